// partial_kernel.cuh -- row f2 (NEXT) of SURVEY §8: settled partial results of online streams;
// included by decoder.cu after frame_kernel.cuh.
//
// P:51 "return intermediate results during online decoding".  The settled prefix of a stream
// after its current layer L is the longest arc sequence shared by the tracebacks of ALL of
// L's survivors, cut after its last emitting arc (reading R15 of DESIGN.md): nothing decoded
// later can change it, because every future path extends one of those survivors.  It ends at
// a token r entered by an emitting arc (or the start token): the deepest layer whose survivor
// paths all pass through one such "root".
//
// One CTA per stream walks back from L: S = the layer's tokens on some survivor path (all of
// layer L at first), closed under epsilon predecessors inside the layer; the roots of S (tokens
// entered by an emitting arc or the start) are found; one root -> done, else S = the roots'
// predecessors in the layer below.  Predecessors are found by state: the wanted source states
// go into a small shared-memory set and the layer's records are scanned against it.  The walk
// stops at the previous settle point at the latest (all paths pass through it), and only the
// arcs settled since then are returned -- the stream's output grows incrementally.
#pragma once
#include "frame_kernel.cuh"

namespace wfst_dev {

struct PartialParams {
  const int4* __restrict__ arcs;
  const int32_t* __restrict__ olabel;
  const int32_t* lanes;     // [n] lanes to report
  const LaneState* lanes_st;
  const int2* rec;          // [lane][R_cap] {arc, state}
  int64_t R_cap;
  const int2* layer_info;   // [lane][TMAX+1]
  int32_t TMAX;
  int2* settled;            // [lane] {layer, record index} of the last settle point (-1: start)
  int32_t cap;              // per-stream output capacity (arcs)
  int32_t* arcs_out;        // [n][cap] newly settled arcs, in order
  int32_t* olab_out;        // [n][cap] their non-zero olabels
  int32_t* n_arcs_out;      // [n]
  int32_t* n_olab_out;      // [n]
  int32_t* layer_out;       // [n] layer (= frames) of the settle point
  int32_t* status_out;      // [n]
  int32_t wcap;             // shared set capacity (slots)
  int32_t fcap;             // shared flag capacity (tokens of one layer)
  int32_t reclaim;          // 1: records and layers below the new settle point are released
  LaneState* lanes_rw;      // (same array as lanes_st; written only to move the floors)
};

__device__ __forceinline__ void pset_put(uint32_t* set, uint32_t cap, uint32_t q) {
  uint32_t b = __umulhi(q * 0x9E3779B1u, cap);
  while (true) {
    const uint32_t old = atomicCAS(set + b, 0xFFFFFFFFu, q);
    if (old == 0xFFFFFFFFu || old == q) return;
    b = (b + 1 == cap) ? 0 : b + 1;
  }
}
__device__ __forceinline__ bool pset_has(const uint32_t* set, uint32_t cap, uint32_t q) {
  uint32_t b = __umulhi(q * 0x9E3779B1u, cap);
  while (true) {
    const uint32_t x = set[b];
    if (x == q) return true;
    if (x == 0xFFFFFFFFu) return false;
    b = (b + 1 == cap) ? 0 : b + 1;
  }
}

template <int BS, int MINB>
__global__ void __launch_bounds__(BS, MINB) partial_kernel(PartialParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* set = (uint32_t*)smem_raw;                       // wanted source states
  unsigned char* flag = (unsigned char*)(set + p.wcap);      // tokens of the current layer in S
  __shared__ int s_changed, s_roots, s_root, s_status, s_len, s_idx, s_arc, s_layer, s_nw, s_nflag;
  // the wanted-state set is sized to what can be wanted (1.5x the tokens flagged), so that
  // clearing it costs O(flagged tokens), not O(capacity), per step
  auto set_cap = [&](int n) { return (uint32_t)min(p.wcap, max(64, n + n / 2 + 1)); };   // load <= 2/3
  const int tid = threadIdx.x;
  const int ln = p.lanes[blockIdx.x];
  const LaneState* Lp = p.lanes_st + ln;
  const int Lcur = __ldcg(&Lp->frames);
  const int2* rec = p.rec + (size_t)ln * p.R_cap;
  const int2* linfo_base = p.layer_info + (size_t)ln * (p.TMAX + 1);
  auto linfo_at = [&](int k) { return linfo_base[k % (p.TMAX + 1)]; };   // layer index ring
  auto R = [&](int64_t i) { return (uint32_t)i % (uint32_t)p.R_cap; };   // record ring (32-bit: R_cap < 2^31)
  const int2 prev = p.settled[ln];
  if (tid == 0) {
    s_status = __ldcg(&Lp->status) != WFST_OK ? __ldcg(&Lp->status)
               : !__ldcg(&Lp->initialized)    ? WFST_ERR_STATE
               : Lcur - __ldcg(&Lp->layer_floor) > p.TMAX ? WFST_ERR_CAPACITY
                                              : WFST_OK;
    s_len = 0;
  }
  __syncthreads();
  auto finish = [&](int n_arcs, int layer) {
    if (tid == 0) {
      p.status_out[blockIdx.x] = s_status;
      p.n_arcs_out[blockIdx.x] = n_arcs;
      p.layer_out[blockIdx.x] = layer;
    }
  };
  if (s_status != WFST_OK) {
    if (tid == 0) p.n_olab_out[blockIdx.x] = 0;
    finish(0, prev.x < 0 ? 0 : prev.x);
    return;
  }
  // ---- walk back from the current layer to the deepest single root
  int k = Lcur;
  int2 Lk = linfo_at(k);
  if (Lk.y > p.fcap) {
    if (tid == 0) {
      s_status = WFST_ERR_CAPACITY;
      p.n_olab_out[blockIdx.x] = 0;
    }
    __syncthreads();
    finish(0, 0);
    return;
  }
  for (int i = tid; i < Lk.y; i += BS) flag[i] = 1;
  if (tid == 0) s_nflag = Lk.y;
  __syncthreads();
  int root = -1;   // record index of the settle point
  while (true) {
    // epsilon predecessors inside layer k (chains are short; repeat until nothing new)
    while (true) {
      const uint32_t wc = set_cap(s_nflag);
      for (uint32_t i = tid; i < wc; i += BS) set[i] = 0xFFFFFFFFu;
      if (tid == 0) {
        s_changed = 0;
        s_nw = 0;
      }
      __syncthreads();
      for (int i = tid; i < Lk.y; i += BS) {
        if (!flag[i]) continue;
        const int a = __ldcg(&rec[R((int64_t)Lk.x + i)].x);
        if (a >= 0 && __ldg(&p.arcs[a].z) < 0) {
          pset_put(set, wc, (uint32_t)(__ldg(&p.arcs[a].w) & 0x7FFFFFFF));
          s_nw = 1;
        }
      }
      __syncthreads();
      if (!s_nw) break;
      for (int i = tid; i < Lk.y; i += BS)
        if (!flag[i] && pset_has(set, wc, (uint32_t)__ldcg(&rec[R((int64_t)Lk.x + i)].y))) {
          flag[i] = 1;
          s_changed = 1;
          atomicAdd(&s_nflag, 1);
        }
      __syncthreads();
      const bool more = s_changed != 0;
      __syncthreads();   // read by every thread before thread 0 clears it for the next pass
      if (!more) break;
    }
    // roots: tokens of S entered by an emitting arc or the start
    if (tid == 0) {
      s_roots = 0;
      s_root = -1;
    }
    __syncthreads();
    for (int i = tid; i < Lk.y; i += BS) {
      if (!flag[i]) continue;
      const int a = __ldcg(&rec[R((int64_t)Lk.x + i)].x);
      if (a < 0 || __ldg(&p.arcs[a].z) >= 0) {
        atomicAdd(&s_roots, 1);
        atomicMax(&s_root, Lk.x + i);   // used only when there is exactly one root
      }
    }
    __syncthreads();
    if (s_roots == 1 || k == 0 || (prev.x >= 0 && k <= prev.x)) {
      root = s_roots == 1 ? s_root : -2;
      break;
    }
    // predecessors of the roots in layer k-1
    const uint32_t wc = set_cap(s_roots);
    for (uint32_t i = tid; i < wc; i += BS) set[i] = 0xFFFFFFFFu;
    if (tid == 0) s_nflag = 0;
    __syncthreads();
    for (int i = tid; i < Lk.y; i += BS) {
      if (!flag[i]) continue;
      const int a = __ldcg(&rec[R((int64_t)Lk.x + i)].x);
      if (a >= 0 && __ldg(&p.arcs[a].z) >= 0)
        pset_put(set, wc, (uint32_t)(__ldg(&p.arcs[a].w) & 0x7FFFFFFF));
    }
    __syncthreads();
    k--;
    Lk = linfo_at(k);
    if (Lk.y > p.fcap) {
      if (tid == 0) s_status = WFST_ERR_CAPACITY;
      break;
    }
    for (int i = tid; i < Lk.y; i += BS) {
      const bool f = pset_has(set, wc, (uint32_t)__ldcg(&rec[R((int64_t)Lk.x + i)].y));
      flag[i] = f;
      if (f) atomicAdd(&s_nflag, 1);
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_status != WFST_OK || root == -2) {   // (-2: the walk met the old settle point unresolved)
    if (tid == 0) {
      if (s_status == WFST_OK) s_status = WFST_ERR_STATE;
      p.n_olab_out[blockIdx.x] = 0;
    }
    __syncthreads();
    finish(0, prev.x < 0 ? 0 : prev.x);
    return;
  }
  // ---- arcs from the old settle point to the new one (traceback walk, layer scans)
  const int stop = prev.x < 0 ? -1 : prev.y;   // record index of the old settle point
  int32_t* out = p.arcs_out + (size_t)blockIdx.x * p.cap;
  if (tid == 0) {
    s_idx = root;
    s_layer = k;
  }
  __syncthreads();
  while (true) {
    const int idx = s_idx;
    if (idx == stop) break;
    const int arc = __ldcg(&rec[R(idx)].x);
    if (arc < 0) break;   // the start token
    __syncthreads();
    if (tid == 0) {
      if (s_len < p.cap) out[s_len] = arc;
      s_len++;
      s_arc = __ldg(&p.arcs[arc].w) & 0x7FFFFFFF;   // source state
      if (__ldg(&p.arcs[arc].z) >= 0) s_layer--;
      s_idx = -1;
    }
    __syncthreads();
    const int2 info = linfo_at(s_layer);
    const int want = s_arc;
    for (int i = tid; i < info.y; i += BS)
      if (__ldcg(&rec[R((int64_t)info.x + i)].y) == want) s_idx = info.x + i;
    __syncthreads();
    if (s_idx < 0) {
      if (tid == 0) s_status = WFST_ERR_STATE;
      break;
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int m = min(s_len, p.cap);
    for (int x = 0; x < m / 2; x++) {
      const int32_t t = out[x];
      out[x] = out[m - 1 - x];
      out[m - 1 - x] = t;
    }
    int nol = 0;
    for (int x = 0; x < m; x++) {
      const int32_t ol = __ldg(p.olabel + out[x]);
      if (ol != 0) p.olab_out[(size_t)blockIdx.x * p.cap + nol++] = ol;
    }
    p.n_olab_out[blockIdx.x] = nol;
    if (s_status == WFST_OK && s_len <= p.cap) {
      p.settled[ln] = make_int2(k, root);
      if (p.reclaim) {   // traceback GC: everything below the settle point is handed out
        p.lanes_rw[ln].rec_floor = linfo_at(k).x;
        p.lanes_rw[ln].layer_floor = k;
      }
    }
    if (s_status == WFST_OK && s_len > p.cap) s_status = WFST_ERR_INVALID_ARG;
  }
  __syncthreads();
  finish(s_len, k);
}

}  // namespace wfst_dev
