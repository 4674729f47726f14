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
// Two launches per call, one CTA per stream each:
// * partial_root_kernel walks back from L: S = the layer's tokens on some survivor path (all of
//   layer L at first), closed under epsilon predecessors inside the layer; the roots of S (tokens
//   entered by an emitting arc or the start) are found; one root -> done, else S = the roots'
//   predecessors in the layer below.  Predecessors are found by state: the wanted source states
//   go into a small shared-memory set and the layer's records are scanned against it.  The walk
//   stops at the previous settle point at the latest (all paths pass through it).
// * partial_trace_kernel returns only the arcs settled since the previous call (the stream's
//   output grows incrementally): from the new root back to the old settle point, one record per
//   step, each found by a scan of its layer for the arc's source state (a layer holds one token
//   per state).  It needs no shared tables, so it runs as small CTAs, many per SM: the walk is a
//   chain of dependent memory round trips, and resident CTAs are what hide them.
// Every pass over a layer's records issues U loads per thread before using any of them.
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
  int32_t* arcs_out;        // [n][cap] scratch rows (the walk's arcs when they do not fit on chip)
  int32_t* packed_arcs;     // newly settled arcs, in order, stream after stream at root_out[b]
  int32_t* packed_olab;     // their non-zero olabels, at the same offsets
  int32_t* packed_count;    // arcs packed so far (zeroed before the launch)
  int32_t* n_arcs_out;      // [n]
  int32_t* n_olab_out;      // [n]
  int32_t* layer_out;       // [n] layer (= frames) of the settle point (root kernel: the root's layer)
  int32_t* status_out;      // [n]
  int32_t* root_out;        // [n] root kernel -> trace kernel: record index of the new settle point;
                            //     trace kernel -> host: the stream's offset in the packed outputs
  int32_t wcap;             // shared set capacity (slots)
  int32_t fcap;             // shared flag capacity (tokens of one layer)
  int32_t reclaim;          // 1: records and layers below the new settle point are released
  LaneState* lanes_rw;      // (same array as lanes_st; written only to move the floors)
};

__device__ __forceinline__ bool pset_put(uint32_t* set, uint32_t cap, uint32_t q) {   // true: q is new
  uint32_t b = __umulhi(q * 0x9E3779B1u, cap);
  while (true) {
    const uint32_t old = atomicCAS(set + b, 0xFFFFFFFFu, q);
    if (old == 0xFFFFFFFFu) return true;
    if (old == q) return false;
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

constexpr int kPU = 8;   // record loads in flight per thread in the layer passes

// one walk-back pass over the n records of a layer starting at logical index x0: f(i, rec, arc)
// for every i with want(i), with the record's arc (arc id >= 0) loaded too; kPU record loads are
// issued before any is used, then the arc loads
template <int BS, typename Want, typename Fn>
__device__ __forceinline__ void layer_pass_arcs(const int4* __restrict__ arcs, const int2* rec, uint32_t R_cap,
                                                int64_t x0, int n, Want want, Fn f) {
  const uint32_t b0 = (uint32_t)(x0 % R_cap);   // the layer's first record in the ring
  for (int i0 = 0; i0 < n; i0 += BS * kPU) {
    int2 r[kPU];
    int4 a[kPU];
#pragma unroll
    for (int u = 0; u < kPU; u++) {
      const int i = i0 + u * BS + (int)threadIdx.x;
      const uint32_t x = b0 + (uint32_t)i;
      r[u] = i < n && want(i) ? __ldcg(rec + (x >= R_cap ? x - R_cap : x)) : make_int2(-3, -1);
    }
#pragma unroll
    for (int u = 0; u < kPU; u++) a[u] = r[u].x >= 0 ? __ldg(arcs + r[u].x) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < kPU; u++)
      if (r[u].x != -3) f(i0 + u * BS + (int)threadIdx.x, r[u], a[u]);
  }
}

// f(i, rec) over the records of a layer in batches of BS * kPU (cheapest first), until done()
// holds after a batch (one decision for the whole CTA); ends with a barrier, so done()'s inputs
// can be reset right after
template <int BS, typename Fn, typename Done>
__device__ __forceinline__ void layer_scan_until(const int2* rec, uint32_t R_cap, int64_t x0, int n, Fn f, Done done) {
  const uint32_t b0 = (uint32_t)(x0 % R_cap);
  for (int i0 = 0; i0 < n; i0 += BS * kPU) {
    int2 r[kPU];
#pragma unroll
    for (int u = 0; u < kPU; u++) {
      const int i = i0 + u * BS + (int)threadIdx.x;
      const uint32_t x = b0 + (uint32_t)i;
      r[u] = i < n ? __ldcg(rec + (x >= R_cap ? x - R_cap : x)) : make_int2(-3, -1);
    }
#pragma unroll
    for (int u = 0; u < kPU; u++)
      if (r[u].x != -3) f(i0 + u * BS + (int)threadIdx.x, r[u]);
    __syncthreads();   // the batch's updates are visible ...
    const bool d = done();
    if (__syncthreads_or(d)) break;   // ... and read by every thread before the next batch changes them
  }
  __syncthreads();
}

constexpr uint32_t kPredTag = 0x80000000u;   // set entries: state (epsilon source) | state + tag (emitting source)

template <int BS, int MINB>
__global__ void __launch_bounds__(BS, MINB) partial_root_kernel(PartialParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* set = (uint32_t*)smem_raw;                       // wanted source states
  unsigned char* flag = (unsigned char*)(set + p.wcap);      // tokens of the current layer in S:
                                                             // 2 unclassified, 1 classified
  __shared__ int s_roots, s_root, s_status, s_nwe, s_nwp, s_found, s_hi;
  // the wanted-state set of a layer holds at most one entry per token of S, so it is sized to
  // the layer (load <= 2/3) and clearing it costs O(layer), not O(capacity)
  auto set_cap = [&](int n) { return (uint32_t)min(p.wcap, max(64, n + n / 2 + 1)); };
  const int tid = threadIdx.x;
  const int ln = p.lanes[blockIdx.x];
  const LaneState* Lp = p.lanes_st + ln;
  const int Lcur = __ldcg(&Lp->frames);
  const int2* rec = p.rec + (size_t)ln * p.R_cap;
  const uint32_t Rc = (uint32_t)p.R_cap;   // record ring (32-bit: R_cap < 2^31)
  const int2* linfo_base = p.layer_info + (size_t)ln * (p.TMAX + 1);
  auto linfo_at = [&](int k) { return linfo_base[k % (p.TMAX + 1)]; };   // layer index ring
  const int2 prev = p.settled[ln];
  if (tid == 0)
    s_status = __ldcg(&Lp->status) != WFST_OK ? __ldcg(&Lp->status)
               : !__ldcg(&Lp->initialized)    ? WFST_ERR_STATE
               : Lcur - __ldcg(&Lp->layer_floor) > p.TMAX ? WFST_ERR_CAPACITY
                                              : WFST_OK;
  __syncthreads();
  auto finish = [&](int status, int root, int layer) {
    if (tid == 0) {
      p.status_out[blockIdx.x] = status;
      p.root_out[blockIdx.x] = root;
      p.layer_out[blockIdx.x] = layer;
    }
  };
  if (s_status != WFST_OK) {
    finish(s_status, -1, prev.x < 0 ? 0 : prev.x);
    return;
  }
  // ---- walk back from the current layer to the deepest single root
  int k = Lcur;
  int2 Lk = linfo_at(k);
  if (Lk.y > p.fcap) {
    finish(WFST_ERR_CAPACITY, -1, prev.x < 0 ? 0 : prev.x);
    return;
  }
  uint32_t wc = set_cap(Lk.y);
  for (int i = tid; i < Lk.y; i += BS) flag[i] = 2;
  for (uint32_t i = tid; i < wc; i += BS) set[i] = 0xFFFFFFFFu;
  if (tid == 0) {
    s_hi = Lk.y;
    s_roots = 0;
    s_root = -1;
    s_nwe = s_nwp = 0;
  }
  __syncthreads();
  int root = -1;   // record index of the settle point
  // Every token of S is classified once, by the arc that entered it: an epsilon arc puts its
  // source (a token of the same layer) into the set, an emitting arc makes it a root and puts
  // its source (a token of the layer below) into the set with kPredTag, the start token is a
  // root.  Epsilon sources join S and are classified in turn.  Tokens on survivor paths are
  // cheap and a layer is stored cheapest bins first, so past the first layer S sits near the
  // front: passes over S stop at s_hi (one past its last index), and a search for a known number
  // of wanted states stops once all are found.
  while (true) {
    while (true) {
      const int hi = s_hi;
      if (tid == 0) s_found = 0;   // (last read before the barrier that ended the previous search)
      bool adde = false;
      layer_pass_arcs<BS>(p.arcs, rec, Rc, Lk.x, hi, [&](int i) { return flag[i] == 2; }, [&](int i, int2 r, int4 a) {
        flag[i] = 1;
        if (r.x < 0 || a.z >= 0) {
          atomicAdd(&s_roots, 1);
          atomicMax(&s_root, Lk.x + i);   // used only when there is exactly one root
          if (r.x >= 0 && pset_put(set, wc, (uint32_t)(a.w & 0x7FFFFFFF) | kPredTag)) atomicAdd(&s_nwp, 1);
        } else if (pset_put(set, wc, (uint32_t)(a.w & 0x7FFFFFFF))) {
          atomicAdd(&s_nwe, 1);
          adde = true;
        }
      });
      if (!__syncthreads_or(adde)) break;   // no new epsilon source wanted
      const int nwe = s_nwe;
      bool newf = false;
      // every wanted epsilon source is a token of this layer: stop when all are seen
      layer_scan_until<BS>(rec, Rc, Lk.x, Lk.y, [&](int i, int2 r) {
        if (pset_has(set, wc, (uint32_t)r.y)) {
          atomicAdd(&s_found, 1);
          if (!flag[i]) {
            flag[i] = 2;
            atomicMax(&s_hi, i + 1);
            newf = true;
          }
        }
      }, [&]() { return s_found >= nwe; });
      if (!__syncthreads_or(newf)) break;
    }
    const int n_roots = s_roots;
    if (n_roots == 1 || k == 0 || (prev.x >= 0 && k <= prev.x)) {
      root = n_roots == 1 ? s_root : -2;
      break;
    }
    // S = the tokens of layer k-1 whose states the roots came from
    const int nwp = s_nwp;
    k--;
    Lk = linfo_at(k);
    if (Lk.y > p.fcap) {
      if (tid == 0) s_status = WFST_ERR_CAPACITY;
      break;
    }
    __syncthreads();   // s_roots, s_root, s_nwp read
    for (int i = tid; i < Lk.y; i += BS) flag[i] = 0;
    if (tid == 0) {
      s_hi = 0;
      s_found = 0;
      s_roots = 0;
      s_root = -1;
      s_nwe = s_nwp = 0;
    }
    __syncthreads();
    layer_scan_until<BS>(rec, Rc, Lk.x, Lk.y, [&](int i, int2 r) {
      if (pset_has(set, wc, (uint32_t)r.y | kPredTag)) {
        flag[i] = 2;
        atomicAdd(&s_found, 1);
        atomicMax(&s_hi, i + 1);
      }
    }, [&]() { return s_found >= nwp; });
    wc = set_cap(Lk.y);
    for (uint32_t i = tid; i < wc; i += BS) set[i] = 0xFFFFFFFFu;
    __syncthreads();
  }
  __syncthreads();
  if (s_status != WFST_OK || root == -2)   // (-2: the walk met the old settle point unresolved)
    finish(s_status != WFST_OK ? s_status : WFST_ERR_STATE, -1, prev.x < 0 ? 0 : prev.x);
  else
    finish(WFST_OK, root, k);
}

// block-wide exclusive prefix sum of 0/1 flags (all threads call it); returns the total
template <int BS>
__device__ __forceinline__ int block_excl_scan01(bool f, int& excl, int* s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, f);
  if (lane == 0) s_w[w] = __popc(m);
  __syncthreads();
  int base = 0, tot = 0;
#pragma unroll
  for (int j = 0; j < BS / 32; j++) {
    const int c = s_w[j];
    base += j < w ? c : 0;
    tot += c;
  }
  excl = base + __popc(m & ((1u << lane) - 1u));
  __syncthreads();
  return tot;
}

constexpr int kTraceSmem = 2048;   // settled arcs kept on chip per call (longer: serial fallback)

template <int BS, int MINB>
__global__ void __launch_bounds__(BS, MINB) partial_trace_kernel(PartialParams p) {
  __shared__ int s_idx[3], s_arc[3], s_src[3], s_emit[3];
  __shared__ int s_path[kTraceSmem];
  __shared__ int s_w[BS / 32];
  __shared__ int s_off;
  const int tid = threadIdx.x;
  const int ln = p.lanes[blockIdx.x];
  const int2* rec = p.rec + (size_t)ln * p.R_cap;
  const uint32_t Rc = (uint32_t)p.R_cap;
  const int2* linfo_base = p.layer_info + (size_t)ln * (p.TMAX + 1);
  const int2 prev = p.settled[ln];
  const int root = p.root_out[blockIdx.x];
  int status = p.status_out[blockIdx.x];
  const int k = p.layer_out[blockIdx.x];
  int32_t* out = p.arcs_out + (size_t)blockIdx.x * p.cap;
  if (status != WFST_OK) {   // the root kernel wrote the status and the old settle layer
    if (tid == 0) {
      p.n_arcs_out[blockIdx.x] = 0;
      p.n_olab_out[blockIdx.x] = 0;
      p.root_out[blockIdx.x] = 0;
    }
    return;
  }
  // ---- arcs from the new settle point back to the old one.  Step j reads slot j%3 (the record
  // found by step j-1: index, arc, the arc's source state and kind), its scan fills slot
  // (j+1)%3, and thread 0 clears slot (j+2)%3, last read in step j-1: one barrier per step.
  const int stop = prev.x < 0 ? -1 : prev.y;   // record index of the old settle point
  auto load_step = [&](int slot, int idx, int2 r) {   // (one thread: the record's finder)
    s_idx[slot] = idx;
    s_arc[slot] = r.x;
    if (r.x >= 0) {
      const int4 a = __ldg(&p.arcs[r.x]);
      s_src[slot] = a.w & 0x7FFFFFFF;
      s_emit[slot] = a.z >= 0;
    }
  };
  if (tid == 0) {
    load_step(0, root, __ldcg(rec + (uint32_t)root % Rc));
    s_idx[1] = -1;
  }
  __syncthreads();
  int len = 0, layer = k, j = 0;
  while (true) {
    const int cur = j % 3, nxt = (j + 1) % 3;
    const int idx = s_idx[cur], arc = s_arc[cur];
    if (idx < 0) {   // the previous scan found no record of the source state
      status = WFST_ERR_STATE;
      break;
    }
    if (idx == stop || arc < 0) break;   // the old settle point / the start token
    if (tid == 0) {
      if (len < p.cap) out[len] = arc;
      if (len < kTraceSmem) s_path[len] = arc;
      s_idx[(j + 2) % 3] = -1;
    }
    len++;
    layer -= s_emit[cur];
    const int want = s_src[cur];
    const int2 info = linfo_base[layer % (p.TMAX + 1)];
    // the path's tokens are cheap and a layer is stored cheapest bins first: the scan usually
    // ends in its first batch (the barrier after each batch is the step's barrier)
    int i0 = 0;
    const uint32_t b0 = (uint32_t)info.x % Rc;   // (R_cap < 2^31; no modulo per record)
    do {
      int2 r[kPU];
#pragma unroll
      for (int u = 0; u < kPU; u++) {
        const int i = i0 + u * BS + tid;
        const uint32_t x = b0 + (uint32_t)i;
        r[u] = i < info.y ? __ldcg(rec + (x >= Rc ? x - Rc : x)) : make_int2(-3, -1);
      }
      bool found = false;
#pragma unroll
      for (int u = 0; u < kPU; u++)
        if (r[u].y == want && r[u].x != -3) {
          load_step(nxt, info.x + i0 + u * BS + tid, r[u]);
          found = true;
        }
      if (__syncthreads_or(found)) break;   // one decision for the CTA (the finder's writes are visible)
      i0 += BS * kPU;
    } while (i0 < info.y);
    j++;
  }
  __syncthreads();
  // ---- reverse into path order, gather the non-zero olabels (in parallel when on chip), and
  // pack both at this stream's offset: the host copies back exactly the arcs that settled
  const int m = min(len, p.cap);
  if (tid == 0) s_off = m > 0 ? atomicAdd(p.packed_count, m) : 0;
  __syncthreads();
  const int off = s_off;
  int32_t* pa = p.packed_arcs + off;
  int32_t* po = p.packed_olab + off;
  int nol = 0;
  if (m <= kTraceSmem) {
    for (int x0 = 0; x0 < m; x0 += BS) {
      const int x = x0 + tid;
      const int32_t arc = x < m ? s_path[m - 1 - x] : 0;
      const int32_t ol = x < m ? __ldg(p.olabel + arc) : 0;
      if (x < m) pa[x] = arc;
      int e = 0;
      const int tot = block_excl_scan01<BS>(ol != 0, e, s_w);
      if (ol != 0) po[nol + e] = ol;
      nol += tot;
    }
  } else if (tid == 0) {   // serial fallback (more than kTraceSmem arcs settled in one call)
    for (int x = 0; x < m; x++) {
      const int32_t arc = out[m - 1 - x];
      pa[x] = arc;
      const int32_t ol = __ldg(p.olabel + arc);
      if (ol != 0) po[nol++] = ol;
    }
  }
  if (tid == 0) {
    p.n_olab_out[blockIdx.x] = nol;
    p.root_out[blockIdx.x] = off;
    if (status == WFST_OK && len <= p.cap) {
      p.settled[ln] = make_int2(k, root);
      if (p.reclaim) {   // traceback GC: everything below the settle point is handed out
        p.lanes_rw[ln].rec_floor = linfo_base[k % (p.TMAX + 1)].x;
        p.lanes_rw[ln].layer_floor = k;
      }
    }
    if (status == WFST_OK && len > p.cap) status = WFST_ERR_INVALID_ARG;
    p.status_out[blockIdx.x] = status;
    p.n_arcs_out[blockIdx.x] = len;
  }
}

}  // namespace wfst_dev
