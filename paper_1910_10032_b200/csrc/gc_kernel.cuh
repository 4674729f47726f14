// gc_kernel.cuh -- traceback GC by live-set compaction (opts.gc_frames).
// Included by decoder.cu after partial_kernel.cuh.
//
// A traceback record {winning arc, state} is needed only while its token lies on the traceback
// of some current survivor (P:37 traceback; "used to generate the final lattice at the end
// of utterance" -- the one-best output reads the same chains).  Every other record is dead: no
// later frame can reach it.  With max-active binding, a stream writes ~10k records per frame but
// only a narrow tree of them stays live (paths coalesce a few frames back), so an utterance's
// records need not grow with its length.  The paper keeps decoder memory independent of the
// utterance by copying lattice tokens to the host every frame (Eq. 2); this
// build keeps the traceback on the device and drops the dead records instead.
//
// One CTA per stream:
//  (1) mark: walk back from the current layer Lc with the live set (all of Lc's survivors at
//      first), closing it under epsilon predecessors inside each layer and stepping to the
//      emitting predecessors in the layer below -- the same walk as the settled-prefix kernel
//      (partial_kernel.cuh), with bit 31 of a record's state word as the live mark.  The walk
//      stops at the floor, or at a layer the previous collection already compacted where the
//      live set is a single token (everything older is that token's ancestry, compacted then).
//  (2) compact: forward over the walked layers, each layer's live records are moved down to a
//      running cursor (order kept, mark cleared) and the layer index entry rewritten; the lane's
//      record cursor ends at the compacted end.  Records only move down, and a chunk is read in
//      full before it is written, so the move is in place.
// Readers of records (best path, settled prefix) look predecessors up by state within a layer,
// so compacted layers need no pointer fix-up; only the settle point's record index is remapped.
#pragma once
#include "frame_kernel.cuh"

namespace wfst_dev {

struct GcParams {
  const int4* __restrict__ arcs;
  const int32_t* lanes;     // [n] lanes to collect
  LaneState* lanes_st;
  int2* rec;                // [lane][R_cap] {arc, state}
  float* rec_cost;          // [lane][R_cap] survivor costs (debug_costs) or null
  int64_t R_cap;
  int2* layer_info;         // [lane][TMAX+1] {record base, survivors}
  int32_t TMAX;
  int2* settled;            // [lane] {layer, record index} of the last settle point (-1: none)
  int32_t wcap;             // shared set capacity (slots)
};

#ifndef WFST_GC_THREADS
#define WFST_GC_THREADS 1024
#endif
#ifndef WFST_GC_CTAS
#define WFST_GC_CTAS 2
#endif
constexpr int kGcThreads = WFST_GC_THREADS;   // the walk is latency-bound: many records in flight
constexpr int kGcCtas = WFST_GC_CTAS;         // resident CTAs (streams) per SM
constexpr int32_t kLive = (int32_t)0x80000000;

template <int BS>
__device__ __forceinline__ int gc_block_excl_scan(int v, int* s_w, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < BS / 32 ? s_w[lane] : 0;
    const int t0 = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    __syncwarp();
    if (lane < BS / 32) s_w[lane] = t - t0;   // exclusive warp offsets
    if (lane == 31) s_w[32] = t;
  }
  __syncthreads();
  total = s_w[32];
  const int r = s_w[w] + x - v;
  __syncthreads();   // s_w is reused by the next call
  return r;
}

template <int BS>
__global__ void __launch_bounds__(BS, kGcCtas) gc_kernel(GcParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* set = (uint32_t*)smem_raw;   // wanted source states
  __shared__ int s_w[33];
  __shared__ int s_nw, s_nlive, s_nlive_next, s_stop, s_wide, s_np[2], s_found;
  const int tid = threadIdx.x;
  const int ln = p.lanes[blockIdx.x];
  LaneState* Lp = p.lanes_st + ln;
  if (__ldcg(&Lp->status) != WFST_OK || !__ldcg(&Lp->initialized)) return;
  const int Lc = __ldcg(&Lp->frames), F = __ldcg(&Lp->layer_floor), prev_gc = __ldcg(&Lp->gc_layer);
  int2* rec = p.rec + (size_t)ln * p.R_cap;
  float* rc = p.rec_cost ? p.rec_cost + (size_t)ln * p.R_cap : nullptr;
  int2* linfo = p.layer_info + (size_t)ln * (p.TMAX + 1);
  auto LI = [&](int k) -> int2& { return linfo[k % (p.TMAX + 1)]; };
  auto R = [&](int64_t i) { return (uint32_t)i % (uint32_t)p.R_cap; };

  // ---- (1) mark.  Per layer k (its live records already marked): one pass over k's records
  // puts the source state of every live record's arc into E (epsilon arc: same layer) or P
  // (emitting arc: layer k-1); while E holds states whose records are not yet marked, a pass
  // marks them and puts their own arcs' sources; a pass over layer k-1 marks the states in P.
  // Records are read UNR per thread before any is used (the walk is latency-bound).
  constexpr int UNR = 4;
  constexpr uint32_t kE = kGcCtas > 1 ? 2048 : 4096;  // epsilon-source set (few live tokens are entered by epsilon)
  const uint32_t kP = (uint32_t)p.wcap / 2 - kE;       // emitting-source set
  // two (E, P) pairs: the current layer's sources (looked up) and the next layer's (built)
  uint32_t* Ebuf[2] = {set, set + p.wcap / 2};
  uint32_t* Pbuf[2] = {set + kE, set + p.wcap / 2 + kE};
  // visit the records [0, n) of a layer, UNR loads in flight per thread
  // (ring position of record i of a layer: b0 + i, wrapped by one conditional subtraction)
  const uint32_t Rc = (uint32_t)p.R_cap;
  auto RI = [&](uint32_t b0, int i) { const uint32_t x = b0 + (uint32_t)i; return x >= Rc ? x - Rc : x; };
  // done() (evaluated by every thread after each batch; one decision for the CTA) ends the visit
  auto visit_until = [&](int2 L, auto&& f, auto&& done) {
    const uint32_t b0 = R((int64_t)L.x);
    for (int i0 = 0; i0 < L.y; i0 += BS * UNR) {
      int2 r[UNR];
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int i = i0 + u * BS + tid;
        r[u] = i < L.y ? __ldcg(&rec[RI(b0, i)]) : make_int2(-1, 0x7FFFFFFF);
      }
#pragma unroll
      for (int u = 0; u < UNR; u++) {
        const int i = i0 + u * BS + tid;
        if (i < L.y) f(RI(b0, i), r[u]);
      }
      __syncthreads();
      const bool d = done();
      if (__syncthreads_or(d)) break;
    }
  };
  auto visit = [&](int2 L, auto&& f) { visit_until(L, f, [] { return false; }); };
  // bounded insert: a full set flags the walk as too wide to track (s_wide)
  auto put = [&](uint32_t* st, uint32_t cap, uint32_t q) {   // true: q is new
    uint32_t b = __umulhi(q * 0x9E3779B1u, cap);
    for (uint32_t n = 0; n < cap; n++) {
      const uint32_t old = atomicCAS(st + b, 0xFFFFFFFFu, q);
      if (old == 0xFFFFFFFFu) return true;
      if (old == q) return false;
      b = (b + 1 == cap) ? 0 : b + 1;
    }
    s_wide = 1;
    return false;
  };
  // bounded lookup (a set filled by a failed put must not loop)
  auto has = [&](const uint32_t* st, uint32_t cap, uint32_t q) {
    uint32_t b = __umulhi(q * 0x9E3779B1u, cap);
    for (uint32_t n = 0; n < cap; n++) {
      const uint32_t x = st[b];
      if (x == q) return true;
      if (x == 0xFFFFFFFFu) return false;
      b = (b + 1 == cap) ? 0 : b + 1;
    }
    return false;
  };
  // a live record (arc a) sends its source state to E (epsilon arc: same layer) or P (layer below)
  // (s_np[w]: distinct states in P of pair w -- the pass over the layer below stops once it has
  // found them all: a layer holds one token per state, and live tokens sit in its cheap front)
  auto put_src = [&](int a, uint32_t* e, uint32_t* pp, int w) {
    if (a < 0) return;
    const int4 arc = __ldg(&p.arcs[a]);
    const uint32_t src = (uint32_t)(arc.w & 0x7FFFFFFF);
    if (arc.z < 0) {
      put(e, kE, src);
      s_nw = 1;
    } else if (put(pp, kP, src)) {
      atomicAdd(&s_np[w], 1);
    }
  };
  auto clear = [&](int w) {
    for (uint32_t i = tid; i < (uint32_t)p.wcap / 2; i += BS) Ebuf[w][i] = 0xFFFFFFFFu;   // E and P of pair w
  };
  // (1) mark.  Layer Lc is all live; its records' sources seed pair 0.  Walking down, the pass
  // over layer k-1 marks the records whose state is in the current P and at once puts the newly
  // live records' own sources into the other pair; epsilon sources found in layer k-1 (E) are
  // marked by further passes over k-1 until none is new.  One pass per layer in the common case.
  int2 Lk = LI(Lc);
  clear(0);
  if (tid == 0) {
    s_nlive = Lk.y;
    s_stop = F;
    s_wide = 0;
    s_nw = 0;
    s_np[0] = s_np[1] = 0;
  }
  __syncthreads();
  visit(Lk, [&](uint32_t x, int2 r) {
    rec[x].y = r.y | kLive;
    put_src(r.x, Ebuf[0], Pbuf[0], 0);
  });
  __syncthreads();
  int cur = 0;
  for (int k = Lc; k >= F; k--) {
    Lk = LI(k);
    // stop: the floor, a walk too wide to track, or an already-compacted layer whose live set
    // is one token (everything older is that token's ancestry, compacted before)
    if (k == F || s_wide || (k <= prev_gc && s_nlive == 1)) {
      if (tid == 0) s_stop = s_wide ? F : k;
      break;
    }
    const int2 Lb = LI(k - 1);
    const int nx = cur ^ 1;
    clear(nx);
    const int np = s_np[cur];   // (complete: the pass that filled P ended with a barrier)
    if (tid == 0) {
      s_nlive_next = 0;
      s_nw = 0;
      s_found = 0;
      s_np[nx] = 0;
    }
    __syncthreads();
    visit_until(Lb, [&](uint32_t x, int2 r) {
      if (has(Pbuf[cur], kP, (uint32_t)(r.y & 0x7FFFFFFF))) {
        rec[x].y = r.y | kLive;
        atomicAdd(&s_nlive_next, 1);
        atomicAdd(&s_found, 1);
        put_src(r.x, Ebuf[nx], Pbuf[nx], nx);
      }
    }, [&] { return !s_wide && s_found >= np; });
    __syncthreads();
    // epsilon predecessors inside layer k-1, to a fixed point
    while (s_nw && !s_wide) {
      __syncthreads();
      if (tid == 0) s_nw = 0;
      __syncthreads();
      visit(Lb, [&](uint32_t x, int2 r) {
        if (r.y >= 0 && has(Ebuf[nx], kE, (uint32_t)r.y)) {
          rec[x].y = r.y | kLive;
          atomicAdd(&s_nlive_next, 1);
          put_src(r.x, Ebuf[nx], Pbuf[nx], nx);
        }
      });
      __syncthreads();
    }
    if (tid == 0) s_nlive = s_nlive_next;
    cur = nx;
    __syncthreads();
  }
  __syncthreads();
  if (s_wide) {   // too wide to track: every record from the floor up stays (conservative, exact)
    for (int k = F; k <= Lc; k++) {
      const int2 Lq = LI(k);
      for (int i = tid; i < Lq.y; i += BS) rec[R((int64_t)Lq.x + i)].y |= kLive;
    }
    __syncthreads();
  }
  // ---- (2) compact layers s_stop..Lc in place
  const int k0 = s_stop;
  int64_t cursor = LI(k0).x;
  const int2 st = p.settled[ln];
  for (int k = k0; k <= Lc; k++) {
    const int2 Lq = LI(k);
    const int64_t nb = cursor;
    const uint32_t qb = R((int64_t)Lq.x);
    for (int i0 = 0; i0 < Lq.y; i0 += BS) {
      const int i = i0 + tid;
      int2 r = make_int2(0, 0);
      float c = 0.0f;
      if (i < Lq.y) {
        r = __ldcg(&rec[RI(qb, i)]);
        if (rc) c = __ldcg(&rc[RI(qb, i)]);
      }
      const bool live = i < Lq.y && r.y < 0;
      int total;
      const int rank = gc_block_excl_scan<BS>(live ? 1 : 0, s_w, total);   // barriers: reads done
      if (live) {
        const int64_t d = cursor + rank;
        rec[R(d)] = make_int2(r.x, r.y & 0x7FFFFFFF);
        if (rc) rc[R(d)] = c;
        if (st.x == k && st.y == Lq.x + i) p.settled[ln].y = (int)d;
      }
      cursor += total;
      __syncthreads();
    }
    if (tid == 0) LI(k) = make_int2((int)nb, (int)(cursor - nb));
  }
  __syncthreads();
  if (tid == 0) {
    const int32_t used = (int32_t)cursor;
    Lp->rec_used = used;
    Lp->rec_phys = (int32_t)R(used);
    Lp->layer_base = LI(Lc).x;
    Lp->gc_layer = Lc;
  }
}

}  // namespace wfst_dev
