// lattice_kernel.cuh -- row f1 (NEXT) of SURVEY §8: per-frame lattice segments and the
// end-of-utterance backward sweep; included by decoder.cu after frame_kernel.cuh.
//
// Segment k of a stream (k = 0: the initial closure, k = t+1: frame t) lists every arc a that
//   * leaves a representative token i (P:139 soft pruning: only representatives have out-arcs) --
//     of layer k-1 if a is emitting, c = (cost_i + w) - L[t][pdf], of layer k if a is an epsilon
//     arc, c = cost_i + w (R1 arithmetic, bit-identical to the frame kernel);
//   * passes frame k's keep() (the cutoff the frame kernel used, R5/R6);
//   * has extra cost s = c - cost_j <= lattice_beam, j the token (representative) of dst(a) in
//     layer k ("computing extra costs", lattice-beam P:146),
// listed in CSR order by j ("listing them in the CSR format"), arc id ascending inside a
// group.  Readings R13-R14 of DESIGN.md.  The segments of one decode call are built by one
// launch after the frame kernel (one work item per (stream, frame)); the frame kernel is not
// touched: it only keeps each survivor's cost beside its record.
#pragma once
#include "frame_kernel.cuh"

namespace wfst_dev {

struct LatParams {
  const int4* __restrict__ state_info;
  const int4* __restrict__ arcs;
  const float* ll;          // the call's log-likelihoods [T][B][P] (mode frames)
  int32_t T, B, P;
  const int32_t* lanes;     // batch index -> lane
  int32_t mode;             // kModeFrames: layers of the call's T frames; kModeInit: layer 0
  int32_t n_items;
  int32_t* q_head;
  float beam, lattice_beam;
  const LaneState* lanes_st;
  const int2* rec;          // [lane][R_cap] {arc, state}
  const float* rec_cost;    // [lane][R_cap]
  const int4* rec_si;       // [lane][R_cap] {e_begin, e_end, eps_end, state}, written by the frame kernel
  int64_t R_cap;
  const int2* layer_info;   // [lane][TMAX+1] {record base, n}
  int32_t TMAX;
  const float* fstats;      // [lane][TMAX][3]
  int4* seg;                // [lane][S_cap] {arc, src token, dst token, slack bits}
  int64_t S_cap;
  unsigned long long* seg_cursor;   // [lane] arena entries used
  int2* seg_index;          // [lane][TMAX+1] {arena offset, n} of segment k
  int32_t* lat_status;      // [lane] sticky lattice status
  u64* g_tab;               // [cta][g_cap] global fallback token map for large layers
  int32_t* g_cnt;           // [cta][FCAP]
  int32_t g_cap, FCAP;
  int4* g_stage;            // [cta][stage_cap] the segment's arcs before placement
  int32_t stage_cap;
  int32_t smem_bytes;       // dynamic shared memory of the launch
};

__device__ __forceinline__ uint32_t lat_bucket(uint32_t q, uint32_t n) { return __umulhi(q * 0x9E3779B1u, n); }

// token map of layer k: state -> token index (states are unique in a layer: insert never matches)
__device__ __forceinline__ void lat_put(u64* tab, uint32_t cap, uint32_t q, uint32_t i) {
  uint32_t b = lat_bucket(q, cap);
  const u64 key = ((u64)q << 32) | i;
  while (atomicCAS(tab + b, kEmpty, key) != kEmpty) b = (b + 1 == cap) ? 0 : b + 1;
}
__device__ __forceinline__ int lat_get(const u64* tab, uint32_t cap, uint32_t q) {
  uint32_t b = lat_bucket(q, cap);
  for (uint32_t n = 0; n < cap; n++) {
    const u64 x = tab[b];
    if (x == kEmpty) return -1;
    if ((uint32_t)(x >> 32) == q) return (int)(uint32_t)x;
    b = (b + 1 == cap) ? 0 : b + 1;
  }
  return -1;
}

template <int BS>
__device__ int block_excl_scan(int x, int* s_tmp /* 33 ints */, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int incl = warp_incl_scan(x);
  if (lane == 31) s_tmp[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int v = lane < BS / 32 ? s_tmp[lane] : 0;
    const int vi = warp_incl_scan(v);
    if (lane < BS / 32) s_tmp[lane] = vi - v;
    if (lane == 31) s_tmp[32] = vi;
  }
  __syncthreads();
  const int r = s_tmp[w] + incl - x;
  total = s_tmp[32];
  __syncthreads();
  return r;
}

constexpr int kLatBig = 64, kLatBigCap = 64;   // tokens with more arcs are expanded CTA-wide
constexpr int kLatU = 4;                        // arcs in flight per thread

#ifndef WFST_LAT_BS
#define WFST_LAT_BS 1024
#endif
#ifndef WFST_LAT_CTAS
#define WFST_LAT_CTAS 1
#endif
constexpr int kLatBS = WFST_LAT_BS, kLatCtas = WFST_LAT_CTAS;   // lattice CTA size, CTAs per SM

template <int BS, int MINB>
__global__ void __launch_bounds__(BS, MINB) lattice_kernel(LatParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_item, s_skip, s_err, s_scan[33], s_nbig, s_nst, s_next, s_big[kLatBigCap];
  __shared__ long long s_base;
  const int tid = threadIdx.x, lane = tid & 31;
  while (true) {
    if (tid == 0) s_item = atomicAdd(p.q_head, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= p.n_items) break;
    const int b = p.mode == kModeInit ? item : item % p.B;
    const int tl = p.mode == kModeInit ? 0 : item / p.B;
    const int ln = p.lanes[b];
    const LaneState* Lp = p.lanes_st + ln;
    const int frames = __ldcg(&Lp->frames);
    const int k = p.mode == kModeInit ? 0 : frames - p.T + 1 + tl;
    if (tid == 0) s_skip = (__ldcg(&Lp->status) != WFST_OK || k < 0 || k > frames || k > p.TMAX ||
                            __ldcg(p.lat_status + ln) != WFST_OK);
    __syncthreads();
    if (s_skip) continue;
    const size_t lo = (size_t)ln * (p.TMAX + 1);
    const int2 Lk = p.layer_info[lo + k];
    const int2 Lp1 = k > 0 ? p.layer_info[lo + k - 1] : make_int2(0, 0);
    const int2* rec = p.rec + (size_t)ln * p.R_cap;
    const float* rco = p.rec_cost + (size_t)ln * p.R_cap;
    float cut_b = __fadd_rn(0.0f, p.beam), cut_a = INFINITY;
    if (k > 0) {
      const float* fs = p.fstats + ((size_t)ln * p.TMAX + (k - 1)) * 3;
      cut_b = fs[1];
      cut_a = fs[2];
    }
    const float* row = k > 0 ? p.ll + ((size_t)tl * p.B + b) * (size_t)p.P : nullptr;
    // the frame's log-likelihood row, the token map and the per-token counts live in shared
    // memory when they fit (else in the CTA's global scratch)
    const int n_k = Lk.y;
    const int row_bytes = (k > 0 && p.P * 4 <= 48 * 1024) ? (p.P * 4 + 15) / 16 * 16 : 0;
    uint32_t cap = (3u * (uint32_t)n_k) / 2u + 32u;
    u64* tab;
    int* cnt;
    const float* cost_k = rco + Lk.x;
    float* s_cost = nullptr;
    if ((size_t)row_bytes + (size_t)cap * 8 + (size_t)n_k * 8 <= (size_t)p.smem_bytes) {
      tab = (u64*)(smem_raw + row_bytes);
      cnt = (int*)(tab + cap);
      s_cost = (float*)(cnt + n_k);
      cost_k = s_cost;
    } else {
      cap = (uint32_t)p.g_cap;
      tab = p.g_tab + (size_t)blockIdx.x * p.g_cap;
      cnt = p.g_cnt + (size_t)blockIdx.x * p.FCAP;
    }
    int4* stg = p.g_stage + (size_t)blockIdx.x * p.stage_cap;
    const float* rowp = row;
    if (row_bytes) {
      float* srow = (float*)smem_raw;
      for (int i = tid; i < p.P; i += BS) srow[i] = __ldg(row + i);
      rowp = srow;
    }
    for (uint32_t i = tid; i < cap; i += BS) tab[i] = kEmpty;
    for (int i = tid; i < n_k; i += BS) cnt[i] = 0;
    if (tid == 0) {
      s_err = WFST_OK;
      s_nbig = 0;
      s_nst = 0;
      s_next = 0;
    }
    __syncthreads();
    for (int i = tid; i < n_k; i += BS) {
      lat_put(tab, cap, (uint32_t)__ldcg(&rec[Lk.x + i].y), (uint32_t)i);
      if (s_cost) s_cost[i] = __ldcg(rco + Lk.x + i);
    }
    __syncthreads();
    // virtual source tokens: u < n_e -> layer k-1 (emitting arcs), else layer k (epsilon arcs)
    const int n_e = k > 0 ? Lp1.y : 0;
    const int n_src = n_e + n_k;
    // one arc: R1 cost, keep(), destination token, extra cost; staged with its group count
    // (warp-collective: every lane calls it, v = the lane has an arc)
    auto proc = [&](bool v, int a, const int4& arc, float co, int u) {   // arc preloaded (MLP)
      bool ok = false;
      int jt = -1;
      float s = 0.f;
      if (v) {
        const bool em = arc.z >= 0;
        const float c = em ? __fadd_rn(__fsub_rn(__fadd_rn(co, __int_as_float(arc.y)), rowp[arc.z]), 0.0f)
                           : __fadd_rn(__fadd_rn(co, __int_as_float(arc.y)), 0.0f);
        if (c < cut_b && c <= cut_a) {
          jt = lat_get(tab, cap, (uint32_t)arc.x);
          if (jt < 0) {   // a kept candidate always has a kept destination
            s_err = WFST_ERR_STATE;
          } else {
            s = __fsub_rn(c, cost_k[jt]);
            ok = s <= p.lattice_beam;
          }
        }
      }
      const int x = warp_append(ok, saddr(&s_nst));
      if (ok) {
        atomicAdd(cnt + jt, 1);
        if (x < p.stage_cap) stg[x] = make_int4(a, u < n_e ? u : u - n_e, jt, __float_as_int(s));
      }
    };
    const int4* rsi = p.rec_si + (size_t)ln * p.R_cap;
    auto src_of = [&](int u, int& e0, int& deg, float& co) {   // contiguous loads, no gathers
      const bool em = u < n_e;
      const int r = em ? Lp1.x + u : Lk.x + (u - n_e);
      co = __ldcg(rco + r);
      const int4 si = __ldcg(rsi + r);
      e0 = em ? si.x : si.y;
      deg = em ? si.y - si.x : si.z - si.y;
    };
    // tokens of small out-degree: groups of 32 handed to warps dynamically, arcs flattened over
    // the warp
    while (true) {
      int u0 = 0;
      if (lane == 0) u0 = atomicAdd(&s_next, 32);
      u0 = __shfl_sync(0xffffffffu, u0, 0);
      if (u0 >= n_src) break;
      const int u = u0 + lane;
      int e0 = 0, deg = 0;
      float co = 0.f;
      if (u < n_src) src_of(u, e0, deg, co);
      if (deg > kLatBig) {   // hub tokens are expanded CTA-wide below (if the list has room)
        const int x = atomicAdd(&s_nbig, 1);
        if (x < kLatBigCap) {
          s_big[x] = u;
          deg = 0;
        }
      }
      const int incl = warp_incl_scan(deg);
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      for (int j0 = 0; j0 < total; j0 += 32 * kLatU) {
        int a[kLatU], own[kLatU];
        float co_o[kLatU];
        int4 arc[kLatU];
#pragma unroll
        for (int x = 0; x < kLatU; x++) {
          const int j = j0 + x * 32 + lane;
          // owner = first lane whose inclusive prefix exceeds j (binary search over the warp)
          int lo_l = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int v = __shfl_sync(0xffffffffu, incl, lo_l + step - 1);
            if (v <= j) lo_l += step;
          }
          own[x] = min(lo_l, 31);
          const int ex_o = __shfl_sync(0xffffffffu, incl - deg, own[x]);
          const int eb_o = __shfl_sync(0xffffffffu, e0, own[x]);
          co_o[x] = __shfl_sync(0xffffffffu, co, own[x]);
          a[x] = eb_o + (j - ex_o);
          arc[x] = j < total ? __ldg(p.arcs + a[x]) : make_int4(0, 0, 0, 0);   // all loads first
        }
#pragma unroll
        for (int x = 0; x < kLatU; x++) proc(j0 + x * 32 + lane < total, a[x], arc[x], co_o[x], u0 + own[x]);
      }
    }
    __syncthreads();
    const int nbig = min(s_nbig, kLatBigCap);
    for (int x = 0; x < nbig; x++) {
      const int u = s_big[x];
      int e0, deg;
      float co;
      src_of(u, e0, deg, co);
      for (int j0 = 0; j0 < deg; j0 += BS * kLatU) {
        int4 arc[kLatU];
#pragma unroll
        for (int y = 0; y < kLatU; y++) {
          const int j = j0 + y * BS + tid;
          arc[y] = j < deg ? __ldg(p.arcs + e0 + j) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int y = 0; y < kLatU; y++) proc(j0 + y * BS + tid < deg, e0 + j0 + y * BS + tid, arc[y], co, u);
      }
    }
    __syncthreads();
    // counts -> CSR offsets; reserve the segment in the stream's arena; scatter the staged arcs
    const int n_st = s_nst;
    int run = 0;
    {   // one block scan: each thread owns a contiguous range of tokens
      const int per = (n_k + BS - 1) / BS, i0 = min(n_k, tid * per), i1 = min(n_k, i0 + per);
      int loc = 0;
      for (int i = i0; i < i1; i++) loc += cnt[i];
      const int ex = block_excl_scan<BS>(loc, s_scan, run);
      int acc = ex;
      for (int i = i0; i < i1; i++) {
        const int c = cnt[i];
        cnt[i] = acc;
        acc += c;
      }
    }
    if (tid == 0) {
      const int err = s_err != WFST_OK ? s_err : n_st > p.stage_cap ? WFST_ERR_CAPACITY : WFST_OK;
      const unsigned long long base = atomicAdd(p.seg_cursor + ln, (unsigned long long)run);
      if (base + run > (unsigned long long)p.S_cap || err != WFST_OK) {
        p.lat_status[ln] = err != WFST_OK ? err : WFST_ERR_CAPACITY;
        s_base = -1;
      } else {
        s_base = (long long)base;
      }
      p.seg_index[lo + k] = make_int2(s_base < 0 ? -1 : (int)s_base, run);
    }
    __syncthreads();
    if (s_base < 0) continue;
    int4* sg = p.seg + (size_t)ln * p.S_cap + s_base;
    for (int i = tid; i < n_st; i += BS) {
      const int4 e = __ldcg(stg + i);
      sg[atomicAdd(cnt + e.z, 1)] = e;
    }
    __syncthreads();
    // group j now spans [cnt[j-1], cnt[j]): order it by arc id (groups are small)
    for (int j = tid; j < n_k; j += BS) {
      const int g0 = j > 0 ? cnt[j - 1] : 0, g1 = cnt[j];
      for (int x = g0 + 1; x < g1; x++) {
        const int4 v = sg[x];
        int y = x - 1;
        while (y >= g0 && sg[y].x > v.x) {
          sg[y + 1] = sg[y];
          y--;
        }
        sg[y + 1] = v;
      }
    }
    __syncthreads();
  }
}

// End of utterance ("used to generate the final lattice at the end of utterance"; R14):
// gamma(j) = slack of the best complete path through token j, swept backwards over the layers
// (emitting arcs of segment k+1 leave layer k; epsilon arcs of segment k to a fixed point), then
// each arc's path slack s_a + gamma(dst(a)).  One CTA per stream.  gamma is kept as orderable u32
// so the per-token minimum is an integer atomic.
struct LatFinParams {
  const int4* __restrict__ state_info;
  const int4* __restrict__ arcs;
  const int32_t* lanes;
  const LaneState* lanes_st;
  const int2* rec;
  const float* rec_cost;
  int64_t R_cap;
  const int2* layer_info;
  int32_t TMAX;
  const int4* seg;
  int64_t S_cap;
  const int2* seg_index;
  uint32_t* gamma;          // [lane][R_cap] orderable
  float* pslack;            // [lane][S_cap]
  float* best_out;          // [n]
  int32_t* reached_out;     // [n]
  int32_t* status_out;      // [n]
  const int32_t* lat_status;
};

template <int BS>
__global__ void __launch_bounds__(BS, 1) lattice_final_kernel(LatFinParams p) {
  __shared__ uint32_t s_fin, s_any;
  __shared__ int s_changed, s_status;
  const int tid = threadIdx.x;
  const int ln = p.lanes[blockIdx.x];
  const LaneState* Lp = p.lanes_st + ln;
  const int T = __ldcg(&Lp->frames);
  if (tid == 0) {
    s_fin = s_any = 0xFFFFFFFFu;
    s_status = __ldcg(&Lp->status) != WFST_OK ? __ldcg(&Lp->status)
               : !__ldcg(&Lp->initialized)    ? WFST_ERR_STATE
               : T > p.TMAX                   ? WFST_ERR_CAPACITY
                                              : p.lat_status[ln];
  }
  __syncthreads();
  if (s_status != WFST_OK) {
    if (tid == 0) {
      p.status_out[blockIdx.x] = s_status;
      p.best_out[blockIdx.x] = INFINITY;
      p.reached_out[blockIdx.x] = 0;
    }
    return;
  }
  const size_t lo = (size_t)ln * (p.TMAX + 1);
  const int2* rec = p.rec + (size_t)ln * p.R_cap;
  const float* rco = p.rec_cost + (size_t)ln * p.R_cap;
  uint32_t* gam = p.gamma + (size_t)ln * p.R_cap;
  const int4* seg = p.seg + (size_t)ln * p.S_cap;
  float* psl = p.pslack + (size_t)ln * p.S_cap;
  const int2 LT = p.layer_info[lo + T];
  // best (R10): min over final survivors of c + F, else min c
  for (int i = tid; i < LT.y; i += BS) {
    const float c = rco[LT.x + i];
    const float F = __int_as_float(__ldg(&p.state_info[rec[LT.x + i].y].w));
    if (F < INFINITY) atomicMin(&s_fin, ord_of(__fadd_rn(c, F)));
    atomicMin(&s_any, ord_of(c));
  }
  const int n_rec = LT.x + LT.y;
  for (int i = tid; i < n_rec; i += BS) gam[i] = 0xFFFFFFFFu;   // ord(+inf) < 0xFFFFFFFF: "unset"
  __syncthreads();
  const bool reached = s_fin != 0xFFFFFFFFu;
  const float best = float_of_ord(reached ? s_fin : s_any);
  for (int i = tid; i < LT.y; i += BS) {
    const float c = rco[LT.x + i];
    const float F = __int_as_float(__ldg(&p.state_info[rec[LT.x + i].y].w));
    const float g = reached ? (F < INFINITY ? __fsub_rn(__fadd_rn(c, F), best) : INFINITY) : __fsub_rn(c, best);
    gam[LT.x + i] = ord_of(g);
  }
  __syncthreads();
  auto gval = [&](int r) {
    const uint32_t o = __ldcg(gam + r);
    return o == 0xFFFFFFFFu ? INFINITY : float_of_ord(o);
  };
  for (int k = T; k >= 0; k--) {
    const int2 Lk = p.layer_info[lo + k];
    if (k < T) {   // emitting arcs of segment k+1: token of layer k -> token of layer k+1
      const int2 Ln = p.layer_info[lo + k + 1];
      const int2 sx = p.seg_index[lo + k + 1];
      for (int m = tid; m < sx.y; m += BS) {
        const int4 e = seg[sx.x + m];
        if (__ldg(&p.arcs[e.x].z) < 0) continue;
        const float v = __fadd_rn(__int_as_float(e.w), gval(Ln.x + e.z));
        if (v < INFINITY) atomicMin(gam + Lk.x + e.y, ord_of(v));
      }
      __syncthreads();
    }
    const int2 sx = p.seg_index[lo + k];
    while (true) {   // epsilon arcs of segment k stay inside layer k
      if (tid == 0) s_changed = 0;
      __syncthreads();
      for (int m = tid; m < sx.y; m += BS) {
        const int4 e = seg[sx.x + m];
        if (__ldg(&p.arcs[e.x].z) >= 0) continue;
        const float v = __fadd_rn(__int_as_float(e.w), gval(Lk.x + e.z));
        if (v < gval(Lk.x + e.y)) {
          atomicMin(gam + Lk.x + e.y, ord_of(v));
          s_changed = 1;
        }
      }
      __syncthreads();
      const bool more = s_changed != 0;
      __syncthreads();   // read by every thread before thread 0 clears it for the next pass
      if (!more) break;
    }
    for (int m = tid; m < sx.y; m += BS) {
      const int4 e = seg[sx.x + m];
      psl[sx.x + m] = __fadd_rn(__int_as_float(e.w), gval(Lk.x + e.z));
    }
    __syncthreads();
  }
  for (int i = tid; i < n_rec; i += BS) {   // hand gamma out as fp32 (+inf: no complete path)
    const float g = gval(i);
    gam[i] = __float_as_uint(g);
  }
  if (tid == 0) {
    p.status_out[blockIdx.x] = WFST_OK;
    p.best_out[blockIdx.x] = best;
    p.reached_out[blockIdx.x] = reached ? 1 : 0;
  }
}

}  // namespace wfst_dev
