// decoder.cu -- the frame kernel (rows a1-a7 of SURVEY §8) and the decoder C ABI.
//
// One persistent CTA per SM owns one lane (stream) at a time and runs whole frames with only
// CTA barriers: load-balanced emitting expansion, running best + beam and exact
// max-active, epsilon closure to a fixed point under the fixed cutoff (P:49,
// P:132), contraction of one representative per state with traceback records.
// Lanes are re-queued every `frames_per_item` frames so all SMs stay busy to the end.
// DESIGN.md §5 describes the data layout and why it looks like this on sm_100a.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "wfst_internal.h"

using namespace wfst;
typedef unsigned long long u64;

namespace {

constexpr u64 kEmpty = 0xFFFFFFFFFFFFFFFFull;
constexpr int kNB = 1024;          // cost bins for the max-active bound
constexpr int kMaxProbeS = 24;     // buckets probed in the on-chip table before overflowing
constexpr int kMaxProbeG = 256;    // buckets probed in the global overflow table
constexpr int32_t kEpsFlag = (int32_t)0x80000000;
constexpr int kModeFrames = 0, kModeInit = 1;

struct LaneState {
  int32_t status;       // wfst_status, sticky
  int32_t initialized;
  int32_t n_front;      // survivors in the current frontier
  int32_t cur;          // frontier buffer holding them
  int32_t frames;       // frames decoded in this utterance
  int32_t layer_base;   // record index of the current layer's first survivor
  int32_t rec_used;
  float front_best;     // min cost of the current survivors
  u64 emit_arcs, eps_arcs, eps_relax, cand, surv, ovf, alpha_frames, frames_total;
};

struct KParams {
  const int4* __restrict__ state_info;
  const int4* __restrict__ arcs;
  int32_t start;
  const float* ll;
  int32_t T, B, P;
  const int32_t* lanes;   // batch index -> lane id
  int32_t mode, K, n_items;
  int32_t* q_head;
  int32_t* lane_round;
  float beam;
  int32_t alpha;
  int32_t C, NBK, C_ovf, FCAP;
  int64_t R_cap;
  int32_t TMAX;
  LaneState* lanes_st;
  int4* front;        // [lane][2][FCAP]  {state, cost bits, e_begin, n_emit}
  int2* claim;        // [lane][FCAP]     {slot, state}
  int32_t* prevg;     // [lane][FCAP]     back-pointer of the slot's winner
  int32_t* slotrec;   // [lane][FCAP]     slot -> survivor index
  int2* fslot;        // [lane][FCAP]     survivor index -> {slot, arc}
  u64* ovf;           // [lane][C_ovf]    global overflow token table
  int2* wl;           // [lane][2][FCAP]  epsilon worklists {slot, state}
  int2* rec;          // [lane][R_cap]    traceback records {arc, prev}
  float* rec_cost;    // [lane][R_cap]    (debug) survivor cost
  float* fstats;      // [lane][TMAX][3]
  long long* fcounts; // [lane][TMAX][5]
  int2* layer_info;   // [lane][TMAX+1]   {record base, survivors}
};

struct SmemCtl {
  int32_t item, lane, b, status;
  uint32_t best_ord;
  int32_t theta;
  int32_t n_claim, n_claim_emit, n_ovf, n_surv, n_in, n_wl, n_wl_next;
  float beam_cut, kalpha, ref, inv_w, min_surv;
  int32_t use_alpha;
  int32_t radix_prefix, radix_k;
  long long emit_arcs, eps_deg, eps_relax;
  int32_t warp_tmp[32];
  long long warp_tmp64[32];
  LaneState L;
};

// ---------------- small helpers ----------------
__device__ __forceinline__ uint32_t ord_of(float c) {
  uint32_t b = __float_as_uint(c);
  return b ^ ((b & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float float_of_ord(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o ^ 0x80000000u) : ~o;
  return __uint_as_float(b);
}
__device__ __forceinline__ uint32_t bucket_of(uint32_t q, uint32_t nb) { return __umulhi(q * 0x9E3779B1u, nb); }
__device__ __forceinline__ uint32_t tag_of(uint32_t q) { return ((q * 0x85EBCA77u) >> 28) << 28; }
__device__ __forceinline__ u64 make_key(float c, uint32_t q, uint32_t arc) {
  return ((u64)ord_of(c) << 32) | (u64)(tag_of(q) | (arc & kArcMask));
}
__device__ __forceinline__ float key_cost(u64 k) { return float_of_ord((uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t key_arc(u64 k) { return (uint32_t)k & kArcMask; }

__device__ __forceinline__ u64 ld_volatile(const u64* p) { return *(const volatile u64*)p; }

// monotone cost -> bin map used both to count and to reject
__device__ __forceinline__ int bin_of(float c, float ref, float inv_w) {
  float x = __fmul_rn(__fsub_rn(c, ref), inv_w);
  x = fminf(fmaxf(x, 0.0f), (float)(kNB - 1));
  return (int)x;
}

// Open-addressing insert of (state q, key) into a table of nb buckets of 4 slots.  The slot's
// state is identified by a 4-bit tag in the key plus the destination of the stored arc.
// Returns slot index or -1 when the probe limit is hit.  claimed: the slot was empty;
// improved: the key is now the slot minimum (claim or atomicMin success).
template <int MAXPROBE>
__device__ __forceinline__ int tab_insert(u64* tab, uint32_t nb, uint32_t q, u64 key, const int4* arcs,
                                          int32_t start, bool& claimed, bool& improved) {
  uint32_t b = bucket_of(q, nb);
  const uint32_t tg = (uint32_t)key & 0xF0000000u;
  claimed = improved = false;
  for (int p = 0; p < MAXPROBE; ++p) {
    u64* bk = tab + (size_t)b * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u64 v = ld_volatile(bk + j);
      if (v == kEmpty) {
        u64 old = atomicCAS(bk + j, kEmpty, key);
        if (old == kEmpty) {
          claimed = improved = true;
          return (int)(b * 4 + j);
        }
        v = old;
      }
      if (((uint32_t)v & 0xF0000000u) == tg) {
        uint32_t a = (uint32_t)v & kArcMask;
        int32_t s = (a == kArcNone) ? start : __ldg(&arcs[a].x);
        if (s == (int32_t)q) {
          u64 old = atomicMin(bk + j, key);
          improved = key < old;
          return (int)(b * 4 + j);
        }
      }
    }
    b = (b + 1 == nb) ? 0 : b + 1;
  }
  return -1;
}

template <int BS>
__device__ __forceinline__ int block_excl_scan(int v, int* s_tmp, int& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = (lane < BS / 32) ? s_tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < BS / 32) s_tmp[lane] = s;
  }
  __syncthreads();
  int prefix = (w > 0) ? s_tmp[w - 1] : 0;
  total = s_tmp[BS / 32 - 1];
  __syncthreads();
  return prefix + x - v;
}

template <int BS>
__device__ __forceinline__ long long block_sum64(long long v, long long* s_tmp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_tmp[w] = v;
  __syncthreads();
  long long t = 0;
  for (int i = 0; i < BS / 32; i++) t += s_tmp[i];
  __syncthreads();
  return t;
}

// ---------------- the frame kernel ----------------
template <int BS, int R>
struct Frame {
  const KParams& p;
  SmemCtl& S;
  u64* tab;
  int* hist;
  int* s_off;
  int* s_eb;
  float* s_cost;
  int* s_aux;   // per-token slot (epsilon) or unused
  // lane buffers
  int4* F[2];
  int2* claim;
  int32_t* prevg;
  int32_t* slotrec;
  int2* fslot;
  u64* ovf;
  int2* wl[2];
  int2* rec;
  float* rec_cost;

  __device__ Frame(const KParams& p_, SmemCtl& S_, u64* tab_, int* hist_, int* s_off_, int* s_eb_, float* s_cost_,
                   int* s_aux_)
      : p(p_), S(S_), tab(tab_), hist(hist_), s_off(s_off_), s_eb(s_eb_), s_cost(s_cost_), s_aux(s_aux_) {}

  __device__ void bind(int lane) {
    size_t L = (size_t)lane, FC = (size_t)p.FCAP;
    F[0] = p.front + L * 2 * FC;
    F[1] = F[0] + FC;
    claim = p.claim + L * FC;
    prevg = p.prevg + L * FC;
    slotrec = p.slotrec + L * FC;
    fslot = p.fslot + L * FC;
    ovf = p.ovf + L * (size_t)p.C_ovf;
    wl[0] = p.wl + L * 2 * FC;
    wl[1] = wl[0] + FC;
    rec = p.rec + L * (size_t)p.R_cap;
    rec_cost = p.rec_cost ? p.rec_cost + L * (size_t)p.R_cap : nullptr;
  }

  __device__ __forceinline__ u64 read_slot(int slot) const {
    return slot < p.C ? ld_volatile(tab + slot) : ld_volatile(ovf + (slot - p.C));
  }

  __device__ __forceinline__ bool keep(float c) const {
    return c < S.beam_cut && (!S.use_alpha || c <= S.kalpha);
  }

  // insert into on-chip table, then the global overflow table; -1 = capacity failure
  __device__ __forceinline__ int insert(uint32_t q, u64 key, bool& claimed, bool& improved) {
    int s = tab_insert<kMaxProbeS>(tab, (uint32_t)p.NBK, q, key, p.arcs, p.start, claimed, improved);
    if (s >= 0) return s;
    s = tab_insert<kMaxProbeG>(ovf, (uint32_t)(p.C_ovf / 4), q, key, p.arcs, p.start, claimed, improved);
    if (s < 0) {
      S.status = WFST_ERR_CAPACITY;
      return -1;
    }
    if (claimed) atomicAdd(&S.n_ovf, 1);
    return s + p.C;
  }

  // claim entry = {slot, state | has_eps << 31}
  __device__ __forceinline__ void add_claim(int slot, uint32_t q, uint32_t eps_flag) {
    int idx = atomicAdd(&S.n_claim, 1);
    if (idx < p.FCAP) claim[idx] = make_int2(slot, (int)(q | (eps_flag << 31)));
    else S.status = WFST_ERR_CAPACITY;
  }

  // winner protocol: after a barrier, the thread whose key is still the slot value writes prev
  __device__ __forceinline__ void write_winner(int slot, u64 key, int32_t prev) {
    if (read_slot(slot) == key) prevg[slot] = prev;
  }

  // tighten theta (warp 0): smallest b such that >= alpha distinct states have first-insert bin < b
  __device__ void update_theta() {
    const int lane = threadIdx.x & 31;
    int base = lane * (kNB / 32);
    int s = 0;
    for (int i = 0; i < kNB / 32; i++) s += *(volatile int*)&hist[base + i];
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    unsigned m = __ballot_sync(0xffffffffu, incl >= p.alpha);
    if (m == 0) return;
    int L = __ffs(m) - 1;
    if (lane == L) {
      int c = incl - s;
      for (int i = 0; i < kNB / 32; i++) {
        c += *(volatile int*)&hist[base + i];
        if (c >= p.alpha) {
          atomicMin(&S.theta, base + i + 1);
          break;
        }
      }
    }
  }

  // ---- row a1 + a2: load-balanced emitting expansion ----
  __device__ void expand(const float* row, int t) {
    const int tid = threadIdx.x;
    const int n_f = S.L.n_front;
    const int4* Fin = F[S.L.cur];
    const int32_t layer_base = S.L.layer_base;
    const float beam = p.beam;
    long long arcs_total = 0;
    for (int cb = 0; cb < n_f; cb += BS) {
      int i = cb + tid, deg = 0, eb = 0;
      float cost = 0.f;
      if (i < n_f) {
        int4 f = __ldcg(Fin + i);
        eb = f.z;
        deg = f.w;
        cost = __int_as_float(f.y);
      }
      int A;
      int off = block_excl_scan<BS>(deg, S.warp_tmp, A);
      s_off[tid] = off;
      s_eb[tid] = eb;
      s_cost[tid] = cost;
      if (tid == 0) s_off[BS] = A;
      __syncthreads();
      arcs_total += A;
      for (int base = 0; base < A; base += BS * R) {
        int wslot[R];
        u64 wkey[R];
        int32_t wprev[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
          wslot[r] = -1;
          int j = base + r * BS + tid;
          if (j >= A) continue;
          // token owning flattened arc j: last k with s_off[k] <= j
          int lo = 0, hi = BS;
          while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (s_off[mid] <= j) lo = mid; else hi = mid;
          }
          const int k = lo;
          const int a = s_eb[k] + (j - s_off[k]);
          const int4 arc = __ldg(p.arcs + a);
          const float L = __ldg(row + arc.z);
          float c = __fsub_rn(__fadd_rn(s_cost[k], __int_as_float(arc.y)), L);
          c = __fadd_rn(c, 0.0f);
          const uint32_t bo = *(volatile uint32_t*)&S.best_ord;
          if (bo != 0xFFFFFFFFu && !(c < __fadd_rn(float_of_ord(bo), beam))) continue;
          const int bin = bin_of(c, S.ref, S.inv_w);
          if (bin >= *(volatile int*)&S.theta) continue;
          const uint32_t o = ord_of(c);
          if (o < bo) atomicMin(&S.best_ord, o);
          const uint32_t q = (uint32_t)arc.x;
          const u64 key = ((u64)o << 32) | (u64)(tag_of(q) | (uint32_t)a);
          bool claimed, improved;
          int slot = insert(q, key, claimed, improved);
          if (slot < 0) continue;
          if (claimed) {
            atomicAdd(&hist[bin], 1);
            add_claim(slot, q, (uint32_t)arc.w >> 31);
          }
          if (improved) {
            wslot[r] = slot;
            wkey[r] = key;
            wprev[r] = layer_base + cb + k;
          }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; r++)
          if (wslot[r] >= 0) write_winner(wslot[r], wkey[r], wprev[r]);
        if (p.alpha > 0 && tid < 32) {
          const int nc = __shfl_sync(0xffffffffu, *(volatile int*)&S.n_claim, 0);
          if (nc >= p.alpha) update_theta();
        }
      }
      __syncthreads();
    }
    if (tid == 0) S.emit_arcs = arcs_total;
  }

  // ---- row a3: beam + exact max-active (readings R5, R6) ----
  __device__ void select_cutoff() {
    const int tid = threadIdx.x;
    const float beam_cut = S.beam_cut;
    const int n_claim = min(S.n_claim, p.FCAP);
    if (p.alpha <= 0 || n_claim <= p.alpha) {   // max-active cannot bind: n_in <= n_claim
      if (tid == 0) {
        S.n_in = -1;
        S.use_alpha = 0;
        S.kalpha = INFINITY;
      }
      __syncthreads();
      return;
    }
    long long cnt = 0;
    for (int i = tid; i < n_claim; i += BS) {
      float c = key_cost(read_slot(claim[i].x));
      if (c < beam_cut) cnt++;
    }
    long long n_in = block_sum64<BS>(cnt, S.warp_tmp64);
    if (tid == 0) {
      S.n_in = (int)n_in;
      S.use_alpha = 0;
      S.kalpha = INFINITY;
    }
    __syncthreads();
    if (p.alpha <= 0 || n_in <= p.alpha) return;
    // exact alpha-th smallest among in-beam costs: 4 radix passes of 8 bits on ord(cost)
    if (tid == 0) {
      S.radix_prefix = 0;
      S.radix_k = p.alpha;
    }
    __syncthreads();
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = tid; i < 256; i += BS) hist[i] = 0;
      __syncthreads();
      const uint32_t prefix = (uint32_t)S.radix_prefix;
      const uint32_t hmask = (shift == 24) ? 0u : (0xFFFFFFFFu << (shift + 8));
      for (int i = tid; i < n_claim; i += BS) {
        float c = key_cost(read_slot(claim[i].x));
        if (!(c < beam_cut)) continue;
        uint32_t o = ord_of(c);
        if ((o & hmask) == (prefix & hmask)) atomicAdd(&hist[(o >> shift) & 255], 1);
      }
      __syncthreads();
      if (tid == 0) {
        int k = S.radix_k, d = 0;
        for (; d < 256; d++) {
          if (hist[d] >= k) break;
          k -= hist[d];
        }
        S.radix_k = k;
        S.radix_prefix = (int)(prefix | ((uint32_t)d << shift));
      }
      __syncthreads();
    }
    if (tid == 0) {
      S.kalpha = float_of_ord((uint32_t)S.radix_prefix);
      S.use_alpha = 1;
    }
    for (int i = tid; i < kNB; i += BS) hist[i] = 0;
    __syncthreads();
  }

  // ---- row a5: epsilon closure under the fixed cutoff (reading R7) ----
  __device__ void eps_closure() {
    const int tid = threadIdx.x;
    if (tid == 0) S.n_wl = 0;
    __syncthreads();
    {
      const int n_claim = min(S.n_claim, p.FCAP);
      for (int i = tid; i < n_claim; i += BS) {
        int2 cl = claim[i];
        if (cl.y >= 0) continue;                  // state has no epsilon arcs
        float c = key_cost(read_slot(cl.x));
        if (!keep(c)) continue;
        int idx = atomicAdd(&S.n_wl, 1);
        wl[0][idx] = make_int2(cl.x, cl.y & 0x7FFFFFFF);
      }
    }
    __syncthreads();
    int cur = 0;
    long long relax = 0;
    while (true) {
      const int n_wl = S.n_wl;
      if (n_wl == 0) break;
      if (tid == 0) S.n_wl_next = 0;
      __syncthreads();
      const int2* W = wl[cur];
      int2* Wn = wl[cur ^ 1];
      for (int cb = 0; cb < n_wl; cb += BS) {
        int i = cb + tid, deg = 0, eb = 0, slot = 0;
        float cost = 0.f;
        if (i < n_wl) {
          int2 e = W[i];
          slot = e.x;
          int4 si = __ldg(p.state_info + e.y);
          eb = si.y;
          deg = si.z - si.y;
          cost = key_cost(read_slot(slot));
        }
        int A;
        int off = block_excl_scan<BS>(deg, S.warp_tmp, A);
        s_off[tid] = off;
        s_eb[tid] = eb;
        s_cost[tid] = cost;
        s_aux[tid] = slot;
        if (tid == 0) s_off[BS] = A;
        __syncthreads();
        for (int base = 0; base < A; base += BS) {
          int wslot = -1;
          u64 wkey = 0;
          int32_t wprev = 0;
          int j = base + tid;
          if (j < A) {
            int lo = 0, hi = BS;
            while (hi - lo > 1) {
              int mid = (lo + hi) >> 1;
              if (s_off[mid] <= j) lo = mid; else hi = mid;
            }
            const int k = lo;
            const int e = s_eb[k] + (j - s_off[k]);
            const int4 arc = __ldg(p.arcs + e);
            float c = __fadd_rn(__fadd_rn(s_cost[k], __int_as_float(arc.y)), 0.0f);
            relax++;
            if (keep(c)) {
              const uint32_t q = (uint32_t)arc.x;
              const u64 key = make_key(c, q, (uint32_t)e);
              bool claimed, improved;
              int sl = insert(q, key, claimed, improved);
              if (sl >= 0) {
                const uint32_t has_eps = (uint32_t)arc.w >> 31;
                if (claimed) add_claim(sl, q, has_eps);
                if (improved) {
                  wslot = sl;
                  wkey = key;
                  wprev = kEpsFlag | s_aux[k];
                  if (has_eps) {
                    int idx = atomicAdd(&S.n_wl_next, 1);
                    if (idx < p.FCAP) Wn[idx] = make_int2(sl, (int)q);
                    else S.status = WFST_ERR_CAPACITY;
                  }
                }
              }
            }
          }
          __syncthreads();
          if (wslot >= 0) write_winner(wslot, wkey, wprev);
        }
        __syncthreads();
      }
      if (tid == 0) S.n_wl = min(S.n_wl_next, p.FCAP);
      cur ^= 1;
      __syncthreads();
    }
    long long tot = block_sum64<BS>(relax, S.warp_tmp64);
    if (tid == 0) S.eps_relax = tot;
  }

  // ---- rows a4 + a6: contraction into the next frontier + traceback records ----
  __device__ void contract() {
    const int tid = threadIdx.x;
    const int n_claim = min(S.n_claim, p.FCAP);
    int4* Fout = F[S.L.cur ^ 1];
    if (tid == 0) {
      S.n_surv = 0;
      S.min_surv = INFINITY;
    }
    __syncthreads();
    long long epsd = 0;
    float mn = INFINITY;
    for (int i = tid; i < n_claim; i += BS) {
      int2 cl = claim[i];
      cl.y &= 0x7FFFFFFF;
      u64 v = read_slot(cl.x);
      if (cl.x < p.C) tab[cl.x] = kEmpty; else ovf[cl.x - p.C] = kEmpty;
      float c = key_cost(v);
      if (!keep(c)) continue;
      int r = atomicAdd(&S.n_surv, 1);
      if (r >= p.FCAP) {
        S.status = WFST_ERR_CAPACITY;
        continue;
      }
      int4 si = __ldg(p.state_info + cl.y);
      Fout[r] = make_int4(cl.y, __float_as_int(c), si.x, si.y - si.x);
      fslot[r] = make_int2(cl.x, (int)key_arc(v));
      slotrec[cl.x] = r;
      epsd += si.z - si.y;
      mn = fminf(mn, c);
    }
    // block min of survivors' cost
    for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if ((tid & 31) == 0) S.warp_tmp[tid >> 5] = __float_as_int(mn);
    long long eps_deg = block_sum64<BS>(epsd, S.warp_tmp64);
    if (tid == 0) {
      float m = INFINITY;
      for (int w = 0; w < BS / 32; w++) m = fminf(m, __int_as_float(S.warp_tmp[w]));
      S.min_surv = m;
      S.eps_deg = eps_deg;
    }
    __syncthreads();
    const int n_surv = min(S.n_surv, p.FCAP);
    const int32_t rb = S.L.rec_used;
    if ((long long)rb + n_surv > p.R_cap) {
      if (tid == 0) S.status = WFST_ERR_CAPACITY;
      __syncthreads();
      return;
    }
    for (int r = tid; r < n_surv; r += BS) {
      int2 fs = fslot[r];
      int32_t pv = prevg[fs.x];
      if (pv < 0 && pv != -1) pv = rb + slotrec[pv & 0x7FFFFFFF];
      int32_t arc = (uint32_t)fs.y == kArcNone ? -1 : fs.y;
      rec[rb + r] = make_int2(arc, pv);
      if (rec_cost) rec_cost[rb + r] = __int_as_float(Fout[r].y);
    }
    __syncthreads();
  }

  __device__ void begin_frame(float beam_cut_fixed) {
    const int tid = threadIdx.x;
    for (int i = tid; i < kNB; i += BS) hist[i] = 0;
    if (tid == 0) {
      S.best_ord = 0xFFFFFFFFu;
      S.theta = kNB;
      S.n_claim = 0;
      S.n_ovf = 0;
      S.use_alpha = 0;
      S.kalpha = INFINITY;
      S.beam_cut = beam_cut_fixed;
      S.emit_arcs = 0;
      S.eps_relax = 0;
      float half = isinf(p.beam) ? 32.0f : 0.5f * p.beam;
      S.ref = S.L.front_best - half;
      S.inv_w = (float)kNB / (4.0f * half);
    }
    __syncthreads();
  }

  // on a sticky error the claim list may be incomplete: wipe both tables
  __device__ void clear_all() {
    for (int i = threadIdx.x; i < p.C; i += BS) tab[i] = kEmpty;
    for (int i = threadIdx.x; i < p.C_ovf; i += BS) ovf[i] = kEmpty;
    __syncthreads();
  }

  __device__ void finish_frame(int t, bool emitting) {
    const int tid = threadIdx.x;
    if (S.status != WFST_OK) clear_all();
    if (tid == 0) {
      LaneState& L = S.L;
      const int n_surv = min(S.n_surv, p.FCAP);
      if (S.status != WFST_OK) L.status = S.status;
      if (L.status == WFST_OK) {
        L.layer_base = L.rec_used;
        L.rec_used += n_surv;
        L.n_front = n_surv;
        L.cur ^= 1;
        L.front_best = S.min_surv;
        int layer = emitting ? L.frames + 1 : 0;
        if (emitting) L.frames++;
        L.eps_arcs += S.eps_deg;
        L.eps_relax += S.eps_relax;
        L.cand += S.n_claim;
        L.surv += n_surv;
        L.ovf += S.n_ovf;
        if (emitting) {
          L.emit_arcs += S.emit_arcs;
          L.alpha_frames += S.use_alpha;
          L.frames_total++;
        }
        size_t lane = (size_t)S.lane;
        if (layer <= p.TMAX) p.layer_info[lane * (p.TMAX + 1) + layer] = make_int2(L.layer_base, n_surv);
        if (emitting && t >= 0 && L.frames - 1 < p.TMAX) {
          size_t fi = lane * p.TMAX + (L.frames - 1);
          p.fstats[fi * 3 + 0] = float_of_ord(S.best_ord);
          p.fstats[fi * 3 + 1] = S.beam_cut;
          p.fstats[fi * 3 + 2] = S.use_alpha ? S.kalpha : INFINITY;
          p.fcounts[fi * 5 + 0] = S.n_claim_emit;
          p.fcounts[fi * 5 + 1] = S.n_in;
          p.fcounts[fi * 5 + 2] = n_surv;
          p.fcounts[fi * 5 + 3] = S.emit_arcs;
          p.fcounts[fi * 5 + 4] = S.eps_deg;
        }
      }
      S.status = WFST_OK;
    }
    __syncthreads();
  }

  // R3: start token + epsilon closure with keep(c) = c < beam
  __device__ void init_lane() {
    const int tid = threadIdx.x;
    if (tid == 0) {
      LaneState& L = S.L;
      // a new utterance: keep the lifetime counters, clear the decode state
      L.n_front = 0;
      L.cur = 0;
      L.frames = 0;
      L.layer_base = 0;
      L.rec_used = 0;
      L.status = WFST_OK;
      L.initialized = 1;
      L.front_best = 0.0f;
    }
    __syncthreads();
    begin_frame(__fadd_rn(0.0f, p.beam));
    if (tid == 0) {
      bool claimed, improved;
      u64 key = make_key(0.0f, (uint32_t)p.start, kArcNone);
      int slot = insert((uint32_t)p.start, key, claimed, improved);
      if (slot >= 0) {
        int4 si = __ldg(p.state_info + p.start);
        add_claim(slot, (uint32_t)p.start, si.z > si.y ? 1u : 0u);
        prevg[slot] = -1;
      }
      S.best_ord = ord_of(0.0f);
      S.n_claim_emit = 1;
      S.n_in = 1;
    }
    __syncthreads();
    eps_closure();
    contract();
    finish_frame(-1, false);
  }

  __device__ void run_frame(int t) {
    const int tid = threadIdx.x;
    const float* row = p.ll + ((size_t)t * p.B + S.b) * (size_t)p.P;
    begin_frame(INFINITY);
    expand(row, t);
    __syncthreads();
    if (tid == 0) {
      S.n_claim_emit = S.n_claim;
      if (S.best_ord == 0xFFFFFFFFu) S.status = WFST_ERR_NO_SURVIVOR;
      else S.beam_cut = __fadd_rn(float_of_ord(S.best_ord), p.beam);
    }
    __syncthreads();
    if (S.status != WFST_OK) {
      // leave the table clean for the next lane
      const int n_claim = min(S.n_claim, p.FCAP);
      for (int i = threadIdx.x; i < n_claim; i += BS) {
        int s = claim[i].x;
        if (s < p.C) tab[s] = kEmpty; else ovf[s - p.C] = kEmpty;
      }
      if (tid == 0) S.n_surv = 0;
      __syncthreads();
      finish_frame(t, true);
      return;
    }
    select_cutoff();
    eps_closure();
    contract();
    finish_frame(t, true);
  }
};

template <int BS, int R>
__global__ void __launch_bounds__(BS, 1) frame_kernel(KParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SmemCtl S;
  u64* tab = (u64*)smem_raw;
  int* hist = (int*)(tab + p.C);
  int* s_off = hist + kNB;
  int* s_eb = s_off + BS + 1;
  float* s_cost = (float*)(s_eb + BS);
  int* s_aux = (int*)(s_cost + BS);
  const int tid = threadIdx.x;
  for (int i = tid; i < p.C; i += BS) tab[i] = kEmpty;
  if (tid == 0) S.status = WFST_OK;
  __syncthreads();
  Frame<BS, R> fr(p, S, tab, hist, s_off, s_eb, s_cost, s_aux);
  while (true) {
    if (tid == 0) S.item = atomicAdd(p.q_head, 1);
    __syncthreads();
    const int item = S.item;
    if (item >= p.n_items) break;
    const int b = item % p.B, r = item / p.B;
    const int lane = p.lanes[b];
    if (tid == 0) {
      volatile int32_t* lr = p.lane_round + b;
      while (*lr != r) __nanosleep(64);
      __threadfence();
      S.lane = lane;
      S.b = b;
      const int* src = (const int*)&p.lanes_st[lane];
      int* dst = (int*)&S.L;
      for (int k = 0; k < (int)(sizeof(LaneState) / 4); k++) dst[k] = __ldcg(src + k);
    }
    __syncthreads();
    fr.bind(lane);
    if (p.mode == kModeInit) {
      fr.init_lane();
    } else {
      const int t_end = min(p.T, (r + 1) * p.K);
      for (int t = r * p.K; t < t_end; t++) {
        if (S.L.status != WFST_OK) break;
        fr.run_frame(t);
      }
    }
    __syncthreads();
    if (tid == 0) {
      p.lanes_st[lane] = S.L;
      __threadfence();
      *(volatile int32_t*)(p.lane_round + b) = r + 1;
    }
    __syncthreads();
  }
}

// ---------------- best path (row a7; readings R10, R11) ----------------
// One CTA per lane: argmin over the last layer's survivors of (c + F, arc) among final states,
// else of (c, arc); then the traceback walk over {arc, prev} records.
__global__ void best_path_kernel(KParams p, const int32_t* __restrict__ lanes, int32_t n, int32_t cap,
                                 float* cost_out, int32_t* reached_out, int32_t* n_arcs_out, int32_t* arcs_out,
                                 int32_t* olab_out, int32_t* n_olab_out, int32_t* status_out) {
  __shared__ u64 s_fin[32], s_any[32];
  __shared__ int s_idx;
  const int li = blockIdx.x;
  const int lane = lanes[li];
  const int tid = threadIdx.x;
  LaneState L;
  {
    const int* src = (const int*)&p.lanes_st[lane];
    int* dst = (int*)&L;
    for (int k = 0; k < (int)(sizeof(LaneState) / 4); k++) dst[k] = __ldcg(src + k);
  }
  if (L.status != WFST_OK || !L.initialized) {
    if (tid == 0) {
      status_out[li] = L.initialized ? L.status : WFST_ERR_STATE;
      n_arcs_out[li] = 0;
      n_olab_out[li] = 0;
      cost_out[li] = INFINITY;
      reached_out[li] = 0;
    }
    return;
  }
  const int4* Fc = p.front + (size_t)lane * 2 * p.FCAP + (size_t)L.cur * p.FCAP;
  const int2* rec = p.rec + (size_t)lane * p.R_cap;
  u64 kf = kEmpty, ka = kEmpty;
  for (int i = tid; i < L.n_front; i += blockDim.x) {
    int4 f = __ldcg(Fc + i);
    float c = __int_as_float(f.y);
    u64 arc = (uint32_t)__ldcg(&rec[L.layer_base + i].x);  // -1 -> 0xFFFFFFFF sorts last (R9)
    float F = __int_as_float(__ldg(&p.state_info[f.x].w));
    if (F < INFINITY) kf = min(kf, ((u64)ord_of(__fadd_rn(c, F)) << 32) | arc);
    ka = min(ka, ((u64)ord_of(c) << 32) | arc);
  }
  for (int o = 16; o > 0; o >>= 1) {
    kf = min(kf, __shfl_xor_sync(0xffffffffu, kf, o));
    ka = min(ka, __shfl_xor_sync(0xffffffffu, ka, o));
  }
  if ((tid & 31) == 0) {
    s_fin[tid >> 5] = kf;
    s_any[tid >> 5] = ka;
  }
  if (tid == 0) s_idx = -1;
  __syncthreads();
  kf = kEmpty;
  ka = kEmpty;
  for (int w = 0; w < (int)(blockDim.x / 32); w++) {
    kf = min(kf, s_fin[w]);
    ka = min(ka, s_any[w]);
  }
  const bool reached = kf != kEmpty;
  const u64 kb = reached ? kf : ka;
  // the arc identifies the survivor uniquely within a layer
  for (int i = tid; i < L.n_front && kb != kEmpty; i += blockDim.x)
    if ((uint32_t)__ldcg(&rec[L.layer_base + i].x) == (uint32_t)kb) s_idx = i;
  __syncthreads();
  if (tid != 0) return;
  const int best_i = s_idx;
  if (kb == kEmpty || best_i < 0) {
    status_out[li] = WFST_ERR_NO_SURVIVOR;
    n_arcs_out[li] = 0;
    n_olab_out[li] = 0;
    cost_out[li] = INFINITY;
    reached_out[li] = 0;
    return;
  }
  cost_out[li] = float_of_ord((uint32_t)(kb >> 32));
  reached_out[li] = reached ? 1 : 0;
  int len = 0;
  int32_t r = L.layer_base + best_i;
  long long guard = (long long)L.rec_used + 2;
  while (r >= 0 && --guard > 0) {
    int2 e = __ldcg(rec + r);
    if (e.x < 0) break;
    len++;
    r = e.y;
  }
  n_arcs_out[li] = len;
  if (guard <= 0) {
    n_olab_out[li] = 0;
    status_out[li] = WFST_ERR_CAPACITY;
    return;
  }
  // second walk writes arcs back to front; olabels are counted from the arc list
  r = L.layer_base + best_i;
  for (int pos = len - 1; pos >= 0; pos--) {
    int2 e = __ldcg(rec + r);
    if (pos < cap) arcs_out[(size_t)li * cap + pos] = e.x;
    r = e.y;
  }
  int nol = 0;
  for (int k = 0; k < len && k < cap; k++) {
    int32_t ol = __ldg(&p.arcs[arcs_out[(size_t)li * cap + k]].w) & 0x7FFFFFFF;
    if (ol != 0) {
      if (nol < cap) olab_out[(size_t)li * cap + nol] = ol;
      nol++;
    }
  }
  n_olab_out[li] = nol;
  status_out[li] = (len > cap) ? WFST_ERR_INVALID_ARG : WFST_OK;
}

}  // namespace

// ---------------- host side ----------------
struct wfst_decoder_s {
  wfst_graph_t g = nullptr;
  int device = 0;
  int32_t n_lanes = 0;
  float beam = 15.f;
  int32_t alpha = 0;
  wfst_decoder_opts_t o{};
  int32_t C = 0, C_ovf = 0, FCAP = 0, TMAX = 0;
  int64_t R_cap = 0;
  int n_sm = 0, threads = 512;
  size_t smem_bytes = 0;
  KParams kp{};
  // device allocations
  LaneState* d_lanes = nullptr;
  void* d_pool = nullptr;
  size_t pool_bytes = 0;
  int32_t* d_qhead = nullptr;
  int32_t* d_round = nullptr;
  int32_t* d_lane_ids = nullptr;   // batch -> lane (n_lanes capacity)
  int32_t* d_path = nullptr;       // best-path scratch
  size_t path_cap = 0;
  float* d_host_stage[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[2] = {nullptr, nullptr}, ev_use[2] = {nullptr, nullptr};
  std::vector<int32_t> h_initialized;
  std::vector<int32_t> cur_ids;    // mapping currently in d_lane_ids
  int64_t device_bytes = 0;
};

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    cudaSetDevice(d);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

template <int BS>
void* kernel_ptr() {
  return (void*)frame_kernel<BS, 2>;
}

cudaError_t launch_frames(wfst_decoder_t d, KParams kp, cudaStream_t st) {
  int grid = std::min(kp.n_items, d->o.max_ctas > 0 ? d->o.max_ctas : d->n_sm);
  if (grid <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(kp.q_head, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(kp.lane_round, 0, sizeof(int32_t) * kp.B, st);
  if (e != cudaSuccess) return e;
  switch (d->threads) {
    case 256: frame_kernel<256, 2><<<grid, 256, d->smem_bytes, st>>>(kp); break;
    case 1024: frame_kernel<1024, 2><<<grid, 1024, d->smem_bytes, st>>>(kp); break;
    default: frame_kernel<512, 2><<<grid, 512, d->smem_bytes, st>>>(kp); break;
  }
  return cudaGetLastError();
}

size_t smem_for(int C, int threads) {
  return (size_t)C * 8 + (size_t)kNB * 4 + (size_t)(threads + 1) * 4 + (size_t)threads * 12 + 16;
}

}  // namespace

extern "C" {

wfst_status wfst_decoder_create(wfst_graph_t g, int32_t n_streams, float beam, int32_t max_active,
                                wfst_decoder_t* out) {
  return wfst_decoder_create_ex(g, n_streams, beam, max_active, nullptr, out);
}

wfst_status wfst_decoder_create_ex(wfst_graph_t g, int32_t n_streams, float beam, int32_t max_active,
                                   const wfst_decoder_opts_t* opts, wfst_decoder_t* out) {
  if (!g || !out) return fail(WFST_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (n_streams <= 0) return fail(WFST_ERR_INVALID_ARG, "n_streams must be > 0");
  if (!(beam > 0.0f)) return fail(WFST_ERR_INVALID_ARG, "beam must be > 0 (may be +inf)");
  DeviceGuard dg(g->device);
  auto* d = new wfst_decoder_s();
  d->g = g;
  d->device = g->device;
  d->n_lanes = n_streams;
  d->beam = beam;
  d->alpha = max_active > 0 ? max_active : 0;
  if (opts) d->o = *opts;
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, g->device);
  if (e != cudaSuccess) {
    delete d;
    return cuda_fail(e, "cudaGetDeviceProperties");
  }
  d->n_sm = prop.multiProcessorCount;
  d->threads = d->o.threads == 256 || d->o.threads == 1024 ? d->o.threads : 512;
  int C = d->o.table_slots > 0 ? d->o.table_slots : 24576;
  C = std::max(64, (C + 3) / 4 * 4);
  size_t max_smem = prop.sharedMemPerBlockOptin;
  while (C > 64 && smem_for(C, d->threads) + sizeof(SmemCtl) + 1024 > max_smem) C -= 1024;
  d->C = C;
  int Co = d->o.overflow_slots > 0 ? d->o.overflow_slots : C;
  d->C_ovf = std::max(64, (Co + 3) / 4 * 4);
  d->FCAP = d->C + d->C_ovf;
  d->TMAX = d->o.max_frames > 0 ? d->o.max_frames : 2048;
  int64_t per_frame = d->alpha > 0 ? std::min<int64_t>((int64_t)d->alpha * 5 / 4 + 1024, d->FCAP) : d->FCAP;
  if (d->o.records_per_stream > 0) {
    d->R_cap = d->o.records_per_stream;
  } else {
    // default: ~max_frames/4 frames at the alpha bound, capped to half of the free device memory
    d->R_cap = (int64_t)(d->TMAX / 4 + 1) * per_frame;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      int64_t per_lane_other = (int64_t)d->FCAP * (32 + 8 + 4 + 4 + 8 + 32) + (int64_t)d->C_ovf * 8 +
                               (int64_t)d->TMAX * 60;
      int64_t budget = (int64_t)(free_b / 2) / n_streams - per_lane_other;
      int64_t cap = budget / (int64_t)(sizeof(int2) + (d->o.debug_costs ? 4 : 0));
      if (cap < d->R_cap) d->R_cap = std::max<int64_t>(cap, per_frame);
    }
  }
  if (d->R_cap > INT32_MAX - 1) d->R_cap = INT32_MAX - 1;
  if (d->o.frames_per_item <= 0) d->o.frames_per_item = 16;
  d->smem_bytes = smem_for(d->C, d->threads);
  void* kfn = d->threads == 256 ? kernel_ptr<256>() : d->threads == 1024 ? kernel_ptr<1024>() : kernel_ptr<512>();
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d->smem_bytes);
  if (e != cudaSuccess) {
    delete d;
    return cuda_fail(e, "cudaFuncSetAttribute");
  }
  // one pool for all per-lane buffers
  const size_t L = (size_t)n_streams, FC = (size_t)d->FCAP;
  struct Part { size_t off, bytes; };
  std::vector<Part> parts;
  size_t total = 0;
  auto add = [&](size_t bytes) {
    total = (total + 255) / 256 * 256;
    parts.push_back({total, bytes});
    total += bytes;
    return parts.size() - 1;
  };
  size_t i_front = add(L * 2 * FC * sizeof(int4));
  size_t i_claim = add(L * FC * sizeof(int2));
  size_t i_prevg = add(L * FC * 4);
  size_t i_slotrec = add(L * FC * 4);
  size_t i_fslot = add(L * FC * sizeof(int2));
  size_t i_ovf = add(L * (size_t)d->C_ovf * 8);
  size_t i_wl = add(L * 2 * FC * sizeof(int2));
  size_t i_rec = add(L * (size_t)d->R_cap * sizeof(int2));
  size_t i_rcost = d->o.debug_costs ? add(L * (size_t)d->R_cap * 4) : (size_t)-1;
  size_t i_fst = add(L * (size_t)d->TMAX * 3 * 4);
  size_t i_fcn = add(L * (size_t)d->TMAX * 5 * 8);
  size_t i_linfo = add(L * (size_t)(d->TMAX + 1) * sizeof(int2));
  e = cudaMalloc(&d->d_pool, total);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_lanes, sizeof(LaneState) * L);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_qhead, 4);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_round, 4 * L);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_lane_ids, 4 * L);
  if (e != cudaSuccess) {
    cudaFree(d->d_pool);
    cudaFree(d->d_lanes);
    cudaFree(d->d_qhead);
    cudaFree(d->d_round);
    cudaFree(d->d_lane_ids);
    delete d;
    return cuda_fail(e, "decoder allocation");
  }
  d->pool_bytes = total;
  char* base = (char*)d->d_pool;
  KParams& kp = d->kp;
  kp.state_info = g->d_state;
  kp.arcs = g->d_arcs;
  kp.start = g->start;
  kp.beam = beam;
  kp.alpha = d->alpha;
  kp.C = d->C;
  kp.NBK = d->C / 4;
  kp.C_ovf = d->C_ovf;
  kp.FCAP = d->FCAP;
  kp.R_cap = d->R_cap;
  kp.TMAX = d->TMAX;
  kp.lanes_st = d->d_lanes;
  kp.front = (int4*)(base + parts[i_front].off);
  kp.claim = (int2*)(base + parts[i_claim].off);
  kp.prevg = (int32_t*)(base + parts[i_prevg].off);
  kp.slotrec = (int32_t*)(base + parts[i_slotrec].off);
  kp.fslot = (int2*)(base + parts[i_fslot].off);
  kp.ovf = (u64*)(base + parts[i_ovf].off);
  kp.wl = (int2*)(base + parts[i_wl].off);
  kp.rec = (int2*)(base + parts[i_rec].off);
  kp.rec_cost = i_rcost != (size_t)-1 ? (float*)(base + parts[i_rcost].off) : nullptr;
  kp.fstats = (float*)(base + parts[i_fst].off);
  kp.fcounts = (long long*)(base + parts[i_fcn].off);
  kp.layer_info = (int2*)(base + parts[i_linfo].off);
  kp.q_head = d->d_qhead;
  kp.lane_round = d->d_round;
  e = cudaMemset(base + parts[i_ovf].off, 0xFF, parts[i_ovf].bytes);
  if (e == cudaSuccess) e = cudaMemset(d->d_lanes, 0, sizeof(LaneState) * L);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    wfst_decoder_destroy(d);
    return cuda_fail(e, "decoder init");
  }
  d->h_initialized.assign(L, 0);
  d->device_bytes = (int64_t)(total + sizeof(LaneState) * L + 12 * L + 4);
  *out = d;
  return WFST_OK;
}

void wfst_decoder_destroy(wfst_decoder_t d) {
  if (!d) return;
  DeviceGuard dg(d->device);
  cudaDeviceSynchronize();
  cudaFree(d->d_pool);
  cudaFree(d->d_lanes);
  cudaFree(d->d_qhead);
  cudaFree(d->d_round);
  cudaFree(d->d_lane_ids);
  cudaFree(d->d_path);
  cudaFree(d->d_host_stage[0]);
  cudaFree(d->d_host_stage[1]);
  if (d->copy_stream) cudaStreamDestroy(d->copy_stream);
  for (int i = 0; i < 2; i++) {
    if (d->ev_copy[i]) cudaEventDestroy(d->ev_copy[i]);
    if (d->ev_use[i]) cudaEventDestroy(d->ev_use[i]);
  }
  delete d;
}

static wfst_status set_lanes(wfst_decoder_t d, const int32_t* streams, int32_t B, cudaStream_t st,
                             bool require_init) {
  std::vector<int32_t> ids(B);
  std::vector<char> seen(d->n_lanes, 0);
  for (int32_t i = 0; i < B; i++) {
    int32_t s = streams ? streams[i] : i;
    if (s < 0 || s >= d->n_lanes) return fail(WFST_ERR_INVALID_ARG, "stream id out of range");
    if (seen[s]) return fail(WFST_ERR_INVALID_ARG, "duplicate stream id");
    seen[s] = 1;
    if (require_init && !d->h_initialized[s]) return fail(WFST_ERR_STATE, "stream " + std::to_string(s) + " not reset");
    ids[i] = s;
  }
  if (ids == d->cur_ids) return WFST_OK;  // same mapping as the work already queued
  // the buffer may be in use by queued kernels: wait for them before replacing it
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(d->d_lane_ids, ids.data(), 4 * (size_t)B, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "lane ids upload");
  d->cur_ids = ids;
  (void)st;
  return WFST_OK;
}

wfst_status wfst_decoder_reset(wfst_decoder_t d, const int32_t* streams, int32_t n, void* cuda_stream) {
  if (!d) return fail(WFST_ERR_INVALID_ARG, "NULL decoder");
  DeviceGuard dg(d->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int32_t B = streams ? n : d->n_lanes;
  if (B <= 0) return WFST_OK;
  wfst_status s = set_lanes(d, streams, B, st, false);
  if (s != WFST_OK) return s;
  KParams kp = d->kp;
  kp.ll = nullptr;
  kp.T = 0;
  kp.B = B;
  kp.P = 0;
  kp.lanes = d->d_lane_ids;
  kp.mode = kModeInit;
  kp.K = 1;
  kp.n_items = B;
  cudaError_t e = launch_frames(d, kp, st);
  if (e != cudaSuccess) return cuda_fail(e, "reset launch");
  for (int32_t i = 0; i < B; i++) d->h_initialized[streams ? streams[i] : i] = 1;
  return WFST_OK;
}

wfst_status wfst_decode_frames(wfst_decoder_t d, const float* d_loglikes, int32_t T, int32_t B, int32_t P,
                               const int32_t* streams, void* cuda_stream) {
  if (!d) return fail(WFST_ERR_INVALID_ARG, "NULL decoder");
  if (T < 0 || B < 0) return fail(WFST_ERR_INVALID_ARG, "negative size");
  if (T == 0 || B == 0) return WFST_OK;
  if (!d_loglikes) return fail(WFST_ERR_INVALID_ARG, "NULL loglikes");
  if (B > d->n_lanes) return fail(WFST_ERR_INVALID_ARG, "B exceeds n_streams");
  if (P <= d->g->max_pdf) return fail(WFST_ERR_PDF_RANGE, "P=" + std::to_string(P) + " <= max pdf " + std::to_string(d->g->max_pdf));
  DeviceGuard dg(d->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  wfst_status s = set_lanes(d, streams, B, st, true);
  if (s != WFST_OK) return s;
  KParams kp = d->kp;
  kp.ll = d_loglikes;
  kp.T = T;
  kp.B = B;
  kp.P = P;
  kp.lanes = d->d_lane_ids;
  kp.mode = kModeFrames;
  // one work item per (round of K frames, lane); fewer lanes than SMs -> one item per lane
  int K = d->o.frames_per_item;
  int max_ctas = d->o.max_ctas > 0 ? d->o.max_ctas : d->n_sm;
  if (B <= max_ctas) K = T;
  kp.K = K;
  long long items = (long long)((T + K - 1) / K) * B;
  if (items > INT32_MAX) return fail(WFST_ERR_INVALID_ARG, "too many work items");
  kp.n_items = (int32_t)items;
  cudaError_t e = launch_frames(d, kp, st);
  if (e != cudaSuccess) return cuda_fail(e, "decode launch");
  return WFST_OK;
}

wfst_status wfst_decode_frames_host(wfst_decoder_t d, const float* h_loglikes, int32_t T, int32_t B, int32_t P,
                                    const int32_t* streams, int32_t chunk_frames, void* cuda_stream) {
  if (!d) return fail(WFST_ERR_INVALID_ARG, "NULL decoder");
  if (T < 0 || B < 0) return fail(WFST_ERR_INVALID_ARG, "negative size");
  if (T == 0 || B == 0) return WFST_OK;
  if (!h_loglikes) return fail(WFST_ERR_INVALID_ARG, "NULL loglikes");
  DeviceGuard dg(d->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int32_t CF = chunk_frames > 0 ? std::min(chunk_frames, T) : std::min(T, 25);
  size_t need = (size_t)CF * B * P * 4;
  cudaError_t e = cudaSuccess;
  if (need > d->stage_bytes) {
    cudaStreamSynchronize(st);
    if (d->copy_stream) cudaStreamSynchronize(d->copy_stream);
    cudaFree(d->d_host_stage[0]);
    cudaFree(d->d_host_stage[1]);
    d->d_host_stage[0] = d->d_host_stage[1] = nullptr;
    d->stage_bytes = 0;
    e = cudaMalloc(&d->d_host_stage[0], need);
    if (e == cudaSuccess) e = cudaMalloc(&d->d_host_stage[1], need);
    if (e != cudaSuccess) return cuda_fail(e, "staging allocation");
    d->stage_bytes = need;
  }
  if (!d->copy_stream) {
    e = cudaStreamCreateWithFlags(&d->copy_stream, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; i++) {
      e = cudaEventCreateWithFlags(&d->ev_copy[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_use[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_fail(e, "copy stream");
  }
  // the staging buffers may still be read by earlier work on st
  e = cudaEventRecord(d->ev_use[0], st);
  if (e == cudaSuccess) e = cudaEventRecord(d->ev_use[1], st);
  if (e != cudaSuccess) return cuda_fail(e, "event");
  int k = 0;
  for (int32_t t0 = 0; t0 < T; t0 += CF, k ^= 1) {
    int32_t n = std::min(CF, T - t0);
    size_t bytes = (size_t)n * B * P * 4;
    e = cudaStreamWaitEvent(d->copy_stream, d->ev_use[k], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d->d_host_stage[k], h_loglikes + (size_t)t0 * B * P, bytes, cudaMemcpyHostToDevice,
                          d->copy_stream);
    if (e == cudaSuccess) e = cudaEventRecord(d->ev_copy[k], d->copy_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, d->ev_copy[k], 0);
    if (e != cudaSuccess) return cuda_fail(e, "H2D chunk");
    wfst_status s = wfst_decode_frames(d, d->d_host_stage[k], n, B, P, streams, cuda_stream);
    if (s != WFST_OK) return s;
    e = cudaEventRecord(d->ev_use[k], st);
    if (e != cudaSuccess) return cuda_fail(e, "event");
  }
  return WFST_OK;
}

wfst_status wfst_decoder_sync(wfst_decoder_t d) {
  if (!d) return fail(WFST_ERR_INVALID_ARG, "NULL decoder");
  DeviceGuard dg(d->device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "sync");
  std::vector<LaneState> L(d->n_lanes);
  e = cudaMemcpy(L.data(), d->d_lanes, sizeof(LaneState) * d->n_lanes, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "lane state");
  for (int i = 0; i < d->n_lanes; i++)
    if (L[i].status != WFST_OK)
      return fail((wfst_status)L[i].status, "stream " + std::to_string(i) + ": " +
                                                 wfst_status_string((wfst_status)L[i].status));
  return WFST_OK;
}

wfst_status wfst_decoder_status(wfst_decoder_t d, int32_t stream) {
  if (!d || stream < 0 || stream >= d->n_lanes) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  DeviceGuard dg(d->device);
  LaneState L;
  cudaError_t e = cudaMemcpy(&L, d->d_lanes + stream, sizeof L, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "lane state");
  if (!d->h_initialized[stream]) return WFST_ERR_STATE;
  return (wfst_status)L.status;
}

wfst_status wfst_get_best_paths(wfst_decoder_t d, const int32_t* streams, int32_t n, float* cost,
                                int32_t* reached_final, int32_t* arcs, int32_t* olabels, int32_t arcs_cap,
                                int32_t* n_arcs, int32_t* n_olabels) {
  if (!d || n < 0 || !cost || !reached_final || !n_arcs) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  if (n == 0) return WFST_OK;
  DeviceGuard dg(d->device);
  if (arcs_cap < 0) arcs_cap = 0;
  for (int i = 0; i < n; i++) {
    int32_t s = streams ? streams[i] : i;
    if (s < 0 || s >= d->n_lanes) return fail(WFST_ERR_INVALID_ARG, "stream id out of range");
    if (!d->h_initialized[s]) return fail(WFST_ERR_STATE, "stream " + std::to_string(s) + " not reset");
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "sync");
  int cap = std::max(arcs_cap, 1);
  size_t need = (size_t)n * (6 + 2 * (size_t)cap);
  if (need > d->path_cap) {
    cudaFree(d->d_path);
    d->d_path = nullptr;
    e = cudaMalloc(&d->d_path, need * 4);
    if (e != cudaSuccess) {
      d->path_cap = 0;
      return cuda_fail(e, "path buffer");
    }
    d->path_cap = need;
  }
  int32_t* p = d->d_path;
  int32_t* d_ids = p;
  float* d_cost = (float*)(p + n);
  int32_t* d_reached = p + 2 * n;
  int32_t* d_nar = p + 3 * n;
  int32_t* d_nol = p + 4 * n;
  int32_t* d_st = p + 5 * n;
  int32_t* d_arcs = p + 6 * n;
  int32_t* d_ol = d_arcs + (size_t)n * cap;
  std::vector<int32_t> ids(n);
  for (int i = 0; i < n; i++) ids[i] = streams ? streams[i] : i;
  e = cudaMemcpy(d_ids, ids.data(), 4 * (size_t)n, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "ids");
  best_path_kernel<<<n, 256>>>(d->kp, d_ids, n, cap, d_cost, d_reached, d_nar, d_arcs, d_ol, d_nol, d_st);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "best path kernel");
  std::vector<int32_t> head(6 * (size_t)n);
  e = cudaMemcpy(head.data(), p, 4 * head.size(), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && arcs && arcs_cap > 0)
    e = cudaMemcpy(arcs, d_arcs, 4 * (size_t)n * cap, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && olabels && arcs_cap > 0)
    e = cudaMemcpy(olabels, d_ol, 4 * (size_t)n * cap, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "path D2H");
  wfst_status first = WFST_OK;
  for (int i = 0; i < n; i++) {
    memcpy(&cost[i], &head[n + i], 4);
    reached_final[i] = head[2 * n + i];
    n_arcs[i] = head[3 * n + i];
    if (n_olabels) n_olabels[i] = head[4 * n + i];
    wfst_status s = (wfst_status)head[5 * n + i];
    if (s != WFST_OK && first == WFST_OK) {
      first = s;
      set_error("stream " + std::to_string(ids[i]) + ": " + wfst_status_string(s));
    }
  }
  return first;
}

wfst_status wfst_get_best_path(wfst_decoder_t d, int32_t stream, int32_t* olabels, int32_t olabels_cap,
                               int32_t* n_olabels, int32_t* arcs, int32_t arcs_cap, int32_t* n_arcs, float* cost,
                               int32_t* reached_final) {
  if (!d || !cost || !reached_final) return fail(WFST_ERR_INVALID_ARG, "NULL argument");
  int32_t cap = std::max(std::max(olabels_cap, arcs_cap), 0);
  int32_t nar = 0, nol = 0;
  std::vector<int32_t> a(std::max(cap, 1)), o(std::max(cap, 1));
  wfst_status s = wfst_get_best_paths(d, &stream, 1, cost, reached_final, a.data(), o.data(), cap, &nar, &nol);
  if (n_arcs) *n_arcs = nar;
  if (n_olabels) *n_olabels = nol;
  if (s != WFST_OK && s != WFST_ERR_INVALID_ARG) return s;
  if ((arcs && nar > arcs_cap) || (olabels && nol > olabels_cap) || s == WFST_ERR_INVALID_ARG)
    return fail(WFST_ERR_INVALID_ARG, "output capacity too small");
  if (arcs) memcpy(arcs, a.data(), 4 * (size_t)std::min(nar, arcs_cap));
  if (olabels) memcpy(olabels, o.data(), 4 * (size_t)std::min(nol, olabels_cap));
  return WFST_OK;
}

wfst_status wfst_decoder_stats(wfst_decoder_t d, wfst_stats_t* s) {
  if (!d || !s) return fail(WFST_ERR_INVALID_ARG, "NULL argument");
  DeviceGuard dg(d->device);
  std::vector<LaneState> L(d->n_lanes);
  cudaError_t e = cudaMemcpy(L.data(), d->d_lanes, sizeof(LaneState) * d->n_lanes, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "stats");
  memset(s, 0, sizeof *s);
  for (auto& x : L) {
    s->frames += x.frames_total;
    s->emit_arcs += x.emit_arcs;
    s->eps_arcs += x.eps_arcs;
    s->eps_relax += x.eps_relax;
    s->candidates += x.cand;
    s->survivors += x.surv;
    s->overflow_inserts += x.ovf;
    s->alpha_frames += x.alpha_frames;
    s->records_used_max = std::max<int64_t>(s->records_used_max, x.rec_used);
  }
  s->device_bytes = d->device_bytes;
  return WFST_OK;
}

wfst_status wfst_decoder_reset_stats(wfst_decoder_t d) {
  if (!d) return fail(WFST_ERR_INVALID_ARG, "NULL decoder");
  DeviceGuard dg(d->device);
  std::vector<LaneState> L(d->n_lanes);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(L.data(), d->d_lanes, sizeof(LaneState) * d->n_lanes, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "stats");
  for (auto& x : L) x.emit_arcs = x.eps_arcs = x.eps_relax = x.cand = x.surv = x.ovf = x.alpha_frames = x.frames_total = 0;
  e = cudaMemcpy(d->d_lanes, L.data(), sizeof(LaneState) * d->n_lanes, cudaMemcpyHostToDevice);
  return e == cudaSuccess ? WFST_OK : cuda_fail(e, "stats");
}

wfst_status wfst_decoder_frame_stats(wfst_decoder_t d, int32_t stream, float* fstats, int64_t* fcounts,
                                     int32_t cap_frames, int32_t* n_frames) {
  if (!d || stream < 0 || stream >= d->n_lanes || !n_frames) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  DeviceGuard dg(d->device);
  cudaError_t e = cudaDeviceSynchronize();
  LaneState L;
  if (e == cudaSuccess) e = cudaMemcpy(&L, d->d_lanes + stream, sizeof L, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "frame stats");
  int n = std::min(std::min(L.frames, d->TMAX), std::max(cap_frames, 0));
  *n_frames = std::min(L.frames, d->TMAX);
  if (fstats && n > 0)
    e = cudaMemcpy(fstats, d->kp.fstats + (size_t)stream * d->TMAX * 3, sizeof(float) * 3 * n, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && fcounts && n > 0)
    e = cudaMemcpy(fcounts, d->kp.fcounts + (size_t)stream * d->TMAX * 5, sizeof(int64_t) * 5 * n,
                   cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? WFST_OK : cuda_fail(e, "frame stats");
}

wfst_status wfst_debug_layer(wfst_decoder_t d, int32_t stream, int32_t layer, int32_t* states, int32_t* arcs,
                             float* costs, int32_t cap, int32_t* n) {
  if (!d || stream < 0 || stream >= d->n_lanes || !n || layer < 0) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  if (layer > d->TMAX) return fail(WFST_ERR_INVALID_ARG, "layer beyond max_frames");
  DeviceGuard dg(d->device);
  cudaError_t e = cudaDeviceSynchronize();
  LaneState L;
  if (e == cudaSuccess) e = cudaMemcpy(&L, d->d_lanes + stream, sizeof L, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "debug layer");
  if (layer > L.frames) return fail(WFST_ERR_INVALID_ARG, "layer not decoded yet");
  int2 info;
  e = cudaMemcpy(&info, d->kp.layer_info + (size_t)stream * (d->TMAX + 1) + layer, sizeof info, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "debug layer");
  *n = info.y;
  if (info.y > cap) return fail(WFST_ERR_INVALID_ARG, "capacity too small");
  std::vector<int2> r(info.y);
  std::vector<float> c(info.y, NAN);
  if (info.y > 0) {
    e = cudaMemcpy(r.data(), d->kp.rec + (size_t)stream * d->R_cap + info.x, sizeof(int2) * info.y,
                   cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && d->kp.rec_cost)
      e = cudaMemcpy(c.data(), d->kp.rec_cost + (size_t)stream * d->R_cap + info.x, 4 * (size_t)info.y,
                     cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "debug layer");
  }
  for (int i = 0; i < info.y; i++) {
    int32_t a = r[i].x;
    if (states) states[i] = a < 0 ? d->g->start : d->g->h_dst[a];
    if (arcs) arcs[i] = a;
    if (costs) costs[i] = c[i];
  }
  return WFST_OK;
}

}  // extern "C"
