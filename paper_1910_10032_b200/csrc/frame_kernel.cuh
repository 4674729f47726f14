// frame_kernel.cuh -- device code of the decoder (rows a1-a7 of SURVEY §8); included by decoder.cu.
//
// One persistent CTA per SM owns one lane (stream) at a time and runs whole frames with CTA
// barriers only between phases: warp-centric load-balanced emitting expansion, running
// best + beam and exact max-active, epsilon closure to a fixed point under the
// fixed cutoff, contraction into a frontier of one representative per state,
// sorted by state id, with traceback records.  DESIGN.md §5 explains the layout.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "wfst_internal.h"

namespace wfst_dev {

typedef unsigned long long u64;

constexpr u64 kEmpty = 0xFFFFFFFFFFFFFFFFull;
constexpr int kNB = 1024;          // cost bins of the max-active bound
#ifndef WFST_MAXPROBE
#define WFST_MAXPROBE 8
#endif
#ifndef WFST_ROWSMEM
#define WFST_ROWSMEM 1
#endif
constexpr int kMaxProbeS = WFST_MAXPROBE;   // buckets probed in the on-chip table before overflowing
constexpr int kMaxProbeG = 512;    // buckets probed in the global overflow table
constexpr int kModeFrames = 0, kModeInit = 1;
#ifndef WFST_PHASES
#define WFST_PHASES 1   // per-phase clock64 marks (wfst_stats_t.phase_cycles): measured free (A/B)
#endif
#ifndef WFST_KBIG
#define WFST_KBIG 64
#endif
#ifndef WFST_EARLY_CURSORS
#define WFST_EARLY_CURSORS 1   // warp 0 places the contraction's cursors before an earlier barrier
#endif
#ifndef WFST_OWNER_BSEARCH
#define WFST_OWNER_BSEARCH 1   // owner of each flattened arc by a shuffle binary search (else head flags + max-scan)
#endif
constexpr int kBig = WFST_KBIG;    // tokens with more emitting arcs are expanded CTA-wide
#ifndef WFST_THSHIFT
#define WFST_THSHIFT 10
#endif
constexpr int kThShift = WFST_THSHIFT;   // the max-active bound is refreshed every 2^kThShift claims
constexpr int kThShiftSorted = 7;        // ... every 128 claims in bin-ordered frames
constexpr int kBigCap = 256;
constexpr int kStage = 32;         // per-warp staging buffer (candidates awaiting insertion)
constexpr int kPlace = 64;         // coarse cost bins ordering the next frontier (kNB / 16 each)
#ifndef WFST_SMALLCLAIMS
#define WFST_SMALLCLAIMS 2048
#endif
constexpr int kSmallClaims = WFST_SMALLCLAIMS;   // frames with at most this many claims use an on-chip claim list
#ifndef WFST_EPSWARP
#define WFST_EPSWARP 32
#endif
constexpr int kEpsWarp = WFST_EPSWARP > 0 ? WFST_EPSWARP : 1;   // epsilon worklists up to this size: warp 0 alone
constexpr bool kEpsWarpOn = WFST_EPSWARP > 0;

struct LaneState {
  int32_t status;       // wfst_status, sticky
  int32_t initialized;
  int32_t n_front;      // survivors in the current frontier (cost-bucketed order)
  int32_t cur;          // frontier buffer holding them
  int32_t frames;       // frames decoded in this utterance
  int32_t layer_base;   // record index of the current layer's first survivor (logical)
  int32_t rec_used;     // records written in this utterance (logical; physical = index % R_cap)
  float front_best;     // min cost of the current survivors
  u64 emit_arcs, eps_arcs, eps_relax, cand, surv, ovf, alpha_frames, frames_total;
  u64 phase[12];        // clock64 cycles per phase (see wfst_stats_t.phase_cycles)
  u64 phase_alpha[12];  // the same, frames where max-active bound only
  int32_t rec_phys;     // rec_used % R_cap: the record ring slot of the next record
  int32_t rec_floor;    // records below this are reclaimed (row f2 traceback GC; 0 otherwise)
  int32_t layer_floor;  // layers below this are reclaimed (layer index ring of TMAX+1 entries)
  int32_t last_alpha;   // max-active bound in the lane's previous frame (selects the insertion order)
  u64 sel_entries;      // table entries read by the max-active selection passes (entries x passes)
  float cpa[2];         // moving average of SM cycles per emitting arc in alpha-bound frames,
                        // arrival order [0] and bin order [1] (insert_order = auto picks the cheaper)
  int32_t n_alpha_seen; // alpha-bound frames seen by the chooser
  int32_t gc_layer;     // newest layer the last traceback GC compacted (-1: none; gc_kernel.cuh)
  int32_t rec_peak;     // most records held at once (rec_used - rec_floor after a frame)
  int32_t pad3_;
};

struct KParams {
  const int4* __restrict__ state_info;   // {e_begin, e_end, eps_end, final bits}
  const int4* __restrict__ arcs;         // {dst, weight bits, pdf, src | dst_has_eps << 31}
  int32_t start, n_states;
  const float* ll;
  int32_t T, B, P;
  const int32_t* lanes;   // batch index -> lane id
  int32_t mode, K, n_items;
  int32_t* q_head;
  int32_t* lane_round;
  float beam;
  int32_t alpha;
  int32_t C, NBK, C_ovf, FCAP;
  int32_t row_floats;     // log-likelihood columns staged on chip per frame (max pdf + 1)
  int32_t row_bytes;      // shared bytes reserved for the staged row
  int64_t R_cap;
  int32_t TMAX;
  LaneState* lanes_st;
  int4* front;        // [lane][2][FCAP]  {state, cost bits, e_begin, n_emit}, cost-bucketed
  uint32_t* claim;    // [cta][C_ovf]     overflow-table slots claimed this frame
                      // (claim, win, ovf, wl: one set per persistent CTA, reset by the end of every frame)
  u64* win;           // [cta][FCAP]      per slot: min (ord(cost) << 32 | canonical arc id)
  u64* ovf;           // [cta][C_ovf]     global overflow token table
  uint32_t* wl;       // [cta][2][FCAP]   epsilon worklists (slots)
  int2* rec;          // [lane][R_cap]    traceback records {winning arc (-1: start), state}
  float* rec_cost;    // [lane][R_cap]    survivor cost (debug_costs or lattice)
  int4* rec_si;       // [lane][R_cap]    survivor's {e_begin, e_end, eps_end, state} (lattice only)
  float* fstats;      // [lane][TMAX][3]
  long long* fcounts; // [lane][TMAX][5]
  int2* layer_info;   // [lane][TMAX+1]   {record base, survivors}
  int4* cbuf;         // [cta][kPlace][cbuf_cap] candidates of a bin-ordered frame, by coarse cost bin
  int32_t cbuf_cap;   // entries per coarse bin (0: bin-ordered insertion off)
  int32_t sort_mode;  // 0 never, 1 after a frame where max-active bound, 2 always (tests)
};

struct SmemCtl {
  int32_t item, lane, b, status;
  uint32_t best_ord;
  int32_t theta;
  int32_t n_claim, n_claim_emit, n_ovf, n_oclaim, n_surv, n_in, n_wl, n_big, next_group;
  int32_t wlc[3];   // epsilon worklist counters (rotating)
  int32_t eps_r, eps_cur;           // where the warp-synchronous epsilon iterations stopped
  int32_t cursors_done;             // warp 0 placed the contraction's cursors early this frame
  uint32_t swl[2][kEpsWarp];        // the first kEpsWarp entries of the epsilon worklists
#ifdef WFST_COUNT
  unsigned long long dbgc[4];   // alpha-bound frames: claims above k_alpha by (0,0.5], (0.5,2], (2,5], >5
#endif
  int32_t bcnt[kPlace];      // bin-ordered frames: candidates appended per coarse cost bin
  int32_t bbase[kPlace + 1]; // bin-ordered frames: their prefix sums (drain order)
  int32_t next_chunk;        // bin-ordered frames: drain cursor
  int32_t sorted;            // this frame inserts its candidates in coarse-bin order
  int32_t choose;            // the order of this frame was chosen by the auto rule
  int32_t pl_base[kPlace];   // placement cursors
  int32_t n_app;             // survivors appended in the cutoff's bin
  long long t_mark;
  u64 ph[12];                    // this frame's phase cycles (thread 0), flushed by flush_phases
  unsigned long long row_mbar;   // mbarrier of the row's bulk copy
  int32_t row_parity, row_pending, row_off, t_cur;
  float beam_cut, kalpha, ref, inv_w, min_surv;
  int32_t use_alpha;
  int32_t radix_prefix, radix_k;
  int32_t sel_mode, sel_bin, sel_cnt, sel_h;   // fast selection: mode, bin b*, its entries, H(bb)
  uint32_t sel_span;
  unsigned long long emit_arcs, eps_deg, eps_relax, sel_entries;
  uint32_t sclaim[kSmallClaims];   // claimed slots while the frame is small
  int32_t warp_tmp[32];
  long long warp_tmp64[32];
  int32_t big[kBigCap];
  LaneState L;
};

// ---------------- primitives ----------------
__device__ __forceinline__ uint32_t ord_of(float c) {
  uint32_t b = __float_as_uint(c);
  return b ^ ((b & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float float_of_ord(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o ^ 0x80000000u) : ~o;
  return __uint_as_float(b);
}
__device__ __forceinline__ uint32_t bucket_of(uint32_t q, uint32_t nb) { return __umulhi(q * 0x9E3779B1u, nb); }
__device__ __forceinline__ float key_cost(u64 k) { return float_of_ord((uint32_t)(k >> 32)); }

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ u64 lds64(uint32_t a) {
  u64 v;
  asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void lds64x2(uint32_t a, u64& x, u64& y) {
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t a, u64 v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ int4 lds128(uint32_t a) {
  int4 v;
  asm volatile("ld.volatile.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
// sum of 4*N consecutive ints at a 16-B aligned shared address (N 128-bit loads in flight).
// Lanes reading blocks 128 B apart start at rotated offsets, so a warp's loads spread over the
// banks instead of all lanes hitting the same four.
template <int N>
__device__ __forceinline__ int lds_sum(uint32_t a) {
  const uint32_t rot = threadIdx.x & (N - 1);
  int4 v[N];
#pragma unroll
  for (int i = 0; i < N; i++) v[i] = lds128(a + 16u * ((i + rot) & (N - 1)));
  int t = 0;
#pragma unroll
  for (int i = 0; i < N; i++) t += v[i].x + v[i].y + v[i].z + v[i].w;
  return t;
}
__device__ __forceinline__ void sts128(uint32_t a, int4 v) {
  asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ u64 atom_cas_s(uint32_t a, u64 cmp, u64 v) {
  u64 old;
  asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "r"(a), "l"(cmp), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_min_s_u32(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.min.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int atom_add_s(uint32_t a, int v) {
  int old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_min_s32(uint32_t a, uint32_t v) {
  asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_s64(uint32_t a, unsigned long long v) {
  asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void red_add_s(uint32_t a, int v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// Predicated forms: the condition becomes an instruction predicate instead of a branch around
// the atomic/store (no BSSY/BSYNC reconvergence per call site in the hot loops).
__device__ __forceinline__ void red_add_s_if(bool c, uint32_t a, int v) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p red.shared.add.u32 [%0], %1;\n}" ::"r"(a), "r"(v),
               "r"((uint32_t)c) : "memory");
}
__device__ __forceinline__ int atom_add_s_if(bool c, uint32_t a, int v) {
  int old = 0;
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %3, 0;\n @p atom.shared.add.u32 %0, [%1], %2;\n}"
               : "+r"(old) : "r"(a), "r"(v), "r"((uint32_t)c) : "memory");
  return old;
}
__device__ __forceinline__ void sts128_if(bool c, uint32_t a, int4 v) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %5, 0;\n @p st.shared.v4.s32 [%0], {%1, %2, %3, %4};\n}"
               ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"((uint32_t)c) : "memory");
}
__device__ __forceinline__ int lds32(uint32_t a) {
  int v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, int v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ u64 ldg_volatile64(const u64* p) { return *(const volatile u64*)p; }
// drop a dead 128-B line of per-frame scratch from L2 without writing it back to DRAM
#ifndef WFST_DISCARD_FRONT
#define WFST_DISCARD_FRONT 1
#endif
#ifndef WFST_DISCARD_BINS
#define WFST_DISCARD_BINS 0   // measured: saves 12 GB of DRAM writes per C3 launch but costs 3.6% (A/B)
#endif
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void red_min_g64(u64* p, u64 v) {
  asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- TMA bulk copy (global -> shared) completing on an mbarrier ----
__device__ __forceinline__ void mbar_init(uint32_t a, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, int parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
  }
}

// monotone cost -> bin map, used both to count and to reject
__device__ __forceinline__ int bin_of(float c, float ref, float inv_w) {
  float x = __fmul_rn(__fsub_rn(c, ref), inv_w);
  x = fminf(fmaxf(x, 0.0f), (float)(kNB - 1));
  return (int)x;
}

// Insert (state q, key = ord(cost) << 32 | q) into a table of nb buckets of 4 slots.
// Returns the slot, or -1 when the probe limit is reached.  claimed: the slot was empty;
// logit: the cost is <= the slot's (an improvement or a tie); strict: <.
#ifndef WFST_BUCKET
#define WFST_BUCKET 4
#endif
constexpr int kBucket = WFST_BUCKET;   // slots per bucket of the on-chip table
__device__ __forceinline__ int insert_s(uint32_t tab_sa, uint32_t nb, uint32_t q, u64 key, bool& claimed,
                                        bool& logit, bool& strict, uint32_t& old_hi) {
  uint32_t b = bucket_of(q, nb);
  const uint32_t hi = (uint32_t)(key >> 32);
  claimed = logit = strict = false;
#pragma unroll 1
  for (int p = 0; p < kMaxProbeS;) {
    const uint32_t ba = tab_sa + b * (8u * kBucket);
    u64 x[kBucket];
#pragma unroll
    for (int j = 0; j < kBucket; j += 2) lds64x2(ba + 8 * j, x[j], x[j + 1]);
    // bit j: slot j holds q / slot j is empty
    uint32_t mq = 0, me = 0;
#pragma unroll
    for (int j = 0; j < kBucket; j++) {
      mq |= (uint32_t)((uint32_t)x[j] == q) << j;
      me |= (uint32_t)((uint32_t)x[j] == 0xFFFFFFFFu) << j;   // (no state word is all ones: state ids < 2^31 - 1)
    }
    int j;
    if (mq) {
      j = __ffs(mq) - 1;
    } else if (me) {
      j = __ffs(me) - 1;
      const u64 old = atom_cas_s(ba + 8 * j, kEmpty, key);
      if (old == kEmpty) {
        claimed = logit = strict = true;
        old_hi = 0xFFFFFFFFu;
        return (int)(b * kBucket + j);
      }
      if ((uint32_t)old != q) continue;   // lost the slot to another state: re-read this bucket
    } else {
      b = (b + 1 == nb) ? 0 : b + 1;
      p++;
      continue;
    }
    // the state half of a slot never changes: a 32-bit min on the cost half (+4 bytes,
    // little-endian) is the 64-bit min and a native shared atomic
    const uint32_t old = atom_min_s_u32(ba + 8 * j + 4, hi);
    logit = hi <= old;
    strict = hi < old;
    old_hi = old;
    return (int)(b * kBucket + j);
  }
  return -1;
}

__device__ __forceinline__ int insert_g(u64* tab, uint32_t nb, uint32_t q, u64 key, bool& claimed, bool& logit,
                                        bool& strict, uint32_t& old_hi) {
  uint32_t b = bucket_of(q, nb);
  claimed = logit = strict = false;
#pragma unroll 1
  for (int p = 0; p < kMaxProbeG; ++p) {
    u64* bk = tab + (size_t)b * 4;
    u64 x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = ldg_volatile64(bk + j);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if ((uint32_t)x[j] == q && x[j] != kEmpty) {
        u64 old = atomicMin(bk + j, key);
        logit = key <= old;
        strict = key < old;
        old_hi = (uint32_t)(old >> 32);
        return (int)(b * 4 + j);
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (x[j] == kEmpty) {
        u64 old = atomicCAS(bk + j, kEmpty, key);
        if (old == kEmpty) {
          claimed = logit = strict = true;
          old_hi = 0xFFFFFFFFu;
          return (int)(b * 4 + j);
        }
        if ((uint32_t)old == q) {
          old = atomicMin(bk + j, key);
          logit = key <= old;
          strict = key < old;
          old_hi = (uint32_t)(old >> 32);
          return (int)(b * 4 + j);
        }
      }
    b = (b + 1 == nb) ? 0 : b + 1;
  }
  return -1;
}

__device__ __forceinline__ int warp_incl_scan(int x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// warp-aggregated append to a shared counter: returns this lane's index (or -1 if !need)
__device__ __forceinline__ int warp_append(bool need, uint32_t counter_sa) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, need);
  if (m == 0) return -1;
  const int leader = __ffs(m) - 1;
  int base = atom_add_s_if(lane == leader, counter_sa, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  return need ? base + __popc(m & ((1u << lane) - 1u)) : -1;
}

template <int BS>
__device__ __forceinline__ long long block_sum64(long long v, long long* s_tmp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_tmp[w] = v;
  __syncthreads();
  if (w == 0) {
    long long t = lane < BS / 32 ? s_tmp[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    __syncwarp();   // lane 31 has read s_tmp[31] before lane 0 overwrites it
    if (lane == 0) s_tmp[32 - 1] = t;
  }
  __syncthreads();
  const long long t = s_tmp[32 - 1];
  __syncthreads();
  return t;
}

// shared address of a field (optionally indexed) of the Frame's SmemCtl
#define SA(field) (S_sa + (uint32_t)offsetof(SmemCtl, field))
#define SAI(field, i) (S_sa + (uint32_t)offsetof(SmemCtl, field) + 4u * (uint32_t)(i))

// ---------------- one lane's frames ----------------
template <int BS, int R, int AM>
struct Frame {   // AM: max-active rule, 0 exact (R6), 1 histogram (R16) -- a template parameter so
                 // the default kernel carries no code of the other mode
  static constexpr int NW = BS / 32;
  const KParams& p;
  SmemCtl& S;
  uint32_t tab_sa;    // shared address of the token table (C slots of 8 B)
  uint32_t hist_sa;   // shared address of the cost histogram (kNB ints)
  uint32_t stage_sa;  // shared address of this warp's staging buffer (kStage x 16 B)
  uint32_t row_sa;    // shared address of the staged log-likelihood row region
  uint32_t S_sa;      // shared address of S (field addresses are S_sa + offsetof: no per-use
                      // generic-to-shared conversion, which re-reads the CTA's window base)
  int* hist;          // exact count of live table entries per fine cost bin (bin_of), kept by every
                      // insert: +1 on a claim, a move between bins on a strict improvement
  int* sel;           // selection scratch (kNB ints): the stage buffers, idle after the expansion
  uint32_t sel_sa;
  int* wbuf;          // this warp's owner buffer (32 ints, -1 when idle)
  // lane buffers
  int4* F0;           // frontier buffer 0; buffer 1 follows at +FCAP
  uint32_t* claim;
  u64* win;
  u64* ovf;
  uint32_t* wl0;      // epsilon worklist 0; worklist 1 follows at +FCAP
  int4* cb;           // this CTA's coarse-bin candidate buffers (bin-ordered frames)
  int2* rec;
  float* rec_cost;
  int4* rec_si;

  __device__ Frame(const KParams& p_, SmemCtl& S_, uint32_t tab_sa_, int* hist_, int* wbuf_, uint32_t stage_sa_,
                   uint32_t row_sa_, int* sel_)
      : p(p_), S(S_), tab_sa(tab_sa_), hist_sa(saddr(hist_)), stage_sa(stage_sa_), row_sa(row_sa_),
        S_sa(saddr(&S_)), hist(hist_), sel(sel_), sel_sa(saddr(sel_)), wbuf(wbuf_) {}

  // ---- row a0: the frame's log-likelihood row is staged in shared memory by one TMA bulk
  // copy (issued by thread 0; the next frame's row is prefetched during this frame's tail)
  __device__ void row_issue(const float* row_g) {   // thread 0 only
    if (S.row_pending) {
      mbar_wait(saddr(&S.row_mbar), S.row_parity);
      S.row_parity ^= 1;
    }
    const uintptr_t a = (uintptr_t)row_g;
    const uintptr_t s = a & ~(uintptr_t)15;
    const uintptr_t e = (a + (uintptr_t)p.row_floats * 4 + 15) & ~(uintptr_t)15;
    const uint32_t bytes = (uint32_t)(e - s);
    S.row_off = (int)(a - s);
    mbar_expect_tx(saddr(&S.row_mbar), bytes);
    bulk_g2s(row_sa, (const void*)s, bytes, saddr(&S.row_mbar));
    S.row_pending = 1;
  }
  const float* rowg;   // the frame's row in global memory (gathers when it is not staged)
  __device__ __forceinline__ float row_ll(uint32_t rowp, int pdf) const {
#if WFST_ROWSMEM
    return __int_as_float(lds32(rowp + 4u * (uint32_t)pdf));
#else
    return __ldg(rowg + pdf);
#endif
  }
  // all threads: wait for the pending row (caller guarantees one is pending)
  __device__ void row_wait() {
    mbar_wait(saddr(&S.row_mbar), S.row_parity);
    __syncthreads();
    if (threadIdx.x == 0) {
      S.row_parity ^= 1;
      S.row_pending = 0;
    }
  }

  __device__ void bind_scratch() {   // intra-frame scratch of this persistent CTA
    const size_t X = (size_t)blockIdx.x, FC = (size_t)p.FCAP;
    claim = p.claim + X * (size_t)p.C_ovf;
    win = p.win + X * FC;
    ovf = p.ovf + X * (size_t)p.C_ovf;
    wl0 = p.wl + X * 2 * FC;
    cb = p.cbuf ? p.cbuf + X * (size_t)kPlace * (size_t)p.cbuf_cap : nullptr;
  }
  __device__ void bind(int lane) {
    const size_t L = (size_t)lane, FC = (size_t)p.FCAP;
    F0 = p.front + L * 2 * FC;
    rec = p.rec + L * (size_t)p.R_cap;
    rec_cost = p.rec_cost ? p.rec_cost + L * (size_t)p.R_cap : nullptr;
    rec_si = p.rec_si ? p.rec_si + L * (size_t)p.R_cap : nullptr;
  }

  __device__ __forceinline__ u64 slot_key(int i) const { return lds64(tab_sa + 8u * (uint32_t)i); }
  __device__ __forceinline__ void clear_slot(int slot) const {
    if (slot < p.C) sts64(tab_sa + 8u * (uint32_t)slot, kEmpty);
    else ovf[slot - p.C] = kEmpty;
  }
  __device__ __forceinline__ u64 read_slot(int slot) const {
    return slot < p.C ? slot_key(slot) : ldg_volatile64(ovf + (slot - p.C));
  }

  // coarse placement bin of a cost: kNB/kPlace consecutive fine bins (monotone in c)
  __device__ __forceinline__ int pbin(float c) const { return bin_of(c, S.ref, S.inv_w) / (kNB / kPlace); }
  __device__ __forceinline__ int fbin(float c) const { return bin_of(c, S.ref, S.inv_w); }
  // keep the fine histogram equal to the table's current costs: +1 on a claim, a move between
  // bins on a strict improvement (DESIGN.md §5.2 contraction, §10 selection)
  // fine: keep every fine bin exact (the emitting phase: the cutoff selection reads fine counts);
  // otherwise only the coarse sums (the epsilon closure and the initial frame: only the
  // contraction's cursors read the histogram after the selection)
  __device__ __forceinline__ void hist_update(int slot, bool claimed, bool strict, uint32_t old_hi, uint32_t new_hi,
                                              bool fine) {
    if (slot < 0) return;
    if (claimed) {
      red_add_s(hist_sa + 4u * (uint32_t)fbin(float_of_ord(new_hi)), 1);
    } else if (strict) {
      const int ob = fbin(float_of_ord(old_hi)), nb = fbin(float_of_ord(new_hi));
      if (fine ? ob != nb : (ob >> 4) != (nb >> 4)) {
        red_add_s(hist_sa + 4u * (uint32_t)ob, -1);
        red_add_s(hist_sa + 4u * (uint32_t)nb, 1);
      }
    }
  }

  // agg_claims: the caller adds the claims to the placement histogram itself (warp-aggregated)
  __device__ __forceinline__ int insert(uint32_t q, u64 key, bool& claimed, bool& logit, bool& strict,
                                        bool agg_claims = false) {
    uint32_t old_hi = 0xFFFFFFFFu;
    int s = insert_s(tab_sa, (uint32_t)p.NBK, q, key, claimed, logit, strict, old_hi);
    if (s < 0) s = insert_g(ovf, (uint32_t)(p.C_ovf / 4), q, key, claimed, logit, strict, old_hi);
    else {
      hist_update(s, claimed && !agg_claims, strict && !claimed, old_hi, (uint32_t)(key >> 32), agg_claims);
      return s;
    }
    if (s < 0) {
      S.status = WFST_ERR_CAPACITY;
      return -1;
    }
    if (claimed) atomicAdd(&S.n_ovf, 1);
    hist_update(s, claimed && !agg_claims, strict && !claimed, old_hi, (uint32_t)(key >> 32), agg_claims);
    return s + p.C;
  }

  // claim bookkeeping (warp-collective: every lane of the warp calls it).  Returns true on
  // the warp whose append crossed a multiple of 1024 claims at or beyond alpha: that warp
  // refreshes the max-active bound.
  __device__ __forceinline__ bool add_claim(int slot, bool claimed, uint32_t eps_flag, int bin, bool seed = true) {
    const int lane = threadIdx.x & 31;
    const unsigned m = __ballot_sync(0xffffffffu, claimed);
    if (m == 0) return false;
    if (seed) {   // claimed states with epsilon arcs seed the closure (no table scan later)
      const bool e = claimed && eps_flag;
      const int idx = warp_append(e, SA(n_wl));
      if (e) {
        wl0[idx] = (uint32_t)slot;
        if (idx < kEpsWarp) S.swl[0][idx] = (uint32_t)slot;
      }
    }
    const int leader = __ffs(m) - 1;
    int base = atom_add_s_if(lane == leader, SA(n_claim), __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (claimed) {
      const int ci = base + __popc(m & ((1u << lane) - 1u));
      if (ci < kSmallClaims) S.sclaim[ci] = (uint32_t)slot;
      if (slot >= p.C) {   // the on-chip table is scanned directly; only overflow slots are listed
        const int oi = atomicAdd(&S.n_oclaim, 1);
        if (oi < p.C_ovf) claim[oi] = (uint32_t)slot;
        else S.status = WFST_ERR_CAPACITY;
      }
      red_add_s_if(bin >= 0 && !S.sorted, hist_sa + 4u * (uint32_t)bin, 1);
    }
    if (S.sorted) {   // bin-ordered frames: a warp's claims share few bins -- one atomic per bin
      const int key = claimed && bin >= 0 ? bin : -1;
      const unsigned grp = __match_any_sync(0xffffffffu, key);
      red_add_s_if(key >= 0 && lane == __ffs(grp) - 1, hist_sa + 4u * (uint32_t)max(key, 0), __popc(grp));
    }
    const int end = base + __popc(m);
    const int sh = S.sorted ? kThShiftSorted : kThShift;   // bin order: claims past alpha are waste
    return p.alpha > 0 && end >= p.alpha && (end >> sh) != (base >> sh);
  }

  // Candidates in bins >= theta are provably above the exact k_alpha (R6).  The histogram rule
  // (R16) cuts at most one histogram bin (beam/1024) above k_alpha, less than one max-active bin
  // (2*beam/1024): its candidates are rejected two bins later, which keeps the test exact.
  static constexpr int kThMargin = AM == 1 ? 2 : 0;

  // theta = smallest b such that >= alpha distinct states have first-insert bin < b (warp-collective)
  __device__ void update_theta() {
    const int lane = threadIdx.x & 31;
    const int base = lane * (kNB / 32);
    const int s = lds_sum<kNB / 128>(hist_sa + 4u * base);
    const int incl = warp_incl_scan(s);
    const unsigned m = __ballot_sync(0xffffffffu, incl >= p.alpha);
    if (m != 0) {
      const int L = __ffs(m) - 1;
      if (lane == L) {
        int c = incl - s;
        for (int i = 0; i < kNB / 32; i++) {
          c += lds32(hist_sa + 4u * (base + i));
          if (c >= p.alpha) {
            atomicMin(&S.theta, base + i + 1 + kThMargin);
            break;
          }
        }
      }
    }
    __syncwarp();
  }

  // Bin-ordered frames: instead of inserting, append the first n staged
  // candidates of this warp to their coarse cost bin's buffer (L2); drain_bins() inserts them
  // cheapest bin first, so the exact max-active bound theta is known after ~alpha claims and
  // whole bins above it are never inserted.  A full bin buffer inserts directly (the result
  // never depends on the insertion order: R7, R9).  Warp-collective.
  __device__ __forceinline__ void append(int n, float beam, uint32_t best_sa, uint32_t theta_sa) {
    const int lane = threadIdx.x & 31;
    int4 e = make_int4(0, 0, 0, 0);
    bool ok = false;
    if (lane < n) {
      e = lds128(stage_sa + 16u * lane);   // {q, ord, arc id, bin | eps flag << 31}
      const uint32_t o = (uint32_t)e.y;
      const uint32_t bo = (uint32_t)lds32(best_sa);
      ok = bo == 0xFFFFFFFFu || float_of_ord(o) < __fadd_rn(float_of_ord(bo), beam);
      if (ok && o < bo) red_min_s32(best_sa, o);
    }
    const int pb = ok ? (e.w & 0x7FFFFFFF) / (kNB / kPlace) : kPlace;
    const unsigned grp = __match_any_sync(0xffffffffu, pb);
    const int leader = __ffs(grp) - 1;
    int base = atom_add_s_if(pb < kPlace && lane == leader, SAI(bcnt, min(pb, kPlace - 1)), __popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    const int idx = base + __popc(grp & ((1u << lane) - 1u));
    const bool direct = ok && idx >= p.cbuf_cap;
    if (ok && !direct) __stcg(cb + (size_t)pb * p.cbuf_cap + idx, e);
    if (__any_sync(0xffffffffu, direct)) {   // bin buffer full: insert those now (rare)
      __syncwarp();
      const int m = __ballot_sync(0xffffffffu, direct);
      if (direct) sts128(stage_sa + 16u * __popc(m & ((1u << lane) - 1u)), e);
      __syncwarp();
      insert_staged(__popc(m), beam, best_sa, theta_sa);
    }
  }

  // insert the first n staged candidates of this warp (warp-collective)
  __device__ __forceinline__ void flush(int n, float beam, uint32_t best_sa, uint32_t theta_sa) {
    if (S.sorted) append(n, beam, best_sa, theta_sa);
    else insert_staged(n, beam, best_sa, theta_sa);
  }

  __device__ __forceinline__ void insert_staged(int n, float beam, uint32_t best_sa, uint32_t theta_sa) {
    const int lane = threadIdx.x & 31;
    bool claimed = false, logit = false, strict = false;
    int slot = -1, bin = -1;
    uint32_t flag = 0;
    if (lane < n) {
      const int4 e = lds128(stage_sa + 16u * lane);   // {q, ord, arc id, bin | eps flag << 31}
      const uint32_t o = (uint32_t)e.y;
      bin = e.w & 0x7FFFFFFF;
      flag = (uint32_t)e.w >> 31;
      // re-check against the bounds as they are now (both only tighten)
      const uint32_t bo = (uint32_t)lds32(best_sa);
      const bool ok = (bo == 0xFFFFFFFFu || float_of_ord(o) < __fadd_rn(float_of_ord(bo), beam)) &&
                      bin < lds32(theta_sa);
      if (ok) {
        if (o < bo) red_min_s32(best_sa, o);
        const uint32_t qf = (uint32_t)e.x | (flag << 31);   // state | has-epsilon flag
        slot = insert(qf, ((u64)o << 32) | qf, claimed, logit, strict, true);
        if (slot >= 0 && logit) red_min_g64(win + slot, ((u64)o << 32) | (uint32_t)e.z);
        if (slot < 0) claimed = false;
      }
    }
    if (add_claim(slot, claimed, flag, bin)) update_theta();   // counts the claims in hist
  }

  // stage one round of candidates (warp-collective); flushes when the buffer fills
  __device__ __forceinline__ void stage(bool pass, const int4& entry, int& staged, float beam, uint32_t best_sa,
                                        uint32_t theta_sa) {
    const int lane = threadIdx.x & 31;
    const unsigned m = __ballot_sync(0xffffffffu, pass);
    const int n = __popc(m);
    const int rank = __popc(m & ((1u << lane) - 1u));
    if (staged + n < kStage) {
      sts128_if(pass, stage_sa + 16u * (staged + rank), entry);
      staged += n;
    } else {
      const int room = kStage - staged;
      if (pass && rank < room) sts128(stage_sa + 16u * (staged + rank), entry);
      __syncwarp();
      flush(kStage, beam, best_sa, theta_sa);
      __syncwarp();
      if (pass && rank >= room) sts128(stage_sa + 16u * (rank - room), entry);
      staged = n - room;
    }
  }

  // ---- rows a1 + a2: load-balanced emitting expansion ----
  // Each warp takes 32 frontier tokens, scans their emitting degrees, walks the flattened arcs
  // 32*R at a time (owner of arc j from head flags + a max-scan), filters the candidates against
  // the running beam and the max-active bound, and stages the survivors so that the table
  // inserts run with full warps.  Each improving insert also does a fire-and-forget 64-bit
  // RED.MIN of (cost, canonical arc id) into the slot's winner word: the min is exactly the
  // (cost, arc) tie-break of R9.
  __device__ void expand() {
    const int tid = threadIdx.x, lane = tid & 31;
    const int n_f = S.L.n_front;
    const int4* Fin = F0 + (size_t)S.L.cur * p.FCAP;
    const float ref = S.ref, inv_w = S.inv_w, beam = p.beam;
    const uint32_t rowp = row_sa + (uint32_t)S.row_off;
    rowg = row_ptr(S.t_cur);
    const uint32_t best_sa = SA(best_ord), theta_sa = SA(theta);
    long long arcs_total = 0;
    int staged = 0;   // warp-uniform
    // token groups of 32 are handed out dynamically (warps whose groups hold long arc lists
    // do not hold the CTA back at the barrier)
    const uint32_t next_sa = SA(next_group);
    while (true) {
      int tb = atom_add_s_if(lane == 0, next_sa, 32);
      tb = __shfl_sync(0xffffffffu, tb, 0);
      if (tb >= n_f) break;
      const int i = tb + lane;
      int deg = 0, eb = 0;
      float cost = 0.f;
      if (i < n_f) {
        const int4 f = __ldcg(Fin + i);
        eb = f.z;
        deg = f.w;
        cost = __int_as_float(f.y);
      }
      arcs_total += deg;
      if (deg > kBig) {
        const int k = atomicAdd(&S.n_big, 1);
        if (k < kBigCap) {
          S.big[k] = i;
          deg = 0;
        }
      }
      const int incl = warp_incl_scan(deg);
      const int excl = incl - deg;
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      for (int r0 = 0; r0 < total; r0 += 32 * R) {
        int a[R], own[R];
        bool v[R];
#pragma unroll
        for (int u = 0; u < R; u++) {
          const int w0 = r0 + u * 32;
#if WFST_OWNER_BSEARCH
          // owner of arc j = the last token t with excl_t <= j (excl is non-decreasing; a token
          // without arcs shares its excl with the next token, so it is never the last): a binary
          // search over the warp's prefix sums, 5 shuffles
          {
            const int j = w0 + lane;
            int lo = 0;
#pragma unroll
            for (int st = 16; st >= 1; st >>= 1) {
              const int e = __shfl_sync(0xffffffffu, excl, lo + st);
              if (e <= j) lo += st;
            }
            own[u] = lo;
            v[u] = j < total;
            const int eb_o = __shfl_sync(0xffffffffu, eb, lo);
            const int ex_o = __shfl_sync(0xffffffffu, excl, lo);
            a[u] = eb_o + (j - ex_o);
            continue;
          }
#endif
          if (deg > 0 && excl >= w0 && excl < w0 + 32) wbuf[excl - w0] = lane;
          const unsigned cm = __ballot_sync(0xffffffffu, deg > 0 && excl <= w0 && w0 < incl);
          __syncwarp();
          int o = wbuf[lane];
          __syncwarp();
          wbuf[lane] = -1;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, o, d);
            if (lane >= d) o = max(o, y);
          }
          if (cm) o = max(o, __ffs(cm) - 1);
          own[u] = o & 31;
          const int j = w0 + lane;
          v[u] = j < total;
          const int eb_o = __shfl_sync(0xffffffffu, eb, own[u]);
          const int ex_o = __shfl_sync(0xffffffffu, excl, own[u]);
          a[u] = eb_o + (j - ex_o);
          __syncwarp();
        }
        int4 arc[R];
#pragma unroll
        for (int u = 0; u < R; u++) arc[u] = v[u] ? __ldg(p.arcs + a[u]) : make_int4(0, 0, 0, 0);
        float L[R];
#pragma unroll
        for (int u = 0; u < R; u++) L[u] = v[u] ? row_ll(rowp, arc[u].z) : 0.0f;
        const uint32_t bo = (uint32_t)lds32(best_sa);
        const int th = lds32(theta_sa);
        const float bound = bo == 0xFFFFFFFFu ? INFINITY : __fadd_rn(float_of_ord(bo), beam);
#pragma unroll
        for (int u = 0; u < R; u++) {
          const float co = __shfl_sync(0xffffffffu, cost, own[u]);
          const float c = __fadd_rn(__fsub_rn(__fadd_rn(co, __int_as_float(arc[u].y)), L[u]), 0.0f);
          const int bin = bin_of(c, ref, inv_w);
          const bool pass = v[u] && c < bound && bin < th;
          const int4 entry = make_int4(arc[u].x, (int)ord_of(c), a[u], bin | (int)(arc[u].w & 0x80000000));
          stage(pass, entry, staged, beam, best_sa, theta_sa);
        }
      }
    }
    __syncwarp();
    if (staged > 0) flush(staged, beam, best_sa, theta_sa);
    staged = 0;
    __syncthreads();
    mark(3);   // warp-expanded tokens done
    // tokens with large out-degree (hub states): all threads share their arcs
    const int nbig = min(S.n_big, kBigCap);
    for (int k = 0; k < nbig; k++) {
      const int i = S.big[k];
      const int4 f = __ldcg(Fin + i);
      const float cost = __int_as_float(f.y);
      const int deg = f.w;
      for (int j0 = 0; j0 < deg; j0 += BS * R) {
        int4 arc[R];
        bool v[R];
#pragma unroll
        for (int u = 0; u < R; u++) {
          const int j = j0 + u * BS + tid;
          v[u] = j < deg;
          arc[u] = v[u] ? __ldg(p.arcs + f.z + j) : make_int4(0, 0, 0, 0);
        }
        float L[R];
#pragma unroll
        for (int u = 0; u < R; u++) L[u] = v[u] ? row_ll(rowp, arc[u].z) : 0.0f;
        const uint32_t bo = (uint32_t)lds32(best_sa);
        const int th = lds32(theta_sa);
        const float bound = bo == 0xFFFFFFFFu ? INFINITY : __fadd_rn(float_of_ord(bo), beam);
#pragma unroll
        for (int u = 0; u < R; u++) {
          const float c = __fadd_rn(__fsub_rn(__fadd_rn(cost, __int_as_float(arc[u].y)), L[u]), 0.0f);
          const int bin = bin_of(c, ref, inv_w);
          const bool pass = v[u] && c < bound && bin < th;
          const int j = j0 + u * BS + tid;
          const int4 entry = make_int4(arc[u].x, (int)ord_of(c), f.z + j, bin | (int)(arc[u].w & 0x80000000));
          stage(pass, entry, staged, beam, best_sa, theta_sa);
        }
      }
    }
    __syncwarp();
    if (staged > 0) flush(staged, beam, best_sa, theta_sa);
    {
      const unsigned long long wsum = warp_sum64((unsigned long long)arcs_total);
      if (lane == 0 && wsum) red_add_s64(SA(emit_arcs), wsum);
    }
    __syncthreads();
    mark(4);   // hub tokens done
    // the consumed frontier is dead (the next contraction writes the other buffer): drop its
    // lines from L2 so they are never written back (buffers are 128-B aligned: FCAP % 8 == 0)
#if WFST_DISCARD_FRONT
    for (int l = tid; l < (n_f + 7) / 8; l += BS) discard_l2(Fin + 8 * l);
#endif
    if (S.sorted) {
      drain_bins(beam, best_sa, theta_sa);
      mark(7);   // bin-ordered insertion done
    }
  }

  // Bin-ordered frames: insert the appended candidates cheapest coarse bin first.  The bins
  // are concatenated (prefix sums of their counts) and warps take 32-entry chunks in that order
  // from a shared cursor, so no barrier separates the bins; candidates in bins >= theta are
  // provably above k_alpha (R6): the first chunk whose bin lies at or beyond theta ends the
  // drain for every warp (later chunks lie in the same or later bins).
  __device__ void drain_bins(float beam, uint32_t best_sa, uint32_t theta_sa) {
    const int tid = threadIdx.x, lane = tid & 31;
    static_assert(kPlace == 64, "warp 0 scans two bins per lane");
    if (tid < 32) {
      const int c0 = min(S.bcnt[2 * lane], p.cbuf_cap), c1 = min(S.bcnt[2 * lane + 1], p.cbuf_cap);
      const int incl = warp_incl_scan(c0 + c1);
      S.bbase[2 * lane] = incl - c0 - c1;
      S.bbase[2 * lane + 1] = incl - c1;
      if (lane == 31) S.bbase[kPlace] = incl;
    }
    __syncthreads();
    const int total = S.bbase[kPlace];
    const uint32_t cur_sa = SA(next_chunk);
    while (true) {
      int c0 = atom_add_s_if(lane == 0, cur_sa, 32);
      c0 = __shfl_sync(0xffffffffu, c0, 0);
      if (c0 >= total) break;
      const int i = c0 + lane;
      int pb = 0;   // bin of entry i: the last b with bbase[b] <= i
#pragma unroll
      for (int step = kPlace / 2; step > 0; step >>= 1)
        if (pb + step < kPlace && S.bbase[pb + step] <= i) pb += step;
      const int pb0 = __shfl_sync(0xffffffffu, pb, 0);
      if (pb0 * (kNB / kPlace) >= lds32(theta_sa)) break;
      if (i < total) sts128(stage_sa + 16u * lane, __ldcg(cb + (size_t)pb * p.cbuf_cap + (i - S.bbase[pb])));
      __syncwarp();
      insert_staged(min(32, total - c0), beam, best_sa, theta_sa);
      __syncwarp();
    }
    __syncthreads();
    // the bin buffers are dead: drop them from L2 without write-back (bins are 128-B aligned)
#if WFST_DISCARD_BINS
    for (int pb = 0; pb < kPlace; pb++) {
      const int nl = (min(S.bcnt[pb], p.cbuf_cap) + 7) / 8;
      for (int l = tid; l < nl; l += BS) discard_l2(cb + (size_t)pb * p.cbuf_cap + 8 * l);
    }
#endif
  }

  // Visit every live token-table entry: the on-chip table is scanned directly (strided, so a
  // warp reads consecutive slots), then the overflow slots listed this frame.  f(slot, value)
  // is called by every lane with value == kEmpty for empty/out-of-range positions, U entries
  // per lane per step so the loads overlap (warp-collective callbacks are allowed).
  template <int U, typename Fn>
  __device__ __forceinline__ void scan_batches(Fn f) {
    const int tid = threadIdx.x;
    const int nc = S.n_claim;
    if (nc <= kSmallClaims) {   // small frame: the on-chip claim list names every live slot
      for (int i0 = 0; i0 < nc; i0 += BS * U) {
        int sl[U];
        u64 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const int i = i0 + u * BS + tid;
          sl[u] = i < nc ? (int)S.sclaim[i] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++) v[u] = sl[u] >= 0 ? read_slot(sl[u]) : kEmpty;
        f(sl, v);
      }
      return;
    }
    for (int i0 = 0; i0 < p.C; i0 += BS * U) {
      int sl[U];
      u64 v[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        sl[u] = i0 + u * BS + tid;
        v[u] = sl[u] < p.C ? slot_key(sl[u]) : kEmpty;
      }
      f(sl, v);
    }
    const int no = min(S.n_oclaim, p.C_ovf);
    for (int i0 = 0; i0 < no; i0 += BS * U) {
      int sl[U];
      u64 v[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int i = i0 + u * BS + tid;
        sl[u] = i < no ? (int)__ldcg(claim + i) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; u++) v[u] = sl[u] >= 0 ? read_slot(sl[u]) : kEmpty;
      f(sl, v);
    }
  }
  // Visit every live token-table entry: the on-chip table is scanned directly (strided, so a
  // warp reads consecutive slots), then the overflow slots listed this frame.  f(slot, value)
  // is called by every lane with value == kEmpty for empty/out-of-range positions, U entries
  // per lane per step so the loads overlap (warp-collective callbacks are allowed).
  template <int U, typename Fn>
  __device__ __forceinline__ void scan_entries(Fn f) {
    scan_batches<U>([&](const int* sl, const u64* v) {
#pragma unroll
      for (int u = 0; u < U; u++) f(sl[u], v[u]);
    });
  }

  // ---- row a3: beam + exact max-active (readings R5, R6) ----
  // beam_cut: the frame's beam cutoff (every thread computes it from the final best: no barrier
  // publishes S.beam_cut before this call).  Every path below ends with a barrier, which also
  // publishes thread 0's S.beam_cut and the epsilon worklist counters (eps_init).
  __device__ void select_cutoff(float beam_cut) {
    const int tid = threadIdx.x;
    if (tid == 0) eps_init();
    const int n_claim = min(S.n_claim, p.FCAP);
    if (p.alpha <= 0 || n_claim <= p.alpha) {   // max-active cannot bind (n_in <= n_claim)
      if (tid == 0) {
        S.n_in = -1;
        S.use_alpha = 0;
        S.kalpha = INFINITY;
      }
#if WFST_EARLY_CURSORS
      // no epsilon seeds: the table is final, so warp 0 places the contraction's cursors now and
      // this barrier publishes them (the contraction skips its own scan and barrier)
      if (tid < 32 && S.n_wl == 0) {
        place_cursors(min(pbin(beam_cut), pbin(INFINITY)));   // (the contraction's bc with cut_a = inf)
        if (tid == 0) S.cursors_done = 1;
      }
#endif
      __syncthreads();
      return;
    }
    if constexpr (AM == 1) {
      select_hist(beam_cut);
      return;
    }
    // Fast path: hist holds the exact count of live entries per fine cost bin.  bin_of is
    // monotone, so the entries of bins < bb = bin(beam_cut) are in beam and every in-beam entry
    // lies in a bin <= bb.  With H(b) = entries in bins < b: H(bb + 1) <= alpha -> max-active
    // cannot bind; H(bb) > alpha -> it binds and k_alpha is the r-th smallest cost of the bin b*
    // where H reaches alpha (r = alpha - H(b*)): one pass collects that bin's costs, a small
    // radix select over them finds k_alpha.  Otherwise (the bound depends on how bin bb splits
    // at the cutoff, or b* holds too many entries) the general radix select below runs.
    const int bb = bin_of(beam_cut, S.ref, S.inv_w);
    if (tid < 32) {
      const int lane = tid;
      int sum = 0;
      sum = lds_sum<8>(hist_sa + 128u * (uint32_t)lane);
      const int incl = warp_incl_scan(sum);
      const int excl = incl - sum;
      if (lane == (bb >> 5)) {   // H(bb), hist[bb]
        int c = excl;
        for (int d = lane * 32; d < bb; d++) c += lds32(hist_sa + 4u * (uint32_t)d);
        S.sel_h = c;
        S.n_in = lds32(hist_sa + 4u * (uint32_t)bb);
      }
      const unsigned m = __ballot_sync(0xffffffffu, incl >= p.alpha);
      const int L = m ? __ffs(m) - 1 : 32;
      if (lane == L) {   // b* and H(b*)
        int c = excl, d = lane * 32;
        for (; d < lane * 32 + 31; d++) {
          const int h = lds32(hist_sa + 4u * (uint32_t)d);
          if (c + h >= p.alpha) break;
          c += h;
        }
        S.radix_k = p.alpha - c;   // rank within bin d (1-based)
        S.sel_bin = d;
        S.sel_cnt = lds32(hist_sa + 4u * (uint32_t)d);
      }
      __syncwarp();
      if (lane == 0) {
        const int Hbb = S.sel_h, hbb = S.n_in;
        int mode;   // 0 cannot bind, 1 binds in bin b*, 2 general select
        if (Hbb + hbb <= p.alpha) mode = 0;
        else if (Hbb > p.alpha && S.sel_cnt <= kNB - 256) mode = 1;
        else mode = 2;
        S.sel_mode = mode;
        S.n_in = -1;                         // exact in-beam count: only the general select has it
        if (mode == 0) {
          S.use_alpha = 0;
          S.kalpha = INFINITY;
        }
      }
    }
    __syncthreads();
    const int smode = S.sel_mode;
    if (smode == 0) return;
    if (smode == 1) {
      // collect the orderable costs of bin b*'s entries (all in beam) into sel[256..], their
      // min into sel[0]; then 8-bit radix digits over ord - min select the r-th smallest
      const int bs = S.sel_bin, cap = kNB - 256;
      if (tid == 0) {
        S.n_app = 0;
        S.sel_span = 0;
        sel[0] = -1;
        S.sel_entries += (unsigned long long)n_claim;
      }
      __syncthreads();
      const uint32_t cnt_sa = SA(n_app);
      scan_entries<4>([&](int, u64 v) {
        const bool in = v != kEmpty && fbin(key_cost(v)) == bs;
        const int i = warp_append(in, cnt_sa);
        if (in && i < cap) {   // i < hist[b*] <= cap: hist is exact
          sel[256 + i] = (int)(uint32_t)(v >> 32);
          atomicMin((unsigned int*)&sel[0], (uint32_t)(v >> 32));
        }
      });
      __syncthreads();
      const int m = min(S.n_app, cap);
      const uint32_t lo = (uint32_t)sel[0];
      uint32_t mx = 0;
      for (int i = tid; i < m; i += BS) mx = max(mx, (uint32_t)sel[256 + i] - lo);
      mx = __reduce_max_sync(0xffffffffu, mx);
      if ((tid & 31) == 0 && mx) atomicMax(&S.sel_span, mx);
      __syncthreads();
      const uint32_t span = S.sel_span;
      int shift = span ? ((32 - __clz(span) + 7) / 8) * 8 - 8 : 0;
      uint32_t prefix = 0;
      int k = S.radix_k;
      while (true) {
        if (tid < 256) sel[tid] = 0;   // sel[0] (the min) is in lo already
        __syncthreads();
        const uint32_t hmask = shift + 8 >= 32 ? 0u : (0xFFFFFFFFu << (shift + 8));
        for (int i = tid; i < m; i += BS) {
          const uint32_t rk = (uint32_t)sel[256 + i] - lo;
          red_add_s_if((rk & hmask) == (prefix & hmask), sel_sa + 4u * ((rk >> shift) & 255u), 1);
        }
        __syncthreads();
        if (tid < 32) {   // warp 0: the digit holding rank k (8 digits per lane)
          const int lane = tid;
          int sum = 0;
          sum = lds_sum<2>(sel_sa + 32u * (uint32_t)lane);
          const int incl = warp_incl_scan(sum);
          const unsigned bm = __ballot_sync(0xffffffffu, incl >= k);
          const int L = __ffs(bm) - 1;
          if (lane == L) {
            int c = incl - sum, d = lane * 8;
            for (; d < lane * 8 + 7; d++) {
              if (c + sel[d] >= k) break;
              c += sel[d];
            }
            S.radix_k = k - c;
            S.radix_prefix = (int)(prefix | ((uint32_t)d << shift));
          }
        }
        __syncthreads();
        prefix = (uint32_t)S.radix_prefix;
        k = S.radix_k;
        if (shift == 0) break;
        shift -= 8;
      }
      if (tid == 0) {
        S.kalpha = float_of_ord(lo + prefix);
        S.use_alpha = 1;
      }
      __syncthreads();
      return;
    }
    // exact alpha-th smallest in-beam cost by radix select on rk = ord(c) - ord(best) (every
    // entry is >= best): digits of up to 10 bits from the top set bit of the span
    // ord(beam_cut) - ord(best) down (every in-beam rk < span), so the first pass spreads the
    // entries over up to 1024 counters (a degenerate 1-2 bit top digit would send them all to
    // the same shared counter); the first pass also counts the in-beam entries.
    const uint32_t ob = S.best_ord;
    const uint32_t span = ord_of(beam_cut) - ob;
    const int nbits = span ? 32 - __clz(span) : 1;
    int hi = nbits, shift = max(nbits - 10, 0);
    if (tid == 0) {
      S.radix_prefix = 0;
      S.radix_k = p.alpha;
    }
    long long cnt = 0;
    bool first = true;
    if (tid == 0) S.sel_entries += (unsigned long long)n_claim;   // the first pass (in-beam count)
    while (true) {
      for (int i = tid; i < kNB; i += BS) sel[i] = 0;
      __syncthreads();
      const uint32_t prefix = (uint32_t)S.radix_prefix;
      const uint32_t hmask = hi >= 32 ? 0u : (0xFFFFFFFFu << hi);
      const uint32_t dmask = (1u << (hi - shift)) - 1u;
      scan_entries<4>([&](int, u64 v) {
        if (v == kEmpty || !(key_cost(v) < beam_cut)) return;
        if (first) cnt++;
        const uint32_t rk = (uint32_t)(v >> 32) - ob;
        red_add_s_if((rk & hmask) == (prefix & hmask), sel_sa + 4u * ((rk >> shift) & dmask), 1);
      });
      if (first) {
        const long long n_in = block_sum64<BS>(cnt, S.warp_tmp64);   // includes a barrier
        if (tid == 0) S.n_in = (int)n_in;
        first = false;
        if (n_in <= p.alpha) {
          if (tid == 0) {
            S.use_alpha = 0;
            S.kalpha = INFINITY;
          }
          break;
        }
      } else {
        __syncthreads();
      }
      if (tid < 32) {   // warp 0: locate the digit holding rank k
        const int lane = tid;
        const int k = S.radix_k;
        int sum = 0;
        sum = lds_sum<8>(sel_sa + 128u * (uint32_t)lane);
        const int incl = warp_incl_scan(sum);
        const unsigned m = __ballot_sync(0xffffffffu, incl >= k);
        const int L = __ffs(m) - 1;
        if (lane == L) {
          int c = incl - sum;
          int d = lane * 32;
          for (; d < lane * 32 + 31; d++) {
            if (c + sel[d] >= k) break;
            c += sel[d];
          }
          S.radix_k = k - c;
          S.radix_prefix = (int)(prefix | ((uint32_t)d << shift));
        }
      }
      __syncthreads();
      if (shift == 0) {
        if (tid == 0) {
          S.kalpha = float_of_ord(ob + (uint32_t)S.radix_prefix);
          S.use_alpha = 1;
        }
        break;
      }
      hi = shift;
      shift = max(hi - 10, 0);
      if (tid == 0) S.sel_entries += (unsigned long long)n_claim;   // one more radix pass
    }
    for (int i = tid; i < kNB; i += BS) sel[i] = 0;
    __syncthreads();
  }

  // ---- row f4 (NEXT): the paper's histogram max-active (Fig. 1; reading R16):
  // one pass counts the in-beam entries into kNB bins of width beam/kNB over [best, best+beam);
  // b = the first bin whose cumulative count reaches alpha; keep c < best + (b+1)*beam/kNB.
  // Same fp32 operations as the oracle's hist_cutoff.
  __device__ void select_hist(float beam_cut) {
    const int tid = threadIdx.x;
    const float best = float_of_ord(S.best_ord);
    const float inv = __fdiv_rn((float)kNB, p.beam), wd = __fdiv_rn(p.beam, (float)kNB);
    for (int i = tid; i < kNB; i += BS) sel[i] = 0;
    if (tid == 0) S.sel_entries += (unsigned long long)min(S.n_claim, p.FCAP);
    __syncthreads();
    long long cnt = 0;
    scan_entries<4>([&](int, u64 v) {
      const float c = key_cost(v);
      if (v == kEmpty || !(c < beam_cut)) return;
      cnt++;
      float x = __fmul_rn(__fsub_rn(c, best), inv);
      x = fmaxf(fminf(x, (float)(kNB - 1)), 0.0f);
      red_add_s(sel_sa + 4u * (uint32_t)(int)x, 1);
    });
    const long long n_in = block_sum64<BS>(cnt, S.warp_tmp64);   // includes a barrier
    if (tid < 32) {
      const int lane = tid;
      if (n_in > p.alpha) {   // warp 0: the bin where the cumulative count reaches alpha
        int sum = 0;
        sum = lds_sum<8>(sel_sa + 128u * (uint32_t)lane);
        const int incl = warp_incl_scan(sum);
        const unsigned m = __ballot_sync(0xffffffffu, incl >= p.alpha);
        const int L = __ffs(m) - 1;
        if (lane == L) {
          int c = incl - sum, d = lane * 32;
          for (; d < lane * 32 + 31; d++) {
            if (c + sel[d] >= p.alpha) break;
            c += sel[d];
          }
          const float ca = __fadd_rn(best, __fmul_rn((float)(d + 1), wd));
          S.kalpha = nextafterf(ca, -INFINITY);
          S.use_alpha = 1;
        }
      } else if (lane == 0) {
        S.use_alpha = 0;
        S.kalpha = INFINITY;
      }
      if (lane == 0) S.n_in = (int)n_in;
    }
    __syncthreads();
    for (int i = tid; i < kNB; i += BS) sel[i] = 0;
    __syncthreads();
  }

  // ---- row a5: epsilon closure under the fixed cutoff (reading R7) ----
  // relax the epsilon arcs of worklist entry `slot` (-1: none); warp-collective.  Improved
  // tokens with epsilon arcs are appended to worklist `wn` (counter wlc[rn]); the first
  // kEpsWarp entries are mirrored on chip for the warp-synchronous iterations.
  __device__ __forceinline__ void relax_eps(int slot, float cut_b, float cut_a, int rn, uint32_t* Wn, int wn,
                                            long long& relax) {
    int e0 = 0, e1 = 0;
    float cp = 0.f;
    if (slot >= 0) {
      const u64 v = read_slot(slot);
      cp = key_cost(v);
      if (cp < cut_b && cp <= cut_a) {   // only kept tokens relax (R7)
        const int4 si = __ldg(p.state_info + ((uint32_t)v & 0x7FFFFFFFu));
        e0 = si.y;
        e1 = si.z;
      }
    }
    // each thread relaxes its token's epsilon arcs (epsilon out-degrees are small)
    const int n_more = e1 - e0;
    int maxd = n_more;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxd = max(maxd, __shfl_xor_sync(0xffffffffu, maxd, o));
    for (int k = 0; k < maxd; k++) {
      const bool v = k < n_more;
      int4 arc = make_int4(0, 0, 0, 0);
      bool claimed = false, logit = false, strict = false;
      int sl = -1;
      if (v) {
        arc = __ldg(p.arcs + e0 + k);
        const float c = __fadd_rn(__fadd_rn(cp, __int_as_float(arc.y)), 0.0f);
        relax++;
        if (c < cut_b && c <= cut_a) {
          const uint32_t o = ord_of(c);
          const uint32_t q = (uint32_t)arc.x | ((uint32_t)arc.w & 0x80000000u);   // state | has-eps
          sl = insert(q, ((u64)o << 32) | q, claimed, logit, strict);
          if (sl >= 0 && logit) red_min_g64(win + sl, ((u64)o << 32) | (uint32_t)(e0 + k));
          if (sl < 0) claimed = strict = false;
        }
      }
      const uint32_t has_eps = (uint32_t)arc.w >> 31;
      add_claim(sl, claimed, has_eps, -1, false);
      const bool push = strict && has_eps;
      const int wi = warp_append(push, SAI(wlc, rn));
      if (push) {
        if (wi < p.FCAP) Wn[wi] = (uint32_t)sl;
        else S.status = WFST_ERR_CAPACITY;
        if (wi < kEpsWarp) S.swl[wn][wi] = (uint32_t)sl;
      }
    }
  }

  // thread 0, once the seeds are final and before a barrier that precedes eps_closure
  __device__ __forceinline__ void eps_init() {
    S.wlc[0] = S.n_wl;
    S.wlc[1] = S.wlc[2] = 0;
    S.eps_r = 0;
    S.eps_cur = 0;
  }

  // seed: the emitting phase listed every claimed state with epsilon arcs (flag in bit 31 of
  // the state word) in worklist 0; the ones the cutoff drops are skipped below
  // Worklist counters rotate over three words: iteration i reads wlc[i%3], appends to
  // wlc[(i+1)%3] and clears wlc[(i+2)%3] (read in iteration i-1, appended to in i+1), so one
  // barrier per iteration suffices.  (Initialised by eps_init before a preceding barrier.)
  __device__ void eps_closure() {
    const int tid = threadIdx.x;
    const float cut_b = S.beam_cut, cut_a = S.use_alpha ? S.kalpha : INFINITY;
    long long relax = 0;
    // Small worklists (the usual case: a few back-off arcs per frame): warp 0 alone runs the
    // iterations, entries from the on-chip mirror, __syncwarp between iterations -- no CTA
    // barrier and no global worklist read per iteration.  A worklist that outgrows a warp is
    // handed to the CTA-wide loop below (the global worklists always hold every entry).
    if (kEpsWarpOn && S.n_wl > 0 && S.n_wl <= kEpsWarp) {
      if (tid < 32) {
        int cur = 0, r = 0;
        while (true) {
          const int n_wl = S.wlc[r];
          if (n_wl == 0 || n_wl > kEpsWarp) break;
          const int rn = r == 2 ? 0 : r + 1;
          if (tid == 0) S.wlc[rn == 2 ? 0 : rn + 1] = 0;
          relax_eps(tid < n_wl ? (int)S.swl[cur][tid] : -1, cut_b, cut_a, rn, wl0 + (size_t)(cur ^ 1) * p.FCAP, cur ^ 1,
                    relax);
          __syncwarp();
          cur ^= 1;
          r = rn;
        }
        if (tid == 0) {
          S.eps_r = r;
          S.eps_cur = cur;
        }
#if WFST_EARLY_CURSORS
        if (S.wlc[r] == 0) {   // closed in warp mode: the table is final, place the cursors now
          __syncwarp();
          place_cursors(min(pbin(cut_b), pbin(cut_a)));
          if (tid == 0) S.cursors_done = 1;
        }
#endif
      }
      __syncthreads();
    }
    int cur = S.eps_cur, r = S.eps_r;
    while (true) {
      const int n_wl = min(S.wlc[r], p.FCAP);
      if (n_wl == 0) break;
      const int rn = r == 2 ? 0 : r + 1;
      if (tid == 0) S.wlc[rn == 2 ? 0 : rn + 1] = 0;
      const uint32_t* W = wl0 + (size_t)cur * p.FCAP;
      uint32_t* Wn = wl0 + (size_t)(cur ^ 1) * p.FCAP;
      for (int i0 = 0; i0 < n_wl; i0 += BS) {
        const int i = i0 + tid;
        relax_eps(i < n_wl ? (int)__ldcg(W + i) : -1, cut_b, cut_a, rn, Wn, cur ^ 1, relax);
      }
      __syncthreads();
      cur ^= 1;
      r = rn;
    }
    {
      const unsigned long long wsum = warp_sum64((unsigned long long)relax);
      if ((tid & 31) == 0 && wsum) red_add_s64(SA(eps_relax), wsum);
    }
  }

  // ---- rows a4 + a6: contraction into the next frontier (cost-bucketed) + records ----
  // A traceback record is {winning arc, state}: the predecessor is the record of src(arc) in
  // the previous layer (emitting arc) or in the same layer (epsilon arc), found by the
  // end-of-stream traceback -- nothing per frame has to map states to records.
  __device__ void contract() {
    const int tid = threadIdx.x, lane = tid & 31;
    const float cut_b = S.beam_cut, cut_a = S.use_alpha ? S.kalpha : INFINITY;
    // The fine histogram counts the table's live entries per cost bin (kept exact by every
    // insert); a coarse placement bin is kNB/kPlace consecutive fine bins.  pbin is monotone, so
    // coarse bins below bc = min(pbin(cut_b), pbin(cut_a)) hold only survivors and no survivor
    // lies above bc: their counts give exact cursors, and the survivors of bin bc are appended
    // after them.  One pass over the table, no counting pass.
    const int bc = min(pbin(cut_b), pbin(cut_a));
    if (!S.cursors_done) {   // (else warp 0 computed them before an earlier barrier of this frame)
      if (tid < 32) place_cursors(bc);
      __syncthreads();
    }
    mark(6);   // cursors ready
    contract_drain(cut_b, cut_a, bc);
  }

  // warp 0: exclusive scan of the coarse placement bins below bc (the contraction's cursors) from
  // the exact histogram -- valid once no insert can change the table any more
  __device__ __forceinline__ void place_cursors(int bc) {
    const int lane = threadIdx.x & 31;
    static_assert(kPlace == 64 && kNB == 1024, "warp 0 scans two coarse (32 fine) bins per lane");
    {   // (per-frame critical path: no serial loop)
      const int b0 = 2 * lane, b1 = b0 + 1;
      const int f0 = lds_sum<4>(hist_sa + 128u * (uint32_t)lane);         // coarse bin b0
      const int f1 = lds_sum<4>(hist_sa + 128u * (uint32_t)lane + 64u);   // coarse bin b1
      const int c0 = b0 < bc ? f0 : 0, c1 = b1 < bc ? f1 : 0;
      const int incl = warp_incl_scan(c0 + c1);
      const int excl = incl - c0 - c1;
      if (b0 < bc) S.pl_base[b0] = excl;
      if (b1 < bc) S.pl_base[b1] = excl + c0;
      const int acc = __shfl_sync(0xffffffffu, incl, 31);
      const int pbc = __shfl_sync(0xffffffffu, (bc & 1) ? f1 : f0, min(bc, kPlace - 1) >> 1);
      if (lane == 0) {
        S.pl_base[bc] = acc;
        S.n_surv = acc + (bc < kPlace ? pbc : 0);   // upper bound until the appended count is known
        S.n_app = 0;
        S.min_surv = INFINITY;
        S.warp_tmp[0] = -1;   // min survivor cost, orderable (0xFFFFFFFF: none)
      }
    }
  }

  __device__ void contract_drain(float cut_b, float cut_a, int bc) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int n_ub = S.n_surv;
    const int32_t rb = S.L.rec_used;
    if (n_ub > p.FCAP || (long long)rb + n_ub - S.L.rec_floor > p.R_cap || (long long)rb + n_ub > INT32_MAX) {
      if (tid == 0) S.status = WFST_ERR_CAPACITY;
      __syncthreads();
      return;
    }
    const int app0 = S.pl_base[bc];
    const int32_t rp = S.L.rec_phys;   // ring slot of the layer's first record
    float mn = INFINITY;
    // pass 2: drain the tables and place each survivor at its bucket cursor: frontier entry
    // (with the state's emitting range, prepared for the next frame: P:78) and traceback record
    int4* Fout = F0 + (size_t)(S.L.cur ^ 1) * p.FCAP;
    unsigned long long epsd = 0;
    constexpr int U2 = 2;
    scan_batches<U2>([&](const int* sl, const u64* v) {
      int pos[U2];
      u64 w[U2];
      int4 si[U2];
#pragma unroll
      for (int u = 0; u < U2; u++) {   // placement + every global round trip issued up front
        const bool live = v[u] != kEmpty;
        const float c = key_cost(v[u]);
        const bool k = live && c < cut_b && c <= cut_a;
        if (k) mn = fminf(mn, c);
        const int bk = k ? min(pbin(c), bc) : kPlace;   // bin bc: the append region
        const unsigned grp = __match_any_sync(0xffffffffu, bk);
        const int leader = __ffs(grp) - 1;
        const bool lead = bk < kPlace && lane == leader;
        int base = atom_add_s_if(lead && bk < bc, SAI(pl_base, min(bk, kPlace - 1)), __popc(grp));
        base += atom_add_s_if(lead && bk >= bc, SA(n_app), __popc(grp));
        if (bk >= bc) base += app0;
        base = __shfl_sync(0xffffffffu, base, leader);
        pos[u] = k ? base + __popc(grp & ((1u << lane) - 1u)) : (live ? -1 : -2);
        if (live) clear_slot(sl[u]);
#ifdef WFST_COUNT
        if (live && !k && S.use_alpha && c < cut_b) {
          const float d = __fsub_rn(c, cut_a);
          red_add_s64((SA(dbgc) + 8u * (d <= 0.5f ? 0u : d <= 2.0f ? 1u : d <= 5.0f ? 2u : 3u)), 1ull);
        }
#endif

        w[u] = kEmpty;
        si[u] = make_int4(0, 0, 0, 0);
        if (k) {
          w[u] = atomicExch(win + sl[u], kEmpty);   // winner word read + reset in one transaction
          si[u] = __ldg(p.state_info + ((uint32_t)v[u] & 0x7FFFFFFFu));
        } else if (live) {
          win[sl[u]] = kEmpty;
        }
      }
#pragma unroll
      for (int u = 0; u < U2; u++) {
        if (pos[u] < 0) continue;
        const uint32_t q = (uint32_t)v[u] & 0x7FFFFFFFu;
        const float c = key_cost(v[u]);
        // the winner word's cost must be the slot's final cost (every improving insert RED's)
        const int32_t arc = (uint32_t)(w[u] >> 32) == (uint32_t)(v[u] >> 32) ? (int32_t)(uint32_t)w[u] : -2;
        if (arc == -2) S.status = WFST_ERR_STATE;
        Fout[pos[u]] = make_int4((int)q, __float_as_int(c), si[u].x, si[u].y - si[u].x);
        const int64_t r = (int64_t)rp + pos[u] - (rp + pos[u] >= p.R_cap ? p.R_cap : 0);   // record ring
        rec[r] = make_int2(arc, (int)q);
        if (rec_cost) rec_cost[r] = c;
        if (rec_si) rec_si[r] = make_int4(si[u].x, si[u].y, si[u].z, (int)q);   // for the lattice pass
        epsd += (unsigned long long)(si[u].z - si[u].y);
      }
    });
    {
      const unsigned long long wsum = warp_sum64(epsd);
      if (lane == 0 && wsum) red_add_s64(SA(eps_deg), wsum);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      if (lane == 0 && mn < INFINITY) atomicMin((unsigned int*)&S.warp_tmp[0], ord_of(mn));
    }
    __syncthreads();
    if (tid == 0) {
      S.n_surv = app0 + S.n_app;
      const uint32_t o = (uint32_t)S.warp_tmp[0];
      S.min_surv = o == 0xFFFFFFFFu ? INFINITY : float_of_ord(o);
    }
    mark(8);   // placement done
  }

  // sync = false: the caller's next barrier publishes the frame's initial state (row_wait)
  __device__ void begin_frame(float beam_cut_fixed, bool emitting, bool sync = true) {
    const int tid = threadIdx.x;
    for (int i = tid; i < kNB; i += BS) hist[i] = 0;
    if (tid < kPlace) S.bcnt[tid] = 0;
    if (tid == 0) {
      // insertion order of this frame (results never depend on it): bin order when forced, or
      // (auto) after an alpha-bound frame when bin order has been the cheaper one per emitting
      // arc on this lane lately; every 8th alpha-bound frame tries the other order
      bool sorted = false;
      if (emitting && p.cbuf_cap > 0 && p.alpha > 0) {
        if (p.sort_mode == 2) sorted = true;
        else if (p.sort_mode == 1 && S.L.last_alpha)
          sorted = (S.L.cpa[1] <= S.L.cpa[0]) != ((S.L.n_alpha_seen & 7) == 7);
      }
      S.sorted = sorted;
      S.choose = emitting && p.cbuf_cap > 0 && p.alpha > 0 && p.sort_mode == 1 && S.L.last_alpha;
      S.best_ord = 0xFFFFFFFFu;
      S.theta = kNB;
      S.n_claim = 0;
      S.n_oclaim = 0;
      S.n_ovf = 0;
      S.n_big = 0;
      S.next_group = 0;
      S.next_chunk = 0;
      S.cursors_done = 0;
#ifdef WFST_COUNT
      S.dbgc[0] = S.dbgc[1] = S.dbgc[2] = S.dbgc[3] = 0;
#endif
      S.n_wl = 0;
      S.use_alpha = 0;
      S.kalpha = INFINITY;
      S.beam_cut = beam_cut_fixed;
      S.emit_arcs = 0;
      S.eps_relax = 0;
      S.eps_deg = 0;
      S.sel_entries = 0;
      S.n_in = -1;
      const float half = isinf(p.beam) ? 32.0f : 0.5f * p.beam;
      S.ref = S.L.front_best - half;
      S.inv_w = (float)kNB / (4.0f * half);
    }
    if (sync) __syncthreads();
  }

  __device__ void clear_all() {
    for (int i = threadIdx.x; i < p.C; i += BS) sts64(tab_sa + 8u * i, kEmpty);
    for (int i = threadIdx.x; i < p.C_ovf; i += BS) ovf[i] = kEmpty;
    for (int i = threadIdx.x; i < p.FCAP; i += BS) win[i] = kEmpty;
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
        L.rec_peak = max(L.rec_peak, L.rec_used - L.rec_floor);
        L.rec_phys += n_surv;
        if (L.rec_phys >= p.R_cap) L.rec_phys -= (int32_t)p.R_cap;
        L.n_front = n_surv;
        L.cur ^= 1;
        L.front_best = S.min_surv;
        const int layer = emitting ? L.frames + 1 : 0;
        if (emitting) L.frames++;
        L.eps_arcs += S.eps_deg;
        L.eps_relax += S.eps_relax;
        L.cand += S.n_claim;
        L.surv += n_surv;
        L.sel_entries += S.sel_entries;
        L.ovf += S.n_ovf;
        if (emitting) {
          L.emit_arcs += S.emit_arcs;
          L.alpha_frames += S.use_alpha;
          L.frames_total++;
          L.last_alpha = S.use_alpha;
        }
        const size_t lane = (size_t)S.lane;
        p.layer_info[lane * (p.TMAX + 1) + layer % (p.TMAX + 1)] = make_int2(L.layer_base, n_surv);
        if (emitting && t >= 0) {
          const size_t fi = lane * p.TMAX + (L.frames - 1) % p.TMAX;
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
    set_mark();   // the contraction's phase marks measure from here
    if (tid == 0) {
      LaneState& L = S.L;   // a new utterance: keep the lifetime counters
      L.n_front = 0;
      L.cur = 0;
      L.frames = 0;
      L.layer_base = 0;
      L.rec_used = 0;
      L.rec_phys = 0;
      L.rec_floor = 0;
      L.layer_floor = 0;
      L.last_alpha = 0;
      L.gc_layer = -1;
      L.rec_peak = 0;
      L.status = WFST_OK;
      L.initialized = 1;
      L.front_best = 0.0f;
    }
    __syncthreads();
    begin_frame(__fadd_rn(0.0f, p.beam), false);
    if (tid < 32) {
      bool claimed = false, logit = false, strict = false;
      int slot = -1;
      const uint32_t o = ord_of(0.0f);
      uint32_t flag = 0;
      if (tid == 0) {
        const int4 si = __ldg(p.state_info + p.start);
        flag = si.z > si.y ? 1u : 0u;
        const uint32_t qf = (uint32_t)p.start | (flag << 31);
        slot = insert(qf, ((u64)o << 32) | qf, claimed, logit, strict);
        if (slot >= 0) win[slot] = ((u64)o << 32) | 0xFFFFFFFFull;   // the start token (arc -1)
        else claimed = false;
      }
      add_claim(slot, claimed, flag, -1);
      __syncwarp();   // (the seed append of add_claim is visible to lane 0)
      if (tid == 0) {
        S.best_ord = o;
        S.n_claim_emit = 1;
        eps_init();
      }
    }
    __syncthreads();
    eps_closure();
    contract();
    finish_frame(-1, false);
    flush_phases(false, 0);
  }

  __device__ __forceinline__ void mark(int ph) {   // thread 0, after a barrier
#if WFST_PHASES
    if (threadIdx.x == 0) {
      const long long t1 = clock64();
      S.ph[ph] += (u64)(t1 - S.t_mark);
      S.t_mark = t1;
    }
#endif
  }
  __device__ __forceinline__ void tick(long long& t0, int ph) {
#if WFST_PHASES
    if (threadIdx.x == 0) {
      const long long t1 = clock64();
      S.ph[ph] += (u64)(t1 - t0);
      t0 = t1;
    }
#endif
  }
  __device__ __forceinline__ void set_mark() {
#if WFST_PHASES
    if (threadIdx.x == 0) S.t_mark = clock64();
#endif
  }
  // a frame's phase cycles go to the lane's totals, and to the alpha-bound totals when
  // max-active bound in it (thread 0, after the frame's last tick)
  // cyc: the frame's SM cycles (thread 0's clock; the insertion-order chooser's measure)
  __device__ __forceinline__ void flush_phases(bool alpha_frame, u64 cyc) {
    if (threadIdx.x == 0) {
#if WFST_PHASES
#pragma unroll
      for (int k = 0; k < 12; k++) {
        S.L.phase[k] += S.ph[k];
        if (alpha_frame) S.L.phase_alpha[k] += S.ph[k];
        S.ph[k] = 0;
      }
#endif
      if (alpha_frame && S.choose) {   // feed the insertion-order chooser
        const float x = (float)cyc / (float)max(1ull, S.emit_arcs);
        float& m = S.L.cpa[S.sorted ? 1 : 0];
        m = m == 0.0f ? x : 0.875f * m + 0.125f * x;
        S.L.n_alpha_seen++;
      }
    }
  }
  // contraction sub-phases are marked inside contract(); this closes the last one
  __device__ __forceinline__ void tick_contract(long long& t0) {
#if WFST_PHASES
    if (threadIdx.x == 0) {
      const long long t1 = clock64();
      S.ph[10] += (u64)(t1 - S.t_mark);
      t0 = t1;
    }
#endif
  }

  __device__ const float* row_ptr(int t) const { return p.ll + ((size_t)t * p.B + S.b) * (size_t)p.P; }

  // t_next < 0: no prefetch of the next frame's row
  __device__ void run_frame(int t, int t_next) {
    const int tid = threadIdx.x;
    if (S.L.frames - S.L.layer_floor >= p.TMAX) {   // the layer index ring is full
      if (tid == 0) S.L.status = WFST_ERR_CAPACITY;
      __syncthreads();
      return;
    }
    long long t0 = clock64();
    const long long t_frame0 = t0;
    if (tid == 0) S.t_cur = t;
#if WFST_ROWSMEM
    if (tid == 0 && !S.row_pending) row_issue(row_ptr(t));   // first frame of a work item
#endif
    begin_frame(INFINITY, true, !WFST_ROWSMEM);   // (row_wait's barrier publishes it)
    tick(t0, 5);
#if WFST_ROWSMEM
    row_wait();
#endif
    tick(t0, 11);
    set_mark();
    expand();
#if WFST_PHASES
    if (tid == 0) t0 = clock64();   // expansion itself is timed by the marks inside expand()
#endif
#ifdef WFST_FRAMECYC
    const long long t_exp = clock64() - t_frame0;
#endif
#if WFST_ROWSMEM
    if (tid == 0 && t_next >= 0) row_issue(row_ptr(t_next));   // overlaps the frame's tail
#endif
    tick(t0, 0);
    // expand() ends with a barrier: the best cost, the claim count and the status are final, so
    // every thread derives the cutoff itself (select_cutoff's barrier publishes thread 0's copies)
    const uint32_t best_o = S.best_ord;
    const bool bad = best_o == 0xFFFFFFFFu || S.status != WFST_OK;
    const float beam_cut = bad ? INFINITY : __fadd_rn(float_of_ord(best_o), p.beam);
    if (bad) {
      __syncthreads();   // every thread has read S.status before thread 0 may set it
      if (tid == 0) {
        if (best_o == 0xFFFFFFFFu && S.status == WFST_OK) S.status = WFST_ERR_NO_SURVIVOR;
        S.n_claim_emit = S.n_claim;
        S.n_surv = 0;
      }
      __syncthreads();
      finish_frame(t, true);   // wipes the tables
      return;
    }
    if (tid == 0) {
      S.n_claim_emit = S.n_claim;
      S.beam_cut = beam_cut;
    }
    select_cutoff(beam_cut);
    tick(t0, 1);
    eps_closure();
    tick(t0, 2);
#ifdef WFST_FRAMECYC
    const long long t_eps = clock64() - t_frame0;
#endif
    set_mark();
    contract();
    tick_contract(t0);
#ifdef WFST_COUNT   // frame cycles split by frame kind: phase[7] alpha-bound frames, phase[9] others
    if (tid == 0) {
      S.ph[7] += S.dbgc[0] + S.dbgc[1];   // (slots reused by this instrumentation build)
      S.ph[9] += S.dbgc[2] + S.dbgc[3];
    }
#endif
    const bool alpha_frame = S.use_alpha != 0;
    finish_frame(t, true);
#ifdef WFST_FRAMECYC   // instrumentation build: the frame's SM cycles replace its epsilon-degree count
    if (tid == 0 && S.L.status == WFST_OK) {   // (and [1] = cycles to the end of the expansion |
                                               //  cycles to the end of the epsilon closure << 32)
      const size_t fi = ((size_t)S.lane * p.TMAX + (S.L.frames - 1) % p.TMAX) * 5;
      p.fcounts[fi + 4] = clock64() - t_frame0;
      p.fcounts[fi + 1] = (long long)(((unsigned long long)t_eps << 32) | (unsigned long long)(uint32_t)t_exp);
    }
#endif
    tick(t0, 5);
    flush_phases(alpha_frame, (u64)(clock64() - t_frame0));
  }
};

template <int BS, int R, int MINB, int AM>
__global__ void __launch_bounds__(BS, MINB) frame_kernel(KParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SmemCtl S;
  __shared__ int s_wbuf[WFST_OWNER_BSEARCH ? 32 : BS];   // owner buffers (head-flag owner map only)
  __shared__ __align__(16) int4 s_stage[(BS / 32) * kStage];
  u64* tab = (u64*)smem_raw;
  int* hist = (int*)(tab + p.C);
  unsigned char* rowmem = (unsigned char*)(hist + kNB);
  const int tid = threadIdx.x;
  const uint32_t tab_sa = saddr(tab);
  for (int i = tid; i < p.C; i += BS) sts64(tab_sa + 8u * i, kEmpty);
  if (!WFST_OWNER_BSEARCH || tid < 32) s_wbuf[tid] = -1;
  if (tid < 12) S.ph[tid] = 0;
  if (tid == 0) {
    S.status = WFST_OK;
    S.row_parity = 0;
    S.row_pending = 0;
    S.row_off = 0;
    mbar_init(saddr(&S.row_mbar), 1);
  }
  __syncthreads();
  static_assert((BS / 32) * kStage * 4 >= kNB, "selection scratch lives in the stage buffers");
  Frame<BS, R, AM> fr(p, S, tab_sa, hist, s_wbuf + (WFST_OWNER_BSEARCH ? 0 : (tid & ~31)), saddr(s_stage + (tid >> 5) * kStage), saddr(rowmem),
                      (int*)s_stage);
  fr.bind_scratch();
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
        fr.run_frame(t, t + 1 < t_end ? t + 1 : -1);
      }
      if (tid == 0 && S.row_pending) {   // a prefetch left unused (lane stopped early)
        mbar_wait(saddr(&S.row_mbar), S.row_parity);
        S.row_parity ^= 1;
        S.row_pending = 0;
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

}  // namespace wfst_dev
