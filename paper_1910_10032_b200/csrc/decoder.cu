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

#include "frame_kernel.cuh"
#include "lattice_kernel.cuh"
#include "partial_kernel.cuh"
#include "gc_kernel.cuh"
#include "wfst_internal.h"

using namespace wfst;
using namespace wfst_dev;

namespace {

// ---------------- best path (row a7; readings R10, R11) ----------------
// One CTA per lane: argmin over the last layer's survivors of (c + F, arc) among final states,
// else of (c, arc); then the traceback: the predecessor of a record {arc, state} is the record
// of src(arc) in the previous layer (emitting arc) or the same layer (epsilon arc), found by a
// CTA-wide scan of that layer's records.  Arcs are written back to front into arcs_out.
#ifndef WFST_BP_THREADS
#define WFST_BP_THREADS 512
#endif
constexpr int kBestPathThreads = WFST_BP_THREADS;   // (<= 1024: s_fin / s_any hold one entry per warp)
constexpr int kPathSmem = 4096;                      // path arcs kept on chip during the walk
__global__ void __launch_bounds__(kBestPathThreads) best_path_kernel(KParams p, const int32_t* __restrict__ olabel, const int32_t* __restrict__ lanes,
                                 int32_t n, int32_t cap, float* cost_out, int32_t* reached_out, int32_t* n_arcs_out,
                                 int32_t* arcs_out, int32_t* olab_out, int32_t* n_olab_out, int32_t* status_out) {
  __shared__ u64 s_fin[32], s_any[32];
  __shared__ int s_idx;
  __shared__ int s_w_arc[3], s_w_src[3], s_w_emit[3], s_w_found[3];
  __shared__ int s_path[kPathSmem];
  __shared__ int s_wsum[kBestPathThreads / 32];
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
  const int64_t lb0 = (uint32_t)L.layer_base % (uint32_t)p.R_cap;   // the last layer's first record (ring)
  auto rix = [&](int i) { const int64_t x = lb0 + i; return x >= p.R_cap ? x - p.R_cap : x; };
  const int2* rec = p.rec + (size_t)lane * p.R_cap;
  const int2* linfo = p.layer_info + (size_t)lane * (p.TMAX + 1);
  u64 kf = kEmpty, ka = kEmpty;
  for (int i = tid; i < L.n_front; i += blockDim.x) {
    const int4 f = __ldcg(Fc + i);
    const float c = __int_as_float(f.y);
    const u64 arc = (uint32_t)__ldcg(&rec[rix(i)].x);  // -1 -> 0xFFFFFFFF sorts last (R9)
    const float F = __int_as_float(__ldg(&p.state_info[f.x].w));
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
    if ((uint32_t)__ldcg(&rec[rix(i)].x) == (uint32_t)kb) s_idx = i;
  __syncthreads();
  if (kb == kEmpty || s_idx < 0) {
    if (tid == 0) {
      status_out[li] = WFST_ERR_NO_SURVIVOR;
      n_arcs_out[li] = 0;
      n_olab_out[li] = 0;
      cost_out[li] = INFINITY;
      reached_out[li] = 0;
    }
    return;
  }
  // ---- walk back.  Step j reads slot j%3 (the record found by step j-1: its arc, the arc's
  // source state and kind), its scan of the source's layer fills slot (j+1)%3 and thread 0 clears
  // slot (j+2)%3, last read in step j-1: one barrier per step.  The path's tokens are cheap and
  // a layer is stored cheapest bins first, so a scan usually ends in its first batch.  The arcs
  // are kept on chip (kPathSmem of them; longer walks also go to arcs_out) and reversed and
  // labelled in parallel at the end.
  int32_t* out = arcs_out + (size_t)li * cap;
  auto load_step = [&](int slot, int arc) {   // (one thread: the record's finder)
    s_w_arc[slot] = arc;
    s_w_found[slot] = 1;
    if (arc >= 0) {
      const int4 a = __ldg(p.arcs + arc);
      s_w_src[slot] = a.w & 0x7FFFFFFF;
      s_w_emit[slot] = a.z >= 0;
    }
  };
  if (tid == 0) {
    cost_out[li] = float_of_ord((uint32_t)(kb >> 32));
    reached_out[li] = reached ? 1 : 0;
    load_step(0, __ldcg(&rec[rix(s_idx)].x));
    s_w_found[1] = 0;
  }
  __syncthreads();
  int len = 0, layer = L.frames, j = 0, nol_far = 0, status = WFST_OK;
  const long long max_steps = (long long)L.rec_used + 2;
  for (; j < max_steps; j++) {
    const int cur = j % 3, nxt = (j + 1) % 3;
    if (!s_w_found[cur]) {   // the previous scan found no record of the source state
      status = WFST_ERR_STATE;   // (broken chain: must not happen)
      break;
    }
    const int arc = s_w_arc[cur];
    if (arc < 0) break;   // the start token
    // traceback GC (row f2): below the settle point the path was already handed out by
    // wfst_get_partial_paths -- stop at the settled root (entered by an emitting arc)
    if (layer == L.layer_floor && L.layer_floor > 0 && s_w_emit[cur]) break;
    if (tid == 0) {
      if (len < cap) out[len] = arc;
      if (len < kPathSmem) s_path[len] = arc;
      else if (__ldg(olabel + arc) != 0) nol_far++;   // counted over the whole walk
      s_w_found[(j + 2) % 3] = 0;
    }
    len++;
    layer -= s_w_emit[cur];
    const int want = s_w_src[cur];
    const int2 info = __ldcg(&linfo[layer % (p.TMAX + 1)]);
    const uint32_t Rc = (uint32_t)p.R_cap, b0 = (uint32_t)info.x % Rc;   // record ring (row f2 GC)
    for (int i0 = 0; i0 < max(info.y, 1); i0 += kBestPathThreads * kPU) {
      int2 r[kPU];
#pragma unroll
      for (int u = 0; u < kPU; u++) {
        const int i = i0 + u * kBestPathThreads + tid;
        const uint32_t x = b0 + (uint32_t)i;
        r[u] = i < info.y ? __ldcg(rec + (x >= Rc ? x - Rc : x)) : make_int2(-3, -1);
      }
      bool found = false;
#pragma unroll
      for (int u = 0; u < kPU; u++)
        if (r[u].y == want && r[u].x != -3) {
          load_step(nxt, r[u].x);
          found = true;
        }
      if (__syncthreads_or(found)) break;   // one decision for the CTA (the finder's writes are visible)
    }
  }
  if (j >= max_steps) status = WFST_ERR_STATE;
  __syncthreads();
  n_arcs_out[li] = len;   // (every thread holds the same len)
  const int m = min(len, cap);
  int nol = 0, nol_all = 0;
  if (m <= kPathSmem) {   // reverse to forward order, olabels compacted in path order
    for (int x0 = 0; x0 < m; x0 += kBestPathThreads) {
      const int x = x0 + tid;
      const int32_t arc = x < m ? s_path[m - 1 - x] : 0;
      const int32_t ol = x < m ? __ldg(olabel + arc) : 0;
      if (x < m) out[x] = arc;
      int e = 0;
      const int tot = block_excl_scan01<kBestPathThreads>(ol != 0, e, s_wsum);
      if (ol != 0) olab_out[(size_t)li * cap + nol + e] = ol;
      nol += tot;
    }
    // olabels of the walk's arcs beyond cap (a truncated path still reports the size it needs)
    for (int x0 = m; x0 < min(len, kPathSmem); x0 += kBestPathThreads) {
      const int x = x0 + tid;
      int e = 0;
      nol_all += block_excl_scan01<kBestPathThreads>(x < min(len, kPathSmem) && __ldg(olabel + s_path[x]) != 0, e,
                                                     s_wsum);
    }
    nol_all += nol;
  } else if (tid == 0) {   // serial fallback (cap and the walk both beyond kPathSmem)
    for (int k = 0; k < m / 2; k++) {
      const int32_t t = out[k];
      out[k] = out[m - 1 - k];
      out[m - 1 - k] = t;
    }
    for (int k = 0; k < m; k++) {
      const int32_t ol = __ldg(olabel + out[k]);
      if (ol != 0) olab_out[(size_t)li * cap + nol++] = ol;
    }
    for (int x = 0; x < kPathSmem; x++) nol_all += __ldg(olabel + s_path[x]) != 0;   // the walk's first arcs
    // (arcs beyond kPathSmem are in nol_far)
  }
  if (tid != 0) return;
  n_olab_out[li] = nol_all + nol_far;   // every olabel of the path, also when the arcs were truncated
  status_out[li] = status != WFST_OK ? status : (len > cap ? WFST_ERR_INVALID_ARG : WFST_OK);
}

}  // namespace

// ---------------- host side ----------------
// kernel variants: (threads per CTA, arcs in flight per lane, resident CTAs per SM)
struct WfstVariant {
  int bs, ctas, am;
  void* fn;
  void (*launch)(int grid, size_t smem, cudaStream_t st, const KParams& kp);
};

struct wfst_decoder_s {
  wfst_graph_t g = nullptr;
  int device = 0;
  int32_t n_lanes = 0;
  float beam = 15.f;
  int32_t alpha = 0;
  wfst_decoder_opts_t o{};
  int32_t C = 0, C_ovf = 0, FCAP = 0, TMAX = 0, row_floats = 0, row_bytes = 0;
  int64_t R_cap = 0;
  int n_sm = 0, threads = 512, ctas_per_sm = 1;
  int n_scratch = 0;   // persistent CTAs (= per-CTA scratch sets)
  int sort_mode = 1, cbuf_cap = 0;   // bin-ordered insertion (opts.insert_order, opts.bin_capacity)
  const WfstVariant* variant = nullptr;
  size_t smem_bytes = 0;
  KParams kp{};
  // device allocations
  LaneState* d_lanes = nullptr;
  void* d_pool = nullptr;
  size_t pool_bytes = 0;
  int32_t* d_qhead = nullptr;
  int32_t* d_round = nullptr;
  int32_t* d_lane_ids = nullptr;   // batch -> lane of the work being enqueued (a slot of the ring)
  // channel -> lane mappings (row f3): a ring of kIdRing device buffers filled from pinned host
  // memory by stream-ordered copies, so a call on a different subset of streams does not
  // synchronise the device; a slot is reused only after the work that read it has finished
  static constexpr int kIdRing = 8;
  int32_t* d_id_ring = nullptr;
  int32_t* h_id_ring = nullptr;
  cudaEvent_t ev_ids[kIdRing] = {};   // after the last work that read the slot
  cudaEvent_t ev_up[kIdRing] = {};    // after the slot's upload
  cudaStream_t ids_stream = nullptr;  // stream of the last call
  int id_slot = 0;
  int32_t* d_path = nullptr;       // best-path scratch
  size_t path_cap = 0;
  static constexpr int kStages = 3;   // host-input staging buffers (copies run ahead of decoding)
  float* d_host_stage[kStages] = {};
  size_t stage_bytes = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[kStages] = {}, ev_use[kStages] = {};
  int2* d_settled = nullptr;        // [lane] last settle point of the partial results (row f2)
  size_t partial_smem = 0;
  size_t gc_smem = 0;               // traceback GC kernel (opts.gc_frames)
  // lattice (row f1)
  bool lattice = false;
  int64_t S_cap = 0;
  int lat_grid = 0;
  size_t lat_smem = 0;
  LatParams lp{};
  float* kp_pslack = nullptr;
  uint32_t* kp_gamma = nullptr;
  int32_t* d_lat_q = nullptr;       // work-queue head of the lattice launch
  int32_t* d_lat_lane = nullptr;    // lane id of the finalize launch
  float* d_lat_out = nullptr;       // finalize outputs {best, reached, status}
  cudaEvent_t ev_lat = nullptr;     // after the last lattice launch (compute stream)
  void* h_lat_stage = nullptr;      // pinned D2H staging
  size_t h_lat_bytes = 0;
  std::vector<int32_t> h_initialized;
  std::vector<int32_t> cur_ids;    // mapping currently in d_lane_ids
  int64_t device_bytes = 0;
  // Stream ordering: every call that enqueues device work first orders its CUDA stream after
  // the decoder's previous work (which shares the scratch, the work queue and the lane states
  // and may have been enqueued on another stream), then records ev_work after its own work.
  // Result calls (best paths, partial paths, stats) run on work_stream and wait for ev_work
  // only -- never for the whole device.
  cudaEvent_t ev_work = nullptr;
  cudaStream_t work_stream = nullptr;
  bool has_work = false;
  int32_t* h_path = nullptr;       // pinned staging of the result calls (path_cap int32)
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

// order stream st after the decoder's previous work (no-op on the same stream)
cudaError_t order_after_previous(wfst_decoder_t d, cudaStream_t st) {
  if (d->has_work && st != d->work_stream) return cudaStreamWaitEvent(st, d->ev_work, 0);
  return cudaSuccess;
}
// st now carries the decoder's latest work
cudaError_t mark_work(wfst_decoder_t d, cudaStream_t st) {
  d->work_stream = st;
  d->has_work = true;
  return cudaEventRecord(d->ev_work, st);
}
// wait for the decoder's work only (and for the copy stream of the lattice / host-input paths)
cudaError_t wait_work(wfst_decoder_t d) {
  cudaError_t e = d->has_work ? cudaEventSynchronize(d->ev_work) : cudaSuccess;
  if (e == cudaSuccess && d->copy_stream) e = cudaStreamSynchronize(d->copy_stream);
  return e;
}
// device -> host copy ordered after the decoder's work, on its stream (no device-wide sync)
cudaError_t d2h(wfst_decoder_t d, void* dst, const void* src, size_t bytes) {
  cudaError_t e = wait_work(d);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, d->work_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(d->work_stream);
  return e;
}
// grow the device + pinned result buffers of the path calls to `need` int32
cudaError_t ensure_path(wfst_decoder_t d, size_t need) {
  if (need <= d->path_cap) return cudaSuccess;
  cudaError_t e = wait_work(d);
  cudaFree(d->d_path);
  if (d->h_path) cudaFreeHost(d->h_path);
  d->d_path = nullptr;
  d->h_path = nullptr;
  d->path_cap = 0;
  if (e == cudaSuccess) e = cudaMalloc(&d->d_path, need * 4);
  // the kernels write each row's used columns only; the D2H copies whole column ranges
  if (e == cudaSuccess) e = cudaMemset(d->d_path, 0, need * 4);
  if (e == cudaSuccess) e = cudaMallocHost(&d->h_path, need * 4);
  if (e == cudaSuccess) d->path_cap = need;
  return e;
}

#ifndef WFST_R1024
#define WFST_R1024 2   // arcs in flight per thread in the default 1024-thread kernel
#endif
template <int BS, int R, int MINB, int AM>
void launch_v(int grid, size_t smem, cudaStream_t st, const KParams& kp) {
  frame_kernel<BS, R, MINB, AM><<<grid, BS, smem, st>>>(kp);
}
#define WFST_VARIANT(BS, R, MINB, AM) {BS, MINB, AM, (void*)frame_kernel<BS, R, MINB, AM>, launch_v<BS, R, MINB, AM>}
const WfstVariant kVariants[] = {
    WFST_VARIANT(512, 4, 1, 0), WFST_VARIANT(256, 4, 1, 0), WFST_VARIANT(1024, WFST_R1024, 1, 0), WFST_VARIANT(256, 4, 2, 0),
    WFST_VARIANT(512, 2, 2, 0), WFST_VARIANT(256, 2, 3, 0), WFST_VARIANT(256, 2, 4, 0),
    WFST_VARIANT(1024, WFST_R1024, 1, 1),   // histogram max-active (row f4): default launch shape only
};
const WfstVariant* find_variant(int bs, int ctas, int am) {
  for (const WfstVariant& v : kVariants)
    if (v.bs == bs && v.ctas == ctas && v.am == am) return &v;
  return nullptr;
}

cudaError_t launch_frames(wfst_decoder_t d, KParams kp, cudaStream_t st) {
  int grid = std::min(kp.n_items, d->n_scratch);
  if (grid <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(kp.q_head, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(kp.lane_round, 0, sizeof(int32_t) * kp.B, st);
  if (e != cudaSuccess) return e;
  d->variant->launch(grid, d->smem_bytes, st, kp);
  return cudaGetLastError();
}

// traceback GC (opts.gc_frames): compact every lane of the current batch (gc_kernel.cuh)
cudaError_t launch_gc(wfst_decoder_t d, int32_t B, cudaStream_t st) {
  GcParams gp{};
  gp.arcs = d->kp.arcs;
  gp.lanes = d->d_lane_ids;
  gp.lanes_st = d->d_lanes;
  gp.rec = d->kp.rec;
  gp.rec_cost = d->kp.rec_cost;
  gp.R_cap = d->R_cap;
  gp.layer_info = d->kp.layer_info;
  gp.TMAX = d->TMAX;
  gp.settled = d->d_settled;
  gp.wcap = 53248 / kGcCtas;   // two (epsilon, emitting) source-set pairs in the SM's shared memory
  const size_t smem = (size_t)gp.wcap * 4;
  if (d->gc_smem != smem) {
    cudaError_t e = cudaFuncSetAttribute(gc_kernel<kGcThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    d->gc_smem = smem;
  }
  gc_kernel<kGcThreads><<<B, kGcThreads, smem, st>>>(gp);
  return cudaGetLastError();
}

// a lane starts a new utterance: its lattice arena and status restart
__global__ void lat_reset_kernel(const int32_t* lanes, int32_t n, unsigned long long* cursor, int32_t* status) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    cursor[lanes[i]] = 0;
    status[lanes[i]] = WFST_OK;
  }
}

// row f2: a lane starts a new utterance: nothing is settled yet
__global__ void settle_reset_kernel(const int32_t* lanes, int32_t n, int2* settled) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) settled[lanes[i]] = make_int2(-1, -1);
}

// row f1: the lattice segments of the layers the last frame-kernel launch produced
cudaError_t launch_lattice(wfst_decoder_t d, const float* ll, int32_t T, int32_t B, int32_t P, int mode,
                           cudaStream_t st) {
  LatParams lp = d->lp;
  lp.ll = ll;
  lp.T = T;
  lp.B = B;
  lp.P = P;
  lp.lanes = d->d_lane_ids;
  lp.mode = mode;
  lp.n_items = mode == kModeInit ? B : T * B;
  lp.q_head = d->d_lat_q;
  cudaError_t e = cudaSuccess;
  if (mode == kModeInit) {
    lat_reset_kernel<<<(B + 255) / 256, 256, 0, st>>>(d->d_lane_ids, B, lp.seg_cursor, lp.lat_status);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(d->d_lat_q, 0, 4, st);
  if (e != cudaSuccess) return e;
  lattice_kernel<kLatBS, kLatCtas><<<std::min(d->lat_grid, lp.n_items), kLatBS, d->lat_smem, st>>>(lp);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventRecord(d->ev_lat, st);
  return e;
}

size_t smem_for(int C, int row_bytes) { return (size_t)C * 8 + (size_t)kNB * 4 + (size_t)row_bytes; }

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
  d->ctas_per_sm = d->o.ctas_per_sm > 0 ? d->o.ctas_per_sm : 1;
  d->n_scratch = d->o.max_ctas > 0 ? d->o.max_ctas : d->n_sm * d->ctas_per_sm;
  d->threads = d->o.threads > 0 ? d->o.threads : (d->ctas_per_sm == 1 ? 1024 : 256);
  if (d->o.ll_columns < 0 || d->o.ll_columns > 1) {
    delete d;
    return fail(WFST_ERR_INVALID_ARG, "opts.ll_columns must be 0 (pdf columns) or 1 (ilabel columns)");
  }
  if (d->o.insert_order < 0 || d->o.insert_order > 2) {
    delete d;
    return fail(WFST_ERR_INVALID_ARG, "insert_order must be 0 (auto), 1 (arrival order) or 2 (bin order)");
  }
  if (d->o.max_active_mode != 0 && d->o.max_active_mode != 1) {
    delete d;
    return fail(WFST_ERR_INVALID_ARG, "max_active_mode must be 0 (exact) or 1 (histogram)");
  }
  d->variant = find_variant(d->threads, d->ctas_per_sm, d->o.max_active_mode);
  if (!d->variant) {
    delete d;
    return fail(WFST_ERR_INVALID_ARG, "unsupported (threads, ctas_per_sm, max_active_mode) combination");
  }
  // on-chip table: what is left of the SM's shared memory per resident CTA
  const size_t static_smem = sizeof(SmemCtl) + (WFST_OWNER_BSEARCH ? 128 : 4 * (size_t)d->threads) +
                             (size_t)(d->threads / 32) * kStage * 16 + 1024;
  const size_t per_cta = std::min((size_t)prop.sharedMemPerBlockOptin,
                                  (size_t)prop.sharedMemPerMultiprocessor / d->ctas_per_sm);
  // the staged log-likelihood row: columns 0..max_pdf (+16 B alignment slack on each side)
  const int row_floats = std::max(g->max_pdf + 1, 1);
#if WFST_ROWSMEM
  const int row_bytes = (row_floats * 4 + 15) / 16 * 16 + 32;
#else
  const int row_bytes = 32;
#endif
  int C = d->o.table_slots > 0 ? d->o.table_slots
                               : (int)((per_cta - static_smem - (size_t)kNB * 4 - (size_t)row_bytes) / 8);
  C = std::max(64, C / 256 * 256);
  while (C > 256 && smem_for(C, row_bytes) + static_smem > per_cta) C -= 256;
  if (smem_for(C, row_bytes) + static_smem > per_cta) {
    delete d;
    return fail(WFST_ERR_INVALID_ARG, "log-likelihood row does not fit in shared memory (too many pdfs)");
  }
  d->row_floats = row_floats;
  d->row_bytes = row_bytes;
  d->C = C;
  // overflow table: room for every distinct candidate a frame can hold beyond the on-chip table
  int Co = d->o.overflow_slots > 0 ? d->o.overflow_slots : std::max(std::max(C, 32768), 4 * d->alpha);
  d->C_ovf = std::max(64, (Co + 7) / 8 * 8);   // FCAP % 8 == 0: frontier buffers are 128-B aligned
  d->FCAP = d->C + d->C_ovf;
  d->TMAX = d->o.max_frames > 0 ? d->o.max_frames : 4096;
  int64_t per_frame = d->alpha > 0 ? std::min<int64_t>((int64_t)d->alpha * 5 / 4 + 1024, d->FCAP) : d->FCAP;
  if (d->o.gc_frames < 0) {
    delete d;
    return fail(WFST_ERR_INVALID_ARG, "opts.gc_frames must be >= 0");
  }
  if (d->o.gc_frames > 0 && d->o.lattice) {
    delete d;
    return fail(WFST_ERR_INVALID_ARG, "opts.gc_frames and opts.lattice are exclusive (the lattice needs every record)");
  }
  if (d->o.records_per_stream > 0) {
    d->R_cap = d->o.records_per_stream;
  } else if (d->o.gc_frames > 0) {
    // traceback GC: a stream holds its live traceback tree plus the records of the frames since
    // the last collection -- gc_frames + 64 frames at the max-active bound
    d->R_cap = (int64_t)(d->o.gc_frames + 64) * per_frame;
  } else {
    // default: ~max_frames/4 frames at the alpha bound, capped to half of the free device memory
    d->R_cap = (int64_t)(d->TMAX / 4 + 1) * per_frame;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      int64_t per_lane_other = (int64_t)d->FCAP * 32 + (int64_t)d->TMAX * 60 +
                               ((int64_t)d->FCAP * (4 + 8 + 8) + (int64_t)d->C_ovf * 8) * d->n_scratch / n_streams;
      int64_t budget = (int64_t)(free_b / 2) / n_streams - per_lane_other;
      // bytes per record: {arc, state} (+ cost with debug_costs or lattice; with lattice also
      // gamma, the state record {e_begin, e_end, eps_end, state} and 2 arena entries of 20 B)
      int64_t per_rec = (int64_t)sizeof(int2) + (d->o.debug_costs || d->o.lattice ? 4 : 0) +
                        (d->o.lattice ? 4 + 16 + 2 * 20 : 0);
      int64_t cap = budget / per_rec;
      if (cap < d->R_cap) d->R_cap = std::max<int64_t>(cap, per_frame);
    }
  }
  if (d->R_cap > INT32_MAX - 1) d->R_cap = INT32_MAX - 1;
  if (d->o.frames_per_item <= 0) d->o.frames_per_item = 16;
  d->smem_bytes = smem_for(d->C, d->row_bytes);
  e = cudaFuncSetAttribute(d->variant->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d->smem_bytes);
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
  // intra-frame scratch (claim list, winner words, overflow table, epsilon worklists) is reset
  // by the end of every frame, so it belongs to the persistent CTA, not to the lane: its
  // working set stays L2-resident however many lanes there are
  const size_t NS = (size_t)d->n_scratch;
  size_t i_claim = add(NS * FC * 4);
  size_t i_win = add(NS * FC * 8);
  size_t i_ovf = add(NS * (size_t)d->C_ovf * 8);
  size_t i_wl = add(NS * 2 * FC * 4);
  // bin-ordered insertion: candidate buffers per CTA and coarse cost bin
  d->sort_mode = d->o.insert_order == 1 ? 0 : d->o.insert_order == 2 ? 2 : 1;
  d->cbuf_cap = d->alpha > 0 && d->sort_mode ? (d->o.bin_capacity > 0 ? d->o.bin_capacity : 8192) : 0;
  d->cbuf_cap = (d->cbuf_cap + 7) / 8 * 8;   // 128-B aligned bins (discarded line by line)
  size_t i_cbuf = d->cbuf_cap ? add(NS * (size_t)kPlace * (size_t)d->cbuf_cap * sizeof(int4)) : (size_t)-1;
  size_t i_rec = add(L * (size_t)d->R_cap * sizeof(int2));
  d->lattice = d->o.lattice != 0;
  if (d->lattice && d->o.reclaim) {
    delete d;
    return fail(WFST_ERR_INVALID_ARG, "opts.lattice and opts.reclaim are exclusive (the lattice needs every layer)");
  }
  if (d->lattice) {
    d->S_cap = d->o.lattice_arcs_per_stream > 0 ? d->o.lattice_arcs_per_stream : 2 * d->R_cap;
    d->S_cap = std::min<int64_t>(d->S_cap, INT32_MAX - 1);   // segment offsets are int32
    if (!(d->o.lattice_beam >= 0.0f)) {
      delete d;
      return fail(WFST_ERR_INVALID_ARG, "lattice_beam must be >= 0 (may be +inf)");
    }
  }
  size_t i_rcost = (d->o.debug_costs || d->lattice) ? add(L * (size_t)d->R_cap * 4) : (size_t)-1;
  size_t i_rsi = d->lattice ? add(L * (size_t)d->R_cap * sizeof(int4)) : (size_t)-1;
  // lattice: arena {arc, src, dst, slack} + path slack per entry, cursor, segment index, status,
  // gamma per record; fallback token maps of the lattice CTAs for layers beyond shared memory
  const size_t NLAT = d->lattice ? (size_t)d->n_sm * kLatCtas : 0;
  const int64_t lat_gcap = 2 * (int64_t)d->FCAP + 32;
  size_t i_seg = d->lattice ? add(L * (size_t)d->S_cap * sizeof(int4)) : 0;
  size_t i_psl = d->lattice ? add(L * (size_t)d->S_cap * 4) : 0;
  size_t i_scur = d->lattice ? add(L * 8) : 0;
  size_t i_sidx = d->lattice ? add(L * (size_t)(d->TMAX + 1) * sizeof(int2)) : 0;
  size_t i_lst = d->lattice ? add(L * 4) : 0;
  size_t i_gam = d->lattice ? add(L * (size_t)d->R_cap * 4) : 0;
  size_t i_gtab = d->lattice ? add(NLAT * (size_t)lat_gcap * 8) : 0;
  size_t i_gcnt = d->lattice ? add(NLAT * (size_t)d->FCAP * 4) : 0;
  const int64_t lat_stage = 4 * (int64_t)d->FCAP;
  size_t i_gstg = d->lattice ? add(NLAT * (size_t)lat_stage * sizeof(int4)) : 0;
  size_t i_fst = add(L * (size_t)d->TMAX * 3 * 4);
  size_t i_fcn = add(L * (size_t)d->TMAX * 5 * 8);
  size_t i_linfo = add(L * (size_t)(d->TMAX + 1) * sizeof(int2));
  e = cudaMalloc(&d->d_pool, total);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_lanes, sizeof(LaneState) * L);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_qhead, 4);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_round, 4 * L);
  if (e == cudaSuccess) e = cudaMalloc(&d->d_id_ring, 4 * L * wfst_decoder_s::kIdRing);
  if (e == cudaSuccess) e = cudaMallocHost(&d->h_id_ring, 4 * L * wfst_decoder_s::kIdRing);
  for (int k = 0; k < wfst_decoder_s::kIdRing && e == cudaSuccess; k++)
    e = cudaEventCreateWithFlags(&d->ev_ids[k], cudaEventDisableTiming);
  for (int k = 0; k < wfst_decoder_s::kIdRing && e == cudaSuccess; k++)
    e = cudaEventCreateWithFlags(&d->ev_up[k], cudaEventDisableTiming);
  if (e == cudaSuccess) d->d_lane_ids = d->d_id_ring;
  if (e == cudaSuccess) e = cudaMalloc(&d->d_settled, sizeof(int2) * L);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_work, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMemset(d->d_settled, 0xFF, sizeof(int2) * L);
  if (e != cudaSuccess) {
    cudaFree(d->d_pool);
    cudaFree(d->d_lanes);
    cudaFree(d->d_qhead);
    cudaFree(d->d_round);
    cudaFree(d->d_id_ring);
    cudaFreeHost(d->h_id_ring);
    delete d;
    return cuda_fail(e, "decoder allocation");
  }
  d->pool_bytes = total;
  char* base = (char*)d->d_pool;
  KParams& kp = d->kp;
  kp.state_info = g->d_state;
  kp.arcs = g->d_arcs;
  kp.start = g->start;
  kp.row_floats = d->row_floats;
  kp.row_bytes = d->row_bytes;
  kp.n_states = g->Q;
  kp.beam = beam;
  kp.alpha = d->alpha;
  kp.C = d->C;
  kp.NBK = d->C / kBucket;
  kp.C_ovf = d->C_ovf;
  kp.FCAP = d->FCAP;
  kp.R_cap = d->R_cap;
  kp.TMAX = d->TMAX;
  kp.lanes_st = d->d_lanes;
  kp.front = (int4*)(base + parts[i_front].off);
  kp.claim = (uint32_t*)(base + parts[i_claim].off);
  kp.win = (u64*)(base + parts[i_win].off);
  kp.ovf = (u64*)(base + parts[i_ovf].off);
  kp.wl = (uint32_t*)(base + parts[i_wl].off);
  kp.rec = (int2*)(base + parts[i_rec].off);
  kp.rec_cost = i_rcost != (size_t)-1 ? (float*)(base + parts[i_rcost].off) : nullptr;
  kp.rec_si = i_rsi != (size_t)-1 ? (int4*)(base + parts[i_rsi].off) : nullptr;
  kp.fstats = (float*)(base + parts[i_fst].off);
  kp.fcounts = (long long*)(base + parts[i_fcn].off);
  kp.layer_info = (int2*)(base + parts[i_linfo].off);
  kp.cbuf = i_cbuf != (size_t)-1 ? (int4*)(base + parts[i_cbuf].off) : nullptr;
  kp.cbuf_cap = d->cbuf_cap;
  kp.sort_mode = d->sort_mode;
  kp.q_head = d->d_qhead;
  kp.lane_round = d->d_round;
  if (d->lattice) {
    LatParams& lp = d->lp;
    lp.state_info = g->d_state;
    lp.arcs = g->d_arcs;
    lp.beam = beam;
    lp.lattice_beam = d->o.lattice_beam;
    lp.lanes_st = d->d_lanes;
    lp.rec = kp.rec;
    lp.rec_cost = kp.rec_cost;
    lp.rec_si = kp.rec_si;
    lp.R_cap = d->R_cap;
    lp.layer_info = kp.layer_info;
    lp.TMAX = d->TMAX;
    lp.fstats = kp.fstats;
    lp.seg = (int4*)(base + parts[i_seg].off);
    lp.S_cap = d->S_cap;
    lp.seg_cursor = (unsigned long long*)(base + parts[i_scur].off);
    lp.seg_index = (int2*)(base + parts[i_sidx].off);
    lp.lat_status = (int32_t*)(base + parts[i_lst].off);
    lp.g_tab = (u64*)(base + parts[i_gtab].off);
    lp.g_cnt = (int32_t*)(base + parts[i_gcnt].off);
    lp.g_cap = (int32_t)lat_gcap;
    lp.g_stage = (int4*)(base + parts[i_gstg].off);
    lp.stage_cap = (int32_t)lat_stage;
    lp.FCAP = d->FCAP;
    d->lat_grid = (int)NLAT;
    d->lat_smem = std::min((size_t)prop.sharedMemPerBlockOptin, (size_t)(220 / kLatCtas) * 1024);
    lp.smem_bytes = (int32_t)d->lat_smem;
    d->kp_pslack = (float*)(base + parts[i_psl].off);
    d->kp_gamma = (uint32_t*)(base + parts[i_gam].off);
    e = cudaFuncSetAttribute(lattice_kernel<kLatBS, kLatCtas>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)d->lat_smem);
    if (e == cudaSuccess) e = cudaMalloc(&d->d_lat_q, 4);
    if (e == cudaSuccess) e = cudaMalloc(&d->d_lat_lane, 4);
    if (e == cudaSuccess) e = cudaMalloc(&d->d_lat_out, 16);
    if (e == cudaSuccess) e = cudaMemset(d->d_lat_out, 0, 16);   // {best, reached, status, unused}
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_lat, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMemset(lp.seg_cursor, 0, L * 8);
    if (e == cudaSuccess) e = cudaMemset(lp.lat_status, 0, L * 4);
    if (e != cudaSuccess) {
      wfst_decoder_destroy(d);
      return cuda_fail(e, "lattice allocation");
    }
  }
  e = cudaMemset(base + parts[i_ovf].off, 0xFF, parts[i_ovf].bytes);
  if (e == cudaSuccess) e = cudaMemset(base + parts[i_win].off, 0xFF, parts[i_win].bytes);
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
  wait_work(d);
  if (d->ev_work) cudaEventDestroy(d->ev_work);
  if (d->h_path) cudaFreeHost(d->h_path);
  cudaFree(d->d_pool);
  cudaFree(d->d_lanes);
  cudaFree(d->d_qhead);
  cudaFree(d->d_round);
  cudaFree(d->d_id_ring);
  if (d->h_id_ring) cudaFreeHost(d->h_id_ring);
  for (int k = 0; k < wfst_decoder_s::kIdRing; k++)
    if (d->ev_ids[k]) cudaEventDestroy(d->ev_ids[k]);
  for (int k = 0; k < wfst_decoder_s::kIdRing; k++)
    if (d->ev_up[k]) cudaEventDestroy(d->ev_up[k]);
  cudaFree(d->d_path);
  cudaFree(d->d_host_stage[0]);
  cudaFree(d->d_host_stage[1]);
  cudaFree(d->d_settled);
  cudaFree(d->d_lat_q);
  cudaFree(d->d_lat_lane);
  cudaFree(d->d_lat_out);
  if (d->ev_lat) cudaEventDestroy(d->ev_lat);
  if (d->h_lat_stage) cudaFreeHost(d->h_lat_stage);
  if (d->copy_stream) cudaStreamDestroy(d->copy_stream);
  for (int i = 0; i < wfst_decoder_s::kStages; i++) {
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
  if (ids == d->cur_ids) {   // same mapping as the work already queued
    if (st != d->ids_stream) {   // another stream: order it after the slot's upload
      cudaError_t e = cudaStreamWaitEvent(st, d->ev_up[d->id_slot], 0);
      if (e != cudaSuccess) return cuda_fail(e, "lane ids event");
      d->ids_stream = st;
    }
    return WFST_OK;
  }
  // next ring slot: wait only for the (old) work that read it, then a stream-ordered upload
  const int k = (d->id_slot + 1) % wfst_decoder_s::kIdRing;
  cudaError_t e = cudaEventSynchronize(d->ev_ids[k]);
  int32_t* h = d->h_id_ring + (size_t)k * d->n_lanes;
  int32_t* dv = d->d_id_ring + (size_t)k * d->n_lanes;
  if (e == cudaSuccess) {
    memcpy(h, ids.data(), 4 * (size_t)B);
    e = cudaMemcpyAsync(dv, h, 4 * (size_t)B, cudaMemcpyHostToDevice, st);
  }
  if (e == cudaSuccess) e = cudaEventRecord(d->ev_up[k], st);
  if (e != cudaSuccess) return cuda_fail(e, "lane ids upload");
  d->id_slot = k;
  d->d_lane_ids = dv;
  d->cur_ids = ids;
  d->ids_stream = st;
  return WFST_OK;
}

wfst_status wfst_decoder_reset(wfst_decoder_t d, const int32_t* streams, int32_t n, void* cuda_stream) {
  if (!d) return fail(WFST_ERR_INVALID_ARG, "NULL decoder");
  DeviceGuard dg(d->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int32_t B = streams ? n : d->n_lanes;
  if (B <= 0) return WFST_OK;
  cudaError_t eo = order_after_previous(d, st);
  if (eo != cudaSuccess) return cuda_fail(eo, "stream order");
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
  settle_reset_kernel<<<(B + 255) / 256, 256, 0, st>>>(d->d_lane_ids, B, d->d_settled);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = launch_frames(d, kp, st);
  if (e != cudaSuccess) return cuda_fail(e, "reset launch");
  if (d->lattice) {
    e = launch_lattice(d, nullptr, 0, B, 0, kModeInit, st);
    if (e != cudaSuccess) return cuda_fail(e, "lattice launch");
  }
  for (int32_t i = 0; i < B; i++) d->h_initialized[streams ? streams[i] : i] = 1;
  e = cudaEventRecord(d->ev_ids[d->id_slot], st);   // the slot is free once this work is done
  if (e == cudaSuccess) e = mark_work(d, st);
  return e == cudaSuccess ? WFST_OK : cuda_fail(e, "event");
}

wfst_status wfst_decode_frames(wfst_decoder_t d, const float* d_loglikes, int32_t T, int32_t B, int32_t P,
                               const int32_t* streams, void* cuda_stream) {
  if (!d) return fail(WFST_ERR_INVALID_ARG, "NULL decoder");
  if (T < 0 || B < 0) return fail(WFST_ERR_INVALID_ARG, "negative size");
  if (T == 0 || B == 0) return WFST_OK;
  if (!d_loglikes) return fail(WFST_ERR_INVALID_ARG, "NULL loglikes");
  if (B > d->n_lanes) return fail(WFST_ERR_INVALID_ARG, "B exceeds n_streams");
  // ll_columns = 1 (SPEC layout): column ilabel = column pdf + 1, so the rows are read from one
  // column in (the stride stays P) and the last column read is max_pdf + 1
  const int32_t col0 = d->o.ll_columns == 1 ? 1 : 0;
  if (P <= d->g->max_pdf + col0)
    return fail(WFST_ERR_PDF_RANGE, "P=" + std::to_string(P) + " too small for max pdf " + std::to_string(d->g->max_pdf) +
                                        (col0 ? " with ilabel columns (P >= max ilabel + 1)" : " (P > max pdf)"));
  d_loglikes += col0;
  DeviceGuard dg(d->device);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  cudaError_t eo = order_after_previous(d, st);
  if (eo != cudaSuccess) return cuda_fail(eo, "stream order");
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
  // traceback GC: the frames run in launches of at most gc_frames frames, each followed by a
  // compaction of the batch's records (stream-ordered, no host synchronisation)
  const int32_t G = d->o.gc_frames > 0 ? d->o.gc_frames : T;
  cudaError_t e = cudaSuccess;
  for (int32_t t0 = 0; t0 < T && e == cudaSuccess; t0 += G) {
    KParams kq = kp;
    kq.T = std::min(G, T - t0);
    kq.ll = d_loglikes + (size_t)t0 * B * P;
    kq.K = std::min(K, kq.T);
    long long items = (long long)((kq.T + kq.K - 1) / kq.K) * B;
    if (items > INT32_MAX) return fail(WFST_ERR_INVALID_ARG, "too many work items");
    kq.n_items = (int32_t)items;
    e = launch_frames(d, kq, st);
    if (e == cudaSuccess && d->o.gc_frames > 0) e = launch_gc(d, B, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "decode launch");
  if (d->lattice) {
    e = launch_lattice(d, d_loglikes, T, B, P, kModeFrames, st);
    if (e != cudaSuccess) return cuda_fail(e, "lattice launch");
  }
  e = cudaEventRecord(d->ev_ids[d->id_slot], st);   // the slot is free once this work is done
  if (e == cudaSuccess) e = mark_work(d, st);
  return e == cudaSuccess ? WFST_OK : cuda_fail(e, "event");
}

static cudaError_t ensure_copy_stream(wfst_decoder_t d) {
  cudaError_t e = cudaSuccess;
  if (!d->copy_stream) {
    e = cudaStreamCreateWithFlags(&d->copy_stream, cudaStreamNonBlocking);
    for (int i = 0; i < wfst_decoder_s::kStages && e == cudaSuccess; i++) {
      e = cudaEventCreateWithFlags(&d->ev_copy[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_use[i], cudaEventDisableTiming);
    }
  }
  return e;
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
  // the staging buffers below are then free once earlier work of ANY stream is done
  cudaError_t e = order_after_previous(d, st);
  if (e != cudaSuccess) return cuda_fail(e, "stream order");
  if (need > d->stage_bytes) {
    wait_work(d);
    cudaStreamSynchronize(st);
    for (int i = 0; i < wfst_decoder_s::kStages; i++) {
      cudaFree(d->d_host_stage[i]);
      d->d_host_stage[i] = nullptr;
    }
    d->stage_bytes = 0;
    for (int i = 0; i < wfst_decoder_s::kStages && e == cudaSuccess; i++) e = cudaMalloc(&d->d_host_stage[i], need);
    if (e != cudaSuccess) return cuda_fail(e, "staging allocation");
    d->stage_bytes = need;
  }
  e = ensure_copy_stream(d);
  if (e != cudaSuccess) return cuda_fail(e, "copy stream");
  // the staging buffers may still be read by earlier work on st
  for (int i = 0; i < wfst_decoder_s::kStages && e == cudaSuccess; i++) e = cudaEventRecord(d->ev_use[i], st);
  if (e != cudaSuccess) return cuda_fail(e, "event");
  int k = 0;
  // chunk schedule: a short first chunk (decoding starts after a fifth of a chunk's copy) and a
  // short last one (little decoding left once the last copy lands); full chunks in between
  std::vector<int32_t> sizes;
  {
    const int32_t small = std::max(1, CF / 5);
    int32_t rem = T;
    if (rem > CF + small) {
      sizes.push_back(small);
      rem -= small;
    }
    while (rem > CF + small) {
      sizes.push_back(CF);
      rem -= CF;
    }
    if (rem > CF) {
      sizes.push_back(rem - small);
      rem = small;
    }
    if (rem > 0) sizes.push_back(rem);
  }
  int32_t t0 = 0;
  for (size_t ci = 0; ci < sizes.size(); t0 += sizes[ci], ci++, k = (k + 1) % wfst_decoder_s::kStages) {
    int32_t n = sizes[ci];
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
  std::vector<LaneState> L(d->n_lanes);
  cudaError_t e = d2h(d, L.data(), d->d_lanes, sizeof(LaneState) * d->n_lanes);
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
  cudaError_t e = d2h(d, &L, d->d_lanes + stream, sizeof L);
  if (e != cudaSuccess) return cuda_fail(e, "lane state");
  if (!d->h_initialized[stream]) return WFST_ERR_STATE;
  return (wfst_status)L.status;
}

wfst_status wfst_get_best_paths_ex(wfst_decoder_t d, const int32_t* streams, int32_t n, float* cost,
                                   int32_t* reached_final, int32_t* arcs, int32_t* olabels, int32_t arcs_cap,
                                   int32_t* n_arcs, int32_t* n_olabels, int32_t* status) {
  if (!d || n < 0 || !cost || !reached_final || !n_arcs) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  if (n == 0) return WFST_OK;
  DeviceGuard dg(d->device);
  if (arcs_cap < 0) arcs_cap = 0;
  for (int i = 0; i < n; i++) {
    int32_t s = streams ? streams[i] : i;
    if (s < 0 || s >= d->n_lanes) return fail(WFST_ERR_INVALID_ARG, "stream id out of range");
    if (!d->h_initialized[s]) return fail(WFST_ERR_STATE, "stream " + std::to_string(s) + " not reset");
  }
  int cap = std::max(arcs_cap, 1);
  cudaError_t e = ensure_path(d, (size_t)n * (6 + 2 * (size_t)cap));
  if (e != cudaSuccess) return cuda_fail(e, "path buffer");
  // on the decoder's work stream, after its last decode: only this decoder's work is awaited
  cudaStream_t st = d->work_stream;
  int32_t* p = d->d_path;
  int32_t* h = d->h_path;
  int32_t* d_ids = p;
  float* d_cost = (float*)(p + n);
  int32_t* d_reached = p + 2 * n;
  int32_t* d_nar = p + 3 * n;
  int32_t* d_nol = p + 4 * n;
  int32_t* d_st = p + 5 * n;
  int32_t* d_arcs = p + 6 * n;
  int32_t* d_ol = d_arcs + (size_t)n * cap;
  for (int i = 0; i < n; i++) h[i] = streams ? streams[i] : i;
  e = cudaMemcpyAsync(d_ids, h, 4 * (size_t)n, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "ids");
  best_path_kernel<<<n, kBestPathThreads, 0, st>>>(d->kp, d->g->d_olabel, d_ids, n, cap, d_cost, d_reached, d_nar,
                                                   d_arcs, d_ol, d_nol, d_st);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, p, 4 * 6 * (size_t)n, cudaMemcpyDeviceToHost, st);
  // only the columns some stream used (a path is ~T arcs, cap is an upper bound)
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "best path kernel");
  int mx_a = 0, mx_o = 0;
  for (int i = 0; i < n; i++) {
    mx_a = std::max(mx_a, std::min(h[3 * n + i], cap));
    mx_o = std::max(mx_o, std::min(h[4 * n + i], cap));
  }
  int32_t* h_arcs = h + 6 * n;
  int32_t* h_ol = h_arcs + (size_t)n * cap;
  const size_t pitch = 4 * (size_t)cap;
  if (arcs && arcs_cap > 0 && mx_a > 0)
    e = cudaMemcpy2DAsync(h_arcs, pitch, d_arcs, pitch, 4 * (size_t)mx_a, n, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && olabels && arcs_cap > 0 && mx_o > 0)
    e = cudaMemcpy2DAsync(h_ol, pitch, d_ol, pitch, 4 * (size_t)mx_o, n, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "path D2H");
  if (arcs && arcs_cap > 0 && mx_a > 0)
    for (int i = 0; i < n; i++) memcpy(arcs + (size_t)i * cap, h_arcs + (size_t)i * cap, 4 * (size_t)mx_a);
  if (olabels && arcs_cap > 0 && mx_o > 0)
    for (int i = 0; i < n; i++) memcpy(olabels + (size_t)i * cap, h_ol + (size_t)i * cap, 4 * (size_t)mx_o);
  wfst_status first = WFST_OK;
  for (int i = 0; i < n; i++) {
    memcpy(&cost[i], &h[n + i], 4);
    reached_final[i] = h[2 * n + i];
    n_arcs[i] = h[3 * n + i];
    if (n_olabels) n_olabels[i] = h[4 * n + i];
    wfst_status s = (wfst_status)h[5 * n + i];
    if (status) status[i] = s;
    if (s != WFST_OK && first == WFST_OK) {
      first = s;
      set_error("stream " + std::to_string(streams ? streams[i] : i) + ": " + wfst_status_string(s));
    }
  }
  return first;
}

wfst_status wfst_get_best_paths(wfst_decoder_t d, const int32_t* streams, int32_t n, float* cost,
                                int32_t* reached_final, int32_t* arcs, int32_t* olabels, int32_t arcs_cap,
                                int32_t* n_arcs, int32_t* n_olabels) {
  return wfst_get_best_paths_ex(d, streams, n, cost, reached_final, arcs, olabels, arcs_cap, n_arcs, n_olabels,
                                nullptr);
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
  cudaError_t e = d2h(d, L.data(), d->d_lanes, sizeof(LaneState) * d->n_lanes);
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
    s->records_used_max = std::max<int64_t>(s->records_used_max, x.rec_peak);
    for (int k = 0; k < 12; k++) s->phase_cycles[k] += (int64_t)x.phase[k];
    for (int k = 0; k < 12; k++) s->phase_cycles_alpha[k] += (int64_t)x.phase_alpha[k];
    s->select_entries += (int64_t)x.sel_entries;
  }
  s->device_bytes = d->device_bytes;
  s->records_per_stream = d->R_cap;
  s->record_bytes = (int64_t)d->n_lanes * d->R_cap * (int64_t)(sizeof(int2) + (d->kp.rec_cost ? 4 : 0) +
                                                               (d->kp.rec_si ? sizeof(int4) : 0));
  return WFST_OK;
}

wfst_status wfst_decoder_reset_stats(wfst_decoder_t d) {
  if (!d) return fail(WFST_ERR_INVALID_ARG, "NULL decoder");
  DeviceGuard dg(d->device);
  std::vector<LaneState> L(d->n_lanes);
  cudaError_t e = d2h(d, L.data(), d->d_lanes, sizeof(LaneState) * d->n_lanes);
  if (e != cudaSuccess) return cuda_fail(e, "stats");
  for (auto& x : L) {
    x.emit_arcs = x.eps_arcs = x.eps_relax = x.cand = x.surv = x.ovf = x.alpha_frames = x.frames_total = 0;
    x.sel_entries = 0;
    for (int k = 0; k < 12; k++) x.phase[k] = x.phase_alpha[k] = 0;
  }
  e = cudaMemcpyAsync(d->d_lanes, L.data(), sizeof(LaneState) * d->n_lanes, cudaMemcpyHostToDevice, d->work_stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(d->work_stream);
  return e == cudaSuccess ? WFST_OK : cuda_fail(e, "stats");
}

wfst_status wfst_decoder_frame_stats(wfst_decoder_t d, int32_t stream, float* fstats, int64_t* fcounts,
                                     int32_t cap_frames, int32_t* n_frames) {
  if (!d || stream < 0 || stream >= d->n_lanes || !n_frames) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  DeviceGuard dg(d->device);
  LaneState L;
  cudaError_t e = d2h(d, &L, d->d_lanes + stream, sizeof L);
  if (e != cudaSuccess) return cuda_fail(e, "frame stats");
  int n = std::min(std::min(L.frames, d->TMAX), std::max(cap_frames, 0));
  *n_frames = std::min(L.frames, d->TMAX);
  if (fstats && n > 0) e = d2h(d, fstats, d->kp.fstats + (size_t)stream * d->TMAX * 3, sizeof(float) * 3 * n);
  if (e == cudaSuccess && fcounts && n > 0)
    e = d2h(d, fcounts, d->kp.fcounts + (size_t)stream * d->TMAX * 5, sizeof(int64_t) * 5 * n);
  return e == cudaSuccess ? WFST_OK : cuda_fail(e, "frame stats");
}

wfst_status wfst_debug_layer(wfst_decoder_t d, int32_t stream, int32_t layer, int32_t* states, int32_t* arcs,
                             float* costs, int32_t cap, int32_t* n) {
  if (!d || stream < 0 || stream >= d->n_lanes || !n || layer < 0) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  if (layer > d->TMAX) return fail(WFST_ERR_INVALID_ARG, "layer beyond max_frames");
  DeviceGuard dg(d->device);
  LaneState L;
  cudaError_t e = d2h(d, &L, d->d_lanes + stream, sizeof L);
  if (e != cudaSuccess) return cuda_fail(e, "debug layer");
  if (layer > L.frames) return fail(WFST_ERR_INVALID_ARG, "layer not decoded yet");
  if (layer < L.layer_floor || L.frames - layer > d->TMAX) return fail(WFST_ERR_INVALID_ARG, "layer reclaimed");
  int2 info;
  e = d2h(d, &info, d->kp.layer_info + (size_t)stream * (d->TMAX + 1) + layer % (d->TMAX + 1), sizeof info);
  if (e != cudaSuccess) return cuda_fail(e, "debug layer");
  *n = info.y;
  if (info.y > cap) return fail(WFST_ERR_INVALID_ARG, "capacity too small");
  std::vector<int2> r(info.y);
  std::vector<float> c(info.y, NAN);
  if (info.y > 0) {
    // the layer's records may wrap around the end of the record ring
    const int64_t r0 = (int64_t)info.x % d->R_cap, n1 = std::min<int64_t>(info.y, d->R_cap - r0);
    const size_t lb = (size_t)stream * d->R_cap;
    e = d2h(d, r.data(), d->kp.rec + lb + r0, sizeof(int2) * n1);
    if (e == cudaSuccess && n1 < info.y) e = d2h(d, r.data() + n1, d->kp.rec + lb, sizeof(int2) * (info.y - n1));
    if (e == cudaSuccess && d->kp.rec_cost) e = d2h(d, c.data(), d->kp.rec_cost + lb + r0, 4 * (size_t)n1);
    if (e == cudaSuccess && d->kp.rec_cost && n1 < info.y)
      e = d2h(d, c.data() + n1, d->kp.rec_cost + lb, 4 * (size_t)(info.y - n1));
    if (e != cudaSuccess) return cuda_fail(e, "debug layer");
  }
  for (int i = 0; i < info.y; i++) {
    int32_t a = r[i].x;
    if (states) states[i] = r[i].y;
    if (arcs) arcs[i] = a;
    if (costs) costs[i] = c[i];
  }
  return WFST_OK;
}

wfst_status wfst_get_lattice(wfst_decoder_t d, int32_t stream, int32_t* seg_n, int32_t layers_cap,
                             int32_t* n_layers, int32_t* arc, int32_t* src, int32_t* dst, float* slack,
                             float* pslack, int64_t arcs_cap, int64_t* n_arcs, float* gamma, int64_t gamma_cap,
                             int64_t* n_tokens, float* best, int32_t* reached_final) {
  if (!d || stream < 0 || stream >= d->n_lanes || !n_layers || !n_arcs || !best || !reached_final)
    return fail(WFST_ERR_INVALID_ARG, "bad argument");
  if (!d->lattice) return fail(WFST_ERR_INVALID_ARG, "decoder created without opts.lattice");
  if (!d->h_initialized[stream]) return fail(WFST_ERR_STATE, "stream not reset");
  DeviceGuard dg(d->device);
  cudaError_t e = ensure_copy_stream(d);
  cudaStream_t cs = d->copy_stream;
  // the backward sweep and the copies run on the copy stream after the lane's last lattice
  // launch; the compute stream is left running
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, d->ev_lat, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d->d_lat_lane, &stream, 4, cudaMemcpyHostToDevice, cs);
  LatFinParams fp{};
  fp.state_info = d->lp.state_info;
  fp.arcs = d->lp.arcs;
  fp.lanes = d->d_lat_lane;
  fp.lanes_st = d->d_lanes;
  fp.rec = d->kp.rec;
  fp.rec_cost = d->kp.rec_cost;
  fp.R_cap = d->R_cap;
  fp.layer_info = d->kp.layer_info;
  fp.TMAX = d->TMAX;
  fp.seg = d->lp.seg;
  fp.S_cap = d->S_cap;
  fp.seg_index = d->lp.seg_index;
  fp.gamma = d->kp_gamma;
  fp.pslack = d->kp_pslack;
  fp.best_out = d->d_lat_out;
  fp.reached_out = (int32_t*)(d->d_lat_out + 1);
  fp.status_out = (int32_t*)(d->d_lat_out + 2);
  fp.lat_status = d->lp.lat_status;
  if (e == cudaSuccess) {
    lattice_final_kernel<1024><<<1, 1024, 0, cs>>>(fp);
    e = cudaGetLastError();
  }
  auto stage = [&](size_t bytes) -> cudaError_t {
    if (bytes <= d->h_lat_bytes) return cudaSuccess;
    cudaError_t x = cudaStreamSynchronize(cs);
    if (d->h_lat_stage) cudaFreeHost(d->h_lat_stage);
    d->h_lat_stage = nullptr;
    d->h_lat_bytes = 0;
    if (x == cudaSuccess) x = cudaMallocHost(&d->h_lat_stage, bytes);
    if (x == cudaSuccess) d->h_lat_bytes = bytes;
    return x;
  };
  struct Head { LaneState L; float out[4]; unsigned long long cursor; };
  if (e == cudaSuccess) e = stage(std::max(sizeof(Head), (size_t)1 << 20));
  Head* h = (Head*)d->h_lat_stage;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h->L, d->d_lanes + stream, sizeof(LaneState), cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->out, d->d_lat_out, 16, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h->cursor, d->lp.seg_cursor + stream, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(e, "lattice finalize");
  const Head H = *h;
  int32_t st_out;
  memcpy(&st_out, &H.out[2], 4);
  if (st_out != WFST_OK)
    return fail((wfst_status)st_out, "stream " + std::to_string(stream) + ": lattice " +
                                         wfst_status_string((wfst_status)st_out));
  const int T = H.L.frames;
  const int64_t n_tok = H.L.rec_used;
  const int64_t n_used = (int64_t)H.cursor;
  *best = H.out[0];
  memcpy(reached_final, &H.out[1], 4);
  *n_layers = T + 1;
  if (n_tokens) *n_tokens = n_tok;
  // layer index, arena and gamma in one staging buffer
  const size_t o_sidx = 0, o_lay = o_sidx + 8 * (size_t)(T + 1), o_seg = o_lay + 8 * (size_t)(T + 1);
  const size_t o_psl = o_seg + 16 * (size_t)n_used, o_gam = o_psl + 4 * (size_t)n_used;
  const size_t total = o_gam + 4 * (size_t)n_tok;
  e = stage(total);
  char* hb = (char*)d->h_lat_stage;
  const size_t lo = (size_t)stream * (d->TMAX + 1);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(hb + o_sidx, d->lp.seg_index + lo, 8 * (size_t)(T + 1), cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(hb + o_lay, d->kp.layer_info + lo, 8 * (size_t)(T + 1), cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess && n_used)
    e = cudaMemcpyAsync(hb + o_seg, d->lp.seg + (size_t)stream * d->S_cap, 16 * (size_t)n_used,
                        cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess && n_used)
    e = cudaMemcpyAsync(hb + o_psl, d->kp_pslack + (size_t)stream * d->S_cap, 4 * (size_t)n_used,
                        cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess && n_tok)
    e = cudaMemcpyAsync(hb + o_gam, d->kp_gamma + (size_t)stream * d->R_cap, 4 * (size_t)n_tok,
                        cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(e, "lattice D2H");
  const int2* sidx = (const int2*)(hb + o_sidx);
  const int4* sg = (const int4*)(hb + o_seg);
  const float* ps = (const float*)(hb + o_psl);
  int64_t n = 0;
  for (int k = 0; k <= T; k++) n += sidx[k].y;
  *n_arcs = n;
  if ((seg_n && T + 1 > layers_cap) || n > arcs_cap || (gamma && n_tok > gamma_cap))
    return fail(WFST_ERR_INVALID_ARG, "lattice output capacity too small");
  // segments in layer order (the arena is filled in completion order)
  int64_t m = 0;
  for (int k = 0; k <= T; k++) {
    if (seg_n) seg_n[k] = sidx[k].y;
    for (int i = 0; i < sidx[k].y; i++, m++) {
      const int4 v = sg[sidx[k].x + i];
      if (arc) arc[m] = v.x;
      if (src) src[m] = v.y;
      if (dst) dst[m] = v.z;
      if (slack) memcpy(&slack[m], &v.w, 4);
      if (pslack) pslack[m] = ps[sidx[k].x + i];
    }
  }
  if (gamma && n_tok) memcpy(gamma, hb + o_gam, 4 * (size_t)n_tok);
  return WFST_OK;
}

constexpr int kTraceThreads = 256, kTraceMinBlocks = 6;

wfst_status wfst_get_partial_paths_packed(wfst_decoder_t d, const int32_t* streams, int32_t n, int32_t* arcs,
                                          int32_t* olabels, int64_t total_cap, int32_t cap, int64_t* offsets,
                                          int64_t* total_out, int32_t* n_arcs, int32_t* n_olabels,
                                          int32_t* settled_frames, int32_t* status) {
  if (!d || n < 0 || !n_arcs || !settled_frames || cap < 0) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  if ((arcs || olabels) && (!offsets || total_cap < (int64_t)n * cap))
    return fail(WFST_ERR_INVALID_ARG, "packed partial paths: offsets needed and total_cap >= n * cap");
  if (total_out) *total_out = 0;
  for (int i = 0; i < n; i++) {   // (a call that fails before the results reports nothing)
    n_arcs[i] = 0;
    if (n_olabels) n_olabels[i] = 0;
    if (offsets) offsets[i] = 0;
  }
  if (n == 0) return WFST_OK;
  DeviceGuard dg(d->device);
  for (int i = 0; i < n; i++) {
    int32_t s = streams ? streams[i] : i;
    if (s < 0 || s >= d->n_lanes) return fail(WFST_ERR_INVALID_ARG, "stream id out of range");
    if (!d->h_initialized[s]) return fail(WFST_ERR_STATE, "stream " + std::to_string(s) + " not reset");
  }
  const int cp = std::max(cap, 1);
  cudaError_t e = ensure_path(d, (size_t)n * (6 + 3 * (size_t)cp) + 1);
  if (e != cudaSuccess) return cuda_fail(e, "path buffer");
  cudaStream_t st = d->work_stream;   // after the decoder's last decode, on its stream
  int32_t* p = d->d_path;
  int32_t* h = d->h_path;
  PartialParams pp{};
  pp.arcs = d->kp.arcs;
  pp.olabel = d->g->d_olabel;
  pp.lanes = p;
  pp.lanes_st = d->d_lanes;
  pp.rec = d->kp.rec;
  pp.R_cap = d->R_cap;
  pp.layer_info = d->kp.layer_info;
  pp.TMAX = d->TMAX;
  pp.settled = d->d_settled;
  pp.reclaim = d->o.reclaim;
  pp.lanes_rw = d->d_lanes;
  pp.cap = cp;
  pp.n_arcs_out = p + n;
  pp.n_olab_out = p + 2 * n;
  pp.layer_out = p + 3 * n;
  pp.status_out = p + 4 * n;
  pp.root_out = p + 5 * n;
  pp.arcs_out = p + 6 * n;
  pp.packed_arcs = pp.arcs_out + (size_t)n * cp;
  pp.packed_olab = pp.packed_arcs + (size_t)n * cp;
  pp.packed_count = pp.packed_olab + (size_t)n * cp;
  // shared memory: a set of wanted source states (1.5 slots per token) + one flag per token
  pp.wcap = 24576;   // 1.5 x fcap: two 512-thread CTAs per SM fit in shared memory
  pp.fcap = 16384;
  const size_t smem = (size_t)pp.wcap * 4 + (size_t)pp.fcap;
  if (d->partial_smem != smem) {
    e = cudaFuncSetAttribute(partial_root_kernel<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "partial kernel attribute");
    d->partial_smem = smem;
  }
  for (int i = 0; i < n; i++) h[i] = streams ? streams[i] : i;
  e = cudaMemcpyAsync(p, h, 4 * (size_t)n, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(pp.packed_count, 0, 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "ids");
  // the walk back to the new settle point needs the shared sets (two 512-thread CTAs per SM);
  // the trace of the newly settled arcs needs none and runs as 256-thread CTAs, several per SM
  partial_root_kernel<512, 2><<<n, 512, smem, st>>>(pp);
  partial_trace_kernel<kTraceThreads, kTraceMinBlocks><<<n, kTraceThreads, 0, st>>>(pp);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = mark_work(d, st);   // the kernel may move the lanes' reclaim floors
  // per stream {n_arcs, n_olabels, settled layer, status, packed offset} and the packed total
  const size_t hp_tot = 6 * (size_t)n + 3 * (size_t)n * cp;
  if (e == cudaSuccess) e = cudaMemcpyAsync(h + n, p + n, 4 * 5 * (size_t)n, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h + hp_tot, pp.packed_count, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "partial kernel");
  const size_t total = (size_t)h[hp_tot];
  if (total_out) *total_out = (int64_t)total;
  // straight into the caller's buffers (pageable memory is staged by the driver)
  if (total > 0 && arcs && cap > 0)
    e = cudaMemcpyAsync(arcs, pp.packed_arcs, 4 * total, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess && total > 0 && olabels && cap > 0)
    e = cudaMemcpyAsync(olabels, pp.packed_olab, 4 * total, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "partial D2H");
  if (offsets)
    for (int i = 0; i < n; i++) offsets[i] = h[5 * n + i];
  wfst_status first = WFST_OK;
  for (int i = 0; i < n; i++) {
    n_arcs[i] = h[n + i];
    if (n_olabels) n_olabels[i] = h[2 * n + i];
    settled_frames[i] = h[3 * n + i];
    wfst_status s = (wfst_status)h[4 * n + i];
    if (status) status[i] = s;
    if (s != WFST_OK && first == WFST_OK) {
      first = s;
      set_error("stream " + std::to_string(streams ? streams[i] : i) + ": " + wfst_status_string(s));
    }
  }
  return first;
}

wfst_status wfst_get_partial_paths_ex(wfst_decoder_t d, const int32_t* streams, int32_t n, int32_t* arcs,
                                      int32_t* olabels, int32_t cap, int32_t* n_arcs, int32_t* n_olabels,
                                      int32_t* settled_frames, int32_t* status) {
  if (!d || n < 0 || !n_arcs || !settled_frames || cap < 0) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  // the packed call, then each stream's range into its row
  const size_t tc = (size_t)n * (size_t)std::max(cap, 0);
  std::vector<int32_t> pa(arcs && cap > 0 ? tc : 0), po(olabels && cap > 0 ? tc : 0);
  std::vector<int64_t> off(n);
  std::vector<int32_t> nol(n);
  wfst_status r = wfst_get_partial_paths_packed(d, streams, n, pa.empty() ? nullptr : pa.data(),
                                                po.empty() ? nullptr : po.data(), (int64_t)tc, cap, off.data(),
                                                nullptr, n_arcs, nol.data(), settled_frames, status);
  for (int i = 0; i < n; i++) {
    if (n_olabels) n_olabels[i] = nol[i];
    const int na = std::max(0, std::min(n_arcs[i], cap)), no = std::max(0, std::min(nol[i], cap));
    if (!pa.empty() && na) memcpy(arcs + (size_t)i * cap, pa.data() + off[i], 4 * (size_t)na);
    if (!po.empty() && no) memcpy(olabels + (size_t)i * cap, po.data() + off[i], 4 * (size_t)no);
  }
  return r;
}

wfst_status wfst_get_partial_paths(wfst_decoder_t d, const int32_t* streams, int32_t n, int32_t* arcs,
                                   int32_t* olabels, int32_t cap, int32_t* n_arcs, int32_t* n_olabels,
                                   int32_t* settled_frames) {
  return wfst_get_partial_paths_ex(d, streams, n, arcs, olabels, cap, n_arcs, n_olabels, settled_frames, nullptr);
}

}  // extern "C"
