// Synthetic log-likelihood generator: the device twin of paper_1910_10032_b200/inputs.py
// loglikes_stream().  Input generation only -- no decoding arithmetic lives here.
//   key = (stream << 40) | (t << 20) | p ; h = mix((key ^ mix(seed + G)) + G)
//   u0 = (h >> 41) * 2^-23 ; u1 = ((h >> 18) & (2^23-1)) * 2^-23
//   L  = fl(fl(fl(u0 + u1) - 1) * s) + (p == planted[t][b] ? boost : 0),  s = fl32(sigma * sqrt 6)
#include <cmath>

#include "wfst_internal.h"

namespace {

constexpr unsigned long long kGold = 0x9E3779B97F4A7C15ull;

__host__ __device__ inline unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_kernel(float* __restrict__ out, int32_t T, int32_t B, int32_t P,
                             const int32_t* __restrict__ sid, int32_t t0, unsigned long long sw,
                             const int32_t* __restrict__ planted, float scale, float boost) {
  const long long n = (long long)T * B * P;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int32_t p = (int32_t)(i % P);
    long long tb = i / P;
    int32_t b = (int32_t)(tb % B);
    int32_t t = (int32_t)(tb / B);
    unsigned long long key = ((unsigned long long)(uint32_t)sid[b] << 40) |
                             ((unsigned long long)(uint32_t)(t0 + t) << 20) | (unsigned long long)p;
    unsigned long long h = mix64((key ^ sw) + kGold);
    float u0 = __fmul_rn(__uint2float_rn((uint32_t)(h >> 41)), 1.1920928955078125e-07f);
    float u1 = __fmul_rn(__uint2float_rn((uint32_t)((h >> 18) & 0x7FFFFFull)), 1.1920928955078125e-07f);
    float x = __fmul_rn(__fsub_rn(__fadd_rn(u0, u1), 1.0f), scale);
    float bb = (planted && planted[(long long)t * B + b] == p) ? boost : 0.0f;
    out[i] = __fadd_rn(x, bb);
  }
}

}  // namespace

extern "C" wfst_status wfst_synth_loglikes(float* d_out, int32_t T, int32_t B, int32_t P,
                                           const int32_t* d_stream_ids, int32_t t0, uint64_t seed,
                                           const int32_t* d_planted, float sigma, float boost,
                                           void* cuda_stream) {
  if (T < 0 || B < 0 || P <= 0 || P >= (1 << 20) || t0 < 0 || t0 + T >= (1 << 20))
    return wfst::fail(WFST_ERR_INVALID_ARG, "synth: bad sizes");
  if ((long long)T * B == 0) return WFST_OK;
  if (!d_out || !d_stream_ids) return wfst::fail(WFST_ERR_INVALID_ARG, "synth: NULL pointer");
  unsigned long long sw = mix64((unsigned long long)seed + kGold);
  float scale = (float)((double)sigma * std::sqrt(6.0));
  long long n = (long long)T * B * P;
  long long blocks = (n + 255) / 256;
  if (blocks > 148LL * 64) blocks = 148LL * 64;
  synth_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)cuda_stream>>>(d_out, T, B, P, d_stream_ids, t0,
                                                                       sw, d_planted, scale, boost);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? WFST_OK : wfst::cuda_fail(e, "synth launch");
}
