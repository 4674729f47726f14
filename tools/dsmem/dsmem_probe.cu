// DSMEM probe (design evidence for DESIGN.md §10): what a token-table insert costs when the table
// is split over a 2-CTA cluster (the peer SM's shared memory through DSMEM) vs the CTA's own
// shared memory.  Throughput: every thread of every CTA issues dependent-free atomic mins on
// random 8-B slots of the local or the peer table; latency: one thread, a dependent chain.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dsmem_probe dsmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kSlots = 22528;   // the frame kernel's on-chip table (~176 KB of 8-B slots)

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ uint32_t atom_min_cl(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cluster.min.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t atom_min_cta(uint32_t a, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.min.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// mode 0: own table (atom.shared), mode 1: own table through the cluster window, mode 2: peer's
template <int MODE, bool CHAIN>
__global__ void __cluster_dims__(2, 1, 1) probe(int iters, unsigned long long* cycles, uint32_t* sink) {
  extern __shared__ uint64_t tab[];
  for (int i = threadIdx.x; i < kSlots; i += blockDim.x) tab[i] = ~0ull;
  cluster_sync();
  const uint32_t me = cta_rank(), peer = me ^ 1u;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  const uint32_t tbase = MODE == 0 ? base : mapa(base, MODE == 1 ? me : peer);
  uint32_t acc = 0, x = hash(blockIdx.x * 1024 + threadIdx.x);
  const long long t0 = clock64();
  if (!CHAIN || threadIdx.x == 0) {
#pragma unroll 4
    for (int i = 0; i < iters; i++) {
      x = hash(x + (CHAIN ? acc : 0));
      const uint32_t a = tbase + 8u * (x % kSlots) + 4u;
      acc += MODE == 0 ? atom_min_cta(a, x) : atom_min_cl(a, x);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  cluster_sync();
  if (threadIdx.x == 0) atomicAdd(cycles, (unsigned long long)(t1 - t0));
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int MODE, bool CHAIN>
void run(const char* name, int ctas, int threads, int iters) {
  unsigned long long* d_cyc;
  uint32_t* d_sink;
  cudaMalloc(&d_cyc, 8);
  cudaMalloc(&d_sink, 4);
  const size_t smem = (size_t)kSlots * 8;
  cudaFuncSetAttribute(probe<MODE, CHAIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; rep++) {
    cudaMemset(d_cyc, 0, 8);
    cudaEventRecord(a);
    probe<MODE, CHAIN><<<ctas, threads, smem>>>(iters, d_cyc, d_sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  const double ops = CHAIN ? (double)ctas * iters : (double)ctas * threads * iters;
  const double cyc_per_cta = (double)cyc / ctas;
  if (CHAIN)
    printf("%-34s latency %.1f cycles per dependent atomic   [%s]\n", name, cyc_per_cta / iters, cudaGetErrorString(e));
  else
    printf("%-34s %.2f G atomics/s total, %.2f atomics/cycle/SM   [%s]\n", name, ops / (ms * 1e6),
           ops / ctas / cyc_per_cta, cudaGetErrorString(e));
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = (sms / 2) * 2;
  printf("SMs %d, CTAs %d (clusters of 2), table %d slots per CTA\n", sms, ctas, kSlots);
  run<0, false>("own table, atom.shared", ctas, 1024, 4096);
  run<1, false>("own table via cluster window", ctas, 1024, 4096);
  run<2, false>("peer table (DSMEM)", ctas, 1024, 4096);
  run<0, true>("own table, atom.shared", ctas, 1024, 4096);
  run<1, true>("own table via cluster window", ctas, 1024, 4096);
  run<2, true>("peer table (DSMEM)", ctas, 1024, 4096);
  return 0;
}
