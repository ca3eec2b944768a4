// Streaming-rate probe for the projection kernels' weight path: G CTAs (one
// per SM) each stream a contiguous share of a buffer through a ring of S
// stages of B bytes with cp.async.bulk (one issuing thread, mbarrier
// complete_tx, consumer = one warp that waits and frees the stage).  Prints
// GB/s for each (CTAs, stages, copy bytes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulk_probe tools/bulk_probe.cu && /tmp/bulk_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
               ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}

__global__ void probe(const uint8_t* src, size_t total, int stages, int chunk, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
  uint64_t* empty = full + stages;
  const size_t per = total / gridDim.x / chunk * chunk;
  const uint8_t* base = src + per * blockIdx.x;
  const int n = (int)(per / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      if (i >= stages) bar_wait(&empty[s], ((i / stages) - 1) & 1);
      bar_expect(&full[s], chunk);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
          ::"r"(sa(sm + (size_t)s * chunk)), "l"(base + (size_t)i * chunk), "r"(chunk), "r"(sa(&full[s])), "l"(pol)
          : "memory");
    }
  } else if (threadIdx.x == 32) {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      bar_wait(&full[s], (i / stages) & 1);
      acc += sm[(size_t)s * chunk + (i & 63)];
      bar_arrive(&empty[s]);
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

int main() {
  const size_t total = 512ull << 20;
  uint8_t* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, total);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grids[] = {64, 96, 128, sms, 2 * sms};
  const int chunks[] = {8192, 16384, 32768};
  for (int g : grids)
    for (int chunk : chunks)
      for (int stages : {4, 8, 12}) {
        const size_t smem = (size_t)stages * chunk + 2 * stages * 8;
        if (smem > 220 * 1024) continue;
        if (g > sms && smem > 110 * 1024) continue;
        probe<<<g, 64, smem>>>(buf, total, stages, chunk, sink);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) probe<<<g, 64, smem>>>(buf, total, stages, chunk, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double moved = 5.0 * (double)(total / g / chunk * chunk) * g;
        printf("ctas %4d chunk %6d stages %2d: %7.1f GB/s  (%.1f GB/s per CTA)\n", g, chunk, stages,
               moved / (ms * 1e-3) / 1e9, moved / (ms * 1e-3) / 1e9 / g);
      }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
