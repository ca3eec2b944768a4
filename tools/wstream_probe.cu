// Weight-stream probe for the projection kernels: G CTAs (one per SM) each
// stream a contiguous share of a 512 MB buffer (HBM, not L2) through a ring of
// S stages of 16 KB, either as plain cp.async.bulk copies (mode 0) or as 2-D
// TMA tensor boxes {64 bf16, 128 rows} over the same bytes viewed as
// [rows][128 B] (mode 1, no swizzle: the smem image is byte-identical).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wsp tools/wstream_probe.cu -lcuda && /tmp/wsp
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

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

constexpr int CHUNK = 16384;

__global__ void probe(const uint8_t* src, const __grid_constant__ CUtensorMap map, size_t total, int stages, int mode,
                      int split, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * CHUNK);
  uint64_t* empty = full + stages;
  const size_t per = total / gridDim.x / CHUNK * CHUNK;
  const size_t off = per * blockIdx.x;
  const int n = (int)(per / CHUNK);
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
      bar_expect(&full[s], CHUNK);
      const size_t g = off + (size_t)i * CHUNK;
      if (mode >= 2) {
        // `mode` interleaved streams: copy i comes from stream i % mode, each stream a
        // contiguous 1/mode of this CTA's share (same bytes, more DRAM locality spread)
        const int per_stream = n / mode;
        const size_t gs = off + ((size_t)(i % mode) * per_stream + i / mode) * CHUNK;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
            ::"r"(sa(sm + (size_t)s * CHUNK)), "l"(src + gs), "r"(CHUNK), "r"(sa(&full[s])), "l"(pol) : "memory");
      } else if (mode == 0) {
        const int part = CHUNK / split;
        for (int k = 0; k < split; ++k)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
              ::"r"(sa(sm + (size_t)s * CHUNK + k * part)), "l"(src + g + k * part), "r"(part), "r"(sa(&full[s])),
                "l"(pol) : "memory");
      } else {
        const int rows = 128 / split;
        for (int k = 0; k < split; ++k)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1, {%2, %3}], [%4], %5;"
              ::"r"(sa(sm + (size_t)s * CHUNK + k * rows * 128)), "l"(&map), "r"(0), "r"((int)(g / 128) + k * rows),
                "r"(sa(&full[s])), "l"(pol) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      bar_wait(&full[s], (i / stages) & 1);
      acc += sm[(size_t)s * CHUNK + (i & 63)];
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
  CUtensorMap maps[3];
  for (int i = 0; i < 3; ++i) {
    const int split = 1 << i;
    cuuint64_t dims[2] = {64, total / 128};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)(128 / split)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&maps[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int g : {64, 96, 128, sms})
    for (int mode : {0, 1, 2, 4, 8})
      for (int split : {1, 2, 4})
        for (int stages : {6, 11}) {
          if ((mode != 0 && mode != 1) && split != 1) continue;
          if (mode == 1 && split != 1) continue;
          const size_t smem = (size_t)stages * CHUNK + 2 * stages * 8;
          probe<<<g, 64, smem>>>(buf, maps[split == 1 ? 0 : split == 2 ? 1 : 2], total, stages, mode, split, sink);
          cudaEventRecord(a);
          for (int r = 0; r < 5; ++r)
            probe<<<g, 64, smem>>>(buf, maps[split == 1 ? 0 : split == 2 ? 1 : 2], total, stages, mode, split, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms = 0;
          cudaEventElapsedTime(&ms, a, b);
          const double moved = 5.0 * (double)(total / g / CHUNK * CHUNK) * g;
          printf("ctas %4d %s x%d streams %d stages %2d: %7.1f GB/s  (%.1f GB/s per SM)\n", g,
                 mode == 1 ? "tensor" : "bulk  ", split, mode >= 2 ? mode : 1,
                 stages, moved / (ms * 1e-3) / 1e9, moved / (ms * 1e-3) / 1e9 / g);
        }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
