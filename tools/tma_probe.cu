// TMA load-rate probe (tools only, not part of librk): one CTA per SM streams
// key tiles of a [keys][row_elems] bf16 tensor into a STAGES-deep smem ring
// with (a) 2-D tensor-map boxes {64 elems, box_rows} (SWIZZLE_128B, the
// prefill/scoring kernels' pattern) or (b) 1-D cp.async.bulk of contiguous
// spans; a consumer warp only waits and frees.  Prints GB/s (whole chip) so
// the per-SM TMA service rate for 128-byte rows can be compared with bulk.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_probe.cu -lcuda -o /tmp/tma_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(sa(dst)), "l"(map), "r"(c0), "r"(c1), "r"(sa(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(bar))
               : "memory");
}

constexpr int STAGES = 8;

// mode 0: tensor boxes {64, box_rows} x boxes_per_tile (column offsets 64*i);
// mode 1: bulk copies of `span` contiguous bytes x boxes_per_tile
__global__ void probe(const __grid_constant__ CUtensorMap map, const uint8_t* base, int mode, int box_rows,
                      int boxes_per_tile, int span, int tiles, int keys, int row_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tile_bytes = mode == 0 ? boxes_per_tile * box_rows * 128 : boxes_per_tile * span;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * tile_bytes);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int rows_per_tile = mode == 0 ? box_rows : 0;
  if (threadIdx.x == 0) {
    for (int t = 0; t < tiles; ++t) {
      const int s = t % STAGES;
      if (t >= STAGES) bar_wait(&empty[s], ((t / STAGES) - 1) & 1);
      bar_expect(&full[s], tile_bytes);
      uint8_t* dst = smem + s * tile_bytes;
      if (mode == 0) {
        const int row0 = (int)(((int64_t)(blockIdx.x * 7919 + t) * rows_per_tile) % (keys - rows_per_tile));
        for (int i = 0; i < boxes_per_tile; ++i) tma_2d(dst + i * box_rows * 128, &map, 64 * i, row0, &full[s]);
      } else {
        const int64_t off = ((int64_t)(blockIdx.x * 7919 + t) * tile_bytes) % ((int64_t)keys * row_bytes - tile_bytes);
        for (int i = 0; i < boxes_per_tile; ++i) bulk_1d(dst + i * span, base + (off & ~15ll) + i * span, span, &full[s]);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int t = 0; t < tiles; ++t) {
      const int s = t % STAGES;
      bar_wait(&full[s], (t / STAGES) & 1);
      bar_arrive(&empty[s]);
    }
  }
  __syncthreads();
}

int main() {
  const int keys = 66048, row_elems = 512;   // [keys][4 heads x 128] bf16, as C3's K
  const int row_bytes = row_elems * 2;
  uint8_t* dev;
  cudaMalloc(&dev, (size_t)keys * row_bytes);
  cudaMemset(dev, 0, (size_t)keys * row_bytes);
  cudaDriverEntryPointQueryResult q;
  void* fp = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int mode, box_rows, boxes, span; const char* name; };
  std::vector<Cfg> cfgs = {
      {0, 64, 2, 0, "tensor box {64,64} x2 (prefill K tile, 16 KB)"},
      {0, 64, 4, 0, "tensor box {64,64} x4 (32 KB)"},
      {0, 128, 2, 0, "tensor box {64,128} x2 (score_tc K tile, 32 KB)"},
      {0, 256, 2, 0, "tensor box {64,256} x2 (64 KB)"},
      {1, 0, 1, 16384, "bulk 16 KB contiguous"},
      {1, 0, 16, 1024, "bulk 16 x 1 KB rows"},
      {1, 0, 64, 256, "bulk 64 x 256 B"},
  };
  for (auto& c : cfgs) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)row_elems, (cuuint64_t)keys};
    cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {64, (cuuint32_t)(c.box_rows ? c.box_rows : 64)};
    cuuint32_t estr[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dev, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int tile_bytes = c.mode == 0 ? c.boxes * c.box_rows * 128 : c.boxes * c.span;
    const size_t smem = (size_t)STAGES * tile_bytes + 256;
    if (smem > 232448) { printf("%-50s skip (smem)\n", c.name); continue; }
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int tiles = (int)(((size_t)2 << 30) / sms / tile_bytes);     // ~2 GB total
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      probe<<<sms, 64, smem>>>(map, dev, c.mode, c.box_rows, c.boxes, c.span, tiles, keys, row_bytes);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)sms * tiles * tile_bytes;
    printf("%-50s %8.1f GB/s  (%.1f B/clk/SM @1.9GHz)  err=%s\n", c.name, bytes / ms / 1e6,
           bytes / ms / 1e6 / sms / 1.9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
