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
__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(sa(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(sa(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(bar))
               : "memory");
}

constexpr int STAGES = 6;   // 192 KB in flight (the cluster decode ring: 3 stages x K+V 32 KB)

// mode 2: 3-D boxes {64, box_rows, 2} (dims: 64 elems, keys, 64-elem column
//         blocks; both halves of a kv-head in one instruction) x boxes_per_tile;
// mode 0: tensor boxes {64, box_rows} x boxes_per_tile (column offsets 64*i);
// mode 1: bulk copies of `span` contiguous bytes x boxes_per_tile
__global__ void probe(const __grid_constant__ CUtensorMap map, const uint8_t* base, int mode, int box_rows,
                      int boxes_per_tile, int span, int tiles, int keys, int row_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tile_bytes = mode == 0 ? boxes_per_tile * box_rows * 128
                       : mode == 2 ? boxes_per_tile * box_rows * 256 : boxes_per_tile * span;
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
  const int rows_per_tile = mode != 1 ? box_rows : 0;
  if (threadIdx.x == 0) {
    for (int t = 0; t < tiles; ++t) {
      const int s = t % STAGES;
      if (t >= STAGES) bar_wait(&empty[s], ((t / STAGES) - 1) & 1);
      bar_expect(&full[s], tile_bytes);
      uint8_t* dst = smem + s * tile_bytes;
      if (mode == 0) {
        // head-slice pattern of the cluster decode: this CTA's kv-head (128 of the row's
        // 1024 elements) as two 64-column boxes per key group, consecutive key groups
        const int span = rows_per_tile * boxes_per_tile / 2;
        const int row0 = (int)(((int64_t)(blockIdx.x / 8 * 7919 + t) * span) % (keys - span));
        const int col = (blockIdx.x % 8) * 128;
        for (int i = 0; i < boxes_per_tile; ++i)
          tma_2d(dst + i * box_rows * 128, &map, col + 64 * (i & 1), row0 + (i >> 1) * box_rows, &full[s]);
      } else if (mode == 2) {
        const int span = rows_per_tile * boxes_per_tile;
        const int row0 = (int)(((int64_t)(blockIdx.x / 8 * 7919 + t) * span) % (keys - span));
        for (int i = 0; i < boxes_per_tile; ++i)
          tma_3d(dst + i * box_rows * 256, &map, 0, row0 + i * box_rows, 2 * (blockIdx.x % 8), &full[s]);
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
  const int keys = 66048, row_elems = 1024;  // [keys][8 heads x 128] bf16, as C2's K
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
      {0, 16, 16, 0, "tensor box {64,16} x16 (32 KB; cluster decode)"},
      {0, 32, 8, 0, "tensor box {64,32} x8 (32 KB)"},
      {0, 64, 4, 0, "tensor box {64,64} x4 (32 KB)"},
      {0, 128, 2, 0, "tensor box {64,128} x2 (32 KB)"},
      {0, 256, 1, 0, "tensor box {64,256} x1 (32 KB)"},
      {2, 64, 2, 0, "3d box {64,64,2} x2 (32 KB)"},
      {2, 128, 1, 0, "3d box {64,128,2} x1 (32 KB; cluster decode stage)"},
      {2, 16, 8, 0, "3d box {64,16,2} x8 (32 KB)"},
      {1, 0, 8, 4096, "bulk 8 x 4 KB"},
      {1, 0, 32, 1024, "bulk 32 x 1 KB rows"},
      {1, 0, 128, 256, "bulk 128 x 256 B"},
  };
  const int grids[2] = {sms, 128};
  for (int gi = 0; gi < 2; ++gi)
  for (auto& c : cfgs) {
    const int grid = grids[gi];
    CUtensorMap map;
    CUresult er;
    if (c.mode == 2) {   // dims {64 elems, keys, column blocks}: strides {row, 128 B} (not monotonic)
      cuuint64_t dims[3] = {64, (cuuint64_t)keys, (cuuint64_t)(row_elems / 64)};
      cuuint64_t strides[2] = {(cuuint64_t)row_bytes, 128};
      cuuint32_t box[3] = {64, (cuuint32_t)c.box_rows, 2};
      cuuint32_t estr[3] = {1, 1, 1};
      er = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, dev, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[2] = {(cuuint64_t)row_elems, (cuuint64_t)keys};
      cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
      cuuint32_t box[2] = {64, (cuuint32_t)(c.box_rows ? c.box_rows : 64)};
      cuuint32_t estr[2] = {1, 1};
      er = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dev, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (er != CUDA_SUCCESS) { printf("%-50s encode failed (%d)\n", c.name, (int)er); continue; }
    const int tile_bytes = c.mode == 0 ? c.boxes * c.box_rows * 128
                         : c.mode == 2 ? c.boxes * c.box_rows * 256 : c.boxes * c.span;
    const size_t smem = (size_t)STAGES * tile_bytes + 256;
    if (smem > 232448) { printf("%-50s skip (smem)\n", c.name); continue; }
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int tiles = (int)(((size_t)2 << 30) / grid / tile_bytes);     // ~2 GB total
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      probe<<<grid, 64, smem>>>(map, dev, c.mode, c.box_rows, c.boxes, c.span, tiles, keys, row_bytes);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)grid * tiles * tile_bytes;
    printf("grid %3d %-46s %8.1f GB/s  (%.1f B/clk/SM @1.9GHz)  err=%s\n", grid, c.name, bytes / ms / 1e6,
           bytes / ms / 1e6 / grid / 1.9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
