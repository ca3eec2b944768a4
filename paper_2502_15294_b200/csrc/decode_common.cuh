// Shared machinery of the pipelined decode kernels (decode_bulk.cu: CUDA-core
// consumers for fp32 KV; decode_mma.cu: tensor-core consumers for bf16 KV):
// mbarrier / bulk-copy / PDL wrappers and the work-segment partition.
#pragma once

#include "decode_bulk.cuh"

namespace rk {

constexpr int kConsumerWarps = 8;
constexpr int kBulkThreads = (kConsumerWarps + 1) * 32;
constexpr int kStages = 3;
constexpr int kStageBytes = 32768;   // per operand (K or V) per stage (CUDA-core kernel)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32)); }


__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + C, fp32 accumulate
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}

constexpr int kMaxBatch = 512;

// Work segments of one CTA.  Uniform mode: the key ranges of all dialogues are
// concatenated (length W) and CTA c owns [c*W/N, (c+1)*W/N) — one wave, equal
// work per SM whatever the batch — split at dialogue boundaries.  Item mode:
// CTA (x, b) owns item x of dialogue b (round-aligned, for fused scoring).
struct Seg {
  int b, lo, hi;
};

struct SegTable {
  int pref[kMaxBatch + 1];
  Seg seg[kMaxBatch];
  int nseg;
};

// all threads of the CTA call this; returns after a __syncthreads
__device__ inline void compute_segments(const BulkParams& p, SegTable& t) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool append = p.k_new != nullptr;
  if (p.items) {
    if (threadIdx.x == 0) {
      const int b = blockIdx.y, x = blockIdx.x;
      t.nseg = 0;
      if (x < p.n_items[b]) {
        const int32_t* it = p.items + ((size_t)b * p.items_stride + x) * 3;
        const int len = p.seq_len[b] + (append ? 1 : 0);
        t.seg[0] = Seg{b, it[0], min((int)it[1], len)};
        t.nseg = 1;
      }
    }
  } else {
    for (int i = threadIdx.x; i < p.B; i += blockDim.x) t.pref[i + 1] = p.seq_len[i] + (append ? 1 : 0);
    __syncthreads();
    if (warp == 0) {          // inclusive scan of the lengths
      int carry = 0;
      for (int base = 0; base < p.B; base += 32) {
        int v = (base + lane < p.B) ? t.pref[base + lane + 1] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (base + lane < p.B) t.pref[base + lane + 1] = v + carry;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
      if (lane == 0) t.pref[0] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t W = t.pref[p.B], N = gridDim.x, c = blockIdx.x;
      const int r0 = (int)(c * W / N), r1 = (int)((c + 1) * W / N);
      int n = 0;
      int lo = 0, hi = p.B;                    // first b with pref[b+1] > r0
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (t.pref[mid + 1] > r0) hi = mid; else lo = mid + 1;
      }
      for (int b = lo; b < p.B && t.pref[b] < r1; ++b) {
        const int a0 = max(r0, t.pref[b]) - t.pref[b], a1 = min(r1, t.pref[b + 1]) - t.pref[b];
        if (a0 < a1) t.seg[n++] = Seg{b, a0, a1};
      }
      t.nseg = n;
    }
  }
  __syncthreads();
}

}  // namespace rk
