// Small-batch decode attention: one thread-block cluster per (dialogue,
// kv-head), the split-K merge done in distributed shared memory.
//
// At a few dialogues the persistent split-K decode (decode_mma.cu) spends more
// time on its fixed per-layer chain (decode grid -> partials in global memory
// -> merge kernel) than on streaming the ~9 MB of a kept-rounds layer.  Here
// the C CTAs of a cluster split one (dialogue b, kv-head h) key range
// [0, len) into C contiguous slices and combine their (m, l, acc) partials
// over DSMEM, so a layer is ONE kernel with no workspace:
//   warp 8      producer: one lane issues 2-D TMA boxes {64 dims, 128 keys}
//               (128-byte swizzle) of head h's K and V columns — 256-byte
//               pieces of the token-major [S][HKV][D] rows, gathered by the
//               tensor unit instead of one bulk copy per key — into a 3-stage
//               ring (full/empty mbarriers); the box, not the byte count, is
//               the TMA's unit of work (tools/tma_probe.cu: {64,16} boxes
//               stream 18 B/clk/SM, {64,128} 36 B/clk/SM);
//   warps 0..7  consumers: warp w owns the 16-key group w of each stage; the
//               math is decode_mma's (mma.sync m16n8k16, q and P split into
//               bf16 hi/lo rows so the products carry ~16 mantissa bits, lazy
//               rescale), with swizzled ldmatrix addresses;
//   epilogue    warps -> CTA partial, pushed with st.async into the inbox of
//               the CTA that finalises each (query head, dim) output (CTA rank
//               r owns a contiguous 1/C of them); the stores count their bytes
//               on the owner's inbox mbarrier, so each CTA just waits for its
//               inbox and reduces it locally (no remote loads, no closing
//               cluster barrier).
// The appended token (k_new/v_new) is written into the cache row len-1 by the
// producer of the slice that owns it, before its TMA reads that row
// (fence.proxy.async orders the generic stores before the async-proxy loads).
// Semantics = rk_decode_attention's uniform mode (pipeline.py:298-313 ->
// engine.py:244-267 with one question row; kernel contract _attn_ext.pyx:20-81).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "decode_common.cuh"
#include "tc_common.cuh"

namespace rk {
namespace {

// 8 consumer warps + 1 producer, 3 stages of 128 keys (~197 KB): one CTA per
// SM.  (A 4-warp, 64-key-stage variant with two CTAs per SM, meant to let the
// next layer's CTAs prefetch under PDL, measured slower at every batch.)
constexpr int kCW = 8;                       // consumer warps
constexpr int kThreads = (kCW + 1) * 32;
#ifndef RK_CL_STAGES
#define RK_CL_STAGES 3
#endif
constexpr int kStg = RK_CL_STAGES;
constexpr int kBoxRows = 16;                 // keys per box (one consumer warp's group)
constexpr int kBoxBytes = kBoxRows * 128;    // 16 keys x 128 bytes (64 bf16 / 32 fp32 dims)

// KV element type: bf16 stages hold 128 keys (8 groups of 16, one per consumer
// warp); fp32 rows are twice as wide, so a stage holds 64 keys (4 groups) and
// the consumer warps form two sets that take alternate stages (warp w: group
// w % 4 of the stages t with t % 2 == w / 4) — same ring bytes, same warps.
template <typename KT>
struct KV;
template <>
struct KV<__nv_bfloat16> {
  static constexpr int ES = 2, GROUPS = 8, SETS = 1;
};
template <>
struct KV<float> {
  static constexpr int ES = 4, GROUPS = 4, SETS = 2;
};

template <typename KT, int D>
struct CTile {
  static constexpr int ES = KV<KT>::ES;
  static constexpr int TK = kBoxRows * KV<KT>::GROUPS;   // keys per stage
  static constexpr int BOXE = 128 / ES;                  // elements per 128-byte box row
  static constexpr int NH = D / BOXE;                    // boxes per key row (128-byte column slabs)
  static constexpr int HALF = TK * 128;                  // one slab of a stage: [TK rows][128 B]
  static constexpr int OP = NH * HALF;                   // bytes of K (or V) per stage
  static constexpr int C16 = D * ES / 16;                // 16-byte chunks per key row
  static constexpr size_t smem = 1024 + 2 * (size_t)kStg * OP + 2 * kStg * sizeof(uint64_t);
  // byte offset of (key row r of group w, 16-byte chunk c16 of the row) in one
  // operand stage; rows of a slab are contiguous, so a full stage is one
  // {BOXE, TK} box per slab and a partial one is {BOXE, 16} boxes per group
  __device__ static __forceinline__ uint32_t off(int w, int r, int c16) {
    const int hf = c16 >> 3, c = c16 & 7;
    return (uint32_t)(hf * HALF + (16 * w + r) * 128 + ((c ^ (r & 7)) << 4));
  }
};

__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(kCW * 32)); }
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// asynchronous remote store that counts its bytes on the destination CTA's mbarrier
__device__ __forceinline__ void st_async(uint32_t addr, float v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
               ::"r"(addr), "r"(__float_as_uint(v)), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ void cl_arrive() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cl_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_box(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                        uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

struct ClusterParams {
  const float* q;          // [B][Hq][D]
  void* k;                 // cache base (k_map / v_map describe the same memory), bf16 or fp32
  void* v;
  int64_t rows_per_b;      // cache rows (keys) per dialogue = batch_stride / (HKV*D)
  const int32_t* seq_len;  // [B]
  const void* k_new;       // [B][HKV][D] or null
  const void* v_new;
  int hq, hkv;
  float scale_log2;
  float* out;              // [B][Hq][D]
  const int32_t* active;   // [B] or null: rows with 0 are skipped (no append, no output)
};

// fp32 K / V rows r, r+1 at 16-byte chunk c16 (+ byte offset) of one stage -> bf16 hi / lo pairs
__device__ __forceinline__ float2 lds_f2(const uint8_t* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
  const float ha = bf16_round(a), hb = bf16_round(b);
  hi = pack_bf16(ha, hb);
  lo = pack_bf16(a - ha, b - hb);
}

// kmap/vmap: {BOXE, TK}-key boxes (whole stages); kmap16/vmap16: {BOXE, 16} (the
// last, partial stage of a slice, so a slice reads at most 15 keys past its end)
template <typename KT, int D, int G>
__global__ void __launch_bounds__(kThreads, 1) decode_cluster_kernel(const __grid_constant__ CUtensorMap kmap,
                                                                     const __grid_constant__ CUtensorMap vmap,
                                                                     const __grid_constant__ CUtensorMap kmap16,
                                                                     const __grid_constant__ CUtensorMap vmap16,
                                                                     const __grid_constant__ ClusterParams p) {
  using T = CTile<KT, D>;
  constexpr int NH = T::NH, OP = T::OP, TK = T::TK, BOXE = T::BOXE;
  constexpr int GROUPS = KV<KT>::GROUPS, SETS = KV<KT>::SETS;
  constexpr bool F32 = sizeof(KT) == 4;
  constexpr int KC = D / 16, NT = D / 8;
  static_assert(G <= 8, "at most 8 query heads per kv-head");
  extern __shared__ uint8_t smem_raw[];
  // 128-byte swizzled TMA boxes need 1024-byte aligned destinations
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* kst = smem;
  uint8_t* vst = smem + kStg * OP;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kStg * OP);
  uint64_t* empty = full + kStg;
  // cluster merge inbox of this CTA: the outputs [rank*per, rank*per + per) it
  // finalises, pushed by every CTA q of the cluster (row q), plus their (m, l)
  __shared__ float in_acc[8 * D + 64];
  __shared__ float in_m[16][8], in_l[16][8];
  __shared__ __align__(8) uint64_t in_bar;      // completes when every peer's bytes have landed

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.z, h = blockIdx.y;
  // an inactive row (a dialogue outside the decode loop this step): every CTA of its
  // cluster leaves before any barrier, so nothing is appended, read or written
  if (p.active != nullptr && !p.active[b]) {
    pdl_trigger();
    return;
  }
  const uint32_t C = cl_size(), rank = cl_rank();
  const bool append = p.k_new != nullptr;
  const int len = p.seq_len[b] + (append ? 1 : 0);
  const int lo = (int)((int64_t)rank * len / C), hi = (int)((int64_t)(rank + 1) * len / C);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStg; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GROUPS);
    }
    mbar_init(&in_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl_arrive();            // this CTA is running: peers may push into its inbox after their wait
  pdl_trigger();          // the next layer's CTAs may start their prologue (no workspace is shared)
  const int64_t row0 = (int64_t)b * p.rows_per_b;

  if (warp == kCW) {
    // ================= producer
    // the cache rows before the appended key do not depend on the previous kernel
    // (PDL): their TMA boxes stream while it finishes.  The appended key (k_new /
    // v_new) is the previous kernel's output (the fused QKV projection): the stage
    // that holds cache row len-1 waits for it, copies head h's 256 bytes of K and
    // V into that row, and fences them for the async proxy before its TMA reads.
    const bool owns_new = append && hi == len && hi > lo;
    const uint64_t pol = evict_first_policy();
    int t = 0;
    for (int j0 = lo; j0 < hi; j0 += TK, ++t) {
      const int nk = min(TK, hi - j0);
      if (owns_new && j0 + nk == hi) {
        pdl_wait();
        const int64_t dst = (row0 + len - 1) * p.hkv * D + (int64_t)h * D;
        const int64_t src = ((int64_t)b * p.hkv + h) * D;
        for (int e = lane; e < T::C16; e += 32) {
          reinterpret_cast<uint4*>(static_cast<KT*>(p.k) + dst)[e] =
              reinterpret_cast<const uint4*>(static_cast<const KT*>(p.k_new) + src)[e];
          reinterpret_cast<uint4*>(static_cast<KT*>(p.v) + dst)[e] =
              reinterpret_cast<const uint4*>(static_cast<const KT*>(p.v_new) + src)[e];
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __syncwarp();
      }
      if (lane == 0) {
        const int s = t % kStg;
        const int ng = (nk + kBoxRows - 1) / kBoxRows;
        if (t >= kStg) mbar_wait(&empty[s], ((t / kStg) - 1) & 1);
        mbar_expect_tx(&full[s], (unsigned)(2 * ng * NH * kBoxBytes));
        const int r = (int)(row0 + j0);
        for (int hf = 0; hf < NH; ++hf) {
          const uint32_t kd = smem_u32(kst + s * OP) + hf * T::HALF, vd = smem_u32(vst + s * OP) + hf * T::HALF;
          if (nk == TK) {
            tma_box(kd, &kmap, h * D + hf * BOXE, r, &full[s], pol);
            tma_box(vd, &vmap, h * D + hf * BOXE, r, &full[s], pol);
          } else {
            for (int w = 0; w < ng; ++w) {
              tma_box(kd + w * kBoxBytes, &kmap16, h * D + hf * BOXE, r + w * kBoxRows, &full[s], pol);
              tma_box(vd + w * kBoxBytes, &vmap16, h * D + hf * BOXE, r + w * kBoxRows, &full[s], pol);
            }
          }
        }
      }
    }
    pdl_wait();   // this warp also writes outputs in the cluster merge
  } else {
    // ================= consumers
    pdl_wait();   // q and out belong to the previous kernels until here
    const int g = lane >> 2, c = lane & 3;
    uint32_t qa[KC][4];
    {
      const bool real = g < G;
      const float* qp = p.q + ((int64_t)b * p.hq + h * G + (real ? g : 0)) * D;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const float2 lo2 = *reinterpret_cast<const float2*>(qp + 16 * kc + 2 * c);
        const float2 hi2 = *reinterpret_cast<const float2*>(qp + 16 * kc + 2 * c + 8);
        float x[4];
        x[0] = real ? lo2.x * p.scale_log2 : 0.f;
        x[1] = real ? lo2.y * p.scale_log2 : 0.f;
        x[2] = real ? hi2.x * p.scale_log2 : 0.f;
        x[3] = real ? hi2.y * p.scale_log2 : 0.f;
        const float h0 = bf16_round(x[0]), h1 = bf16_round(x[1]), h2 = bf16_round(x[2]), h3 = bf16_round(x[3]);
        qa[kc][0] = pack_bf16(h0, h1);
        qa[kc][1] = pack_bf16(x[0] - h0, x[1] - h1);
        qa[kc][2] = pack_bf16(h2, h3);
        qa[kc][3] = pack_bf16(x[2] - h2, x[3] - h3);
      }
    }
    float o[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m = -INFINITY, lsum = 0.f;
    const int grp = warp % GROUPS, set = warp / GROUPS;
    for (int j0 = lo + set * TK, t = set; j0 < hi; j0 += SETS * TK, t += SETS) {
      const int s = t % kStg;
      const int nkw = min(kBoxRows, max(0, min(TK, hi - j0) - kBoxRows * grp));
      mbar_wait(&full[s], (t / kStg) & 1);
      if (nkw > 0) {
        const uint8_t* kb = kst + s * OP;
        uint8_t* vb = vst + s * OP;
        if (nkw < kBoxRows) {   // rows past the slice are other keys (or unwritten rows): zero their V
          for (int e = lane; e < (kBoxRows - nkw) * T::C16; e += 32) {
            const int r = nkw + e / T::C16, c16 = e % T::C16;
            *reinterpret_cast<uint4*>(vb + T::off(grp, r, c16)) = make_uint4(0, 0, 0, 0);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
        }
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (F32) {
          // fp32 K rows split into bf16 hi + lo on the fly: S = [q_hi; q_lo] (K_hi + K_lo),
          // ~16 mantissa bits per operand (the bf16 cache's products keep the same class)
#pragma unroll
          for (int kc = 0; kc < KC; ++kc) {
            const int cb = 4 * kc + (c >> 1), ob = (c & 1) * 8;     // dims 16kc + 2c (+8): chunks cb, cb + 2
            uint32_t bh0, bl0, bh1, bl1;
            float2 x0 = lds_f2(kb + T::off(grp, g, cb) + ob), x1 = lds_f2(kb + T::off(grp, g, cb + 2) + ob);
            split_pair(x0.x, x0.y, bh0, bl0);
            split_pair(x1.x, x1.y, bh1, bl1);
            mma_bf16_16816(s0, qa[kc], bh0, bh1);
            mma_bf16_16816(s0, qa[kc], bl0, bl1);
            x0 = lds_f2(kb + T::off(grp, 8 + g, cb) + ob);
            x1 = lds_f2(kb + T::off(grp, 8 + g, cb + 2) + ob);
            split_pair(x0.x, x0.y, bh0, bl0);
            split_pair(x1.x, x1.y, bh1, bl1);
            mma_bf16_16816(s1, qa[kc], bh0, bh1);
            mma_bf16_16816(s1, qa[kc], bl0, bl1);
          }
        } else {
#pragma unroll
          for (int kk = 0; kk < KC / 2; ++kk) {
            uint32_t r[4];
            const int c8 = 4 * kk + (lane >> 3);
            ldmatrix_x4(r, kb + T::off(grp, lane & 7, c8));
            mma_bf16_16816(s0, qa[2 * kk], r[0], r[1]);
            mma_bf16_16816(s0, qa[2 * kk + 1], r[2], r[3]);
            ldmatrix_x4(r, kb + T::off(grp, 8 + (lane & 7), c8));
            mma_bf16_16816(s1, qa[2 * kk], r[0], r[1]);
            mma_bf16_16816(s1, qa[2 * kk + 1], r[2], r[3]);
          }
        }
        float sc[4];
        sc[0] = (2 * c < nkw) ? s0[0] + s0[2] : -INFINITY;
        sc[1] = (2 * c + 1 < nkw) ? s0[1] + s0[3] : -INFINITY;
        sc[2] = (2 * c + 8 < nkw) ? s1[0] + s1[2] : -INFINITY;
        sc[3] = (2 * c + 9 < nkw) ? s1[1] + s1[3] : -INFINITY;
        float tmax = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
        const bool grow = tmax > m + 8.f || (m == -INFINITY && tmax != -INFINITY);
        if (__any_sync(0xffffffffu, grow)) {
          const float m_new = grow ? tmax : m;
          const float corr = (m == -INFINITY) ? 0.f : fast_exp2(m - m_new);
          m = m_new;
          lsum *= corr;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            o[nt][0] *= corr; o[nt][1] *= corr; o[nt][2] *= corr; o[nt][3] *= corr;
          }
        }
        const float mu = (m == -INFINITY) ? 0.f : m;
        float pr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) pr[i] = fast_exp2(sc[i] - mu);
        lsum += (pr[0] + pr[1]) + (pr[2] + pr[3]);
        uint32_t pa[4];
        {
          const float h0 = bf16_round(pr[0]), h1 = bf16_round(pr[1]), h2 = bf16_round(pr[2]), h3 = bf16_round(pr[3]);
          pa[0] = pack_bf16(h0, h1);
          pa[1] = pack_bf16(pr[0] - h0, pr[1] - h1);
          pa[2] = pack_bf16(h2, h3);
          pa[3] = pack_bf16(pr[2] - h2, pr[3] - h3);
        }
        if constexpr (F32) {
          // V rows (keys 2c, 2c+1, 2c+8, 2c+9) x dims 16jj + 2g, +1: tile 2jj holds the even
          // dims, tile 2jj+1 the odd ones, so one 8-byte load feeds both tiles (the
          // epilogue writes dims 16jj + 4c .. +3 from o[2jj][*], o[2jj+1][*])
#pragma unroll
          for (int jj = 0; jj < NT / 2; ++jj) {
            const int cb = 4 * jj + (g >> 1), ob = (g & 1) * 8;
            const float2 v0 = lds_f2(vb + T::off(grp, 2 * c, cb) + ob);
            const float2 v1 = lds_f2(vb + T::off(grp, 2 * c + 1, cb) + ob);
            const float2 v8 = lds_f2(vb + T::off(grp, 2 * c + 8, cb) + ob);
            const float2 v9 = lds_f2(vb + T::off(grp, 2 * c + 9, cb) + ob);
            uint32_t eh0, el0, eh1, el1, oh0, ol0, oh1, ol1;
            split_pair(v0.x, v1.x, eh0, el0);
            split_pair(v8.x, v9.x, eh1, el1);
            split_pair(v0.y, v1.y, oh0, ol0);
            split_pair(v8.y, v9.y, oh1, ol1);
            mma_bf16_16816(o[2 * jj], pa, eh0, eh1);
            mma_bf16_16816(o[2 * jj], pa, el0, el1);
            mma_bf16_16816(o[2 * jj + 1], pa, oh0, oh1);
            mma_bf16_16816(o[2 * jj + 1], pa, ol0, ol1);
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < NT / 2; ++jj) {
            uint32_t r[4];
            ldmatrix_x4_trans(r, vb + T::off(grp, (lane & 7) + 8 * ((lane >> 3) & 1), 2 * jj + (lane >> 4)));
            mma_bf16_16816(o[2 * jj], pa, r[0], r[1]);
            mma_bf16_16816(o[2 * jj + 1], pa, r[2], r[3]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    // ---- warps -> CTA partial; every TMA has landed (all tiles were waited), so
    // the K ring is free for the per-warp partials after the consumer barrier
    csync();
    float* wm = reinterpret_cast<float*>(kst);            // [kCW][8]
    float* wl = wm + kCW * 8;                              // [kCW][8]
    float* wacc = wl + kCW * 8;                            // [kCW][8][D]
    if (g < G) {
      if constexpr (F32) {
#pragma unroll
        for (int jj = 0; jj < NT / 2; ++jj)
          *reinterpret_cast<float4*>(wacc + (warp * 8 + g) * D + 16 * jj + 4 * c) =
              make_float4(o[2 * jj][0] + o[2 * jj][2], o[2 * jj + 1][0] + o[2 * jj + 1][2],
                          o[2 * jj][1] + o[2 * jj][3], o[2 * jj + 1][1] + o[2 * jj + 1][3]);
      } else {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          *reinterpret_cast<float2*>(wacc + (warp * 8 + g) * D + 8 * nt + 2 * c) =
              make_float2(o[nt][0] + o[nt][2], o[nt][1] + o[nt][3]);
      }
      if (c == 0) {
        wm[warp * 8 + g] = m;
        wl[warp * 8 + g] = lsum;
      }
    }
    csync();
  }
  // ---- cluster merge, push model: every CTA scatters its partial (m, l, acc) into
  // the inbox of the CTA that finalises each output with st.async, whose bytes count
  // on the owner's inbox mbarrier; each CTA waits for its own inbox only (no closing
  // cluster barrier, no GPU-scope fence) and reduces it locally
  if (C == 1) {           // one CTA per (dialogue, kv-head): its partial is the answer
    __syncwarp();
    cl_wait();
    if (warp < kCW) {
      const float* wm = reinterpret_cast<const float*>(kst);
      const float* wl = wm + kCW * 8;
      const float* wacc = wl + kCW * 8;
      for (int e = threadIdx.x; e < G * D; e += kCW * 32) {
        const int gg = e / D, dd = e % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kCW; ++w) M = fmaxf(M, wm[w * 8 + gg]);
        const float mu = (M == -INFINITY) ? 0.f : M;
        float L = 0.f, A = 0.f;
#pragma unroll
        for (int w = 0; w < kCW; ++w) {
          const float sc = fast_exp2(wm[w * 8 + gg] - mu);
          L += wl[w * 8 + gg] * sc;
          A += wacc[(w * 8 + gg) * D + dd] * sc;
        }
        p.out[((int64_t)b * p.hq + h * G + gg) * D + dd] = A / L;
      }
    }
    return;
  }
  const int per = ((G * D + (int)C - 1) / (int)C + 3) & ~3;      // outputs finalised per CTA
  const int mine = max(0, min(per, G * D - (int)rank * per));    // outputs this CTA finalises
  if (threadIdx.x == 0)
    mbar_expect_tx(&in_bar, (unsigned)(C * (mine + 2 * G) * 4));
  __syncwarp();
  cl_wait();              // every peer has started (its inbox and barrier exist)
  if (warp < kCW) {
    const float* wm = reinterpret_cast<const float*>(kst);
    const float* wl = wm + kCW * 8;
    const float* wacc = wl + kCW * 8;
    for (int e = threadIdx.x; e < G * D; e += kCW * 32) {
      const int gg = e / D, dd = e % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kCW; ++w) M = fmaxf(M, wm[w * 8 + gg]);
      const float mu = (M == -INFINITY) ? 0.f : M;
      float L = 0.f, A = 0.f;
#pragma unroll
      for (int w = 0; w < kCW; ++w) {
        const float sc = fast_exp2(wm[w * 8 + gg] - mu);
        L += wl[w * 8 + gg] * sc;
        A += wacc[(w * 8 + gg) * D + dd] * sc;
      }
      const int r = e / per;
      st_async(cl_map(&in_acc[rank * per + (e - r * per)], r), A, cl_map(&in_bar, r));
      if (dd == 0)
        for (uint32_t q = 0; q < C; ++q) {
          st_async(cl_map(&in_m[rank][gg], q), M, cl_map(&in_bar, q));
          st_async(cl_map(&in_l[rank][gg], q), L, cl_map(&in_bar, q));
        }
    }
  }
  mbar_wait(&in_bar, 0);  // every peer's share of this CTA's outputs has landed
  for (int el = threadIdx.x; el < per; el += kThreads) {
    const int e = (int)rank * per + el;
    if (e >= G * D) break;
    const int gg = e / D, dd = e % D;
    float M = -INFINITY;
    for (uint32_t q = 0; q < C; ++q) M = fmaxf(M, in_m[q][gg]);
    const float mu = (M == -INFINITY) ? 0.f : M;
    float L = 0.f, A = 0.f;
    for (uint32_t q = 0; q < C; ++q) {
      const float sc = fast_exp2(in_m[q][gg] - mu);
      L += in_l[q][gg] * sc;
      A += in_acc[q * per + el] * sc;
    }
    p.out[((int64_t)b * p.hq + h * G + gg) * D + dd] = A / L;
  }
}

int g_max_clusters[17] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};   // by cluster size

template <typename KT, int D, int G>
cudaError_t configure(int C) {
  auto kern = decode_cluster_kernel<KT, D, G>;
  static bool done = false;
  if (!done) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CTile<KT, D>::smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    done = true;
  }
  (void)C;
  return cudaSuccess;
}

template <typename KT, int D, int G>
cudaError_t launch(int C, int B, int hkv, const CUtensorMap* m, const ClusterParams& p, cudaStream_t st) {
  cudaError_t e = configure<KT, D, G>(C);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C, hkv, B);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = CTile<KT, D>::smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, decode_cluster_kernel<KT, D, G>, m[0], m[1], m[2], m[3], p);
}

template <typename KT, int D>
cudaError_t launch_by_g(int G, int C, int B, int hkv, const CUtensorMap* m, const ClusterParams& p,
                        cudaStream_t st) {
  switch (G) {
    case 1: return launch<KT, D, 1>(C, B, hkv, m, p, st);
    case 2: return launch<KT, D, 2>(C, B, hkv, m, p, st);
    case 4: return launch<KT, D, 4>(C, B, hkv, m, p, st);
    case 7: return launch<KT, D, 7>(C, B, hkv, m, p, st);
    case 8: return launch<KT, D, 8>(C, B, hkv, m, p, st);
  }
  return cudaErrorInvalidValue;
}

int max_clusters(int C) {
  const int i = C;
  if (g_max_clusters[i] < 0) {
    if (configure<__nv_bfloat16, 128, 4>(C) != cudaSuccess) return g_max_clusters[i] = 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C, 1, 1);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = CTile<__nv_bfloat16, 128>::smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, decode_cluster_kernel<__nv_bfloat16, 128, 4>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    g_max_clusters[i] = n;
    if (std::getenv("RK_DECODE_CLUSTER_VERBOSE")) std::fprintf(stderr, "[rk] cluster %d: %d co-resident\n", C, n);
  }
  return g_max_clusters[i];
}

}  // namespace

// cluster size for (batch, kv-heads, longest dialogue); 0 = use the persistent
// split-K kernel.  Applies when every (dialogue, kv-head) pair gets >= 1 CTA
// in one wave; C = the largest of 16/12/8/6/4/3/2/1 that fits the SMs with
// >= 64 keys per CTA and whose clusters are all co-resident (B200, 1 CTA/SM:
// 7 clusters of 16 or 12, 15 of 8, 22 of 6, 33 of 4 — so one dialogue with 8
// kv-heads runs 8 x 8 CTAs).  Slices follow each dialogue's own length, so a batch whose lengths
// differ widely runs at the pace of its longest dialogue (the persistent
// kernel balances keys across SMs instead).  RK_DECODE_CLUSTER=0 disables
// (A/B runs, tests of the persistent kernel).
int cluster_decode_size(int kv_dtype, int d, int hkv, int G, int batch, int max_len, int64_t batch_stride,
                        bool multiwave) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = std::getenv("RK_DECODE_CLUSTER");
    mode = e ? std::atoi(e) : 1;
  }
  // fp32 and bf16 stages have the same bytes and warps (CTile), so the same co-residency
  if (mode == 0 || (kv_dtype != RK_BF16 && kv_dtype != RK_F32) || (d != 128 && d != 64)) return 0;
  if (!(G == 1 || G == 2 || G == 4 || G == 7 || G == 8)) return 0;
  const int64_t row = (int64_t)hkv * d;
  if (batch > 1 && (batch_stride % row != 0 || batch_stride <= 0)) return 0;
  static int cmax = -1;        // RK_DECODE_CLUSTER_CMAX caps the cluster size (experiments)
  if (cmax < 0) {
    const char* e = std::getenv("RK_DECODE_CLUSTER_CMAX");
    cmax = e ? std::atoi(e) : 16;
  }
  const int pairs = batch * hkv;
  // RK_DECODE_CLUSTER=2 (experiment): beyond one wave, one CTA per pair in several
  // waves.  Measured vs the persistent kernel (C2 shapes, equal lengths): better when
  // the waves are nearly full (B=32: 45.5 vs 50.1 us upper, 297.6 vs 301.4 us lower;
  // B=48 67.0 vs 70.5 us), worse otherwise (B=20: 38.5 vs 33.4 us) and exposed to
  // ragged lengths, so the default keeps the persistent kernel there
  if ((mode == 2 || multiwave) && pairs > sm_count()) return 1;
  for (int C : {16, 12, 8, 6, 4, 3, 2, 1}) {   // 10 (11 co-resident) measured slower at B=1 upper layers
    if (C > cmax) continue;
    if ((int64_t)pairs * C > sm_count()) continue;
    if (C > 1 && max_len / C < 64) continue;          // >= 64 keys per CTA
    if (max_clusters(C) < pairs) continue;             // one co-resident wave
    // a long single-dialogue layer on under half the SMs streams faster through the
    // persistent kernel's full wave (B=1: 65 K keys 45.1 vs 42.9 us, 131 K keys 87.7 vs
    // 81.9 us; at 32 K keys they tie and below it the cluster decode wins)
    if (2 * (int64_t)pairs * C < sm_count() && max_len / C > 6144) return 0;
    return C;
  }
  return 0;
}

int launch_decode_cluster(int C, int kv_dtype, const float* q, int batch, int hq, int d, void* k_cache,
                          void* v_cache, int hkv, int64_t batch_stride, const int32_t* seq_len, int max_len,
                          const void* k_new, const void* v_new, float* out, cudaStream_t st,
                          const int32_t* active) {
  const bool f32 = kv_dtype == RK_F32;
  const int es = f32 ? 4 : 2;
  const uint32_t tk = f32 ? (uint32_t)CTile<float, 128>::TK : (uint32_t)CTile<__nv_bfloat16, 128>::TK;
  const int64_t row = (int64_t)hkv * d;
  const int64_t rows_per_b = batch > 1 ? batch_stride / row : (int64_t)max_len;
  // the map ends at the last dialogue's max_len-th row (max_len bounds seq_len+1
  // and the capacity): the 16-key tail boxes of a slice may run up to 15 rows
  // past a dialogue's length — inside the next dialogue's rows (masked), or
  // past the map's end, where TMA fills zeros instead of reading unowned memory
  const uint64_t rows = (uint64_t)rows_per_b * (batch - 1) + (uint64_t)max_len;
  CUtensorMap m[4];   // K, V whole-stage boxes; K, V 16-key boxes
  int r = 0;
  for (int i = 0; i < 4 && !r; ++i)
    r = tc::make_map(&m[i], (i & 1) ? v_cache : k_cache, (uint64_t)row, rows, (uint64_t)row * es,
                     i < 2 ? tk : (uint32_t)kBoxRows, es);
  if (r) return r;
  ClusterParams p{};
  p.q = q;
  p.k = k_cache;
  p.v = v_cache;
  p.rows_per_b = rows_per_b;
  p.seq_len = seq_len;
  p.k_new = k_new;
  p.v_new = v_new;
  p.hq = hq;
  p.hkv = hkv;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
  p.out = out;
  p.active = active;
  const int G = hq / hkv;
  cudaError_t e;
  if (f32)
    e = d == 128 ? launch_by_g<float, 128>(G, C, batch, hkv, m, p, st) : launch_by_g<float, 64>(G, C, batch, hkv, m, p, st);
  else
    e = d == 128 ? launch_by_g<__nv_bfloat16, 128>(G, C, batch, hkv, m, p, st)
                 : launch_by_g<__nv_bfloat16, 64>(G, C, batch, hkv, m, p, st);
  if (e != cudaSuccess) return cuda_status(e, "decode_cluster_kernel launch");
  return RK_OK;
}

}  // namespace rk
