// Multi-row watershed round scoring on the 5th-generation tensor cores.
//
// For a question of n_q rows at layer Lw-1 (pipeline.py:225-245, C3: 512 rows
// x 66K keys x 28 heads) the work is S = Q K^T over every visible key followed
// by a softmax and a per-round sum (stats.py:59-94).  This kernel produces, per
// (question row, query head, round-aligned item), the log2-domain running max
// m and sum l of exp2(s - m); score_rows_kernel turns them into Eq. 1 masses.
//
// CTA roles (192 threads, one CTA per SM, persistent over work units):
//   warps 0-3  epilogue: thread = accumulator row = (head g, question row i);
//              tcgen05.ld the 128 scores of a tile from TMEM, causal mask,
//              online (m, l) per item — no cross-thread reduction at all;
//   warp 4     TMA producer: K tiles [128 keys x 128 dims] of one kv-head
//              (two 64-element boxes, SWIZZLE_128B) into a 4-stage ring;
//              Q tiles (split bf16: q_hi, q_lo) when the M tile changes;
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer:
//              S[128 x 128] = Q_hi K^T + Q_lo K^T (16 x m128n128k16, fp32 in
//              TMEM, double-buffered), tcgen05.commit -> mbarriers.
// The split q = q_hi + q_lo (bf16 each) keeps ~16 mantissa bits of the fp32
// query so the masses match the fp64 oracle to ~1e-6 relative.
// Work unit = (M tile, item); units are dealt to CTAs as contiguous ranges so a
// CTA reloads Q only when its range crosses an M tile.
#include <cmath>

#include "tc_common.cuh"

namespace rk {
namespace tc {

constexpr int BM = 128, BN = 128, BK = 128;          // rows, keys, head dim (fixed 128)
constexpr int STAGES = 4;
constexpr int SUB = BM * 64 * 2;                     // one 64-element swizzled box: 16 KB
constexpr int KT_BYTES = 2 * SUB;                    // K tile: 32 KB
constexpr int QT_BYTES = 4 * SUB;                    // Q tile hi+lo: 64 KB
constexpr int THREADS = 192;
constexpr size_t SMEM = 1024 + QT_BYTES + STAGES * KT_BYTES + 256;

struct Params {
  int n_q, hq, hkv, G, mpad, n_items, n_units, mtiles;
  const int64_t* q_pos;            // question row positions (visibility), [n_q]
  const int64_t* k_pos;            // key positions (visibility), [s]
  const int32_t* items;            // [n_items][3]
  float* part_m;                   // [n_q][hq][n_items]
  float* part_l;
};

// kind::f16, F32 accumulate, BF16 A/B, both K-major, M = N = 128
constexpr uint32_t kIdesc = idesc_f16(BM, BN);

// unit u -> (mtile, item); mtile = kvh * mtiles + mt
__device__ __forceinline__ void unit_of(const Params& p, int u, int& mtile, int& item) {
  mtile = u / p.n_items;
  item = u - mtile * p.n_items;
}

__global__ void __launch_bounds__(THREADS, 1)
score_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qs = smem;                                // [hi|lo][chunk0|chunk1] 4 x 16 KB
  uint8_t* ks = smem + QT_BYTES;                     // STAGES x 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(ks + STAGES * KT_BYTES);
  uint64_t* k_full = bars;                           // [STAGES]
  uint64_t* k_empty = bars + STAGES;                 // [STAGES]
  uint64_t* q_full = bars + 2 * STAGES;
  uint64_t* q_empty = q_full + 1;
  uint64_t* s_full = q_full + 2;                     // [2]
  uint64_t* s_empty = q_full + 4;                    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 6);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = (int)((int64_t)blockIdx.x * p.n_units / gridDim.x);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * p.n_units / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&k_full[s], 1);
      bar_init(&k_empty[s], 1);
    }
    bar_init(q_full, 1);
    bar_init(q_empty, 1);
    for (int b = 0; b < 2; ++b) {
      bar_init(&s_full[b], 1);
      bar_init(&s_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {   // 256 TMEM columns: two 128-column fp32 score buffers
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ================= TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&qmap) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
      int cur_mtile = -1, qn = 0, t = 0;
      for (int u = u0; u < u1; ++u) {
        int mtile, item;
        unit_of(p, u, mtile, item);
        const int kvh = mtile / p.mtiles, mt = mtile - kvh * p.mtiles;
        if (mtile != cur_mtile) {
          if (qn > 0) bar_wait(q_empty, (qn - 1) & 1);
          bar_expect(q_full, QT_BYTES);
          const int row0 = kvh * 2 * p.mpad + mt * BM;
          tma_2d(qs + 0 * SUB, &qmap, 0, row0, q_full);                 // hi, dims 0-63
          tma_2d(qs + 1 * SUB, &qmap, 64, row0, q_full);                // hi, dims 64-127
          tma_2d(qs + 2 * SUB, &qmap, 0, row0 + p.mpad, q_full);        // lo
          tma_2d(qs + 3 * SUB, &qmap, 64, row0 + p.mpad, q_full);
          cur_mtile = mtile;
          ++qn;
        }
        const int lo = p.items[item * 3 + 0], hi = p.items[item * 3 + 1];
        for (int j0 = lo; j0 < hi; j0 += BN, ++t) {
          const int s = t % STAGES;
          if (t >= STAGES) bar_wait(&k_empty[s], ((t / STAGES) - 1) & 1);
          bar_expect(&k_full[s], KT_BYTES);
          tma_2d(ks + s * KT_BYTES, &kmap, kvh * BK, j0, &k_full[s]);
          tma_2d(ks + s * KT_BYTES + SUB, &kmap, kvh * BK + 64, j0, &k_full[s]);
        }
      }
    }
  } else if (warp == 5) {
    // ================= MMA issuer (one elected thread)
    if (lane == 0) {
      int cur_mtile = -1, qn = 0, t = 0;
      for (int u = u0; u < u1; ++u) {
        int mtile, item;
        unit_of(p, u, mtile, item);
        if (mtile != cur_mtile) {
          if (qn > 0) umma_commit(q_empty);          // Q slot free once prior MMAs finish
          bar_wait(q_full, qn & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          cur_mtile = mtile;
          ++qn;
        }
        const int lo = p.items[item * 3 + 0], hi = p.items[item * 3 + 1];
        for (int j0 = lo; j0 < hi; j0 += BN, ++t) {
          const int s = t % STAGES, buf = t & 1;
          bar_wait(&k_full[s], (t / STAGES) & 1);
          if (t >= 2) bar_wait(&s_empty[buf], ((t / 2) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t d = tmem + buf * BN;
#pragma unroll
          for (int hl = 0; hl < 2; ++hl)
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint8_t* a = qs + (2 * hl + k / 4) * SUB + 32 * (k % 4);
              const uint8_t* b = ks + s * KT_BYTES + (k / 4) * SUB + 32 * (k % 4);
              umma(d, umma_desc(a), umma_desc(b), kIdesc, (hl | k) ? 1u : 0u);
            }
          umma_commit(&k_empty[s]);                 // smem stage free when these MMAs finish
          umma_commit(&s_full[buf]);                // scores ready for the epilogue
        }
      }
    }
  } else {
    // ================= epilogue: warps 0-3, thread = accumulator row
    const int r = warp * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    int t = 0;
    for (int u = u0; u < u1; ++u) {
      int mtile, item;
      unit_of(p, u, mtile, item);
      const int kvh = mtile / p.mtiles, mt = mtile - kvh * p.mtiles;
      const int R = mt * BM + r;                    // row within the kv-head's (g, i) rows
      const bool real = R < p.G * p.n_q;
      const int g = real ? R / p.n_q : 0, qi = real ? R - g * p.n_q : 0;
      const int64_t qpos = p.q_pos[qi];
      const int lo = p.items[item * 3 + 0], hi = p.items[item * 3 + 1];
      float m = -INFINITY, l = 0.f;
      for (int j0 = lo; j0 < hi; j0 += BN, ++t) {
        const int buf = t & 1;
        bar_wait(&s_full[buf], (t / 2) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float sc[BN];
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          tmem_ld32(lane_addr + buf * BN + 32 * c, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) sc[32 * c + i] = v[i];
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) bar_arrive(&s_empty[buf]);    // TMEM buffer may be overwritten
        // causal / range mask: key j visible iff j < hi and pos(j) <= pos(row)
        const bool all_vis = (j0 + BN <= hi) && (p.k_pos[min(j0 + BN, hi) - 1] <= qpos);
        float tmax = -INFINITY;
        if (all_vis) {
#pragma unroll
          for (int i = 0; i < BN; ++i) tmax = fmaxf(tmax, sc[i]);
        } else {
#pragma unroll
          for (int i = 0; i < BN; ++i) {
            const int j = j0 + i;
            const bool vis = j < hi && p.k_pos[j] <= qpos;
            sc[i] = vis ? sc[i] : -INFINITY;
            tmax = fmaxf(tmax, sc[i]);
          }
        }
        const float mn = fmaxf(m, tmax);
        const float mu = (mn == -INFINITY) ? 0.f : mn;
        float acc = l * fast_exp2(m - mu);
#pragma unroll
        for (int i = 0; i < BN; ++i) acc += fast_exp2(sc[i] - mu);
        m = mn;
        l = acc;
      }
      if (real) {
        const int64_t o = ((int64_t)qi * p.hq + kvh * p.G + g) * p.n_items + item;
        p.part_m[o] = m;
        p.part_l[o] = l;
      }
    }
  }
  __syncthreads();
  if (warp == 5) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// q [n_q][hq][128] fp32 -> Qs [hkv][2][mpad][128] bf16, rows (g, i), scaled into
// log2 units and split into hi = bf16(x), lo = bf16(x - hi); padding rows zero.
__global__ void prep_q_kernel(const float* __restrict__ q, int n_q, int hq, int hkv, int G, int mpad,
                              float scale_log2, __nv_bfloat16* __restrict__ qs) {
  const int64_t total = (int64_t)hkv * mpad * BK;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(x % BK);
    const int64_t rr = x / BK;
    const int R = (int)(rr % mpad), kvh = (int)(rr / mpad);
    float v = 0.f;
    if (R < G * n_q) {
      const int g = R / n_q, i = R - g * n_q;
      v = q[((int64_t)i * hq + kvh * G + g) * BK + e] * scale_log2;
    }
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
    qs[(((int64_t)kvh * 2 + 0) * mpad + R) * BK + e] = h;
    qs[(((int64_t)kvh * 2 + 1) * mpad + R) * BK + e] = l;
  }
}

}  // namespace tc

bool score_tc_supported(int kv_dtype, int d, int n_q, int G) {
  return kv_dtype == RK_BF16 && d == 128 && (int64_t)n_q * G >= 64 && G <= 8;
}

size_t score_tc_scratch_bytes(int n_q, int hkv, int G) {
  const int mpad = (G * n_q + tc::BM - 1) / tc::BM * tc::BM;
  return (size_t)hkv * 2 * mpad * tc::BK * 2;
}

// q [n_q][hq][128] f32, k [s][hkv][128] bf16; items [n_items][3] sorted by bin;
// writes part_m/part_l [n_q][hq][n_items]; qs_scratch >= score_tc_scratch_bytes
int launch_score_tc(const float* q, int n_q, int hq, const void* k, int s, int hkv, const int64_t* q_pos,
                    const int64_t* k_pos, const int32_t* items, int n_items, float* part_m, float* part_l,
                    void* qs_scratch, cudaStream_t st) {
  const int G = hq / hkv;
  const int mpad = (G * n_q + tc::BM - 1) / tc::BM * tc::BM;
  tc::prep_q_kernel<<<(int)std::min<int64_t>(4096, ((int64_t)hkv * mpad * tc::BK + 255) / 256), 256, 0, st>>>(
      q, n_q, hq, hkv, G, mpad, (float)(1.4426950408889634 / std::sqrt(128.0)),
      reinterpret_cast<__nv_bfloat16*>(qs_scratch));
  RK_CHECK_LAUNCH("prep_q_kernel");
  CUtensorMap qmap, kmap;
  int r = tc::make_map(&qmap, qs_scratch, tc::BK, (uint64_t)hkv * 2 * mpad, tc::BK * 2);
  if (r) return r;
  r = tc::make_map(&kmap, k, (uint64_t)hkv * tc::BK, (uint64_t)s, (uint64_t)hkv * tc::BK * 2);
  if (r) return r;
  tc::Params p{};
  p.n_q = n_q; p.hq = hq; p.hkv = hkv; p.G = G; p.mpad = mpad; p.n_items = n_items;
  p.mtiles = mpad / tc::BM;
  p.n_units = hkv * p.mtiles * n_items;
  p.q_pos = q_pos; p.k_pos = k_pos; p.items = items;
  p.part_m = part_m; p.part_l = part_l;
  static bool configured = false;
  if (!configured) {
    RK_CUDA(cudaFuncSetAttribute(tc::score_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tc::SMEM),
            "score_tc smem attribute");
    configured = true;
  }
  const int grid = std::min(sm_count(), p.n_units);
  tc::score_tc_kernel<<<grid, tc::THREADS, tc::SMEM, st>>>(qmap, kmap, p);
  RK_CHECK_LAUNCH("score_tc_kernel");
  return RK_OK;
}

}  // namespace rk
