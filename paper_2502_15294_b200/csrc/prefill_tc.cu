// Multi-row (question prefill) attention on the 5th-generation tensor cores,
// with the watershed round scoring fused in.
//
// Reference: the question rows of a turn run Model.forward_range over the
// lower layers (full history, pipeline.py:225-230) and the upper layers (kept
// rounds + the question, pipeline.py:292-296); every per-layer call is the
// kernel contract attention_forward (_attn_ext.pyx:20-81: causal by position,
// optional `allowed` mask, fp64 softmax).  At layer Lw-1 the capture matrix is
// reduced to per-round masses (aggregate_round_attention, stats.py:59-94);
// here that reduction is fused: the kernel leaves per-(row, head, round item)
// softmax statistics that score_rows_kernel turns into Eq. 1 masses, so the
// scoring costs no extra pass over K.
//
// Per work unit (M tile of 128 stacked query rows (g, i) of one kv-head, key
// chunk = a run of items) the CTA streams 64-key tiles of K and V:
//   S  = Q_hi K^T + Q_lo K^T            tcgen05.mma m128n64k16 x 16, TMEM
//   P  = exp2(S - m) (online, lazy rescale), split P = P_hi + P_lo (bf16)
//   O += P_hi V + P_lo V                tcgen05.mma m128n128k16 x 8, TMEM,
//                                        V read MN-major straight from its TMA tile
// The q and P splits keep ~16 mantissa bits (fp32-class outputs; the reference
// tolerance is 1e-3 relative, fp64 accumulation on its side).
//
// CTA roles (192 threads, one CTA per SM, persistent over a contiguous range
// of units so Q is reloaded only when the range crosses an M tile):
//   warps 0-3  softmax / epilogue: thread = TMEM lane = stacked row; reads S
//              with tcgen05.ld, masks, online softmax, writes P (swizzled
//              smem) and the per-item scoring statistics; rescales O in TMEM
//              when its running max moves by more than 2^8; at unit end reads
//              O and writes the unit's partial (m, l, O) for the merge;
//   warp 4     TMA producer: Q hi/lo [128 x 128] per M tile, K and V
//              [64 keys x 128] per tile (4-stage ring, SWIZZLE_128B);
//   warp 5     TMEM allocation + single-thread MMA issue, QK of tile t issued
//              ahead of PV of tile t-1 so the tensor pipe has work while the
//              softmax runs.
#include <cmath>

#include <algorithm>

#include "prefill_tc.cuh"
#include "tc_common.cuh"

namespace rk {
namespace pf {

using namespace tc;

constexpr int BM = 128, BN = 64, D = 128;
constexpr int STAGES = 4;
constexpr int QBOX = BM * 64 * 2;        // 128 rows x 64 bf16, swizzled: 16 KB
constexpr int Q_BYTES = 4 * QBOX;        // q_hi, q_lo x two 64-dim halves
constexpr int KBOX = BN * 64 * 2;        // 64 keys x 64 bf16: 8 KB
constexpr int KV_STAGE = 4 * KBOX;       // K (2 boxes) + V (2 boxes): 32 KB
constexpr int P_BYTES = 2 * QBOX;        // P_hi, P_lo: 128 rows x 64 keys each
constexpr int THREADS = 192;
constexpr size_t SMEM = 1024 + Q_BYTES + P_BYTES + STAGES * KV_STAGE + 256;
constexpr float TAU = 8.f;               // lazy rescale threshold (log2 units)
constexpr float FALLBACK = 100.f;        // item statistics recomputed when a tile sits this far below m

constexpr uint32_t kIdescQK = idesc_f16(BM, BN);             // S[128 x 64]  = Q K^T
constexpr uint32_t kIdescPV = idesc_f16(BM, D, true);        // O[128 x 128] += P V, V MN-major

struct Params {
  int n_q, hq, hkv, G, mpad, mtiles;
  int n_items, n_chunks, items_per_chunk, n_units;
  int item_keys;                   // uniform items when items == nullptr
  int s;                           // keys
  const int64_t* q_pos;            // [n_q]
  const int64_t* k_pos;            // [s]
  const uint8_t* allowed;          // [s] or null
  const int32_t* items;            // [n_items][3] (lo, hi, bin) or null (uniform)
  float* item_m;                   // [n_q][hq][n_items] scoring statistics or null
  float* item_l;
  float* part_m;                   // [n_q][hq][n_chunks]
  float* part_l;
  float* part_o;                   // [n_q][hq][n_chunks][128]
};

__device__ __forceinline__ void item_range(const Params& p, int it, int& lo, int& hi) {
  if (p.items) {
    lo = p.items[it * 3 + 0];
    hi = min(p.items[it * 3 + 1], p.s);
  } else {
    lo = it * p.item_keys;
    hi = min(p.s, lo + p.item_keys);
  }
}

__device__ __forceinline__ void unit_of(const Params& p, int u, int& mtile, int& it0, int& it1) {
  mtile = u / p.n_chunks;
  const int c = u - mtile * p.n_chunks;
  it0 = c * p.items_per_chunk;
  it1 = min(p.n_items, it0 + p.items_per_chunk);
}

__device__ __forceinline__ int ntiles(int lo, int hi) { return hi > lo ? (hi - lo + BN - 1) / BN : 0; }

// exp2 of a pair and packing into (hi, lo) bf16x2 words
__device__ __forceinline__ void split_pack(float a, float b, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  float2 hf = __bfloat1622float2(h);
  __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<uint32_t*>(&h);
  lo = *reinterpret_cast<uint32_t*>(&l);
}

__global__ void __launch_bounds__(THREADS, 1)
prefill_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                  const __grid_constant__ CUtensorMap vmap, const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qs = smem;                               // [hi d0-63 | hi d64-127 | lo d0-63 | lo d64-127]
  uint8_t* ps = qs + Q_BYTES;                       // [P_hi | P_lo], 128 rows x 64 keys each
  uint8_t* kvs = ps + P_BYTES;                      // STAGES x [K d0-63 | K d64-127 | V d0-63 | V d64-127]
  uint64_t* bars = reinterpret_cast<uint64_t*>(kvs + STAGES * KV_STAGE);
  uint64_t* kv_full = bars;                         // [STAGES]
  uint64_t* kv_empty = bars + STAGES;               // [STAGES]
  uint64_t* q_full = bars + 2 * STAGES;
  uint64_t* q_empty = q_full + 1;
  uint64_t* s_full = q_full + 2;                    // [2]
  uint64_t* s_empty = q_full + 4;                   // [2]
  uint64_t* p_full = q_full + 6;                    // P tile written (4 warp arrivals)
  uint64_t* pv_done = q_full + 7;                   // PV of the last issued tile complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_full + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u0 = (int)((int64_t)blockIdx.x * p.n_units / gridDim.x);
  const int u1 = (int)((int64_t)(blockIdx.x + 1) * p.n_units / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&kv_full[s], 1);
      bar_init(&kv_empty[s], 1);
    }
    bar_init(q_full, 1);
    bar_init(q_empty, 1);
    for (int b = 0; b < 2; ++b) {
      bar_init(&s_full[b], 1);
      bar_init(&s_empty[b], 4);
    }
    bar_init(p_full, 4);
    bar_init(pv_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {   // 256 TMEM columns: S double buffer (2 x 64) + O (128)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(sa(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_o = tmem + 2 * BN;

  if (warp == 4) {
    // ================= TMA producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&qmap) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&vmap) : "memory");
      int cur_mtile = -1, qn = 0, t = 0;
      for (int u = u0; u < u1; ++u) {
        int mtile, it0, it1;
        unit_of(p, u, mtile, it0, it1);
        const int kvh = mtile / p.mtiles, mt = mtile - kvh * p.mtiles;
        int nt = 0;
        for (int it = it0; it < it1; ++it) {
          int lo, hi;
          item_range(p, it, lo, hi);
          nt += ntiles(lo, hi);
        }
        if (nt == 0) continue;
        if (mtile != cur_mtile) {
          if (qn > 0) bar_wait(q_empty, (qn - 1) & 1);
          bar_expect(q_full, Q_BYTES);
          const int row0 = kvh * 2 * p.mpad + mt * BM;
          tma_2d(qs + 0 * QBOX, &qmap, 0, row0, q_full);
          tma_2d(qs + 1 * QBOX, &qmap, 64, row0, q_full);
          tma_2d(qs + 2 * QBOX, &qmap, 0, row0 + p.mpad, q_full);
          tma_2d(qs + 3 * QBOX, &qmap, 64, row0 + p.mpad, q_full);
          cur_mtile = mtile;
          ++qn;
        }
        for (int it = it0; it < it1; ++it) {
          int lo, hi;
          item_range(p, it, lo, hi);
          for (int j0 = lo; j0 < hi; j0 += BN, ++t) {
            const int s = t % STAGES;
            if (t >= STAGES) bar_wait(&kv_empty[s], ((t / STAGES) - 1) & 1);
            uint8_t* st = kvs + s * KV_STAGE;
            bar_expect(&kv_full[s], KV_STAGE);
            tma_2d(st + 0 * KBOX, &kmap, kvh * D, j0, &kv_full[s]);
            tma_2d(st + 1 * KBOX, &kmap, kvh * D + 64, j0, &kv_full[s]);
            tma_2d(st + 2 * KBOX, &vmap, kvh * D, j0, &kv_full[s]);
            tma_2d(st + 3 * KBOX, &vmap, kvh * D + 64, j0, &kv_full[s]);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ================= MMA issuer (one thread)
    if (lane == 0) {
      int cur_mtile = -1, qn = 0, t = 0;
      int pending = -1;            // global index of the tile whose PV is not issued yet
      bool pending_first = false;  // that tile opens its unit (PV overwrites O)
      auto issue_pv = [&](int tp, bool first) {
        bar_wait(p_full, tp & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* vst = kvs + (tp % STAGES) * KV_STAGE + 2 * KBOX;
#pragma unroll
        for (int hl = 0; hl < 2; ++hl)
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk) {
            const uint8_t* a = ps + hl * QBOX + 32 * kk;          // P (K-major: keys along the row)
            const uint8_t* b = vst + kk * 16 * 128;              // V (MN-major: d along the row)
            umma(tmem_o, umma_desc(a), umma_desc(b, KBOX), kIdescPV, (first && hl == 0 && kk == 0) ? 0u : 1u);
          }
        umma_commit(&kv_empty[tp % STAGES]);
        umma_commit(pv_done);
      };
      for (int u = u0; u < u1; ++u) {
        int mtile, it0, it1;
        unit_of(p, u, mtile, it0, it1);
        bool first_tile = true;
        for (int it = it0; it < it1; ++it) {
          int lo, hi;
          item_range(p, it, lo, hi);
          for (int j0 = lo; j0 < hi; j0 += BN, ++t) {
            if (mtile != cur_mtile) {
              if (qn > 0) umma_commit(q_empty);      // Q slot free once the QKs issued so far finish
              bar_wait(q_full, qn & 1);
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
              cur_mtile = mtile;
              ++qn;
            }
            const int s = t % STAGES, buf = t & 1;
            bar_wait(&kv_full[s], (t / STAGES) & 1);
            if (t >= 2) bar_wait(&s_empty[buf], ((t / 2) - 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t dS = tmem + buf * BN;
            const uint8_t* kst = kvs + s * KV_STAGE;
#pragma unroll
            for (int hl = 0; hl < 2; ++hl)
#pragma unroll
              for (int k = 0; k < D / 16; ++k) {
                const uint8_t* a = qs + (2 * hl + k / 4) * QBOX + 32 * (k % 4);
                const uint8_t* b = kst + (k / 4) * KBOX + 32 * (k % 4);
                umma(dS, umma_desc(a), umma_desc(b), kIdescQK, (hl | k) ? 1u : 0u);
              }
            umma_commit(&s_full[buf]);
            if (pending >= 0) issue_pv(pending, pending_first);
            pending = t;
            pending_first = first_tile;
            first_tile = false;
          }
        }
      }
      if (pending >= 0) issue_pv(pending, pending_first);
    }
  } else {
    // ================= softmax / epilogue: warps 0-3, thread = TMEM lane = stacked row
    const int r = warp * 32 + lane;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    uint8_t* prow_hi = ps + r * 128;
    uint8_t* prow_lo = ps + QBOX + r * 128;
    const int sw = r & 7;
    int t = 0;
    int pv_seen = 0;               // PV completions consumed
    for (int u = u0; u < u1; ++u) {
      int mtile, it0, it1;
      unit_of(p, u, mtile, it0, it1);
      const int kvh = mtile / p.mtiles, mt = mtile - kvh * p.mtiles;
      const int c = u - mtile * p.n_chunks;
      const int R = mt * BM + r;
      const bool real = R < p.G * p.n_q;
      const int g = real ? R / p.n_q : 0, qi = real ? R - g * p.n_q : 0;
      const int h = kvh * p.G + g;
      const int64_t qpos = p.q_pos[qi];
      float m_run = -INFINITY, l_run = 0.f;   // O's reference max and running sum
      bool any_tile = false;
      for (int it = it0; it < it1; ++it) {
        int lo, hi;
        item_range(p, it, lo, hi);
        float m_it = -INFINITY, l_it = 0.f;    // this item's scoring statistics
        for (int j0 = lo; j0 < hi; j0 += BN, ++t) {
          const int buf = t & 1;
          // ---- visibility of the tile's keys (warp-cooperative, positions shared by all rows)
          const int nv = min(BN, hi - j0);
          int64_t kp0 = INT64_MAX, kp1 = INT64_MAX;
          if (lane < nv) {
            kp0 = p.k_pos[j0 + lane];
            if (p.allowed && !p.allowed[j0 + lane]) kp0 = INT64_MAX;
          }
          if (lane + 32 < nv) {
            kp1 = p.k_pos[j0 + 32 + lane];
            if (p.allowed && !p.allowed[j0 + 32 + lane]) kp1 = INT64_MAX;
          }
          int64_t kmax = kp0 > kp1 ? kp0 : kp1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const int64_t x = __shfl_xor_sync(0xffffffffu, kmax, o);
            kmax = x > kmax ? x : kmax;
          }
          const bool all_vis = kmax <= qpos;           // INT64_MAX (masked / past the item) fails

          bar_wait(&s_full[buf], (t / 2) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          float sc[BN];
          {
            float v0[32], v1[32];
            tmem_ld32(tmem + lane_base + buf * BN, v0);
            tmem_ld32(tmem + lane_base + buf * BN + 32, v1);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              sc[i] = v0[i];
              sc[32 + i] = v1[i];
            }
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) bar_arrive(&s_empty[buf]);

          if (!__all_sync(0xffffffffu, all_vis)) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int64_t a = __shfl_sync(0xffffffffu, kp0, i);
              const int64_t b = __shfl_sync(0xffffffffu, kp1, i);
              if (a > qpos) sc[i] = -INFINITY;
              if (b > qpos) sc[32 + i] = -INFINITY;
            }
          }
          float tmax = -INFINITY;
#pragma unroll
          for (int i = 0; i < BN; ++i) tmax = fmaxf(tmax, sc[i]);
          // ---- lazy online softmax: move the reference max only when it grows by > TAU
          const bool first = !any_tile;
          float m_new = m_run;
          if (first) m_new = tmax;
          else if (tmax > m_run + TAU) m_new = tmax;
          const float mu = (m_new == -INFINITY) ? 0.f : m_new;
          const float fac = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - mu);
          const bool rescale = !first && (m_new != m_run);
          float rs = 0.f;
          uint32_t hw[BN / 2], lw[BN / 2];
#pragma unroll
          for (int i = 0; i < BN; i += 2) {
            const float a = fast_exp2(sc[i] - mu), b = fast_exp2(sc[i + 1] - mu);
            rs += a + b;
            split_pack(a, b, hw[i / 2], lw[i / 2]);
          }
          l_run = (rescale ? l_run * fac : l_run) + rs;
          // ---- per-item scoring statistics (exact (m, l) pair of the item's keys)
          if (p.item_m && tmax != -INFINITY) {
            float tm = mu, tl = rs;
            if (tmax < mu - FALLBACK) {        // tile far below the reference: recompute exactly
              tm = tmax;
              tl = 0.f;
#pragma unroll
              for (int i = 0; i < BN; ++i) tl += fast_exp2(sc[i] - tmax);
            }
            if (m_it == -INFINITY) {
              m_it = tm;
              l_it = tl;
            } else {
              const float M = fmaxf(m_it, tm);
              l_it = l_it * fast_exp2(m_it - M) + tl * fast_exp2(tm - M);
              m_it = M;
            }
          }
          // ---- P (and O) may be touched once the previous tile's PV is complete
          if (t > 0 && pv_seen < t) {
            bar_wait(pv_done, (t - 1) & 1);
            pv_seen = t;
          }
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (__any_sync(0xffffffffu, rescale)) {
            const float f = rescale ? fac : 1.f;
#pragma unroll
            for (int cc = 0; cc < D / 32; ++cc) {
              float o[32];
              tmem_ld32(tmem_o + lane_base + 32 * cc, o);
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] *= f;
              tmem_st32(tmem_o + lane_base + 32 * cc, o);
            }
          }
          m_run = m_new;
          any_tile = true;
#pragma unroll
          for (int ch = 0; ch < BN / 8; ++ch) {
            const int off = ((ch ^ sw) << 4);
            *reinterpret_cast<uint4*>(prow_hi + off) =
                make_uint4(hw[4 * ch], hw[4 * ch + 1], hw[4 * ch + 2], hw[4 * ch + 3]);
            *reinterpret_cast<uint4*>(prow_lo + off) =
                make_uint4(lw[4 * ch], lw[4 * ch + 1], lw[4 * ch + 2], lw[4 * ch + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) bar_arrive(p_full);
        }
        if (p.item_m && real) {
          const int64_t o = ((int64_t)qi * p.hq + h) * p.n_items + it;
          p.item_m[o] = m_it;
          p.item_l[o] = l_it;
        }
      }
      // ---- unit end: O of the last tile, partial (m, l, O) for the merge
      const int64_t po = ((int64_t)qi * p.hq + h) * p.n_chunks + c;
      if (any_tile) {
        bar_wait(pv_done, (t - 1) & 1);
        pv_seen = t;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc) {
          float o[32];
          tmem_ld32(tmem_o + lane_base + 32 * cc, o);
          if (real) {
            float4* dst = reinterpret_cast<float4*>(p.part_o + po * D + 32 * cc);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      } else if (real) {
        float4* dst = reinterpret_cast<float4*>(p.part_o + po * D);
        for (int i = 0; i < D / 4; ++i) dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (real) {
        p.part_m[po] = m_run;
        p.part_l[po] = l_run;
      }
    }
  }
  __syncthreads();
  if (warp == 5) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// q [n_q][hq][128] fp32 -> Qs [hkv][2][mpad][128] bf16 (rows (g, i), log2 units, hi/lo split)
__global__ void prep_q_kernel(const float* __restrict__ q, int n_q, int hq, int hkv, int G, int mpad,
                              float scale_log2, __nv_bfloat16* __restrict__ qs) {
  const int64_t total = (int64_t)hkv * mpad * D;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(x % D);
    const int64_t rr = x / D;
    const int R = (int)(rr % mpad), kvh = (int)(rr / mpad);
    float v = 0.f;
    if (R < G * n_q) {
      const int g = R / n_q, i = R - g * n_q;
      v = q[((int64_t)i * hq + kvh * G + g) * D + e] * scale_log2;
    }
    const __nv_bfloat16 hb = __float2bfloat16_rn(v);
    const __nv_bfloat16 lb = __float2bfloat16_rn(v - __bfloat162float(hb));
    qs[(((int64_t)kvh * 2 + 0) * mpad + R) * D + e] = hb;
    qs[(((int64_t)kvh * 2 + 1) * mpad + R) * D + e] = lb;
  }
}

// out[i][h][:] = sum_c O_c 2^(m_c - M) / sum_c l_c 2^(m_c - M); one warp per (i, h).
// stat_m/stat_l (nullable): merged log2-domain max and sum (capture path).
__global__ void prefill_merge_kernel(const float* __restrict__ part_m, const float* __restrict__ part_l,
                                     const float* __restrict__ part_o, int n_rows_heads, int hq, int n_chunks,
                                     float* __restrict__ out, float* __restrict__ stat_m, float* __restrict__ stat_l,
                                     int32_t* __restrict__ bad_row) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= n_rows_heads) return;
  const float* pm = part_m + (int64_t)w * n_chunks;
  const float* pl = part_l + (int64_t)w * n_chunks;
  float M = -INFINITY;
  for (int c = 0; c < n_chunks; ++c) M = fmaxf(M, pm[c]);
  const float mu = M == -INFINITY ? 0.f : M;
  float L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c = 0; c < n_chunks; ++c) {
    const float lc = pl[c];
    if (lc == 0.f) continue;
    const float f = exp2f(pm[c] - mu);
    L += lc * f;
    const float4 o = reinterpret_cast<const float4*>(part_o + ((int64_t)w * n_chunks + c) * D)[lane];
    acc.x += o.x * f;
    acc.y += o.y * f;
    acc.z += o.z * f;
    acc.w += o.w * f;
  }
  const float inv = L > 0.f ? 1.f / L : 0.f;
  reinterpret_cast<float4*>(out + (int64_t)w * D)[lane] =
      make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  if (lane == 0) {
    if (stat_m) {
      stat_m[w] = M;
      stat_l[w] = L;
    }
    if (L == 0.f && bad_row) atomicMin(bad_row, w / hq);
  }
}

}  // namespace pf

bool prefill_tc_supported(int kv_dtype, int d, int n_q, int G) {
  return kv_dtype == RK_BF16 && d == 128 && (int64_t)n_q * G >= 64 && G <= 16;
}

// item table: `items` (n_items given) or uniform items of item_keys keys over s
PrefillPlan prefill_plan(int n_q, int hq, int hkv, int s, int n_items_in, bool stats) {
  PrefillPlan pl{};
  const int G = hq / hkv;
  pl.mpad = (G * n_q + pf::BM - 1) / pf::BM * pf::BM;
  pl.mtiles = pl.mpad / pf::BM;
  const int mt_total = hkv * pl.mtiles;
  if (n_items_in > 0) {
    pl.n_items = n_items_in;
    pl.item_keys = 0;
  } else {
    pl.item_keys = 512;
    pl.n_items = s > 0 ? (s + pl.item_keys - 1) / pl.item_keys : 1;
  }
  // ~8 units per SM: balance over the persistent CTAs, >= 1 item per chunk
  const int target = 8 * sm_count();
  int nc = (target + mt_total - 1) / mt_total;
  nc = std::max(1, std::min(nc, pl.n_items));
  pl.items_per_chunk = (pl.n_items + nc - 1) / nc;
  pl.n_chunks = (pl.n_items + pl.items_per_chunk - 1) / pl.items_per_chunk;
  pl.n_units = mt_total * pl.n_chunks;
  pl.qs_bytes = align_up((size_t)hkv * 2 * pl.mpad * pf::D * 2, 256);
  const size_t rh = (size_t)n_q * hq;
  pl.part_bytes = align_up(rh * pl.n_chunks * 4, 256) * 2 + align_up(rh * pl.n_chunks * pf::D * 4, 256);
  pl.item_bytes = stats ? align_up(rh * pl.n_items * 4, 256) * 2 : 0;
  pl.total = pl.qs_bytes + pl.part_bytes + pl.item_bytes + align_up(rh * 4, 256) * 2;
  return pl;
}

// Launch prep + tensor-core pass + merge.  ws must hold prefill_plan(...).total
// bytes.  item_m/item_l (stats) are carved from ws and returned for the
// scoring finalisation; stat_m/stat_l likewise (capture path).
int launch_prefill_tc(const float* q, int n_q, int hq, const void* k, const void* v, int s, int hkv,
                      const int64_t* q_pos, const int64_t* k_pos, const uint8_t* allowed, const int32_t* items,
                      int n_items_in, bool stats, float* out, int32_t* bad_row, void* ws, size_t ws_bytes,
                      float** item_m_out, float** item_l_out, float** stat_m_out, float** stat_l_out,
                      cudaStream_t st) {
  const int G = hq / hkv;
  PrefillPlan pl = prefill_plan(n_q, hq, hkv, s, items ? n_items_in : 0, stats);
  if (pl.total > ws_bytes) return fail(RK_ERR_CAPACITY, "prefill workspace %zu < %zu", ws_bytes, pl.total);
  char* b = static_cast<char*>(ws);
  const size_t rh = (size_t)n_q * hq;
  __nv_bfloat16* qs = reinterpret_cast<__nv_bfloat16*>(b);
  b += pl.qs_bytes;
  float* part_m = reinterpret_cast<float*>(b);
  b += align_up(rh * pl.n_chunks * 4, 256);
  float* part_l = reinterpret_cast<float*>(b);
  b += align_up(rh * pl.n_chunks * 4, 256);
  float* part_o = reinterpret_cast<float*>(b);
  b += align_up(rh * pl.n_chunks * pf::D * 4, 256);
  float* item_m = nullptr;
  float* item_l = nullptr;
  if (stats) {
    item_m = reinterpret_cast<float*>(b);
    b += align_up(rh * pl.n_items * 4, 256);
    item_l = reinterpret_cast<float*>(b);
    b += align_up(rh * pl.n_items * 4, 256);
  }
  float* stat_m = reinterpret_cast<float*>(b);
  b += align_up(rh * 4, 256);
  float* stat_l = reinterpret_cast<float*>(b);
  if (item_m_out) *item_m_out = item_m;
  if (item_l_out) *item_l_out = item_l;
  if (stat_m_out) *stat_m_out = stat_m;
  if (stat_l_out) *stat_l_out = stat_l;

  pf::prep_q_kernel<<<(int)std::min<int64_t>(4096, ((int64_t)hkv * pl.mpad * pf::D + 255) / 256), 256, 0, st>>>(
      q, n_q, hq, hkv, G, pl.mpad, (float)(1.4426950408889634 / std::sqrt(128.0)), qs);
  RK_CHECK_LAUNCH("prefill prep_q_kernel");
  CUtensorMap qmap, kmap, vmap;
  int r = tc::make_map(&qmap, qs, pf::D, (uint64_t)hkv * 2 * pl.mpad, pf::D * 2, pf::BM);
  if (r) return r;
  r = tc::make_map(&kmap, k, (uint64_t)hkv * pf::D, (uint64_t)s, (uint64_t)hkv * pf::D * 2, pf::BN);
  if (r) return r;
  r = tc::make_map(&vmap, v, (uint64_t)hkv * pf::D, (uint64_t)s, (uint64_t)hkv * pf::D * 2, pf::BN);
  if (r) return r;
  pf::Params p{};
  p.n_q = n_q; p.hq = hq; p.hkv = hkv; p.G = G; p.mpad = pl.mpad; p.mtiles = pl.mtiles;
  p.n_items = pl.n_items; p.n_chunks = pl.n_chunks; p.items_per_chunk = pl.items_per_chunk;
  p.n_units = pl.n_units; p.item_keys = pl.item_keys; p.s = s;
  p.q_pos = q_pos; p.k_pos = k_pos; p.allowed = allowed; p.items = items;
  p.item_m = item_m; p.item_l = item_l;
  p.part_m = part_m; p.part_l = part_l; p.part_o = part_o;
  static bool configured = false;
  if (!configured) {
    RK_CUDA(cudaFuncSetAttribute(pf::prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pf::SMEM),
            "prefill_tc smem attribute");
    configured = true;
  }
  const int grid = std::min(sm_count(), pl.n_units);
  pf::prefill_tc_kernel<<<grid, pf::THREADS, pf::SMEM, st>>>(qmap, kmap, vmap, p);
  RK_CHECK_LAUNCH("prefill_tc_kernel");
  const int nrh = (int)rh;
  pf::prefill_merge_kernel<<<(nrh * 32 + 255) / 256, 256, 0, st>>>(part_m, part_l, part_o, nrh, hq, pl.n_chunks,
                                                                   out, stat_m, stat_l, bad_row);
  RK_CHECK_LAUNCH("prefill_merge_kernel");
  return RK_OK;
}

}  // namespace rk
