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
// chunk = a run of items) the CTA streams 128-key tiles of K and V:
//   S  = Q_hi K^T + Q_lo K^T            tcgen05.mma m128n128k16 x 16 -> TMEM
//   P  = exp2(S - m) (online, lazy rescale), split P = P_hi + P_lo (bf16),
//        written back over its own S columns in TMEM (bf16x2 per column)
//   O += P_hi V + P_lo V                tcgen05.mma m128n128k16 x 8, A = P from
//                                        TMEM, B = V read MN-major from its TMA tile
// The q and P splits keep ~16 mantissa bits (fp32-class outputs; the reference
// tolerance is 1e-3 relative, fp64 accumulation on its side).  Three S/P
// buffers let QK run a tile ahead of the softmax, and the softmax never
// waits for the previous tile's PV (only the rare O rescale does).
//
// CTA roles (352 threads, one CTA per SM, persistent over a contiguous range
// of units so Q is reloaded only when the range crosses an M tile):
//   warps 0-7  softmax / epilogue: TMEM lane quarter = warp & 3 (a thread owns
//              one stacked row), column half = warp >> 2 — the two warps of a
//              row (same SMSP) agree on the row max through a 64-thread named
//              barrier per tile.  They read S with tcgen05.ld, mask, run the
//              online softmax (packed f32x2 math), write P with tcgen05.st and
//              the per-item scoring statistics; rescale their half of O in
//              TMEM when the running max moves by more than 2^8; at unit end
//              read O and write the unit's partial (m, l, O) for the merge;
//   warp 8     TMEM allocation + single-thread MMA issue;
//   warp 9     TMA producer of Q hi/lo [128 x 128] per M tile and K [128 keys
//              x 128] per tile (2-stage ring, freed after its QK); the warp
//              also reduces each tile's key positions to one maximum so fully
//              visible tiles skip the per-key causal mask;
//   warp 10    TMA producer of V [128 keys x 128] per tile (2-stage ring, freed
//              after its PV).  All tiles SWIZZLE_128B.
#include <cmath>
#include <cstdlib>

#include <algorithm>

#include "prefill_tc.cuh"
#include "tc_common.cuh"

namespace rk {
namespace pf {

using namespace tc;

constexpr int BM = 128, BN = 128, D = 128;   // rows, keys per tile, head dim
constexpr int STAGES = 4;                // K ring and V ring depth
constexpr int MR = 8;                    // tile-visibility metadata ring
constexpr int NB = 3;                    // S/P buffers in TMEM (3 x 128 columns + O = 512)
constexpr int LA = NB - 1;               // QK runs LA tiles ahead (its buffer is freed by the PV queued before)
constexpr int QBOX = BM * 64 * 2;        // 128 rows x 64 bf16, swizzled: 16 KB
constexpr int Q_BYTES = 4 * QBOX;        // q_hi, q_lo x two 64-dim halves
// CTA pair (cta_group::2): an M tile is 256 stacked rows, CTA rank r owns rows
// [128r, 128r+128) (its Q, S, P, O); the B operands are split by N: CTA r holds
// keys [64r, 64r+64) of a K tile and head dims [64r, 64r+64) of a V tile.
constexpr int PM = 2 * BM;               // rows per pair M tile
constexpr int KBOX = (BN / 2) * 64 * 2;  // 64 keys x 64 bf16: 8 KB
constexpr int K_STAGE = 2 * KBOX;        // this CTA's K half-tile (64 keys x 128 dims): 16 KB
constexpr int VBOX = BN * 64 * 2;        // 128 keys x 64 dims: 16 KB
constexpr int V_STAGE = VBOX;            // this CTA's V half-tile (128 keys x 64 dims): 16 KB
constexpr int kSoftmaxWarps = 8, kMmaWarp = 8, kProducerWarp = 9, kVProducerWarp = 10;
constexpr int THREADS = 352;
constexpr int BAR_BYTES = 512;           // mbarriers, TMEM slot, per-stage tile maxima
constexpr int XCH_BYTES = (2 * 256 + 3 * 128) * 4;  // row-max exchange (2 tiles x 2 halves) + item / unit sums
constexpr size_t SMEM = 1024 + Q_BYTES + STAGES * (K_STAGE + V_STAGE) + BAR_BYTES + XCH_BYTES;
constexpr uint32_t TMEM_COLS = 512;      // S/P buffers NB x 128 at 0.., O (128) at NB * 128 (= 384)
constexpr float TAU = 8.f;               // lazy rescale threshold (log2 units)

constexpr uint32_t kIdescQK = idesc_f16(PM, BN);             // S[256 x 128] = Q K^T (both K-major, smem)
constexpr uint32_t kIdescPV = idesc_f16(PM, D, true);        // O[256 x 128] += P V (P from TMEM, V MN-major)

struct Params {
  int n_q, hq, hkv, G, mpad, mtiles;
  int n_items, n_chunks, items_per_chunk, n_units;
  int item_keys;                   // uniform items when items == nullptr
  int s;                           // keys
  const int64_t* q_pos;            // [n_q]
  const int64_t* k_pos;            // [s]
  const uint8_t* allowed;          // [s] or null
  const int32_t* items;            // [n_items][3] (lo, hi, bin) or null (uniform)
  float* item_m;                   // [n_q][hq][n_items][2 column halves] scoring statistics or null
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

// Units are chunk-major: at any moment the persistent CTAs work on the M tiles
// of (about) one key chunk, so the chunk's K/V (all kv-heads: the rows are
// contiguous) is fetched from DRAM once and served to every M tile from L2.
__device__ __forceinline__ int unit_chunk(const Params& p, int u) { return u / (p.hkv * p.mtiles); }

__device__ __forceinline__ void unit_of(const Params& p, int u, int& mtile, int& it0, int& it1) {
  const int c = unit_chunk(p, u);
  mtile = u - c * (p.hkv * p.mtiles);
  it0 = c * p.items_per_chunk;
  it1 = min(p.n_items, it0 + p.items_per_chunk);
}

// Walks the 128-key tiles of the CTA's units in order (units without keys are skipped).
struct TileIter {
  const Params* p;
  int u, u1, it, it1, lo, hi, j0, mtile;
  bool first, valid;
  __device__ void init(const Params& P, int ua, int ub) {
    p = &P;
    u = ua - 1;
    u1 = ub;
    valid = true;
    next_unit();
  }
  __device__ void next_unit() {
    while (true) {
      if (++u >= u1) {
        valid = false;
        return;
      }
      unit_of(*p, u, mtile, it, it1);
      for (; it < it1; ++it) {
        item_range(*p, it, lo, hi);
        if (hi > lo) {
          j0 = lo;
          first = true;
          return;
        }
      }
    }
  }
  __device__ void advance() {
    first = false;
    j0 += BN;
    if (j0 < hi) return;
    for (++it; it < it1; ++it) {
      item_range(*p, it, lo, hi);
      if (hi > lo) {
        j0 = lo;
        return;
      }
    }
    next_unit();
  }
};

#ifdef PF_PROF
// [role][slot] accumulated cycles; role 0 softmax (warp 0 lane 0), 1 MMA, 2 K producer, 3 V producer
__device__ unsigned long long g_pf_prof[4][16];
#define PWAIT(bar, par, role, slot)                                                     \
  do {                                                                                  \
    const long long _t0 = clock64();                                                    \
    bar_wait(bar, par);                                                                 \
    if ((threadIdx.x & 31) == 0 && (role != 0 || threadIdx.x == 0))                     \
      atomicAdd(&g_pf_prof[role][slot], (unsigned long long)(clock64() - _t0));         \
  } while (0)
#else
#define PWAIT(bar, par, role, slot) bar_wait(bar, par)
#endif

// TMA into this CTA's smem, completion bytes counted on the pair leader's
// barrier (bar_cluster: shared::cluster address from mapa(.., 0))
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of a shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sa(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void bar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// pair MMAs (issued by the leader; A rows and B columns split across the pair)
__device__ __forceinline__ void umma2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}
// completion of the leader's MMAs issued so far -> the barrier at this offset in both CTAs
__device__ __forceinline__ void umma2_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      ::"r"(sa(bar)), "h"((unsigned short)3)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// SWIZZLE_128B descriptor from a 32-bit shared address (see tc::umma_desc);
// later k-slices add (byte offset >> 4) to the start-address field
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo_bytes) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// 2^x for a pair on the FMA pipe (the MUFU ex2 pipe does 16/clk/SM and is the
// softmax's bottleneck): x = j + f with j = rint(x) from the 1.5*2^23 magic
// add, 2^f by a degree-5 minimax polynomial on [-1/2, 1/2] (max rel. error
// 2.2e-7 in fp32 Horner, the class of ex2.approx), j added to the exponent
// bits; x < -126.5 gives 0 like ex2.approx.ftz.
// Pairs (of every 8) whose exp2 runs on the FMA pipe.  Measured at C3
// (tools/bench_prefill.py, n_q 512): prefill 0.788 / 0.797 / 0.808 / 0.851 ms
// for 0 / 1 / 2 / 3 of 8 — the attention softmax is issue-bound, not MUFU-bound;
// the scores-only pass (no PV) is: 0.630 / 0.594 / 0.601 / 0.624 ms.
#ifndef PF_POLY_OF8
#define PF_POLY_OF8 0                    // attention (prefill) softmax
#endif
#ifndef PF_POLY_OF8_SCORE
#define PF_POLY_OF8_SCORE 1              // scores-only pass
#endif
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  const float2 one = make_float2(1.f, 1.f), mone = make_float2(-1.f, -1.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 xc = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
  const float2 t = ffma2(xc, one, magic);                 // 1.5*2^23 + rint(x)
  const float2 j = ffma2(magic, mone, t);                 // rint(x)
  const float2 f = ffma2(j, mone, xc);                    // x - rint(x) in [-1/2, 1/2]
  float2 p = make_float2(0.0013291972f, 0.0013291972f);
  p = ffma2(p, f, make_float2(0.009675695561f, 0.009675695561f));
  p = ffma2(p, f, make_float2(0.05550665781f, 0.05550665781f));
  p = ffma2(p, f, make_float2(0.2402211577f, 0.2402211577f));
  p = ffma2(p, f, make_float2(0.6931470037f, 0.6931470037f));
  p = ffma2(p, f, make_float2(1.0000001192f, 1.0000001192f));
  float2 r;
  r.x = __int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23));
  r.y = __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23));
  r.x = x.x < -126.5f ? 0.f : r.x;
  r.y = x.y < -126.5f ? 0.f : r.y;
  return r;
}

__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// tcgen05.mma with A from TMEM (kind::f16, A K-major: row = lane, 2 bf16 per column)
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_st32u(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
        "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SCORE_ONLY: the watershed scorer (rk_round_scores) — QK^T and the per-item
// softmax statistics only: no V, no PV, no O, no row-max exchange.
// SPLIT (default): q and P as bf16 hi + lo, two MMA passes each (fp32-class
// outputs).  !SPLIT: the single-pass bf16 path (bf16 q and P, one pass each,
// bf16-class outputs; rk_prefill_attention flag RK_PREFILL_SINGLE_PASS).
template <bool SCORE_ONLY, bool SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
prefill_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                  const __grid_constant__ CUtensorMap vmap, const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* qs = smem;                               // [hi d0-63 | hi d64-127 | lo d0-63 | lo d64-127]
  uint8_t* ks = qs + Q_BYTES;                       // STAGES x [K d0-63 | K d64-127] of this CTA's 64 keys
  uint8_t* vs = ks + STAGES * K_STAGE;              // STAGES x [V, this CTA's 64 dims] of 128 keys
  uint64_t* bars = reinterpret_cast<uint64_t*>(vs + STAGES * V_STAGE);
  uint64_t* k_full = bars;                          // [STAGES] both CTAs' TMA -> leader's MMA (leader's copy used)
  uint64_t* k_empty = k_full + STAGES;              // [STAGES] QK done -> producers (multicast)
  uint64_t* v_full = k_empty + STAGES;              // [STAGES] both CTAs' TMA -> leader's MMA
  uint64_t* v_empty = v_full + STAGES;              // [STAGES] PV done -> producers (multicast)
  uint64_t* meta_full = v_empty + STAGES;           // [MR] producer -> softmax (tile_max)
  uint64_t* q_full = meta_full + MR;
  uint64_t* q_empty = q_full + 1;
  uint64_t* s_full = q_full + 2;                    // [NB] QK done -> softmax
  uint64_t* p_full = s_full + NB;                   // [NB] P written (8 + 8 softmax warps of the pair) -> leader
  uint64_t* buf_free = p_full + NB;                 // [NB] PV done: S/P buffer reusable, O stable
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(buf_free + NB);
  // per tile (ring of MR): the largest effective key position of the tile
  // (masked or out-of-item keys count as +inf), published through meta_full
  int64_t* tile_max = reinterpret_cast<int64_t*>(buf_free + NB + 1);
  float* xmax = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + BAR_BYTES);   // [2][2][128]
  float* xm_it = xmax + 512;                        // [128]
  float* xl_it = xm_it + 128;                       // [128]
  float* xl_u = xl_it + 128;                        // [128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int u0 = (int)((int64_t)pair * p.n_units / npairs);
  const int u1 = (int)((int64_t)(pair + 1) * p.n_units / npairs);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&k_full[s], 1);
      bar_init(&k_empty[s], 1);
      bar_init(&v_full[s], 1);
      bar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < MR; ++s) bar_init(&meta_full[s], 1);
    bar_init(q_full, 1);
    bar_init(q_empty, 1);
    for (int b = 0; b < NB; ++b) {
      bar_init(&s_full[b], 1);
      bar_init(&p_full[b], 2 * kSoftmaxWarps);
      bar_init(&buf_free[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // both CTAs' barriers initialised before any remote arrive; also orders the
  // pair allocation below after both CTAs' start-up writes of the reserved
  // shared-memory words tcgen05.alloc.cta_group::2 reads (compute-sanitizer
  // racecheck reported that read, at reserved offsets 0x58-0x5f of both CTAs,
  // as a RAW hazard against the launch preamble when the alloc came first)
  cluster_sync();
  if (warp == kMmaWarp) {     // same warp in both CTAs: the pair's TMEM (same columns on both SMs)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  __syncthreads();            // the TMEM address is in this CTA's slot
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_o = tmem + NB * BN;
#ifdef PF_PROF
  const long long prof_t0 = clock64();
#endif

  if (warp == kProducerWarp) {
    // ================= K (+ Q) producer (lane 0 issues; the warp computes tile visibility)
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&qmap) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&kmap) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&vmap) : "memory");
    }
    const uint32_t qs_a = sa(qs), ks_a = sa(ks);
    const uint32_t q_full_l = mapa(q_full, 0);     // the leader's barriers count both CTAs' bytes
    TileIter ti, ta;                                // ta runs PF tiles ahead: key-position prefetch
    ti.init(p, u0, u1);
    ta.init(p, u0, u1);
    constexpr int PF = 3;
    int64_t pk[PF][BN / 32];                        // prefetched effective positions, pk[0] = current tile
    // shift the ring by one tile and load the tile `ta` points at into its tail
    auto fetch = [&]() {
#pragma unroll
      for (int sl = 0; sl + 1 < PF; ++sl)
#pragma unroll
        for (int i = 0; i < BN / 32; ++i) pk[sl][i] = pk[sl + 1][i];
#pragma unroll
      for (int i = 0; i < BN / 32; ++i) pk[PF - 1][i] = INT64_MAX;
      if (ta.valid) {
        const int nv = min(BN, ta.hi - ta.j0);
#pragma unroll
        for (int i = 0; i < BN / 32; ++i) {
          const int jj = 32 * i + lane;
          if (jj < nv && (!p.allowed || p.allowed[ta.j0 + jj])) pk[PF - 1][i] = p.k_pos[ta.j0 + jj];
        }
        ta.advance();
      }
    };
#pragma unroll
    for (int i = 0; i < PF; ++i) fetch();
    int cur_mtile = -1, qn = 0;
    for (int t = 0; ti.valid; ++t, ti.advance()) {
      const int kvh = ti.mtile / p.mtiles, mt = ti.mtile - kvh * p.mtiles;
      if (ti.mtile != cur_mtile) {
        if (qn > 0) PWAIT(q_empty, (qn - 1) & 1, 2, 1);
        if (elect_one()) {
          if (leader) bar_expect(q_full, 2 * Q_BYTES);
          const int row0 = kvh * 2 * p.mpad + mt * PM + BM * (int)rank;   // this CTA's 128 rows
          tma_2d_pair(qs_a + 0 * QBOX, &qmap, 0, row0, q_full_l);
          tma_2d_pair(qs_a + 1 * QBOX, &qmap, 64, row0, q_full_l);
          tma_2d_pair(qs_a + 2 * QBOX, &qmap, 0, row0 + p.mpad, q_full_l);
          tma_2d_pair(qs_a + 3 * QBOX, &qmap, 64, row0 + p.mpad, q_full_l);
        }
        __syncwarp();
        cur_mtile = ti.mtile;
        ++qn;
      }
      const int s = t % STAGES, j0 = ti.j0;
      // effective positions of the tile's keys, loaded PF tiles ago
      int64_t kmax = INT64_MIN;
#pragma unroll
      for (int i = 0; i < BN / 32; ++i) kmax = pk[0][i] > kmax ? pk[0][i] : kmax;
      fetch();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t x = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmax = x > kmax ? x : kmax;
      }
      if (t >= STAGES) PWAIT(&k_empty[s], ((t / STAGES) - 1) & 1, 2, 0);
      if (elect_one()) {
        tile_max[t % MR] = kmax;
        bar_arrive(&meta_full[t % MR]);               // release: tile_max visible with the phase
        if (leader) bar_expect(&k_full[s], 2 * K_STAGE);
        const uint32_t kb = mapa(&k_full[s], 0);
        const int jr = j0 + (BN / 2) * (int)rank;      // this CTA's 64 keys of the tile
        tma_2d_pair(ks_a + s * K_STAGE, &kmap, kvh * D, jr, kb);
        tma_2d_pair(ks_a + s * K_STAGE + KBOX, &kmap, kvh * D + 64, jr, kb);
      }
      __syncwarp();
    }
  } else if (warp == kVProducerWarp) {
    if (!SCORE_ONLY) {
      // ================= V producer: V of tile t once PV_{t-STAGES} freed its slot
      // (a separate warp so the K loads, needed a tile earlier, never queue behind it)
      TileIter ti;
      ti.init(p, u0, u1);
      const uint32_t vs_a = sa(vs);
      for (int t = 0; ti.valid; ++t, ti.advance()) {
        const int kvh = ti.mtile / p.mtiles, s = t % STAGES;
        if (t >= STAGES) PWAIT(&v_empty[s], ((t / STAGES) - 1) & 1, 3, 0);
        if (elect_one()) {                           // this CTA's 64 head dims of all 128 keys
          if (leader) bar_expect(&v_full[s], 2 * V_STAGE);
          tma_2d_pair(vs_a + s * V_STAGE, &vmap, kvh * D + 64 * (int)rank, ti.j0, mapa(&v_full[s], 0));
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    if (leader) {
      // ================= MMA issuer.  The whole warp runs the (uniform) control
      // flow and one elected lane issues, so descriptors live in uniform
      // registers; each tile's descriptors are built once and advanced by
      // compile-time offsets.  Order: QK of the LA tiles ahead, then per tile t:
      // PV_t (after its P), QK_{t+LA} into the buffer PV_{t-1} frees — the
      // issuer never waits on the PV it just issued, and the tensor pipe always
      // holds queued work.  (LA = NB - 1: QK_{t+LA} reuses the buffer of PV_{t-1},
      // which sits ahead of PV_t in the tensor queue and is normally done.)
      // Only the pair leader issues (cta_group::2 MMAs over both SMs' operands);
      // every commit arrives on the barrier at the same offset in both CTAs.
      TileIter qi, pi;
      qi.init(p, u0, u1);
      pi.init(p, u0, u1);
      const uint32_t qs_a = sa(qs), ks_a = sa(ks), vs_a = sa(vs);
      int tq = 0, tp = 0, cur_mtile = -1, qn = 0;
      auto issue_qk = [&]() {
        if (qi.mtile != cur_mtile) {
          if (qn > 0 && elect_one()) umma2_commit(q_empty);   // Q slot free once the QKs issued so far finish
          __syncwarp();
          PWAIT(q_full, qn & 1, 1, 0);
          cur_mtile = qi.mtile;
          ++qn;
        }
        const int b = tq % NB, s = tq % STAGES;
        if (tq >= NB) PWAIT(&buf_free[b], ((tq / NB) - 1) & 1, 1, 1);
        PWAIT(&k_full[s], (tq / STAGES) & 1, 1, 2);
        fence_after();
        if (elect_one()) {
          const uint32_t dS = tmem + b * BN;
          const uint64_t a0 = desc_sw128(qs_a, 16);
          const uint64_t b0 = desc_sw128(ks_a + s * K_STAGE, 16);     // this CTA's 64 keys (peer: same offset)
  #pragma unroll
          for (int hl = 0; hl < (SPLIT ? 2 : 1); ++hl)          // q_hi, q_lo
  #pragma unroll
            for (int k = 0; k < D / 16; ++k) {
#ifdef PF_MMA_ONE                                       // timing experiment only (wrong scores)
              if (SCORE_ONLY && (hl | k)) continue;
#endif
              umma2(dS, a0 + (uint64_t)((((2 * hl + k / 4) * QBOX) + 32 * (k % 4)) >> 4),
                   b0 + (uint64_t)((((k / 4) * KBOX) + 32 * (k % 4)) >> 4), kIdescQK, (hl | k) ? 1u : 0u);
            }
          umma2_commit(&k_empty[s]);                   // K slots free once this QK completes
          umma2_commit(&s_full[b]);
        }
        __syncwarp();
        ++tq;
        qi.advance();
      };
      for (int i = 0; i < LA && qi.valid; ++i) issue_qk();
      while (pi.valid) {
        const int b = tp % NB, s = tp % STAGES;
        PWAIT(&p_full[b], (tp / NB) & 1, 1, 3);
        if (SCORE_ONLY) {               // S_tp consumed: its buffer is free (nothing async to wait for)
          if (elect_one()) bar_arrive(&buf_free[b]);
          __syncwarp();
          ++tp;
          pi.advance();
          if (qi.valid) issue_qk();
          continue;
        }
        PWAIT(&v_full[s], (tp / STAGES) & 1, 1, 4);
        fence_after();
        if (elect_one()) {
          const uint64_t b0 = desc_sw128(vs_a + s * V_STAGE, VBOX);    // V MN-major, one 64-dim atom per CTA
          const uint32_t a0 = tmem + b * BN;                             // P_hi | P_lo (16 keys = 8 columns)
          const bool first = pi.first;
  #pragma unroll
          for (int hl = 0; hl < (SPLIT ? 2 : 1); ++hl)          // P_hi, P_lo
  #pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk) {
              umma2_ts(tmem_o, a0 + hl * (BN / 2) + kk * 8, b0 + (uint64_t)((kk * 16 * 128) >> 4), kIdescPV,
                      (first && hl == 0 && kk == 0) ? 0u : 1u);
            }
          umma2_commit(&v_empty[s]);
          umma2_commit(&buf_free[b]);
        }
        __syncwarp();
        ++tp;
        pi.advance();
        if (qi.valid) issue_qk();
      }
    }
  } else {
    // ================= softmax / epilogue: warps 0-7.  TMEM lane quarter q4 =
    // warp & 3 (rows 32*q4 ..), column half = warp >> 2: each row's 64 scores
    // and 128 O columns are split over two warps (same SMSP), which agree on
    // the row max through a 64-thread named barrier per tile.
    const int q4 = warp & 3, half = warp >> 2;
    const int r = q4 * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const int bar_id = 1 + q4;
    int t = 0;
    for (int u = u0; u < u1; ++u) {
      int mtile, it0, it1;
      unit_of(p, u, mtile, it0, it1);
      const int kvh = mtile / p.mtiles, mt = mtile - kvh * p.mtiles;
      const int c = unit_chunk(p, u);
      const int R = mt * PM + BM * (int)rank + r;   // stacked row of this CTA's half of the pair tile
      const bool real = R < p.G * p.n_q;
      const int g = real ? R / p.n_q : 0, qi = real ? R - g * p.n_q : 0;
      const int h = kvh * p.G + g;
      const int64_t qpos = p.q_pos[qi];
      float m_run = -INFINITY, l_half = 0.f;  // O's reference max (shared by the pair), this half's sum
      bool any_tile = false;
      for (int it = it0; it < it1; ++it) {
        int lo, hi;
        item_range(p, it, lo, hi);
        float m_it = -INFINITY, l_it = 0.f;    // this half's scoring statistics of the item
        for (int j0 = lo; j0 < hi; j0 += BN, ++t) {
          const int b = t % NB;
          // ---- visibility: the producer's tile maximum
          PWAIT(&meta_full[t % MR], (t / MR) & 1, 0, 0);
          const bool all_vis = tile_max[t % MR] <= qpos;   // +inf (masked / past the item) fails

          PWAIT(&s_full[b], (t / NB) & 1, 0, 1);
          fence_after();
          constexpr int HK = BN / 2;                    // keys per column half
          float sc[HK];
          {
            float v0[32], v1[32];
            tmem_ld32(tmem + lane_base + b * BN + HK * half, v0);
            tmem_ld32(tmem + lane_base + b * BN + HK * half + 32, v1);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              sc[i] = v0[i];
              sc[32 + i] = v1[i];
            }
          }
          if (SCORE_ONLY) {                             // S is in registers: release the buffer now
            fence_before();
            __syncwarp();
            if (lane == 0) {
              if (leader) bar_arrive(&p_full[b]);
              else bar_arrive_cluster(mapa(&p_full[b], 0));
            }
          }

          if (!__all_sync(0xffffffffu, all_vis)) {     // diagonal / masked tile: per-key check
            const int nv = min(BN, hi - j0);
#pragma unroll
            for (int c = 0; c < HK / 32; ++c) {
              const int jj = HK * half + 32 * c + lane;
              int64_t kp = INT64_MAX;
              if (jj < nv && (!p.allowed || p.allowed[j0 + jj])) kp = p.k_pos[j0 + jj];
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (__shfl_sync(0xffffffffu, kp, i) > qpos) sc[32 * c + i] = -INFINITY;
            }
          }
          // four independent FMNMX3 chains (one serial chain of 32 sat on the
          // softmax's per-tile critical path); the max is order-free
          float hm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int i = 0; i < HK; i += 8)
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) hm[c4] = fmaxf(fmaxf(hm[c4], sc[i + 2 * c4]), sc[i + 2 * c4 + 1]);
          const float hmax = fmaxf(fmaxf(hm[0], hm[1]), fmaxf(hm[2], hm[3]));
          if (SCORE_ONLY) {
            // this half's (max, sum) of the tile, folded into the item statistics
#ifdef PF_EXP_OFF                                   // timing experiment only (wrong masses)
            if (false) {
#else
            if (hmax != -INFINITY) {
#endif
              float2 acc[4];                           // four independent sum chains
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) acc[c4] = make_float2(0.f, 0.f);
              const float2 nm = make_float2(-hmax, -hmax), one = make_float2(1.f, 1.f);
#pragma unroll
              for (int i = 0; i < HK; i += 2) {
                const float2 dlt = ffma2(make_float2(sc[i], sc[i + 1]), one, nm);
                const float2 e = ((i >> 1) & 7) < PF_POLY_OF8_SCORE ? exp2_poly2(dlt)
                                                                    : make_float2(fast_exp2(dlt.x), fast_exp2(dlt.y));
                acc[(i >> 1) & 3] = ffma2(e, one, acc[(i >> 1) & 3]);
              }
              const float2 a01 = ffma2(acc[0], one, acc[1]), a23 = ffma2(acc[2], one, acc[3]);
              const float2 a2 = ffma2(a01, one, a23);
              const float tl = a2.x + a2.y;
              if (m_it == -INFINITY) {
                m_it = hmax;
                l_it = tl;
              } else {
                const float M = fmaxf(m_it, hmax);
                l_it = l_it * fast_exp2(m_it - M) + tl * fast_exp2(hmax - M);
                m_it = M;
              }
            }
            any_tile = true;
            continue;
          }
          xmax[(t & 1) * 256 + half * 128 + r] = hmax;
          fence_before();                                // our S reads precede the partner's P writes
#ifdef PF_PROF
          { const long long _t0 = clock64(); named_sync(bar_id, 64);
            if (threadIdx.x == 0) atomicAdd(&g_pf_prof[0][4], (unsigned long long)(clock64() - _t0)); }
#else
          named_sync(bar_id, 64);
#endif
          fence_after();
          const float tmax = fmaxf(hmax, xmax[(t & 1) * 256 + (half ^ 1) * 128 + r]);
          // ---- lazy online softmax: move the reference max only when it grows by > TAU
          const bool first = !any_tile;
          float m_new = m_run;
          if (first) m_new = tmax;
          else if (tmax > m_run + TAU) m_new = tmax;
          const float mu = (m_new == -INFINITY) ? 0.f : m_new;
          const float fac = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - mu);
          const bool rescale = !first && (m_new != m_run);
          float2 acc[4];                                 // four independent sum chains
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) acc[c4] = make_float2(0.f, 0.f);
          uint32_t hw[HK / 2], lw[HK / 2];
          const float2 nmu = make_float2(-mu, -mu), one = make_float2(1.f, 1.f), mone = make_float2(-1.f, -1.f);
#pragma unroll
          for (int i = 0; i < HK; i += 2) {
            const float2 dlt = ffma2(make_float2(sc[i], sc[i + 1]), one, nmu);
            const float2 e = ((i >> 1) & 7) < PF_POLY_OF8 ? exp2_poly2(dlt)
                                                          : make_float2(fast_exp2(dlt.x), fast_exp2(dlt.y));
            acc[(i >> 1) & 3] = ffma2(e, one, acc[(i >> 1) & 3]);
            __nv_bfloat162 hb = __floats2bfloat162_rn(e.x, e.y);
            const uint32_t hu = *reinterpret_cast<uint32_t*>(&hb);
            hw[i / 2] = hu;
            if constexpr (SPLIT) {
              const float2 lo2 = ffma2(make_float2(__uint_as_float(hu << 16), __uint_as_float(hu & 0xffff0000u)),
                                       mone, e);
              __nv_bfloat162 lb = __floats2bfloat162_rn(lo2.x, lo2.y);
              lw[i / 2] = *reinterpret_cast<uint32_t*>(&lb);
            }
          }
          const float2 a01 = ffma2(acc[0], one, acc[1]), a23 = ffma2(acc[2], one, acc[3]);
          const float2 a2 = ffma2(a01, one, a23);
          const float rs = a2.x + a2.y;
          l_half = (rescale ? l_half * fac : l_half) + rs;
          // ---- per-item scoring statistics from the softmax's own sum: this half's
          // tile sum rs is relative to the reference max mu, so (mu, rs) folds into the
          // item's (m, l) like a tile-local (max, sum) — no second exp per score.  The
          // masses equal the tile-local form up to fp32 rounding (identical rounds may
          // differ in the last bits); a kept set decided by such a near-tie has a
          // K-boundary margin below the engines' refine threshold, and the fp64 exact
          // re-score (rk_round_scores_exact) decides it as the reference does
          if (p.item_m && hmax != -INFINITY) {
            if (m_it == -INFINITY) {
              m_it = mu;
              l_it = rs;
            } else {
              const float M = fmaxf(m_it, mu);
              l_it = l_it * fast_exp2(m_it - M) + rs * fast_exp2(mu - M);
              m_it = M;
            }
          }
          // ---- O rescale (rare): O is stable once PV_{t-1} has completed
          if (__any_sync(0xffffffffu, rescale)) {
            const int tl1 = t - 1;
            PWAIT(&buf_free[tl1 % NB], (tl1 / NB) & 1, 0, 2);
            fence_after();
            const float f = rescale ? fac : 1.f;
            const float2 f2 = make_float2(f, f);
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              float o[32];
              const uint32_t oa = tmem_o + lane_base + 64 * half + 32 * cc;
              tmem_ld32(oa, o);
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const float2 x = fmul2(make_float2(o[i], o[i + 1]), f2);
                o[i] = x.x;
                o[i + 1] = x.y;
              }
              tmem_st32(oa, o);
            }
          }
          m_run = m_new;
          any_tile = true;
          // ---- P over its own S columns: [P_hi keys 0-63 | P_lo keys 0-63], bf16x2 per column
          tmem_st32u(tmem + lane_base + b * BN + (HK / 2) * half, hw);            // P_hi columns
          if constexpr (SPLIT) tmem_st32u(tmem + lane_base + b * BN + BN / 2 + (HK / 2) * half, lw);   // P_lo
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          fence_before();
          __syncwarp();
          if (lane == 0) {                               // the leader issues this tile's PV
            if (leader) bar_arrive(&p_full[b]);
            else bar_arrive_cluster(mapa(&p_full[b], 0));
          }
        }
        if (p.item_m && real) {                // this column half's statistics: slot (item, half); the
          // finalisation (score_rows_kernel, 2 slots per item) combines the halves — no barrier here
          const int64_t o = (((int64_t)qi * p.hq + h) * p.n_items + it) * 2 + half;
          p.item_m[o] = m_it;
          p.item_l[o] = l_it;
        }
      }
      if (SCORE_ONLY) continue;
      // ---- unit end: O after the last PV, partial (m, l, O) for the merge
      const int64_t po = ((int64_t)qi * p.hq + h) * p.n_chunks + c;
      if (any_tile) {
        const int tl1 = t - 1;
        PWAIT(&buf_free[tl1 % NB], (tl1 / NB) & 1, 0, 3);
        fence_after();
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          float o[32];
          tmem_ld32(tmem_o + lane_base + 64 * half + 32 * cc, o);
          if (real) {
            float4* dst = reinterpret_cast<float4*>(p.part_o + po * D + 64 * half + 32 * cc);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
          }
        }
        fence_before();
      } else if (real) {
        float4* dst = reinterpret_cast<float4*>(p.part_o + po * D + 64 * half);
        for (int i = 0; i < 16; ++i) dst[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (half == 1) xl_u[r] = l_half;
      named_sync(bar_id, 64);
      if (half == 0 && real) {
        p.part_m[po] = m_run;
        p.part_l[po] = l_half + xl_u[r];
      }
      named_sync(bar_id, 64);
    }
  }
#ifdef PF_PROF
  if (threadIdx.x == 0 || threadIdx.x == 32 * kMmaWarp || threadIdx.x == 32 * kProducerWarp ||
      threadIdx.x == 32 * kVProducerWarp) {
    const int role = threadIdx.x == 0 ? 0 : threadIdx.x == 32 * kMmaWarp ? 1 : threadIdx.x == 32 * kProducerWarp ? 2 : 3;
    atomicAdd(&g_pf_prof[role][15], (unsigned long long)(clock64() - prof_t0));
  }
#endif
  fence_before();
  cluster_sync();             // the leader's last MMAs touched both SMs' TMEM; both CTAs are done
  if (warp == kMmaWarp) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
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

// CTA pairs the persistent prefill grid may occupy: all SMs by default;
// RK_PREFILL_MAX_PAIRS caps it so a concurrent decode keeps SMs of its own
// (experiment: C3 with 48 / 37 / 26 pairs ran 2.94 / 2.93 / 2.92 K tok/s vs ~2.98 K
// uncapped — the other group's decode speeds up exactly as much as the prefill slows)
static int prefill_pairs() {
  static int cap = -1;
  if (cap < 0) {
    const char* e = std::getenv("RK_PREFILL_MAX_PAIRS");
    cap = e ? std::max(0, std::atoi(e)) : 0;       // 0 = no cap
  }
  const int all = std::max(1, sm_count() / 2);
  return cap > 0 ? std::min(cap, all) : all;
}

// item table: `items` (n_items given) or uniform items of item_keys keys over s
PrefillPlan prefill_plan(int n_q, int hq, int hkv, int s, int n_items_in, bool stats, bool with_output) {
  PrefillPlan pl{};
  const int G = hq / hkv;
  pl.mpad = (G * n_q + pf::PM - 1) / pf::PM * pf::PM;      // pair M tiles of 256 stacked rows
  pl.mtiles = pl.mpad / pf::PM;
  const int mt_total = hkv * pl.mtiles;
  if (n_items_in > 0) {
    pl.n_items = n_items_in;
    pl.item_keys = 0;
  } else {
    pl.item_keys = 512;
    pl.n_items = s > 0 ? (s + pl.item_keys - 1) / pl.item_keys : 1;
  }
  // ~8 units per SM: balance over the persistent CTAs, >= 1 item per chunk
  static int per_pair = -1;                                 // RK_PREFILL_UNITS overrides (experiments)
  if (per_pair < 0) {
    const char* e = std::getenv("RK_PREFILL_UNITS");
    per_pair = e ? std::max(1, std::atoi(e)) : 8;
  }
  // the scores-only pass (no V / PV) has cheaper units: finer, plain chunking balances it
  // better (C3 512 rows: 0.60 -> 0.58 ms with 12 units per pair and no wave model)
  static int score_units = -1;                              // RK_SCORE_UNITS overrides (experiments)
  if (score_units < 0) {
    const char* e = std::getenv("RK_SCORE_UNITS");
    score_units = e ? std::max(1, std::atoi(e)) : 12;
  }
  const int target = (with_output ? per_pair : score_units) * prefill_pairs();   // units per CTA pair
  int nc = (target + mt_total - 1) / mt_total;
  nc = std::max(1, std::min(nc, pl.n_items));
  pl.items_per_chunk = (pl.n_items + nc - 1) / nc;
  pl.n_chunks = (pl.n_items + pl.items_per_chunk - 1) / pl.items_per_chunk;
  static int balance = -1;                                  // RK_PREFILL_BALANCE=0: the plain target
  if (balance < 0) {
    const char* e = std::getenv("RK_PREFILL_BALANCE");
    balance = e ? std::atoi(e) : 1;
  }
  if (balance && with_output) {
    // units are dealt round-robin to the persistent pairs, so the pairs' time is
    // ceil(units / pairs) units: pick the chunking (items per chunk) that minimises
    // waves x (work per unit + a fixed per-unit cost), around the target count
    // (C3, 56 M tiles x 11 chunks = 616 units = 8.3 waves on 74 pairs; 13 chunks:
    // 728 units = 9.8 waves)
    const int pairs = prefill_pairs();
    const double unit_cost = 0.03;                          // per unit, in whole-M-tile work (fitted: n_q 128..1024)
    double best = 1e30;
    for (int ipc = 1; ipc <= pl.n_items; ++ipc) {
      const int ncks = (pl.n_items + ipc - 1) / ipc;
      if (ipc > 1 && (pl.n_items + ipc - 2) / (ipc - 1) == ncks) continue;   // same chunk count, fewer items
      const int64_t units = (int64_t)mt_total * ncks;
      if (units > 4 * (int64_t)target) continue;
      const int64_t waves = (units + pairs - 1) / pairs;
      const double cost = (double)waves * (1.0 / ncks + unit_cost);
      if (cost < best - 1e-12) {
        best = cost;
        pl.items_per_chunk = ipc;
        pl.n_chunks = ncks;
      }
    }
  }
  pl.n_units = mt_total * pl.n_chunks;
  pl.qs_bytes = align_up((size_t)hkv * 2 * pl.mpad * pf::D * 2, 256);
  const size_t rh = (size_t)n_q * hq;
  pl.part_bytes = with_output ? align_up(rh * pl.n_chunks * 4, 256) * 2 + align_up(rh * pl.n_chunks * pf::D * 4, 256)
                              : 0;
  pl.item_bytes = stats ? align_up(rh * pl.n_items * 2 * 4, 256) * 2 : 0;     // (m, l) per (item, column half)
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
                      cudaStream_t st, bool single_pass) {
  const int G = hq / hkv;
  const bool score_only = out == nullptr;          // the watershed scorer: statistics only
  if (score_only && !stats) return fail(RK_ERR_DOMAIN, "prefill without output needs the scoring statistics");
  PrefillPlan pl = prefill_plan(n_q, hq, hkv, s, items ? n_items_in : 0, stats, !score_only);
  if (pl.total > ws_bytes) return fail(RK_ERR_CAPACITY, "prefill workspace %zu < %zu", ws_bytes, pl.total);
  char* b = static_cast<char*>(ws);
  const size_t rh = (size_t)n_q * hq;
  __nv_bfloat16* qs = reinterpret_cast<__nv_bfloat16*>(b);
  b += pl.qs_bytes;
  float *part_m = nullptr, *part_l = nullptr, *part_o = nullptr;
  if (!score_only) {
    part_m = reinterpret_cast<float*>(b);
    b += align_up(rh * pl.n_chunks * 4, 256);
    part_l = reinterpret_cast<float*>(b);
    b += align_up(rh * pl.n_chunks * 4, 256);
    part_o = reinterpret_cast<float*>(b);
    b += align_up(rh * pl.n_chunks * pf::D * 4, 256);
  }
  float* item_m = nullptr;
  float* item_l = nullptr;
  if (stats) {
    item_m = reinterpret_cast<float*>(b);
    b += align_up(rh * pl.n_items * 2 * 4, 256);
    item_l = reinterpret_cast<float*>(b);
    b += align_up(rh * pl.n_items * 2 * 4, 256);
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
  r = tc::make_map(&kmap, k, (uint64_t)hkv * pf::D, (uint64_t)s, (uint64_t)hkv * pf::D * 2, pf::BN / 2);
  if (r) return r;
  r = tc::make_map(&vmap, score_only ? k : v, (uint64_t)hkv * pf::D, (uint64_t)s, (uint64_t)hkv * pf::D * 2, pf::BN);
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
    RK_CUDA(cudaFuncSetAttribute(pf::prefill_tc_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pf::SMEM), "prefill_tc smem attribute");
    RK_CUDA(cudaFuncSetAttribute(pf::prefill_tc_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pf::SMEM), "prefill_tc smem attribute");
    RK_CUDA(cudaFuncSetAttribute(pf::prefill_tc_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pf::SMEM), "prefill_tc smem attribute");
    configured = true;
  }
  const int grid = 2 * std::min(prefill_pairs(), pl.n_units);   // CTA pairs (__cluster_dims__(2,1,1))
  if (score_only) {
    pf::prefill_tc_kernel<true, true><<<grid, pf::THREADS, pf::SMEM, st>>>(qmap, kmap, vmap, p);
    RK_CHECK_LAUNCH("prefill_tc_kernel<score>");
    return RK_OK;
  }
  if (single_pass)
    pf::prefill_tc_kernel<false, false><<<grid, pf::THREADS, pf::SMEM, st>>>(qmap, kmap, vmap, p);
  else
    pf::prefill_tc_kernel<false, true><<<grid, pf::THREADS, pf::SMEM, st>>>(qmap, kmap, vmap, p);
  RK_CHECK_LAUNCH("prefill_tc_kernel");
  const int nrh = (int)rh;
  pf::prefill_merge_kernel<<<(nrh * 32 + 255) / 256, 256, 0, st>>>(part_m, part_l, part_o, nrh, hq, pl.n_chunks,
                                                                   out, stat_m, stat_l, bad_row);
  RK_CHECK_LAUNCH("prefill_merge_kernel");
  return RK_OK;
}

}  // namespace rk

#ifdef PF_PROF
extern "C" int rk_pf_prof_read(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, rk::pf::g_pf_prof, sizeof(rk::pf::g_pf_prof));
  unsigned long long z[4][16] = {};
  cudaMemcpyToSymbol(rk::pf::g_pf_prof, z, sizeof(z));
  return 0;
}
#endif
