// The decode step's layer body on the GPU (engine.py:244-251,267-271 of the
// reference: q,k = RoPE(x W_q), RoPE(x W_k); v = x W_v; append; attention;
// x += out W_o; logits = x E^T; argmax) for B dialogues at once.
//
// Every projection is a skinny GEMM (m = B tokens <= 64 per launch, K = 4096,
// N = 6144 / 4096): the weights are read once per token step, so the kernel is
// bound by HBM on the weight bytes (Llama-3-8B-shaped: 84 MB per layer).
//
// Layout: a weight W [K][N] (x @ W) is stored once (rk_pack_weight) as 16 KB
// tiles [N_pad/128][K/64] of W^T — 128 features x 64 k, each tile already in
// the 128-byte-swizzled K-major image a tcgen05.mma M=128 A operand reads from
// shared memory (16-byte chunk c of feature row r at chunk c ^ (r & 7)); N is
// padded to 128 with zero rows.  A tile is one contiguous bulk copy, and a
// CTA's run of tiles is one contiguous stream (a TMA tensor box of W^T would
// gather 128 separate 128-byte rows 8 KB apart: measured 2.9 TB/s).
//
// Work: units (strip group sg = 128 features, k-chunk kc = 64 k) in sg-major
// order; a persistent grid of min(#SMs, units) CTAs takes contiguous equal
// runs of units, so every SM streams the same number of weight bytes whatever
// the shape.  Per CTA (12 warps):
//   warp 0   weight producer: bulk copy of each unit's 16 KB tile into a deep ring —
//            issued BEFORE griddepcontrol.wait (weights do not depend on the
//            previous kernel), so the ring fills while that kernel drains;
//   warps 4-7 converters (after griddepcontrol.wait): the unit's fp32
//            activation slice x[0:m][kc*64 : kc*64+64] straight from L2, several
//            units ahead in registers, -> bf16 hi + lo (x = hi + lo keeps ~16
//            mantissa bits; the reference's projections are fp32 BLAS) written
//            as two swizzled K-major B operands [NP tokens][64 k];
//   warp 2   MMA issuer (one elected lane): per unit 4 k16 steps x (hi, lo)
//            tcgen05.mma m128 n=NP k16 into a TMEM accumulator (double
//            buffered across the CTA's strip-group segments);
//   warps 8-11 epilogue (TMEM lane quarter = warp % 4, thread = feature):
//            a segment covering the whole K of its strip group runs the fused
//            epilogue directly; otherwise the partial goes to the workspace and
//            the last CTA to arrive on the group's ticket adds the partials in
//            CTA order (deterministic) and runs it:
//   qkv : RoPE on q and k (interleaved pairs, fp64 angles from the host-computed
//         reference frequency table, engine.py:162-164,175-185), q -> fp32,
//         k, v -> bf16 rows for the cache append;
//   out : x += attention_out W_o (the residual, engine.py:267);
//   head: logits (engine.py:270-271), then rk_argmax_embed picks the first
//         maximum (pipeline.py:308, np.argmax) and looks up the next input.
#include <cstdlib>
#include <type_traits>

#include "decode_common.cuh"
#include "rk_common.cuh"
#include "tc_common.cuh"

namespace rk {
namespace pj {

using namespace rk::tc;

#ifdef PJ_TRACE   // timing experiments: per-CTA %globaltimer stamps of the last launch
__device__ unsigned long long g_pj_trace[1024 * 16];
__device__ unsigned long long g_pj_units[3 * 64];
#define PJU(kind, i)                                                                     \
  do {                                                                                   \
    if (blockIdx.x == 0 && (i) < 64) {                                                   \
      unsigned long long _t;                                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                             \
      g_pj_units[(kind) * 64 + (i)] = _t;                                                \
    }                                                                                    \
  } while (0)
#define PJT(slot)                                                                        \
  do {                                                                                   \
    unsigned long long _t;                                                               \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                               \
    g_pj_trace[blockIdx.x * 16 + (slot)] = _t;                                            \
  } while (0)
#else
#define PJT(slot)
#define PJU(kind, i)
#endif

constexpr int BM = 128;                    // features per strip group (MMA M)
constexpr int BK = 64;                     // k per unit (one 128-byte swizzle row of bf16)
constexpr int W_BYTES = BM * BK * 2;       // 16 KB weight box
constexpr int kWarps = 12;
constexpr int kThreads = kWarps * 32;
constexpr int kWProducer = 0, kMma = 2, kConv0 = 4, kEpi0 = 8;
#ifndef PJ_BUDGET_KB
#define PJ_BUDGET_KB 200
#endif
constexpr int kSmemBudget = PJ_BUDGET_KB * 1024;

enum { PJ_QKV = 0, PJ_OUT = 1, PJ_HEAD = 2 };

template <int NP>
struct Cfg {
  static constexpr int XHL = 2 * NP * 128;            // hi tile | lo tile
  static constexpr int XH = NP >= 64 ? 2 : 3;
  static constexpr int EPT = NP / 8;                  // float4 of a unit's x slice per converter thread
  static constexpr int PD = 16 / EPT < 1 ? 1 : 16 / EPT;   // units of x in flight (registers)
  static constexpr int ROPE = NP <= 32 ? NP * (BM / 2) * 8 : 0;    // (cos, sin) table [t][pair]
  static constexpr int RED = NP * BM * 4;             // cluster mode: this CTA's partial [NP][128] f32
  static constexpr int WS = (kSmemBudget - 1024 - XH * XHL - ROPE - RED - 1024) / W_BYTES;
  static constexpr int SMEM = 1024 + WS * W_BYTES + XH * XHL + ROPE + RED + 1024;
  static constexpr int TMEM_COLS = 4 * NP < 32 ? 32 : 4 * NP;   // 2 buffers x [hi | lo] columns
  static_assert(WS >= 3, "weight ring too shallow");
};

struct Params {
  int cs;                                  // cluster mode: CTAs per strip group (the cluster size)
  const void* w;                           // tiled, swizzled W^T (rk_pack_weight)
  const float* x;                          // [m][K] activations
  int m, K, N, Npad, mode;
  int KC, n_units, maxc;                   // k-chunks per strip group, units, partial slots per group
  // qkv
  int hq, hkv, d;
  const int32_t* pos;
  const double* freq;
  float* q_out;
  void* k_out;                             // bf16 or (kv_f32) fp32 cache rows
  void* v_out;
  int64_t kv_stride;
  int kv_f32;
  // out
  float* resid;
  const int32_t* row_active;               // out: rows with 0 keep their residual (nullable = all rows)
  // head
  float* logits;
  // split-K reduction
  int* tickets;                            // [n_sg], zero between launches
  float* part;                             // [n_sg][maxc][m][128]
};

__device__ __forceinline__ int owner(int u, int n_units, int G) {    // CTA whose run holds unit u
  return (int)(((int64_t)(u + 1) * G - 1) / n_units);
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ bool elect() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void split_bf16(float2 p, uint32_t& hi, uint32_t& lo) {
  hi = pack_bf16(p.x, p.y);
  const float2 h = bf16x2_to_f2(hi);
  lo = pack_bf16(p.x - h.x, p.y - h.y);
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 2, 128;" ::: "memory"); }

// the fused epilogue of one strip group: thread `row` holds feature
// n = sg * 128 + row for tokens 0..NP-1.  `rope` (QKV) is the CTA's table of
// (cos, sin) of pos[t] * freq[pair] (angle and sincos in float64 as
// engine.py:175-185, stored rounded to float32), [t][row / 2], filled while the
// weights stream (nullptr: computed here); the rotation itself runs in float64.
// one k / v cache element (or an adjacent pair) in the cache's dtype
__device__ __forceinline__ void store_kv(const Params& p, void* base, size_t i, float y) {
  if (p.kv_f32)
    static_cast<float*>(base)[i] = y;
  else
    static_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(y);
}
__device__ __forceinline__ void store_kv2(const Params& p, void* base, size_t i, float a, float b) {
  if (p.kv_f32)
    *reinterpret_cast<float2*>(static_cast<float*>(base) + i) = make_float2(a, b);
  else
    *reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(base) + i) = pack_bf16(a, b);
}

template <int NP>
__device__ __forceinline__ void finish(const Params& p, int sg, int row, float (&v)[NP], const float2* rope) {
  const int n = sg * BM + row;
  if (p.mode == PJ_QKV) {
    const int qd = p.hq * p.d, kd = p.hkv * p.d;
    const bool even = (n & 1) == 0, valid = n < p.N, rot = n < qd + kd;
    const double f = rot ? p.freq[(n % p.d) >> 1] : 0.0;
#pragma unroll
    for (int t = 0; t < NP; ++t) {
      if (t >= p.m) break;                                          // uniform: every lane has the same m
      const float other = __shfl_xor_sync(0xffffffffu, v[t], 1);   // the pair partner (all lanes take part)
      if (!valid) continue;
      if (rot) {
        double sn, cs;
        if (rope) {
          const float2 e = rope[t * (BM / 2) + (row >> 1)];
          cs = e.x;
          sn = e.y;
        } else {
          sincos((double)p.pos[t] * f, &sn, &cs);
        }
        const double x0 = even ? v[t] : other, x1 = even ? other : v[t];
        const float y = even ? (float)(x0 * cs - x1 * sn) : (float)(x0 * sn + x1 * cs);
        if (n < qd)
          p.q_out[(size_t)t * qd + n] = y;
        else
          store_kv(p, p.k_out, (size_t)t * p.kv_stride + (n - qd), y);
      } else {
        store_kv(p, p.v_out, (size_t)t * p.kv_stride + (n - qd - kd), v[t]);
      }
    }
  } else if (p.mode == PJ_OUT) {
    if (n >= p.N) return;
    float r[NP];
#pragma unroll
    for (int t = 0; t < NP; ++t) r[t] = t < p.m ? p.resid[(size_t)t * p.N + n] : 0.f;   // all loads in flight
#pragma unroll
    for (int t = 0; t < NP; ++t)
      if (t < p.m && (p.row_active == nullptr || p.row_active[t])) p.resid[(size_t)t * p.N + n] = r[t] + v[t];
  } else {
#pragma unroll
    for (int t = 0; t < NP; ++t) {
      if (t >= p.m) break;
      p.logits[(size_t)t * p.Npad + n] = v[t];
    }
  }
}

// the fused epilogue for one feature pair (n, n + 1), n = sg * 128 + 2 pr, of
// token t (cluster mode): same arithmetic as finish()
__device__ __forceinline__ void finish_pair(const Params& p, int sg, int pr, int t, float y0, float y1,
                                            const float2* rope) {
  const int n = sg * BM + 2 * pr;
  if (n >= p.N) return;
  if (p.mode == PJ_QKV) {
    const int qd = p.hq * p.d, kd = p.hkv * p.d;
    if (n < qd + kd) {
      double sn, cs;
      if (rope) {
        const float2 e = rope[t * (BM / 2) + pr];
        cs = e.x;
        sn = e.y;
      } else {
        sincos((double)p.pos[t] * p.freq[(n % p.d) >> 1], &sn, &cs);
      }
      const float a = (float)((double)y0 * cs - (double)y1 * sn), b = (float)((double)y0 * sn + (double)y1 * cs);
      if (n < qd)
        *reinterpret_cast<float2*>(p.q_out + (size_t)t * qd + n) = make_float2(a, b);
      else
        store_kv2(p, p.k_out, (size_t)t * p.kv_stride + (n - qd), a, b);
    } else {
      store_kv2(p, p.v_out, (size_t)t * p.kv_stride + (n - qd - kd), y0, y1);
    }
  } else if (p.mode == PJ_OUT) {
    if (p.row_active != nullptr && !p.row_active[t]) return;
    float2* r = reinterpret_cast<float2*>(p.resid + (size_t)t * p.N + n);
    const float2 o = *r;
    *r = make_float2(o.x + y0, o.y + y1);
  } else {
    *reinterpret_cast<float2*>(p.logits + (size_t)t * p.Npad + n) = make_float2(y0, y1);
  }
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float2 ld_dsmem_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

// v = the sum over the strip group's contributors (CTA order) of their
// partials: the loads of 4 contributors x 16 tokens are in flight at once
template <int NP>
__device__ __forceinline__ void reduce_partials(const Params& p, int sg, int row, int ncontrib, float (&v)[NP]) {
  constexpr int TC = NP < 16 ? NP : 16, CC = 4;
  const float* base = p.part + (size_t)sg * p.maxc * p.m * BM + row;
#pragma unroll
  for (int t0 = 0; t0 < NP; t0 += TC) {
    if (t0 >= p.m) break;
    float acc[TC];
#pragma unroll
    for (int tt = 0; tt < TC; ++tt) acc[tt] = 0.f;
    for (int c0 = 0; c0 < ncontrib; c0 += CC) {
      float x[CC][TC];
#pragma unroll
      for (int cc = 0; cc < CC; ++cc)
#pragma unroll
        for (int tt = 0; tt < TC; ++tt)
          x[cc][tt] = (c0 + cc < ncontrib && t0 + tt < p.m)
                          ? __ldcg(base + ((size_t)(c0 + cc) * p.m + t0 + tt) * BM) : 0.f;
#pragma unroll
      for (int cc = 0; cc < CC; ++cc)
#pragma unroll
        for (int tt = 0; tt < TC; ++tt) acc[tt] += x[cc][tt];      // fixed order: deterministic
    }
#pragma unroll
    for (int tt = 0; tt < TC; ++tt) v[t0 + tt] = acc[tt];
  }
}

__device__ __forceinline__ int ticket_acq_rel(int* t) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
  return old;
}

// CL = cluster mode: a cluster of p.cs CTAs per strip group, each a contiguous
// k range, partials added through distributed shared memory (no global round
// trips in the kernel's tail); otherwise the ticketed split-K over a flat run
// of units per CTA.
template <int NP, bool CL>
__global__ void __launch_bounds__(kThreads, 1)
proj_tc_kernel(const __grid_constant__ Params p) {
  using C = Cfg<NP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* wring = smem;                              // WS x 16 KB (SW128 K-major A tiles)
  uint8_t* xhl = wring + C::WS * W_BYTES;             // XH x [hi NP x 128 B | lo NP x 128 B]
  float2* rope_tab = reinterpret_cast<float2*>(xhl + C::XH * C::XHL);
  float* red = reinterpret_cast<float*>(xhl + C::XH * C::XHL + C::ROPE);     // [NP][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xhl + C::XH * C::XHL + C::ROPE + C::RED);
  uint64_t* wfull = bars;
  uint64_t* wempty = wfull + C::WS;
  uint64_t* hfull = wempty + C::WS;
  uint64_t* hempty = hfull + C::XH;
  uint64_t* accfull = hempty + C::XH;
  uint64_t* accempty = accfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  int* flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  int u0, u1;
  if constexpr (CL) {               // strip group c / cs, k chunks [r KC / cs, (r + 1) KC / cs)
    const int sg = c / p.cs, r = c - sg * p.cs;
    u0 = sg * p.KC + r * p.KC / p.cs;
    u1 = sg * p.KC + (r + 1) * p.KC / p.cs;
  } else {
    u0 = (int)((int64_t)c * p.n_units / G);
    u1 = (int)((int64_t)(c + 1) * p.n_units / G);
  }
  const int n = u1 - u0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::WS; ++s) { bar_init(&wfull[s], 1); bar_init(&wempty[s], 1); }
    for (int s = 0; s < C::XH; ++s) { bar_init(&hfull[s], 128); bar_init(&hempty[s], 1); }
    for (int b = 0; b < 2; ++b) { bar_init(&accfull[b], 1); bar_init(&accempty[b], 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) PJT(0);
  // every CTA of this grid is running: the next kernel on the stream may start
  // its prologue (it reads nothing this kernel writes before its own
  // griddepcontrol.wait, which waits for this whole grid)
  pdl_trigger();

  if (warp == kWProducer) {
    // ===== weights: independent of the previous kernel, streamed from launch
    if (elect()) {
      const uint64_t pol = evict_first_policy();     // read once per token step
      const uint8_t* src = reinterpret_cast<const uint8_t*>(p.w) + (size_t)u0 * W_BYTES;
      for (int i = 0; i < n; ++i) {
        const int s = i % C::WS;
        if (i >= C::WS) bar_wait(&wempty[s], ((i / C::WS) - 1) & 1);
#ifdef PJ_NO_W
        bar_arrive(&wfull[s]);
#else
        bar_expect(&wfull[s], W_BYTES);
        bulk_g2s(wring + s * W_BYTES, src + (size_t)i * W_BYTES, W_BYTES, &wfull[s], pol);
#endif
      }
    }
    __syncwarp();
  } else if (warp >= kConv0 && warp < kConv0 + 4) {
    // ===== x -> bf16 hi + lo, swizzled K-major B operands.  The fp32 slice
    // x[0:m][kc*64 : kc*64+64] of each unit is loaded straight from L2 (the
    // previous kernel's output) PD units ahead in registers, so the activations
    // never throttle the weight stream
    pdl_wait();
    const int tid = threadIdx.x - kConv0 * 32;
    float4 pre[C::PD][C::EPT];
    auto load = [&](int i, float4(&dst)[C::EPT]) {
      const int kc = (u0 + i) % p.KC;
#pragma unroll
      for (int e = 0; e < C::EPT; ++e) {
        const int idx = tid + 128 * e, r = idx >> 4, c4 = idx & 15;
        dst[e] = (i < n && r < p.m) ? __ldcg(reinterpret_cast<const float4*>(p.x + (size_t)r * p.K + kc * BK) + c4)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
#pragma unroll
    for (int d = 0; d < C::PD; ++d) load(d, pre[d]);
    for (int i0 = 0; i0 < n; i0 += C::PD) {
#pragma unroll
      for (int d = 0; d < C::PD; ++d) {
        const int i = i0 + d;
        if (i >= n) break;
        const int h = i % C::XH;
        if (i >= C::XH) bar_wait(&hempty[h], ((i / C::XH) - 1) & 1);
        uint8_t* hi = xhl + h * C::XHL;
        uint8_t* lo = hi + NP * 128;
#pragma unroll
        for (int e = 0; e < C::EPT; ++e) {
          const int idx = tid + 128 * e, r = idx >> 4, c4 = idx & 15;
          uint2 vh, vl;
          split_bf16(make_float2(pre[d][e].x, pre[d][e].y), vh.x, vl.x);
          split_bf16(make_float2(pre[d][e].z, pre[d][e].w), vh.y, vl.y);
          // 16-byte chunk c4 / 2 of row r holds k 8 (c4 / 2) .. +7; this float4 is its half c4 & 1
          const int off = r * 128 + (((c4 >> 1) ^ (r & 7)) << 4) + ((c4 & 1) << 3);
          *reinterpret_cast<uint2*>(hi + off) = vh;
          *reinterpret_cast<uint2*>(lo + off) = vl;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core reads
        bar_arrive(&hfull[h]);
        if (tid == 0) PJU(2, i);
        load(i + C::PD, pre[d]);
      }
    }
  } else if (warp == kMma) {
    // ===== MMA issuer
    // B = [x_hi; x_lo] stacked (2 NP rows): one MMA per k16 step gives W x_hi in
    // accumulator columns [0, NP) and W x_lo in [NP, 2 NP) — the weight tile is
    // read once per k16 step, not once per half; the epilogue adds the halves
    constexpr uint32_t idesc = idesc_f16(BM, 2 * NP);
    const uint32_t w_a = sa(wring), h_a = sa(xhl);
    int q = 0;                                        // segment counter (accumulator buffer q & 1)
    bool fresh = true;
    for (int i = 0; i < n; ++i) {
      const int u = u0 + i, kc = u % p.KC, s = i % C::WS, h = i % C::XH;
      const int b = q & 1;
      if (fresh && q >= 2) bar_wait(&accempty[b], ((q / 2) - 1) & 1);
      bar_wait(&wfull[s], (i / C::WS) & 1);
      if (i == 0 && lane == 0) PJT(1);
      if (lane == 0) PJU(0, i);
#ifndef PJ_NO_X
      bar_wait(&hfull[h], (i / C::XH) & 1);
#endif
      if (lane == 0) PJU(1, i);
      if (i == 0 && lane == 0) PJT(3);
      if (i == n - 1 && lane == 0) PJT(4);
      fence_after();
      if (elect()) {
        const uint64_t da = umma_desc(wring + s * W_BYTES), db = umma_desc(xhl + h * C::XHL);
        (void)w_a; (void)h_a;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          umma(tmem + b * 2 * NP, da + (uint64_t)((32 * k) >> 4), db + (uint64_t)((32 * k) >> 4), idesc,
               (fresh && k == 0) ? 0u : 1u);
        umma_commit(&wempty[s]);
        umma_commit(&hempty[h]);
        if (i == n - 1 || kc == p.KC - 1) umma_commit(&accfull[b]);
      }
      __syncwarp();
      fresh = false;
      if (i == n - 1 || kc == p.KC - 1) { ++q; fresh = true; }
    }
  } else if (warp >= kEpi0) {
    // ===== epilogue: thread = feature row of the strip group
    pdl_wait();
    const int wq = warp & 3, row = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    // RoPE table of this launch's rows (the pair index of row r is the same in
    // every strip group when 128 % d == 0), built while the weights stream
    const bool tab = C::ROPE > 0 && p.mode == PJ_QKV && BM % p.d == 0;
    if (tab) {
      const double f = p.freq[(row % p.d) >> 1];
      for (int t = row & 1; t < p.m; t += 2) {
        double sn, cs;
        sincos((double)p.pos[t] * f, &sn, &cs);
        rope_tab[t * (BM / 2) + (row >> 1)] = make_float2((float)cs, (float)sn);
      }
      epi_sync();
    }
    const float2* rope = tab ? rope_tab : nullptr;
    int q = 0;
    for (int i = 0; i < n;) {
      const int u = u0 + i, sg = u / p.KC, kc_a = u - sg * p.KC;
      const int len = min(n - i, p.KC - kc_a);
      const int b = q & 1;
      bar_wait(&accfull[b], (q / 2) & 1);
      fence_after();
      float v[NP];
#pragma unroll
      for (int c16 = 0; c16 < NP / 16; ++c16) {
        float lo16[16];
        tmem_ld16(tmem + lane_base + b * 2 * NP + 16 * c16, v + 16 * c16);
        tmem_ld16(tmem + lane_base + b * 2 * NP + NP + 16 * c16, lo16);
#pragma unroll
        for (int e = 0; e < 16; ++e) v[16 * c16 + e] += lo16[e];      // W x_hi + W x_lo
      }
      fence_before();
      bar_arrive(&accempty[b]);
      if (threadIdx.x == kEpi0 * 32) PJT(7);
      if constexpr (CL) {             // this CTA's partial -> smem; the cluster adds them below
#pragma unroll
        for (int t = 0; t < NP; ++t) red[t * BM + row] = v[t];
      } else if (len == p.KC) {
        finish<NP>(p, sg, row, v, rope);
      } else {
        // split-K: publish the partial; the last of the group's contributors
        // (ticket) adds them in CTA order and runs the epilogue
        const int cf = owner(sg * p.KC, p.n_units, G), cl = owner(sg * p.KC + p.KC - 1, p.n_units, G);
        float* slot = p.part + ((size_t)(sg * p.maxc + (c - cf)) * p.m) * BM + row;
#pragma unroll
        for (int t = 0; t < NP; ++t)
          if (t < p.m) __stcg(slot + (size_t)t * BM, v[t]);
        epi_sync();                                   // the group's stores precede the release below
        if (threadIdx.x == kEpi0 * 32) PJT(8);
        if (threadIdx.x == kEpi0 * 32) *flag = ticket_acq_rel(&p.tickets[sg]) == cl - cf;
        epi_sync();
        if (threadIdx.x == kEpi0 * 32) PJT(9);
        if (*flag) {
          reduce_partials<NP>(p, sg, row, cl - cf + 1, v);
          if (threadIdx.x == kEpi0 * 32) PJT(10);
          finish<NP>(p, sg, row, v, rope);
          if (threadIdx.x == kEpi0 * 32) PJT(11);
          if (threadIdx.x == kEpi0 * 32) p.tickets[sg] = 0;   // ready for the next launch
        }
        epi_sync();
      }
      i += len;
      ++q;
    }
    if (threadIdx.x == kEpi0 * 32) PJT(5);
  }
  if constexpr (CL) {
    cluster_sync_all();               // every CTA's partial is in its shared memory
    if (warp >= kEpi0) {
      // rank r finishes feature pairs [r 64 / cs, (r + 1) 64 / cs) of the strip
      // group: the cluster's partials added in rank order (deterministic)
      const int sg = c / p.cs, r = c - sg * p.cs, tid = threadIdx.x - kEpi0 * 32;
      const int p0 = r * (BM / 2) / p.cs, np_ = (r + 1) * (BM / 2) / p.cs - p0;
      const bool tab = C::ROPE > 0 && p.mode == PJ_QKV && BM % p.d == 0;
      const float2* rope = tab ? rope_tab : nullptr;
      const uint32_t red_a = sa(red);
      constexpr int IT = 4;                                    // items per thread with all loads in flight
      for (int e0 = tid; e0 < np_ * p.m; e0 += 128 * IT) {
        float2 z[IT][8];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          const int e = e0 + 128 * it;
          const int t = e / np_, pr = p0 + (e - t * np_);
          const uint32_t off = (uint32_t)(t * BM + 2 * pr) * 4;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            z[it][q] = (q < p.cs && e < np_ * p.m) ? ld_dsmem_f2(mapa_u32(red_a + off, (uint32_t)q))
                                                   : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
          const int e = e0 + 128 * it;
          if (e >= np_ * p.m) break;
          const int t = e / np_, pr = p0 + (e - t * np_);
          float2 y = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < 8; ++q) {                      // rank order: deterministic
            y.x += z[it][q].x;
            y.y += z[it][q].y;
          }
          finish_pair(p, sg, pr, t, y.x, y.y, rope);
        }
      }
    }
    cluster_sync_all();               // the peers are done reading this CTA's partial
  }
  fence_before();
  __syncthreads();
  if (warp == kMma) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::TMEM_COLS));
  }
  if (threadIdx.x == 0) PJT(6);
}

}  // namespace pj

// tiles[sg][kc] (16 KB, swizzled K-major image) <- W[k][n] (x @ W), rows n >= n_valid zero
template <typename T>
__global__ void pack_weight_kernel(const T* __restrict__ w, int K, int n_valid, int Npad,
                                   __nv_bfloat16* __restrict__ out) {
  // one thread per (feature row n, 16-byte chunk of 8 k)
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int kchunks = K / 8;
  if (idx >= (size_t)Npad * kchunks) return;
  const int n = (int)(idx % Npad), kq = (int)(idx / Npad);   // consecutive threads: consecutive n (coalesced reads)
  const int k0 = kq * 8, sg = n / pj::BM, r = n % pj::BM, kc = k0 / pj::BK, c = (k0 % pj::BK) / 8;
  __nv_bfloat16 v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e)
    v[e] = __float2bfloat16_rn(n < n_valid ? (float)w[(size_t)(k0 + e) * n_valid + n] : 0.f);
  const size_t tile = (size_t)sg * (K / pj::BK) + kc;
  uint8_t* dst = reinterpret_cast<uint8_t*>(out) + tile * pj::W_BYTES + r * 128 + ((c ^ (r & 7)) << 4);
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
}

constexpr int kMaxStripGroups = 1024;      // n_pad <= 131072 outputs

struct ProjPlan {
  int Npad, KC, n_sg, n_units, grid, maxc;
  size_t part_off, part_bytes, logits_off, total;
};

static ProjPlan proj_plan(int m, int K, int N) {
  ProjPlan pl{};
  pl.Npad = (N + pj::BM - 1) / pj::BM * pj::BM;
  pl.n_sg = pl.Npad / pj::BM;
  pl.KC = K / pj::BK;
  pl.n_units = pl.n_sg * pl.KC;
#ifndef PJ_CTAS_PER_SM
#define PJ_CTAS_PER_SM 1
#endif
  const int slots = PJ_CTAS_PER_SM * sm_count();
  pl.grid = pl.n_units < slots ? pl.n_units : slots;
  pl.maxc = 1;
  for (int sg = 0; sg < pl.n_sg; ++sg) {
    auto own = [&](int u) { return (int)(((int64_t)(u + 1) * pl.grid - 1) / pl.n_units); };
    const int cnt = own(sg * pl.KC + pl.KC - 1) - own(sg * pl.KC) + 1;
    pl.maxc = cnt > pl.maxc ? cnt : pl.maxc;
  }
  const int mm = m < 1 ? 1 : (m > 64 ? 64 : m);
  // tickets live in a fixed leading region, so calls of any shape can share one
  // workspace: no shape's partials ever land where another keeps its tickets
  pl.part_off = sizeof(int) * kMaxStripGroups;
  pl.part_bytes = sizeof(float) * (size_t)pl.n_sg * pl.maxc * mm * pj::BM;
  pl.logits_off = align_up(pl.part_off + pl.part_bytes, 256);
  pl.total = pl.logits_off + sizeof(float) * (size_t)mm * pl.Npad;
  return pl;
}

template <int NP, bool CL>
static int launch_np(const pj::Params& p, int grid, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    RK_CUDA(cudaFuncSetAttribute(pj::proj_tc_kernel<NP, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 pj::Cfg<NP>::SMEM), "proj smem attribute");
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(pj::kThreads);
  cfg.dynamicSmemBytes = pj::Cfg<NP>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CL ? p.cs : 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CL ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, pj::proj_tc_kernel<NP, CL>, p);
  if (e != cudaSuccess) return cuda_status(e, "proj_tc_kernel launch");
  return RK_OK;
}

// clusters of `cs` CTAs of the NP kernel that can be co-resident on this GPU (0 = unknown)
template <int NP>
static int max_clusters(int cs) {
  static int cache[17] = {0};
  if (cs < 1 || cs > 16) return 0;
  if (cache[cs] == 0) {
    if (cudaFuncSetAttribute(pj::proj_tc_kernel<NP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             pj::Cfg<NP>::SMEM) != cudaSuccess)
      return 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(pj::kThreads);
    cfg.dynamicSmemBytes = pj::Cfg<NP>::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, pj::proj_tc_kernel<NP, true>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      nc = -1;
    }
    cache[cs] = nc;
  }
  return cache[cs] > 0 ? cache[cs] : 0;
}

// the cluster size for a launch: the largest cs <= 8 with n_sg clusters of cs
// co-resident on the GPU (one wave), or 0 = ticketed split-K over every SM.
// Measured (C2 token step, 16 rows): the qkv projection as 48 clusters of 2
// (96 SMs) beats the ticketed split-K over 148 SMs (the SMs left free start
// the next kernel early, and the DSMEM tail is short); bench 7.03 K -> 7.63 K tok/s
template <int NP>
static int pick_cs(int n_sg, int KC) {
  if (getenv("RK_PROJ_NO_CLUSTER")) return 0;
  int best = 0;
  for (int cs = 2; cs <= 8 && cs <= KC; ++cs)
    if (n_sg * cs <= sm_count() && max_clusters<NP>(cs) >= n_sg) best = cs;
  return best;
}

// y = x W for rows [0, m) in launches of <= 64 rows
static int launch_proj(pj::Params p, const float* x, const void* w_packed, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
  if (p.m <= 0) return RK_OK;
  if (p.K % pj::BK != 0) return fail(RK_ERR_DOMAIN, "projection K=%d (multiple of %d)", p.K, pj::BK);
  const ProjPlan pl = proj_plan(p.m, p.K, p.N);
  if (pl.n_sg > kMaxStripGroups) return fail(RK_ERR_DOMAIN, "projection N=%d too large", p.N);
  if (ws == nullptr || ws_bytes < pl.total)
    return fail(RK_ERR_CAPACITY, "projection workspace %zu < %zu bytes", ws_bytes, pl.total);
  int r = RK_OK;
  p.w = w_packed;
  p.Npad = pl.Npad;
  p.KC = pl.KC;
  p.n_units = pl.n_units;
  p.maxc = pl.maxc;
  p.tickets = reinterpret_cast<int*>(ws);
  p.part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + pl.part_off);
  if (p.mode == pj::PJ_HEAD) p.logits = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + pl.logits_off);
  const int m_all = p.m;
  for (int m0 = 0; m0 < m_all; m0 += 64) {
    pj::Params q = p;
    q.m = m_all - m0 < 64 ? m_all - m0 : 64;
    const int qd = p.hq * p.d;
    if (p.mode == pj::PJ_QKV) {
      q.pos = p.pos + m0;
      q.q_out = p.q_out + (size_t)m0 * qd;
      const size_t kv_off = (size_t)m0 * p.kv_stride * (p.kv_f32 ? 4 : 2);
      q.k_out = static_cast<uint8_t*>(p.k_out) + kv_off;
      q.v_out = static_cast<uint8_t*>(p.v_out) + kv_off;
    } else if (p.mode == pj::PJ_OUT) {
      q.resid = p.resid + (size_t)m0 * p.N;
      if (p.row_active) q.row_active = p.row_active + m0;
    } else if (m0 > 0) {
      return fail(RK_ERR_DOMAIN, "lm_head rows %d > 64 per call", m_all);
    }
    q.x = x + (size_t)m0 * p.K;
    auto run = [&](auto np_tag) -> int {
      constexpr int NP = decltype(np_tag)::value;
      const int cs = pick_cs<NP>(pl.n_sg, pl.KC);
      if (cs > 1) {
        q.cs = cs;
        return launch_np<NP, true>(q, pl.n_sg * cs, st);
      }
      q.cs = 0;
      return launch_np<NP, false>(q, pl.grid, st);
    };
    if (q.m <= 16)
      r = run(std::integral_constant<int, 16>{});
    else if (q.m <= 32)
      r = run(std::integral_constant<int, 32>{});
    else
      r = run(std::integral_constant<int, 64>{});
    if (r != RK_OK) return r;
  }
  return RK_OK;
}

// tokens[b] = first argmax of logits[b][0:V) (np.argmax); x[b] = emb[token];
// pos[b] += 1 when given; tokens_log[b * log_stride] = token when given
__global__ void argmax_embed_kernel(const float* __restrict__ logits, int ld, int V,
                                    const __nv_bfloat16* __restrict__ emb, int D, float* __restrict__ x,
                                    int32_t* __restrict__ tokens, int32_t* __restrict__ pos,
                                    int32_t* __restrict__ tokens_log, int log_stride,
                                    const int32_t* __restrict__ row_active, int log_pos_base) {
  pdl_wait();
  __shared__ float sv[256];
  __shared__ int si[256];
  const int b = blockIdx.x;
  if (row_active != nullptr && !row_active[b]) {   // an inactive row keeps its token, position and input
    pdl_trigger();
    return;
  }
  const float* lg = logits + (size_t)b * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const float z = lg[v];
    if (z > best || (z == best && v < bi)) { best = z; bi = v; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const float z = sv[threadIdx.x + o];
      const int i = si[threadIdx.x + o];
      if (z > sv[threadIdx.x] || (z == sv[threadIdx.x] && i < si[threadIdx.x])) {
        sv[threadIdx.x] = z;
        si[threadIdx.x] = i;
      }
    }
    __syncthreads();
  }
  const int tok = si[0];
  for (int e = threadIdx.x; e < D; e += blockDim.x) x[(size_t)b * D + e] = __bfloat162float(emb[(size_t)tok * D + e]);
  if (threadIdx.x == 0) {
    if (tokens) tokens[b] = tok;
    // log_pos_base >= 0: the token goes to entry pos[b] - log_pos_base + 1 of the row (rows of a cohort
    // batch sit at different steps); otherwise to the row's entry at tokens_log
    if (tokens_log) {
      const int64_t at = log_pos_base >= 0 && pos ? (int64_t)(pos[b] - log_pos_base + 1) : 0;
      tokens_log[(size_t)b * log_stride + at] = tok;
    }
    if (pos) pos[b] += 1;
  }
  pdl_trigger();
}

__global__ void embed_kernel(const int32_t* __restrict__ tokens, int m, const __nv_bfloat16* __restrict__ emb,
                             int D, float* __restrict__ x) {
  pdl_wait();
  const int b = blockIdx.x;
  const int tok = tokens[b];
  for (int e = threadIdx.x; e < D; e += blockDim.x) x[(size_t)b * D + e] = __bfloat162float(emb[(size_t)tok * D + e]);
  pdl_trigger();
}

// RoPE + cache append for projections computed elsewhere (the multi-row
// question prefill's GEMMs): qkv [m][(hq + 2 hkv) d] f32 -> q_out [m][hq][d]
// f32, k / v rows (bf16) of row r at k_out + (r / rows_per_group) *
// group_stride + (r % rows_per_group) * row_stride (one group per dialogue).
__global__ void rope_rows_kernel(const float* __restrict__ qkv, int m, int hq, int hkv, int d,
                                 const int32_t* __restrict__ pos, const double* __restrict__ freq,
                                 float* __restrict__ q_out, __nv_bfloat16* __restrict__ k_out,
                                 __nv_bfloat16* __restrict__ v_out, int64_t row_stride, int rows_per_group,
                                 int64_t group_stride) {
  const int r = blockIdx.x;
  const int qd = hq * d, kd = hkv * d, W = qd + 2 * kd;
  const float* src = qkv + (size_t)r * W;
  const int64_t kv_off = (int64_t)(r / rows_per_group) * group_stride + (int64_t)(r % rows_per_group) * row_stride;
  for (int pr = threadIdx.x; pr < W / 2; pr += blockDim.x) {
    const int n = 2 * pr;
    const float x0 = src[n], x1 = src[n + 1];
    if (n < qd + kd) {
      const int i = (n % d) >> 1;
      double sn, cs;
      sincos((double)pos[r] * freq[i], &sn, &cs);
      const float y0 = (float)((double)x0 * cs - (double)x1 * sn);
      const float y1 = (float)((double)x0 * sn + (double)x1 * cs);
      if (n < qd) {
        q_out[(size_t)r * qd + n] = y0;
        q_out[(size_t)r * qd + n + 1] = y1;
      } else {
        *reinterpret_cast<uint32_t*>(k_out + kv_off + (n - qd)) = pack_bf16(y0, y1);
      }
    } else {
      *reinterpret_cast<uint32_t*>(v_out + kv_off + (n - qd - kd)) = pack_bf16(x0, x1);
    }
  }
}

}  // namespace rk

using namespace rk;

extern "C" {

size_t rk_packed_weight_bytes(int k, int n) {
  return (size_t)((n + pj::BM - 1) / pj::BM * pj::BM) * (size_t)k * sizeof(__nv_bfloat16);
}

int rk_pack_weight(const void* w, int w_dtype, int k, int n, void* packed, rk_stream_t stream) {
  if (k <= 0 || n <= 0 || k % pj::BK != 0)
    return fail(RK_ERR_DOMAIN, "pack_weight k=%d (multiple of %d), n=%d", k, pj::BK, n);
  const int np = (n + pj::BM - 1) / pj::BM * pj::BM;
  const size_t threads = (size_t)np * (k / 8);
  const int blocks = (int)((threads + 255) / 256);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (w_dtype == RK_F32)
    pack_weight_kernel<float><<<blocks, 256, 0, st>>>((const float*)w, k, n, np, (__nv_bfloat16*)packed);
  else if (w_dtype == RK_BF16)
    pack_weight_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)w, k, n, np,
                                                              (__nv_bfloat16*)packed);
  else
    return fail(RK_ERR_DOMAIN, "weight dtype %d", w_dtype);
  RK_CHECK_LAUNCH("pack_weight_kernel");
  return RK_OK;
}

size_t rk_proj_workspace_bytes(int m, int k, int n) {
  if (m <= 0 || k <= 0 || n <= 0) return 256;
  return proj_plan(m, k, n).total;
}

int rk_qkv_rope(const float* x, int m, int d_model, const void* w_qkv_packed, int hq, int hkv, int d,
                const int32_t* pos, const double* rope_freq, float* q_out, void* k_out, void* v_out,
                int64_t kv_row_stride, void* workspace, size_t workspace_bytes, rk_stream_t stream) {
  return rk_qkv_rope_kv(x, m, d_model, w_qkv_packed, hq, hkv, d, pos, rope_freq, q_out, k_out, v_out, RK_BF16,
                        kv_row_stride, workspace, workspace_bytes, stream);
}

int rk_qkv_rope_kv(const float* x, int m, int d_model, const void* w_qkv_packed, int hq, int hkv, int d,
                   const int32_t* pos, const double* rope_freq, float* q_out, void* k_out, void* v_out,
                   int kv_dtype, int64_t kv_row_stride, void* workspace, size_t workspace_bytes,
                   rk_stream_t stream) {
  if (hkv <= 0 || hq % hkv != 0 || d % 2 != 0) return fail(RK_ERR_DOMAIN, "qkv heads %d/%d, d %d", hq, hkv, d);
  if (kv_dtype != RK_BF16 && kv_dtype != RK_F32) return fail(RK_ERR_DOMAIN, "kv dtype %d", kv_dtype);
  pj::Params p{};
  p.m = m;
  p.K = d_model;
  p.N = (hq + 2 * hkv) * d;
  p.mode = pj::PJ_QKV;
  p.hq = hq;
  p.hkv = hkv;
  p.d = d;
  p.pos = pos;
  p.freq = rope_freq;
  p.q_out = q_out;
  p.k_out = k_out;
  p.v_out = v_out;
  p.kv_stride = kv_row_stride;
  p.kv_f32 = kv_dtype == RK_F32;
  return launch_proj(p, x, w_qkv_packed, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int rk_out_proj(const float* a, int m, int k, const void* w_o_packed, int d_model, float* resid,
                void* workspace, size_t workspace_bytes, rk_stream_t stream) {
  return rk_out_proj_rows(a, m, k, w_o_packed, d_model, resid, nullptr, workspace, workspace_bytes, stream);
}

int rk_out_proj_rows(const float* a, int m, int k, const void* w_o_packed, int d_model, float* resid,
                     const int32_t* row_active, void* workspace, size_t workspace_bytes, rk_stream_t stream) {
  pj::Params p{};
  p.row_active = row_active;
  p.m = m;
  p.K = k;
  p.N = d_model;
  p.mode = pj::PJ_OUT;
  p.resid = resid;
  return launch_proj(p, a, w_o_packed, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

size_t rk_lm_head_workspace_bytes(int m, int vocab, int d_model) {
  if (m <= 0 || vocab <= 0 || d_model <= 0) return 256;
  return proj_plan(m, d_model, vocab).total;
}

int rk_lm_head(const float* x, int m, int d_model, const void* emb_packed, int vocab, const void* emb,
               float* x_next, int32_t* tokens, int32_t* pos, int32_t* tokens_log, int log_stride,
               void* workspace, size_t workspace_bytes, rk_stream_t stream) {
  return rk_lm_head_rows(x, m, d_model, emb_packed, vocab, emb, x_next, tokens, pos, tokens_log, log_stride, nullptr,
                         -1, workspace, workspace_bytes, stream);
}

int rk_lm_head_rows(const float* x, int m, int d_model, const void* emb_packed, int vocab, const void* emb,
                    float* x_next, int32_t* tokens, int32_t* pos, int32_t* tokens_log, int log_stride,
                    const int32_t* row_active, int log_pos_base, void* workspace, size_t workspace_bytes,
                    rk_stream_t stream) {
  if (m <= 0) return RK_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // rows in chunks of 64 (the projection's MMA N bound); each chunk's logits reuse the
  // workspace after the previous chunk's argmax (stream order; the projection's epilogue
  // writes only after griddepcontrol.wait)
  for (int m0 = 0; m0 < m; m0 += 64) {
    const int mc = m - m0 < 64 ? m - m0 : 64;
    pj::Params p{};
    p.m = mc;
    p.K = d_model;
    p.N = vocab;
    p.mode = pj::PJ_HEAD;
    int rc = launch_proj(p, x + (size_t)m0 * d_model, emb_packed, workspace, workspace_bytes, st);
    if (rc != RK_OK) return rc;
    const ProjPlan pl = proj_plan(mc, d_model, vocab);
    const float* logits = reinterpret_cast<const float*>(reinterpret_cast<const uint8_t*>(workspace) + pl.logits_off);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(mc);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, argmax_embed_kernel, logits, pl.Npad, vocab,
                                       (const __nv_bfloat16*)emb, d_model, x_next + (size_t)m0 * d_model,
                                       tokens ? tokens + m0 : tokens, pos ? pos + m0 : pos,
                                       tokens_log ? tokens_log + (size_t)m0 * log_stride : tokens_log, log_stride,
                                       row_active ? row_active + m0 : row_active, log_pos_base);
    if (e != cudaSuccess) return cuda_status(e, "argmax_embed_kernel launch");
  }
  return RK_OK;
}

int rk_rope_rows(const float* qkv, int m, int hq, int hkv, int d, const int32_t* pos, const double* rope_freq,
                 float* q_out, void* k_out, void* v_out, int64_t kv_row_stride, int rows_per_group,
                 int64_t kv_group_stride, rk_stream_t stream) {
  if (m <= 0) return RK_OK;
  if (rows_per_group <= 0 || d % 2) return fail(RK_ERR_DOMAIN, "rope_rows: rows_per_group %d, d %d", rows_per_group, d);
  rope_rows_kernel<<<m, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      qkv, m, hq, hkv, d, pos, rope_freq, q_out, reinterpret_cast<__nv_bfloat16*>(k_out),
      reinterpret_cast<__nv_bfloat16*>(v_out), kv_row_stride, rows_per_group, kv_group_stride);
  RK_CHECK_LAUNCH("rope_rows_kernel");
  return RK_OK;
}

int rk_embed(const int32_t* tokens, int m, const void* emb, int d_model, float* x, rk_stream_t stream) {
  if (m <= 0) return RK_OK;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(m);
  cfg.blockDim = dim3(256);
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, embed_kernel, tokens, m, (const __nv_bfloat16*)emb, d_model, x);
  if (e != cudaSuccess) return cuda_status(e, "embed_kernel launch");
  return RK_OK;
}

#ifdef PJ_TRACE
int rk_debug_proj_trace(unsigned long long* out, int n) {  // n <= 16384
  return cudaMemcpyFromSymbol(out, pj::g_pj_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}
int rk_debug_proj_units(unsigned long long* out) {       // 3 x 64
  return cudaMemcpyFromSymbol(out, pj::g_pj_units, sizeof(unsigned long long) * 192) == cudaSuccess ? 0 : -1;
}
#endif

}  // extern "C"
