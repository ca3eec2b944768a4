// The whole decode token step in ONE persistent launch (small batches).
//
// The layered path runs every layer as qkv -> attention -> out kernels (97
// launches per token at C2 shapes); at B <= 16 each launch is short and the
// token step is bound by that dependency chain: each kernel pays the previous
// one's completion, an L2 round trip for its activations and a split-K tail
// (B = 1 at 0.52 of the copy peak).  Here one CTA per SM runs the
// entire step — for every layer l: QKV(l) (projection + RoPE + KV append),
// ATT(l) (split-K decode attention over the cached keys), MRG(l) (merge of the
// split-K partials + the new key), OUT(l) (projection + residual); then the
// tied logits and the first-max argmax + embedding of the next token
// (engine.py:244-271, pipeline.py:298-313 of the reference).
//
// What makes it faster is that the BYTES of the step do not depend on its
// arithmetic: the weights of every projection and the cached K/V of every
// layer (all rows but the one appended this step) are known at launch.  Each
// CTA's producer warp streams its fixed share of them — weight tiles by bulk
// copy, K/V boxes by TMA — through one ring of 16 KB stages in schedule order,
// never waiting on a dependency, only on free stages; the consumer warps
// follow the same schedule and wait on device-scope phase counters only for
// their activations.  While a CTA waits for the slowest strip of the previous
// phase, its ring keeps filling with the next phase's bytes, so the HBM stream
// does not stop at phase boundaries the way a kernel boundary stops it.
//
// Schedule (identical in producer and consumers): per layer the units of a
// phase are split into equal contiguous runs over the CTAs (so every SM
// streams the same bytes):
//   QKV/OUT unit (strip sg of 128 features, k-chunk kc of 64): one 16 KB tile of
//     the rk_pack_weight image (swizzled K-major W^T), consumed by mma.sync
//     m16n8k16 (bf16 hi/lo split of the fp32 activations, fp32 accumulate;
//     warp w owns features 16w..16w+15); a run's partial per strip goes to the
//     workspace and the last contributor (ticket) adds them in CTA order and
//     runs the epilogue (RoPE + q / KV row stores; residual add; logits);
//   ATT tile (dialogue b, kv-head h, 64 keys): K then V, each two 64 x 64 TMA
//     boxes (128-byte swizzle); warp w takes keys 8w..8w+7 (S = Q K^T with
//     the q hi/lo split, online softmax in log2 units, O += P V with the
//     probabilities split hi/lo); a run's state per (b, h) is merged over the
//     warps and written as a split-K partial (m, l, O);
//   MRG item (b, h): the partials in CTA order + the appended key -> the
//     attention output rows of the group's query heads.
// Counters are monotonic (targets = (epoch + 1) x count), so nothing is
// reset between launches; every wait is bounded (trap, never a hang).
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "decode_common.cuh"
#include "tc_common.cuh"

namespace rk {
namespace stp {

constexpr int kCW = 8;                         // consumer warps
constexpr int kThreads = (kCW + 1) * 32;       // + the producer warp
constexpr int kStage = 16384;                  // ring stage: one weight tile / half an attention tile
constexpr int BM = 128, BK = 64, KEYS = 64;
constexpr int kMaxB = 16, kMaxG = 8, kMaxL = 128;
constexpr int kSmemMax = 227 * 1024;

enum { QKV = 0, OUT = 1, HEAD = 2 };
enum { C_QKV = 0, C_ATT = 1, C_MRG = 2, C_OUT = 3 };

struct Proj {
  int n_sg, KC, n_units, Gp, maxc;
  float* part;                // [n_sg][maxc][B][128]
  unsigned* tickets;          // [L][n_sg] (HEAD: [n_sg])
};

struct Params {
  CUtensorMap map_lo, map_up;                  // 4-D: d, hkv, seq, (b * layers + l) * 2 + kv
  int B, L, lw, hq, hkv, d, D, vocab, Gq, NS, xs_bytes;
  int64_t s_lo, s_up;
  float* x;                                    // [B][D] residual stream
  float* q;                                    // [B][hq][d] (workspace)
  float* attn;                                 // [B][D] (workspace)
  float* logits;                               // [B][npad] (workspace)
  int npad;
  __nv_bfloat16* lower;
  __nv_bfloat16* upper;
  int32_t* lower_len;
  int32_t* upper_len;
  int32_t* pos;
  const double* freq;
  const void* const* w_qkv;
  const void* const* w_o;
  const void* emb_packed;
  const __nv_bfloat16* emb;
  int32_t* tokens;
  int32_t* tokens_log;
  int log_stride;
  Proj pj[3];
  float* part_att;                             // [B][hkv][maxs][2 Gq + Gq d]
  int maxs, mrg_split;                         // merge items split d into mrg_split slices
  unsigned* hdr;                               // [0] epoch, [1] watchdog code
  unsigned* cnt;                               // [L][4] + [4 L] head
  float scale_log2;
};

#ifdef STP_TRACE   // timing experiments: %globaltimer per (CTA, layer, point) of the last launch
constexpr int kTP = 10;
__device__ unsigned long long g_stp_trace[160 * 64 * kTP];
#define STT(l, k)                                                                          \
  do {                                                                                     \
    if (threadIdx.x == 0 && (l) < 64) {                                                    \
      unsigned long long _t;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                               \
      g_stp_trace[(blockIdx.x * 64 + (l)) * kTP + (k)] = _t;                               \
    }                                                                                      \
  } while (0)
#define STP_PROD(l, k)                                                                     \
  do {                                                                                     \
    if ((l) < 64) {                                                                        \
      unsigned long long _t;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                               \
      g_stp_trace[(blockIdx.x * 64 + (l)) * kTP + (k)] = _t;                               \
    }                                                                                      \
  } while (0)
#else
#define STT(l, k)
#define STP_PROD(l, k)
#endif

__device__ __forceinline__ int run_lo(int c, int n, int G) { return (int)((int64_t)c * n / G); }
__device__ __forceinline__ int owner(int u, int n, int G) { return (int)(((int64_t)(u + 1) * G - 1) / n); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void watchdog(unsigned* hdr, unsigned code) {
  atomicExch(hdr + 1, code);
  __threadfence();
  asm volatile("trap;");
}
// bounded waits: SM clocks before a wait traps (~2 s by default; RK_STEP_PATIENCE_S for
// slowed-down runs such as compute-sanitizer)
__device__ long long g_patience = 4ll << 30;

__device__ __forceinline__ bool bar_try(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bar_wait_b(uint64_t* bar, unsigned parity, unsigned* hdr, unsigned code) {
#ifdef STP_PLAIN_WAIT      // sanitizer experiments: the unbounded wait loop of the other kernels
  mbar_wait(bar, parity);
  return;
#endif
  if (bar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!bar_try(bar, parity))
    if (clock64() - t0 > g_patience) watchdog(hdr, code);
}
// every consumer thread calls this: thread 0 polls, the rest wait at the barrier
__device__ __forceinline__ void wait_count(const unsigned* c, unsigned target, unsigned* hdr, unsigned code) {
  if (threadIdx.x == 0 && (int)(ld_acquire(c) - target) < 0) {
    const long long t0 = clock64();
    while ((int)(ld_acquire(c) - target) < 0) {
      __nanosleep(32);
      if (clock64() - t0 > g_patience) watchdog(hdr, code);
    }
  }
  consumer_sync();
}

__device__ __forceinline__ void tma_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                       uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ float2 ldcg2(const float* p) { return __ldcg(reinterpret_cast<const float2*>(p)); }

__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const float ha = bf16_round(a), hb = bf16_round(b);
  hi = pack_bf16(ha, hb);
  lo = pack_bf16(a - ha, b - hb);
}

// the cache row of dialogue b at layer l (k: kv = 0, v: 1), `row` keys in
__device__ __forceinline__ __nv_bfloat16* cache_row(const Params& p, int l, int b, int kv, int row) {
  const bool lo = l < p.lw;
  const int Lt = lo ? p.lw : p.L - p.lw, lt = lo ? l : l - p.lw;
  const int64_t S = lo ? p.s_lo : p.s_up;
  __nv_bfloat16* base = lo ? p.lower : p.upper;
  return base + ((((int64_t)b * Lt + lt) * 2 + kv) * S + row) * (int64_t)(p.hkv * p.d);
}

struct AttLoc {
  int b, h, j, first, nt;
};
// tile idx of the layer's flattened (b, h, 64-key block) list
__device__ __forceinline__ AttLoc att_locate(int idx, const int* ntl, int B, int hkv) {
  int pre = 0;
  for (int b = 0; b < B; ++b) {
    const int span = ntl[b] * hkv;
    if (idx < pre + span) {
      const int r = idx - pre, h = r / ntl[b];
      return AttLoc{b, h, r - h * ntl[b], pre + h * ntl[b], ntl[b]};
    }
    pre += span;
  }
  return AttLoc{0, 0, 0, 0, 0};
}

struct Smem {
  uint8_t* ring;
  uint8_t* xs;
  float2* rope;             // [B][64] (cos, sin)
  uint64_t* full;
  uint64_t* empty;
  int* len_lo;              // [kMaxB] (consumers)
  int* len_up;
  int* nt_lo;               // tiles per dialogue, per tier
  int* nt_up;
  int* flag;
  int* tok;                 // [kMaxB]
};

// ----------------------------------------------------------------------------------------------
// consumer side
template <int NT>
struct Consumer {
  const Params& p;
  Smem s;
  unsigned E;               // launch epoch
  uint32_t seq;             // ring position
  int c, G, tid, warp, lane;

  __device__ unsigned* counter(int l, int k) { return p.cnt + l * 4 + k; }
  __device__ unsigned* head_counter() { return p.cnt + p.L * 4; }

  __device__ void signal(unsigned* ctr, unsigned v) {
    __threadfence();
    consumer_sync();
    if (tid == 0) atom_add_acq_rel(ctr, v);
  }

  // ---------------------------------------------------------------- projections
  __device__ void epilogue(int ph, int l, int sg, int pr, int t, float y0, float y1) {
    const int n = sg * BM + 2 * pr;
    if (ph == QKV) {
      const int qd = p.hq * p.d, kd = p.hkv * p.d;
      if (n >= qd + 2 * kd) return;
      if (n < qd + kd) {
        const float2 e = s.rope[t * 64 + ((n % p.d) >> 1)];
        const double cs = e.x, sn = e.y;
        const float a = (float)((double)y0 * cs - (double)y1 * sn), b = (float)((double)y0 * sn + (double)y1 * cs);
        if (n < qd)
          __stcg(reinterpret_cast<float2*>(p.q + (size_t)t * qd + n), make_float2(a, b));
        else
          *reinterpret_cast<uint32_t*>(cache_row(p, l, t, 0, t_len(l, t)) + (n - qd)) = pack_bf16(a, b);
      } else {
        *reinterpret_cast<uint32_t*>(cache_row(p, l, t, 1, t_len(l, t)) + (n - qd - kd)) = pack_bf16(y0, y1);
      }
    } else if (ph == OUT) {
      if (n >= p.D) return;
      float2* r = reinterpret_cast<float2*>(p.x + (size_t)t * p.D + n);
      const float2 o = __ldcg(r);
      __stcg(r, make_float2(o.x + y0, o.y + y1));
    } else {
      __stcg(reinterpret_cast<float2*>(p.logits + (size_t)t * p.npad + n), make_float2(y0, y1));
    }
  }
  __device__ int t_len(int l, int b) { return l < p.lw ? s.len_lo[b] : s.len_up[b]; }

  __device__ void finalize(int ph, int l, int sg, int ncontrib) {
    const Proj& P = p.pj[ph];
    const float* base = P.part + (size_t)sg * P.maxc * p.B * BM;
    for (int e = tid; e < 64 * p.B; e += kCW * 32) {
      const int t = e >> 6, pr = e & 63;
      const float* src = base + (size_t)t * BM + 2 * pr;
      float2 y = make_float2(0.f, 0.f);
      int s0 = 0;
      for (; s0 + 4 <= ncontrib; s0 += 4) {           // 4 loads in flight, added in contributor order
        float2 z[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) z[q] = ldcg2(src + (size_t)(s0 + q) * p.B * BM);
#pragma unroll
        for (int q = 0; q < 4; ++q) { y.x += z[q].x; y.y += z[q].y; }
      }
      for (; s0 < ncontrib; ++s0) {
        const float2 z = ldcg2(src + (size_t)s0 * p.B * BM);
        y.x += z.x;
        y.y += z.y;
      }
      epilogue(ph, l, sg, pr, t, y.x, y.y);
    }
  }

  __device__ void argmax_finish() {
    for (int b = warp; b < p.B; b += kCW) {
      const float* lg = p.logits + (size_t)b * p.npad;
      float best = -INFINITY;
      int bi = 0x7fffffff;
      for (int v = lane; v < p.vocab; v += 32) {
        const float z = __ldcg(lg + v);
        if (z > best) { best = z; bi = v; }          // ascending v per lane: keeps the first maximum
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float z = __shfl_xor_sync(0xffffffffu, best, o);
        const int i = __shfl_xor_sync(0xffffffffu, bi, o);
        if (z > best || (z == best && i < bi)) { best = z; bi = i; }
      }
      if (lane == 0) s.tok[b] = bi;
    }
    consumer_sync();
    if (tid < p.B) {
      const int b = tid, tok = s.tok[b];
      if (p.tokens) p.tokens[b] = tok;
      if (p.tokens_log) p.tokens_log[(size_t)b * p.log_stride] = tok;
      if (p.pos) p.pos[b] += 1;
      if (p.lower_len) p.lower_len[b] += 1;
      if (p.upper_len) p.upper_len[b] += 1;
    }
    for (int e = tid; e < p.B * p.D; e += kCW * 32) {
      const int b = e / p.D, i = e - b * p.D;
      p.x[e] = __bfloat162float(p.emb[(size_t)s.tok[b] * p.D + i]);
    }
    __threadfence();
    consumer_sync();
    if (tid == 0) atomicExch(p.hdr, E + 1);           // the next launch's epoch (read after griddepcontrol.wait)
  }

  __device__ void proj_phase(int ph, int l, const float* src) {
    const Proj& P = p.pj[ph];
    if (c >= P.Gp) return;
    const int u0 = run_lo(c, P.n_units, P.Gp), n = run_lo(c + 1, P.n_units, P.Gp) - u0;
    if (n <= 0) return;
    const int K = P.KC * BK;
    uint32_t* xs = reinterpret_cast<uint32_t*>(s.xs);
    // the run's activations as mma B fragments, [unit][k16 step][n-tile][hi, lo][lane] x (b0, b1):
    // one float4 (4 consecutive k of token t) per work element, up to kU in flight per thread
    constexpr int kU = 12;
    const int total = n * NT * 8 * 16;                       // units x tokens x float4 per 64 k
    for (int e0 = tid; e0 < total; e0 += kU * kCW * 32) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kCW * 32, f = e & 15, t = (e >> 4) % (NT * 8), i = (e >> 4) / (NT * 8);
        v[u] = (e < total && t < p.B)
                   ? __ldcg(reinterpret_cast<const float4*>(src + (size_t)t * K + ((u0 + i) % P.KC) * BK) + f)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int e = e0 + u * kCW * 32;
        if (e >= total) break;
        const int f = e & 15, t = (e >> 4) % (NT * 8), i = (e >> 4) / (NT * 8);
        const int ks = f >> 2, kk = 4 * (f & 3), nt = t >> 3, g = t & 7;
        // pairs (kk, kk+1) and (kk+2, kk+3) of the k16 step: b0 (kk < 8) or b1 of lanes g*4 + (kk % 8) / 2 (+1)
        const int half_b = kk >= 8 ? 1 : 0, cc0 = (kk & 7) >> 1;
        uint32_t h0, l0, h1, l1;
        split2(v[u].x, v[u].y, h0, l0);
        split2(v[u].z, v[u].w, h1, l1);
        const size_t hi_base = (size_t)(((i * 4 + ks) * NT + nt) * 2 + 0) * 32;
        const size_t lo_base = hi_base + 32;
        const int ln0 = g * 4 + cc0;
        xs[(hi_base + ln0) * 2 + half_b] = h0;
        xs[(lo_base + ln0) * 2 + half_b] = l0;
        xs[(hi_base + ln0 + 1) * 2 + half_b] = h1;
        xs[(lo_base + ln0 + 1) * 2 + half_b] = l1;
      }
    }
    consumer_sync();
    STT(l, ph == OUT ? 7 : 1);
    const int g = lane >> 2, cc = lane & 3;
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
    for (int i = 0; i < n; ++i) {
      const int st = seq % p.NS;
      bar_wait_b(&s.full[st], (seq / p.NS) & 1, p.hdr, 10 + ph);
      const uint8_t* tile = s.ring + (size_t)st * kStage;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t a[4];
        const int j = lane >> 3, row = 16 * warp + ((j & 1) << 3) + (lane & 7), ch = 2 * ks + (j >> 1);
        ldmatrix_x4(a, tile + row * 128 + ((ch ^ (row & 7)) << 4));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint2 bh = reinterpret_cast<const uint2*>(xs)[(size_t)(((i * 4 + ks) * NT + nt) * 2 + 0) * 32 + lane];
          const uint2 bl = reinterpret_cast<const uint2*>(xs)[(size_t)(((i * 4 + ks) * NT + nt) * 2 + 1) * 32 + lane];
          mma_bf16_16816(acc[nt], a, bh.x, bh.y);
          mma_bf16_16816(acc[nt], a, bl.x, bl.y);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.empty[st]);
      ++seq;
      const int u = u0 + i, kc = u % P.KC;
      if (i == n - 1 || kc == P.KC - 1) {
        // segment end: this run's partial of strip sg, then the strip's ticket
        const int sg = u / P.KC;
        const int cf = owner(sg * P.KC, P.n_units, P.Gp), cl = owner(sg * P.KC + P.KC - 1, P.n_units, P.Gp);
        float* part = P.part + ((size_t)(sg * P.maxc + (c - cf)) * p.B) * BM;
        const int r0 = 16 * warp + g;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int t0 = nt * 8 + 2 * cc;
          if (t0 < p.B) {
            __stcg(part + (size_t)t0 * BM + r0, acc[nt][0]);
            __stcg(part + (size_t)t0 * BM + r0 + 8, acc[nt][2]);
          }
          if (t0 + 1 < p.B) {
            __stcg(part + (size_t)(t0 + 1) * BM + r0, acc[nt][1]);
            __stcg(part + (size_t)(t0 + 1) * BM + r0 + 8, acc[nt][3]);
          }
          acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
        }
        __threadfence();
        consumer_sync();
        unsigned* tk = P.tickets + (ph == HEAD ? 0 : l * P.n_sg) + sg;
        const unsigned nc = (unsigned)(cl - cf + 1);
        if (tid == 0) *s.flag = atom_add_acq_rel(tk, 1u) == (E + 1) * nc - 1;
        consumer_sync();
        if (*s.flag) {
          finalize(ph, l, sg, (int)nc);
          __threadfence();
          consumer_sync();
          if (ph == HEAD) {
            if (tid == 0) *s.flag = atom_add_acq_rel(head_counter(), 1u) == (E + 1) * (unsigned)P.n_sg - 1;
            consumer_sync();
            if (*s.flag) argmax_finish();
          } else if (tid == 0) {
            atom_add_acq_rel(counter(l, ph == QKV ? C_QKV : C_OUT), 1u);
          }
        }
        consumer_sync();        // *s.flag is rewritten at the next segment end
      }
    }
  }

  // ---------------------------------------------------------------- attention
  __device__ void att_phase(int l) {
    const bool lo = l < p.lw;
    const int* ntl = lo ? s.nt_lo : s.nt_up;
    const int* lens = lo ? s.len_lo : s.len_up;
    int T = 0;
    for (int b = 0; b < p.B; ++b) T += ntl[b] * p.hkv;
    const int Ga = min(G, T);
    if (c >= Ga) return;
    const int a0 = run_lo(c, T, Ga), a1 = run_lo(c + 1, T, Ga);
    const int g = lane >> 2, cc = lane & 3;
    float* sm_m = reinterpret_cast<float*>(s.xs);            // [8 warps][8]
    float* sm_l = sm_m + kCW * kMaxG;
    float* sm_o = sm_l + kCW * kMaxG;                        // [8 warps][Gq][d]
    for (int idx = a0; idx < a1;) {
      const AttLoc at = att_locate(idx, ntl, p.B, p.hkv);
      const int end = min(a1, at.first + at.nt), len = lens[at.b];
      // q fragments (rows 0-7: hi, 8-15: lo of the group's heads; pre-scaled to log2 units)
      uint32_t qa[8][4];
      {
        const bool real = g < p.Gq;
        const float* qp = p.q + ((size_t)at.b * p.hq + at.h * p.Gq + (real ? g : 0)) * p.d;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          float2 x0 = ldcg2(qp + 16 * ks + 2 * cc), x1 = ldcg2(qp + 16 * ks + 2 * cc + 8);
          const float sc = real ? p.scale_log2 : 0.f;
          split2(x0.x * sc, x0.y * sc, qa[ks][0], qa[ks][1]);
          split2(x1.x * sc, x1.y * sc, qa[ks][2], qa[ks][3]);
        }
      }
      float o[16][4];
#pragma unroll
      for (int nt = 0; nt < 16; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
      float m = -INFINITY, lsum = 0.f;
      for (int j = at.j; idx < end; ++idx, ++j) {
        // ---- K stage: S = Q K^T for keys 8w..8w+7 of the block
        int st = seq % p.NS;
        bar_wait_b(&s.full[st], (seq / p.NS) & 1, p.hdr, 20);
        const uint8_t* kt = s.ring + (size_t)st * kStage;
        const int r = 8 * warp + (lane & 7);
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kp = 0; kp < 4; ++kp) {
          uint32_t kb[4];
          const int ch = 4 * kp + (lane >> 3);
          ldmatrix_x4(kb, kt + (ch >> 3) * 8192 + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
          mma_bf16_16816(sacc, qa[2 * kp], kb[0], kb[1]);
          mma_bf16_16816(sacc, qa[2 * kp + 1], kb[2], kb[3]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.empty[st]);
        ++seq;
        const int key0 = KEYS * j + 8 * warp + 2 * cc;
        float s0 = sacc[0] + sacc[2], s1 = sacc[1] + sacc[3];
        if (key0 >= len) s0 = -INFINITY;
        if (key0 + 1 >= len) s1 = -INFINITY;
        float mt = fmaxf(s0, s1);
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
        const float mn = fmaxf(m, mt);
        float p0 = 0.f, p1 = 0.f, alpha = 1.f;
        if (mn != -INFINITY) {
          alpha = exp2f(m - mn);                         // m = -inf -> 0
          p0 = exp2f(s0 - mn);
          p1 = exp2f(s1 - mn);
        }
        m = mn;
        lsum = lsum * alpha + p0 + p1;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt) {
          o[nt][0] *= alpha;
          o[nt][1] *= alpha;
          o[nt][2] *= alpha;
          o[nt][3] *= alpha;
        }
        uint32_t pa[4];
        split2(p0, p1, pa[0], pa[1]);
        pa[2] = pa[3] = 0u;
        // ---- V stage: O += P V
        st = seq % p.NS;
        bar_wait_b(&s.full[st], (seq / p.NS) & 1, p.hdr, 21);
        uint8_t* vt = s.ring + (size_t)st * kStage;
        if (KEYS * j + 8 * warp + 7 >= len) {
          // rows past the dialogue's keys hold stale bytes (possibly non-finite): zero them
          for (int e = lane; e < 8 * 16; e += 32) {
            const int rr = 8 * warp + (e >> 4), ch = e & 15;
            if (KEYS * j + rr >= len)
              *reinterpret_cast<uint4*>(vt + (ch >> 3) * 8192 + rr * 128 + ((ch & 7) << 4)) = make_uint4(0, 0, 0, 0);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint32_t vb[4];
          const int ch = 4 * q4 + (lane >> 3);
          ldmatrix_x4_trans(vb, vt + (ch >> 3) * 8192 + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) mma_bf16_16816(o[4 * q4 + jj], pa, vb[jj], 0u);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.empty[st]);
        ++seq;
      }
      // ---- the run's state for (b, h): merge the 8 warps, write the split-K partial
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
      if (g < p.Gq) {
        if (cc == 0) {
          sm_m[warp * kMaxG + g] = m;
          sm_l[warp * kMaxG + g] = lsum;
        }
        float* ow = sm_o + ((size_t)warp * p.Gq + g) * p.d;
#pragma unroll
        for (int nt = 0; nt < 16; ++nt)
          *reinterpret_cast<float2*>(ow + 8 * nt + 2 * cc) = make_float2(o[nt][0] + o[nt][2], o[nt][1] + o[nt][3]);
      }
      consumer_sync();
      const int slot = c - owner(at.first, T, Ga);
      float* pa = p.part_att + (((size_t)at.b * p.hkv + at.h) * p.maxs + slot) * (size_t)(2 * p.Gq + p.Gq * p.d);
      for (int e = tid; e < p.Gq * p.d; e += kCW * 32) {
        const int gg = e / p.d, dim = e - gg * p.d;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kCW; ++w) M = fmaxf(M, sm_m[w * kMaxG + gg]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kCW; ++w) {
          const float mw = sm_m[w * kMaxG + gg];
          const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
          L += f * sm_l[w * kMaxG + gg];
          O += f * sm_o[((size_t)w * p.Gq + gg) * p.d + dim];
        }
        __stcg(pa + 2 * p.Gq + e, O);
        if (dim == 0) {
          __stcg(pa + gg, M);
          __stcg(pa + p.Gq + gg, L);
        }
      }
      consumer_sync();            // the scratch is rewritten by the next run
    }
  }

  // items (b, h, slice of d / ds dims): the partials' (m, l) into shared memory while each
  // thread's O values of up to kZ slots are already in flight; then the appended key
  __device__ void merge_phase(int l, int items) {
    const bool lo = l < p.lw;
    const int* ntl = lo ? s.nt_lo : s.nt_up;
    const int* lens = lo ? s.len_lo : s.len_up;
    int T = 0;
    for (int b = 0; b < p.B; ++b) T += ntl[b] * p.hkv;
    const int Ga = max(1, min(G, T));
    const int ds = p.mrg_split, dper = p.d / ds;
    const size_t psz = (size_t)(2 * p.Gq + p.Gq * p.d);
    float* sm_m = reinterpret_cast<float*>(s.xs);            // [maxs][Gq]
    float* sm_l = sm_m + p.maxs * kMaxG;
    float* sm_s = sm_l + p.maxs * kMaxG;                     // [Gq] new-key logits
    constexpr int kZ = 24;
    for (int it = c; it < items; it += G) {
      const int part = it % ds, bh = it / ds, b = bh / p.hkv, h = bh - b * p.hkv;
      int pre = 0;
      for (int bb = 0; bb < b; ++bb) pre += ntl[bb] * p.hkv;
      const int first = pre + h * ntl[b], nt = ntl[b];
      const int ns = nt > 0 ? owner(first + nt - 1, T, Ga) - owner(first, T, Ga) + 1 : 0;
      const float* pa = p.part_att + ((size_t)b * p.hkv + h) * p.maxs * psz;
      const __nv_bfloat16* kn = cache_row(p, l, b, 0, lens[b]) + h * p.d;
      const __nv_bfloat16* vn = cache_row(p, l, b, 1, lens[b]) + h * p.d;
      const int e = tid, g = e / dper, dim = part * dper + (e - g * dper);
      const bool mine = e < p.Gq * dper;
      float z[kZ];
#pragma unroll
      for (int q = 0; q < kZ; ++q) z[q] = (mine && q < ns) ? __ldcg(pa + q * psz + 2 * p.Gq + g * p.d + dim) : 0.f;
      const float vnew = mine ? __bfloat162float(__ldcg(vn + dim)) : 0.f;
      for (int f = tid; f < ns * p.Gq; f += kCW * 32) {
        const int sl = f / p.Gq, gg = f - sl * p.Gq;
        sm_m[f] = __ldcg(pa + sl * psz + gg);
        sm_l[f] = __ldcg(pa + sl * psz + p.Gq + gg);
      }
      if (warp < p.Gq) {
        const float* qp = p.q + ((size_t)b * p.hq + h * p.Gq + warp) * p.d;
        float dot = 0.f;
        for (int i = lane; i < p.d / 4; i += 32) {
          const float4 qv = __ldcg(reinterpret_cast<const float4*>(qp) + i);
          const uint2 kw = __ldcg(reinterpret_cast<const uint2*>(kn) + i);
          const float2 k0 = bf16x2_to_f2(kw.x), k1 = bf16x2_to_f2(kw.y);
          dot += qv.x * k0.x + qv.y * k0.y + qv.z * k1.x + qv.w * k1.y;
        }
        dot = group_sum<32>(dot);
        if (lane == 0) sm_s[warp] = dot * p.scale_log2;
      }
      consumer_sync();
      if (mine) {
        const float snew = sm_s[g];
        float M = snew;
        for (int sl = 0; sl < ns; ++sl) M = fmaxf(M, sm_m[sl * p.Gq + g]);
        const float fn = exp2f(snew - M);
        float L = fn, acc = fn * vnew;
#pragma unroll
        for (int q = 0; q < kZ; ++q) {
          if (q >= ns) break;
          const float ms = sm_m[q * p.Gq + g];
          const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
          L += w * sm_l[q * p.Gq + g];
          acc += w * z[q];
        }
        for (int sl = kZ; sl < ns; ++sl) {
          const float ms = sm_m[sl * p.Gq + g];
          const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
          L += w * sm_l[sl * p.Gq + g];
          acc += w * __ldcg(pa + sl * psz + 2 * p.Gq + g * p.d + dim);
        }
        __stcg(p.attn + (size_t)b * p.D + (h * p.Gq + g) * p.d + dim, acc / L);
      }
      consumer_sync();
    }
  }

  __device__ void run() {
    const int npj[2] = {p.pj[QKV].n_sg, p.pj[OUT].n_sg};
    for (int l = 0; l < p.L; ++l) {
      if (l > 0) wait_count(counter(l - 1, C_OUT), (E + 1) * (unsigned)npj[1], p.hdr, 1);
      STT(l, 0);
      proj_phase(QKV, l, p.x);
      STT(l, 2);
      wait_count(counter(l, C_QKV), (E + 1) * (unsigned)npj[0], p.hdr, 2);
      STT(l, 3);
      att_phase(l);
      signal(counter(l, C_ATT), 1u);
      STT(l, 4);
      const int items = p.B * p.hkv * p.mrg_split;
      if (c < items) {
        wait_count(counter(l, C_ATT), (E + 1) * (unsigned)G, p.hdr, 3);
        merge_phase(l, items);
        int mine = 0;
        for (int it = c; it < items; it += G) ++mine;
        signal(counter(l, C_MRG), (unsigned)mine);
      }
      STT(l, 5);
      wait_count(counter(l, C_MRG), (E + 1) * (unsigned)items, p.hdr, 4);
      STT(l, 6);
      proj_phase(OUT, l, p.attn);
      STT(l, 8);
    }
    if (c < p.pj[HEAD].Gp) {
      wait_count(counter(p.L - 1, C_OUT), (E + 1) * (unsigned)npj[1], p.hdr, 5);
      proj_phase(HEAD, p.L - 1, p.x);
    }
  }
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) step_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Smem s;
  s.ring = base;
  s.xs = base + (size_t)p.NS * kStage;
  s.rope = reinterpret_cast<float2*>(s.xs + p.xs_bytes);
  s.full = reinterpret_cast<uint64_t*>(s.rope + kMaxB * 64);
  s.empty = s.full + p.NS;
  s.len_lo = reinterpret_cast<int*>(s.empty + p.NS);
  s.len_up = s.len_lo + kMaxB;
  s.nt_lo = s.len_up + kMaxB;
  s.nt_up = s.nt_lo + kMaxB;
  s.tok = s.nt_up + kMaxB;
  s.flag = s.tok + kMaxB;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.NS; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // every CTA is resident: the next step's grid may launch and take SMs as they free
  pdl_trigger();

  if (warp == kCW) {
    // ================= producer: the CTA's bytes of the whole step, in schedule order
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      uint32_t seq = 0;
      auto stage = [&]() -> int {
        const int st = seq % p.NS;
        if (seq >= (uint32_t)p.NS) bar_wait_b(&s.empty[st], ((seq / p.NS) - 1) & 1, p.hdr, 30);
        return st;
      };
      auto put_w = [&](const void* src) {
        const int st = stage();
        mbar_expect_tx(&s.full[st], kStage);
        bulk_g2s(s.ring + (size_t)st * kStage, src, kStage, &s.full[st], pol);
        ++seq;
      };
      auto proj_tiles = [&](int ph, const void* w) {
        const Proj& P = p.pj[ph];
        if (c >= P.Gp) return;
        const int u0 = run_lo(c, P.n_units, P.Gp), u1 = run_lo(c + 1, P.n_units, P.Gp);
        for (int u = u0; u < u1; ++u) put_w(static_cast<const uint8_t*>(w) + (size_t)u * kStage);
      };
      int nt_lo[kMaxB], nt_up[kMaxB];
      bool waited = false;
      for (int l = 0; l < p.L; ++l) {
        proj_tiles(QKV, p.w_qkv[l]);
        if (!waited) {
          pdl_wait();            // the cached rows appended by the previous step, the lengths
          for (int b = 0; b < p.B; ++b) {
            nt_lo[b] = (__ldcg(p.lower_len + b) + KEYS - 1) / KEYS;
            nt_up[b] = (__ldcg(p.upper_len + b) + KEYS - 1) / KEYS;
          }
          waited = true;
        }
        const bool lo = l < p.lw;
        const int* ntl = lo ? nt_lo : nt_up;
        const CUtensorMap* map = lo ? &p.map_lo : &p.map_up;
        const int Lt = lo ? p.lw : p.L - p.lw, lt = lo ? l : l - p.lw;
        int T = 0;
        for (int b = 0; b < p.B; ++b) T += ntl[b] * p.hkv;
        const int Ga = min(G, T);
        const int a0 = c < Ga ? run_lo(c, T, Ga) : 0, a1 = c < Ga ? run_lo(c + 1, T, Ga) : 0;
        for (int idx = a0; idx < a1; ++idx) {
          const AttLoc at = att_locate(idx, ntl, p.B, p.hkv);
          for (int kv = 0; kv < 2; ++kv) {
            const int st = stage();
            uint8_t* dst = s.ring + (size_t)st * kStage;
            const int blk = (at.b * Lt + lt) * 2 + kv;
            mbar_expect_tx(&s.full[st], kStage);
            tma_4d(dst, map, 0, at.h, KEYS * at.j, blk, &s.full[st], pol);
            tma_4d(dst + 8192, map, 64, at.h, KEYS * at.j, blk, &s.full[st], pol);
            ++seq;
          }
        }
        proj_tiles(OUT, p.w_o[l]);
        STP_PROD(l, 9);
      }
      proj_tiles(HEAD, p.emb_packed);
    }
    return;
  }

  // ================= consumers
  pdl_wait();
  const int tid = threadIdx.x;
  if (tid < p.B) {
    const int a = __ldcg(p.lower_len + tid), b = __ldcg(p.upper_len + tid);
    s.len_lo[tid] = a;
    s.len_up[tid] = b;
    s.nt_lo[tid] = (a + KEYS - 1) / KEYS;
    s.nt_up[tid] = (b + KEYS - 1) / KEYS;
  }
  for (int e = tid; e < p.B * 64; e += kCW * 32) {
    const int t = e >> 6, pr = e & 63;
    double sn, cs;
    sincos((double)__ldcg(p.pos + t) * p.freq[pr], &sn, &cs);
    s.rope[e] = make_float2((float)cs, (float)sn);
  }
  Consumer<NT> cons{p, s, __ldcg(p.hdr), 0u, c, G, tid, warp, lane};
  consumer_sync();
  cons.run();
}

}  // namespace stp

struct StepPlan {
  int G, Gq, KC, maxs, maxrun, NT, NS, xs_bytes, npad;
  int n_sg[3], n_units[3], Gp[3], maxc[3];
  size_t off_cnt, off_tk[3], off_part[3], off_att, off_q, off_attn, off_logits, total, smem;
};

static StepPlan step_plan(int B, int L, int hq, int hkv, int d, int vocab) {
  StepPlan pl{};
  pl.G = sm_count();
  pl.Gq = hq / hkv;
  const int D = hq * d;
  pl.KC = D / stp::BK;
  pl.npad = (vocab + stp::BM - 1) / stp::BM * stp::BM;
  const int N[3] = {(hq + 2 * hkv) * d, D, vocab};
  size_t off = 256;                                        // header: epoch, watchdog code
  pl.off_cnt = off;
  off += align_up(sizeof(unsigned) * (size_t)(4 * L + 4), 256);
  pl.maxrun = 1;
  for (int ph = 0; ph < 3; ++ph) {
    pl.n_sg[ph] = (N[ph] + stp::BM - 1) / stp::BM;
    pl.n_units[ph] = pl.n_sg[ph] * pl.KC;
    // logits: few units; runs of >= 4 tiles keep the strips' contributor counts (and their
    // final reduction) small
    pl.Gp[ph] = ph == stp::HEAD ? std::max(1, std::min(pl.G, pl.n_units[ph] / 4)) : std::min(pl.G, pl.n_units[ph]);
    int maxc = 1, maxrun = 1;
    for (int c = 0; c < pl.Gp[ph]; ++c) {
      const int r = (int)((int64_t)(c + 1) * pl.n_units[ph] / pl.Gp[ph]) - (int)((int64_t)c * pl.n_units[ph] / pl.Gp[ph]);
      maxrun = std::max(maxrun, r);
    }
    for (int sg = 0; sg < pl.n_sg[ph]; ++sg) {
      auto own = [&](int u) { return (int)(((int64_t)(u + 1) * pl.Gp[ph] - 1) / pl.n_units[ph]); };
      maxc = std::max(maxc, own(sg * pl.KC + pl.KC - 1) - own(sg * pl.KC) + 1);
    }
    pl.maxc[ph] = maxc;
    pl.maxrun = std::max(pl.maxrun, maxrun);
    pl.off_tk[ph] = off;
    off += align_up(sizeof(unsigned) * (size_t)pl.n_sg[ph] * (ph == stp::HEAD ? 1 : L), 256);
  }
  for (int ph = 0; ph < 3; ++ph) {
    pl.off_part[ph] = off;
    off += align_up(sizeof(float) * (size_t)pl.n_sg[ph] * pl.maxc[ph] * B * stp::BM, 256);
  }
  pl.maxs = pl.G + 1;
  pl.off_att = off;
  off += align_up(sizeof(float) * (size_t)B * hkv * pl.maxs * (2 * pl.Gq + pl.Gq * d), 256);
  pl.off_q = off;
  off += align_up(sizeof(float) * (size_t)B * D, 256);
  pl.off_attn = off;
  off += align_up(sizeof(float) * (size_t)B * D, 256);
  pl.off_logits = off;
  off += align_up(sizeof(float) * (size_t)B * pl.npad, 256);
  pl.total = off;
  pl.NT = B <= 8 ? 1 : 2;
  const int x_frag = pl.maxrun * 4 * pl.NT * 2 * 32 * 8;   // [unit][k16][n-tile][hi, lo][lane] uint2
  const int scratch_att = sizeof(float) * (2 * stp::kCW * stp::kMaxG + stp::kCW * pl.Gq * d);
  const int scratch_mrg = sizeof(float) * (2 * stp::kMaxG * pl.maxs + stp::kMaxG);
  pl.xs_bytes = (int)align_up((size_t)std::max(x_frag, std::max(scratch_att, scratch_mrg)), 1024);
  const int fixed = 1024 + pl.xs_bytes + stp::kMaxB * 64 * 8 + 2 * 64 * 8 + 6 * stp::kMaxB * 4 + 256;
  pl.NS = (stp::kSmemMax - fixed) / stp::kStage;
  if (pl.NS > 24) pl.NS = 24;
  pl.smem = (size_t)pl.NS * stp::kStage + fixed;
  return pl;
}

static int make_cache_map(CUtensorMap* map, const void* base, int hkv, int d, int64_t seq, int64_t blocks) {
  auto fn = tc::encode_fn();
  if (!fn) return fail(RK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)hkv, (cuuint64_t)seq, (cuuint64_t)blocks};
  cuuint64_t strides[3] = {(cuuint64_t)d * 2, (cuuint64_t)hkv * d * 2, (cuuint64_t)seq * hkv * d * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)stp::KEYS, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(RK_ERR_CUDA, "cuTensorMapEncodeTiled (cache) failed (%d)", (int)r);
  return RK_OK;
}

template <int NT>
static int launch_step(const stp::Params& p, const StepPlan& pl, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    if (const char* e = getenv("RK_STEP_PATIENCE_S")) {
      const long long cycles = (long long)(atof(e) * 2.0e9);
      if (cycles > 0) RK_CUDA(cudaMemcpyToSymbol(stp::g_patience, &cycles, sizeof(cycles)), "step patience");
    }
    RK_CUDA(cudaFuncSetAttribute(stp::step_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem),
            "step smem attribute");
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.G);
  cfg.blockDim = dim3(stp::kThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, stp::step_kernel<NT>, p);
  if (e != cudaSuccess) return cuda_status(e, "step_kernel launch");
  return RK_OK;
}

}  // namespace rk

using namespace rk;

extern "C" {

size_t rk_decode_step_workspace_bytes(int batch, int num_layers, int hq, int hkv, int head_dim, int vocab) {
  if (batch <= 0 || num_layers <= 0 || hkv <= 0 || hq % hkv != 0 || head_dim <= 0 || vocab <= 0) return 256;
  return step_plan(batch, num_layers, hq, hkv, head_dim, vocab).total;
}

int rk_decode_step_supported(int batch, int hq, int hkv, int head_dim, int kv_dtype) {
  if (!(batch >= 1 && batch <= stp::kMaxB && hkv > 0 && hq % hkv == 0 && hq / hkv <= stp::kMaxG &&
        head_dim == 128 && kv_dtype == RK_BF16))
    return 0;
  // every CTA must hold QKV projection units (each reads the launch epoch before contributing)
  const int64_t qkv_units = (int64_t)(hq + 2 * hkv) * head_dim / stp::BM * (hq * head_dim / stp::BK);
  return qkv_units >= sm_count();
}

int rk_decode_step(const rk_decode_step_args* a, rk_stream_t stream) {
  if (a == nullptr) return fail(RK_ERR_DOMAIN, "decode_step: null arguments");
  const int B = a->batch, L = a->num_layers, lw = a->watershed;
  if (!rk_decode_step_supported(B, a->hq, a->hkv, a->head_dim, RK_BF16))
    return fail(RK_ERR_DOMAIN,
                "decode_step: batch %d (1..%d), heads %d/%d (group <= %d), head_dim %d (128), QKV units >= SMs", B,
                stp::kMaxB, a->hq, a->hkv, stp::kMaxG, a->head_dim);
  if (L <= 0 || L > stp::kMaxL || lw < 0 || lw > L)
    return fail(RK_ERR_DOMAIN, "decode_step: layers %d (<= %d), watershed %d", L, stp::kMaxL, lw);
  if (a->vocab <= 0 || a->x == nullptr || a->rope_freq == nullptr || a->w_qkv == nullptr || a->w_o == nullptr ||
      a->emb_packed == nullptr || a->emb == nullptr || a->lower_len == nullptr || a->upper_len == nullptr ||
      a->pos == nullptr || (lw > 0 && a->lower == nullptr) || (lw < L && a->upper == nullptr))
    return fail(RK_ERR_DOMAIN, "decode_step: missing buffer");
  const StepPlan pl = step_plan(B, L, a->hq, a->hkv, a->head_dim, a->vocab);
  if (a->workspace == nullptr || a->workspace_bytes < pl.total)
    return fail(RK_ERR_CAPACITY, "decode_step workspace %zu < %zu bytes", a->workspace_bytes, pl.total);
  if (pl.NS < 4) return fail(RK_ERR_DOMAIN, "decode_step: shared memory leaves %d ring stages", pl.NS);
  if (pl.n_units[0] < pl.G)
    return fail(RK_ERR_DOMAIN, "decode_step: %d projection units < %d SMs", pl.n_units[0], pl.G);
  stp::Params p{};
  const int d = a->head_dim;
  if (lw > 0) {
    int r = make_cache_map(&p.map_lo, a->lower, a->hkv, d, a->lower_seq, (int64_t)B * lw * 2);
    if (r != RK_OK) return r;
  }
  if (lw < L) {
    int r = make_cache_map(&p.map_up, a->upper, a->hkv, d, a->upper_seq, (int64_t)B * (L - lw) * 2);
    if (r != RK_OK) return r;
  }
  uint8_t* ws = static_cast<uint8_t*>(a->workspace);
  p.B = B;
  p.L = L;
  p.lw = lw;
  p.hq = a->hq;
  p.hkv = a->hkv;
  p.d = d;
  p.D = a->hq * d;
  p.vocab = a->vocab;
  p.Gq = pl.Gq;
  p.NS = pl.NS;
  p.xs_bytes = pl.xs_bytes;
  p.s_lo = a->lower_seq;
  p.s_up = a->upper_seq;
  p.x = a->x;
  p.q = reinterpret_cast<float*>(ws + pl.off_q);
  p.attn = reinterpret_cast<float*>(ws + pl.off_attn);
  p.logits = reinterpret_cast<float*>(ws + pl.off_logits);
  p.npad = pl.npad;
  p.lower = static_cast<__nv_bfloat16*>(a->lower);
  p.upper = static_cast<__nv_bfloat16*>(a->upper);
  p.lower_len = a->lower_len;
  p.upper_len = a->upper_len;
  p.pos = a->pos;
  p.freq = a->rope_freq;
  p.w_qkv = a->w_qkv;
  p.w_o = a->w_o;
  p.emb_packed = a->emb_packed;
  p.emb = static_cast<const __nv_bfloat16*>(a->emb);
  p.tokens = a->tokens;
  p.tokens_log = a->tokens_log;
  p.log_stride = a->log_stride;
  for (int ph = 0; ph < 3; ++ph) {
    p.pj[ph].n_sg = pl.n_sg[ph];
    p.pj[ph].KC = pl.KC;
    p.pj[ph].n_units = pl.n_units[ph];
    p.pj[ph].Gp = pl.Gp[ph];
    p.pj[ph].maxc = pl.maxc[ph];
    p.pj[ph].part = reinterpret_cast<float*>(ws + pl.off_part[ph]);
    p.pj[ph].tickets = reinterpret_cast<unsigned*>(ws + pl.off_tk[ph]);
  }
  p.part_att = reinterpret_cast<float*>(ws + pl.off_att);
  p.maxs = pl.maxs;
  p.mrg_split = 1;
  while (pl.Gq * d / p.mrg_split > stp::kCW * 32) p.mrg_split *= 2;
  p.hdr = reinterpret_cast<unsigned*>(ws);
  p.cnt = reinterpret_cast<unsigned*>(ws + pl.off_cnt);
  p.scale_log2 = kLog2e / sqrtf((float)d);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return pl.NT == 1 ? launch_step<1>(p, pl, st) : launch_step<2>(p, pl, st);
}

#ifdef STP_TRACE
int rk_debug_step_trace(unsigned long long* out, int n) {   // n <= 160 * 64 * 10
  return cudaMemcpyFromSymbol(out, stp::g_stp_trace, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : -1;
}
#endif

int rk_decode_step_watchdog(const void* workspace, unsigned* code_out, rk_stream_t stream) {
  if (workspace == nullptr || code_out == nullptr) return fail(RK_ERR_DOMAIN, "decode_step_watchdog: null");
  RK_CUDA(cudaMemcpyAsync(code_out, static_cast<const unsigned*>(workspace) + 1, sizeof(unsigned),
                          cudaMemcpyDeviceToHost, reinterpret_cast<cudaStream_t>(stream)),
          "decode_step_watchdog copy");
  return RK_OK;
}

}  // extern "C"
