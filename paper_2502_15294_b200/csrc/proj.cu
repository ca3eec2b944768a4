// The decode step's layer body on the GPU (engine.py:244-251,267-271 of the
// reference: q,k = RoPE(x W_q), RoPE(x W_k); v = x W_v; append; attention;
// x += out W_o; logits = x E^T; argmax) for B dialogues at once.
//
// Every projection is a skinny GEMM (m = B tokens <= 32 per pass, K = 4096,
// N = 6144 / 4096): the weights are read once per token step, so the kernels
// are bound by HBM on the weight bytes (Llama-3-8B-shaped: 84 MB per layer).
//
// Layout: weights are packed once (rk_pack_weight) into mma.m16n8k16 A-fragment
// order — one 16 (output features) x 16 (inputs) tile = 512 contiguous bytes,
// lane L's 8 bf16 at 16 L, so a warp fetches a whole A operand with one
// coalesced 16-byte load per lane and no shared-memory staging.  The tiles of
// one 16-row output strip are consecutive along K.
//
// Kernel: a CTA of 8 warps owns RT = 2 output strips (32 features); the 8
// warps are RT strips x KS = 4 K-quarters.  Each warp streams its weights with
// 8 tiles (4 KB) in flight, converts the fp32 activations of its K range into
// bf16 hi + lo fragments on the fly (x = hi + lo keeps ~16 mantissa bits, the
// reference's projections are fp32 BLAS) and issues 2 MMAs per (tile, 8-token
// block).  The K-quarter partials meet in shared memory and are added in a
// fixed order (deterministic), then the fused epilogue runs:
//   qkv : RoPE on q and k (interleaved pairs, fp64 angles from the host-computed
//         reference frequency table, engine.py:162-164,175-185), q -> fp32,
//         k, v -> bf16 rows for the cache append;
//   out : x += attention_out W_o (the residual, engine.py:267);
//   head: logits (engine.py:270-271), then rk_argmax_embed picks the first
//         maximum (pipeline.py:308, np.argmax) and looks up the next input.
#include "decode_common.cuh"
#include "rk_common.cuh"

namespace rk {

constexpr int kPjWarps = 8;
constexpr int kPjRT = 2;                  // output strips (16 features) per CTA
constexpr int kPjKS = kPjWarps / kPjRT;   // K splits per strip
constexpr int kPjU = 8;                   // weight tiles in flight per warp
constexpr int kPjMaxNT = 4;               // 8-token blocks per pass (32 tokens)

enum { PJ_QKV = 0, PJ_OUT = 1, PJ_HEAD = 2 };

struct ProjParams {
  const float* x;          // [m][K] fp32 input rows
  int m, K, N;
  const uint4* w;          // packed [N/16][K/16][32 lanes] x 16 B
  int mode;
  // qkv
  int hq, hkv, d;
  const int32_t* pos;      // [m] absolute positions
  const double* freq;      // [d/2] RoPE frequencies (host: theta ** (-2i/d))
  float* q_out;            // [m][hq*d]
  __nv_bfloat16* k_out;    // row j at k_out + j * kv_stride
  __nv_bfloat16* v_out;
  int64_t kv_stride;
  // out
  float* resid;            // [m][N] += result
  // head
  float* logits;           // [m][N]
};

__device__ __forceinline__ void split_bf16(float2 p, uint32_t& hi, uint32_t& lo) {
  hi = pack_bf16(p.x, p.y);
  const float2 h = bf16x2_to_f2(hi);
  lo = pack_bf16(p.x - h.x, p.y - h.y);
}

template <int NT>
__global__ void __launch_bounds__(kPjWarps * 32, 2) proj_kernel(ProjParams p) {
  __shared__ float red[kPjWarps][NT][32][4];
  __shared__ float tile[kPjRT * 16][NT * 8 + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int strip = blockIdx.x * kPjRT + (warp % kPjRT);
  const int ks = warp / kPjRT;
  const int KT = p.K / 16;
  const int n_strips = p.N / 16;
  const int kt0 = ks * KT / kPjKS, kt1 = (ks + 1) * KT / kPjKS;
  const bool active = strip < n_strips;
  const uint4* wp = p.w + ((size_t)(active ? strip : 0) * KT) * 32 + lane;
  // the weights do not depend on the previous kernel: the first batch is in
  // flight before griddepcontrol.wait (programmatic dependent launch)
  uint4 nxt[kPjU];
#pragma unroll
  for (int u = 0; u < kPjU; ++u)
    if (active && kt0 + u < kt1) nxt[u] = ld_stream(wp + (size_t)(kt0 + u) * 32);
  pdl_wait();                              // the activations of the previous kernel are complete
  for (int m0 = 0; m0 < p.m; m0 += NT * 8) {
    float acc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[nt][i] = 0.f;
    if (active) {
      const float* xr[NT];
      bool tok_ok[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int tok = m0 + nt * 8 + g;
        tok_ok[nt] = tok < p.m;
        xr[nt] = p.x + (size_t)(tok_ok[nt] ? tok : 0) * p.K + 2 * t;
      }
      if (m0 > 0) {                        // later passes (multi-row prefill): reload the first batch
#pragma unroll
        for (int u = 0; u < kPjU; ++u)
          if (kt0 + u < kt1) nxt[u] = ld_stream(wp + (size_t)(kt0 + u) * 32);
      }
      for (int kt = kt0; kt < kt1; kt += kPjU) {
        uint4 a[kPjU];
#pragma unroll
        for (int u = 0; u < kPjU; ++u) a[u] = nxt[u];
#pragma unroll
        for (int u = 0; u < kPjU; ++u)     // next batch in flight while this one computes
          if (kt + kPjU + u < kt1) nxt[u] = ld_stream(wp + (size_t)(kt + kPjU + u) * 32);
#pragma unroll
        for (int u = 0; u < kPjU; ++u) {
          if (kt + u >= kt1) break;
          const uint32_t af[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            float2 x0 = make_float2(0.f, 0.f), x1 = make_float2(0.f, 0.f);
            if (tok_ok[nt]) {
              const float* xp = xr[nt] + (kt + u) * 16;
              x0 = *reinterpret_cast<const float2*>(xp);
              x1 = *reinterpret_cast<const float2*>(xp + 8);
            }
            uint32_t h0, l0, h1, l1;
            split_bf16(x0, h0, l0);
            split_bf16(x1, h1, l1);
            mma_bf16_16816(acc[nt], af, h0, h1);
            mma_bf16_16816(acc[nt], af, l0, l1);
          }
        }
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) red[warp][nt][lane][i] = acc[nt][i];
    __syncthreads();
    if (warp < kPjRT) {                    // K-quarters in a fixed order
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        float s[4] = {0.f, 0.f, 0.f, 0.f};
        for (int q = 0; q < kPjKS; ++q)
#pragma unroll
          for (int i = 0; i < 4; ++i) s[i] += red[q * kPjRT + warp][nt][lane][i];
        // C fragment: c0,c1 = (row g, tokens 2t, 2t+1); c2,c3 = (row g + 8, ...)
        const int r = warp * 16 + g, c = nt * 8 + 2 * t;
        tile[r][c] = s[0];
        tile[r][c + 1] = s[1];
        tile[r + 8][c] = s[2];
        tile[r + 8][c + 1] = s[3];
      }
    }
    __syncthreads();
    // ---- fused epilogue over this CTA's 32 features x the pass's tokens
    const int n0 = blockIdx.x * kPjRT * 16;
    const int mt = min(NT * 8, p.m - m0);
    if (p.mode == PJ_QKV) {
      const int qd = p.hq * p.d, kd = p.hkv * p.d;
      for (int e = threadIdx.x; e < kPjRT * 8 * mt; e += blockDim.x) {
        const int pr = e / mt, j = e - pr * mt;          // feature pair (2pr, 2pr+1), token j
        const int n = n0 + 2 * pr;
        if (n >= p.N) continue;
        const int tok = m0 + j;
        const float x0 = tile[2 * pr][j], x1 = tile[2 * pr + 1][j];
        if (n < qd + kd) {
          const int i = (n % p.d) >> 1;
          const double ang = (double)p.pos[tok] * p.freq[i];
          double sn, cs;
          sincos(ang, &sn, &cs);
          const float y0 = (float)((double)x0 * cs - (double)x1 * sn);
          const float y1 = (float)((double)x0 * sn + (double)x1 * cs);
          if (n < qd) {
            float* qo = p.q_out + (size_t)tok * qd + n;
            qo[0] = y0;
            qo[1] = y1;
          } else {
            __nv_bfloat16* ko = p.k_out + (size_t)tok * p.kv_stride + (n - qd);
            *reinterpret_cast<uint32_t*>(ko) = pack_bf16(y0, y1);
          }
        } else {
          __nv_bfloat16* vo = p.v_out + (size_t)tok * p.kv_stride + (n - qd - kd);
          *reinterpret_cast<uint32_t*>(vo) = pack_bf16(x0, x1);
        }
      }
    } else {
      for (int e = threadIdx.x; e < kPjRT * 16 * mt; e += blockDim.x) {
        const int r = e / mt, j = e - r * mt;
        const int n = n0 + r;
        if (n >= p.N) continue;
        const int tok = m0 + j;
        if (p.mode == PJ_OUT)
          p.resid[(size_t)tok * p.N + n] += tile[r][j];
        else
          p.logits[(size_t)tok * p.N + n] = tile[r][j];
      }
    }
    __syncthreads();
  }
  pdl_trigger();
}

// tokens[b] = first argmax of logits[b][0:V) (np.argmax); x[b] = emb[token];
// pos[b] += 1 when given; tokens_log[b * log_stride] = token when given
__global__ void argmax_embed_kernel(const float* __restrict__ logits, int ld, int V,
                                    const __nv_bfloat16* __restrict__ emb, int D, float* __restrict__ x,
                                    int32_t* __restrict__ tokens, int32_t* __restrict__ pos,
                                    int32_t* __restrict__ tokens_log, int log_stride) {
  pdl_wait();
  __shared__ float sv[256];
  __shared__ int si[256];
  const int b = blockIdx.x;
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
    if (tokens_log) tokens_log[(size_t)b * log_stride] = tok;
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

// packed[strip][kt][lane] <- W[k][n] (row-major [K][N], x @ W), fp32 or bf16 source
template <typename T>
__global__ void pack_weight_kernel(const T* __restrict__ w, int K, int N, int n_valid, __nv_bfloat16* __restrict__ out) {
  const size_t tiles = (size_t)(N / 16) * (K / 16);
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;   // one (tile, lane)
  if (idx >= tiles * 32) return;
  const int lane = idx & 31;
  const size_t tl = idx >> 5;
  const int KT = K / 16;
  const int strip = (int)(tl / KT), kt = (int)(tl % KT);
  const int g = lane >> 2, t = lane & 3;
  const int rows[8] = {g, g, g + 8, g + 8, g, g, g + 8, g + 8};
  const int cols[8] = {2 * t, 2 * t + 1, 2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9, 2 * t + 8, 2 * t + 9};
  __nv_bfloat16* o = out + idx * 8;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int n = strip * 16 + rows[e], k = kt * 16 + cols[e];
    const float v = n < n_valid ? (float)w[(size_t)k * n_valid + n] : 0.f;
    o[e] = __float2bfloat16_rn(v);
  }
}

static int launch_proj(const ProjParams& p, cudaStream_t st) {
  if (p.m <= 0) return RK_OK;
  if (p.K % (16 * kPjKS) != 0 || p.N % 16 != 0)
    return fail(RK_ERR_DOMAIN, "projection K=%d (multiple of %d), N=%d (multiple of 16)", p.K, 16 * kPjKS, p.N);
  const int grid = (p.N / 16 + kPjRT - 1) / kPjRT;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kPjWarps * 32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  const int nt = (p.m + 7) / 8;
  if (nt <= 1)
    e = cudaLaunchKernelEx(&cfg, proj_kernel<1>, p);
  else if (nt <= 2)
    e = cudaLaunchKernelEx(&cfg, proj_kernel<2>, p);
  else
    e = cudaLaunchKernelEx(&cfg, proj_kernel<4>, p);
  if (e != cudaSuccess) return cuda_status(e, "proj_kernel launch");
  return RK_OK;
}

}  // namespace rk

using namespace rk;

extern "C" {

size_t rk_packed_weight_bytes(int k, int n) {
  return (size_t)((n + 15) / 16 * 16) * (size_t)k * sizeof(__nv_bfloat16);
}

int rk_pack_weight(const void* w, int w_dtype, int k, int n, void* packed, rk_stream_t stream) {
  if (k <= 0 || n <= 0 || k % 16 != 0) return fail(RK_ERR_DOMAIN, "pack_weight k=%d (multiple of 16), n=%d", k, n);
  const int np = (n + 15) / 16 * 16;
  const size_t threads = (size_t)(np / 16) * (k / 16) * 32;
  const int blocks = (int)((threads + 255) / 256);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (w_dtype == RK_F32)
    pack_weight_kernel<float><<<blocks, 256, 0, st>>>((const float*)w, k, np, n, (__nv_bfloat16*)packed);
  else if (w_dtype == RK_BF16)
    pack_weight_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)w, k, np, n,
                                                              (__nv_bfloat16*)packed);
  else
    return fail(RK_ERR_DOMAIN, "weight dtype %d", w_dtype);
  RK_CHECK_LAUNCH("pack_weight_kernel");
  return RK_OK;
}

int rk_qkv_rope(const float* x, int m, int d_model, const void* w_qkv_packed, int hq, int hkv, int d,
                const int32_t* pos, const double* rope_freq, float* q_out, void* k_out, void* v_out,
                int64_t kv_row_stride, rk_stream_t stream) {
  if (hkv <= 0 || hq % hkv != 0 || d % 2 != 0) return fail(RK_ERR_DOMAIN, "qkv heads %d/%d, d %d", hq, hkv, d);
  ProjParams p{};
  p.x = x;
  p.m = m;
  p.K = d_model;
  p.N = (hq + 2 * hkv) * d;
  p.w = reinterpret_cast<const uint4*>(w_qkv_packed);
  p.mode = PJ_QKV;
  p.hq = hq;
  p.hkv = hkv;
  p.d = d;
  p.pos = pos;
  p.freq = rope_freq;
  p.q_out = q_out;
  p.k_out = reinterpret_cast<__nv_bfloat16*>(k_out);
  p.v_out = reinterpret_cast<__nv_bfloat16*>(v_out);
  p.kv_stride = kv_row_stride;
  if (p.N % 32 != 0) return fail(RK_ERR_DOMAIN, "qkv width %d (multiple of 32)", p.N);
  return launch_proj(p, reinterpret_cast<cudaStream_t>(stream));
}

int rk_out_proj(const float* a, int m, int k, const void* w_o_packed, int d_model, float* resid,
                rk_stream_t stream) {
  ProjParams p{};
  p.x = a;
  p.m = m;
  p.K = k;
  p.N = d_model;
  p.w = reinterpret_cast<const uint4*>(w_o_packed);
  p.mode = PJ_OUT;
  p.resid = resid;
  return launch_proj(p, reinterpret_cast<cudaStream_t>(stream));
}

size_t rk_lm_head_workspace_bytes(int m, int vocab) {
  return sizeof(float) * (size_t)m * ((vocab + 15) / 16 * 16);
}

int rk_lm_head(const float* x, int m, int d_model, const void* emb_packed, int vocab, const void* emb,
               float* x_next, int32_t* tokens, int32_t* pos, int32_t* tokens_log, int log_stride,
               void* workspace, size_t workspace_bytes, rk_stream_t stream) {
  if (m <= 0) return RK_OK;
  const int vp = (vocab + 15) / 16 * 16;
  if (workspace_bytes < rk_lm_head_workspace_bytes(m, vocab))
    return fail(RK_ERR_CAPACITY, "lm_head workspace %zu", workspace_bytes);
  ProjParams p{};
  p.x = x;
  p.m = m;
  p.K = d_model;
  p.N = vp;
  p.w = reinterpret_cast<const uint4*>(emb_packed);
  p.mode = PJ_HEAD;
  p.logits = reinterpret_cast<float*>(workspace);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc = launch_proj(p, st);
  if (rc != RK_OK) return rc;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(m);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, argmax_embed_kernel, (const float*)p.logits, vp, vocab,
                                     (const __nv_bfloat16*)emb, d_model, x_next, tokens, pos, tokens_log,
                                     log_stride);
  if (e != cudaSuccess) return cuda_status(e, "argmax_embed_kernel launch");
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

}  // extern "C"
