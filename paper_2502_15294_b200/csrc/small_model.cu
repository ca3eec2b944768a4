// The layer body of the reference-compatible drop-in model (engine.Model: the
// reference's toy transformer with float32 weights, default d_model 32), on the
// GPU in float32 — the reference computes these products with float32 BLAS:
//   rk_small_qkv_rope     q, k = RoPE(x W_q), RoPE(x W_k); v = x W_v
//                         (engine.py:244-251; RoPE in float64, engine.py:175-185)
//   rk_small_out_proj     x_out = x + a W_o                 (engine.py:267)
//   rk_small_logits       logits = x E^T, first-max argmax  (engine.py:270-271, pipeline.py:308)
//   rk_capture_pre        the capture_mode="pre" score matrix (engine.py:187-200), float64
// These shapes are tiny (the batched engine's tcgen05 projections, proj.cu,
// serve the large bf16 models): one CTA per (row, column block), the row of x
// in shared memory, one output column per thread, coalesced weight reads
// (consecutive threads read consecutive columns of the row-major weight).
#include "rk_common.cuh"

namespace rk {
namespace sm {

constexpr int kThreads = 256;
constexpr int kMaxDm = 4096;

// out[col] = sum_k x[k] W[k][col] (four interleaved partial sums, then added)
__device__ __forceinline__ float dot_col(const float* xs, const float* __restrict__ w, int dm, int ld, int col) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  int k = 0;
  for (; k + 4 <= dm; k += 4) {
    a0 = fmaf(xs[k], w[(size_t)k * ld + col], a0);
    a1 = fmaf(xs[k + 1], w[(size_t)(k + 1) * ld + col], a1);
    a2 = fmaf(xs[k + 2], w[(size_t)(k + 2) * ld + col], a2);
    a3 = fmaf(xs[k + 3], w[(size_t)(k + 3) * ld + col], a3);
  }
  for (; k < dm; ++k) a0 = fmaf(xs[k], w[(size_t)k * ld + col], a0);
  return (a0 + a1) + (a2 + a3);
}

// grid (n, ceil(dm / 256), 3): z = 0 q, 1 k, 2 v; RoPE pairs are within one
// column block when 256 % d_k == 0 — else each thread recomputes its partner
__global__ void __launch_bounds__(kThreads) small_qkv_rope_kernel(
    const float* __restrict__ x, int dm, const float* __restrict__ wq, const float* __restrict__ wk,
    const float* __restrict__ wv, int dk, const int64_t* __restrict__ pos, const double* __restrict__ freq,
    float* __restrict__ q_out, float* __restrict__ k_out, float* __restrict__ v_out) {
  __shared__ float xs[kMaxDm];
  const int row = blockIdx.x, which = blockIdx.z, col = blockIdx.y * kThreads + threadIdx.x;
  for (int k = threadIdx.x; k < dm; k += kThreads) xs[k] = x[(size_t)row * dm + k];
  __syncthreads();
  if (col >= dm) return;
  const float* w = which == 0 ? wq : which == 1 ? wk : wv;
  const float y = dot_col(xs, w, dm, dm, col);
  float* out = which == 0 ? q_out : which == 1 ? k_out : v_out;
  if (which == 2) {
    out[(size_t)row * dm + col] = y;
    return;
  }
  const float other = dot_col(xs, w, dm, dm, col ^ 1);     // the rotation partner (same head: d_k even)
  const int i = (col % dk) >> 1;
  const double ang = (double)pos[row] * freq[i];
  const double cs = cos(ang), sn = sin(ang);
  const bool even = (col & 1) == 0;
  const double ev = even ? (double)y : (double)other, od = even ? (double)other : (double)y;
  out[(size_t)row * dm + col] = even ? (float)(ev * cs - od * sn) : (float)(ev * sn + od * cs);
}

__global__ void __launch_bounds__(kThreads) small_out_proj_kernel(const float* __restrict__ a, int dm,
                                                                  const float* __restrict__ wo,
                                                                  const float* __restrict__ x,
                                                                  float* __restrict__ x_out) {
  __shared__ float as[kMaxDm];
  const int row = blockIdx.x, col = blockIdx.y * kThreads + threadIdx.x;
  for (int k = threadIdx.x; k < dm; k += kThreads) as[k] = a[(size_t)row * dm + k];
  __syncthreads();
  if (col >= dm) return;
  x_out[(size_t)row * dm + col] = x[(size_t)row * dm + col] + dot_col(as, wo, dm, dm, col);
}

// one CTA per row: logits[v] = sum_k x[k] E[v][k], then the first maximum
__global__ void __launch_bounds__(kThreads) small_logits_kernel(const float* __restrict__ x, int dm,
                                                                const float* __restrict__ emb, int vocab,
                                                                float* __restrict__ logits,
                                                                int32_t* __restrict__ argmax) {
  __shared__ float xs[kMaxDm];
  __shared__ float bv[kThreads / 32];
  __shared__ int bi[kThreads / 32];
  const int row = blockIdx.x;
  for (int k = threadIdx.x; k < dm; k += kThreads) xs[k] = x[(size_t)row * dm + k];
  __syncthreads();
  float best = -INFINITY;
  int besti = 0x7fffffff;
  for (int v = threadIdx.x; v < vocab; v += kThreads) {
    const float* e = emb + (size_t)v * dm;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    int k = 0;
    for (; k + 4 <= dm; k += 4) {
      a0 = fmaf(xs[k], e[k], a0);
      a1 = fmaf(xs[k + 1], e[k + 1], a1);
      a2 = fmaf(xs[k + 2], e[k + 2], a2);
      a3 = fmaf(xs[k + 3], e[k + 3], a3);
    }
    for (; k < dm; ++k) a0 = fmaf(xs[k], e[k], a0);
    const float z = (a0 + a1) + (a2 + a3);
    if (logits) logits[(size_t)row * vocab + v] = z;
    if (z > best) { best = z; besti = v; }        // ascending v per thread: the first maximum
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float z = __shfl_xor_sync(0xffffffffu, best, o);
    const int i = __shfl_xor_sync(0xffffffffu, besti, o);
    if (z > best || (z == best && i < besti)) { best = z; besti = i; }
  }
  if (lane == 0) {
    bv[warp] = best;
    bi[warp] = besti;
  }
  __syncthreads();
  if (threadIdx.x == 0 && argmax) {
    for (int w = 1; w < kThreads / 32; ++w)
      if (bv[w] > best || (bv[w] == best && bi[w] < besti)) { best = bv[w]; besti = bi[w]; }
    // NaN rows: no comparison succeeds; report index 0 like np.argmax over an all-NaN row
    argmax[row] = besti == 0x7fffffff ? 0 : besti;
  }
}

// capture_mode="pre" (engine.py:187-200): one float64 softmax per query row over
// the head-summed logits sum_h q_h . k_h / (H sqrt(d_k)) of the visible keys
// (k_pos <= q_pos, allowed); products of the float32 inputs are exact in float64.
// Row with no visible key: NaN (the reference's -inf - -inf).
__global__ void __launch_bounds__(kThreads) capture_pre_kernel(
    const float* __restrict__ q, int hd, const float* __restrict__ k, int s, const int64_t* __restrict__ q_pos,
    const int64_t* __restrict__ k_pos, const uint8_t* __restrict__ allowed, double denom, double* __restrict__ out) {
  extern __shared__ double qs[];
  __shared__ double red[kThreads / 32];
  const int row = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < hd; e += kThreads) qs[e] = (double)q[(size_t)row * hd + e];
  __syncthreads();
  const int64_t qp = q_pos[row];
  double* o = out + (size_t)row * s;
  double m = -INFINITY;
  for (int j = threadIdx.x; j < s; j += kThreads) {
    double v = -INFINITY;
    if (k_pos[j] <= qp && (allowed == nullptr || allowed[j])) {
      const float* kr = k + (size_t)j * hd;
      double acc = 0.0;
      for (int e = 0; e < hd; ++e) acc = fma(qs[e], (double)kr[e], acc);
      v = acc / denom;
    }
    o[j] = v;
    m = fmax(m, v);
  }
  auto block_reduce = [&](double v, bool is_max) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, v, off);
      v = is_max ? fmax(v, w) : v + w;
    }
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double r = red[0];
    for (int w = 1; w < kThreads / 32; ++w) r = is_max ? fmax(r, red[w]) : r + red[w];
    return r;
  };
  const double M = block_reduce(m, true);
  double sum = 0.0;
  for (int j = threadIdx.x; j < s; j += kThreads) {
    const double e = M == -INFINITY ? NAN : exp(o[j] - M);
    o[j] = e;
    sum += e;
  }
  const double S = block_reduce(sum, false);
  for (int j = threadIdx.x; j < s; j += kThreads) o[j] = o[j] / S;
}

}  // namespace sm
}  // namespace rk

using namespace rk;

extern "C" {

int rk_small_qkv_rope(const float* x, int n, int d_model, const float* w_q, const float* w_k, const float* w_v,
                      int heads, const int64_t* pos, const double* rope_freq, float* q_out, float* k_out,
                      float* v_out, rk_stream_t stream) {
  if (n <= 0) return RK_OK;
  if (d_model <= 0 || d_model > sm::kMaxDm || heads <= 0 || d_model % heads || (d_model / heads) % 2)
    return fail(RK_ERR_DOMAIN, "small_qkv_rope: d_model %d (<= %d), heads %d (even d_k)", d_model, sm::kMaxDm, heads);
  dim3 grid(n, (d_model + sm::kThreads - 1) / sm::kThreads, 3);
  sm::small_qkv_rope_kernel<<<grid, sm::kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      x, d_model, w_q, w_k, w_v, d_model / heads, pos, rope_freq, q_out, k_out, v_out);
  RK_CHECK_LAUNCH("small_qkv_rope_kernel");
  return RK_OK;
}

int rk_small_out_proj(const float* a, int n, int d_model, const float* w_o, const float* x, float* x_out,
                      rk_stream_t stream) {
  if (n <= 0) return RK_OK;
  if (d_model <= 0 || d_model > sm::kMaxDm) return fail(RK_ERR_DOMAIN, "small_out_proj: d_model %d", d_model);
  dim3 grid(n, (d_model + sm::kThreads - 1) / sm::kThreads);
  sm::small_out_proj_kernel<<<grid, sm::kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a, d_model, w_o, x,
                                                                                               x_out);
  RK_CHECK_LAUNCH("small_out_proj_kernel");
  return RK_OK;
}

int rk_small_logits(const float* x, int n, int d_model, const float* emb, int vocab, float* logits,
                    int32_t* argmax, rk_stream_t stream) {
  if (n <= 0) return RK_OK;
  if (d_model <= 0 || d_model > sm::kMaxDm || vocab <= 0)
    return fail(RK_ERR_DOMAIN, "small_logits: d_model %d, vocab %d", d_model, vocab);
  sm::small_logits_kernel<<<n, sm::kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, d_model, emb, vocab,
                                                                                         logits, argmax);
  RK_CHECK_LAUNCH("small_logits_kernel");
  return RK_OK;
}

int rk_capture_pre(const float* q, int n, int heads, int d_k, const float* k, int s, const int64_t* q_pos,
                   const int64_t* k_pos, const uint8_t* allowed, double* out, rk_stream_t stream) {
  if (n <= 0 || s <= 0) return RK_OK;
  const int hd = heads * d_k;
  if (heads <= 0 || d_k <= 0 || hd > 6144) return fail(RK_ERR_DOMAIN, "capture_pre: heads %d x d_k %d", heads, d_k);
  const double denom = (double)heads * sqrt((double)d_k);
  sm::capture_pre_kernel<<<n, sm::kThreads, sizeof(double) * hd, reinterpret_cast<cudaStream_t>(stream)>>>(
      q, hd, k, s, q_pos, k_pos, allowed, denom, out);
  RK_CHECK_LAUNCH("capture_pre_kernel");
  return RK_OK;
}

}  // extern "C"
