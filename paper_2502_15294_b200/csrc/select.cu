// normalize + select on the device (stats.py:97-115, selection.py:63-126) and
// Eq. 1 aggregation over a materialised capture matrix (stats.py:59-94).
//
// Bit-exactness: the reference thresholds depend on float64 values produced by
// NumPy reductions — raw.sum() (normalize), masses.mean() and masses.std()
// (adaptive).  For a contiguous 1-D float64 array NumPy sums pairwise: blocks
// of <= 128 elements with an 8-way unrolled accumulator, larger ranges split
// at n/2 rounded down to a multiple of 8.  pw_sum below evaluates exactly that
// tree with explicit round-to-nearest intrinsics (no FMA contraction), so the
// same raw values give the same masses and the same kept set.
#include "rk_common.cuh"

namespace rk {

template <typename F>
__device__ double pw_sum(const F& f, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, f(lo + i));
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(lo + i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_sum(f, lo, n2), pw_sum(f, lo + n2, n - n2));
}

constexpr int kSelMax = 16384;

// One distribution per block: normalize (pairwise sum), then the policy's kept
// positions (ascending) into kept[0, *n_kept).  raw may live in shared memory.
__device__ void select_core(const double* raw, int n, int normalize, int kind, double v, int k_top, double kappa,
                            double* __restrict__ masses, int32_t* __restrict__ kept, int32_t* __restrict__ n_kept,
                            int32_t* __restrict__ degenerate, int32_t* __restrict__ status,
                            unsigned char* __restrict__ flag) {
  __shared__ double s_total, s_cut;
  __shared__ int s_neg, s_any;
  const int t = threadIdx.x;
  if (t == 0) { s_neg = 0; s_any = 0; }
  __syncthreads();
  for (int i = t; i < n; i += blockDim.x)
    if (raw[i] < 0.0) s_neg = 1;
  __syncthreads();
  if (s_neg) {
    if (t == 0) { *status = RK_ERR_DOMAIN; *n_kept = 0; }
    __syncthreads();
    return;
  }
  if (t == 0) {
    s_total = normalize ? pw_sum([&](int i) { return raw[i]; }, 0, n) : 1.0;
    *status = RK_OK;
    *degenerate = (s_total > 0.0) ? 0 : 1;
  }
  __syncthreads();
  const double total = s_total;
  const bool ok = total > 0.0;
  for (int i = t; i < n; i += blockDim.x)
    masses[i] = !normalize ? raw[i] : ok ? __ddiv_rn(raw[i], total) : __ddiv_rn(1.0, (double)n);
  __syncthreads();
  if (kind == RK_SEL_ADAPTIVE && t == 0) {
    // _methods._mean / _var: pairwise sum, true divide, squared deviations
    double mean = __ddiv_rn(pw_sum([&](int i) { return masses[i]; }, 0, n), (double)n);
    double var = __ddiv_rn(pw_sum([&](int i) {
                             double dv = __dsub_rn(masses[i], mean);
                             return __dmul_rn(dv, dv);
                           }, 0, n), (double)n);
    s_cut = __dadd_rn(mean, __dmul_rn(kappa, __dsqrt_rn(var)));
  }
  __syncthreads();
  for (int i = t; i < n; i += blockDim.x) {
    const double mi = masses[i];
    bool f;
    if (kind == RK_SEL_ALL) {
      f = true;
    } else if (kind == RK_SEL_TOP_PERCENT) {
      // stable rank of -mass (np.argsort(-masses, kind="stable")): ties -> lower index
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const double mj = masses[j];
        rank += (mj > mi) || (mj == mi && j < i);
      }
      f = rank < k_top;
    } else if (kind == RK_SEL_FIXED) {
      f = mi > v;
    } else {
      f = mi > s_cut;
    }
    flag[i] = f;
    if (f) s_any = 1;
  }
  __syncthreads();
  if (t == 0) {
    int c = 0;
    if (!s_any && n > 0) {      // _argmax_fallback: first maximum (selection.py:71-73)
      int best = 0;
      for (int i = 1; i < n; ++i)
        if (masses[i] > masses[best]) best = i;
      kept[c++] = best;
    } else {
      for (int i = 0; i < n; ++i)
        if (flag[i]) kept[c++] = i;
    }
    *n_kept = c;
  }
  __syncthreads();
}

// one block per distribution (blockIdx.x = batch row, rows `ld` apart)
__global__ void select_kernel(const double* __restrict__ raw, int n, int ld, int normalize, int kind, double v,
                              int k_top, double kappa, double* __restrict__ masses, int32_t* __restrict__ kept,
                              int32_t* __restrict__ n_kept, int32_t* __restrict__ degenerate,
                              int32_t* __restrict__ status) {
  __shared__ unsigned char flag[kSelMax];
  const size_t o = (size_t)blockIdx.x * ld;
  select_core(raw + o, n, normalize, kind, v, k_top, kappa, masses + o, kept + o, n_kept + blockIdx.x,
              degenerate + blockIdx.x, status + blockIdx.x, flag);
}

// Decision margin of one selection (relative distance of the deciding masses
// from the decision threshold; +inf when nothing is decided by a comparison):
//   top_percent: (m_(K) - m_(K+1)) / m_(K), the K-th and (K+1)-th largest masses;
//   fixed:       min_i |m_i - v| / v;
//   adaptive:    min_i |m_i - cut| / |cut|, cut = mean + kappa * std;
//   all:         +inf.
// A kept set computed from masses accurate to a relative error e is the
// reference's kept set whenever margin > 2e (exact ties, margin 0, are decided
// by index on both sides when the masses tie exactly).
__device__ void margin_core(const double* __restrict__ masses, int n, int kind, double v, int k_top, double kappa,
                            double* __restrict__ margin) {
  __shared__ double red[256];
  __shared__ double s_cut, s_a, s_b;
  const int t = threadIdx.x;
  if (t == 0) {
    s_a = -1.0;
    s_b = -1.0;
    if (kind == RK_SEL_ADAPTIVE) {
      double mean = __ddiv_rn(pw_sum([&](int i) { return masses[i]; }, 0, n), (double)n);
      double var = __ddiv_rn(pw_sum([&](int i) {
                               double dv = __dsub_rn(masses[i], mean);
                               return __dmul_rn(dv, dv);
                             }, 0, n), (double)n);
      s_cut = __dadd_rn(mean, __dmul_rn(kappa, __dsqrt_rn(var)));
    } else {
      s_cut = v;
    }
  }
  __syncthreads();
  double best = INFINITY;
  if (kind == RK_SEL_TOP_PERCENT) {
    if (k_top > 0 && k_top < n) {
      for (int i = t; i < n; i += blockDim.x) {    // stable rank as select_kernel
        const double mi = masses[i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
          const double mj = masses[j];
          rank += (mj > mi) || (mj == mi && j < i);
        }
        if (rank == k_top - 1) s_a = mi;
        if (rank == k_top) s_b = mi;
      }
    }
  } else if (kind == RK_SEL_FIXED || kind == RK_SEL_ADAPTIVE) {
    const double cut = s_cut;
    const double den = fabs(cut) > 0.0 ? fabs(cut) : 1.0;
    for (int i = t; i < n; i += blockDim.x) best = fmin(best, fabs(masses[i] - cut) / den);
  }
  red[t] = best;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (t < o) red[t] = fmin(red[t], red[t + o]);
    __syncthreads();
  }
  if (t == 0) {
    double m = red[0];
    if (kind == RK_SEL_TOP_PERCENT && k_top > 0 && k_top < n)
      m = s_a > 0.0 ? (s_a - s_b) / s_a : 0.0;
    *margin = m;
  }
  __syncthreads();
}

__global__ void margin_kernel(const double* __restrict__ masses, int n, int ld, int kind, double v, int k_top,
                              double kappa, double* __restrict__ margin) {
  margin_core(masses + (size_t)blockIdx.x * ld, n, kind, v, k_top, kappa, margin + blockIdx.x);
}

constexpr int kSelActMax = 2048;   // static shared memory: flags + masses + ids

// Selection over each dialogue's ACTIVE rounds (the inactivity drop policy,
// selection.py:183-204 + pipeline.py:238-245): raw [batch][ld] holds one Eq. 1
// mass per round (inactive rounds included, as the scorer's row normalisation
// needs every key); the block compacts its active rounds in ascending order
// (the reference's active_rounds list), normalizes and selects over them
// exactly as select_kernel, and reports the kept ROUND IDS.  top_percent with
// k_top <= 0 takes k = min(n_b, max(min_rounds, ceil(fraction * n_b - 1e-9)))
// per dialogue (selection.py:87-97).  masses [batch][ld] at compacted positions;
// margin [batch] as margin_kernel (nullable).
__global__ void select_active_kernel(const double* __restrict__ raw, int n, int ld,
                                     const uint8_t* __restrict__ active, int normalize, int kind, double v, int k_top,
                                     double fraction, int min_rounds, double kappa, double* __restrict__ masses,
                                     int32_t* __restrict__ kept, int32_t* __restrict__ n_kept,
                                     int32_t* __restrict__ degenerate, int32_t* __restrict__ status,
                                     double* __restrict__ margin) {
  __shared__ unsigned char flag[kSelActMax];
  __shared__ double vals[kSelActMax];
  __shared__ int32_t ids[kSelActMax];
  __shared__ int s_n;
  const int b = blockIdx.x, t = threadIdx.x;
  const size_t o = (size_t)b * ld;
  if (t < 32) {                               // ordered compaction by warp ballots
    int base = 0;
    for (int i0 = 0; i0 < n; i0 += 32) {
      const int i = i0 + t;
      const bool a = i < n && (active == nullptr || active[o + i]);
      const unsigned m = __ballot_sync(0xffffffffu, a);
      if (a) {
        const int p = base + __popc(m & ((1u << t) - 1u));
        ids[p] = i;
        vals[p] = raw[o + i];
      }
      base += __popc(m);
    }
    if (t == 0) s_n = base;
  }
  __syncthreads();
  const int nb = s_n;
  int k = k_top;
  if (kind == RK_SEL_TOP_PERCENT && k_top <= 0) {
    k = max(min_rounds, (int)ceil(fraction * (double)nb - 1e-9));
    k = min(k, nb);
  }
  if (nb == 0) {                              // no history: the reference's empty result
    if (t == 0) {
      n_kept[b] = 0;
      degenerate[b] = 0;
      status[b] = RK_OK;
      if (margin) margin[b] = INFINITY;
    }
    return;
  }
  select_core(vals, nb, normalize, kind, v, k, kappa, masses + o, kept + o, n_kept + b, degenerate + b, status + b,
              flag);
  const int c = n_kept[b];
  for (int i = t; i < c; i += blockDim.x) kept[o + i] = ids[kept[o + i]];
  if (margin) margin_core(masses + o, nb, kind, v, k, kappa, margin + b);
}

__global__ void aggregate_kernel(const double* __restrict__ scores, int64_t ld, int row_lo, int row_hi,
                                 const int64_t* __restrict__ spans, double* __restrict__ raw) {
  __shared__ double red[256];
  const int a = blockIdx.x;
  const int64_t q0 = spans[a * 4 + 0], q1 = spans[a * 4 + 1], a0 = spans[a * 4 + 2], a1 = spans[a * 4 + 3];
  const int64_t wq = q1 - q0, wa = a1 - a0, w = wq + wa;
  const int64_t total = (int64_t)(row_hi - row_lo) * w;
  double acc = 0.0;
  for (int64_t idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int64_t r = idx / w, c = idx - r * w;
    int64_t col = c < wq ? q0 + c : a0 + (c - wq);
    acc += scores[(row_lo + r) * ld + col];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) raw[a] = red[0];
}

}  // namespace rk

using namespace rk;

extern "C" {

int rk_select(const double* raw, int n, int normalize, int kind, double v, int k_top, double kappa, double* masses_out,
              int32_t* kept_out, int32_t* n_kept_out, int32_t* degenerate_out, int32_t* status_out,
              rk_stream_t stream) {
  if (n < 0 || n > kSelMax) return fail(RK_ERR_DOMAIN, "selection over %d rounds (max %d)", n, kSelMax);
  if (kind < RK_SEL_FIXED || kind > RK_SEL_ALL) return fail(RK_ERR_DOMAIN, "selection kind %d unknown", kind);
  select_kernel<<<1, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      raw, n, n, normalize, kind, v, k_top, kappa, masses_out, kept_out, n_kept_out, degenerate_out, status_out);
  RK_CHECK_LAUNCH("select_kernel");
  return RK_OK;
}

int rk_select_batch(const double* raw, int n, int ld, int batch, int normalize, int kind, double v, int k_top,
                    double kappa, double* masses_out, int32_t* kept_out, int32_t* n_kept_out,
                    int32_t* degenerate_out, int32_t* status_out, rk_stream_t stream) {
  if (n < 0 || n > kSelMax || ld < n) return fail(RK_ERR_DOMAIN, "selection over %d rounds (max %d)", n, kSelMax);
  if (kind < RK_SEL_FIXED || kind > RK_SEL_ALL) return fail(RK_ERR_DOMAIN, "selection kind %d unknown", kind);
  if (batch <= 0) return RK_OK;
  select_kernel<<<batch, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      raw, n, ld, normalize, kind, v, k_top, kappa, masses_out, kept_out, n_kept_out, degenerate_out, status_out);
  RK_CHECK_LAUNCH("select_kernel");
  return RK_OK;
}

int rk_select_batch_active(const double* raw, int n, int ld, int batch, const uint8_t* active, int normalize,
                           int kind, double v, int k_top, double fraction, int min_rounds, double kappa,
                           double* masses_out, int32_t* kept_out, int32_t* n_kept_out, int32_t* degenerate_out,
                           int32_t* status_out, double* margin_out, rk_stream_t stream) {
  if (n < 0 || n > kSelActMax || ld < n)
    return fail(RK_ERR_DOMAIN, "active selection over %d rounds (max %d)", n, kSelActMax);
  if (kind < RK_SEL_FIXED || kind > RK_SEL_ALL) return fail(RK_ERR_DOMAIN, "selection kind %d unknown", kind);
  if (kind == RK_SEL_TOP_PERCENT && k_top <= 0 && (!(fraction > 0.0 && fraction <= 1.0) || min_rounds < 1))
    return fail(RK_ERR_DOMAIN, "top_percent needs k_top > 0 or fraction in (0, 1] and min_rounds >= 1");
  if (batch <= 0) return RK_OK;
  select_active_kernel<<<batch, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      raw, n, ld, active, normalize, kind, v, k_top, fraction, min_rounds, kappa, masses_out, kept_out, n_kept_out,
      degenerate_out, status_out, margin_out);
  RK_CHECK_LAUNCH("select_active_kernel");
  return RK_OK;
}

int rk_selection_margin(const double* masses, int n, int ld, int batch, int kind, double v, int k_top,
                        double kappa, double* margin_out, rk_stream_t stream) {
  if (n < 0 || n > kSelMax || ld < n) return fail(RK_ERR_DOMAIN, "selection over %d rounds (max %d)", n, kSelMax);
  if (kind < RK_SEL_FIXED || kind > RK_SEL_ALL) return fail(RK_ERR_DOMAIN, "selection kind %d unknown", kind);
  if (batch <= 0) return RK_OK;
  margin_kernel<<<batch, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(masses, n, ld, kind, v, k_top, kappa,
                                                                           margin_out);
  RK_CHECK_LAUNCH("margin_kernel");
  return RK_OK;
}

int rk_aggregate_rounds(const double* scores, int64_t ld, int row_lo, int row_hi, const int64_t* spans,
                        int n_active, double* raw_out, rk_stream_t stream) {
  if (n_active <= 0) return RK_OK;
  if (row_hi < row_lo) return fail(RK_ERR_DOMAIN, "row range reversed");
  aggregate_kernel<<<n_active, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(scores, ld, row_lo, row_hi,
                                                                                  spans, raw_out);
  RK_CHECK_LAUNCH("aggregate_kernel");
  return RK_OK;
}

}  // extern "C"
