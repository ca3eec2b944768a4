// Host entry points for the attention family: kernel contract, decode, round
// scoring.  See include/roundkv_b200.h for the ABI and attn_split.cuh for the
// main kernel.
#include <climits>
#include <cmath>

#include "attn_dispatch.cuh"
#include "decode_bulk.cuh"
#include "prefill_tc.cuh"
#include <cstdlib>



namespace rk {

// ---------------------------------------------------------------- config
static int check_heads(int hq, int hkv, int d, Shape* s) {
  if (hq <= 0 || hkv <= 0 || hq % hkv != 0)
    return fail(RK_ERR_DOMAIN, "query heads %d not a multiple of key heads %d", hq, hkv);
  if (d <= 0) return fail(RK_ERR_DOMAIN, "head_dim must be positive");
  if (!pick_shape(d, hq / hkv, s)) return fail(RK_ERR_UNSUPPORTED, "head_dim %d not supported", d);
  return RK_OK;
}

static int dispatch_split(int kv_dtype, bool decode, bool score, int G, const Shape& s, dim3 grid,
                          cudaStream_t st, const SplitParams& p) {
  int r;
  if (kv_dtype == RK_F32) r = dispatch_f32(decode, score, G, s, grid, st, p);
  else if (kv_dtype == RK_BF16) r = dispatch_bf16(decode, score, G, s, grid, st, p);
  else return fail(RK_ERR_DOMAIN, "kv_dtype %d unknown", kv_dtype);
  if (r == 1) return fail(RK_ERR_UNSUPPORTED, "GQA group %d not supported (1, 2, 4, 7, 8)", G);
  if (r == 2) return cuda_status(cudaGetLastError(), "attn_split_kernel launch");
  return RK_OK;
}

// workspace carving ----------------------------------------------------------
struct SplitWs {
  unsigned* counters;
  float *part_m, *part_l, *part_acc, *stat_m, *stat_l;
  size_t bytes;
};

static SplitWs carve(void* base, int rows, int hq, int hkv, int splits, int d) {
  SplitWs w{};
  size_t off = 0;
  char* b = static_cast<char*>(base);
  auto take = [&](size_t n) { size_t o = off; off = align_up(off + n, 256); return b ? b + o : nullptr; };
  w.counters = reinterpret_cast<unsigned*>(take(sizeof(unsigned) * rows * hkv));
  w.part_m = reinterpret_cast<float*>(take(sizeof(float) * (size_t)rows * hq * splits));
  w.part_l = reinterpret_cast<float*>(take(sizeof(float) * (size_t)rows * hq * splits));
  w.part_acc = reinterpret_cast<float*>(take(sizeof(float) * (size_t)rows * hq * splits * d));
  w.stat_m = reinterpret_cast<float*>(take(sizeof(float) * (size_t)rows * hq));
  w.stat_l = reinterpret_cast<float*>(take(sizeof(float) * (size_t)rows * hq));
  w.bytes = off;
  return w;
}

static int general_splits(int n, int hkv, int s, int d, int G) {
  Shape sh;
  if (!pick_shape(d, G, &sh)) return 1;
  int target = 4 * sm_count();
  int per_row = (target + n * hkv - 1) / (n * hkv);
  int max_useful = (s + tile_keys(sh) - 1) / tile_keys(sh);
  int sp = per_row < max_useful ? per_row : max_useful;
  if (sp > 256) sp = 256;
  return sp < 1 ? 1 : sp;
}

// ---------------------------------------------------------------- capture
// cap[i][j] = sum_h exp2(s_hij - M_ih) / L_ih  (fp64 over heads, in head order),
// 0 where key j is not visible — head-summed probabilities, _attn_ext.pyx:75-76
template <typename T>
__global__ void capture_kernel(const float* __restrict__ q, const T* __restrict__ k, int n, int hq,
                               int hkv, int d, int s, const int64_t* __restrict__ q_pos,
                               const int64_t* __restrict__ k_pos, const uint8_t* __restrict__ allowed,
                               const float* __restrict__ stat_m, const float* __restrict__ stat_l,
                               float scale_log2, double* __restrict__ cap) {
  int i = blockIdx.y;
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s) return;
  double acc = 0.0;
  bool vis = k_pos[j] <= q_pos[i] && (allowed == nullptr || allowed[j]);
  if (vis) {
    int G = hq / hkv;
    for (int h = 0; h < hq; ++h) {
      const float* qp = q + ((int64_t)i * hq + h) * d;
      const T* kp = k + ((int64_t)j * hkv + h / G) * d;
      float dot = 0.f;
      for (int e = 0; e < d; ++e) dot = fmaf(qp[e] * scale_log2, KV<T>::get(kp, e), dot);
      float mm = stat_m[(int64_t)i * hq + h];
      acc += (double)exp2f(dot - mm) / (double)stat_l[(int64_t)i * hq + h];
    }
  }
  cap[(int64_t)i * s + j] = acc;
}

// row-normalise (cap /= cap.sum(axis=1), _attn_ext.pyx:113-114)
__global__ void rownorm_kernel(double* cap, int s) {
  __shared__ double red[256];
  double* row = cap + (int64_t)blockIdx.x * s;
  double acc = 0.0;
  for (int j = threadIdx.x; j < s; j += blockDim.x) acc += row[j];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  double tot = red[0];
  for (int j = threadIdx.x; j < s; j += blockDim.x) row[j] = row[j] / tot;
}

__global__ void fill_i32(int32_t* p, int32_t v) { *p = v; }

__global__ void advance_kernel(int32_t* len, int n, int delta) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) len[i] += delta;
}

// the same, launched as a programmatic dependent of a decode kernel: it becomes
// resident while the decode runs and waits for its completion (every reader of
// the lengths is done); it never triggers early, so the kernel after it starts
// only once the lengths are advanced
__global__ void advance_after_kernel(int32_t* len, int n, int delta) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) len[i] += delta;
}

__global__ void advance_after_rows_kernel(int32_t* len, int n, int delta, const int32_t* active) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && active[i]) len[i] += delta;
}

static int advance_after_rows(int32_t* len, int n, const int32_t* active, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((n + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, advance_after_rows_kernel, len, n, 1, active);
  if (e != cudaSuccess) return cuda_status(e, "advance_after_rows_kernel launch");
  return RK_OK;
}

static int advance_after(int32_t* len, int n, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((n + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, advance_after_kernel, len, n, 1);
  if (e != cudaSuccess) return cuda_status(e, "advance_after_kernel launch");
  return RK_OK;
}

// ---------------------------------------------------------------- score finalize
// Per row: per head M_h, L_h over items; per bin mass = sum_h sum_items(bin)
// l*exp2(m - M_h)/L_h (fp64); row sum over all bins (incl. current and
// inactive, as the reference's row normalisation); massn = mass / rowsum.
// mode 0 (multi-row question): massn -> rowmass[row][bin] then summed over rows;
// mode 1 (batched decode): massn -> raw[row][bin] directly.
// slots: partial slots per item (warps per kv-head of the bulk decode kernel,
// 1 for the split kernel); slot of (item, slice) = item * slots + slice.
__global__ void score_rows_kernel(const float* __restrict__ part_m, const float* __restrict__ part_l,
                                  int nsplit, int slots, int hq, const int32_t* __restrict__ items, int items_stride,
                                  const int32_t* __restrict__ n_items_dev, int n_items_static, int n_bins,
                                  const uint8_t* __restrict__ active, double* __restrict__ out_rows) {
  extern __shared__ double sh[];
  double* mass = sh;                                   // [n_bins + 1]
  double* Lh = mass + n_bins + 1;                      // [hq] fp64 1 / denominators
  float* Mh = reinterpret_cast<float*>(Lh + hq);       // [hq]
  int* bin_lo = reinterpret_cast<int*>(Mh + hq);       // [n_bins + 2]
  float* sm_m = reinterpret_cast<float*>(bin_lo + n_bins + 2);   // the row's [hq][nsplit] statistics
  float* sm_l = sm_m + (size_t)hq * nsplit;
  const int row = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int32_t* tab = items + (size_t)row * items_stride * 3;
  const int n_items = n_items_dev ? n_items_dev[items_stride ? row : 0] : n_items_static;
  const float* pm = part_m + (size_t)row * hq * nsplit;
  const float* pl = part_l + (size_t)row * hq * nsplit;
  const int n_slots = n_items * slots;
  // the row's statistics into shared memory: up to 2 x 16 loads per thread in flight at once
  constexpr int kU = 16;
  const int n_stat = hq * nsplit;
  for (int e0 = threadIdx.x; e0 < n_stat; e0 += kU * blockDim.x) {
    float a[kU], b[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * blockDim.x;
      a[u] = e < n_stat ? pm[e] : 0.f;
      b[u] = e < n_stat ? pl[e] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < n_stat) {
        sm_m[e] = a[u];
        sm_l[e] = b[u];
      }
    }
  }
  // first item of each bin (items are sorted by bin), one thread per item
  if (n_items == 0) {
    for (int b = threadIdx.x; b <= n_bins + 1; b += blockDim.x) bin_lo[b] = 0;
  }
  for (int it = threadIdx.x; it < n_items; it += blockDim.x) {
    const int bin = tab[it * 3 + 2], prev = it > 0 ? tab[(it - 1) * 3 + 2] : -1;
    for (int b = max(prev + 1, 0); b <= min(bin, n_bins + 1); ++b) bin_lo[b] = it;
    if (it == n_items - 1)
      for (int b = max(bin + 1, 0); b <= n_bins + 1; ++b) bin_lo[b] = n_items;
  }
  __syncthreads();
  // per head: M_h = max over items, L_h = sum l exp2(m - M_h) (warp per head, fixed lane order)
  for (int h = warp; h < hq; h += nw) {
    float mx = -INFINITY;
    for (int it = lane; it < n_slots; it += 32) mx = fmaxf(mx, sm_m[h * nsplit + it]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double L = 0.0;
    for (int it = lane; it < n_slots; it += 32)
      L += (double)sm_l[h * nsplit + it] * (double)exp2f(sm_m[h * nsplit + it] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane == 0) {
      Mh[h] = mx;
      Lh[h] = 1.0 / L;                         // the head's reciprocal denominator
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b <= n_bins; b += blockDim.x) {
    double acc = 0.0;
    for (int h = 0; h < hq; ++h) {
      double hs = 0.0;
      for (int it = bin_lo[b] * slots; it < bin_lo[b + 1] * slots; ++it)
        hs += (double)sm_l[h * nsplit + it] * (double)exp2f(sm_m[h * nsplit + it] - Mh[h]);
      acc += hs * Lh[h];
    }
    mass[b] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int b = 0; b <= n_bins; ++b) tot += mass[b];
    mass[n_bins] = tot;                        // (the current round's own entry is not written out)
  }
  __syncthreads();
  const double tot = mass[n_bins];
  for (int b = threadIdx.x; b < n_bins; b += blockDim.x) {
    const bool on = active == nullptr || active[b];
    out_rows[(size_t)row * n_bins + b] = on ? mass[b] / tot : 0.0;
  }
}

// raw[a] over active bins (ascending) = sum over rows of massn[row][bin]: one block per bin,
// a fixed-order tree over the rows (deterministic)
constexpr int kSumThreads = 256;
__global__ void __launch_bounds__(kSumThreads) score_sum_rows_kernel(const double* __restrict__ rows_mass,
                                                                     int n_rows, int n_bins,
                                                                     const uint8_t* __restrict__ active,
                                                                     double* __restrict__ raw) {
  __shared__ double red[kSumThreads];
  const int b = blockIdx.x;
  if (active && !active[b]) return;            // uniform over the block
  int a = 0;                                   // this bin's rank among the active bins
  if (active)
    for (int x0 = 0; x0 < b; x0 += kSumThreads)
      a += __syncthreads_count(x0 + (int)threadIdx.x < b && active[x0 + threadIdx.x]);
  else
    a = b;
  double acc = 0.0;
  for (int r = threadIdx.x; r < n_rows; r += kSumThreads) acc += rows_mass[(size_t)r * n_bins + b];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kSumThreads / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) raw[a] = red[0];
}

static size_t score_rows_smem(int n_bins, int hq, int nsplit) {
  return sizeof(double) * (n_bins + 1 + hq) + sizeof(float) * hq + sizeof(int) * (n_bins + 2) +
         2 * sizeof(float) * (size_t)hq * nsplit;
}

// launches score_rows_kernel with its shared memory (the row's statistics staged)
static int launch_score_rows(int rows, const float* part_m, const float* part_l, int nsplit, int slots, int hq,
                             const int32_t* items, int items_stride, const int32_t* n_items_dev, int n_items_static,
                             int n_bins, const uint8_t* active, double* out_rows, cudaStream_t st) {
  const size_t smem = score_rows_smem(n_bins, hq, nsplit);
  if (smem > 227 * 1024) return fail(RK_ERR_CAPACITY, "score_rows: %zu bytes of statistics per row", smem);
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    RK_CUDA(cudaFuncSetAttribute(score_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "score_rows smem attribute");
    attr = smem;
  }
  score_rows_kernel<<<rows, 128, smem, st>>>(part_m, part_l, nsplit, slots, hq, items, items_stride, n_items_dev,
                                             n_items_static, n_bins, active, out_rows);
  RK_CHECK_LAUNCH("score_rows_kernel");
  return RK_OK;
}

// the tensor-core multi-row path (prefill_tc.cu) serves bf16 K/V, d = 128,
// >= 64 stacked rows; RK_PREFILL_TC=0 forces the CUDA-core split kernel
static bool use_prefill_tc(int kv_dtype, int d, int n, int G) {
  static int env = -1;
  if (env < 0) {
    const char* e = std::getenv("RK_PREFILL_TC");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env && prefill_tc_supported(kv_dtype, d, n, G);
}

// capture matrix from merged (stat_m, stat_l): head-summed, row-normalised
static int launch_capture(const float* q, int n, int hq, int hkv, int d, int s, const void* k, int kv_dtype,
                          const int64_t* q_pos, const int64_t* k_pos, const uint8_t* allowed, const float* stat_m,
                          const float* stat_l, float scale_log2, double* scores, cudaStream_t cs) {
  dim3 g2((s + 255) / 256, n);
  if (kv_dtype == RK_F32)
    capture_kernel<float><<<g2, 256, 0, cs>>>(q, (const float*)k, n, hq, hkv, d, s, q_pos, k_pos, allowed,
                                             stat_m, stat_l, scale_log2, scores);
  else
    capture_kernel<__nv_bfloat16><<<g2, 256, 0, cs>>>(q, (const __nv_bfloat16*)k, n, hq, hkv, d, s, q_pos,
                                                     k_pos, allowed, stat_m, stat_l, scale_log2, scores);
  RK_CHECK_LAUNCH("capture_kernel");
  rownorm_kernel<<<n, 256, 0, cs>>>(scores, s);
  RK_CHECK_LAUNCH("rownorm_kernel");
  return RK_OK;
}

}  // namespace rk

using namespace rk;

extern "C" {

size_t rk_attention_workspace_bytes(int n, int hq, int hkv, int s, int d) {
  if (n <= 0 || hq <= 0 || hkv <= 0 || d <= 0) return 256;
  int sp = general_splits(n, hkv, s, d, hq / hkv);
  size_t a = carve(nullptr, n, hq, hkv, sp, d).bytes;
  // the tensor-core path (bf16 K/V only; the kv dtype is not an argument here)
  if (hq % hkv == 0 && prefill_tc_supported(RK_BF16, d, n, hq / hkv)) {
    size_t b = prefill_plan(n, hq, hkv, s, 0, false).total;
    if (b > a) a = b;
  }
  return a;
}

int rk_attention_forward(const float* q, int n, int hq, int d, const void* k, const void* v,
                         int kv_dtype, int s, int hkv, const int64_t* q_pos, const int64_t* k_pos,
                         const uint8_t* allowed, float* out, double* scores, int32_t* bad_row,
                         void* workspace, size_t workspace_bytes, rk_stream_t stream) {
  Shape sh;
  int st = check_heads(hq, hkv, d, &sh);
  if (st) return st;
  if (n < 0 || s < 0) return fail(RK_ERR_DOMAIN, "negative row count");
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (bad_row) {
    fill_i32<<<1, 1, 0, cs>>>(bad_row, INT_MAX);
    RK_CHECK_LAUNCH("fill bad_row");
  }
  if (n == 0) return RK_OK;
  if (s == 0) {
    if (bad_row) { fill_i32<<<1, 1, 0, cs>>>(bad_row, 0); RK_CHECK_LAUNCH("fill bad_row"); }
    return RK_OK;
  }
  const float scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
  if (use_prefill_tc(kv_dtype, d, n, hq / hkv)) {
    // tensor-core multi-row path (prefill_tc.cu); statistics feed the capture
    float *stat_m = nullptr, *stat_l = nullptr;
    st = launch_prefill_tc(q, n, hq, k, v, s, hkv, q_pos, k_pos, allowed, nullptr, 0, false, out, bad_row,
                           workspace, workspace_bytes, nullptr, nullptr, &stat_m, &stat_l, cs);
    if (st) return st;
    if (scores) return launch_capture(q, n, hq, hkv, d, s, k, kv_dtype, q_pos, k_pos, allowed, stat_m, stat_l,
                                      scale_log2, scores, cs);
    return RK_OK;
  }
  int sp = general_splits(n, hkv, s, d, hq / hkv);
  SplitWs w = carve(workspace, n, hq, hkv, sp, d);
  if (w.bytes > workspace_bytes)
    return fail(RK_ERR_CAPACITY, "workspace %zu bytes < required %zu", workspace_bytes, w.bytes);
  SplitParams p{};
  p.q = q; p.k = k; p.v = v;
  p.row_stride = (int64_t)hkv * d;
  p.s_static = s;
  p.q_pos = q_pos; p.k_pos = k_pos; p.allowed = allowed;
  p.rows = n; p.hq = hq; p.hkv = hkv; p.d = d;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
  p.out = out;
  p.part_m = w.part_m; p.part_l = w.part_l; p.part_acc = w.part_acc;
  p.counters = w.counters; p.bad_row = bad_row;
  p.stat_m = scores ? w.stat_m : nullptr;
  p.stat_l = scores ? w.stat_l : nullptr;
  // the arrival counters must be zero; the arena is shared by calls of other shapes
  RK_CUDA(cudaMemsetAsync(w.counters, 0, sizeof(unsigned) * (size_t)n * hkv, cs), "counter reset");
  dim3 grid(sp, n, hkv);
  st = dispatch_split(kv_dtype, false, false, hq / hkv, sh, grid, cs, p);
  if (st) return st;
  if (scores)
    return launch_capture(q, n, hq, hkv, d, s, k, kv_dtype, q_pos, k_pos, allowed, w.stat_m, w.stat_l,
                          p.scale_log2, scores, cs);
  return RK_OK;
}

size_t rk_decode_workspace_bytes(int batch, int hq, int hkv, int d, int max_splits) {
  if (batch <= 0 || hq <= 0 || hkv <= 0 || d <= 0) return 256;
  if (max_splits < 148 * 4) max_splits = 148 * 4;   // persistent CTAs x warps per head
  return carve(nullptr, batch, hq, hkv, max_splits, d).bytes;
}

static int decode_splits(int batch, int hkv, int max_seq_len, int d, int G) {
  Shape sh;
  if (!pick_shape(d, G, &sh)) return 1;
  int target = 4 * sm_count();
  int per = (target + batch * hkv - 1) / (batch * hkv);
  int useful = (max_seq_len + 2 * tile_keys(sh) - 1) / (2 * tile_keys(sh));
  int sp = per < useful ? per : useful;
  if (sp > 128) sp = 128;
  return sp < 1 ? 1 : sp;
}

int rk_decode_attention(const float* q, int batch, int hq, int d, void* k_cache, void* v_cache,
                        int kv_dtype, int hkv, int64_t cache_stride, const int32_t* seq_len,
                        int max_seq_len, const void* k_new, const void* v_new, const int32_t* items,
                        const int32_t* n_items, int items_stride, float* out, int32_t* advance_len,
                        void* workspace, size_t workspace_bytes, rk_stream_t stream) {
  Shape sh;
  int st = check_heads(hq, hkv, d, &sh);
  if (st) return st;
  if (batch <= 0) return RK_OK;
  if (max_seq_len <= 0) return fail(RK_ERR_DOMAIN, "max_seq_len must be positive");
  if ((k_new == nullptr) != (v_new == nullptr)) return fail(RK_ERR_DOMAIN, "k_new and v_new go together");
  if (items && (items_stride <= 0 || items_stride > 512 || n_items == nullptr))
    return fail(RK_ERR_DOMAIN, "item table needs 0 < items_stride <= 512 and n_items");
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  const int G = hq / hkv;
  if (!items) {   // small batches: one cluster per (dialogue, kv-head), merge in DSMEM (decode_cluster.cu)
    const int C = cluster_decode_size(kv_dtype, d, hkv, G, batch, max_seq_len, cache_stride);
    if (C) {
      st = launch_decode_cluster(C, kv_dtype, q, batch, hq, d, k_cache, v_cache, hkv, cache_stride, seq_len,
                                 max_seq_len, k_new, v_new, out, cs);
      if (st) return st;
      if (advance_len) return advance_after(advance_len, batch, cs);
      return RK_OK;
    }
  }
  if (bulk_supported(kv_dtype, d, hkv, G)) {
    int sp = items ? items_stride * (8 / hkv) : bulk_splits(batch, max_seq_len, hkv);
    SplitWs w = carve(workspace, batch, hq, hkv, sp, d);
    if (w.bytes > workspace_bytes)
      return fail(RK_ERR_CAPACITY, "decode workspace %zu bytes < required %zu", workspace_bytes, w.bytes);
    BulkParams p{};
    p.q = q; p.k = k_cache; p.v = v_cache; p.batch_stride = cache_stride;
    p.seq_len = seq_len; p.k_new = const_cast<void*>(k_new); p.v_new = const_cast<void*>(v_new);
    p.items = items; p.n_items = n_items; p.items_stride = items ? items_stride : 0;
    p.B = batch; p.hq = hq; p.nsplit = sp;
    p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
    p.part_m = w.part_m; p.part_l = w.part_l; p.part_acc = w.part_acc;
    return launch_decode_bulk(kv_dtype, d, hkv, G, sp, p, out, advance_len, cs, true);
  }
  int sp = items ? items_stride : decode_splits(batch, hkv, max_seq_len, d, G);
  SplitWs w = carve(workspace, batch, hq, hkv, sp, d);
  if (w.bytes > workspace_bytes)
    return fail(RK_ERR_CAPACITY, "decode workspace %zu bytes < required %zu (splits %d)", workspace_bytes,
                w.bytes, sp);
  SplitParams p{};
  p.q = q; p.k = k_cache; p.v = v_cache;
  p.row_stride = (int64_t)hkv * d;
  p.batch_stride = cache_stride;
  p.seq_len = seq_len;
  p.s_static = max_seq_len;
  p.k_new = const_cast<void*>(k_new); p.v_new = const_cast<void*>(v_new);
  p.items = items; p.n_items = n_items; p.items_row_stride = items ? items_stride : 0;
  p.rows = batch; p.hq = hq; p.hkv = hkv; p.d = d;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
  p.out = out;
  p.part_m = w.part_m; p.part_l = w.part_l; p.part_acc = w.part_acc;
  p.counters = w.counters;
  RK_CUDA(cudaMemsetAsync(w.counters, 0, sizeof(unsigned) * (size_t)batch * hkv, cs), "counter reset");
  dim3 grid(sp, batch, hkv);
  st = dispatch_split(kv_dtype, true, false, G, sh, grid, cs, p);
  if (st) return st;
  if (advance_len) return rk_advance_lengths(advance_len, batch, 1, stream);
  return RK_OK;
}

int rk_decode_attention_rows(const float* q, int batch, int hq, int d, void* k_cache, void* v_cache,
                             int kv_dtype, int hkv, int64_t cache_stride, const int32_t* seq_len,
                             int max_seq_len, const void* k_new, const void* v_new, const int32_t* row_active,
                             float* out, int32_t* advance_len, rk_stream_t stream) {
  Shape sh;
  int st = check_heads(hq, hkv, d, &sh);
  if (st) return st;
  if (batch <= 0) return RK_OK;
  if (max_seq_len <= 0) return fail(RK_ERR_DOMAIN, "max_seq_len must be positive");
  if ((k_new == nullptr) != (v_new == nullptr)) return fail(RK_ERR_DOMAIN, "k_new and v_new go together");
  if (row_active == nullptr) return fail(RK_ERR_DOMAIN, "rk_decode_attention_rows needs row_active");
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  const int C = cluster_decode_size(kv_dtype, d, hkv, hq / hkv, batch, max_seq_len, cache_stride, true);
  if (C <= 0)
    return fail(RK_ERR_DOMAIN, "row-masked decode runs the cluster kernel (bf16/fp32, d 64/128, G 1/2/4/7/8)");
  st = launch_decode_cluster(C, kv_dtype, q, batch, hq, d, k_cache, v_cache, hkv, cache_stride, seq_len,
                             max_seq_len, k_new, v_new, out, cs, row_active);
  if (st) return st;
  if (advance_len) return advance_after_rows(advance_len, batch, row_active, cs);
  return RK_OK;
}

int rk_decode_plan(int batch, int hq, int hkv, int d, int kv_dtype, int max_seq_len, int64_t cache_stride,
                   int has_items) {
  if (batch <= 0 || hkv <= 0 || hq <= 0 || hq % hkv) return -1;
  const int G = hq / hkv;
  if (!has_items) {
    const int C = cluster_decode_size(kv_dtype, d, hkv, G, batch, max_seq_len, cache_stride);
    if (C) return C;
  }
  return bulk_supported(kv_dtype, d, hkv, G) ? 0 : -1;
}

int rk_advance_lengths(int32_t* seq_len, int n, int delta, rk_stream_t stream) {
  if (n <= 0) return RK_OK;
  advance_kernel<<<(n + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(seq_len, n, delta);
  RK_CHECK_LAUNCH("advance_kernel");
  return RK_OK;
}

// the tcgen05 path (prefill_tc.cu, scores-only kernel) serves bf16 K, d = 128,
// >= 64 stacked rows; RK_SCORE_TC=0 forces the CUDA-core split kernel (tests compare both)
static bool use_tc(int kv_dtype, int d, int n_q, int G) {
  static int env = -1;
  if (env < 0) {
    const char* e = std::getenv("RK_SCORE_TC");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env && prefill_tc_supported(kv_dtype, d, n_q, G);
}

size_t rk_round_scores_workspace_bytes(int n_q, int hq, int hkv, int n_items, int d, int n_bins) {
  if (n_q <= 0 || n_items <= 0 || hkv <= 0 || hq % hkv) return 256;
  size_t a = carve(nullptr, n_q, hq, hkv, n_items, d).bytes;
  a = align_up(a + sizeof(double) * (size_t)n_q * (n_bins > 0 ? n_bins : 1), 256);
  if (prefill_tc_supported(RK_BF16, d, n_q, hq / hkv))
    a = align_up(a + prefill_plan(n_q, hq, hkv, 0, n_items, true, false).total, 256);
  return a;
}

int rk_round_scores(const float* q, int n_q, int hq, int d, const void* k, int kv_dtype, int s, int hkv,
                    const int64_t* q_pos, const int64_t* k_pos, const int32_t* items, int n_items,
                    int n_bins, const uint8_t* active, double* raw_out, void* workspace,
                    size_t workspace_bytes, rk_stream_t stream) {
  Shape sh;
  int st = check_heads(hq, hkv, d, &sh);
  if (st) return st;
  if (n_q <= 0 || n_items <= 0 || n_bins <= 0) return fail(RK_ERR_DOMAIN, "round scoring needs rows, items, bins");
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  SplitWs w = carve(workspace, n_q, hq, hkv, n_items, d);
  size_t need = align_up(w.bytes + sizeof(double) * (size_t)n_q * n_bins, 256);
  if (need > workspace_bytes) return fail(RK_ERR_CAPACITY, "score workspace %zu < %zu", workspace_bytes, need);
  double* rows_mass = reinterpret_cast<double*>(static_cast<char*>(workspace) + w.bytes);
  const float* part_m = w.part_m;
  const float* part_l = w.part_l;
  int nsplit = n_items, slots = 1;                  // the tensor-core pass: 2 slots (column halves) per item
  if (use_tc(kv_dtype, d, n_q, hq / hkv)) {
    const size_t tc_bytes = prefill_plan(n_q, hq, hkv, s, n_items, true, false).total;
    if (need + tc_bytes > workspace_bytes)
      return fail(RK_ERR_CAPACITY, "score workspace too small for the tensor-core path");
    float *im = nullptr, *il = nullptr;
    st = launch_prefill_tc(q, n_q, hq, k, nullptr, s, hkv, q_pos, k_pos, nullptr, items, n_items, true, nullptr,
                           nullptr, static_cast<char*>(workspace) + need, tc_bytes, &im, &il, nullptr, nullptr, cs);
    if (st) return st;
    part_m = im;
    part_l = il;
    nsplit = 2 * n_items;
    slots = 2;
  } else {
  SplitParams p{};
  p.q = q; p.k = k; p.v = k;
  p.row_stride = (int64_t)hkv * d;
  p.s_static = s;
  p.q_pos = q_pos; p.k_pos = k_pos;
  p.items = items; p.items_row_stride = 0;
  p.rows = n_q; p.hq = hq; p.hkv = hkv; p.d = d;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)d));
  p.part_m = w.part_m; p.part_l = w.part_l; p.part_acc = w.part_acc;
  p.counters = w.counters;
  dim3 grid(n_items, n_q, hkv);
  st = dispatch_split(kv_dtype, false, true, hq / hkv, sh, grid, cs, p);
  if (st) return st;
  }
  st = launch_score_rows(n_q, part_m, part_l, nsplit, slots, hq, items, 0, nullptr, n_items, n_bins, nullptr,
                         rows_mass, cs);
  if (st) return st;
  score_sum_rows_kernel<<<n_bins, kSumThreads, 0, cs>>>(rows_mass, n_q, n_bins, active, raw_out);
  RK_CHECK_LAUNCH("score_sum_rows_kernel");
  return RK_OK;
}

int rk_round_scores_finalize(int batch, int hq, int hkv, int d, int kv_dtype, int items_stride,
                             const int32_t* items, const int32_t* n_items, int n_bins, const uint8_t* active,
                             double* raw_out, void* workspace, rk_stream_t stream) {
  if (batch <= 0 || n_bins <= 0) return RK_OK;
  if (items == nullptr || n_items == nullptr || items_stride <= 0)
    return fail(RK_ERR_DOMAIN, "finalize needs the item table used by rk_decode_attention");
  // same partial-slot layout rk_decode_attention used for this shape
  const int slots = bulk_supported(kv_dtype, d, hkv, hq / hkv) ? 8 / hkv : 1;
  const int nsplit = items_stride * slots;
  SplitWs w = carve(workspace, batch, hq, hkv, nsplit, d);
  return launch_score_rows(batch, w.part_m, w.part_l, nsplit, slots, hq, items, items_stride, n_items, 0, n_bins,
                           active, raw_out, reinterpret_cast<cudaStream_t>(stream));
}

size_t rk_prefill_workspace_bytes(int n_q, int hq, int hkv, int s, int d, int n_items, int n_bins) {
  if (n_q <= 0 || hq <= 0 || hkv <= 0 || d <= 0 || hq % hkv) return 256;
  size_t a = prefill_plan(n_q, hq, hkv, s, n_items > 0 ? n_items : 0, n_bins > 0).total;
  if (n_bins > 0) a = align_up(a + sizeof(double) * (size_t)n_q * n_bins, 256);
  return a;
}

int rk_prefill_attention(const float* q, int n_q, int hq, int d, const void* k, const void* v, int kv_dtype,
                         int s, int hkv, const int64_t* q_pos, const int64_t* k_pos, const uint8_t* allowed,
                         const int32_t* items, int n_items, int n_bins, const uint8_t* active, float* out,
                         double* raw_out, int32_t* bad_row, void* workspace, size_t workspace_bytes,
                         int flags, rk_stream_t stream) {
  Shape sh;
  int st = check_heads(hq, hkv, d, &sh);
  if (st) return st;
  if (n_q <= 0 || s <= 0) return fail(RK_ERR_DOMAIN, "prefill needs rows and keys");
  if (!prefill_tc_supported(kv_dtype, d, n_q, hq / hkv))
    return fail(RK_ERR_UNSUPPORTED, "prefill path needs bf16 K/V, head_dim 128 and >= 64 stacked rows");
  const bool stats = raw_out != nullptr;
  if (stats && (items == nullptr || n_items <= 0 || n_bins <= 0))
    return fail(RK_ERR_DOMAIN, "round scoring needs the round-aligned item table and n_bins");
  const bool single_pass = (flags & RK_PREFILL_SINGLE_PASS) != 0;
  if (stats && single_pass)
    return fail(RK_ERR_DOMAIN, "round scoring needs the two-pass (fp32-class) path: selection is bit-exact");
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (bad_row) {
    fill_i32<<<1, 1, 0, cs>>>(bad_row, INT_MAX);
    RK_CHECK_LAUNCH("fill bad_row");
  }
  PrefillPlan pl = prefill_plan(n_q, hq, hkv, s, items ? n_items : 0, stats);
  size_t need = stats ? align_up(pl.total + sizeof(double) * (size_t)n_q * n_bins, 256) : pl.total;
  if (need > workspace_bytes) return fail(RK_ERR_CAPACITY, "prefill workspace %zu < %zu", workspace_bytes, need);
  float *item_m = nullptr, *item_l = nullptr;
  st = launch_prefill_tc(q, n_q, hq, k, v, s, hkv, q_pos, k_pos, allowed, items, items ? n_items : 0, stats, out,
                         bad_row, workspace, pl.total, &item_m, &item_l, nullptr, nullptr, cs, single_pass);
  if (st) return st;
  if (stats) {
    double* rows_mass = reinterpret_cast<double*>(static_cast<char*>(workspace) + pl.total);
    st = launch_score_rows(n_q, item_m, item_l, 2 * n_items, 2, hq, items, 0, nullptr, n_items, n_bins, nullptr,
                           rows_mass, cs);
    if (st) return st;
    score_sum_rows_kernel<<<n_bins, kSumThreads, 0, cs>>>(rows_mass, n_q, n_bins, active, raw_out);
    RK_CHECK_LAUNCH("score_sum_rows_kernel");
  }
  return RK_OK;
}

}  // extern "C"
