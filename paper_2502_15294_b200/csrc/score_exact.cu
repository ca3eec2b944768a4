// Exact (fp64) watershed round scoring: the Eq. 1 masses with the reference
// kernel's arithmetic, so the kept-round indices are bit-exact by
// construction rather than within a tolerance.
//
// Reference (_attn_ext.pyx:52-76, 113-114; stats.py:59-94): for query row i and
// head h, score_j = (sum_t (double)q[t] * (double)k[j][t]) * (1/sqrt(d)) summed
// sequentially over t; w_j = exp(score_j - max); p_hj = w_j / sum_j w_j;
// cap_ij = sum_h p_hj; capn = cap / rowsum; raw_k = sum over the question rows
// and round k's keys of capn.
//
// Here:
//  * logits: q is fp32 and K fp32 or bf16, so every product q*k is EXACT in fp64
//    (<= 48 of 53 mantissa bits).  bf16 keys with d 64 / 128 run on the FP64
//    tensor pipe (exact_stats_dmma_kernel: the sum over t in four interleaved
//    partial sums, ~1e-16 relative from the reference's sequential sum); other
//    shapes run one thread per key with the reference's sequential fp64 sum
//    (an FMA and its separate multiply + add round identically: bit-identical);
//  * per (row, head, round-aligned item): (m, l = sum exp(s - m)) in fp64,
//    reduced in a fixed tree relative to the item's first key, so identical
//    rounds get bit-identical statistics wherever they sit (exact ties go to
//    the lower index, as the reference's stable argsort);
//  * finalize: per (row, head) M = max m, D = sum l exp(m - M); per bin
//    sum_h (sum_items l exp(m - M)) / D; rowsum over every bin (the current
//    question's keys and inactive rounds' keys included, as the reference's
//    row normalisation); raw = sum over rows of mass / rowsum.
// The remaining differences from the reference are fp64 roundings in the exp and
// in the summation order (~1e-16 relative); a kept-set flip needs a K-boundary gap
// below ~1e-14, which rk_selection_margin reports.
//
// Cost (C2, one decode row): 16 K keys x 32 heads x 128 DFMA = 67 M DFMA per
// dialogue plus one read of layer Lw-1's K (32 MiB): ~5 us per dialogue.
#include "rk_common.cuh"

namespace rk {

constexpr int kExThreads = 128;
constexpr int kExMaxG = 8;       // query heads per kv-head handled per block
constexpr int kExWarps = kExThreads / 32;

template <typename KT>
struct KLoad;

template <>
struct KLoad<__nv_bfloat16> {
  // 8 bf16 -> 8 doubles (exact)
  static __device__ __forceinline__ void load8(const __nv_bfloat16* p, double* out) {
    uint4 w = *reinterpret_cast<const uint4*>(p);
    uint32_t a[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = bf16x2_to_f2(a[i]);
      out[2 * i] = (double)f.x;
      out[2 * i + 1] = (double)f.y;
    }
  }
};

template <>
struct KLoad<float> {
  static __device__ __forceinline__ void load8(const float* p, double* out) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  }
};

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One key sub-chunk's logits (acc * scale; masked keys -> -inf) folded into the
// running (m, l) per (row, head): sub-chunk max by a fixed warp/block tree, then
// sum exp(s - max), merged into the running statistics.
template <int RT, int G>
__device__ __forceinline__ void chunk_stats(const double (&acc)[RT][G], bool in, int64_t kp, const int64_t (&qp)[RT],
                                            double scale, double (*red)[RT * G], double* sub_m, double* run_m,
                                            double* run_l) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double s[RT][G];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const bool vis = in && kp <= qp[r];
      s[r][h] = vis ? (scale > 0.0 ? __dmul_rn(acc[r][h], scale) : __ddiv_rn(acc[r][h], -scale)) : -INFINITY;
      double m = warp_max_d(s[r][h]);
      if (lane == 0) red[warp][r * G + h] = m;
    }
    __syncthreads();
    if (tid < RT * G) {
      double m = red[0][tid];
#pragma unroll
      for (int w = 1; w < kExWarps; ++w) m = fmax(m, red[w][tid]);
      sub_m[tid] = m;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int h = 0; h < G; ++h) {
        const double m = sub_m[r * G + h];
        double e = (s[r][h] == -INFINITY) ? 0.0 : exp(__dsub_rn(s[r][h], m));
        e = warp_sum_d(e);
        if (lane == 0) red[warp][r * G + h] = e;
      }
    __syncthreads();
    if (tid < RT * G) {
      double l = red[0][tid];
#pragma unroll
      for (int w = 1; w < kExWarps; ++w) l = __dadd_rn(l, red[w][tid]);
      const double m = sub_m[tid];
      if (m != -INFINITY) {
        const double M = run_m[tid];
        if (M == -INFINITY) {
          run_m[tid] = m;
          run_l[tid] = l;
        } else if (m > M) {
          run_l[tid] = __fma_rn(run_l[tid], exp(__dsub_rn(M, m)), l);
          run_m[tid] = m;
        } else {
          run_l[tid] = __fma_rn(l, exp(__dsub_rn(m, M)), run_l[tid]);
        }
      }
    }
    __syncthreads();
}

// grid (items_stride, hkv, batch * row_tiles), block kExThreads.
// part_m / part_l: [batch][n_q][hq][items_stride] fp64.
template <typename KT, int RT, int G>
__global__ void __launch_bounds__(kExThreads) exact_stats_kernel(
    const float* __restrict__ q, int n_q, int hq, int d, const KT* __restrict__ k, int64_t k_bstride, int hkv,
    const int32_t* __restrict__ seq_len, int s_static, const int64_t* __restrict__ q_pos,
    const int64_t* __restrict__ k_pos, const int32_t* __restrict__ items, int items_stride,
    const int32_t* __restrict__ n_items_dev, double scale, int row_tiles, double* __restrict__ part_m,
    double* __restrict__ part_l) {
  extern __shared__ double qs[];                       // [RT][G][d]
  __shared__ double red[kExWarps][RT * G];
  __shared__ double run_m[RT * G], run_l[RT * G], sub_m[RT * G];
  const int it = blockIdx.x, g = blockIdx.y;
  const int b = blockIdx.z / row_tiles;
  const int r0 = (blockIdx.z % row_tiles) * RT;
  const int n_items = n_items_dev ? n_items_dev[b] : items_stride;
  if (it >= n_items) return;
  const int32_t* tab = items + ((size_t)b * items_stride + it) * 3;
  const int s_b = seq_len ? seq_len[b] : s_static;
  const int lo = tab[0];
  const int hi = min(tab[1], s_b);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = min(RT, n_q - r0);

  for (int x = tid; x < RT * G * d; x += kExThreads) {
    const int r = x / (G * d), rem = x - r * G * d;
    const int h = rem / d, t = rem - h * d;
    qs[x] = r < nr ? (double)q[(((size_t)b * n_q + r0 + r) * hq + g * G + h) * d + t] : 0.0;
  }
  for (int x = tid; x < RT * G; x += kExThreads) {
    run_m[x] = -INFINITY;
    run_l[x] = 0.0;
  }
  int64_t qp[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) qp[r] = r < nr ? q_pos[r0 + r] : INT64_MIN;
  __syncthreads();

  const KT* kb = k + (size_t)b * k_bstride + (size_t)g * d;
  const int64_t row_stride = (int64_t)hkv * d;
  for (int c0 = lo; c0 < hi; c0 += kExThreads) {
    const int j = c0 + tid;
    const bool in = j < hi;
    const int64_t kp = in ? (k_pos ? k_pos[j] : (int64_t)j) : 0;
    double acc[RT][G];
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
      for (int h = 0; h < G; ++h) acc[r][h] = 0.0;
    if (in) {
      const KT* kr = kb + (int64_t)j * row_stride;
      for (int t0 = 0; t0 < d; t0 += 8) {
        double kv[8];
        KLoad<KT>::load8(kr + t0, kv);
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
#pragma unroll
          for (int r = 0; r < RT; ++r) {
#pragma unroll
            for (int h = 0; h < G; ++h) {
              // sequential over t as the reference; the product is exact in fp64
              acc[r][h] = __fma_rn(qs[(r * G + h) * d + t0 + tt], kv[tt], acc[r][h]);
            }
          }
        }
      }
    }
    chunk_stats<RT, G>(acc, in, kp, qp, scale, red, sub_m, run_m, run_l);
  }
  if (tid < RT * G) {
    const int r = tid / G, h = tid % G;
    if (r < nr) {
      const size_t o = (((size_t)b * n_q + r0 + r) * hq + g * G + h) * items_stride + it;
      part_m[o] = run_m[tid];
      part_l[o] = run_l[tid];
    }
  }
}

// Multi-row questions on the FP64 tensor pipe (mma.sync m8n8k4 f64): the
// DFMA kernel above reads one q operand from shared memory per FMA and runs at
// ~1/3 of the FP64 peak; here a warp computes 8 keys x 8 (row, head) combos per
// instruction with both operands in registers.  The products q*k are exact in
// fp64 as before; the sum over t is split into 4 interleaved partial sums that
// the tensor core adds (dims j*D/4 + s for lane j of the k4 step s), so a logit
// may differ from the sequential sum by fp64 rounding (~1e-16 relative) — the
// same class as the exp and summation roundings the masses already carry (a
// kept-set flip needs a K-boundary gap below ~1e-14).  Each key's logit depends
// only on its own values (not its position), and the statistics are reduced per
// 128-key sub-chunk aligned to the item start in a fixed order, so identical
// rounds still get bit-identical masses.
// Block = 4 warps over 128-key sub-chunks (warp w: keys 32w..32w+31 as 4 n8
// tiles); combos c = r * G + h (r < 4 rows of the tile, h < G heads) padded to
// MT x 8.  K: bf16, D % 32 == 0.  grid (items_stride, hkv, batch * row_tiles).
template <int RT, int MT, int D>
__global__ void __launch_bounds__(kExThreads) exact_stats_dmma_kernel(
    const float* __restrict__ q, int n_q, int hq, int G, const __nv_bfloat16* __restrict__ k, int64_t k_bstride,
    int hkv, const int32_t* __restrict__ seq_len, int s_static, const int64_t* __restrict__ q_pos,
    const int64_t* __restrict__ k_pos, const int32_t* __restrict__ items, int items_stride,
    const int32_t* __restrict__ n_items_dev, double scale, int row_tiles, double* __restrict__ part_m,
    double* __restrict__ part_l) {
  constexpr int NC = MT * 8, DS = D / 4, JS = DS + 1;        // combos, k4 steps, padded j-stride (doubles)
  __shared__ double qs[NC * 4 * JS];                          // [combo][j][s] = q[combo][j * DS + s]
  __shared__ double red[kExWarps][NC];
  __shared__ double run_m[NC], run_l[NC], sub_m[NC];
  const int it = blockIdx.x, g = blockIdx.y;
  const int b = blockIdx.z / row_tiles;
  const int r0 = (blockIdx.z % row_tiles) * RT;
  const int n_items = n_items_dev ? n_items_dev[b] : items_stride;
  if (it >= n_items) return;
  const int32_t* tab = items + ((size_t)b * items_stride + it) * 3;
  const int s_b = seq_len ? seq_len[b] : s_static;
  const int lo = tab[0];
  const int hi = min(tab[1], s_b);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = min(RT, n_q - r0);
  const int ncombo = RT * G;

  for (int x = tid; x < NC * D; x += kExThreads) {
    const int c = x / D, t = x - c * D;
    const int r = c / G, h = c - r * G;
    const double v = (c < ncombo && r < nr) ? (double)q[(((size_t)b * n_q + r0 + r) * hq + g * G + h) * D + t] : 0.0;
    qs[c * 4 * JS + (t / DS) * JS + (t % DS)] = v;
  }
  for (int x = tid; x < NC; x += kExThreads) {
    run_m[x] = -INFINITY;
    run_l[x] = 0.0;
  }
  // this thread's combo rows (one per M tile) and their query positions
  int64_t qp[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int c = mt * 8 + (lane >> 2), r = c / G;
    qp[mt] = (c < ncombo && r < nr) ? q_pos[r0 + r] : INT64_MIN;
  }
  __syncthreads();

  const __nv_bfloat16* kb = k + (size_t)b * k_bstride + (size_t)g * D;
  const int64_t row_stride = (int64_t)hkv * D;
  const int j = lane & 3, kn = lane >> 2;                   // k4 lane (dim quarter), key of the n8 tile
  const double* qa = qs + (lane >> 2) * 4 * JS + j * JS;     // + mt * 8 * 4 * JS + s
  for (int c0 = lo; c0 < hi; c0 += kExThreads) {
    double acc[4][MT][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) acc[nt][mt][0] = acc[nt][mt][1] = 0.0;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int key = c0 + 32 * warp + 8 * nt + kn;
      // dims j*DS .. j*DS + DS-1 of this key (bf16), 8 per 16-byte load
      const uint4* src = reinterpret_cast<const uint4*>(kb + (int64_t)min(key, hi - 1) * row_stride + j * DS);
      const bool kin = key < hi;
#pragma unroll 2
      for (int v = 0; v < DS / 8; ++v) {
        uint4 w4 = src[v];
        if (!kin) w4 = make_uint4(0u, 0u, 0u, 0u);
        const uint32_t ww[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t w = ww[e >> 1];
          const double bv = (double)__uint_as_float((e & 1) ? (w & 0xffff0000u) : (w << 16));
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const double av = qa[mt * 8 * 4 * JS + 8 * v + e];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(acc[nt][mt][0]), "+d"(acc[nt][mt][1]) : "d"(av), "d"(bv));
          }
        }
      }
    }
    // logits of this thread's 8 keys per combo row: C[row lane/4][cols 2j, 2j+1] of each n8 tile
    double sv[MT][8];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = c0 + 32 * warp + 8 * nt + 2 * j + e;
        const bool in = key < hi;
        const int64_t kp = in ? (k_pos ? k_pos[key] : (int64_t)key) : 0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          sv[mt][2 * nt + e] = (in && kp <= qp[mt]) ? __dmul_rn(acc[nt][mt][e], scale) : -INFINITY;
      }
    // sub-chunk max per combo: thread -> 4-lane group -> warp order
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      double m = sv[mt][0];
#pragma unroll
      for (int e = 1; e < 8; ++e) m = fmax(m, sv[mt][e]);
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, 2));
      if (j == 0) red[warp][mt * 8 + kn] = m;
    }
    __syncthreads();
    if (tid < NC) {
      double m = red[0][tid];
#pragma unroll
      for (int w = 1; w < kExWarps; ++w) m = fmax(m, red[w][tid]);
      sub_m[tid] = m;
    }
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const double m = sub_m[mt * 8 + kn];
      double l = 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) l = __dadd_rn(l, sv[mt][e] == -INFINITY ? 0.0 : exp(__dsub_rn(sv[mt][e], m)));
      l = __dadd_rn(l, __shfl_xor_sync(0xffffffffu, l, 1));
      l = __dadd_rn(l, __shfl_xor_sync(0xffffffffu, l, 2));
      if (j == 0) red[warp][mt * 8 + kn] = l;
    }
    __syncthreads();
    if (tid < NC) {
      double l = red[0][tid];
#pragma unroll
      for (int w = 1; w < kExWarps; ++w) l = __dadd_rn(l, red[w][tid]);
      const double m = sub_m[tid];
      if (m != -INFINITY) {
        const double M = run_m[tid];
        if (M == -INFINITY) {
          run_m[tid] = m;
          run_l[tid] = l;
        } else if (m > M) {
          run_l[tid] = __fma_rn(run_l[tid], exp(__dsub_rn(M, m)), l);
          run_m[tid] = m;
        } else {
          run_l[tid] = __fma_rn(l, exp(__dsub_rn(m, M)), run_l[tid]);
        }
      }
    }
    __syncthreads();
  }
  if (tid < ncombo) {
    const int r = tid / G, h = tid - r * G;
    if (r < nr) {
      const size_t o = (((size_t)b * n_q + r0 + r) * hq + g * G + h) * items_stride + it;
      part_m[o] = run_m[tid];
      part_l[o] = run_l[tid];
    }
  }
}

// capture_mode="pre" (engine.py:187-200): ONE logit per (row, key), the
// head-summed dot product sum_h q_h . k_kv(h) in fp64 (h ascending, t sequential
// within a head, as the einsum "nhd,shd->ns"), divided by Hq * sqrt(d); one
// softmax over the keys per row.  The statistics are those of a single "head".
// grid (items_stride, 1, batch * row_tiles); part_m / part_l [batch][n_q][1][items_stride].
template <typename KT, int RT>
__global__ void __launch_bounds__(kExThreads) exact_pre_stats_kernel(
    const float* __restrict__ q, int n_q, int hq, int d, const KT* __restrict__ k, int64_t k_bstride, int hkv,
    const int32_t* __restrict__ seq_len, int s_static, const int64_t* __restrict__ q_pos,
    const int64_t* __restrict__ k_pos, const int32_t* __restrict__ items, int items_stride,
    const int32_t* __restrict__ n_items_dev, double denom, int row_tiles, double* __restrict__ part_m,
    double* __restrict__ part_l) {
  extern __shared__ double qs[];                       // [RT][hq][d]
  __shared__ double red[kExWarps][RT];
  __shared__ double run_m[RT], run_l[RT], sub_m[RT];
  const int it = blockIdx.x;
  const int b = blockIdx.z / row_tiles;
  const int r0 = (blockIdx.z % row_tiles) * RT;
  const int n_items = n_items_dev ? n_items_dev[b] : items_stride;
  if (it >= n_items) return;
  const int32_t* tab = items + ((size_t)b * items_stride + it) * 3;
  const int s_b = seq_len ? seq_len[b] : s_static;
  const int lo = tab[0];
  const int hi = min(tab[1], s_b);
  const int tid = threadIdx.x;
  const int nr = min(RT, n_q - r0);
  const int G = hq / hkv;

  for (int x = tid; x < RT * hq * d; x += kExThreads) {
    const int r = x / (hq * d), rem = x - r * hq * d;
    qs[x] = r < nr ? (double)q[((size_t)b * n_q + r0 + r) * hq * d + rem] : 0.0;
  }
  for (int x = tid; x < RT; x += kExThreads) {
    run_m[x] = -INFINITY;
    run_l[x] = 0.0;
  }
  int64_t qp[RT];
#pragma unroll
  for (int r = 0; r < RT; ++r) qp[r] = r < nr ? q_pos[r0 + r] : INT64_MIN;
  __syncthreads();

  const KT* kb = k + (size_t)b * k_bstride;
  const int64_t row_stride = (int64_t)hkv * d;
  for (int c0 = lo; c0 < hi; c0 += kExThreads) {
    const int j = c0 + tid;
    const bool in = j < hi;
    const int64_t kp = in ? (k_pos ? k_pos[j] : (int64_t)j) : 0;
    double acc[RT][1];
#pragma unroll
    for (int r = 0; r < RT; ++r) acc[r][0] = 0.0;
    if (in) {
      const KT* kr = kb + (int64_t)j * row_stride;
      for (int h = 0; h < hq; ++h) {
        const KT* kh = kr + (size_t)(h / G) * d;
        for (int t0 = 0; t0 < d; t0 += 8) {
          double kv[8];
          KLoad<KT>::load8(kh + t0, kv);
#pragma unroll
          for (int tt = 0; tt < 8; ++tt)
#pragma unroll
            for (int r = 0; r < RT; ++r) acc[r][0] = __fma_rn(qs[(r * hq + h) * d + t0 + tt], kv[tt], acc[r][0]);
        }
      }
    }
    chunk_stats<RT, 1>(acc, in, kp, qp, -denom, red, sub_m, run_m, run_l);
  }
  if (tid < nr) {
    const size_t o = ((size_t)b * n_q + r0 + tid) * items_stride + it;
    part_m[o] = run_m[tid];
    part_l[o] = run_l[tid];
  }
}

// one block per (dialogue, row): row mass per bin / rowsum -> rowmass[b][row][bin]
__global__ void exact_rows_kernel(const double* __restrict__ part_m, const double* __restrict__ part_l, int n_q,
                                  int hq, const int32_t* __restrict__ items, int items_stride,
                                  const int32_t* __restrict__ n_items_dev, int n_bins,
                                  double* __restrict__ rowmass) {
  extern __shared__ double sh[];
  double* mass = sh;                       // [n_bins + 1]
  double* Mh = mass + n_bins + 1;          // [hq]
  double* Dh = Mh + hq;                    // [hq]
  int* bin_lo = reinterpret_cast<int*>(Dh + hq);   // [n_bins + 2]
  const int b = blockIdx.x / n_q, row = blockIdx.x % n_q;
  const int n_items = n_items_dev ? n_items_dev[b] : items_stride;
  const int32_t* tab = items + (size_t)b * items_stride * 3;
  const double* pm = part_m + ((size_t)b * n_q + row) * hq * items_stride;
  const double* pl = part_l + ((size_t)b * n_q + row) * hq * items_stride;
  for (int h = threadIdx.x; h < hq; h += blockDim.x) {
    double mx = -INFINITY;
    for (int it = 0; it < n_items; ++it) mx = fmax(mx, pm[h * items_stride + it]);
    double D = 0.0;
    for (int it = 0; it < n_items; ++it) {
      const double m = pm[h * items_stride + it];
      if (m != -INFINITY) D = __fma_rn(pl[h * items_stride + it], exp(__dsub_rn(m, mx)), D);
    }
    Mh[h] = mx;
    Dh[h] = D;
  }
  if (threadIdx.x == 0) {                  // items are sorted by bin: first item of each bin
    int it = 0;
    for (int bn = 0; bn <= n_bins + 1; ++bn) {
      while (it < n_items && tab[it * 3 + 2] < bn) ++it;
      bin_lo[bn] = it;
    }
  }
  __syncthreads();
  for (int bn = threadIdx.x; bn <= n_bins; bn += blockDim.x) {
    double acc = 0.0;
    for (int h = 0; h < hq; ++h) {         // head order as the reference's cap accumulation
      if (Dh[h] <= 0.0) continue;
      double hs = 0.0;
      for (int it = bin_lo[bn]; it < bin_lo[bn + 1]; ++it) {
        const double m = pm[h * items_stride + it];
        if (m != -INFINITY) hs = __fma_rn(pl[h * items_stride + it], exp(__dsub_rn(m, Mh[h])), hs);
      }
      acc = __dadd_rn(acc, __ddiv_rn(hs, Dh[h]));
    }
    mass[bn] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int bn = 0; bn <= n_bins; ++bn) tot = __dadd_rn(tot, mass[bn]);
    double* out = rowmass + ((size_t)b * n_q + row) * n_bins;
    for (int bn = 0; bn < n_bins; ++bn) out[bn] = tot > 0.0 ? __ddiv_rn(mass[bn], tot) : 0.0;
  }
}

// raw[b][a] over active bins (ascending) = sum over rows (in order) of rowmass
__global__ void exact_sum_rows_kernel(const double* __restrict__ rowmass, int n_q, int n_bins,
                                      const uint8_t* __restrict__ active, int n_out, double* __restrict__ raw) {
  const int b = blockIdx.y;
  const int bn = blockIdx.x * blockDim.x + threadIdx.x;
  if (bn >= n_bins) return;
  if (active && !active[bn]) return;
  int a = bn;
  if (active) {
    a = 0;
    for (int x = 0; x < bn; ++x) a += active[x] ? 1 : 0;
  }
  double acc = 0.0;
  for (int r = 0; r < n_q; ++r) acc = __dadd_rn(acc, rowmass[((size_t)b * n_q + r) * n_bins + bn]);
  raw[(size_t)b * n_out + a] = acc;
}

static size_t exact_ws_parts(int batch, int n_q, int hq, int items_stride, int n_bins, size_t* off_l,
                             size_t* off_rows) {
  const size_t part = align_up(sizeof(double) * (size_t)batch * n_q * hq * items_stride, 256);
  *off_l = part;
  *off_rows = 2 * part;
  return 2 * part + align_up(sizeof(double) * (size_t)batch * n_q * n_bins, 256);
}

template <typename KT, int RT, int G>
static int launch_exact_stats_g(const float* q, int batch, int n_q, int hq, int d, const void* k, int64_t k_bstride,
                                int hkv, const int32_t* seq_len, int s, const int64_t* q_pos, const int64_t* k_pos,
                                const int32_t* items, int items_stride, const int32_t* n_items, double scale,
                                double* pm, double* pl, cudaStream_t st) {
  const int row_tiles = (n_q + RT - 1) / RT;
  dim3 grid(items_stride, hkv, batch * row_tiles);
  const size_t smem = sizeof(double) * RT * G * d;
  auto kern = exact_stats_kernel<KT, RT, G>;
  if (smem > 48 * 1024) RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                                "exact_stats smem");
  kern<<<grid, kExThreads, smem, st>>>(q, n_q, hq, d, reinterpret_cast<const KT*>(k), k_bstride, hkv, seq_len, s,
                                       q_pos, k_pos, items, items_stride, n_items, scale, row_tiles, pm, pl);
  RK_CHECK_LAUNCH("exact_stats_kernel");
  return RK_OK;
}

template <typename KT, int RT>
static int launch_exact_stats(const float* q, int batch, int n_q, int hq, int d, const void* k, int64_t k_bstride,
                              int hkv, const int32_t* seq_len, int s, const int64_t* q_pos, const int64_t* k_pos,
                              const int32_t* items, int items_stride, const int32_t* n_items, double scale,
                              double* pm, double* pl, cudaStream_t st) {
#define RK_EXACT_G(GG)                                                                                          \
  case GG:                                                                                                      \
    return launch_exact_stats_g<KT, RT, GG>(q, batch, n_q, hq, d, k, k_bstride, hkv, seq_len, s, q_pos, k_pos,  \
                                            items, items_stride, n_items, scale, pm, pl, st);
  switch (hq / hkv) {
    RK_EXACT_G(1) RK_EXACT_G(2) RK_EXACT_G(3) RK_EXACT_G(4) RK_EXACT_G(5) RK_EXACT_G(6) RK_EXACT_G(7) RK_EXACT_G(8)
    default:
      return fail(RK_ERR_DOMAIN, "exact scoring: group %d", hq / hkv);
  }
#undef RK_EXACT_G
}

// bf16 keys with d 64 / 128 on the FP64 tensor pipe, 1-row (decode questions: 4 row tiles would
// waste 3/4 of the combos) or 4-row tiles (RK_EXACT_DMMA=0: the DFMA kernels)
static bool use_dmma(int kv_dtype, int n_q, int d, int G) {
  static const int mode = getenv("RK_EXACT_DMMA") ? atoi(getenv("RK_EXACT_DMMA")) : 1;
  return mode != 0 && kv_dtype == RK_BF16 && (d == 128 || d == 64) && G >= 1 && G <= 8;
}

template <int RT, int MT, int D>
static int launch_dmma_md(const float* q, int batch, int n_q, int hq, int G, const void* k, int64_t k_bstride,
                          int hkv, const int32_t* seq_len, int s, const int64_t* q_pos, const int64_t* k_pos,
                          const int32_t* items, int items_stride, const int32_t* n_items, double scale, double* pm,
                          double* pl, cudaStream_t st) {
  const int row_tiles = (n_q + RT - 1) / RT;
  dim3 grid(items_stride, hkv, batch * row_tiles);
  exact_stats_dmma_kernel<RT, MT, D><<<grid, kExThreads, 0, st>>>(
      q, n_q, hq, G, reinterpret_cast<const __nv_bfloat16*>(k), k_bstride, hkv, seq_len, s, q_pos, k_pos, items,
      items_stride, n_items, scale, row_tiles, pm, pl);
  RK_CHECK_LAUNCH("exact_stats_dmma_kernel");
  return RK_OK;
}

static int launch_exact_dmma(const float* q, int batch, int n_q, int hq, int d, const void* k, int64_t k_bstride,
                             int hkv, const int32_t* seq_len, int s, const int64_t* q_pos, const int64_t* k_pos,
                             const int32_t* items, int items_stride, const int32_t* n_items, double scale,
                             double* pm, double* pl, cudaStream_t st) {
  const int G = hq / hkv;
  if (n_q == 1) {
    if (d == 128) return launch_dmma_md<1, 1, 128>(q, batch, n_q, hq, G, k, k_bstride, hkv, seq_len, s, q_pos, k_pos,
                                                   items, items_stride, n_items, scale, pm, pl, st);
    return launch_dmma_md<1, 1, 64>(q, batch, n_q, hq, G, k, k_bstride, hkv, seq_len, s, q_pos, k_pos, items,
                                    items_stride, n_items, scale, pm, pl, st);
  }
  const int mt = (4 * G + 7) / 8;
#define RK_DM(MTV, DV)                                                                                             \
  if (mt == MTV && d == DV)                                                                                        \
    return launch_dmma_md<4, MTV, DV>(q, batch, n_q, hq, G, k, k_bstride, hkv, seq_len, s, q_pos, k_pos, items,     \
                                      items_stride, n_items, scale, pm, pl, st);
  RK_DM(1, 128) RK_DM(2, 128) RK_DM(3, 128) RK_DM(4, 128) RK_DM(1, 64) RK_DM(2, 64) RK_DM(3, 64) RK_DM(4, 64)
#undef RK_DM
  return fail(RK_ERR_DOMAIN, "exact scoring (dmma): group %d, d %d", G, d);
}

template <typename KT>
static int launch_exact_pre(const float* q, int batch, int n_q, int hq, int d, const void* k, int64_t k_bstride,
                            int hkv, const int32_t* seq_len, int s, const int64_t* q_pos, const int64_t* k_pos,
                            const int32_t* items, int items_stride, const int32_t* n_items, double denom, double* pm,
                            double* pl, cudaStream_t st) {
  constexpr int RT = 4;
  const int rt = n_q == 1 ? 1 : RT;
  const int row_tiles = (n_q + rt - 1) / rt;
  dim3 grid(items_stride, 1, batch * row_tiles);
  const size_t smem = sizeof(double) * rt * hq * d;
  if (smem > 200 * 1024) return fail(RK_ERR_DOMAIN, "exact pre scoring: %d heads x %d dims", hq, d);
  if (n_q == 1) {
    auto kern = exact_pre_stats_kernel<KT, 1>;
    if (smem > 48 * 1024)
      RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "exact_pre smem");
    kern<<<grid, kExThreads, smem, st>>>(q, n_q, hq, d, reinterpret_cast<const KT*>(k), k_bstride, hkv, seq_len, s,
                                         q_pos, k_pos, items, items_stride, n_items, denom, row_tiles, pm, pl);
  } else {
    auto kern = exact_pre_stats_kernel<KT, RT>;
    if (smem > 48 * 1024)
      RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "exact_pre smem");
    kern<<<grid, kExThreads, smem, st>>>(q, n_q, hq, d, reinterpret_cast<const KT*>(k), k_bstride, hkv, seq_len, s,
                                         q_pos, k_pos, items, items_stride, n_items, denom, row_tiles, pm, pl);
  }
  RK_CHECK_LAUNCH("exact_pre_stats_kernel");
  return RK_OK;
}

}  // namespace rk

using namespace rk;

extern "C" {

size_t rk_round_scores_exact_workspace_bytes(int batch, int n_q, int hq, int items_stride, int n_bins) {
  size_t a, b;
  return exact_ws_parts(batch, n_q, hq, items_stride, n_bins, &a, &b);
}

}  // extern "C"

namespace rk {

static int round_scores_exact_impl(int pre, const float* q, int batch, int n_q, int hq, int d, const void* k, int kv_dtype, int hkv,
                          int64_t k_batch_stride, const int32_t* seq_len, int s, const int64_t* q_pos,
                          const int64_t* k_pos, const int32_t* items, int items_stride, const int32_t* n_items,
                          int n_bins, const uint8_t* active, int n_out, double* raw_out, void* workspace,
                          size_t workspace_bytes, rk_stream_t stream) {
  if (batch <= 0 || n_q <= 0 || n_bins <= 0) return RK_OK;
  if (hkv <= 0 || hq % hkv != 0 || hq / hkv > kExMaxG)
    return fail(RK_ERR_DOMAIN, "exact scoring: %d query heads over %d kv-heads (group <= %d)", hq, hkv, kExMaxG);
  if (d <= 0 || d % 8 != 0 || d > 256) return fail(RK_ERR_DOMAIN, "exact scoring: head_dim %d (multiple of 8, <= 256)", d);
  if (kv_dtype != RK_F32 && kv_dtype != RK_BF16) return fail(RK_ERR_DOMAIN, "kv dtype %d", kv_dtype);
  if (items == nullptr || items_stride <= 0 || q_pos == nullptr || raw_out == nullptr)
    return fail(RK_ERR_DOMAIN, "exact scoring needs items, q_pos and raw_out");
  size_t off_l, off_rows;
  const size_t need = exact_ws_parts(batch, n_q, hq, items_stride, n_bins, &off_l, &off_rows);
  if (workspace_bytes < need) return fail(RK_ERR_CAPACITY, "exact scoring workspace %zu < %zu", workspace_bytes, need);
  char* ws = reinterpret_cast<char*>(workspace);
  double* pm = reinterpret_cast<double*>(ws);
  double* pl = reinterpret_cast<double*>(ws + off_l);
  double* rows = reinterpret_cast<double*>(ws + off_rows);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double scale = 1.0 / sqrt((double)d);        // the reference's inv_scale (_attn_ext.pyx:36)
  int rc;
  if (pre) {
    const double denom = (double)hq * sqrt((double)d);   // num_heads * sqrt(d_k) (engine.py:191)
    rc = kv_dtype == RK_BF16
             ? launch_exact_pre<__nv_bfloat16>(q, batch, n_q, hq, d, k, k_batch_stride, hkv, seq_len, s, q_pos, k_pos,
                                               items, items_stride, n_items, denom, pm, pl, st)
             : launch_exact_pre<float>(q, batch, n_q, hq, d, k, k_batch_stride, hkv, seq_len, s, q_pos, k_pos, items,
                                       items_stride, n_items, denom, pm, pl, st);
  } else if (use_dmma(kv_dtype, n_q, d, hq / hkv)) {
    rc = launch_exact_dmma(q, batch, n_q, hq, d, k, k_batch_stride, hkv, seq_len, s, q_pos, k_pos, items,
                           items_stride, n_items, scale, pm, pl, st);
  } else if (kv_dtype == RK_BF16)
    rc = n_q == 1 ? launch_exact_stats<__nv_bfloat16, 1>(q, batch, n_q, hq, d, k, k_batch_stride, hkv, seq_len, s,
                                                         q_pos, k_pos, items, items_stride, n_items, scale, pm, pl, st)
                  : launch_exact_stats<__nv_bfloat16, 4>(q, batch, n_q, hq, d, k, k_batch_stride, hkv, seq_len, s,
                                                         q_pos, k_pos, items, items_stride, n_items, scale, pm, pl, st);
  else
    rc = n_q == 1 ? launch_exact_stats<float, 1>(q, batch, n_q, hq, d, k, k_batch_stride, hkv, seq_len, s, q_pos,
                                                 k_pos, items, items_stride, n_items, scale, pm, pl, st)
                  : launch_exact_stats<float, 4>(q, batch, n_q, hq, d, k, k_batch_stride, hkv, seq_len, s, q_pos,
                                                 k_pos, items, items_stride, n_items, scale, pm, pl, st);
  if (rc != RK_OK) return rc;
  const int heads = pre ? 1 : hq;          // "pre": one softmax per row
  const size_t smem = sizeof(double) * (n_bins + 1 + 2 * heads) + sizeof(int) * (n_bins + 2);
  if (smem > 48 * 1024) {
    RK_CUDA(cudaFuncSetAttribute(exact_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
            "exact_rows smem");
  }
  exact_rows_kernel<<<batch * n_q, 128, smem, st>>>(pm, pl, n_q, heads, items, items_stride, n_items, n_bins, rows);
  RK_CHECK_LAUNCH("exact_rows_kernel");
  dim3 g2((n_bins + 127) / 128, batch);
  exact_sum_rows_kernel<<<g2, 128, 0, st>>>(rows, n_q, n_bins, active, n_out, raw_out);
  RK_CHECK_LAUNCH("exact_sum_rows_kernel");
  return RK_OK;
}

}  // namespace rk

extern "C" {

int rk_round_scores_exact(const float* q, int batch, int n_q, int hq, int d, const void* k, int kv_dtype, int hkv,
                          int64_t k_batch_stride, const int32_t* seq_len, int s, const int64_t* q_pos,
                          const int64_t* k_pos, const int32_t* items, int items_stride, const int32_t* n_items,
                          int n_bins, const uint8_t* active, int n_out, double* raw_out, void* workspace,
                          size_t workspace_bytes, rk_stream_t stream) {
  return round_scores_exact_impl(0, q, batch, n_q, hq, d, k, kv_dtype, hkv, k_batch_stride, seq_len, s, q_pos, k_pos,
                                 items, items_stride, n_items, n_bins, active, n_out, raw_out, workspace,
                                 workspace_bytes, stream);
}

int rk_round_scores_exact_pre(const float* q, int batch, int n_q, int hq, int d, const void* k, int kv_dtype, int hkv,
                              int64_t k_batch_stride, const int32_t* seq_len, int s, const int64_t* q_pos,
                              const int64_t* k_pos, const int32_t* items, int items_stride, const int32_t* n_items,
                              int n_bins, const uint8_t* active, int n_out, double* raw_out, void* workspace,
                              size_t workspace_bytes, rk_stream_t stream) {
  return round_scores_exact_impl(1, q, batch, n_q, hq, d, k, kv_dtype, hkv, k_batch_stride, seq_len, s, q_pos, k_pos,
                                 items, items_stride, n_items, n_bins, active, n_out, raw_out, workspace,
                                 workspace_bytes, stream);
}

}  // extern "C"
