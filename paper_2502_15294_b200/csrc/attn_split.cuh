// Split-K attention over work items, shared by
//   * rk_decode_attention  — batched single-token decode over a contiguous,
//     round-spliced KV cache [S][Hkv][D] per dialogue;
//   * rk_attention_forward — the reference kernel contract (rows x keys with
//     causal positions and an `allowed` mask, _attn_ext.pyx:20-81);
//   * rk_round_scores      — the same pass with round-aligned work items whose
//     per-(row, head, item) softmax statistics feed the Eq. 1 round masses
//     (stats.py:59-94) without materialising the capture matrix.
//
// One CTA = (work item x, row y, kv-head z).  It streams its key range once
// with 128-bit loads, keeps G = Hq/Hkv query heads' online-softmax state in
// registers (scores in log2 units), reduces across warps through shared
// memory, writes its partial (m, l, acc[D]) and the last CTA of (row, kv-head)
// merges all partials into the fp32 output (self-resetting counter).
#pragma once

#include "rk_common.cuh"

namespace rk {

constexpr int kWarps = 4;
constexpr int kThreads = kWarps * 32;

struct SplitParams {
  const float* q;             // [rows][hq][d]
  const void* k;              // key rows, element (j, kvh, e) at k + b*batch_stride + j*row_stride + kvh*d + e
  const void* v;
  int64_t row_stride;         // hkv * d
  int64_t batch_stride;       // decode: elements between dialogues; general: 0
  const int32_t* seq_len;     // decode: keys cached before this token, per dialogue (device); null -> s_static
  int s_static;
  void* k_new;                // decode append: [rows][hkv][d] (same dtype as cache) or null
  void* v_new;
  const int64_t* q_pos;       // general mode masks (null in decode mode)
  const int64_t* k_pos;
  const uint8_t* allowed;
  const int32_t* items;       // [items_stride * rows or 1][3] = (lo, hi, bin) or null -> uniform split
  const int32_t* n_items;     // per item-table count (device) or null (-> gridDim.x)
  int items_row_stride;       // item-table stride per row (0: shared table)
  int rows, hq, hkv, d;
  float scale_log2;           // log2(e) / sqrt(d)
  float* out;                 // [rows][hq][d]
  float* part_m;              // [rows][hq][gridDim.x]
  float* part_l;
  float* part_acc;            // [rows][hq][gridDim.x][d]
  unsigned* counters;         // [rows][hkv], zero at rest
  int32_t* bad_row;           // atomicMin of rows with no visible key (general mode), or null
  float* stat_m;              // [rows][hq] merged log2-domain max (capture path) or null
  float* stat_l;              // [rows][hq] merged sum of exp2(s - m) or null
};

// SCORE: statistics only (no V, no output, no merge): part_m/part_l per item.
template <typename T, int G, int LPK, int NCH, bool VEC, int U, bool DECODE, bool SCORE>
__global__ void __launch_bounds__(kThreads, 2) attn_split_kernel(SplitParams p) {
  constexpr int KPW = 32 / LPK;                  // keys per warp instruction
  constexpr int EPL = VEC ? NCH * 8 : NCH;       // elements per lane
  constexpr int TILE = kWarps * KPW * U;         // keys per CTA iteration
  static_assert(!VEC || EPL % 2 == 0, "vector path works on float2 pairs");

  const int item = blockIdx.x, row = blockIdx.y, kvh = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LPK, gl = lane % LPK;
  const int d = p.d;

  // ---- key range of this CTA
  int n_eff = gridDim.x;
  int len;
  int64_t base = 0;
  if (DECODE) {
    base = (int64_t)row * p.batch_stride;
    len = (p.seq_len ? p.seq_len[row] : p.s_static) + (p.k_new ? 1 : 0);
  } else {
    len = p.s_static;
  }
  int lo, hi;
  if (p.items) {
    const int32_t* tab = p.items + (size_t)row * p.items_row_stride * 3;
    n_eff = p.n_items ? p.n_items[p.items_row_stride ? row : 0] : gridDim.x;
    if (item >= n_eff) return;                   // not counted by the merge
    lo = tab[item * 3 + 0];
    hi = min(tab[item * 3 + 1], len);
  } else {
    int per = (len + gridDim.x - 1) / gridDim.x;
    per = (per + TILE - 1) / TILE * TILE;
    lo = min(len, item * per);
    hi = min(len, lo + per);
  }
  int new_idx = (DECODE && p.k_new) ? len - 1 : -1;     // appended key index

  const T* K = reinterpret_cast<const T*>(p.k) + base + (int64_t)kvh * d;
  const T* V = reinterpret_cast<const T*>(p.v) + base + (int64_t)kvh * d;
  const T* Kn = DECODE && p.k_new ? reinterpret_cast<const T*>(p.k_new) + ((int64_t)row * p.hkv + kvh) * d : nullptr;
  const T* Vn = DECODE && p.k_new ? reinterpret_cast<const T*>(p.v_new) + ((int64_t)row * p.hkv + kvh) * d : nullptr;

  // ---- queries (pre-scaled into log2 units)
  const int h0 = kvh * G;
  int64_t qpos = 0;
  if (!DECODE) qpos = p.q_pos[row];
  float2 q2[G][VEC ? EPL / 2 : 1];
  float qs[G][VEC ? 1 : EPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float* qp = p.q + ((int64_t)row * p.hq + h0 + g) * d;
    if constexpr (VEC) {
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int e = (c * LPK + gl) * 8 + 2 * i;
          q2[g][c * 4 + i] = make_float2(qp[e] * p.scale_log2, qp[e + 1] * p.scale_log2);
        }
    } else {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        int e = c * 32 + gl;
        qs[g][c] = e < d ? qp[e] * p.scale_log2 : 0.f;
      }
    }
  }

  // ---- per-lane online-softmax state for the keys of this lane's group
  float m[G], l[G];
  float2 acc2[G][VEC ? EPL / 2 : 1];
  float accs[G][VEC ? 1 : EPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int i = 0; i < (VEC ? EPL / 2 : 1); ++i) acc2[g][i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < (VEC ? 1 : EPL); ++i) accs[g][i] = 0.f;
  }

  for (int tile = lo; tile < hi; tile += TILE) {
    float s[U][G];
    float2 kv2[U][VEC ? EPL / 2 : 1], vv2[U][VEC ? EPL / 2 : 1];
    float ks[U][VEC ? 1 : EPL], vs[U][VEC ? 1 : EPL];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = tile + (warp * U + u) * KPW + grp;
      bool vis = j < hi;
      if (!DECODE && vis) {
        vis = p.k_pos[j] <= qpos && (p.allowed == nullptr || p.allowed[j]);
      }
      ok[u] = vis;
      const T* kr = (j == new_idx) ? Kn : K + (int64_t)j * p.row_stride;
      const T* vr = (j == new_idx) ? Vn : V + (int64_t)j * p.row_stride;
      if constexpr (VEC) {
        if (vis) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            float2 t[4];
            KV<T>::load8(kr + (c * LPK + gl) * 8, t);
#pragma unroll
            for (int i = 0; i < 4; ++i) kv2[u][c * 4 + i] = t[i];
            if constexpr (!SCORE) {
              KV<T>::load8(vr + (c * LPK + gl) * 8, t);
#pragma unroll
              for (int i = 0; i < 4; ++i) vv2[u][c * 4 + i] = t[i];
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < EPL / 2; ++i) kv2[u][i] = vv2[u][i] = make_float2(0.f, 0.f);
        }
      } else {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          int e = c * 32 + gl;
          bool in = vis && e < d;
          ks[u][c] = in ? KV<T>::get(kr, e) : 0.f;
          vs[u][c] = (in && !SCORE) ? KV<T>::get(vr, e) : 0.f;
        }
      }
    }
    // scores
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float dot;
        if constexpr (VEC) {
          float2 a = make_float2(0.f, 0.f);
#pragma unroll
          for (int i = 0; i < EPL / 2; ++i) a = ffma2(q2[g][i], kv2[u][i], a);
          dot = a.x + a.y;
        } else {
          dot = 0.f;
#pragma unroll
          for (int c = 0; c < NCH; ++c) dot = fmaf(qs[g][c], ks[u][c], dot);
        }
        dot = group_sum<LPK>(dot);
        s[u][g] = ok[u] ? dot : -INFINITY;
      }
    }
    // online softmax update + PV
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mx = m[g];
#pragma unroll
      for (int u = 0; u < U; ++u) mx = fmaxf(mx, s[u][g]);
      float mu = (mx == -INFINITY) ? 0.f : mx;
      float corr = fast_exp2(m[g] - mu);
      m[g] = mx;
      float lsum = l[g] * corr;
      if constexpr (SCORE) {
#pragma unroll
        for (int u = 0; u < U; ++u) lsum += fast_exp2(s[u][g] - mu);
        l[g] = lsum;
        continue;
      }
      if constexpr (VEC) {
        float2 c2 = make_float2(corr, corr);
#pragma unroll
        for (int i = 0; i < EPL / 2; ++i) acc2[g][i] = fmul2(acc2[g][i], c2);
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) accs[g][i] *= corr;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float pr = fast_exp2(s[u][g] - mu);
        lsum += pr;
        if constexpr (VEC) {
          float2 p2 = make_float2(pr, pr);
#pragma unroll
          for (int i = 0; i < EPL / 2; ++i) acc2[g][i] = ffma2(p2, vv2[u][i], acc2[g][i]);
        } else {
#pragma unroll
          for (int i = 0; i < EPL; ++i) accs[g][i] = fmaf(pr, vs[u][i], accs[g][i]);
        }
      }
      l[g] = lsum;
    }
  }

  // ---- combine the KPW key groups of each warp (lanes with equal gl)
#pragma unroll
  for (int o = LPK; o < 32; o <<= 1) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mo = __shfl_xor_sync(0xffffffffu, m[g], o);
      float lo_ = __shfl_xor_sync(0xffffffffu, l[g], o);
      float mx = fmaxf(m[g], mo);
      float mu = (mx == -INFINITY) ? 0.f : mx;
      float ca = fast_exp2(m[g] - mu), cb = fast_exp2(mo - mu);
      m[g] = mx;
      l[g] = l[g] * ca + lo_ * cb;
      if constexpr (SCORE) continue;
      if constexpr (VEC) {
#pragma unroll
        for (int i = 0; i < EPL / 2; ++i) {
          float2 a = acc2[g][i];
          float2 b;
          b.x = __shfl_xor_sync(0xffffffffu, a.x, o);
          b.y = __shfl_xor_sync(0xffffffffu, a.y, o);
          acc2[g][i] = make_float2(a.x * ca + b.x * cb, a.y * ca + b.y * cb);
        }
      } else {
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          float b = __shfl_xor_sync(0xffffffffu, accs[g][i], o);
          accs[g][i] = accs[g][i] * ca + b * cb;
        }
      }
    }
  }

  // ---- combine warps through shared memory, write this CTA's partial
  extern __shared__ float smem[];
  float* sm_m = smem;                           // [kWarps][G]
  float* sm_l = sm_m + kWarps * G;              // [kWarps][G]
  float* sm_acc = sm_l + kWarps * G;            // [kWarps][G][d]
  if (grp == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (gl == 0) {
        sm_m[warp * G + g] = m[g];
        sm_l[warp * G + g] = l[g];
      }
      float* dst = sm_acc + (warp * G + g) * d;
      if constexpr (SCORE) continue;
      if constexpr (VEC) {
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            int e = (c * LPK + gl) * 8 + 2 * i;
            dst[e] = acc2[g][c * 4 + i].x;
            dst[e + 1] = acc2[g][c * 4 + i].y;
          }
      } else {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          int e = c * 32 + gl;
          if (e < d) dst[e] = accs[g][c];
        }
      }
    }
  }
  __syncthreads();

  const int nsplit = gridDim.x;
  if constexpr (SCORE) {
    if (threadIdx.x < G) {
      int g = threadIdx.x;
      float mx = -INFINITY;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) mx = fmaxf(mx, sm_m[w * G + g]);
      float mu = (mx == -INFINITY) ? 0.f : mx;
      float ls = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) ls += sm_l[w * G + g] * fast_exp2(sm_m[w * G + g] - mu);
      int64_t slot = ((int64_t)row * p.hq + h0 + g) * nsplit + item;
      p.part_m[slot] = mx;
      p.part_l[slot] = ls;
    }
    return;
  }
  for (int idx = threadIdx.x; idx < G * d; idx += kThreads) {
    int g = idx / d, e = idx - g * d;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) mx = fmaxf(mx, sm_m[w * G + g]);
    float mu = (mx == -INFINITY) ? 0.f : mx;
    float ls = 0.f, as = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      float c = fast_exp2(sm_m[w * G + g] - mu);
      ls += sm_l[w * G + g] * c;
      as += sm_acc[(w * G + g) * d + e] * c;
    }
    int64_t slot = ((int64_t)row * p.hq + h0 + g) * nsplit + item;
    p.part_acc[slot * d + e] = as;
    if (e == 0) {
      p.part_m[slot] = mx;
      p.part_l[slot] = ls;
    }
  }

  // decode append: the CTA that owns the appended key writes it into the cache
  if (DECODE && p.k_new && new_idx >= lo && new_idx < hi) {
    T* kd = const_cast<T*>(K) + (int64_t)new_idx * p.row_stride;
    T* vd = const_cast<T*>(V) + (int64_t)new_idx * p.row_stride;
    for (int e = threadIdx.x; e < d; e += kThreads) {
      kd[e] = Kn[e];
      vd[e] = Vn[e];
    }
  }

  // ---- last CTA of (row, kvh) merges all partials
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* ctr = p.counters + (int64_t)row * p.hkv + kvh;
    unsigned prev = atomicAdd(ctr, 1u);
    s_last = (prev + 1 == (unsigned)n_eff);
    if (s_last) *ctr = 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  for (int idx = threadIdx.x; idx < G * d; idx += kThreads) {
    int g = idx / d, e = idx - g * d;
    int64_t slot0 = ((int64_t)row * p.hq + h0 + g) * nsplit;
    float mx = -INFINITY;
    for (int it = 0; it < n_eff; ++it) mx = fmaxf(mx, __ldcg(p.part_m + slot0 + it));
    float out;
    if (mx == -INFINITY) {
      out = 0.f;
      if (p.bad_row && e == 0) atomicMin(p.bad_row, row);
    } else {
      float ls = 0.f, as = 0.f;
      for (int it = 0; it < n_eff; ++it) {
        float c = fast_exp2(__ldcg(p.part_m + slot0 + it) - mx);
        ls += __ldcg(p.part_l + slot0 + it) * c;
        as += __ldcg(p.part_acc + (slot0 + it) * d + e) * c;
      }
      out = as / ls;
      if (p.stat_m && e == 0) {
        p.stat_m[(int64_t)row * p.hq + h0 + g] = mx;
        p.stat_l[(int64_t)row * p.hq + h0 + g] = ls;
      }
    }
    p.out[((int64_t)row * p.hq + h0 + g) * d + e] = out;
  }
}

}  // namespace rk
