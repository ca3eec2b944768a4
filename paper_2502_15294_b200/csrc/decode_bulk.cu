// Pipelined split-K decode attention over round-spliced caches (the sparse
// decode hot loop, pipeline.py:298-313 -> engine.py:244-267 with one row).
//
// Layout: dialogue b's cache is [S_cap][HKV][D] (token-major), so the keys
// [j0, j0+TK) of ALL kv-heads are one contiguous run of TK*HKV*D elements.
// A CTA = (split, dialogue) streams its key range through shared memory:
//   warp 8      producer: one elected lane issues two cp.async.bulk copies
//               (K tile, V tile) per stage into a STAGES-deep ring guarded by
//               full/empty mbarriers (complete_tx byte counting);
//   warps 0..7  consumers: warp w owns kv-head w % HKV (8/HKV warps per head
//               split the tile's keys); LPK=8 lanes per key, 128-bit LDS,
//               FFMA2 dot products, online softmax in log2 units, FFMA2 PV.
// Partials (m, l, acc[D]) per (dialogue, q-head, split) go to global memory;
// decode_merge_kernel combines them.  Both kernels are launched with
// programmatic dependent launch: the next layer's CTAs initialise barriers and
// start prefetching K/V tiles while the previous merge is still running, and
// wait (griddepcontrol.wait) only before touching q / the workspace.
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <type_traits>

#include "decode_common.cuh"

namespace rk {

template <typename T>
__device__ __forceinline__ void lds8(const T* p, float2 (&out)[4]);
template <>
__device__ __forceinline__ void lds8<__nv_bfloat16>(const __nv_bfloat16* p, float2 (&out)[4]) {
  uint4 a = *reinterpret_cast<const uint4*>(p);
  out[0] = bf16x2_to_f2(a.x);
  out[1] = bf16x2_to_f2(a.y);
  out[2] = bf16x2_to_f2(a.z);
  out[3] = bf16x2_to_f2(a.w);
}
template <>
__device__ __forceinline__ void lds8<float>(const float* p, float2 (&out)[4]) {
  float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  out[0] = make_float2(a.x, a.y);
  out[1] = make_float2(a.z, a.w);
  out[2] = make_float2(b.x, b.y);
  out[3] = make_float2(b.z, b.w);
}

template <typename T, int D, int G, int HKV>
__global__ void __launch_bounds__(kBulkThreads, 1) decode_bulk_kernel(const __grid_constant__ BulkParams p) {
  // lanes per key: D/8 (8 elements = one 16-byte bf16 load per lane).  With 9
  // warps one SMSP hosts 3 warps, capping registers at 168/thread; 8 elements
  // per lane keeps q + acc for G <= 8 query heads in registers.
  constexpr int LPK = D / 8;
  constexpr int KPW = 32 / LPK;                   // keys per warp instruction
  constexpr int ROW = HKV * D;                    // elements per key (all heads)
  constexpr int TK = kStageBytes / (ROW * (int)sizeof(T));
  constexpr int P = kConsumerWarps / HKV;         // warps per kv-head
  constexpr int U = G <= 4 ? 4 : 2;               // keys per lane per softmax update
  constexpr int GROUPS = TK / KPW;                // key groups per tile
  static_assert(TK >= KPW && TK % KPW == 0, "tile must hold whole key groups");
  static_assert(kConsumerWarps % HKV == 0, "kv heads must divide the consumer warps");

  extern __shared__ __align__(128) uint8_t smem[];
  T* kst = reinterpret_cast<T*>(smem);
  T* vst = reinterpret_cast<T*>(smem + kStages * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  T* newrow = reinterpret_cast<T*>(empty + kStages);   // [2][ROW] appended K,V row
  __shared__ SegTable segs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool append = p.k_new != nullptr;
  compute_segments(p, segs);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const Seg* s_seg = segs.seg;
  const int nseg = segs.nseg;
  const int slot_base = (p.items ? blockIdx.x : blockIdx.x) * P;

  if (warp == kConsumerWarps) {
    // ================= producer: one lane streams every tile of every segment
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int t = 0;
      for (int sg = 0; sg < nseg; ++sg) {
        const Seg sgm = s_seg[sg];
        const int len = p.seq_len[sgm.b] + (append ? 1 : 0);
        const int chi = append ? min(sgm.hi, len - 1) : sgm.hi;
        const T* kb = reinterpret_cast<const T*>(p.k) + (int64_t)sgm.b * p.batch_stride;
        const T* vb = reinterpret_cast<const T*>(p.v) + (int64_t)sgm.b * p.batch_stride;
        for (int j0 = sgm.lo; j0 < chi; j0 += TK, ++t) {
          const int s = t % kStages;
          if (t >= kStages) mbar_wait(&empty[s], ((t / kStages) - 1) & 1);
          const unsigned bytes = (unsigned)(min(TK, chi - j0) * ROW * sizeof(T));
          mbar_expect_tx(&full[s], 2 * bytes);
          bulk_g2s(kst + (size_t)s * (kStageBytes / sizeof(T)), kb + (int64_t)j0 * ROW, bytes, &full[s], pol);
          bulk_g2s(vst + (size_t)s * (kStageBytes / sizeof(T)), vb + (int64_t)j0 * ROW, bytes, &full[s], pol);
        }
      }
    }
    return;
  }

  // ================= consumers
  pdl_wait();   // q and the workspace belong to the previous kernels until here
  const int h = warp % HKV, slice = warp / HKV;
  const int grp = lane / LPK, gl = lane % LPK;
  const int h0 = h * G;
  int t = 0;

  for (int sg = 0; sg < nseg; ++sg) {
    const Seg sgm = s_seg[sg];
    const int b = sgm.b;
    const int len = p.seq_len[b] + (append ? 1 : 0);
    const int chi = append ? min(sgm.hi, len - 1) : sgm.hi;
    const bool owns_new = append && sgm.hi == len;
    if (owns_new) {   // stage the appended row (all heads) in smem and write it to the cache
      const T* kn = reinterpret_cast<const T*>(p.k_new) + (int64_t)b * ROW;
      const T* vn = reinterpret_cast<const T*>(p.v_new) + (int64_t)b * ROW;
      T* kd = reinterpret_cast<T*>(const_cast<void*>(p.k)) + (int64_t)b * p.batch_stride + (int64_t)(len - 1) * ROW;
      T* vd = reinterpret_cast<T*>(const_cast<void*>(p.v)) + (int64_t)b * p.batch_stride + (int64_t)(len - 1) * ROW;
      for (int e = threadIdx.x; e < ROW; e += kConsumerWarps * 32) {
        T kv = kn[e], vv = vn[e];
        newrow[e] = kv;
        newrow[ROW + e] = vv;
        kd[e] = kv;
        vd[e] = vv;
      }
      consumer_sync();
    }

    float2 q2[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float* qp = p.q + ((int64_t)b * p.hq + h0 + g) * D + gl * 8;
      const float4 a = *reinterpret_cast<const float4*>(qp);
      const float4 bq = *reinterpret_cast<const float4*>(qp + 4);
      q2[g][0] = make_float2(a.x * p.scale_log2, a.y * p.scale_log2);
      q2[g][1] = make_float2(a.z * p.scale_log2, a.w * p.scale_log2);
      q2[g][2] = make_float2(bq.x * p.scale_log2, bq.y * p.scale_log2);
      q2[g][3] = make_float2(bq.z * p.scale_log2, bq.w * p.scale_log2);
    }
    float m[G], l[G];
    float2 acc[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m[g] = -INFINITY;
      l[g] = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[g][i] = make_float2(0.f, 0.f);
    }

    // NU keys per lane-group (rows krow[u]/vrow[u], validity ok[u]): scores for
    // G heads, one rescale per update, PV with FFMA2
    auto update = [&](const T* const* krow, const T* const* vrow, const bool* ok, auto nu_tag) {
      constexpr int NU = decltype(nu_tag)::value;
      float2 kk[NU][4], vv[NU][4];
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        lds8<T>(krow[u] + gl * 8, kk[u]);
        lds8<T>(vrow[u] + gl * 8, vv[u]);
      }
      float s[NU][G];
#pragma unroll
      for (int u = 0; u < NU; ++u)
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float2 a = fmul2(q2[g][0], kk[u][0]);
#pragma unroll
          for (int i = 1; i < 4; ++i) a = ffma2(q2[g][i], kk[u][i], a);
          const float dot = group_sum<LPK>(a.x + a.y);   // every lane shuffles (sync mask)
          s[u][g] = ok[u] ? dot : -INFINITY;
        }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float mx = m[g];
#pragma unroll
        for (int u = 0; u < NU; ++u) mx = fmaxf(mx, s[u][g]);
        const float mu = (mx == -INFINITY) ? 0.f : mx;
        const float corr = fast_exp2(m[g] - mu);
        m[g] = mx;
        float ls = l[g] * corr;
        const float2 c2 = make_float2(corr, corr);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[g][i] = fmul2(acc[g][i], c2);
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const float pr = fast_exp2(s[u][g] - mu);
          ls += pr;
          const float2 p2 = make_float2(pr, pr);
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[g][i] = ffma2(p2, vv[u][i], acc[g][i]);
        }
        l[g] = ls;
      }
    };

    for (int j0 = sgm.lo; j0 < chi; j0 += TK, ++t) {
      const int s = t % kStages;
      mbar_wait(&full[s], (t / kStages) & 1);
      const int nk = min(TK, chi - j0);
      const T* ks = kst + (size_t)s * (kStageBytes / sizeof(T)) + h * D;
      const T* vs = vst + (size_t)s * (kStageBytes / sizeof(T)) + h * D;
      // this warp's key groups: slice, slice + P, ...  processed U at a time
      for (int gi = slice; gi < GROUPS; gi += P * U) {
        const T* kr[U];
        const T* vr[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int key = (gi + u * P) * KPW + grp;
          ok[u] = (gi + u * P) < GROUPS && key < nk;
          const int kc = ok[u] ? key : 0;
          kr[u] = ks + kc * ROW;
          vr[u] = vs + kc * ROW;
        }
        update(kr, vr, ok, std::integral_constant<int, U>{});
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (owns_new && slice == 0) {
      const T* kr[1] = {newrow + h * D};
      const T* vr[1] = {newrow + ROW + h * D};
      const bool ok[1] = {grp == 0};
      update(kr, vr, ok, std::integral_constant<int, 1>{});
    }

    // ---- combine the key groups of the warp, write this warp's partial slot
#pragma unroll
    for (int o = LPK; o < 32; o <<= 1) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float mo = __shfl_xor_sync(0xffffffffu, m[g], o);
        const float lo2 = __shfl_xor_sync(0xffffffffu, l[g], o);
        const float mx = fmaxf(m[g], mo);
        const float mu = (mx == -INFINITY) ? 0.f : mx;
        const float ca = fast_exp2(m[g] - mu), cb = fast_exp2(mo - mu);
        m[g] = mx;
        l[g] = l[g] * ca + lo2 * cb;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float2 bo;
          bo.x = __shfl_xor_sync(0xffffffffu, acc[g][i].x, o);
          bo.y = __shfl_xor_sync(0xffffffffu, acc[g][i].y, o);
          acc[g][i] = make_float2(acc[g][i].x * ca + bo.x * cb, acc[g][i].y * ca + bo.y * cb);
        }
      }
    }
    if (grp == 0) {
      const int slot = slot_base + slice;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int64_t sl = ((int64_t)b * p.hq + h0 + g) * p.nsplit + slot;
        float4* dst = reinterpret_cast<float4*>(p.part_acc + sl * D + gl * 8);
        dst[0] = make_float4(acc[g][0].x, acc[g][0].y, acc[g][1].x, acc[g][1].y);
        dst[1] = make_float4(acc[g][2].x, acc[g][2].y, acc[g][3].x, acc[g][3].y);
        if (gl == 0) {
          p.part_m[sl] = m[g];
          p.part_l[sl] = l[g];
        }
      }
    }
    if (owns_new) consumer_sync();   // newrow is reused by a later segment
  }
  pdl_trigger();
}

// Merge the partial slots of (dialogue b, q-head h):
//   out = sum_s acc_s 2^(m_s - M) / sum_s l_s 2^(m_s - M).
// Uniform mode recomputes which CTAs overlapped dialogue b from the lengths
// (same flattened partition as the decode kernels); their slots are
// contiguous.  Item mode uses n_items[b].  8 warps split the slots, lanes own
// 4 consecutive dims, 4 slots' loads are issued together.
// advance (nullable): advance[b] += 1 (lengths of the next step).
// NW warps per (dialogue, head): 4 when the grid is large (fits beside a
// resident decode CTA); 16 for small batches, where only B*hq blocks exist and
// each must fetch its ~150 partials in one round of loads, not ten.
template <int NW>
__global__ void __launch_bounds__(NW * 32) decode_merge_kernel(const float* __restrict__ part_m,
                                                           const float* __restrict__ part_l,
                                                           const float* __restrict__ part_acc,
                                                           const int32_t* __restrict__ seq_len, int append,
                                                           const int32_t* __restrict__ n_items, int B, int nsplit,
                                                           int slices, int ncta, int hq, int d,
                                                           float* __restrict__ out, int32_t* advance) {
  // the next kernel may start its prologue (reads seq_len, prefetches K/V)
  // while this merge runs — unless this merge advances the lengths: then the
  // trigger is the implicit one at exit, after the increment
  if (advance == nullptr) pdl_trigger();
  pdl_wait();
  const int b = blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int s_c0, s_c1, s_sparse;
  __shared__ int64_t s_W, s_P0, s_P1;
  __shared__ float s_red[NW];
  __shared__ __align__(16) float s_acc[NW][256];
  __shared__ float s_l[NW];
  if (n_items) {
    if (threadIdx.x == 0) { s_c0 = 0; s_c1 = n_items[b] - 1; s_sparse = 0; }
  } else {
    int64_t before = 0, all = 0;
    for (int i = threadIdx.x; i < B; i += blockDim.x) {
      const int64_t L = seq_len[i] + append;
      all += L;
      if (i < b) before += L;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    __shared__ int64_t red[2][NW];
    if (lane == 0) { red[0][warp] = before; red[1][warp] = all; }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t P0 = 0, W = 0;
      for (int w = 0; w < NW; ++w) { P0 += red[0][w]; W += red[1][w]; }
      const int64_t P1 = P0 + seq_len[b] + append, N = ncta;
      s_W = W; s_P0 = P0; s_P1 = P1;
      s_c0 = W > 0 ? (int)min((long long)(N - 1), (long long)(((P0 + 1) * N - 1) / W)) : 0;
      s_c1 = W > 0 ? (int)min((long long)(N - 1), (long long)((P1 * N - 1) / W)) : -1;
      s_sparse = W < N;          // some CTAs own empty ranges: check each slot
    }
  }
  __syncthreads();
  const int c0 = s_c0, c1 = s_c1, sparse = s_sparse;
  const int64_t base = ((int64_t)b * hq + h) * nsplit + (int64_t)c0 * slices;
  const int nslot = (c1 - c0 + 1) * slices;
  auto live = [&](int k) {
    if (!sparse) return true;
    const int64_t c = c0 + k / slices;
    const int64_t r0 = c * s_W / ncta, r1 = (c + 1) * s_W / ncta;
    return max(r0, s_P0) < min(r1, s_P1);
  };
  float mx = -INFINITY;
  for (int k = threadIdx.x; k < nslot; k += blockDim.x)
    if (live(k)) mx = fmaxf(mx, part_m[base + k]);
  mx = group_max<32>(mx);
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < NW; ++w) M = fmaxf(M, s_red[w]);
  const float mu = (M == -INFINITY) ? 0.f : M;
  float ls = 0.f;
  float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
  const bool d0 = lane * 4 < d, d1 = lane * 4 + 128 < d;
  for (int k0 = warp; k0 < nslot; k0 += 4 * NW) {
    float wgt[4], lv[4];
    float4 v0[4], v1[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + u * NW;
      const bool ok = k < nslot && live(k);
      const int64_t sl = base + (ok ? k : 0);
      wgt[u] = ok ? part_m[sl] : -INFINITY;
      lv[u] = ok ? part_l[sl] : 0.f;
      const float4* src = reinterpret_cast<const float4*>(part_acc + sl * d);
      v0[u] = (ok && d0) ? src[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
      v1[u] = (ok && d1) ? src[lane + 32] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float w = fast_exp2(wgt[u] - mu);
      ls += lv[u] * w;
      a0.x += v0[u].x * w; a0.y += v0[u].y * w; a0.z += v0[u].z * w; a0.w += v0[u].w * w;
      a1.x += v1[u].x * w; a1.y += v1[u].y * w; a1.z += v1[u].z * w; a1.w += v1[u].w * w;
    }
  }
  if (lane == 0) s_l[warp] = ls;
  if (d0) *reinterpret_cast<float4*>(&s_acc[warp][lane * 4]) = a0;
  if (d1) *reinterpret_cast<float4*>(&s_acc[warp][lane * 4 + 128]) = a1;
  __syncthreads();
  float L = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) L += s_l[w];
  const float inv = 1.f / L;
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    float as = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) as += s_acc[w][e];
    out[((int64_t)b * hq + h) * d + e] = as * inv;
  }
  if (advance && h == 0 && threadIdx.x == 0) advance[b] += 1;
}

// ------------------------------------------------------------------ host side
template <typename T, int D, int G, int HKV>
static cudaError_t launch_bulk(dim3 grid, cudaStream_t st, const BulkParams& p, bool pdl) {
  constexpr int ROW = HKV * D;
  const size_t smem = 2 * kStages * kStageBytes + 2 * kStages * sizeof(uint64_t) + 2 * ROW * sizeof(T);
  auto kern = decode_bulk_kernel<T, D, G, HKV>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kBulkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <typename T, int D, int HKV>
static int bulk_by_g(int G, dim3 grid, cudaStream_t st, const BulkParams& p, bool pdl, cudaError_t* e) {
  switch (G) {
    case 1: *e = launch_bulk<T, D, 1, HKV>(grid, st, p, pdl); return 0;
    case 2: *e = launch_bulk<T, D, 2, HKV>(grid, st, p, pdl); return 0;
    case 4: *e = launch_bulk<T, D, 4, HKV>(grid, st, p, pdl); return 0;
    case 7: *e = launch_bulk<T, D, 7, HKV>(grid, st, p, pdl); return 0;
    case 8: *e = launch_bulk<T, D, 8, HKV>(grid, st, p, pdl); return 0;
    default: return 1;
  }
}

template <typename T, int D>
static int bulk_by_hkv(int hkv, int G, dim3 grid, cudaStream_t st, const BulkParams& p, bool pdl, cudaError_t* e) {
  switch (hkv) {
    case 2: return bulk_by_g<T, D, 2>(G, grid, st, p, pdl, e);
    case 4: return bulk_by_g<T, D, 4>(G, grid, st, p, pdl, e);
    case 8: return bulk_by_g<T, D, 8>(G, grid, st, p, pdl, e);
    default: return 1;
  }
}

bool bulk_supported(int kv_dtype, int d, int hkv, int G) {
  bool dt = kv_dtype == RK_BF16 || kv_dtype == RK_F32;
  bool dd = d == 64 || d == 128;
  bool hh = hkv == 2 || hkv == 4 || hkv == 8;
  bool gg = G == 1 || G == 2 || G == 4 || G == 7 || G == 8;
  return dt && dd && hh && gg;
}

// partial slots of the uniform mode: one persistent CTA per SM (capped so each
// CTA streams >= 32 keys), times the warps-per-head slices
int bulk_splits(int batch, int max_seq_len, int hkv) {
  static int min_keys = -1;        // keys per CTA floor; RK_DECODE_MIN_KEYS overrides (experiments)
  if (min_keys < 0) {
    const char* e = std::getenv("RK_DECODE_MIN_KEYS");
    min_keys = e ? std::max(1, std::atoi(e)) : 32;
  }
  int64_t total = (int64_t)batch * max_seq_len;
  int64_t ctas = total / min_keys;
  int n = (int)(ctas < sm_count() ? (ctas < 1 ? 1 : ctas) : sm_count());
  return n * (8 / hkv);
}

int launch_decode_bulk(int kv_dtype, int d, int hkv, int G, int nsplit, const BulkParams& p, float* out,
                       int32_t* advance, cudaStream_t st, bool pdl) {
  // uniform mode: one persistent wave of CTAs; item mode: (items, batch)
  const int slices = 8 / hkv;
  dim3 grid = p.items ? dim3(p.items_stride, p.B) : dim3(nsplit / slices, 1);
  cudaError_t e = cudaSuccess;
  int r;
  if (kv_dtype == RK_BF16)
    r = launch_decode_mma(d, hkv, G, grid, p, st, pdl, &e);
  else
    r = d == 64 ? bulk_by_hkv<float, 64>(hkv, G, grid, st, p, pdl, &e)
                : bulk_by_hkv<float, 128>(hkv, G, grid, st, p, pdl, &e);
  if (r) return fail(RK_ERR_UNSUPPORTED, "bulk decode: hkv %d / group %d unsupported", hkv, G);
  if (e != cudaSuccess) return cuda_status(e, "decode_bulk_kernel launch");
  const bool wide = p.B * p.hq <= sm_count();   // at most one (dialogue, head) block per SM: 16 warps each
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.B, p.hq);
  cfg.blockDim = dim3(wide ? 512 : 128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, wide ? decode_merge_kernel<16> : decode_merge_kernel<4>, (const float*)p.part_m,
                         (const float*)p.part_l,
                         (const float*)p.part_acc, p.seq_len, p.k_new ? 1 : 0,
                         p.items ? p.n_items : (const int32_t*)nullptr, p.B, p.nsplit, slices,
                         (int)(p.items ? p.items_stride : nsplit / slices), p.hq, d, out, advance);
  if (e != cudaSuccess) return cuda_status(e, "decode_merge_kernel launch");
  return RK_OK;
}

}  // namespace rk
