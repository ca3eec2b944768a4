// Tensor-core consumers for the pipelined bf16 decode attention.
//
// Same CTA organisation as decode_bulk_kernel (persistent flattened split-K or
// round-aligned items, producer warp + 8 consumer warps, 3-stage mbarrier
// ring, PDL), but the math of a 16-key group of one kv-head runs on
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate):
//   S[16 x 8]  = Qsplit[16 x D] . K^T[D x 8]        rows 0-7: q_hi, rows 8-15: q_lo
//   O[16 x D] += Psplit[16 x 16] . V[16 x D]        rows 0-7: p_hi, rows 8-15: p_lo
// where x_hi = bf16(x), x_lo = bf16(x - x_hi): the split keeps q (fp32, pre-
// scaled by log2(e)/sqrt(d)) and the probabilities at ~16 mantissa bits, so
// the result matches fp32 arithmetic (the reference tolerance is 1e-3
// relative; measured ~1e-6).  K and V are exact bf16.  G <= 8 query heads of a
// group occupy rows 0..G-1 of each half.  This removes the per-key shuffle
// reductions and bf16 unpacking that made the CUDA-core consumer
// instruction-bound (profiles/r01_decode_bulk_ncu.txt).
//
// Shared-memory tiles hold key rows ([HKV][D] bf16, token-major as in the
// cache) in runs of GK consecutive keys, ~4 KB per run, each run padded by 16
// bytes; the producer fills a run with one cp.async.bulk (32 lanes in
// parallel).  The appended token's row is copied from k_new straight into its
// slot of the last run.
#include <cmath>

#include "decode_common.cuh"

namespace rk {

constexpr float kRescaleLog2 = 8.f;   // lazy softmax rescale threshold (log2 units)

template <int D, int HKV>
struct MmaTile {
  static constexpr int ROW = HKV * D;               // bf16 elements per key
  static constexpr int ROWB = ROW * 2;              // bytes per key row (all kv-heads)
  // keys are copied in runs of GK consecutive rows (contiguous in the token-major
  // cache), so every bulk copy moves >= ~4 KB whatever the head count: per-copy
  // issue, not bandwidth, limited 1 KB rows to ~4.5 TB/s and 512 B rows to
  // ~2.4 TB/s; each run is padded by 16 B (GK-way ldmatrix bank conflicts,
  // cheap beside the memory stream)
#ifndef RK_RUN_BYTES
#define RK_RUN_BYTES 4096
#endif
  static constexpr int GK = ROWB >= RK_RUN_BYTES ? 1 : RK_RUN_BYTES / ROWB;
  static constexpr int GS = GK * ROWB + 16;         // run stride, bytes
  static constexpr int P = kConsumerWarps / HKV;    // warps per kv-head
  static constexpr int TK = 16 * P;                 // keys per stage: one 16-key group per warp
  static_assert(TK % GK == 0, "a stage holds whole runs");
  static constexpr int SB = (TK / GK) * GS;         // bytes per operand per stage
  __host__ __device__ static constexpr int row_off(int r) { return (r / GK) * GS + (r % GK) * ROWB; }
  // Key of row i (0..7) of n-tile t (0/1) of a warp's 16-key group.  Rows of one
  // run are ROWB (a multiple of 128 B) apart, i.e. on the same banks, so the 8
  // rows an ldmatrix reads are taken from as many different runs as the group
  // has (runs are GS = k*128 + 16 B apart: distinct 16-byte bank slots): with
  // GK = 2 (C2: 8 kv-heads x 128 dims) every row of a matrix sits in its own
  // run — conflict-free; GK = 1 keeps the natural order.  The softmax and the
  // PV product only need P's key order to match V's, which uses the same map.
  static constexpr int R = GK >= 16 ? 1 : (16 / GK < 8 ? 16 / GK : 8);   // runs one matrix spans
  __host__ __device__ static constexpr int key(int t, int i) {
    return GK == 1 ? 8 * t + i : (i % R) * GK + i / R + t * (8 / R);
  }
  static constexpr size_t smem = 2 * kStages * (size_t)SB + 2 * kStages * sizeof(uint64_t);
};

template <int D, int G, int HKV>
__global__ void __launch_bounds__(kBulkThreads, 1) decode_mma_kernel(const __grid_constant__ BulkParams p) {
  using Tl = MmaTile<D, HKV>;
  constexpr int ROW = Tl::ROW, P = Tl::P, TK = Tl::TK, SB = Tl::SB, GK = Tl::GK;
  constexpr int KC = D / 16;                        // k-chunks of the QK product
  constexpr int NT = D / 8;                         // n-tiles of the PV product
  static_assert(G <= 8 && D % 32 == 0, "group <= 8 rows per half, D multiple of 32");

  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* kst = smem;
  uint8_t* vst = smem + kStages * SB;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kStages * SB);
  uint64_t* empty = full + kStages;
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
  // let the merge kernel become resident now: it only reads the partials after
  // griddepcontrol.wait (full completion of this grid), so its launch latency
  // hides under this kernel's streaming
  pdl_trigger();
  const int nseg = segs.nseg;
  const __nv_bfloat16* kbase = reinterpret_cast<const __nv_bfloat16*>(p.k);
  const __nv_bfloat16* vbase = reinterpret_cast<const __nv_bfloat16*>(p.v);

  if (warp == kConsumerWarps) {
    // ================= producer warp: per-key bulk copies into padded rows
    const uint64_t pol = evict_first_policy();
    int t = 0;
    for (int sg = 0; sg < nseg; ++sg) {
      const Seg sgm = segs.seg[sg];
      const int len = p.seq_len[sgm.b] + (append ? 1 : 0);
      const int new_j = append ? len - 1 : -1;
      const __nv_bfloat16* kb = kbase + (int64_t)sgm.b * p.batch_stride;
      const __nv_bfloat16* vb = vbase + (int64_t)sgm.b * p.batch_stride;
      for (int j0 = sgm.lo; j0 < sgm.hi; j0 += TK, ++t) {
        const int s = t % kStages;
        const int nk = min(TK, sgm.hi - j0);
        if (lane == 0) {
          if (t >= kStages) mbar_wait(&empty[s], ((t / kStages) - 1) & 1);
          mbar_expect_tx(&full[s], (unsigned)(2 * nk * ROW * 2));
        }
        __syncwarp();
        for (int i = lane * GK; i < nk; i += 32 * GK) {      // one run of <= GK rows per lane
          const int j = j0 + i;
          int cnt = min(GK, nk - i);
          // the appended key (the dialogue's last, new_j) comes from k_new / v_new
          const bool has_new = new_j >= j && new_j < j + cnt;
          const int from_cache = has_new ? new_j - j : cnt;
          uint8_t* kd = kst + (size_t)s * SB + Tl::row_off(i);
          uint8_t* vd = vst + (size_t)s * SB + Tl::row_off(i);
          if (from_cache > 0) {
            bulk_g2s(kd, kb + (int64_t)j * ROW, (unsigned)(from_cache * ROW * 2), &full[s], pol);
            bulk_g2s(vd, vb + (int64_t)j * ROW, (unsigned)(from_cache * ROW * 2), &full[s], pol);
          }
          if (has_new) {
            pdl_wait();   // k_new / v_new are the previous kernel's output (the fused QKV projection)
            bulk_g2s(kd + from_cache * ROW * 2, reinterpret_cast<const __nv_bfloat16*>(p.k_new) + (int64_t)sgm.b * ROW,
                     ROW * 2, &full[s], pol);
            bulk_g2s(vd + from_cache * ROW * 2, reinterpret_cast<const __nv_bfloat16*>(p.v_new) + (int64_t)sgm.b * ROW,
                     ROW * 2, &full[s], pol);
          }
        }
      }
    }
    return;
  }

  // ================= consumers
  pdl_wait();   // q and the workspace belong to the previous kernels until here
  const int h = warp % HKV, slice = warp / HKV;
  const int g = lane >> 2, c = lane & 3;            // mma fragment coordinates
  int t = 0;

  for (int sg = 0; sg < nseg; ++sg) {
    const Seg sgm = segs.seg[sg];
    const int b = sgm.b;
    const int len = p.seq_len[b] + (append ? 1 : 0);
    if (append && sgm.hi == len) {     // the owner of the appended key writes it to the cache
      const __nv_bfloat16* kn = reinterpret_cast<const __nv_bfloat16*>(p.k_new) + (int64_t)b * ROW;
      const __nv_bfloat16* vn = reinterpret_cast<const __nv_bfloat16*>(p.v_new) + (int64_t)b * ROW;
      __nv_bfloat16* kd = const_cast<__nv_bfloat16*>(kbase) + (int64_t)b * p.batch_stride + (int64_t)(len - 1) * ROW;
      __nv_bfloat16* vd = const_cast<__nv_bfloat16*>(vbase) + (int64_t)b * p.batch_stride + (int64_t)(len - 1) * ROW;
      for (int e = threadIdx.x; e < ROW / 8; e += kConsumerWarps * 32) {
        reinterpret_cast<uint4*>(kd)[e] = reinterpret_cast<const uint4*>(kn)[e];
        reinterpret_cast<uint4*>(vd)[e] = reinterpret_cast<const uint4*>(vn)[e];
      }
    }

    // Q fragments (A operand, rows g / g+8 = hi / lo of query head g)
    uint32_t qa[KC][4];
    {
      const bool real = g < G;
      const float* qp = p.q + ((int64_t)b * p.hq + h * G + (real ? g : 0)) * D;
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        float x[4];
        const float2 lo2 = *reinterpret_cast<const float2*>(qp + 16 * kc + 2 * c);
        const float2 hi2 = *reinterpret_cast<const float2*>(qp + 16 * kc + 2 * c + 8);
        x[0] = real ? lo2.x * p.scale_log2 : 0.f;
        x[1] = real ? lo2.y * p.scale_log2 : 0.f;
        x[2] = real ? hi2.x * p.scale_log2 : 0.f;
        x[3] = real ? hi2.y * p.scale_log2 : 0.f;
        const float h0 = bf16_round(x[0]), h1 = bf16_round(x[1]), h2 = bf16_round(x[2]), h3 = bf16_round(x[3]);
        qa[kc][0] = pack_bf16(h0, h1);
        qa[kc][1] = pack_bf16(x[0] - h0, x[1] - h1);
        qa[kc][2] = pack_bf16(h2, h3);
        qa[kc][3] = pack_bf16(x[2] - h2, x[3] - h3);
      }
    }
    float o[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
    float m = -INFINITY, lsum = 0.f;

    for (int j0 = sgm.lo; j0 < sgm.hi; j0 += TK, ++t) {
      const int s = t % kStages;
      const int nk = min(TK, sgm.hi - j0);
      const int nkw = min(16, max(0, nk - 16 * slice));        // valid keys of this warp's group
      mbar_wait(&full[s], (t / kStages) & 1);
      if (nkw > 0) {
        const uint8_t* kb = kst + (size_t)s * SB + h * D * 2;    // + Tl::row_off(key row)
        uint8_t* vb = vst + (size_t)s * SB + h * D * 2;
        if (nkw < 16) {   // rows past the valid keys hold stale bytes: zero this head's V columns
          for (int e = lane; e < (16 - nkw) * (D / 8); e += 32) {
            const int r = nkw + e / (D / 8), q16 = e % (D / 8);
            reinterpret_cast<uint4*>(vb + Tl::row_off(16 * slice + r))[q16] = make_uint4(0, 0, 0, 0);
          }
          // generic-proxy writes to a buffer the bulk copies refill later
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
        }
        // ---- S = Q K^T for keys 0-7 (s0) and 8-15 (s1)
        float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < KC / 2; ++kk) {
          uint32_t r[4];
          ldmatrix_x4(r, kb + Tl::row_off(16 * slice + Tl::key(0, lane & 7)) + (32 * kk + 8 * (lane >> 3)) * 2);
          mma_bf16_16816(s0, qa[2 * kk], r[0], r[1]);
          mma_bf16_16816(s0, qa[2 * kk + 1], r[2], r[3]);
          ldmatrix_x4(r, kb + Tl::row_off(16 * slice + Tl::key(1, lane & 7)) + (32 * kk + 8 * (lane >> 3)) * 2);
          mma_bf16_16816(s1, qa[2 * kk], r[0], r[1]);
          mma_bf16_16816(s1, qa[2 * kk + 1], r[2], r[3]);
        }
        float sc[4];
        sc[0] = (Tl::key(0, 2 * c) < nkw) ? s0[0] + s0[2] : -INFINITY;
        sc[1] = (Tl::key(0, 2 * c + 1) < nkw) ? s0[1] + s0[3] : -INFINITY;
        sc[2] = (Tl::key(1, 2 * c) < nkw) ? s1[0] + s1[2] : -INFINITY;
        sc[3] = (Tl::key(1, 2 * c + 1) < nkw) ? s1[1] + s1[3] : -INFINITY;
        float tmax = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
        // ---- lazy online softmax: move the reference max only when the tile
        // exceeds it by 2^8 (probabilities stay <= 256, exact in the split)
        const bool grow = tmax > m + kRescaleLog2 || (m == -INFINITY && tmax != -INFINITY);
        if (__any_sync(0xffffffffu, grow)) {
          const float m_new = grow ? tmax : m;
          const float corr = (m == -INFINITY) ? 0.f : fast_exp2(m - m_new);
          m = m_new;
          lsum *= corr;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            o[nt][0] *= corr; o[nt][1] *= corr; o[nt][2] *= corr; o[nt][3] *= corr;
          }
        }
        const float mu = (m == -INFINITY) ? 0.f : m;
        float pr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) pr[i] = fast_exp2(sc[i] - mu);
        lsum += (pr[0] + pr[1]) + (pr[2] + pr[3]);
        uint32_t pa[4];
        {
          const float h0 = bf16_round(pr[0]), h1 = bf16_round(pr[1]), h2 = bf16_round(pr[2]), h3 = bf16_round(pr[3]);
          pa[0] = pack_bf16(h0, h1);
          pa[1] = pack_bf16(pr[0] - h0, pr[1] - h1);
          pa[2] = pack_bf16(h2, h3);
          pa[3] = pack_bf16(pr[2] - h2, pr[3] - h3);
        }
        // ---- O += P V
#pragma unroll
        for (int jj = 0; jj < NT / 2; ++jj) {
          uint32_t r[4];
          ldmatrix_x4_trans(r, vb + Tl::row_off(16 * slice + Tl::key((lane >> 3) & 1, lane & 7)) +
                                   (16 * jj + 8 * (lane >> 4)) * 2);
          mma_bf16_16816(o[2 * jj], pa, r[0], r[1]);
          mma_bf16_16816(o[2 * jj + 1], pa, r[2], r[3]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // ---- partial slot of this warp: head h*G+g, dims 8nt+2c, 8nt+2c+1
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
    lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
    if (g < G) {
      const int slot = blockIdx.x * P + slice;
      const int64_t sl = ((int64_t)b * p.hq + h * G + g) * p.nsplit + slot;
      float* dst = p.part_acc + sl * D;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        *reinterpret_cast<float2*>(dst + 8 * nt + 2 * c) = make_float2(o[nt][0] + o[nt][2], o[nt][1] + o[nt][3]);
      if (c == 0) {
        p.part_m[sl] = m;
        p.part_l[sl] = lsum;
      }
    }
  }
}

template <int D, int G, int HKV>
static cudaError_t launch_mma(dim3 grid, cudaStream_t st, const BulkParams& p, bool pdl) {
  const size_t smem = MmaTile<D, HKV>::smem;
  auto kern = decode_mma_kernel<D, G, HKV>;
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

template <int D, int HKV>
static int mma_by_g(int G, dim3 grid, cudaStream_t st, const BulkParams& p, bool pdl, cudaError_t* e) {
  switch (G) {
    case 1: *e = launch_mma<D, 1, HKV>(grid, st, p, pdl); return 0;
    case 2: *e = launch_mma<D, 2, HKV>(grid, st, p, pdl); return 0;
    case 4: *e = launch_mma<D, 4, HKV>(grid, st, p, pdl); return 0;
    case 7: *e = launch_mma<D, 7, HKV>(grid, st, p, pdl); return 0;
    case 8: *e = launch_mma<D, 8, HKV>(grid, st, p, pdl); return 0;
    default: return 1;
  }
}

int launch_decode_mma(int d, int hkv, int G, dim3 grid, const BulkParams& p, cudaStream_t st, bool pdl,
                      cudaError_t* e) {
  if (d == 128) {
    switch (hkv) {
      case 2: return mma_by_g<128, 2>(G, grid, st, p, pdl, e);
      case 4: return mma_by_g<128, 4>(G, grid, st, p, pdl, e);
      case 8: return mma_by_g<128, 8>(G, grid, st, p, pdl, e);
    }
  } else if (d == 64) {
    switch (hkv) {
      case 2: return mma_by_g<64, 2>(G, grid, st, p, pdl, e);
      case 4: return mma_by_g<64, 4>(G, grid, st, p, pdl, e);
      case 8: return mma_by_g<64, 8>(G, grid, st, p, pdl, e);
    }
  }
  return 1;
}

}  // namespace rk
