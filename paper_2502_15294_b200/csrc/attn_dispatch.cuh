// Lane-layout selection and the per-dtype dispatch of attn_split_kernel.
// Instantiations live in attn_inst_f32.cu / attn_inst_bf16.cu (compiled in
// parallel); only layouts pick_shape can return are instantiated.
#pragma once

#include "attn_split.cuh"

namespace rk {

struct Shape {
  int lpk, nch, u;
  bool vec;
};

// Lane layout per (d, G): 128-bit vector path when d is 64/128/256 (LPK lanes
// per key, NCH 8-element chunks per lane), generic warp-per-key path (lanes
// stride over d, NCH rounded up to a power of two) otherwise.
inline bool pick_shape(int d, int G, Shape* s) {
  if (d == 64) { *s = {8, 1, 2, true}; return true; }
  if (d == 128) { *s = G <= 4 ? Shape{8, 2, 2, true} : Shape{16, 1, 2, true}; return true; }
  if (d == 256) { *s = G <= 2 ? Shape{16, 2, 1, true} : Shape{32, 1, 2, true}; return true; }
  if (d > 0 && d <= 256) {
    int n = (d + 31) / 32, p = 1;
    while (p < n) p <<= 1;
    *s = {32, p, p <= 2 ? 2 : 1, false};
    return true;
  }
  return false;
}

inline int tile_keys(const Shape& s) { return kWarps * (32 / s.lpk) * s.u; }

inline size_t split_smem(int G, int d) { return sizeof(float) * (2 * kWarps * G + kWarps * G * d); }

// returns 0 ok, 1 unsupported group, 2 launch error (see cudaGetLastError)
int dispatch_f32(bool decode, bool score, int G, const Shape& s, dim3 grid, cudaStream_t st, const SplitParams& p);
int dispatch_bf16(bool decode, bool score, int G, const Shape& s, dim3 grid, cudaStream_t st, const SplitParams& p);

template <typename T, int G, bool DEC, bool SC>
int launch_g(const Shape& s, dim3 grid, cudaStream_t st, const SplitParams& p) {
  size_t smem = split_smem(G, p.d);
#define RK_L(LPK, NCH, VEC, U) attn_split_kernel<T, G, LPK, NCH, VEC, U, DEC, SC><<<grid, kThreads, smem, st>>>(p)
  if (s.vec) {
    if (s.lpk == 8 && s.nch == 1) RK_L(8, 1, true, 2);
    else if constexpr (G <= 4) {
      if (s.lpk == 8) RK_L(8, 2, true, 2);
      else if (s.lpk == 16 && s.nch == 2) { if constexpr (G <= 2) RK_L(16, 2, true, 1); }
      else RK_L(32, 1, true, 2);
    } else {
      if (s.lpk == 16) RK_L(16, 1, true, 2);
      else RK_L(32, 1, true, 2);
    }
  } else {
    switch (s.nch) {
      case 1: RK_L(32, 1, false, 2); break;
      case 2: RK_L(32, 2, false, 2); break;
      case 4: RK_L(32, 4, false, 1); break;
      default: RK_L(32, 8, false, 1); break;
    }
  }
#undef RK_L
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 2;
}

template <typename T>
int dispatch_t(bool decode, bool score, int G, const Shape& s, dim3 grid, cudaStream_t st, const SplitParams& p) {
#define RK_G(GG)                                                    \
  case GG:                                                         \
    if (decode) return launch_g<T, GG, true, false>(s, grid, st, p); \
    if (score) return launch_g<T, GG, false, true>(s, grid, st, p);  \
    return launch_g<T, GG, false, false>(s, grid, st, p);
  switch (G) {
    RK_G(1) RK_G(2) RK_G(4) RK_G(7) RK_G(8)
    default: return 1;
  }
#undef RK_G
}

}  // namespace rk
