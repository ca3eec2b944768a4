// float32-KV instantiations of attn_split_kernel.
#include "attn_dispatch.cuh"

namespace rk {
int dispatch_f32(bool decode, bool score, int G, const Shape& s, dim3 grid, cudaStream_t st, const SplitParams& p) {
  return dispatch_t<float>(decode, score, G, s, grid, st, p);
}
}  // namespace rk
