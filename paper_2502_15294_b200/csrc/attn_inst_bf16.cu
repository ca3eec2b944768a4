// bf16-KV instantiations of attn_split_kernel.
#include "attn_dispatch.cuh"

namespace rk {
int dispatch_bf16(bool decode, bool score, int G, const Shape& s, dim3 grid, cudaStream_t st, const SplitParams& p) {
  return dispatch_t<__nv_bfloat16>(decode, score, G, s, grid, st, p);
}
}  // namespace rk
