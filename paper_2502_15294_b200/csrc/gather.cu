// Batched host<->HBM block movement for the tiered round store.
//
// A kept round's upper-layer block lives in pinned host memory as
// [upper_layer][K|V][tokens][hkv][d] (the reference payload layout,
// store.py:225-242).  The device working cache of the upper layers is
// [layer][K|V][capacity][hkv][d], so one kept round is ONE strided DMA:
// (L-Lw)*2 rows of tokens*hkv*d elements, source pitch = row width, destination
// pitch = capacity*hkv*d.  rk_h2d_gather issues one cudaMemcpy2DAsync per
// kept round on the caller's copy stream and records `done_event` at the end,
// so the consumer stream waits on the event, not on the host.
#include "rk_common.cuh"

extern "C" {

static int copy_batch(int n, const void* const* src, const size_t* sp, void* const* dst, const size_t* dp,
                      const size_t* w, const size_t* h, cudaMemcpyKind kind, rk_stream_t stream,
                      void* done_event, const char* what) {
  if (n < 0) return rk::fail(RK_ERR_DOMAIN, "%s: negative copy count", what);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  for (int i = 0; i < n; ++i) {
    if (w[i] == 0 || h[i] == 0) continue;
    if (sp[i] < w[i] || dp[i] < w[i]) return rk::fail(RK_ERR_DOMAIN, "%s: pitch smaller than width", what);
    RK_CUDA(cudaMemcpy2DAsync(dst[i], dp[i], src[i], sp[i], w[i], h[i], kind, cs), what);
  }
  if (done_event) RK_CUDA(cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), cs), "event record");
  return RK_OK;
}

int rk_h2d_gather(int n, const void* const* src_host, const size_t* src_pitch, void* const* dst,
                  const size_t* dst_pitch, const size_t* width, const size_t* height, rk_stream_t stream,
                  void* done_event) {
  return copy_batch(n, src_host, src_pitch, dst, dst_pitch, width, height, cudaMemcpyHostToDevice, stream,
                    done_event, "rk_h2d_gather");
}

int rk_peer_gather(int n, const void* const* src, const size_t* src_pitch, void* const* dst,
                   const size_t* dst_pitch, const size_t* width, const size_t* height, rk_stream_t stream,
                   void* done_event) {
  // source blocks in HBM (this GPU's, or a peer's over NVLink once peer access is
  // enabled): unified addressing picks the path
  return copy_batch(n, src, src_pitch, dst, dst_pitch, width, height, cudaMemcpyDefault, stream, done_event,
                    "rk_peer_gather");
}

int rk_enable_peer_access(int peer_device) {
  int cur = 0;
  RK_CUDA(cudaGetDevice(&cur), "cudaGetDevice");
  if (peer_device == cur) return RK_OK;
  int can = 0;
  RK_CUDA(cudaDeviceCanAccessPeer(&can, cur, peer_device), "cudaDeviceCanAccessPeer");
  if (!can) return rk::fail(RK_ERR_CUDA, "GPU %d cannot access GPU %d's memory", cur, peer_device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return RK_OK;
  }
  RK_CUDA(e, "cudaDeviceEnablePeerAccess");
  return RK_OK;
}

int rk_d2h_scatter(int n, const void* const* src, const size_t* src_pitch, void* const* dst_host,
                   const size_t* dst_pitch, const size_t* width, const size_t* height, rk_stream_t stream,
                   void* done_event) {
  return copy_batch(n, src, src_pitch, dst_host, dst_pitch, width, height, cudaMemcpyDeviceToHost, stream,
                    done_event, "rk_d2h_scatter");
}

}  // extern "C"
