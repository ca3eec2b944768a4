// MUFU ex2 throughput probe: lanes of ex2.approx.ftz.f32 per clock per SM on this part,
// for 1..16 warps per SM (independent chains, so latency is hidden once enough are in flight).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_probe tools/mufu_probe.cu && /tmp/mufu_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8, IT = 4096;

__global__ void ex2_kernel(float* out, long long* clk, float seed) {
  float v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = seed * (threadIdx.x + c) * 1e-9f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += v[c];
  if (s == 123.f) out[0] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  long long* clk;
  cudaMalloc(&out, 4);
  cudaMalloc(&clk, sizeof(long long) * sms);
  long long h[1024];
  for (int warps : {1, 2, 4, 8, 12, 16, 32}) {
    ex2_kernel<<<sms, 32 * warps>>>(out, clk, 1.f);
    ex2_kernel<<<sms, 32 * warps>>>(out, clk, 1.f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    const double lanes = 32.0 * warps * CH * IT;
    printf("warps/SM %2d: %.2f ex2 lanes/clk/SM\n", warps, lanes / mx);
  }
  return 0;
}
