// FP64 throughput on this part: DFMA chains vs mma.sync m8n8k4 f64 (DMMA), register operands only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dm tools/dmma_probe.cu && /tmp/dm
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters) {
  double a[8], x = threadIdx.x * 1e-3, y = 1.0000001;
  for (int i = 0; i < 8; ++i) a[i] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], y, x);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* o;
  cudaMalloc(&o, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int blocks_per_sm : {2, 4, 8}) {
    dfma_loop<<<sms * blocks_per_sm, 256>>>(o, 100);
    cudaEventRecord(e0);
    dfma_loop<<<sms * blocks_per_sm, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * 256.0 * sms * blocks_per_sm;
    printf("DFMA  %d blocks/SM: %.1f TFLOP/s\n", blocks_per_sm, fl / ms / 1e9);
    dmma_loop<<<sms * blocks_per_sm, 256>>>(o, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms * blocks_per_sm, 256>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 4 * iters * (256 / 32) * (double)sms * blocks_per_sm;
    printf("DMMA  %d blocks/SM: %.1f TFLOP/s (%s)\n", blocks_per_sm, fl / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
