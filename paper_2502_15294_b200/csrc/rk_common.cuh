// Shared device/host helpers for librk (round-attention hot path, sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/roundkv_b200.h"

namespace rk {

// ---------------------------------------------------------------- errors
// thread-local message behind rk_last_error(); set by every failing entry point
void set_error(const char* fmt, ...);
int fail(int status, const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

#define RK_CHECK_LAUNCH(what)                                   \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::rk::cuda_status(_e, what);  \
  } while (0)

#define RK_CUDA(call, what)                                     \
  do {                                                          \
    cudaError_t _e = (call);                                    \
    if (_e != cudaSuccess) return ::rk::cuda_status(_e, what);  \
  } while (0)

int sm_count();

static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------- device math
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  // packed fp32x2 FMA (FFMA2 on sm_100): a*b + c, both lanes round-to-nearest
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}

__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}

// two bf16 packed in a 32-bit word -> two floats (exact)
__device__ __forceinline__ float2 bf16x2_to_f2(uint32_t w) {
  float2 r;
  r.x = __uint_as_float(w << 16);
  r.y = __uint_as_float(w & 0xffff0000u);
  return r;
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 16-byte streaming load that does not allocate in L1 (KV is read once)
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int WIDTH>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int WIDTH>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
  for (int o = WIDTH / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- KV element access
template <typename T> struct KV;
template <> struct KV<float> {
  static constexpr int kBytes = 4;
  // 8 consecutive elements -> 4 float2
  __device__ __forceinline__ static void load8(const float* p, float2 (&out)[4]) {
    uint4 a = ld_stream(p), b = ld_stream(p + 4);
    out[0] = make_float2(__uint_as_float(a.x), __uint_as_float(a.y));
    out[1] = make_float2(__uint_as_float(a.z), __uint_as_float(a.w));
    out[2] = make_float2(__uint_as_float(b.x), __uint_as_float(b.y));
    out[3] = make_float2(__uint_as_float(b.z), __uint_as_float(b.w));
  }
  __device__ __forceinline__ static float get(const float* p, size_t i) { return p[i]; }
  __device__ __forceinline__ static void put(float* p, size_t i, float v) { p[i] = v; }
};
template <> struct KV<__nv_bfloat16> {
  static constexpr int kBytes = 2;
  __device__ __forceinline__ static void load8(const __nv_bfloat16* p, float2 (&out)[4]) {
    uint4 a = ld_stream(p);
    out[0] = bf16x2_to_f2(a.x);
    out[1] = bf16x2_to_f2(a.y);
    out[2] = bf16x2_to_f2(a.z);
    out[3] = bf16x2_to_f2(a.w);
  }
  __device__ __forceinline__ static float get(const __nv_bfloat16* p, size_t i) {
    return __bfloat162float(p[i]);
  }
  __device__ __forceinline__ static void put(__nv_bfloat16* p, size_t i, float v) {
    p[i] = __float2bfloat16_rn(v);
  }
};

}  // namespace rk
