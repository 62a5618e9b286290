// Shared helpers for the srpgpu sm_100a kernels and their C-ABI entry points.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdarg.h>
#include <stdio.h>

#include <algorithm>

#include "../../include/srpgpu.h"

namespace srpgpu {

// Thread-local message for srpgpu_last_error(); status codes cross the ABI.
void set_error(const char* fmt, ...);
// Count of kernel launches issued through the library (bench `gpu_launches`).
void count_launch(int n = 1);

#define SRPGPU_CHECK_ARG(cond, code, ...)        \
  do {                                           \
    if (!(cond)) {                               \
      ::srpgpu::set_error(__VA_ARGS__);          \
      return (code);                             \
    }                                            \
  } while (0)

#define SRPGPU_CHECK_LAUNCH(what)                                                   \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) {                                                        \
      ::srpgpu::set_error("%s: launch failed: %s", what, cudaGetErrorString(_e));   \
      return SRPGPU_ERR_LAUNCH;                                                     \
    }                                                                               \
    ::srpgpu::count_launch();                                                       \
  } while (0)

inline int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// ---- packed argmax keys ---------------------------------------------------
// key = (ordered_bits(z) << 32) | (0xFFFFFFFF - i): the largest key is the
// largest value, ties resolved to the LOWEST index (np.argmax, srp.py:74-80).
__device__ __forceinline__ uint32_t ordered_bits(float x) {
  x = x + 0.0f;  // -0.0 -> +0.0 so signed zeros tie like np.argmax
  uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ unsigned long long make_key(float z, uint32_t i) {
  return ((unsigned long long)ordered_bits(z) << 32) | (unsigned long long)(0xFFFFFFFFu - i);
}

__device__ __forceinline__ unsigned long long key_max(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

__device__ __forceinline__ unsigned long long warp_key_max(unsigned long long k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) k = key_max(k, __shfl_xor_sync(0xffffffffu, k, o));
  return k;
}

// round-to-nearest-even to TF32 (keeps 10 explicit mantissa bits)
__device__ __forceinline__ float tf32_rne(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7F800000u) != 0x7F800000u) u += 0xFFFu + ((u >> 13) & 1u);
  return __uint_as_float(u & 0xFFFFE000u);
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

inline cudaStream_t as_stream(srpgpu_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace srpgpu
