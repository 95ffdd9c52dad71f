// common.cuh -- shared device helpers for the dose kernels (sm_100a).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dosegpu.h"

#define DG_CUDA(expr)                                                   \
  do {                                                                  \
    cudaError_t _e = (expr);                                            \
    if (_e != cudaSuccess) return DG_ERR_CUDA_BASE + static_cast<int>(_e); \
  } while (0)

#define DG_TRY(expr)              \
  do {                            \
    int _s = (expr);              \
    if (_s != DG_OK) return _s;   \
  } while (0)

namespace dg {

constexpr unsigned kFull = 0xffffffffu;

// Exact binary16 -> double (ddm::decode_half, src/half.cpp:50-64): binary16 -> binary32 is exact
// for every pattern (subnormals become normals, Inf/NaN stay), binary32 -> binary64 is exact.
// SASS: HADD2.F32 + F2F.F64.F32.
__device__ __forceinline__ double widen(uint16_t h) {
  return static_cast<double>(__half2float(__ushort_as_half(h)));
}
__device__ __forceinline__ double widen(float v) { return static_cast<double>(v); }
__device__ __forceinline__ double widen(double v) { return v; }

__device__ __forceinline__ float widen_f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ float widen_f(float v) { return v; }
__device__ __forceinline__ float widen_f(double v) { return static_cast<float>(v); }

// Streaming loads of the matrix: read once, keep out of L1 so x keeps the cache.
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
  return __ldcs(p);
}

}  // namespace dg
