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

// Exact binary16 -> double (ddm::decode_half, src/half.cpp:50-64): cvt.f64.f16 is an exact
// widening for every pattern (subnormals become normals, Inf/NaN stay).  SASS: one
// F2F.F64.F16 reading the low half of the packed word directly (instead of HADD2.F32 +
// F2F.F64.F32).
__device__ __forceinline__ double widen(uint16_t h) {
  double d;
  asm("{ .reg .f16 t; mov.b16 t, %1; cvt.f64.f16 %0, t; }" : "=d"(d) : "h"(h));
  return d;
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

// ---- matrix element streams ----------------------------------------------------------------
// SoA: the reference's separate column / value arrays, any value precision and index width.
template <typename V, typename I>
struct SoA {
  using Val = V;
  using Idx = I;
  struct Raw {
    I c;
    V v;
  };
  const I* col;
  const V* val;
  __device__ __forceinline__ Raw load(uint64_t j) const { return {ld_stream(col + j), ld_stream(val + j)}; }
  __device__ __forceinline__ Idx col_at(uint64_t j) const { return col[j]; }
  __device__ __forceinline__ static I c_of(const Raw& r) { return r.c; }
  __device__ __forceinline__ static V v_of(const Raw& r) { return r.v; }
  // a placeholder element for masked-off lanes: a valid column, value bits 0
  __device__ __forceinline__ static Raw filler(uint32_t col) { return {static_cast<I>(col), V(0)}; }
  // L2 prefetch of the 128-byte lines of 32 * U positions starting at p: lines [0, lc) are the
  // column lines, [lc, lc + lv) the value lines; line k goes to lane k % 32
  template <int U>
  __device__ __forceinline__ void prefetch_batch(uint64_t p, uint32_t room, uint32_t lane) const {
    constexpr uint32_t lc = U * sizeof(I) / 4, lv = U * sizeof(V) / 4;
#pragma unroll
    for (uint32_t k0 = 0; k0 < lc + lv; k0 += 32) {
      const uint32_t k = k0 + lane;
      const char* a = nullptr;
      if (k < lc) {
        if (k * (128 / sizeof(I)) < room) a = reinterpret_cast<const char*>(col + p) + 128 * k;
      } else if (k < lc + lv) {
        if ((k - lc) * (128 / sizeof(V)) < room)
          a = reinterpret_cast<const char*>(val + p) + 128 * (k - lc);
      }
      if (a) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
  }
};

// Packed16: the native (binary16 value, u16 column) pair of one nonzero in one 32-bit word,
// column in the high half.  Same 4 bytes per nonzero as the SoA pair (no expansion), but one
// 128-byte request serves 32 lanes' positions instead of two 64-byte requests.
struct Packed16 {
  using Val = uint16_t;
  using Idx = uint16_t;
  using Raw = uint32_t;
  const uint32_t* w;
  __device__ __forceinline__ Raw load(uint64_t j) const { return ld_stream(w + j); }
  __device__ __forceinline__ Idx col_at(uint64_t j) const { return static_cast<uint16_t>(w[j] >> 16); }
  __device__ __forceinline__ static uint16_t c_of(Raw r) { return static_cast<uint16_t>(r >> 16); }
  __device__ __forceinline__ static uint16_t v_of(Raw r) { return static_cast<uint16_t>(r & 0xFFFFu); }
  __device__ __forceinline__ static Raw filler(uint32_t col) { return col << 16; }
  // lines of positions [p, p + min(32 * U, room)): no line past the segment is fetched
  template <int U>
  __device__ __forceinline__ void prefetch_batch(uint64_t p, uint32_t room, uint32_t lane) const {
    if (lane < U && 32 * lane < room) asm volatile("prefetch.global.L2 [%0];" ::"l"(w + p + 32 * lane));
  }
};

// Fused d gather (dg_set_gather_targets): each finished row is also stored into every rank's
// full-d buffer (peer memory over NVLink) at its global row.
constexpr uint32_t kMaxGatherTargets = 8;
struct GatherTargets {
  double* t[kMaxGatherTargets];
  uint32_t n;
  uint64_t row_off;
  // kernels take it as `const __grid_constant__`: indexed in the parameter space directly (a
  // by-value parameter indexed at run time was copied to the stack -- r01's 88-byte frame)
  __device__ __forceinline__ void store(uint64_t row, double v) const {
    for (uint32_t i = 0; i < n; ++i) t[i][row_off + row] = v;
  }
};

// Host side: every dg_* entry point that selects a device restores the caller's current device
// when it returns (a host thread driving several GPUs keeps its own device selection).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      cudaGetLastError();
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

__device__ __forceinline__ uint32_t pack16(uint16_t col, uint16_t half_bits) {
  return (static_cast<uint32_t>(col) << 16) | half_bits;
}

}  // namespace dg
