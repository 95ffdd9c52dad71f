// spmv_kernels.cuh -- row-list kernels of the dose SpMV (d = A.x), sm_100a.
//
// Semantics (exact family) are those of ddm::rowchunk_rows<V> (src/spmv.cpp:48-68): for a row
// with positions [start, end), lane l of L accumulates widen(v[j]) * x[col[j]] for
// j = start + l, start + l + L, ... in increasing order starting from +0.0 (no FMA: __dmul_rn /
// __dadd_rn), then partial[l] += partial[l + w] for w = L/2 ... 1, and d[i] = partial[0].  Empty
// rows are left at +0.0 (the caller zero-fills d).  Because a row of length len <= G <= L gives
// every lane at most one product and pads the rest with +0.0 partials (never -0.0: 0.0 + p is
// +0.0 for p = -0.0), the tree over L lanes equals the tree over G lanes: short rows run G lanes
// wide and still match L = 32 bit for bit.
//
// These kernels take the matrix as an element stream M (SoA or Packed16, common.cuh).  Rows
// longer than 32 under lane_width 32 go to the column-windowed tile kernel (spmv_tiles.cuh); the
// warp-per-row kernel here is the v0 plan, kept selectable (DG_PLAN=warp) for A/B measurement.
#pragma once

#include "common.cuh"

namespace dg {

template <typename Acc>
struct AccOps;
template <>
struct AccOps<double> {
  template <typename V>
  __device__ static __forceinline__ double prod(V v, double xv) { return __dmul_rn(widen(v), xv); }
  __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <>
struct AccOps<float> {
  template <typename V>
  __device__ static __forceinline__ float prod(V v, float xv) { return __fmul_rn(widen_f(v), xv); }
  __device__ static __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};

// ------------------------------------------------------------------------------------------
// G lanes per row, G in {1,2,4,8,16,32}; lane-strided with stride G.  Serves the general
// lane_width = G <= 32 engine (all rows) and the L = 32 engine's short-row bins (len <= G).
template <int G, class M, typename Acc>
__global__ void __launch_bounds__(256) k_group(M mat, const uint64_t* __restrict__ rp,
                                               const Acc* __restrict__ x,
                                               const uint32_t* __restrict__ rows,
                                               uint32_t n_rows, double* __restrict__ y,
                                               const __grid_constant__ GatherTargets gt) {
  using Ops = AccOps<Acc>;
  const uint32_t lane = threadIdx.x & (G - 1);
  const uint64_t group = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  const uint64_t n_groups = static_cast<uint64_t>(gridDim.x) * blockDim.x / G;
  for (uint64_t g = group; g < ((n_rows + n_groups - 1) / n_groups) * n_groups; g += n_groups) {
    const bool live = g < n_rows;
    uint32_t r = 0;
    Acc acc = Acc(0);
    if (live) {
      r = rows[g];
      const uint64_t start = rp[r], end = rp[r + 1];
      for (uint64_t j = start + lane; j < end; j += G) {
        const auto e = mat.load(j);
        acc = Ops::add(acc, Ops::prod(M::v_of(e), __ldg(x + M::c_of(e))));
      }
    }
#pragma unroll
    for (int w = G / 2; w >= 1; w /= 2) acc = Ops::add(acc, __shfl_down_sync(kFull, acc, w, G));
    if (live && lane == 0) {
      y[r] = static_cast<double>(acc);
      gt.store(r, static_cast<double>(acc));
    }
  }
}

// ------------------------------------------------------------------------------------------
// v0: one warp per long row (L = 32), 8-deep unrolled, x gathered through L1.
template <class M, typename Acc>
__global__ void __launch_bounds__(256) k_warp(M mat, const uint64_t* __restrict__ rp,
                                              const Acc* __restrict__ x,
                                              const uint32_t* __restrict__ rows, uint32_t n_rows,
                                              double* __restrict__ y, const __grid_constant__ GatherTargets gt) {
  using Ops = AccOps<Acc>;
  constexpr int U = 8;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t w = warp; w < n_rows; w += n_warps) {
    const uint32_t r = rows[w];
    const uint64_t start = rp[r], end = rp[r + 1];
    Acc acc = Acc(0);
    uint64_t base = start;
    for (; base + 32 * U <= end; base += 32 * U) {
      typename M::Raw e[U];
#pragma unroll
      for (int u = 0; u < U; ++u) e[u] = mat.load(base + lane + 32 * u);
      Acc xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + M::c_of(e[u]));
#pragma unroll
      for (int u = 0; u < U; ++u) acc = Ops::add(acc, Ops::prod(M::v_of(e[u]), xv[u]));
    }
    for (uint64_t j = base + lane; j < end; j += 32) {
      const auto e = mat.load(j);
      acc = Ops::add(acc, Ops::prod(M::v_of(e), __ldg(x + M::c_of(e))));
    }
#pragma unroll
    for (int off = 16; off >= 1; off /= 2) acc = Ops::add(acc, __shfl_down_sync(kFull, acc, off));
    if (lane == 0) {
      y[r] = static_cast<double>(acc);
      gt.store(r, static_cast<double>(acc));
    }
  }
}

// ------------------------------------------------------------------------------------------
// lane_width L in {64, ..., 1024}: one CTA of L threads per row, stride-halving tree in smem.
template <class M>
__global__ void k_block_exact(M mat, const uint64_t* __restrict__ rp, const double* __restrict__ x,
                              const uint32_t* __restrict__ rows, uint32_t n_rows,
                              double* __restrict__ y, const __grid_constant__ GatherTargets gt) {
  extern __shared__ double partial[];
  const uint32_t L = blockDim.x, l = threadIdx.x;
  for (uint32_t b = blockIdx.x; b < n_rows; b += gridDim.x) {
    const uint32_t r = rows[b];
    const uint64_t start = rp[r], end = rp[r + 1];
    double acc = 0.0;
    for (uint64_t j = start + l; j < end; j += L) {
      const auto e = mat.load(j);
      acc = __dadd_rn(acc, __dmul_rn(widen(M::v_of(e)), __ldg(x + M::c_of(e))));
    }
    partial[l] = acc;
    __syncthreads();
    for (uint32_t w = L / 2; w >= 1; w /= 2) {
      if (l < w) partial[l] = __dadd_rn(partial[l], partial[l + w]);
      __syncthreads();
    }
    if (l == 0) {
      y[r] = partial[0];
      gt.store(r, partial[0]);
    }
    __syncthreads();
  }
}

static __global__ void k_x_to_f32(const double* __restrict__ x, float* __restrict__ xf, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    xf[i] = static_cast<float>(x[i]);
}

// ------------------------------------------------------------------------------------------
// upload-time (and generator) validation (ddm::validate, src/sparse.cpp:197-255): per row, columns strictly
// increasing and < cols; every value finite.  Flags are OR-ed into *bad.
template <class M>
__global__ void k_validate(M mat, const uint64_t* __restrict__ rp, uint64_t rows, uint64_t cols,
                           unsigned* __restrict__ bad) {
  const uint64_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  unsigned flag = 0;
  for (uint64_t r = warp; r < rows; r += n_warps) {
    const uint64_t s = rp[r], e = rp[r + 1];
    for (uint64_t j = s + lane; j < e; j += 32) {
      const auto el = mat.load(j);
      const uint64_t c = M::c_of(el);
      if (c >= cols) flag |= 1u;
      if (j > s && c <= static_cast<uint64_t>(mat.col_at(j - 1))) flag |= 2u;
      if (!isfinite(widen(M::v_of(el)))) flag |= 4u;
    }
  }
  flag = __reduce_or_sync(kFull, flag);
  if (lane == 0 && flag) atomicOr(bad, flag);
}


}  // namespace dg
