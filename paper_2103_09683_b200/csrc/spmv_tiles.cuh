// spmv_tiles.cuh -- column-windowed tile kernel: x staged in shared memory by 1-D TMA.
//
// Why: the dose gather x[col[j]] is the dominant L1 cost of a lane-strided CSR SpMV (32 lanes of
// a sparse row touch ~16 sectors of x per request; v0 ncu: 6.5 sectors/request, 42% of HBM).  The
// row plan (plan.cu) sorts row segments by first column and cuts them into tiles whose column
// window [xlo, xlo + xlen) fits in shared memory; one CTA stages the tile's window with
// cp.async.bulk (UBLKCP) and its warps gather x from shared memory instead of L1/L2.
//
// Exactness: a segment is a contiguous position range [p0, p0 + n) of one row; physical lane l
// owns the row's logical lane l (positions j with (j - row_start) % 32 == l), accumulates them in
// increasing j from +0.0 (or from the carried partial of the row's previous segment, written by
// the previous wave), and the last segment applies the stride-halving tree.  This is exactly
// ddm::rowchunk_rows with lane_width 32 (src/spmv.cpp:48-68), split over waves only at segment
// boundaries, where the lane partials are stored and reloaded unchanged.
#pragma once

#include "common.cuh"

namespace dg {

struct Segment {  // 24 bytes
  uint64_t p0;     // first position (shard-local nnz index)
  uint32_t n;      // positions [p0, p0 + n)
  uint32_t row;    // shard-local row
  uint32_t slot;   // carried-partials slot (split rows), else unused
  uint16_t lane0;  // (p0 - row_start) % 32
  uint16_t flags;  // kSegFirst | kSegLast
};
constexpr uint16_t kSegFirst = 1, kSegLast = 2;

struct Tile {  // 16 bytes
  uint32_t xlo, xlen;  // x window (xlo even, xlen even)
  uint32_t seg0, seg1;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "DG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra DG_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA: global -> shared, completion counted on the mbarrier (SASS: UBLKCP.S.G).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

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

// Persistent: CTAs pull tiles from *counter in plan order; warps pull the tile's segments.
template <typename V, typename I, typename Acc, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 2)
    k_tiles(const I* __restrict__ col, const V* __restrict__ val, const Acc* __restrict__ x,
            const Tile* __restrict__ tiles, uint32_t n_tiles, const Segment* __restrict__ segs,
            Acc* __restrict__ state, double* __restrict__ y, uint32_t* __restrict__ counter) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Acc* xs = reinterpret_cast<Acc*>(smem_raw);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tile, s_next;
  using Ops = AccOps<Acc>;
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      s_tile = atomicAdd(counter, 1u);
      s_next = 0;
    }
    __syncthreads();
    const uint32_t t = s_tile;
    if (t >= n_tiles) break;
    const Tile T = tiles[t];
    if (threadIdx.x == 0) {
      // order this CTA's earlier generic-proxy reads of xs before the async-proxy overwrite
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t bytes = (T.xlen * sizeof(Acc) + 15u) & ~15u;
      mbar_arrive_expect_tx(&bar, bytes);
      const char* src = reinterpret_cast<const char*>(x + T.xlo);
      for (uint32_t off = 0; off < bytes; off += 32768u)
        tma_load_1d(reinterpret_cast<char*>(xs) + off, src + off, min(32768u, bytes - off), &bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1u;
    const uint32_t xlo = T.xlo;  // xs[c - xlo] == x[c] for c in the window
    const uint32_t nseg = T.seg1 - T.seg0;
    for (;;) {
      uint32_t k = 0;
      if (lane == 0) k = atomicAdd(&s_next, 1u);
      k = __shfl_sync(kFull, k, 0);
      if (k >= nseg) break;
      const Segment S = segs[T.seg0 + k];
      const uint64_t p0 = S.p0, p1 = S.p0 + S.n;
      Acc acc = (S.flags & kSegFirst) ? Acc(0) : state[static_cast<uint64_t>(S.slot) * 32 + lane];
      uint64_t base = p0 - S.lane0;
      {  // head chunk (positions before p0 belong to the previous segment)
        const uint64_t j = base + lane;
        if (j >= p0 && j < p1) acc = Ops::add(acc, Ops::prod(ld_stream(val + j), xs[ld_stream(col + j) - xlo]));
        base += 32;
      }
      constexpr int U = 8;
      for (; base + 32 * U <= p1; base += 32 * U) {
        I c[U];
        V v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          c[u] = ld_stream(col + base + lane + 32 * u);
          v[u] = ld_stream(val + base + lane + 32 * u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc = Ops::add(acc, Ops::prod(v[u], xs[c[u] - xlo]));
      }
      for (; base < p1; base += 32) {
        const uint64_t j = base + lane;
        if (j < p1) acc = Ops::add(acc, Ops::prod(ld_stream(val + j), xs[ld_stream(col + j) - xlo]));
      }
      if (S.flags & kSegLast) {
#pragma unroll
        for (int off = 16; off >= 1; off /= 2) acc = Ops::add(acc, __shfl_down_sync(kFull, acc, off));
        if (lane == 0) y[S.row] = static_cast<double>(acc);
      } else {
        state[static_cast<uint64_t>(S.slot) * 32 + lane] = acc;
      }
    }
    __syncthreads();  // every warp is done with xs before the next tile's TMA
  }
}

}  // namespace dg
