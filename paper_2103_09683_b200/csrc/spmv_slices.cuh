// spmv_slices.cuh -- the tile kernel over the slice stream (warp-contiguous, 128-bit streaming).
//
// The slice stream is the binary16 matrix re-laid out once at dg_create for the tile kernel:
//   * per tile, 2 x warps contiguous runs of 4-chunk blocks (the plan groups the tile's segments
//     into runs, LPT on chunks, longest run first; the CTA's warps pull runs dynamically), tiles in
//     claim order;
//   * a chunk is 32 words, one per logical lane of ONE segment: word l of a segment's chunk j is
//     the nonzero at position base0 + 32 j + l (base0 = the row's lane grid, Segment::lane0), so
//     lane l still owns the reference's lane l (positions start + l, start + l + 32, ...);
//     positions outside the segment are neutral words (value +0, the window's zero slot);
//   * a word is (slot << 16) | binary16 bits: the slot indexes the tile's x-window buffer
//     directly (column - xlo, or the replica slot of spmv_tiles.cuh) -- 4 bytes per nonzero,
//     for U32-indexed matrices too;
//   * 4 consecutive chunks form one 512-byte block stored lane-major (word 4 l + k = chunk k,
//     lane l), so each lane fetches its next 4 chunk words with one 16-byte load: a batch of
//     8 chunks is two fully coalesced LDG.128 per lane, aligned to 128-byte lines.
// Compared with the row-ordered stream (k_tiles): no segment-edge lines fetched twice (adjacent
// rows of the row-ordered stream sit in unrelated tiles), no misaligned 2-line chunk requests, no
// masked edge batches; the price is the neutral padding (< 32 words per segment end, < 8 chunks
// per run).  Results are bit-identical: each lane adds the same products in the same
// order from +0.0, and a neutral word adds +0 * (+0.0) = +0.0, the identity of an accumulator
// that is never -0.0.
#pragma once

#include "common.cuh"
#include "spmv_kernels.cuh"
#include "spmv_tiles.cuh"

namespace dg {

// per (tile, warp): first chunk and first segment of the warp's run; entry t * WARPS + w, with one
// sentinel at the end (runs are contiguous in tile order)
struct WarpRange {
  uint32_t chunk;
  uint32_t seg;
};
// the kernel's segment descriptor (16 bytes, one LDG.128)
struct SliceSeg {
  uint32_t row;
  uint32_t slot;   // carried-partials slot (split rows)
  uint32_t nch;    // chunks
  uint32_t flags;  // kSegFirst | kSegLast
};

constexpr int kSliceU = 8;      // chunks per batch (two 512-byte blocks)
#ifndef DG_SLICE_PAD
#define DG_SLICE_PAD 8
#endif
constexpr int kSliceBlock = 4;  // chunks per block
constexpr int kSlicePad = DG_SLICE_PAD;  // runs are padded to whole multiples of this many chunks (whole batches)

__device__ __forceinline__ uint4 ld_stream16(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// One warp's run: nblk 4-chunk blocks starting at chunk c0 (a multiple of 8), consumed in batches
// of two blocks (runs are padded to whole batches with neutral words: the zero slot, value +0).
// Software pipeline: batch b + 1 is in flight in registers while batch b is gathered and
// accumulated; lanes 0..7 prefetch the 8 lines of batch b + 1 + P into L2.  r02: whole-batch
// padding (no guarded second load, no neutral fill), a pointer-stepped prefetch stream and
// mask-predicated segment ends (products once) trimmed the per-batch instructions.
// x sources of a run: the tile's shared-memory window (indexed by slot) or global x (dense rows:
// their 32 lanes read consecutive columns, through L1 / L2)
template <typename Acc>
struct XSmem {
  const Acc* base;
  __device__ __forceinline__ Acc operator[](uint32_t i) const { return base[i]; }
};
template <typename Acc>
struct XGlob {
  const Acc* __restrict__ x;
  __device__ __forceinline__ Acc operator[](uint32_t i) const { return __ldg(x + i); }
};

template <typename Acc, int P, bool CARRY, class XS = XSmem<Acc>, int U = kSliceU>
__device__ __forceinline__ void run_slice(const uint4* __restrict__ blocks, uint32_t c0, uint32_t nblk,
                                          const SliceSeg* __restrict__ sseg, uint32_t s0,
                                          uint32_t s1, const XS xs, const Carry<Acc>& carry, double* __restrict__ y,
                                          const GatherTargets& gt, uint32_t lane) {
  using Ops = AccOps<Acc>;
  static_assert(U == 4 || U == 8, "a batch is one or two 4-chunk blocks");
  constexpr uint32_t BL = U / kSliceBlock;  // blocks per batch
  if (nblk == 0) return;
  // runs are padded to whole batches (kSlicePad = 8 chunks = 2 blocks): every block of every
  // batch exists, so the loads need no guard and no neutral fill
  static_assert(kSlicePad % (BL * kSliceBlock) == 0, "runs must hold whole batches");
  const uint32_t nb = nblk / BL;  // batches
  // current segment and the next one's descriptor (loaded one segment ahead)
  uint32_t si = s0;
  SliceSeg cur = sseg[si];
  SliceSeg nxt = si + 1 < s1 ? sseg[si + 1] : SliceSeg{0, 0, 0, 0};
  uint32_t left = cur.nch;
  Acc acc = CARRY ? carry.in(cur.slot, cur.flags, lane) : Acc(0);
  const uint4* p = blocks + static_cast<uint64_t>(c0 / 4) * 32 + lane;  // block c0/4, lane's 16 B
  uint4 a0 = ld_stream16(p), a1 = BL > 1 ? ld_stream16(p + 32) : a0, b0, b1;
  // L2 prefetch stream: lanes 0 .. 4 BL - 1 each own one 128-byte line of a batch (512 BL bytes),
  // P batches ahead
  constexpr uint32_t kBatchBytes = 512 * BL;
  const char* pf = reinterpret_cast<const char*>(p - lane) + 128 * lane;
  if constexpr (P > 0) {
#pragma unroll
    for (int k = 1; k <= P; ++k)
      if (lane < 4 * BL && static_cast<uint32_t>(k) < nb)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + kBatchBytes * k));
    pf += kBatchBytes * (P + 1);
  }
  auto finish = [&]() {  // the current segment ends with the chunk just added
    if (!CARRY || (cur.flags & kSegLast)) {
#pragma unroll
      for (int off = 16; off >= 1; off /= 2) acc = Ops::add(acc, __shfl_down_sync(kFull, acc, off));
      if (lane == 0) {
        y[cur.row] = static_cast<double>(acc);
        gt.store(cur.row, static_cast<double>(acc));
      }
    } else {
      if constexpr (CARRY) carry.out(cur.slot, cur.flags, lane, acc);
    }
    ++si;
    if (si < s1) {
      cur = nxt;
      left = cur.nch;
      acc = CARRY ? carry.in(cur.slot, cur.flags, lane) : Acc(0);
      if (si + 1 < s1) nxt = sseg[si + 1];
    } else {
      left = 0xFFFFFFFFu;  // the run's padding chunks: neutral words, no segment
      acc = Acc(0);
    }
  };
  auto consume = [&](const uint4& q0, const uint4& q1) {
    const uint32_t r[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    Acc xv[U];
#pragma unroll
    for (int k = 0; k < U; ++k) xv[k] = xs[r[k] >> 16];
    if (left > static_cast<uint32_t>(U)) {  // the whole batch inside one segment
#pragma unroll
      for (int k = 0; k < U; ++k)
        acc = Ops::add(acc, Ops::prod(static_cast<uint16_t>(r[k] & 0xFFFFu), xv[k]));
      left -= U;
      return;
    }
    // segment end(s) inside the batch: the products once, then each segment's chunks [k, e)
    // added in position order under a warp-uniform bit mask, one finish() per segment end
    Acc pr[U];
#pragma unroll
    for (int j = 0; j < U; ++j) pr[j] = Ops::prod(static_cast<uint16_t>(r[j] & 0xFFFFu), xv[j]);
    uint32_t k = 0;
    do {
      const uint32_t e = left >= U - k ? static_cast<uint32_t>(U) : k + left;
      const uint32_t m = (0xFFu >> (8 - (e - k))) << k;  // chunks k .. e-1
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (m & (1u << j)) acc = Ops::add(acc, pr[j]);
      left -= e - k;
      k = e;
      if (left == 0) finish();
    } while (k < static_cast<uint32_t>(U));
  };
  constexpr uint32_t kStep = 32 * BL;  // uint4 per lane-major batch
  uint32_t bi = 0;
  for (;;) {
    // step A: consume a, load b
    if (bi + 1 < nb) {
      b0 = ld_stream16(p + kStep);
      if constexpr (BL > 1) b1 = ld_stream16(p + kStep + 32);
    }
    if constexpr (P > 0) {
      if (lane < 4 * BL && bi + 1 + P < nb) asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
      pf += kBatchBytes;
    }
    consume(a0, a1);
    if (++bi == nb) break;
    p += kStep;
    // step B: consume b, load a
    if (bi + 1 < nb) {
      a0 = ld_stream16(p + kStep);
      if constexpr (BL > 1) a1 = ld_stream16(p + kStep + 32);
    }
    if constexpr (P > 0) {
      if (lane < 4 * BL && bi + 1 + P < nb) asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
      pf += kBatchBytes;
    }
    consume(b0, b1);
    if (++bi == nb) break;
    p += kStep;
  }
}

// Persistent: one CTA per SM, NB x-window buffers of wcap elements (dynamic smem), element
// wcap - 1 of each buffer is the zero slot the neutral words gather.
template <typename Acc, int WARPS, int P, bool CARRY, int NB = 2, int U = kSliceU>
__global__ void __launch_bounds__(WARPS * 32, 1)
    k_slices(const uint4* __restrict__ blocks, XSource<Acc> xsrc, const Tile* __restrict__ tiles,
             uint32_t n_tiles, uint32_t runs, const WarpRange* __restrict__ ranges,
             const SliceSeg* __restrict__ sseg, Carry<Acc> carry, double* __restrict__ y,
             uint32_t* __restrict__ counter, uint32_t wcap, BlockSignal sig,
             const __grid_constant__ GatherTargets gt, TileTrace tr) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // full[b]: the window of buffer b has landed (TMA complete_tx); empty[b]: every warp has left
  // buffer b (WARPS x 32 arrivals) -- the refill of b waits on it, so the window's readers are ordered
  // before its next TMA overwrite by barrier operations (visible to compute-sanitizer racecheck)
  __shared__ __align__(8) uint64_t full[NB], empty[NB];
  __shared__ uint32_t tile_of[NB], done[NB], run_next[NB];
  Acc* const xbuf0 = reinterpret_cast<Acc*>(smem_raw);
  const uint32_t lane = threadIdx.x & 31;
  const Acc* __restrict__ x = xsrc.x;

  __shared__ uint32_t blk_of[NB];
  // warp-collective: put tile t into buffer b -- stage its x window by TMA (lane 0) and prefetch
  // the first 2 KB of each of its runs plus its segment descriptors into L2 (the lanes in
  // parallel), so the warps start the tile's runs on L2 hits.  The tile_of / done / run_next
  // stores precede lane 0's arrive on full[b] (release), which every reader acquires.
  auto refill = [&](int b, uint32_t t) {
    if (t < n_tiles) {
      const Tile T = tiles[t];
      if (lane == 0) {
        tile_of[b] = t;
        blk_of[b] = T.blk;
        done[b] = 0;
        run_next[b] = 0;
        if (tr.cta) {
          tr.tile[3ull * t] = gtimer_ns();
          tr.tile[3ull * t + 2] = blockIdx.x | (static_cast<unsigned long long>(T.seg1 - T.seg0) << 16);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        char* const dst0 = reinterpret_cast<char*>(xbuf0 + b * wcap);
        constexpr uint32_t kAl = 16 / sizeof(Acc);
        uint32_t total = 0;
        const uint32_t nrep = T.nrep;
        for (uint32_t r = 0; r < nrep; ++r)
          total += (T.xlen + rep_shift(r) + kAl - 1) / kAl * kAl * static_cast<uint32_t>(sizeof(Acc));
        mbar_arrive_expect_tx(&full[b], total);
        for (uint32_t r = 0; r < nrep; ++r) {
          const uint32_t sh = rep_shift(r);
          const uint32_t bytes = (T.xlen + sh + kAl - 1) / kAl * kAl * static_cast<uint32_t>(sizeof(Acc));
          const Acc* base = (sh % kAl) ? xsrc.x1 : x;
          const char* src = reinterpret_cast<const char*>(base + T.xlo) - sh * sizeof(Acc);
          char* dst = dst0 + static_cast<size_t>(r) * xsrc.rep_stride * sizeof(Acc);
          for (uint32_t off = 0; off < bytes; off += 32768u)
            tma_load_1d(dst + off, src + off, min(32768u, bytes - off), &full[b]);
        }
      }
      const WarpRange* R = ranges + static_cast<uint64_t>(t) * runs;
      for (uint32_t w = lane; w < runs; w += 32) {
        const uint32_t c = R[w].chunk, ce = R[w + 1].chunk;
        if (ce > c)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(blocks + static_cast<uint64_t>(c / 4) * 32),
                       "r"(min(2048u, (ce - c) * 128u)));
      }
      if (lane == 0) {
        const uint64_t sb = reinterpret_cast<uint64_t>(sseg + R[0].seg) & ~15ull;
        const uint64_t se = reinterpret_cast<uint64_t>(sseg + R[runs].seg);
        if (se > sb)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sb),
                       "r"(static_cast<uint32_t>(se - sb)));
      }
    } else if (lane == 0) {
      tile_of[b] = t;
      mbar_arrive(&full[b]);  // terminal: completes the phase with tile_of[b] >= n_tiles
    }
    __syncwarp();
  };

  if (threadIdx.x < NB) xbuf0[threadIdx.x * wcap + wcap - 1] = Acc(0);  // zero slots
  if (threadIdx.x == 0)
    for (int i = 0; i < NB; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], WARPS * 32);  // every thread arrives
    }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  // the first NB tiles are static (CTA i: tiles i, i + grid, ...; no claim latency at the start),
  // staged by warps 0 .. NB-1 in parallel; later tiles are claimed in order from the counter
  const uint32_t warp = threadIdx.x / 32;
  if (warp < NB) refill(static_cast<int>(warp), blockIdx.x + warp * gridDim.x);

  uint32_t phases = 0;
  int b = 0;
  const long long clk0 = clock64();
  long long wait_cyc = 0;
  if (tr.cta && threadIdx.x == 0) tr.cta[4ull * blockIdx.x] = gtimer_ns();
  for (;;) {
    if (tr.cta) {
      const long long w0 = clock64();
      mbar_wait(&full[b], (phases >> b) & 1u);
      wait_cyc += clock64() - w0;
    } else {
      mbar_wait(&full[b], (phases >> b) & 1u);
    }
    phases ^= 1u << b;
    const uint32_t t = *reinterpret_cast<volatile uint32_t*>(&tile_of[b]);
    if (t >= n_tiles) break;
    // pull the tile's runs (longest first) until none is left
#ifndef DG_SLICE_DYN
#define DG_SLICE_DYN 1
#endif
    for (uint32_t it = 0;; ++it) {
      uint32_t k = 0;
      if (DG_SLICE_DYN) {
        if (lane == 0) k = atomicAdd(&run_next[b], 1u);
        k = __shfl_sync(kFull, k, 0);
      } else {
        k = it == 0 ? threadIdx.x / 32 : runs;  // static: run = warp (runs == WARPS)
      }
      if (k >= runs) break;
      const WarpRange r0 = ranges[static_cast<uint64_t>(t) * runs + k];
      const WarpRange r1 = ranges[static_cast<uint64_t>(t) * runs + k + 1];
      run_slice<Acc, P, CARRY, XSmem<Acc>, U>(blocks, r0.chunk, (r1.chunk - r0.chunk) / kSliceBlock, sseg,
                                              r0.seg, r1.seg, XSmem<Acc>{xbuf0 + b * wcap}, carry, y,
                                              gt, lane);
    }
    __syncwarp();
    if (lane == 0) {
      if (sig.left) __threadfence(); else __threadfence_block();
    }
    __syncwarp();
    // release: every lane's reads of buffer b (the window, tile_of[b]) are done -- each thread
    // arrives for itself, so the ordering does not rest on __syncwarp (racecheck models it so)
    mbar_arrive(&empty[b]);
    uint32_t next = 0xFFFFFFFFu;  // the last warp to leave refills b with the next claimed tile
    if (lane == 0 && atomicAdd(&done[b], 1u) == WARPS - 1) {
      mbar_wait(&empty[b], ((phases >> b) & 1u) ^ 1u);  // acquire every warp's release
      const uint32_t blk = blk_of[b];
      if (tr.cta) tr.tile[3ull * t + 1] = gtimer_ns();
      if (sig.left && blk != kNoBlock) {
        __threadfence();
        if (atomicSub(&sig.left[blk], 1u) == 1u) {
          __threadfence();
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(sig.flag + blk),
                       "r"(sig.epoch)
                       : "memory");
        }
      }
      next = atomicAdd(counter, 1u) + NB * gridDim.x;
    }
    next = __shfl_sync(kFull, next, 0);
    if (next != 0xFFFFFFFFu) refill(b, next);
    __syncwarp();
    b = b + 1 == NB ? 0 : b + 1;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tr.cta && lane == 0) {
    atomicAdd(&tr.cta[4ull * blockIdx.x + 2], static_cast<unsigned long long>(wait_cyc));
    atomicAdd(&tr.cta[4ull * blockIdx.x + 3], static_cast<unsigned long long>(clock64() - clk0));
    atomicMax(&tr.cta[4ull * blockIdx.x + 1], gtimer_ns());
  }
}

// ---- dense rows over the slice layout ---------------------------------------------------------
// The dense rows k_dense owns (>= 3/4 of their span, the longest rows) as runs of one segment
// each, longest first, in the same lane-major 4-chunk blocks: each row starts on a 1-KB batch
// (its lane grid = the row's, lane0 0) and is padded to whole batches with neutral words whose
// column is `cols` (x[cols] is a staged +0.0).  Warps of persistent 8-warp CTAs pull rows
// longest first and stream them with the tile kernel's run pipeline (two LDG.128 per lane per
// 8-chunk batch, L2 prefetch P batches ahead); x comes from global memory through L1.
template <typename Acc, int P>
__global__ void __launch_bounds__(256)
    k_dense_slices(const uint4* __restrict__ blocks, const WarpRange* __restrict__ ranges,
                   const SliceSeg* __restrict__ sseg, uint32_t n_rows, const Acc* __restrict__ x,
                   uint32_t* __restrict__ counter, double* __restrict__ y,
                   const __grid_constant__ GatherTargets gt) {
  // programmatic dependent launch: the tile kernel that follows may take each SM as soon as this
  // grid's CTAs there have exited (it touches other rows)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t lane = threadIdx.x & 31;
  const Carry<Acc> no_carry{nullptr};
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(counter, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (k >= n_rows) break;
    const uint32_t c0 = ranges[k].chunk, c1 = ranges[k + 1].chunk;
    run_slice<Acc, P, false>(blocks, c0, (c1 - c0) / kSliceBlock, sseg, k, k + 1, XGlob<Acc>{x},
                             no_carry, y, gt, lane);
  }
}

// ---- contiguous rows as values only ----------------------------------------------------------
// A row whose columns are lo, lo + 1, ..., lo + len - 1 needs no column words: position p reads
// x[lo + p].  k_dense_values streams such rows as binary16 values alone -- 2 bytes per nonzero
// instead of 4 -- in lane-major 8-chunk blocks (512 bytes: lane l's 16 bytes are its 8 values of
// chunks 8b .. 8b + 7, positions 32 c + l), each row starting on a block and padded to whole
// blocks with +0 values.  Lane l adds the same products in the same order from +0.0 as the
// reference's lane l (spmv.cpp:58-63); padding positions read x[zero_col] (a staged +0.0, never
// the caller's x: +0 * Inf would be NaN), so they add +0.0 exactly.  Warps of persistent 8-warp
// CTAs pull rows longest first; a batch is 16 chunks (two LDG.128 per lane), the next batch in
// flight in registers and an L2 prefetch stream P batches ahead; x comes through L1 (32 lanes
// read 32 consecutive elements per chunk).
struct DenseRow {
  uint32_t row;
  uint32_t lo;   // first column (written by k_build_values)
  uint32_t len;
  uint32_t blk;  // first 512-byte block of the row in the value stream
};
constexpr int kValueChunks = 8;  // chunks per 512-byte value block

template <typename Acc, int P>
__global__ void __launch_bounds__(256)
    k_dense_values(const uint4* __restrict__ vs, const DenseRow* __restrict__ rows, uint32_t n_rows,
                   const Acc* __restrict__ x, uint32_t zero_col, uint32_t* __restrict__ counter,
                   double* __restrict__ y, const __grid_constant__ GatherTargets gt) {
  // programmatic dependent launch: the kernel that follows may take each SM as soon as this
  // grid's CTAs there have exited (it touches other rows)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  using Ops = AccOps<Acc>;
  const uint32_t lane = threadIdx.x & 31;
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(counter, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (k >= n_rows) break;
    const DenseRow R = rows[k];
    const uint32_t nblk = ((R.len + 31) / 32 + kValueChunks - 1) / kValueChunks;
    const uint32_t nb = (nblk + 1) / 2;  // batches of two blocks
    const uint4* p = vs + static_cast<uint64_t>(R.blk) * 32 + lane;
    const Acc* xr = x + R.lo;
    const uint4 zero = make_uint4(0, 0, 0, 0);
    uint4 a0 = ld_stream16(p), a1 = nblk > 1 ? ld_stream16(p + 32) : zero, b0 = zero, b1 = zero;
    if constexpr (P > 0) {
#pragma unroll
      for (int j = 1; j <= P; ++j)
        if (lane < 8 && 2 * j + (lane >= 4 ? 1u : 0u) < nblk)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(p - lane + 64 * j) + 128 * lane));
    }
    Acc acc = Acc(0);
    for (uint32_t bi = 0; bi < nb; ++bi) {
      if (bi + 1 < nb) {
        b0 = ld_stream16(p + 64);
        b1 = 2 * bi + 3 < nblk ? ld_stream16(p + 96) : zero;
      }
      if constexpr (P > 0)
        if (lane < 8 && 2 * (bi + 1 + P) + (lane >= 4 ? 1u : 0u) < nblk)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(p - lane + 64 * (1 + P)) + 128 * lane));
      const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const uint32_t pos0 = bi * (2 * kValueChunks * 32) + lane;
      Acc xv[2 * kValueChunks];
      if (pos0 + (2 * kValueChunks - 1) * 32 < R.len) {  // interior batch
#pragma unroll
        for (int c = 0; c < 2 * kValueChunks; ++c) xv[c] = __ldg(xr + pos0 + 32 * c);
      } else {  // the row's last batch: positions past the end read the staged +0.0
#pragma unroll
        for (int c = 0; c < 2 * kValueChunks; ++c) {
          const uint32_t pos = pos0 + 32 * c;
          xv[c] = __ldg(pos < R.len ? xr + pos : x + zero_col);
        }
      }
#pragma unroll
      for (int c = 0; c < 2 * kValueChunks; ++c)
        acc = Ops::add(acc, Ops::prod(static_cast<uint16_t>(w[c / 2] >> (16 * (c & 1))), xv[c]));
      a0 = b0;
      a1 = b1;
      p += 64;
    }
#pragma unroll
    for (int off = 16; off >= 1; off /= 2) acc = Ops::add(acc, __shfl_down_sync(kFull, acc, off));
    if (lane == 0) {
      y[R.row] = static_cast<double>(acc);
      gt.store(R.row, static_cast<double>(acc));
    }
  }
}

// word index of (chunk c, lane l) in the lane-major 4-chunk blocks
__host__ __device__ __forceinline__ uint64_t slice_word(uint64_t c, uint32_t l) {
  return (c >> 2) * 128 + 4 * l + (c & 3);
}

}  // namespace dg
