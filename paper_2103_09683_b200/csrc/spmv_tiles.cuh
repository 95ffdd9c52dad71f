// spmv_tiles.cuh -- column-windowed tile kernel: x staged in shared memory by 1-D TMA.
//
// Why: the dose gather x[col[j]] is the dominant L1 cost of a lane-strided CSR SpMV (32 lanes of
// a sparse row touch ~16 sectors of x per request; v0 ncu: 6.5 sectors/request, 42% of HBM).  The
// row plan (plan.cu) sorts row segments by first column and cuts them into tiles whose column
// window [xlo, xlo + xlen) fits in shared memory; the CTA stages windows with cp.async.bulk
// (SASS UBLKCP) into a 2-buffer ring, and its warps gather x with LDS instead of L1/L2 loads.
//
// Pipeline (one CTA of WARPS warps per SM, no CTA-wide barrier in the steady state):
//   buffer b holds tile tile_of[b]; warps pull its segments with a shared-memory counter; the last
//   warp to leave buffer b claims the next tile from the global counter and re-arms b (TMA +
//   mbarrier expect_tx) while the other warps already work on buffer b^1.
// Inside a segment each lane software-pipelines its matrix loads: batch k+1 (U positions per
// lane) is in flight while batch k is gathered and accumulated.
//
// Exactness: a segment is a contiguous position range [p0, p0 + n) of one row; physical lane l
// owns the row's logical lane l (positions j with (j - row_start) % 32 == l), accumulates them in
// increasing j from +0.0 (or from the carried partial of the row's previous segment, written by
// the previous wave), and the last segment applies the stride-halving tree.  This is exactly
// ddm::rowchunk_rows with lane_width 32 (src/spmv.cpp:48-68), split over waves only at segment
// boundaries, where the lane partials are stored and reloaded unchanged.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "spmv_kernels.cuh"

// DG_ROTATE=1: rotated lane grid (aligned chunk loads).  Bit-identical, measured: C2 kernel
// 2.634 vs 2.633 ms, C1 0.156 vs 0.141, C4 6.69 vs 6.65 (every row's first batch becomes an
// edge batch) -- off.
#ifndef DG_ROTATE
#define DG_ROTATE 0
#endif

namespace dg {

constexpr bool kRotate = DG_ROTATE;  // rotated lane grid (SegRun) in k_tiles and k_dense

struct Segment {  // 24 bytes
  uint64_t p0;     // first position (shard-local nnz index)
  uint32_t n;      // positions [p0, p0 + n)
  uint32_t row;    // shard-local row
  uint32_t slot;   // carried-partials slot (split rows), else unused
  uint16_t lane0;  // (p0 - row_start) % 32
  uint16_t flags;  // kSegFirst | kSegLast
};
constexpr uint16_t kSegFirst = 1, kSegLast = 2, kSegGlobalX = 4;
constexpr uint32_t kSegWaveShift = 8;  // flags >> 8: the segment's index within its row (wave)

// Lane partials carried between the segments (waves) of a split row.  Segment k of a row writes
// its 32 lane partials to slot (row, k) -- Segment::slot -- and segment k + 1 reads them from
// slot - 1.  Slots hold kCarryEmpty (a signalling NaN: arithmetic never produces one, every
// partial is a quieted sum) until written, and the reader puts kCarryEmpty back for the next
// dose, so a lane's partial is its own readiness flag: lane l of segment k + 1 spins only on its
// own 8 bytes (one naturally aligned store / load: never torn), with no acquire/release pair and
// no warp-wide flag.  That lets the warp `peek` the next segment's carried partials when it
// grabs that segment (one segment ahead) and find them already in registers at the switch.
// The same code serves one launch per wave and all waves in one launch (fused).  Fused, the
// wait is deadlock-free in a persistent grid: the plan lists a row's segment k before its
// segment k + 1 (plan.cu), tiles are claimed in list order and a warp takes its segments in
// claim order, so a waiting segment only waits on an earlier-listed segment, and the earliest
// unfinished segment never waits.
template <typename Acc>
struct CarryBits;
template <>
struct CarryBits<double> {
  static constexpr unsigned long long kEmpty = 0x7FF0000000000DC5ull;  // sNaN
  __device__ static __forceinline__ bool empty(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == kEmpty;
  }
  __device__ static __forceinline__ double empty_value() {
    return __longlong_as_double(static_cast<long long>(kEmpty));
  }
};
template <>
struct CarryBits<float> {
  static constexpr unsigned kEmpty = 0x7F800DC5u;  // sNaN
  __device__ static __forceinline__ bool empty(float v) { return __float_as_uint(v) == kEmpty; }
  __device__ static __forceinline__ float empty_value() { return __uint_as_float(kEmpty); }
};

template <typename Acc>
struct Carry {
  using B = CarryBits<Acc>;
  Acc* state;  // 32 partials per slot
  __device__ __forceinline__ Acc* at(uint32_t slot, uint32_t lane) const {
    return state + static_cast<uint64_t>(slot) * 32 + lane;
  }
  // start loading the partials segment (slot, flags) continues from (first segments: none).
  // ld.global.cg: from L2, the coherence point (never a stale L1 line)
  __device__ __forceinline__ Acc peek(uint32_t slot, uint32_t flags, uint32_t lane) const {
    return (flags & kSegFirst) ? Acc(0) : __ldcg(at(slot - 1, lane));
  }
  // the partial to start from: the peeked value, re-read (ld.global.cv: fetched again every
  // time) until the writer has stored it; the slot is emptied again for the next dose
  __device__ __forceinline__ Acc take(uint32_t slot, uint32_t flags, uint32_t lane, Acc v) const {
    if (flags & kSegFirst) return Acc(0);
    Acc* p = at(slot - 1, lane);
    while (B::empty(v)) {
      __nanosleep(32);
      v = __ldcv(p);
    }
    __stcg(p, B::empty_value());
    return v;
  }
  __device__ __forceinline__ Acc in(uint32_t slot, uint32_t flags, uint32_t lane) const {
    return take(slot, flags, lane, peek(slot, flags, lane));
  }
  __device__ __forceinline__ void out(uint32_t slot, uint32_t /*flags*/, uint32_t lane, Acc acc) const {
    __stcg(at(slot, lane), acc);
  }
};

// fill every carry slot with kCarryEmpty (at dg_create)
template <typename Acc>
__global__ void k_carry_init(Acc* __restrict__ state, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    state[i] = CarryBits<Acc>::empty_value();
}

struct Tile {  // 16 bytes
  uint32_t xlo;   // x window start (16-byte aligned)
  uint16_t xlen;  // x window length in elements (16-byte multiple; 0: global-x tile)
  uint8_t blk;    // output row block whose rows this tile finishes (kNoBlock: none)
  uint8_t nrep;   // x replicas in the window: 1 (column mode) or kReplicas (slot mode)
  uint32_t seg0, seg1;
};
constexpr uint8_t kNoBlock = 0xFF;

// ---- replicated x windows (slot mode) -------------------------------------------------------
// A warp's 8-byte x gather is served half-warp by half-warp, each half in as many shared-memory
// wavefronts as the most-loaded of the 16 bank pairs (distinct words; scripts/micro/lds_model.cu
// measured it on B200).  Sparse rows gather random columns, so a half-warp's 16 columns land on
// ~2.45 words per bank pair at worst on average: 4.9 wavefronts per 32 nonzeros instead of 2
// (r01 ncu: 41% of the kernel's shared wavefronts were conflicts).  A slot-mode tile holds its
// x window kReplicas times, replica r shifted by kRepShift[r] bank pairs, and the plan rewrites
// each nonzero's 16-bit column of the Packed16 stream into the *slot* it gathers from: replica
// chosen per nonzero so that every half-warp's lanes spread over the bank pairs with the smallest
// possible maximum load (an exact b-matching per half-chunk, k_assign_slots in plan.cu).  Same
// 4 bytes per nonzero; the column is recovered from (tile.xlo, slot) -- the decode is exact.
constexpr uint32_t kReplicas = 3;
__host__ __device__ constexpr uint32_t rep_shift(uint32_t r) { return r == 0 ? 0u : r == 1 ? 4u : 11u; }
// slot of column c in replica r of a window starting at xlo, replica regions `stride` apart
__host__ __device__ __forceinline__ uint32_t slot_of(uint32_t c, uint32_t xlo, uint32_t r,
                                                     uint32_t stride) {
  return r * stride + (c - xlo) + rep_shift(r);
}
__host__ __device__ __forceinline__ uint32_t col_of_slot(uint32_t slot, uint32_t xlo, uint32_t stride) {
  const uint32_t r = slot / stride;
  return xlo + (slot - r * stride) - rep_shift(r);
}

// Row-block completion signals: the CTA finishing the last tile of output row block k publishes
// flag[k] = epoch, which a copy stream waits on (cuStreamWaitValue32) to move block k of d to the
// host while the kernel still works on later blocks.  left == nullptr disables signalling.
struct BlockSignal {
  uint32_t* left;  // tiles still to finish per block (reset before each dose)
  uint32_t* flag;
  uint32_t epoch;
};

// Diagnostic timeline (DG_TRACE, dg_debug_trace): per CTA {start ns, end ns, cycles warps spent
// waiting for a window buffer, warp-cycles alive}; per tile {claim ns, finish ns, CTA}.
// cta == nullptr disables it (the default).
struct TileTrace {
  unsigned long long* cta;
  unsigned long long* tile;
};
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

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
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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

// ---- slot assignment ---------------------------------------------------------------------------
// One half-chunk: the <= 16 positions of a segment that one half-warp gathers in one LDS.64.
// Each position may read its column from any of the kReplicas replicas (bank pair
// (c - xlo + shift_r) mod 16); masked-off lanes of a partial half read one filler slot (bank
// pair fb).  Find the replica choice minimising the largest number of distinct words on one bank
// pair -- the wavefronts that half costs -- by raising the per-bank capacity L from its lower
// bound until a b-matching of positions to bank pairs exists (BFS augmenting paths; <= 16 x 3
// edges).  Deterministic: the same stream and plan always give the same slots.
struct HalfMatch {
  uint8_t opt[16][kReplicas];  // bank pair per (position, replica)
  int8_t asg[16];              // replica chosen per position (-1: none yet)
  uint8_t load[16];
  int n;

  __device__ int bank(int i) const { return opt[i][asg[i]]; }
  // one augmenting path from position s under capacities cap[]; false if none
  __device__ bool augment(int s, const uint8_t* cap) {
    int8_t via[16];          // via[b]: position that reached bank pair b
    uint8_t q[16];
    uint32_t seen_b = 0, seen_p = 1u << s;
    int qh = 0, qt = 0;
    q[qt++] = static_cast<uint8_t>(s);
    int found = -1;
    while (qh < qt && found < 0) {
      const int u = q[qh++];
      for (int r = 0; r < static_cast<int>(kReplicas) && found < 0; ++r) {
        const int b = opt[u][r];
        if ((seen_b >> b) & 1u) continue;
        seen_b |= 1u << b;
        via[b] = static_cast<int8_t>(u);
        if (load[b] < cap[b]) { found = b; break; }
        for (int v = 0; v < n; ++v)
          if (asg[v] >= 0 && bank(v) == b && !((seen_p >> v) & 1u)) {
            seen_p |= 1u << v;
            q[qt++] = static_cast<uint8_t>(v);
          }
      }
    }
    if (found < 0) return false;
    int b = found;
    for (;;) {  // shift every position on the path one step: only `found` gains a word
      const int u = via[b];
      const int prev = asg[u] >= 0 ? bank(u) : -1;
      for (int r = 0; r < static_cast<int>(kReplicas); ++r)
        if (opt[u][r] == b) { asg[u] = static_cast<int8_t>(r); break; }
      if (prev < 0) break;
      b = prev;
    }
    ++load[found];
    return true;
  }
  __device__ void solve(bool filler, int fb) {
    for (int L = (n + 15) / 16 > 0 ? (n + 15) / 16 : 1;; ++L) {
      uint8_t cap[16];
      for (int b = 0; b < 16; ++b) {
        cap[b] = static_cast<uint8_t>(L - (filler && b == fb ? 1 : 0));
        load[b] = 0;
      }
      for (int i = 0; i < n; ++i) asg[i] = -1;
      bool ok = true;
      for (int i = 0; i < n && ok; ++i) ok = augment(i, cap);
      if (ok) return;
    }
  }
};

// x sources: the tile's shared-memory window, or global x (L1/L2) for dense wide rows whose
// column span exceeds a window (kSegGlobalX) -- their 32 lanes read 32 consecutive x entries.
// The window is indexed by the stream's 16-bit field directly: `base` is the buffer minus xlo in
// column mode (field = column) and the buffer itself in slot mode (field = slot); `safe` is a
// valid field value for masked-off lanes.
template <typename Acc>
struct XWindow {
  const Acc* base;
  uint32_t safe;
  __device__ __forceinline__ Acc operator()(uint32_t c) const { return base[c]; }
};
template <typename Acc>
struct XGlobal {
  const Acc* x;
  __device__ __forceinline__ Acc operator()(uint32_t c) const { return __ldg(x + c); }
};

// A segment as the warp's pipeline sees it: batches of U chunks of 32 positions aligned to the
// row's lane grid (chunk c covers base0 + 32c + lane); positions outside [p0, p1) are masked.
struct SegRun {
  uint64_t base0;   // chunk grid start: positions base0 + rel, rel in [lo, hi) are the segment's
  uint32_t lo, hi;  // (unrotated: base0 = the row's lane grid, lo = lane0, hi = lane0 + n)
  uint32_t nbatch, row, slot, flags;
  uint32_t rot;     // rotated grid: physical lane p holds the row's logical lane (p - rot) & 31
};
// Rotated lane grid (ROT): chunks start on 128-byte boundaries of the stream (base0 rounded down
// to a multiple of 32 positions), so every chunk load is one aligned line instead of straddling
// two.  Physical lane p then holds the row's logical lane (p - rot) & 31 with rot = row_start &
// 31 -- the same for every segment of a row, so carried partials stay lane-consistent -- and
// still sees that lane's positions in increasing order; positions before the row are masked
// like any edge; the final tree shuffles by (lane + w) & 31 and lane rot holds the result.
template <int U, bool ROT = false>
__device__ __forceinline__ SegRun seg_run_at(uint64_t base0, uint32_t lo, uint32_t n) {
  SegRun r;
  const uint32_t rot = ROT ? static_cast<uint32_t>(base0 & 31u) : 0u;
  r.base0 = base0 - rot;
  r.lo = lo + rot;
  r.hi = lo + n + rot;
  r.rot = rot;
  r.nbatch = ((r.hi + 31) / 32 + U - 1) / U;
  return r;
}
template <int U, bool ROT = false>
__device__ __forceinline__ SegRun seg_run(const Segment& S) {
  SegRun r = seg_run_at<U, ROT>(S.p0 - S.lane0, S.lane0, S.n);
  r.row = S.row;
  r.slot = S.slot;
  r.flags = S.flags;
  return r;
}
// The reference's stride-halving tree (src/spmv.cpp:64-65) over the 32 logical lanes; returns
// true on the lane that holds the row's result.
template <bool ROT, typename Acc>
__device__ __forceinline__ bool row_tree(Acc& acc, uint32_t lane, uint32_t rot) {
  using Ops = AccOps<Acc>;
#pragma unroll
  for (int off = 16; off >= 1; off /= 2) {
    if constexpr (ROT) acc = Ops::add(acc, __shfl_sync(kFull, acc, (lane + off) & 31u));
    else acc = Ops::add(acc, __shfl_down_sync(kFull, acc, off));
  }
  return lane == (ROT ? rot : 0u);
}

// Issue batch b of segment s: U predicated requests (one 128-B request per chunk for Packed16).
// Masked-off lanes get a filler element whose column (`safe_col`, the tile's window start) is a
// valid x index, so the gather below needs no predicate; only the accumulation is masked.
// Interior batches (every lane's U chunks inside the segment; warp-uniform test) load unmasked
// and report kFullMask; edge batches are masked per chunk.
template <int U>
constexpr uint32_t kFullMask = (1u << U) - 1u;


template <int U, class M>
__device__ __forceinline__ uint32_t load_batch(const M& mat, typename M::Raw* r, const SegRun& s,
                                               uint32_t b, uint32_t lane, uint32_t safe_col) {
  const uint32_t b0 = b * (32 * U);
  const uint64_t base = s.base0 + b0 + lane;
  if (b0 >= s.lo && b0 + 32 * U <= s.hi) {
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = mat.load(base + 32 * u);
    return kFullMask<U>;
  }
  // chunk u holds position rel = b0 + lane + 32u: valid for u in [ulo, uhi) with
  // uhi = ceil((hi - b0 - lane) / 32) and ulo = ceil((lo - b0 - lane) / 32), clamped to [0, U]
  const int t0 = static_cast<int>(b0 + lane);
  const int th = static_cast<int>(s.hi) - t0, tl = static_cast<int>(s.lo) - t0;
  const uint32_t uhi = th <= 0 ? 0u : min(static_cast<uint32_t>(U), static_cast<uint32_t>(th + 31) >> 5);
  const uint32_t ulo = tl <= 0 ? 0u : min(static_cast<uint32_t>(U), static_cast<uint32_t>(tl + 31) >> 5);
  const uint32_t mask = ((1u << uhi) - 1u) & ~((1u << ulo) - 1u);
  // (measured, rejected: skipping the chunks no lane needs -- a warp-uniform count guarding
  //  each chunk's load, gather and add -- C2 kernel 2.76 vs 2.63 ms, C4 7.55 vs 6.68: the
  //  guarded chunks no longer batch their LDS gathers ahead of the arithmetic)
#pragma unroll
  for (int u = 0; u < U; ++u) {
    r[u] = M::filler(safe_col);
    if (mask & (1u << u)) r[u] = mat.load(base + 32 * u);
  }
  return mask;
}

// L2 prefetch of batches [b, b + P) of segment s: lane l < U touches line l of each batch.
// Prefetches hold no registers, so the stream runs P batches ahead of the register pipeline.
template <int U, int P, class M>
__device__ __forceinline__ void prefetch_batches(const M& mat, const SegRun& s, uint32_t b,
                                                 uint32_t lane) {
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const uint32_t rel = (b + k) * (32 * U);
    if (rel < s.hi) mat.template prefetch_batch<U>(s.base0 + rel, s.hi - rel, lane);
  }
}

// Gather x for a loaded batch and accumulate in position order.  Masked chunks add +0.0, which
// is the identity here: an accumulator that starts at +0.0 and only ever adds is never -0.0
// (round-to-nearest turns exact cancellation into +0.0), and x + (+0.0) == x for x != -0.0.
template <int U, class M, typename Acc, class X>
__device__ __forceinline__ void consume_batch(const typename M::Raw* r, uint32_t mask, const X& xr,
                                              Acc& acc) {
  using Ops = AccOps<Acc>;
  // wide batches gather x in groups of 8 (bounded live registers); U = 8 is one group
  constexpr int G = U > 8 ? 4 : U;
#pragma unroll
  for (int g = 0; g < U; g += G) {
    Acc xv[G];
#pragma unroll
    for (int u = 0; u < G; ++u) xv[u] = xr(M::c_of(r[g + u]));
    if (mask == kFullMask<U>) {
#pragma unroll
      for (int u = 0; u < G; ++u) acc = Ops::add(acc, Ops::prod(M::v_of(r[g + u]), xv[u]));
    } else {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const Acc p = Ops::prod(M::v_of(r[g + u]), xv[u]);
        acc = Ops::add(acc, (mask & (1u << (g + u))) ? p : Acc(0));
      }
    }
  }
}

// Drain one tile's segment pool on one warp, software-pipelined across segment boundaries: the
// next batch -- of the current segment, or batch 0 of the next segment -- is in flight while the
// current batch is consumed; the next segment's descriptor is claimed one segment ahead.
// CARRY = false: the plan has no split rows (every segment is a whole row), so the carry code
// and its registers are compiled out.  PEEK: load the next segment's carried partials when it
// is grabbed (2 more registers per lane; only where the register budget allows it -- spills in
// this loop cost more than the load latency they hide).
template <int U, int P, bool CARRY, bool PEEK, class M, typename Acc, class GrabFn>
__device__ __forceinline__ void run_segments(const M& mat, const XWindow<Acc>& xw,
                                             const XGlobal<Acc>& xg, GrabFn&& grab,
                                             const Carry<Acc>& carry, double* __restrict__ y,
                                             const GatherTargets& gt, uint32_t lane) {
  using Ops = AccOps<Acc>;
  using Raw = typename M::Raw;
  Segment sd;
  if (!grab(sd)) return;
  SegRun cur = seg_run<U, kRotate>(sd);
  Segment sn;
  bool have_next = grab(sn);
  Acc carried_next = PEEK && have_next ? carry.peek(sn.slot, sn.flags, lane) : Acc(0);
  Raw ra[U], rb[U];
  const uint32_t safe = xw.safe;
  uint32_t ma = load_batch<U>(mat, ra, cur, 0, lane, safe), mb = 0;
  prefetch_batches<U, P>(mat, cur, 1, lane);
  bool sn_pf = false;  // the next segment's head (P + 1 batches) has been prefetched
  Acc acc = CARRY ? carry.in(cur.slot, cur.flags, lane) : Acc(0);
  uint32_t bi = 0;
  // one pipeline step: consume (rc, mc), prefetch into (rn, mn); false when the pool is drained
  auto step = [&](const Raw* rc, uint32_t mc, Raw* rn, uint32_t& mn) -> bool {
    const bool more = bi + 1 < cur.nbatch;
    if (more) mn = load_batch<U>(mat, rn, cur, bi + 1, lane, safe);
    else if (have_next) mn = load_batch<U>(mat, rn, seg_run<U, kRotate>(sn), 0, lane, safe);
    if constexpr (P > 0) {  // the L2 prefetch stream runs P batches ahead of the loads; once
      // it passes the end of this segment, the next segment's first P + 1 batches go at once
      const uint32_t pf = bi + 1 + P;
      if (pf < cur.nbatch) {
        prefetch_batches<U, 1>(mat, cur, pf, lane);
      } else if (have_next && !sn_pf) {
        sn_pf = true;
        prefetch_batches<U, P + 1>(mat, seg_run<U, kRotate>(sn), 0, lane);
      }
    }
    if (cur.flags & kSegGlobalX) consume_batch<U, M>(rc, mc, xg, acc);
    else consume_batch<U, M>(rc, mc, xw, acc);
    if (more) {
      ++bi;
      return true;
    }
    if (!CARRY || (cur.flags & kSegLast)) {
      if (row_tree<kRotate>(acc, lane, cur.rot)) {
        y[cur.row] = static_cast<double>(acc);
        gt.store(cur.row, static_cast<double>(acc));
      }
    } else {
      if constexpr (CARRY) carry.out(cur.slot, cur.flags, lane, acc);
    }
    if (!have_next) return false;
    cur = seg_run<U, kRotate>(sn);
    bi = 0;
    if constexpr (PEEK) acc = carry.take(cur.slot, cur.flags, lane, carried_next);
    else acc = CARRY ? carry.in(cur.slot, cur.flags, lane) : Acc(0);
    have_next = grab(sn);
    sn_pf = false;
    if (PEEK && have_next) carried_next = carry.peek(sn.slot, sn.flags, lane);
    return true;
  };
  for (;;) {
    if (!step(ra, ma, rb, mb)) break;
    if (!step(rb, mb, ra, ma)) break;
  }
}

// ---- dense rows ------------------------------------------------------------------------------
// Rows at least 3/4 dense (columns nearly consecutive) need no shared-memory window: their 32
// lanes read 32 (nearly) consecutive x entries, which stay in L1 (this kernel uses no shared
// memory, so L1 holds most of x).  They are the longest rows (C2: every row longer than the
// 4,096-column locality window is fully dense -- 42% of the nonzeros), so inside the tile kernel
// they set both the per-tile imbalance and the kernel tail (one warp streams a 40,000-nonzero
// row at the speed of its own pipeline).  Here each warp pulls whole rows, longest first, with a
// wider batch (U chunks in flight in registers) and a deeper L2 prefetch stream (P batches
// ahead), so one row streams several times faster and the pool ends with the shortest rows.
// Semantics are the tile kernel's: lane l accumulates positions l, l + 32, ... from +0.0, then
// the stride-halving tree -- ddm::rowchunk_rows with lane_width 32 (src/spmv.cpp:48-68).
template <class M, typename Acc, int U, int P>
__global__ void __launch_bounds__(256)
    k_dense(M mat, const uint64_t* __restrict__ rp, const Acc* __restrict__ x,
            const uint32_t* __restrict__ rows, uint32_t n_rows, uint32_t* __restrict__ counter,
            double* __restrict__ y, const __grid_constant__ GatherTargets gt) {
  using Ops = AccOps<Acc>;
  using Raw = typename M::Raw;
  // programmatic dependent launch: the tile kernel that follows may take each SM as soon as
  // this grid's CTAs there have exited (it touches other rows; it waits for this grid only
  // before it completes)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t lane = threadIdx.x & 31;
  const XGlobal<Acc> xg{x};
  auto grab = [&](SegRun& r) -> bool {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(counter, 1u);
    k = __shfl_sync(kFull, k, 0);
    if (k >= n_rows) return false;
    const uint32_t row = rows[k];
    const uint64_t s = rp[row], e = rp[row + 1];
    r = seg_run_at<U, kRotate>(s, 0u, static_cast<uint32_t>(e - s));
    r.row = row;
    r.slot = 0;
    r.flags = kSegFirst | kSegLast;
    return true;
  };
  SegRun cur, nxt;
  if (!grab(cur)) return;
  bool have_next = grab(nxt);
  Raw ra[U], rb[U];
  uint32_t ma = load_batch<U>(mat, ra, cur, 0, lane, 0u), mb = 0;
  prefetch_batches<U, P>(mat, cur, 1, lane);
  bool nx_pf = false;
  Acc acc = Acc(0);
  uint32_t bi = 0;
  auto step = [&](const Raw* rc, uint32_t mc, Raw* rn, uint32_t& mn) -> bool {
    const bool more = bi + 1 < cur.nbatch;
    if (more) mn = load_batch<U>(mat, rn, cur, bi + 1, lane, 0u);
    else if (have_next) mn = load_batch<U>(mat, rn, nxt, 0, lane, 0u);
    const uint32_t pf = bi + 1 + P;
    if (pf < cur.nbatch) {
      prefetch_batches<U, 1>(mat, cur, pf, lane);
    } else if (have_next && !nx_pf) {
      nx_pf = true;
      prefetch_batches<U, P + 1>(mat, nxt, 0, lane);
    }
    consume_batch<U, M>(rc, mc, xg, acc);
    if (more) {
      ++bi;
      return true;
    }
    if (row_tree<kRotate>(acc, lane, cur.rot)) {
      y[cur.row] = static_cast<double>(acc);
      gt.store(cur.row, static_cast<double>(acc));
    }
    if (!have_next) return false;
    cur = nxt;
    bi = 0;
    acc = Acc(0);
    have_next = grab(nxt);
    nx_pf = false;
    return true;
  };
  for (;;) {
    if (!step(ra, ma, rb, mb)) break;
    if (!step(rb, mb, ra, ma)) break;
  }
}

// Persistent: one CTA per SM; dynamic smem = NB * wcap * sizeof(Acc) (the x-window buffers).
#ifndef DG_PREFETCH_SEGS
#define DG_PREFETCH_SEGS 1
#endif
constexpr bool kPrefetchSegs = DG_PREFETCH_SEGS;

// x as the tile kernel reads it: `x` (16-byte aligned, readable 16 elements before x[0] and past
// x[cols - 1]) and `x1`, the same values one element further on (x1 + i holds x[i] at an address
// 8 bytes off x's 16-byte phase), so a replica with an odd bank shift is still one 16-byte-aligned
// bulk copy.  `rep_stride`: elements between the replica regions of a window buffer.
template <typename Acc>
struct XSource {
  const Acc* x;
  const Acc* x1;
  uint32_t rep_stride;
};

template <class M, typename Acc, int WARPS, int U, int P = 0, int NB = 2, bool CARRY = true>
__global__ void __launch_bounds__(WARPS * 32, 1)
    k_tiles(M mat, XSource<Acc> xsrc, const Tile* __restrict__ tiles, uint32_t n_tiles,
            const Segment* __restrict__ segs, Carry<Acc> carry, double* __restrict__ y,
            uint32_t* __restrict__ counter, uint32_t wcap, BlockSignal sig, const __grid_constant__ GatherTargets gt,
            TileTrace tr) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // full[b]: the window of buffer b has landed (TMA complete_tx); empty[b]: every warp has left
  // buffer b (WARPS arrivals) -- the refill of b waits on it, so the window's readers are ordered
  // before its next TMA overwrite by barrier operations (visible to compute-sanitizer racecheck)
  __shared__ __align__(8) uint64_t full[NB], empty[NB];
  __shared__ uint32_t tile_of[NB], seg_next[NB], done[NB];
  Acc* const xbuf0 = reinterpret_cast<Acc*>(smem_raw);
  const uint32_t lane = threadIdx.x & 31;
  const Acc* __restrict__ x = xsrc.x;

  // claim the next tile for buffer b and start its window transfer (one thread)
  auto refill = [&](int b) {
    const uint32_t t = atomicAdd(counter, 1u);
    tile_of[b] = t;
    seg_next[b] = 0;
    done[b] = 0;
    if (t < n_tiles) {
      const Tile T = tiles[t];
      if (tr.cta) {  // {claim ns, -, CTA | n_segments << 16 | global-x << 62}
        tr.tile[3ull * t] = gtimer_ns();
        tr.tile[3ull * t + 2] = blockIdx.x | (static_cast<unsigned long long>(T.seg1 - T.seg0) << 16) |
                                (static_cast<unsigned long long>(T.xlen == 0) << 62);
      }
      // order earlier generic-proxy reads of this buffer before the async-proxy overwrite
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      char* const dst0 = reinterpret_cast<char*>(xbuf0 + b * wcap);
      if (T.nrep <= 1) {
        const uint32_t bytes = T.xlen * static_cast<uint32_t>(sizeof(Acc));  // 0: global-x tile
        mbar_arrive_expect_tx(&full[b], bytes);
        const char* src = reinterpret_cast<const char*>(x + T.xlo);
        for (uint32_t off = 0; off < bytes; off += 32768u)
          tma_load_1d(dst0 + off, src + off, min(32768u, bytes - off), &full[b]);
      } else {
        // replica r: elements [xlo - shift_r, xlo - shift_r + len_r) at dst + r * stride, so
        // column c sits at slot r * stride + (c - xlo) + shift_r (slot_of)
        constexpr uint32_t kAl = 16 / sizeof(Acc);
        uint32_t total = 0;
#pragma unroll
        for (uint32_t r = 0; r < kReplicas; ++r)
          total += (T.xlen + rep_shift(r) + kAl - 1) / kAl * kAl * static_cast<uint32_t>(sizeof(Acc));
        mbar_arrive_expect_tx(&full[b], total);
#pragma unroll
        for (uint32_t r = 0; r < kReplicas; ++r) {
          const uint32_t sh = rep_shift(r);
          const uint32_t bytes = (T.xlen + sh + kAl - 1) / kAl * kAl * static_cast<uint32_t>(sizeof(Acc));
          const Acc* base = (sh & 1u) ? xsrc.x1 : x;
          const char* src = reinterpret_cast<const char*>(base + T.xlo) - sh * sizeof(Acc);
          char* dst = dst0 + static_cast<size_t>(r) * xsrc.rep_stride * sizeof(Acc);
          for (uint32_t off = 0; off < bytes; off += 32768u)
            tma_load_1d(dst + off, src + off, min(32768u, bytes - off), &full[b]);
        }
      }
      // the tile's segment descriptors into L2 (one bulk prefetch): the warps' grabs then wait
      // on an L2 hit, not DRAM -- short segments need the next descriptor almost at once
      const uint64_t sb = reinterpret_cast<uint64_t>(segs + T.seg0) & ~15ull;
      const uint64_t se = (reinterpret_cast<uint64_t>(segs + T.seg1) + 15) & ~15ull;
      if (kPrefetchSegs && se > sb)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sb),
                     "r"(static_cast<uint32_t>(se - sb))
                     : "memory");
    } else {
      mbar_arrive(&full[b]);  // terminal: completes the phase with tile_of[b] >= n_tiles
    }
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], WARPS * 32);  // every thread arrives
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < NB; ++i) refill(i);
  __syncthreads();

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
    const Tile T = tiles[t];
    const bool slots = T.nrep > 1;
    const XWindow<Acc> xw{xbuf0 + b * wcap - (slots ? 0u : T.xlo), slots ? 0u : T.xlo};
    const XGlobal<Acc> xg{x};
    const uint32_t nseg = T.seg1 - T.seg0;
    auto grab = [&](Segment& s) -> bool {
      uint32_t k = 0;
      if (lane == 0) k = atomicAdd(&seg_next[b], 1u);
      k = __shfl_sync(kFull, k, 0);
      if (k >= nseg) return false;
      s = segs[T.seg0 + k];
      return true;
    };
    // peek only with >= 96 registers per thread
    constexpr bool kPeek = CARRY && WARPS * 32 * 96 <= 65536;
    run_segments<U, P, CARRY, kPeek>(mat, xw, xg, grab, carry, y, gt, lane);
    __syncwarp();
    if (lane == 0) {
      // this warp's reads of buffer b (and, when signalling, its d stores) happen before the count
      if (sig.left) __threadfence(); else __threadfence_block();
    }
    __syncwarp();
    mbar_arrive(&empty[b]);  // release: every lane's reads of buffer b are done (each arrives)
    if (lane == 0) {
      if (atomicAdd(&done[b], 1u) == WARPS - 1) {  // the tile is finished
        mbar_wait(&empty[b], ((phases >> b) & 1u) ^ 1u);  // acquire every warp's release
        if (tr.cta) tr.tile[3ull * t + 1] = gtimer_ns();
        if (sig.left && T.blk != kNoBlock) {
          __threadfence();
          if (atomicSub(&sig.left[T.blk], 1u) == 1u) {
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(sig.flag + T.blk),
                         "r"(sig.epoch)
                         : "memory");
          }
        }
        refill(b);
      }
    }
    __syncwarp();
    b = b + 1 == NB ? 0 : b + 1;
  }
  // launched programmatically after k_dense: complete only after it (and its d rows)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (tr.cta && lane == 0) {
    atomicAdd(&tr.cta[4ull * blockIdx.x + 2], static_cast<unsigned long long>(wait_cyc));
    atomicAdd(&tr.cta[4ull * blockIdx.x + 3], static_cast<unsigned long long>(clock64() - clk0));
    atomicMax(&tr.cta[4ull * blockIdx.x + 1], gtimer_ns());
  }
}

}  // namespace dg
