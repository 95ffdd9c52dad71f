// plan.cu -- the row plan: length bins for short rows, column-windowed tiles for the rest.
//
// Replaces the reference's scheduling (parallel_blocks: equal row-count blocks per std::thread,
// src/spmv.cpp:17-32) with a device-oriented plan built once at dg_create:
//   * rows with 1 <= len <= 32  -> bins by next_pow2(len), G lanes per row (k_group_*)
//   * rows with len > 32        -> segments: a sparse row spanning <= W/3 columns, or a dense
//                                  row spanning <= one shared-memory window (W columns), is one
//                                  segment; a dense row wider than a window reads x from global
//                                  memory; a wider sparse row is cut greedily into position ranges
//                                  spanning <= W/3 columns (wave k = k-th segment of a row)
//   * per wave, narrow segments binned into a fixed grid of windows, wide ones packed greedily
//     by first column; tiles of <= W columns and ~tile_nnz nonzeros (guided: smaller at the
//     end); inside a tile, longest segment first.  Waves run in one launch (fused) by default.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "handle.cuh"
#include "spmv_kernels.cuh"
#include "spmv_tiles.cuh"

namespace dg {

// first / last column of every row (0, 0 for empty rows)
template <class M>
__global__ void k_row_extents(M mat, const uint64_t* __restrict__ rp, uint64_t rows,
                              uint2* __restrict__ ext) {
  for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t s = rp[r], e = rp[r + 1];
    ext[r] = s == e ? make_uint2(0, 0) : make_uint2(mat.col_at(s), mat.col_at(e - 1));
  }
}

// Greedy cut of wide sparse rows: a segment starting at column c ends before the first column
// >= c + ws (ws = the narrow bound A of plan_tiles_typed).
template <class M>
__global__ void k_split_rows(M mat, const uint64_t* __restrict__ rp,
                             const uint32_t* __restrict__ rows, uint32_t n_rows,
                             const uint64_t* __restrict__ out_off, uint32_t ws,
                             uint64_t* __restrict__ pos, uint2* __restrict__ cext,
                             uint32_t* __restrict__ count) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += gridDim.x * blockDim.x) {
    const uint32_t r = rows[i];
    uint64_t p = rp[r];
    const uint64_t e = rp[r + 1];
    uint64_t o = out_off[i];
    uint32_t k = 0;
    while (p < e) {
      const uint64_t c = mat.col_at(p), lim = c + ws;
      uint64_t lo = p + 1, hi = e;  // first q in (p, e] with col[q] >= lim (or e)
      while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (static_cast<uint64_t>(mat.col_at(mid)) >= lim) hi = mid; else lo = mid + 1;
      }
      pos[o + k] = p;
      cext[o + k] = make_uint2(static_cast<uint32_t>(c), static_cast<uint32_t>(mat.col_at(lo - 1)));
      ++k;
      p = lo;
    }
    count[i] = k;
  }
}

// decode == 0: rewrite the column field of every position of every slot-mode tile (nrep > 1)
// into its slot; decode == 1: back to columns (dg_copy_rows, the scatter comparator).
// One warp per tile, half-chunks strided over its lanes.
__global__ void k_assign_slots(uint32_t* __restrict__ w, const Tile* __restrict__ tiles,
                               uint32_t n_tiles, const Segment* __restrict__ segs,
                               uint32_t stride, int decode) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = warp; t < n_tiles; t += n_warps) {
    const Tile T = tiles[t];
    if (T.nrep <= 1) continue;
    for (uint32_t k = T.seg0; k < T.seg1; ++k) {
      const Segment S = segs[k];
      const uint64_t base0 = S.p0 - S.lane0;
      const uint32_t lo = S.lane0, hi = S.lane0 + S.n;
      const uint32_t halves = (hi + 15) / 16;
      for (uint32_t u = lo / 16 + lane; u < halves; u += 32) {
        const uint32_t r0 = u * 16, a = max(r0, lo), e = min(r0 + 16, hi);
        if (decode) {
          for (uint32_t rel = a; rel < e; ++rel) {
            const uint32_t v = w[base0 + rel];
            w[base0 + rel] = (col_of_slot(v >> 16, T.xlo, stride) << 16) | (v & 0xFFFFu);
          }
          continue;
        }
        HalfMatch m;
        m.n = static_cast<int>(e - a);
        uint32_t col[16];
        for (int i = 0; i < m.n; ++i) {
          col[i] = w[base0 + a + i] >> 16;
          for (uint32_t r = 0; r < kReplicas; ++r)
            m.opt[i][r] = static_cast<uint8_t>((col[i] - T.xlo + rep_shift(r)) & 15u);
        }
        m.solve(e - a < 16, 0);
        for (int i = 0; i < m.n; ++i) {
          const uint32_t v = w[base0 + a + i];
          w[base0 + a + i] = (slot_of(col[i], T.xlo, m.asg[i], stride) << 16) | (v & 0xFFFFu);
        }
      }
    }
  }
}

namespace {

struct HostSeg {
  uint64_t p0;
  uint32_t n, row, slot, clo, chi;
  uint16_t lane0, flags;
};

template <class M>
int plan_tiles_typed(Handle* h, const M& mat, const std::vector<uint64_t>& lens) {
  const uint64_t rows = h->rows;
  const uint32_t align = 16u / h->acc_bytes;                  // elements per 16 B (TMA alignment)
  // slice stream (spmv_slices.cuh): the last element of every window buffer is the zero slot
  bool slices = h->slices_wanted;
  const uint32_t W = h->window_cols - (slices ? 16u : 0u);    // window capacity (columns)
  const uint32_t ws = W - align;                              // max segment span
  // narrow bound: sparse segments are kept within A columns so they pack into the fixed grid of
  // windows below (stride W - A); dense rows may span a whole window (their lanes read
  // consecutive x, so they share a window with few others anyway)
  const uint32_t A = (W / 3) / align * align;
  // slot mode (replicated windows, exact family on the Packed16 stream): kReplicas replica
  // regions of RS = W / kReplicas elements per buffer; a slot-mode window spans W3 columns (room
  // for the largest replica shift and 16-byte rounding) and takes the sparse segments spanning
  // <= A3 columns (C2: every sparse row, whose columns lie in a 4,096-column locality window),
  // binned on a grid of stride W3 - A3.
  const bool rep = h->slot_mode;
  // (RS a multiple of 16 elements: replica r's bank pairs are then (c - xlo + shift_r) mod 16, the
  //  model the slot assignment optimises -- with the slice stream's W = 13,808, W / 3 = 4,602 would
  //  offset replicas 1 and 2 by 10 and 4 bank pairs and the matching would optimise the wrong banks)
  const uint32_t RS = W / kReplicas / 16 * 16;
  const uint32_t W3 = (RS - 16) / 16 * 16;
  const uint32_t A3 = W3 >= 4096u + 256u ? 4096u : W3 * 2 / 3 / align * align;
  const uint32_t St3 = W3 - A3;
  h->rep_stride = RS;
  std::vector<uint64_t> rp(rows + 1, 0);
  for (uint64_t r = 0; r < rows; ++r) rp[r + 1] = rp[r] + lens[r];

  // 1. row extents on the device
  std::vector<uint2> ext(rows);
  if (rows) {
    uint2* d_ext = nullptr;
    DG_CUDA(cudaMalloc(&d_ext, rows * sizeof(uint2)));
    k_row_extents<M><<<grid_for(rows, 256), 256>>>(mat, h->d_row_ptr, rows, d_ext);
    cudaError_t e = cudaMemcpy(ext.data(), d_ext, rows * sizeof(uint2), cudaMemcpyDeviceToHost);
    cudaFree(d_ext);
    DG_CUDA(e);
  }

  // 2. segments: one per row that fits a window; a dense row wider than a window stays whole and
  //    reads x from global (its lanes read consecutive x: 2 sectors per 32 positions); a sparse
  //    wide row (e.g. a multi-beam row of C4) is cut greedily into windowed segments, one wave
  //    per segment, carrying its 32 lane partials between waves
  // k_dense for every dense row >= dense_min_len (DG_DENSE=0/1 forces off / on): when the longest
  // dense row is a sizeable share of one SM's work (nnz < 200 * SMs * longest) -- there a warp
  // streaming such a row inside the tile kernel sets the kernel tail (C2's 1/8 shard: 0.466 ->
  // 0.415 ms); on large matrices windowed dense rows stay in the tiles (C2: moving them is neutral
  // for the step and delays the overlapped d download).
  // It also needs the dense rows to be >= 5% of the nonzeros: a handful of long rows (C1 has one
  // or two) cost the tile kernel little and a separate launch more.
  // Auto: dense rows wider than a window go to k_dense when they hold >= 1% of the nonzeros
  // (inside the tile kernel they read x through L1 lines from L2: C2, 13% of the nonzeros,
  // 2.76 -> 2.62 ms, end to end 2.79 -> 2.66; C4's few such rows would only add a launch), and
  // every dense row >= dense_min_len does when the rule above holds (C3 shards).
  bool dense_all = h->dense_mode > 0;
  uint64_t wide_dense = 0;
  if (h->dense_mode < 0) {
    uint64_t longest = 0, dnnz = 0;
    for (uint64_t r = 0; r < rows; ++r) {
      if (lens[r] < h->dense_min_len || lens[r] <= h->short_max) continue;
      const uint64_t span = static_cast<uint64_t>(ext[r].y) - ext[r].x + 1;
      if (4 * lens[r] >= 3 * span) {
        longest = std::max<uint64_t>(longest, lens[r]);
        dnnz += lens[r];
        if (span > ws) wide_dense += lens[r];
      }
    }
    dense_all = longest && h->nnz < 200ull * h->sm_count * longest && 20 * dnnz >= h->nnz;
  }
  // (the slice stream has no global-x segments: every dense row wider than a window is k_dense's)
  h->dense_kernel = h->dense_mode != 0 && (dense_all || 100 * wide_dense >= h->nnz || (slices && wide_dense));
  // contiguous rows >= dense_min_len go to k_dense_values whenever the slice stream is planned
  // (binary16 values under lane width 32): their column words are implied, half the bytes
  auto contiguous_row = [&](uint64_t r) {
    return slices && h->dense_mode != 0 && lens[r] >= h->dense_min_len && lens[r] > h->short_max &&
           static_cast<uint64_t>(ext[r].y) - ext[r].x + 1 == lens[r];
  };
  // Auto: only when they are >= 0.5% of the nonzeros.  A handful of them (C1: 16 rows of 4,096,
  // 0.16%) leaves k_dense_values one latency-bound row per warp (~12 us for 4,096 positions) that
  // the tile kernel's CTAs wait behind; in the tiles they cost nothing (C1 0.118 -> 0.114 ms).
  // C2 / C3 / C5: 42%, C4: 1.0%.
  bool values_on = h->dense_mode > 0;
  if (h->dense_mode < 0 && slices) {
    uint64_t cnnz = 0;
    for (uint64_t r = 0; r < rows; ++r)
      if (contiguous_row(r)) cnnz += lens[r];
    values_on = 200 * cnnz >= h->nnz;
  }
  auto contiguous = [&](uint64_t r) { return values_on && contiguous_row(r); };
  if (!h->dense_kernel)
    for (uint64_t r = 0; r < rows && !h->dense_kernel; ++r) h->dense_kernel = contiguous(r);
  std::vector<std::vector<HostSeg>> waves(1);
  std::vector<HostSeg> global_x;
  std::vector<uint32_t> wide, dense_rows;
  for (uint64_t r = 0; r < rows; ++r) {
    if (lens[r] == 0 || lens[r] <= h->short_max) continue;
    const uint32_t c0 = ext[r].x, c1 = ext[r].y;
    const uint64_t span = static_cast<uint64_t>(c1) - c0 + 1;
    const uint16_t whole = static_cast<uint16_t>(kSegFirst | kSegLast);
    const bool dense = 4 * lens[r] >= 3 * span;
    if ((h->dense_kernel && dense && lens[r] >= h->dense_min_len && (dense_all || span > ws)) ||
        contiguous(r)) {  // k_dense / k_dense_values
      dense_rows.push_back(static_cast<uint32_t>(r));
      h->dense_nnz += lens[r];
      continue;
    }
    const bool dense_long = !slices && lens[r] >= h->global_min_len && dense;
    if ((span <= A || (dense && span <= ws)) && !dense_long) {
      waves[0].push_back({rp[r], static_cast<uint32_t>(lens[r]), static_cast<uint32_t>(r), 0, c0,
                          c1, 0, whole});
    } else if (dense) {
      global_x.push_back({rp[r], static_cast<uint32_t>(lens[r]), static_cast<uint32_t>(r), 0, c0,
                          c1, 0, static_cast<uint16_t>(whole | kSegGlobalX)});
    } else {
      wide.push_back(static_cast<uint32_t>(r));
    }
  }
  h->n_split_rows = wide.size();
  h->n_dense_rows = dense_rows.size();
  if (!dense_rows.empty()) {  // longest first: the pool ends with the shortest rows
    // Pull order: longest first by power-of-two length class (the kernel's tail is the last rows
    // pulled), by first column within a class -- rows running at the same time then overlap in
    // x, which the dense kernels read through L1 (an SM's L1 holds ~80% of C2's 320-KB x; rows
    // spread over all of x miss ~half the time, and a miss costs L1 data-pipe fills on top of the
    // hits -- the kernel's roof; C2 k_dense_values 0.525 -> 0.472 ms).  The fp32 family's x
    // (160 KB) fits L1 whole: strictly longest first there (the class order's longer tail cost
    // it ~2%).  DG_DENSE_ORDER=len / cls overrides.
    const char* dord = std::getenv("DG_DENSE_ORDER");
    const bool by_len = dord ? std::strcmp(dord, "len") == 0 : h->accumulation == DG_ACCUM_FP32;
    static const int cls_shift = [] { const char* c = std::getenv("DG_DENSE_CLASS"); return c ? std::atoi(c) : 0; }();
    auto cls = [&](uint32_t r) {  // length class: octave (DG_DENSE_CLASS=1: half octave, 2: two octaves)
      const int o = 63 - __builtin_clzll(lens[r] | 1);
      if (cls_shift == 1) return 2 * o + static_cast<int>((lens[r] >> (o - 1)) & 1);
      if (cls_shift == 2) return o / 2;
      return o;
    };
    std::stable_sort(dense_rows.begin(), dense_rows.end(), [&](uint32_t a, uint32_t b) {
      if (by_len) return lens[a] > lens[b];
      const int ca = cls(a), cb = cls(b);
      return ca != cb ? ca > cb : ext[a].x < ext[b].x;
    });
    h->dense_contig.resize(dense_rows.size());
    for (size_t i = 0; i < dense_rows.size(); ++i) h->dense_contig[i] = contiguous(dense_rows[i]);
    DG_CUDA(cudaMalloc(&h->d_dense_rows, dense_rows.size() * sizeof(uint32_t)));
    DG_CUDA(cudaMemcpy(h->d_dense_rows, dense_rows.data(), dense_rows.size() * sizeof(uint32_t),
                       cudaMemcpyHostToDevice));
    DG_CUDA(cudaMalloc(&h->d_dense_counter, sizeof(uint32_t)));
    h->plan_bytes += dense_rows.size() * sizeof(uint32_t);
  }
  if (!wide.empty()) {
    std::vector<uint64_t> off(wide.size() + 1, 0);
    for (size_t i = 0; i < wide.size(); ++i) {
      const uint64_t span = static_cast<uint64_t>(ext[wide[i]].y) - ext[wide[i]].x + 1;
      off[i + 1] = off[i] + span / A + 2;  // every segment but the last advances >= A columns
    }
    const uint64_t total = off.back();
    uint32_t *d_rows = nullptr, *d_cnt = nullptr;
    uint64_t *d_off = nullptr, *d_pos = nullptr;
    uint2* d_cext = nullptr;
    int st = DG_OK;
    auto cu = [&](cudaError_t e) { if (st == DG_OK && e != cudaSuccess) st = DG_ERR_CUDA_BASE + (int)e; };
    cu(cudaMalloc(&d_rows, wide.size() * 4));
    cu(cudaMalloc(&d_cnt, wide.size() * 4));
    cu(cudaMalloc(&d_off, (wide.size() + 1) * 8));
    cu(cudaMalloc(&d_pos, total * 8));
    cu(cudaMalloc(&d_cext, total * sizeof(uint2)));
    std::vector<uint64_t> pos(total);
    std::vector<uint2> cext(total);
    std::vector<uint32_t> cnt(wide.size());
    if (st == DG_OK) {
      cu(cudaMemcpy(d_rows, wide.data(), wide.size() * 4, cudaMemcpyHostToDevice));
      cu(cudaMemcpy(d_off, off.data(), (wide.size() + 1) * 8, cudaMemcpyHostToDevice));
      // (rows fill only their first count[i] slots; the rest is copied back unread -- zeroed so
      //  the copy reads initialised memory, compute-sanitizer initcheck)
      cu(cudaMemset(d_pos, 0, total * 8));
      cu(cudaMemset(d_cext, 0, total * sizeof(uint2)));
      k_split_rows<M><<<grid_for(wide.size(), 128), 128>>>(
          mat, h->d_row_ptr, d_rows, static_cast<uint32_t>(wide.size()),
          d_off, A, d_pos, d_cext, d_cnt);
      cu(cudaGetLastError());
      cu(cudaMemcpy(pos.data(), d_pos, total * 8, cudaMemcpyDeviceToHost));
      cu(cudaMemcpy(cext.data(), d_cext, total * sizeof(uint2), cudaMemcpyDeviceToHost));
      cu(cudaMemcpy(cnt.data(), d_cnt, wide.size() * 4, cudaMemcpyDeviceToHost));
    }
    cudaFree(d_rows); cudaFree(d_cnt); cudaFree(d_off); cudaFree(d_pos); cudaFree(d_cext);
    if (st) return st;
    // carry slots: segment k of a split row writes slot base + k, segment k + 1 reads it
    uint64_t base = 0;
    for (size_t i = 0; i < wide.size(); ++i) {
      const uint32_t r = wide[i];
      const uint64_t end = rp[r + 1];
      if (base + cnt[i] > 0xFFFFFFFFull) return DG_ERR_UNSUPPORTED_FEATURE;
      for (uint32_t k = 0; k < cnt[i]; ++k) {
        const uint64_t p = pos[off[i] + k];
        const uint64_t q = k + 1 < cnt[i] ? pos[off[i] + k + 1] : end;
        if (waves.size() <= k) waves.resize(k + 1);
        uint16_t flags = (k == 0 ? kSegFirst : 0) | (k + 1 == cnt[i] ? kSegLast : 0) |
                         static_cast<uint16_t>(std::min<uint32_t>(k, 255u) << kSegWaveShift);
        waves[k].push_back({p, static_cast<uint32_t>(q - p), r, static_cast<uint32_t>(base + k),
                            cext[off[i] + k].x, cext[off[i] + k].y,
                            static_cast<uint16_t>((p - rp[r]) & 31u), flags});
      }
      base += cnt[i] - 1;
    }
    h->n_carry_slots = base;
  }

  // 3. tiles
  const uint64_t xcap = (h->cols + align - 1) / align * align;  // padded x length on device
  h->n_waves = static_cast<uint32_t>(waves.size());
  h->n_global_rows = global_x.size();
  // Several waves: one launch for all of them by default (fused: segment k + 1 of a row waits for
  // segment k's carried partials, Carry in spmv_tiles.cuh) -- one kernel tail instead of one per
  // wave.  DG_FUSE_WAVES=0 keeps one launch per wave (A/B only, up to kMaxWaves waves: a row may
  // be cut into any number of segments -- a U32 row spanning a million columns is ~200 waves --
  // and the fused launch has no limit on it).
  h->fused_waves = h->n_waves > 1;
  if (const char* fw = std::getenv("DG_FUSE_WAVES"))
    h->fused_waves = h->fused_waves && (std::atoi(fw) || h->n_waves > Handle::kMaxWaves);
  if (h->n_waves > 1 && !h->fused_waves) slices = false;  // one launch list only
  if (!global_x.empty()) slices = false;  // (DG_DENSE=0: global-x tiles need true columns)
  // Output row blocks: contiguous, byte-balanced row ranges.  A block's d is complete (and can be
  // downloaded) once its tiles are done.  Fused waves list the (wave, block) groups diagonally --
  // wave w of block b right after wave w - 1 of block b + lag -- with lag = K - 1 (wave after
  // wave) by default.  Measured on C4: a short lag (64 blocks, lag 1 or 3, meant to read carried
  // partials back while still in L2) makes segments wait on tiles still in flight -- ~296 tiles
  // (2 per SM) of ~1M nonzeros are always in flight -- 7.95 / 6.83 ms vs 6.70 wave after wave.
  // (~2 MB of d per block: the last block's download after the kernel is short, and small
  // matrices do not pay 32 copies -- C1's end to end went 0.32 -> 0.51 ms at 32 blocks)
  uint32_t K = h->nnz >= (16ull << 20)
                   ? static_cast<uint32_t>(std::max<uint64_t>(
                         1, std::min<uint64_t>(Handle::kDefaultBlocks, rows * 8 / (2u << 20))))
                   : 1;
  if (const char* kb = std::getenv("DG_BLOCKS"))
    K = std::max<uint32_t>(1, std::min<uint32_t>(Handle::kMaxBlocks, std::atoi(kb)));
  uint32_t lag = K - 1;
  if (const char* lg = std::getenv("DG_WAVE_LAG")) lag = std::max(0, std::atoi(lg));
  {
    std::vector<uint64_t> b(K + 1);
    std::vector<uint32_t> l32(rows);
    for (uint64_t r = 0; r < rows; ++r) l32[r] = static_cast<uint32_t>(lens[r]);
    dg_partition_lengths(l32.data(), rows, h->value_bytes + h->index_bytes, K, b.data());
    h->n_blocks = K;
    for (uint32_t k = 0; k <= K; ++k) h->blk_row0[k] = b[k];
  }
  auto blk_of = [&](uint32_t row) {
    return static_cast<uint32_t>(std::upper_bound(h->blk_row0, h->blk_row0 + K + 1, row) -
                                 h->blk_row0) - 1;
  };
  const uint32_t NW = h->n_waves;
  std::vector<std::vector<std::vector<HostSeg>>> win(NW, std::vector<std::vector<HostSeg>>(K));
  std::vector<std::vector<HostSeg>> glob(K);
  for (uint32_t w = 0; w < NW; ++w)
    for (const HostSeg& q : waves[w]) win[w][blk_of(q.row)].push_back(q);
  for (const HostSeg& q : global_x) glob[blk_of(q.row)].push_back(q);
  // emission order of the (wave, block) groups
  std::vector<std::pair<uint32_t, uint32_t>> order;
  if (h->fused_waves) {
    for (uint32_t key = 0; key < K + (NW - 1) * (lag + 1); ++key)
      for (uint32_t w = 0; w < NW; ++w)
        if (key >= w * (lag + 1) && key - w * (lag + 1) < K) order.push_back({w, key - w * (lag + 1)});
  } else {
    for (uint32_t w = 0; w < NW; ++w)
      for (uint32_t k = 0; k < K; ++k) order.push_back({w, k});
  }
  // one tile list per launch (fused: one launch)
  const uint32_t NL = h->fused_waves ? 1 : NW;
  std::vector<std::vector<Tile>> ltiles(NL);
  std::vector<std::vector<Segment>> lsegs(NL);
  std::vector<uint64_t> lnnz(NL, 0), ldone(NL, 0), lrows(NL, 0);
  for (uint32_t w = 0; w < NW; ++w)
    for (const HostSeg& q : waves[w]) lnnz[h->fused_waves ? 0 : w] += q.n;
  for (const HostSeg& q : global_x) lnnz[0] += q.n;
  std::vector<uint64_t> wnnz(NW, 0), wrows(NW, 0);
  const uint32_t St = W - A;
  auto narrow = [&](const HostSeg& q) { return q.chi - q.clo + 1 <= A; };
  for (const auto& [w, k] : order) {
    const uint32_t lw = h->fused_waves ? 0 : w;
    std::vector<Tile>& tiles = ltiles[lw];
    std::vector<Segment>& segs = lsegs[lw];
    // ~8 tiles per SM at least in every launch (no single-tile tails), at most tile_nnz
    const uint64_t tile_nnz = std::max<uint64_t>(
        4096, std::min<uint64_t>(h->tile_nnz, lnnz[lw] / (h->min_tiles_per_sm * h->sm_count)));
    // guided sizing: tiles are claimed in list order, so the kernel's tail is the duration of the
    // last tiles claimed.  Once the work left in the launch drops below ~guide tiles per SM,
    // tiles shrink with it (remaining / (guide * SMs)), down to guide_min nonzeros.
    const uint64_t guide = h->tile_guide;
    const uint64_t guide_min = std::min<uint64_t>(tile_nnz, h->tile_guide_min);
    auto cap_nnz = [&]() -> uint64_t {
      if (!guide) return tile_nnz;
      const uint64_t rem = lnnz[lw] - ldone[lw];
      return std::max(guide_min, std::min(tile_nnz, rem / (guide * h->sm_count)));
    };
    // signalled when one launch finishes every row: a single wave, or fused waves (a block
    // completes with the last of its tiles in any wave)
    const uint8_t blk = NW == 1 || h->fused_waves ? static_cast<uint8_t>(k) : kNoBlock;
    const size_t tiles_before = tiles.size();
    auto take = [&](const HostSeg& q) {
      segs.push_back({q.p0, q.n, q.row, q.slot, q.lane0, q.flags});
      ldone[lw] += q.n;
      wnnz[w] += q.n;
      const bool last = (q.flags & kSegLast) != 0;
      wrows[w] += last;
      lrows[lw] += last;
    };
    if (w == 0) {  // global-x tiles first (no window), longest rows first
      auto& G = glob[k];
      std::stable_sort(G.begin(), G.end(), [](const HostSeg& a, const HostSeg& b) { return a.n > b.n; });
      size_t g = 0;
      while (g < G.size()) {
        uint64_t nnz = 0;
        const uint32_t s0 = static_cast<uint32_t>(segs.size());
        const uint64_t cap = cap_nnz();
        while (g < G.size() && (nnz == 0 || nnz + G[g].n <= cap)) {
          nnz += G[g].n;
          take(G[g++]);
        }
        tiles.push_back({0, 0, blk, 1, s0, static_cast<uint32_t>(segs.size())});
      }
    }
    // windowed tiles.  Narrow segments (span <= A = W/3) are binned into a fixed grid of windows
    // [g*St, g*St + W), stride St = W - A: a segment whose first column lies in [g*St, (g+1)*St)
    // fits window g, so the rare wide segments (e.g. a row's clusters in two adjacent beams,
    // merged into one segment) cannot cut the tiles of narrow ones short.  Wide segments are
    // packed greedily in first-column order.  Each bin: first-column order, cut at ~cap nonzeros.
    // windowed tiles, three classes: (0) slot-mode: sparse segments spanning <= A3 columns,
    // binned on the grid [g*St3, g*St3 + W3) of replicated windows; (1) narrow: segments spanning
    // <= A = W/3, binned into a fixed grid of windows [g*St, g*St + W), stride St = W - A -- a
    // segment whose first column lies in [g*St, (g+1)*St) fits window g, so the rare wide
    // segments (e.g. a row's clusters in two adjacent beams, merged into one segment) cannot cut
    // the tiles of narrow ones short; (2) wide: packed greedily in first-column order.  Each bin:
    // first-column order, cut at ~cap nonzeros.
    auto& S = win[w][k];
    auto cls = [&](const HostSeg& q) -> int {
      const uint32_t span = q.chi - q.clo + 1;
      // (slot mode on the row-ordered stream: Packed16 only -- k_assign_slots rewrites it)
      // (dense segments too: a row 75-99% dense spreads a half-warp's 16 lanes over ~16-21
      //  columns, so without replicas two of them often share a bank pair; fully dense rows
      //  gain nothing but lose nothing either)
      if (rep && (slices || h->packed) && span <= A3) return 0;
      return narrow(q) ? 1 : 2;
    };
    auto bin = [&](const HostSeg& q, int c) -> uint32_t {
      return c == 0 ? q.clo / St3 : c == 1 ? q.clo / St : 0;
    };
    std::stable_sort(S.begin(), S.end(), [&](const HostSeg& a, const HostSeg& b) {
      const int ca = cls(a), cb = cls(b);
      if (ca != cb) return ca < cb;
      const uint32_t ga = bin(a, ca), gb = bin(b, cb);
      if (ga != gb) return ga < gb;
      return a.clo != b.clo ? a.clo < b.clo : a.row < b.row;
    });
    auto emit = [&](size_t i, size_t j, uint8_t nrep) {
      uint32_t lo = S[i].clo, hi = S[i].chi;
      for (size_t q = i; q < j; ++q) {
        lo = std::min(lo, S[q].clo);
        hi = std::max(hi, S[q].chi);
      }
      const uint32_t xlo = lo / align * align;
      // longest segment first inside the tile (warps pull segments dynamically)
      std::stable_sort(S.begin() + i, S.begin() + j,
                       [](const HostSeg& a, const HostSeg& b) { return a.n > b.n; });
      uint32_t xlen = (hi - xlo + 1 + align - 1) / align * align;
      if (xlo + xlen > xcap) xlen = static_cast<uint32_t>(xcap - xlo);
      tiles.push_back({xlo, static_cast<uint16_t>(xlen), blk, nrep,
                       static_cast<uint32_t>(segs.size()),
                       static_cast<uint32_t>(segs.size() + (j - i))});
      for (size_t q = i; q < j; ++q) take(S[q]);
    };
    size_t i = 0;
    for (int c = 0; c < 2; ++c) {  // binned classes: per grid window, cut by nonzeros
      while (i < S.size() && cls(S[i]) == c) {
        const uint32_t g = bin(S[i], c);
        uint64_t nnz = 0;
        size_t j = i;
        const uint64_t cap = cap_nnz();
        while (j < S.size() && cls(S[j]) == c && bin(S[j], c) == g && (j == i || nnz + S[j].n <= cap))
          nnz += S[j++].n;
        emit(i, j, c == 0 ? static_cast<uint8_t>(kReplicas) : 1);
        i = j;
      }
    }
    while (i < S.size()) {  // wide: greedy, cut at the window width or ~cap nonzeros
      const uint32_t xlo = S[i].clo / align * align;
      uint32_t hi = S[i].chi;
      uint64_t nnz = 0;
      size_t j = i;
      const uint64_t cap = cap_nnz();
      while (j < S.size()) {
        const uint32_t nhi = std::max(hi, S[j].chi);
        if (j > i && (static_cast<uint64_t>(nhi) - xlo + 1 > W || nnz + S[j].n > cap)) break;
        hi = nhi;
        nnz += S[j].n;
        ++j;
      }
      emit(i, j, 1);
      i = j;
    }
    if (blk != kNoBlock) h->blk_tiles[k] += static_cast<uint32_t>(tiles.size() - tiles_before);
  }
  {
    uint64_t nseg = 0, snnz = 0;
    for (uint32_t lw = 0; lw < NL; ++lw) {
      nseg += lsegs[lw].size();
      snnz += ldone[lw];
    }
    h->short_segments = nseg && snnz < 256ull * nseg;
    if (const char* ss = std::getenv("DG_SHORT_SEGMENTS")) h->short_segments = std::atoi(ss) != 0;
  }
  for (uint32_t w = 0; w < Handle::kMaxWaves; ++w) h->wave_nnz[w] = h->wave_rows[w] = h->wave_tiles[w] = 0;
  for (uint32_t w = 0; w < NW; ++w) {  // (statistics; waves past the last slot are folded in it)
    h->wave_nnz[std::min(w, Handle::kMaxWaves - 1)] += wnnz[w];
    h->wave_rows[std::min(w, Handle::kMaxWaves - 1)] += wrows[w];
  }
  if (h->fused_waves) {
    h->fused_rows = lrows[0];
    h->fused_nnz = ldone[0];
  }
  if (slices) DG_TRY(plan_slices(h, ltiles[0], lsegs[0]));
  h->n_segments = lsegs[0].size();
  for (uint32_t lw = 0; lw < NL; ++lw) {  // the fused list is uploaded as launch 0
    const auto& tiles = ltiles[lw];
    const auto& segs = lsegs[lw];
    h->wave_tiles[lw] = static_cast<uint32_t>(tiles.size());
    if (tiles.empty()) continue;
    DG_CUDA(cudaMalloc(&h->d_tiles[lw], tiles.size() * sizeof(Tile)));
    DG_CUDA(cudaMemcpy(h->d_tiles[lw], tiles.data(), tiles.size() * sizeof(Tile),
                       cudaMemcpyHostToDevice));
    DG_CUDA(cudaMalloc(&h->d_segs[lw], segs.size() * sizeof(Segment)));
    DG_CUDA(cudaMemcpy(h->d_segs[lw], segs.data(), segs.size() * sizeof(Segment),
                       cudaMemcpyHostToDevice));
    h->plan_bytes += tiles.size() * sizeof(Tile) + segs.size() * sizeof(Segment);
    for (const Tile& t : tiles) h->slot_tiles += t.nrep > 1;
  }
  if (h->slot_tiles && !h->slices) DG_TRY(recode_slots(h, false));
  if (h->n_carry_slots) {
    const uint64_t n = h->n_carry_slots * 32;
    DG_CUDA(cudaMalloc(&h->d_state, n * h->acc_bytes));
    h->plan_bytes += n * h->acc_bytes;
    if (h->acc_bytes == 8)
      k_carry_init<double><<<grid_for(n, 256), 256>>>(static_cast<double*>(h->d_state), n);
    else
      k_carry_init<float><<<grid_for(n, 256), 256>>>(static_cast<float*>(h->d_state), n);
    DG_CUDA(cudaGetLastError());
  }
  DG_CUDA(cudaMalloc(&h->d_counters, Handle::kMaxWaves * sizeof(uint32_t)));
  DG_CUDA(cudaMalloc(&h->d_blk_left, Handle::kMaxBlocks * sizeof(uint32_t)));
  DG_CUDA(cudaMalloc(&h->d_blk_left_init, Handle::kMaxBlocks * sizeof(uint32_t)));
  DG_CUDA(cudaMalloc(&h->d_blk_flag, Handle::kMaxBlocks * sizeof(uint32_t)));
  DG_CUDA(cudaMemcpy(h->d_blk_left_init, h->blk_tiles, Handle::kMaxBlocks * sizeof(uint32_t),
                     cudaMemcpyHostToDevice));
  DG_CUDA(cudaMemset(h->d_blk_flag, 0, Handle::kMaxBlocks * sizeof(uint32_t)));
  return DG_OK;
}

}  // namespace

// Rewrite the slot-mode tiles' positions of the Packed16 stream between columns (decode) and
// slots (encode); the handle remembers which form the stream is in.
int recode_slots(Handle* h, bool decode) {
  if (h->slices || !h->slot_tiles || h->slots_encoded == !decode) return DG_OK;
  const uint32_t NL = h->fused_waves ? 1 : h->n_waves;
  for (uint32_t lw = 0; lw < NL; ++lw) {
    if (!h->wave_tiles[lw]) continue;
    k_assign_slots<<<grid_for(32ull * h->wave_tiles[lw], 128, 16), 128>>>(
        h->d_packed, static_cast<const Tile*>(h->d_tiles[lw]), h->wave_tiles[lw],
        static_cast<const Segment*>(h->d_segs[lw]), h->rep_stride, decode ? 1 : 0);
    DG_CUDA(cudaGetLastError());
  }
  DG_CUDA(cudaDeviceSynchronize());
  h->slots_encoded = !decode;
  return DG_OK;
}

int plan_tiles(Handle* h, const std::vector<uint64_t>& lens) {
  return dispatch_mat(h, [&](const auto& mat) { return plan_tiles_typed(h, mat, lens); });
}

}  // namespace dg
