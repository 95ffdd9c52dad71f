// slices.cu -- building the slice stream (spmv_slices.cuh) from the row-ordered upload, the
// rest stream of the rows the tile kernel does not own, and decoding both back to the
// reference's row-ordered encoding (dg_copy_rows, the scatter comparator).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "handle.cuh"
#include "spmv_slices.cuh"

namespace dg {

// ---- plan: segments of every tile grouped into runs ------------------------------------------
// A tile's segments are grouped into R = kRunsPerWarp x WARPS runs by LPT on chunks (longest
// segment to the least-loaded run), the runs listed longest first; the CTA's warps pull runs
// dynamically, so the runs still left when a warp frees up are the shortest (online LPT): the
// tile's window is released when the slowest warp is done, and a static run per warp left ~25% of
// warp time waiting on a window on C2's 1/8 shard (DG_TRACE).  Each run is padded to whole
// 8-chunk batches (two 512-byte blocks), so the kernel's loads need no guards.
int plan_slices(Handle* h, const std::vector<Tile>& tiles, std::vector<Segment>& segs) {
  const int WARPS = h->n_carry_slots ? Handle::kSliceWarpsCarry
                    : h->short_segments ? Handle::kSliceWarpsShort : Handle::kSliceWarps;
  int RUNS = WARPS * Handle::kRunsPerWarp;
  if (const char* rw = std::getenv("DG_RUNS_PER_WARP")) RUNS = WARPS * std::max(1, std::atoi(rw));
  std::vector<WarpRange> R;
  R.reserve(tiles.size() * RUNS + 1);
  std::vector<SliceSeg> ss(segs.size());
  std::vector<Segment> out(segs.size());
  uint64_t chunk = 0;
  std::vector<uint32_t> idx, order(RUNS);
  std::vector<std::vector<uint32_t>> lists(RUNS);
  std::vector<uint64_t> load(RUNS);
  auto nch = [](const Segment& s) { return (static_cast<uint32_t>(s.lane0) + s.n + 31) / 32; };
  for (const Tile& T : tiles) {
    idx.resize(T.seg1 - T.seg0);
    std::iota(idx.begin(), idx.end(), T.seg0);
    std::stable_sort(idx.begin(), idx.end(),
                     [&](uint32_t a, uint32_t b) { return nch(segs[a]) > nch(segs[b]); });
    for (auto& l : lists) l.clear();
    std::fill(load.begin(), load.end(), 0);
    for (uint32_t i : idx) {
      const int w = static_cast<int>(std::min_element(load.begin(), load.end()) - load.begin());
      lists[w].push_back(i);
      load[w] += nch(segs[i]);
    }
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return load[a] > load[b]; });
    uint32_t k = T.seg0;
    for (int q = 0; q < RUNS; ++q) {
      const uint32_t w = order[q];
      R.push_back({static_cast<uint32_t>(chunk), k});
      for (uint32_t i : lists[w]) {
        const Segment& S = segs[i];
        out[k] = S;
        ss[k] = {S.row, S.slot, nch(S), S.flags};
        ++k;
      }
      chunk += (load[w] + kSlicePad - 1) / kSlicePad * kSlicePad;
      if (chunk > 0xFFFFFFFFull) return DG_ERR_UNSUPPORTED_FEATURE;
    }
  }
  R.push_back({static_cast<uint32_t>(chunk), static_cast<uint32_t>(segs.size())});
  segs.swap(out);
  h->slice_warps = WARPS;
  h->slice_runs = RUNS;
  h->slice_chunks = chunk;
  DG_CUDA(cudaMalloc(&h->d_ranges, R.size() * sizeof(WarpRange)));
  DG_CUDA(cudaMemcpy(h->d_ranges, R.data(), R.size() * sizeof(WarpRange), cudaMemcpyHostToDevice));
  DG_CUDA(cudaMalloc(&h->d_sseg, std::max<size_t>(1, ss.size()) * sizeof(SliceSeg)));
  DG_CUDA(cudaMemcpy(h->d_sseg, ss.data(), ss.size() * sizeof(SliceSeg), cudaMemcpyHostToDevice));
  h->plan_bytes += R.size() * sizeof(WarpRange) + ss.size() * sizeof(SliceSeg);
  h->slices = true;
  return DG_OK;
}

namespace {

// One warp per (tile, run) run: the run's chunks in the lane-major block layout.  Slot-mode
// tiles (nrep > 1) choose every position's replica with the per-half-warp b-matching
// (HalfMatch), solved by the half's first lane.
template <class M>
__global__ void k_build_slices(M mat, const Tile* __restrict__ tiles, const Segment* __restrict__ segs,
                               const WarpRange* __restrict__ ranges, uint32_t n_runs, uint32_t warps,
                               uint32_t* __restrict__ out, uint32_t rep_stride, uint32_t zero_slot) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t n_gw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t neutral = zero_slot << 16;
  for (uint32_t i = gw; i < n_runs; i += n_gw) {
    const Tile T = tiles[i / warps];
    const WarpRange r0 = ranges[i], r1 = ranges[i + 1];
    uint64_t c = r0.chunk;
    for (uint32_t s = r0.seg; s < r1.seg; ++s) {
      const Segment S = segs[s];
      const uint64_t base0 = S.p0 - S.lane0;
      const uint32_t nch = (static_cast<uint32_t>(S.lane0) + S.n + 31) / 32;
      for (uint32_t j = 0; j < nch; ++j, ++c) {
        const uint32_t rel = 32 * j + lane;
        const bool valid = rel >= S.lane0 && rel < S.lane0 + S.n;
        uint32_t col = 0, val = 0;
        if (valid) {
          const auto e = mat.load(base0 + rel);
          col = static_cast<uint32_t>(M::c_of(e));
          val = static_cast<uint16_t>(M::v_of(e));
        }
        uint32_t slot = zero_slot;
        if (T.nrep <= 1) {
          if (valid) slot = col - T.xlo;
        } else {
          // the half's first lane solves its half-warp; choices come back 2 bits per lane
          const uint32_t half = lane & 16u;
          HalfMatch m;
          m.n = 0;
          int8_t pos_of[16];
          bool any_invalid = false;
          for (uint32_t q = 0; q < 16; ++q) {
            const uint32_t cq = __shfl_sync(kFull, col, half + q);
            const bool vq = __shfl_sync(kFull, valid, half + q);
            if ((lane & 15u) == 0) {
              pos_of[q] = -1;
              if (vq) {
                pos_of[q] = static_cast<int8_t>(m.n);
                for (uint32_t r = 0; r < kReplicas; ++r)
                  m.opt[m.n][r] = static_cast<uint8_t>((cq - T.xlo + rep_shift(r)) & 15u);
                ++m.n;
              } else {
                any_invalid = true;
              }
            }
          }
          uint32_t packed = 0;
          if ((lane & 15u) == 0 && m.n) {
            m.solve(any_invalid, static_cast<int>(zero_slot & 15u));
            for (uint32_t q = 0; q < 16; ++q)
              if (pos_of[q] >= 0) packed |= static_cast<uint32_t>(m.asg[pos_of[q]]) << (2 * q);
          }
          packed = __shfl_sync(kFull, packed, half);
          if (valid) slot = slot_of(col, T.xlo, (packed >> (2 * (lane & 15u))) & 3u, rep_stride);
        }
        out[slice_word(c, lane)] = (slot << 16) | val;
      }
    }
    for (; c < r1.chunk; ++c) out[slice_word(c, lane)] = neutral;
  }
}

// Dense rows (k_dense_slices): one warp per row, the row's chunks in lane-major blocks from its
// run's first chunk; positions past the row end are neutral words (column `cols`, value +0).
__global__ void k_build_dense(Packed16 mat, const uint64_t* __restrict__ rp,
                              const SliceSeg* __restrict__ sseg, const WarpRange* __restrict__ ranges,
                              uint32_t n_rows, uint32_t* __restrict__ out, uint32_t neutral) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_gw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t k = gw; k < n_rows; k += n_gw) {
    const uint32_t row = sseg[k].row;
    const uint64_t s = rp[row], n = rp[row + 1] - s;
    const uint64_t c0 = ranges[k].chunk, c1 = ranges[k + 1].chunk;
    for (uint64_t c = c0; c < c1; ++c) {
      const uint64_t rel = 32 * (c - c0) + lane;
      out[slice_word(c, lane)] = rel < n ? mat.load(s + rel) : neutral;
    }
  }
}

__global__ void k_decode_dense(const uint32_t* __restrict__ w, const SliceSeg* __restrict__ sseg,
                               const WarpRange* __restrict__ ranges, uint32_t n_rows,
                               const uint64_t* __restrict__ rp, uint64_t r0, uint64_t r1, uint64_t b,
                               uint32_t* __restrict__ col, uint16_t* __restrict__ val) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_gw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t k = gw; k < n_rows; k += n_gw) {
    const uint32_t row = sseg[k].row;
    if (row < r0 || row >= r1) continue;
    const uint64_t s = rp[row], n = rp[row + 1] - s, c0 = ranges[k].chunk;
    for (uint64_t rel = lane; rel < n; rel += 32) {
      const uint32_t v = w[slice_word(c0 + rel / 32, lane)];
      col[s + rel - b] = v >> 16;
      val[s + rel - b] = static_cast<uint16_t>(v & 0xFFFFu);
    }
  }
}

// Contiguous rows as values only (k_dense_values): one warp per row, which also records the row's
// first column in its descriptor.
template <class M>
__global__ void k_build_values(M mat, const uint64_t* __restrict__ rp, DenseRow* __restrict__ rows,
                               uint32_t n_rows, uint16_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_gw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t k = gw; k < n_rows; k += n_gw) {
    const DenseRow R = rows[k];
    const uint64_t s = rp[R.row];
    if (lane == 0) rows[k].lo = static_cast<uint32_t>(mat.col_at(s));
    const uint32_t nblk = ((R.len + 31) / 32 + kValueChunks - 1) / kValueChunks;
    for (uint32_t b = 0; b < nblk; ++b)
      for (uint32_t i = 0; i < kValueChunks; ++i) {
        const uint32_t pos = 32 * (kValueChunks * b + i) + lane;
        out[(static_cast<uint64_t>(R.blk) + b) * (32 * kValueChunks) + kValueChunks * lane + i] =
            pos < R.len ? static_cast<uint16_t>(M::v_of(mat.load(s + pos))) : uint16_t(0);
      }
  }
}

__global__ void k_decode_values(const uint16_t* __restrict__ vs, const DenseRow* __restrict__ rows,
                                uint32_t n_rows, const uint64_t* __restrict__ rp, uint64_t r0,
                                uint64_t r1, uint64_t b, uint32_t* __restrict__ col,
                                uint16_t* __restrict__ val) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_gw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t k = gw; k < n_rows; k += n_gw) {
    const DenseRow R = rows[k];
    if (R.row < r0 || R.row >= r1) continue;
    const uint64_t s = rp[R.row];
    for (uint32_t rel = lane; rel < R.len; rel += 32) {
      const uint32_t c = rel / 32;
      col[s + rel - b] = R.lo + rel;
      val[s + rel - b] = vs[(static_cast<uint64_t>(R.blk) + c / kValueChunks) * (32 * kValueChunks) +
                            kValueChunks * lane + c % kValueChunks];
    }
  }
}

// rows not owned by tiles (k_dense, the short-row bins): copied into a compacted stream of the
// upload's format; rest_rp is a row pointer over it (tile rows have length 0)
template <class M>
__global__ void k_copy_rest(M src, const uint64_t* __restrict__ rp, const uint64_t* __restrict__ rest_rp,
                            uint64_t rows, uint32_t* __restrict__ out_w, void* __restrict__ out_col,
                            uint16_t* __restrict__ out_val) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = warp; r < rows; r += n_warps) {
    const uint64_t d = rest_rp[r], n = rest_rp[r + 1] - d;
    if (!n) continue;
    const uint64_t s = rp[r];
    for (uint64_t j = lane; j < n; j += 32) {
      const auto e = src.load(s + j);
      if constexpr (std::is_same_v<M, Packed16>) {
        out_w[d + j] = e;
      } else {
        static_cast<typename M::Idx*>(out_col)[d + j] = M::c_of(e);
        out_val[d + j] = M::v_of(e);
      }
    }
  }
}

// Decode positions [b, e) of the row-ordered encoding from the slice stream (one warp per run)
__global__ void k_decode_slices(const uint32_t* __restrict__ w, const Tile* __restrict__ tiles,
                                const Segment* __restrict__ segs, const WarpRange* __restrict__ ranges,
                                uint32_t n_runs, uint32_t warps, uint32_t rep_stride, uint64_t b,
                                uint64_t e, uint32_t* __restrict__ col, uint16_t* __restrict__ val) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t n_gw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = gw; i < n_runs; i += n_gw) {
    const Tile T = tiles[i / warps];
    const WarpRange r0 = ranges[i], r1 = ranges[i + 1];
    uint64_t c = r0.chunk;
    for (uint32_t s = r0.seg; s < r1.seg; ++s) {
      const Segment S = segs[s];
      const uint32_t nch = (static_cast<uint32_t>(S.lane0) + S.n + 31) / 32;
      const uint64_t base0 = S.p0 - S.lane0;
      if (S.p0 + S.n <= b || S.p0 >= e) {
        c += nch;
        continue;
      }
      for (uint32_t j = 0; j < nch; ++j, ++c) {
        const uint32_t rel = 32 * j + lane;
        const uint64_t p = base0 + rel;
        if (rel < S.lane0 || rel >= S.lane0 + S.n || p < b || p >= e) continue;
        const uint32_t v = w[slice_word(c, lane)];
        const uint32_t slot = v >> 16;
        col[p - b] = T.nrep <= 1 ? T.xlo + slot : col_of_slot(slot, T.xlo, rep_stride);
        val[p - b] = static_cast<uint16_t>(v & 0xFFFFu);
      }
    }
  }
}

template <class M>
__global__ void k_decode_rest(M rest, const uint64_t* __restrict__ rp, const uint64_t* __restrict__ rest_rp,
                              uint64_t r0, uint64_t r1, uint64_t b, uint32_t* __restrict__ col,
                              uint16_t* __restrict__ val) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t r = r0 + warp; r < r1; r += n_warps) {
    const uint64_t d = rest_rp[r], n = rest_rp[r + 1] - d, o = rp[r] - b;
    for (uint64_t j = lane; j < n; j += 32) {
      const auto e = rest.load(d + j);
      col[o + j] = static_cast<uint32_t>(M::c_of(e));
      val[o + j] = static_cast<uint16_t>(M::v_of(e));
    }
  }
}

}  // namespace

// After plan_tiles (plan_slices): write the slice stream, compact the other rows into the rest
// stream, free the row-ordered upload.  Peak device memory: the upload plus the slice stream.
int build_slices(Handle* h) {
  if (!h->slices) return DG_OK;
  const uint64_t words = h->slice_chunks * 32;
  DG_CUDA(cudaMalloc(&h->d_slices, std::max<uint64_t>(words, 4) * 4));
  const uint32_t zero_slot = h->window_cols - 1;
  const uint32_t n_runs = h->wave_tiles[0] * h->slice_runs;
  // rest rows: non-empty rows no segment belongs to
  std::vector<uint64_t> rp(h->rows + 1);
  DG_CUDA(cudaMemcpy(rp.data(), h->d_row_ptr, (h->rows + 1) * 8, cudaMemcpyDeviceToHost));
  std::vector<uint8_t> tile_row(h->rows, 0);
  {
    std::vector<Segment> segs(h->n_segments);
    DG_CUDA(cudaMemcpy(segs.data(), h->d_segs[0], segs.size() * sizeof(Segment), cudaMemcpyDeviceToHost));
    for (const Segment& s : segs) tile_row[s.row] = 1;
  }
  // contiguous dense rows as values only (k_dense_values); the others stay k_dense's
  if (h->n_dense_rows && h->dense_contig.size() == h->n_dense_rows) {
    std::vector<uint32_t> drows(h->n_dense_rows), vrows, wrows;
    DG_CUDA(cudaMemcpy(drows.data(), h->d_dense_rows, drows.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < drows.size(); ++i) (h->dense_contig[i] ? vrows : wrows).push_back(drows[i]);
    if (!vrows.empty()) {
      std::vector<DenseRow> V(vrows.size());
      uint64_t blk = 0, vnnz = 0;
      for (size_t k = 0; k < vrows.size(); ++k) {
        const uint32_t r = vrows[k];
        const uint64_t len = rp[r + 1] - rp[r];
        V[k] = {r, 0, static_cast<uint32_t>(len), static_cast<uint32_t>(blk)};
        blk += ((len + 31) / 32 + kValueChunks - 1) / kValueChunks;
        if (blk > 0xFFFFFFFFull) return DG_ERR_UNSUPPORTED_FEATURE;
        vnnz += len;
        tile_row[r] = 1;  // not in the rest stream
      }
      h->n_value_rows = vrows.size();
      h->value_nnz = vnnz;
      h->value_blocks = blk;
      DG_CUDA(cudaMalloc(&h->d_vrows, V.size() * sizeof(DenseRow)));
      DG_CUDA(cudaMemcpy(h->d_vrows, V.data(), V.size() * sizeof(DenseRow), cudaMemcpyHostToDevice));
      DG_CUDA(cudaMalloc(&h->d_vstream, std::max<uint64_t>(blk, 1) * 32 * kValueChunks * 2));
      DG_CUDA(cudaMalloc(&h->d_value_counter, sizeof(uint32_t)));
      h->plan_bytes += V.size() * sizeof(DenseRow);
      const int st = dispatch_mat(h, [&](const auto& mat) {
        using M = std::decay_t<decltype(mat)>;
        if constexpr (std::is_same_v<typename M::Val, uint16_t>) {
          k_build_values<M><<<grid_for(32ull * vrows.size(), 256, 8), 256>>>(
              mat, h->d_row_ptr, static_cast<DenseRow*>(h->d_vrows), static_cast<uint32_t>(vrows.size()),
              h->d_vstream);
          return DG_OK;
        } else {
          return DG_ERR_UNSUPPORTED_FEATURE;
        }
      });
      if (st) return st;
      DG_CUDA(cudaGetLastError());
      // the word rows stay in d_dense_rows (longest first)
      h->n_dense_rows = wrows.size();
      h->dense_nnz -= vnnz;
      if (!wrows.empty())
        DG_CUDA(cudaMemcpy(h->d_dense_rows, wrows.data(), wrows.size() * 4, cudaMemcpyHostToDevice));
    }
  }
  // dense rows as one-segment runs (k_dense_slices): Packed16 (column field < 65536, so the
  // neutral column `cols` fits), DG_DENSE_SLICES=0 keeps k_dense on the rest stream
  h->dense_slices = h->packed && h->n_dense_rows > 0;
  if (const char* ds = std::getenv("DG_DENSE_SLICES")) h->dense_slices = h->dense_slices && std::atoi(ds) != 0;
  if (h->dense_slices) {
    std::vector<uint32_t> drows(h->n_dense_rows);
    DG_CUDA(cudaMemcpy(drows.data(), h->d_dense_rows, drows.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<WarpRange> R(drows.size() + 1);
    std::vector<SliceSeg> S(drows.size());
    uint64_t c = 0;
    for (size_t k = 0; k < drows.size(); ++k) {
      const uint32_t r = drows[k];
      const uint32_t nch = static_cast<uint32_t>((rp[r + 1] - rp[r] + 31) / 32);
      R[k] = {static_cast<uint32_t>(c), static_cast<uint32_t>(k)};
      S[k] = {r, 0, nch, static_cast<uint32_t>(kSegFirst | kSegLast)};
      c += (nch + kSlicePad - 1) / kSlicePad * kSlicePad;
      if (c > 0xFFFFFFFFull) return DG_ERR_UNSUPPORTED_FEATURE;
      tile_row[r] = 1;  // not in the rest stream
    }
    R[drows.size()] = {static_cast<uint32_t>(c), static_cast<uint32_t>(drows.size())};
    h->dense_chunks = c;
    DG_CUDA(cudaMalloc(&h->d_dslices, std::max<uint64_t>(c * 32, 4) * 4));
    DG_CUDA(cudaMalloc(&h->d_dranges, R.size() * sizeof(WarpRange)));
    DG_CUDA(cudaMemcpy(h->d_dranges, R.data(), R.size() * sizeof(WarpRange), cudaMemcpyHostToDevice));
    DG_CUDA(cudaMalloc(&h->d_dsseg, S.size() * sizeof(SliceSeg)));
    DG_CUDA(cudaMemcpy(h->d_dsseg, S.data(), S.size() * sizeof(SliceSeg), cudaMemcpyHostToDevice));
    h->plan_bytes += R.size() * sizeof(WarpRange) + S.size() * sizeof(SliceSeg);
    k_build_dense<<<grid_for(32ull * drows.size(), 256, 8), 256>>>(
        Packed16{h->d_packed}, h->d_row_ptr, static_cast<const SliceSeg*>(h->d_dsseg),
        static_cast<const WarpRange*>(h->d_dranges), static_cast<uint32_t>(drows.size()), h->d_dslices,
        static_cast<uint32_t>(h->cols) << 16);
    DG_CUDA(cudaGetLastError());
  }
  std::vector<uint64_t> rest_rp(h->rows + 1, 0);
  for (uint64_t r = 0; r < h->rows; ++r)
    rest_rp[r + 1] = rest_rp[r] + (tile_row[r] ? 0 : rp[r + 1] - rp[r]);
  const uint64_t rest_nnz = rest_rp[h->rows];
  uint64_t* d_rest_rp = nullptr;
  DG_CUDA(cudaMalloc(&d_rest_rp, (h->rows + 1) * 8));
  DG_CUDA(cudaMemcpy(d_rest_rp, rest_rp.data(), (h->rows + 1) * 8, cudaMemcpyHostToDevice));
  uint32_t* rw = nullptr;
  void* rc = nullptr;
  uint16_t* rv = nullptr;
  int st = DG_OK;
  auto cu = [&](cudaError_t e) { if (st == DG_OK && e != cudaSuccess) st = DG_ERR_CUDA_BASE + (int)e; };
  if (h->packed) {
    cu(cudaMalloc(&rw, std::max<uint64_t>(rest_nnz, 1) * 4 + 16));
  } else {
    cu(cudaMalloc(&rc, std::max<uint64_t>(rest_nnz, 1) * h->index_bytes));
    cu(cudaMalloc(reinterpret_cast<void**>(&rv), std::max<uint64_t>(rest_nnz, 1) * 2));
  }
  if (st == DG_OK) {
    st = dispatch_mat(h, [&](const auto& mat) {
      using M = std::decay_t<decltype(mat)>;
      if constexpr (std::is_same_v<typename M::Val, uint16_t>) {
        if (n_runs)
          k_build_slices<M><<<grid_for(32ull * n_runs, 256, 8), 256>>>(
              mat, static_cast<const Tile*>(h->d_tiles[0]), static_cast<const Segment*>(h->d_segs[0]),
              static_cast<const WarpRange*>(h->d_ranges), n_runs, h->slice_runs, h->d_slices,
              h->rep_stride, zero_slot);
        if (rest_nnz)
          k_copy_rest<M><<<grid_for(32ull * h->rows, 256, 8), 256>>>(mat, h->d_row_ptr, d_rest_rp,
                                                                    h->rows, rw, rc, rv);
        return DG_OK;
      } else {
        return DG_ERR_UNSUPPORTED_FEATURE;  // slices are planned for binary16 values only
      }
    });
  }
  cu(cudaGetLastError());
  cu(cudaDeviceSynchronize());
  if (st) {
    cudaFree(d_rest_rp);
    cudaFree(rw);
    cudaFree(rc);
    cudaFree(rv);
    return st;
  }
  // the row-ordered upload is no longer needed: the rest stream takes its place
  cudaFree(h->d_packed);
  cudaFree(h->d_col);
  cudaFree(h->d_val);
  h->d_packed = rw;
  h->d_col = rc;
  h->d_val = rv;
  h->d_row_ptr_orig = h->d_row_ptr;
  h->d_row_ptr = d_rest_rp;
  h->rest_nnz = rest_nnz;
  // resident matrix bytes now: both row pointers, the slice / dense-slice / value streams and the
  // rest stream (dg_get_info.device_bytes)
  h->matrix_bytes = 2 * (h->rows + 1) * 8 + (h->slice_chunks + h->dense_chunks) * 32 * 4 +
                    h->value_blocks * 32 * kValueChunks * 2 +
                    rest_nnz * (h->packed ? 4 : h->index_bytes + 2);
  return DG_OK;
}

// Positions of rows [r0, r1) in the row-ordered encoding -> col (u32) / val (binary16 bits),
// device arrays of rp[r1] - rp[r0] entries.
int decode_rows(const Handle* h, uint64_t r0, uint64_t r1, uint32_t* d_col, uint16_t* d_val) {
  uint64_t b = 0, e = 0;
  DG_CUDA(cudaMemcpy(&b, h->d_row_ptr_orig + r0, 8, cudaMemcpyDeviceToHost));
  DG_CUDA(cudaMemcpy(&e, h->d_row_ptr_orig + r1, 8, cudaMemcpyDeviceToHost));
  if (e == b) return DG_OK;
  const uint32_t n_runs = h->wave_tiles[0] * h->slice_runs;
  if (n_runs)
    k_decode_slices<<<grid_for(32ull * n_runs, 256, 8), 256>>>(
        h->d_slices, static_cast<const Tile*>(h->d_tiles[0]), static_cast<const Segment*>(h->d_segs[0]),
        static_cast<const WarpRange*>(h->d_ranges), n_runs, h->slice_runs, h->rep_stride, b, e,
        d_col, d_val);
  if (h->n_value_rows)
    k_decode_values<<<grid_for(32ull * h->n_value_rows, 256, 8), 256>>>(
        h->d_vstream, static_cast<const DenseRow*>(h->d_vrows), static_cast<uint32_t>(h->n_value_rows),
        h->d_row_ptr_orig, r0, r1, b, d_col, d_val);
  if (h->dense_slices)
    k_decode_dense<<<grid_for(32ull * h->n_dense_rows, 256, 8), 256>>>(
        h->d_dslices, static_cast<const SliceSeg*>(h->d_dsseg), static_cast<const WarpRange*>(h->d_dranges),
        static_cast<uint32_t>(h->n_dense_rows), h->d_row_ptr_orig, r0, r1, b, d_col, d_val);
  if (h->rest_nnz) {
    const int st = dispatch_mat(h, [&](const auto& mat) {
      using M = std::decay_t<decltype(mat)>;
      if constexpr (std::is_same_v<typename M::Val, uint16_t>) {
        k_decode_rest<M><<<grid_for(32ull * (r1 - r0), 256, 8), 256>>>(
            mat, h->d_row_ptr_orig, h->d_row_ptr, r0, r1, b, d_col, d_val);
        return DG_OK;
      } else {
        return DG_ERR_UNSUPPORTED_FEATURE;
      }
    });
    if (st) return st;
  }
  DG_CUDA(cudaGetLastError());
  DG_CUDA(cudaDeviceSynchronize());
  return DG_OK;
}

template <typename Acc>
int launch_slices(Handle* h, const Acc* x, double* y, cudaStream_t s) {
  const size_t smem = 2ull * h->window_cols * sizeof(Acc);
  const bool carry = h->n_carry_slots != 0;
#ifndef DG_SLICE_P_EXACT
#define DG_SLICE_P_EXACT 3  // r02 at 28 warps: P = 2 / 3 / 4: C2 slices 1.229 / 1.211 / 1.210 ms, C4 3.546 / 3.509
#endif
  constexpr int kP = std::is_same_v<Acc, float> ? 4 : DG_SLICE_P_EXACT;
  // short segments (mean < 256 nonzeros, C1: 136): 4-chunk batches -- fewer chunks per batch
  // behind each segment end
  auto kern = carry                ? k_slices<Acc, Handle::kSliceWarpsCarry, kP, true>
              : h->short_segments ? k_slices<Acc, Handle::kSliceWarpsShort, kP, false, 2, 4>
                                   : k_slices<Acc, Handle::kSliceWarps, kP, false>;
  const int warps = carry ? Handle::kSliceWarpsCarry
                    : h->short_segments ? Handle::kSliceWarpsShort : Handle::kSliceWarps;
  if (!h->tiles_attr) {
    DG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    h->tiles_attr = true;
  }
  if (!h->pdl_next) DG_CUDA(cudaMemsetAsync(h->d_counters, 0, Handle::kMaxWaves * sizeof(uint32_t), s));
  BlockSignal sig{nullptr, nullptr, 0};
  if (h->signal_blocks) {
    DG_CUDA(cudaMemcpyAsync(h->d_blk_left, h->d_blk_left_init, h->n_blocks * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, s));
    sig = {h->d_blk_left, h->d_blk_flag, h->epoch};
    DG_CUDA(cudaEventRecord(h->ev_tiles_start, s));
  }
  TileTrace tr{nullptr, nullptr};
  if (h->d_trace) {
    const uint64_t n = 4ull * h->sm_count + 3ull * h->wave_tiles[0];
    DG_CUDA(cudaMemsetAsync(h->d_trace, 0, n * sizeof(unsigned long long), s));
    tr = {h->d_trace, h->d_trace + 4ull * h->sm_count};
  }
  if (!h->wave_tiles[0]) return DG_OK;
  const Carry<Acc> cr{static_cast<Acc*>(h->d_state)};
  const XSource<Acc> xsrc{x, std::is_same_v<Acc, double> ? reinterpret_cast<const Acc*>(h->d_x1) : nullptr,
                          h->rep_stride};
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(std::min<int>(h->sm_count, static_cast<int>(h->wave_tiles[0])));
  lc.blockDim = dim3(warps * 32);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  if (h->pdl_next) {
    lc.attrs = at;
    lc.numAttrs = 1;
  }
  DG_CUDA(cudaLaunchKernelEx(&lc, kern, reinterpret_cast<const uint4*>(h->d_slices), xsrc,
                             static_cast<const Tile*>(h->d_tiles[0]), h->wave_tiles[0],
                             static_cast<uint32_t>(h->slice_runs),
                             static_cast<const WarpRange*>(h->d_ranges),
                             static_cast<const SliceSeg*>(h->d_sseg), cr, y, h->d_counters,
                             h->window_cols, sig, h->gt, tr));
  h->post(s, h->n_waves > 1 ? "slices[fused]" : "slices", h->fused_waves ? h->fused_rows : h->wave_rows[0],
          h->fused_waves ? h->fused_nnz : h->wave_nnz[0]);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}
// the contiguous rows (k_dense_values); `last`: no other dense launch follows, so the tile
// kernel may follow it as a programmatic dependent launch
template <typename Acc>
int launch_values(Handle* h, const Acc* x, double* y, cudaStream_t s, bool last) {
  if (!h->n_value_rows) return DG_OK;
  DG_CUDA(cudaMemsetAsync(h->d_value_counter, 0, sizeof(uint32_t), s));
  h->pdl_next = last && h->pdl && h->n_waves && !h->profiling && !h->signal_blocks && !h->d_trace;
  if (h->pdl_next) DG_CUDA(cudaMemsetAsync(h->d_counters, 0, Handle::kMaxWaves * sizeof(uint32_t), s));
  const int grid = h->pdl_next ? h->sm_count * 4 : grid_for(h->n_value_rows * 32ull, 256, 8);
  static const int cfg = [] { const char* c = std::getenv("DG_VALUES_CFG"); return c ? std::atoi(c) : 0; }();
  auto kern = cfg == 1 ? k_dense_values<Acc, 4> : cfg == 2 ? k_dense_values<Acc, 8> :
              cfg == 3 ? k_dense_values<Acc, 0> : k_dense_values<Acc, 2>;
  kern<<<grid, 256, 0, s>>>(
      reinterpret_cast<const uint4*>(h->d_vstream), static_cast<const DenseRow*>(h->d_vrows),
      static_cast<uint32_t>(h->n_value_rows), x, static_cast<uint32_t>(h->cols), h->d_value_counter, y, h->gt);
  h->post(s, "dense_values", h->n_value_rows, h->value_nnz);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}
template int launch_values<double>(Handle*, const double*, double*, cudaStream_t, bool);
template int launch_values<float>(Handle*, const float*, double*, cudaStream_t, bool);

template <typename Acc>
int launch_dense_slices(Handle* h, const Acc* x, double* y, cudaStream_t s) {
  if (!h->n_dense_rows) return DG_OK;
  h->pdl_next = false;
  DG_CUDA(cudaMemsetAsync(h->d_dense_counter, 0, sizeof(uint32_t), s));
  // the tile kernel follows as a programmatic dependent launch unless something must sit between
  // the two launches (per-launch profiling events, the row-block signals, the trace)
  h->pdl_next = h->pdl && h->n_waves && !h->profiling && !h->signal_blocks && !h->d_trace;
  if (h->pdl_next) DG_CUDA(cudaMemsetAsync(h->d_counters, 0, Handle::kMaxWaves * sizeof(uint32_t), s));
  const int grid = h->pdl_next ? h->sm_count * 4 : grid_for(h->n_dense_rows * 32ull, 256, 8);
  constexpr int kP = 4;
  k_dense_slices<Acc, kP><<<grid, 256, 0, s>>>(
      reinterpret_cast<const uint4*>(h->d_dslices), static_cast<const WarpRange*>(h->d_dranges),
      static_cast<const SliceSeg*>(h->d_dsseg), static_cast<uint32_t>(h->n_dense_rows), x,
      h->d_dense_counter, y, h->gt);
  h->post(s, "dense", h->n_dense_rows, h->dense_nnz);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}
template int launch_dense_slices<double>(Handle*, const double*, double*, cudaStream_t);
template int launch_dense_slices<float>(Handle*, const float*, double*, cudaStream_t);

template int launch_slices<double>(Handle*, const double*, double*, cudaStream_t);
template int launch_slices<float>(Handle*, const float*, double*, cudaStream_t);

}  // namespace dg
