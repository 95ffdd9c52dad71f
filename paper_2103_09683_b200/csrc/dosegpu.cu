// dosegpu.cu -- C-ABI implementation: validation, row plan, one-time native-encoding upload and
// the dose evaluation (include/dosegpu.h).  No CPU fallback: every dose is computed on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"
#include "handle.cuh"
#include "spmv_kernels.cuh"
#include "spmv_tiles.cuh"

namespace dg {

__global__ void k_narrow_u32_u16(const uint32_t* __restrict__ in, uint16_t* __restrict__ out,
                                 uint64_t n, uint64_t cols, unsigned* __restrict__ bad) {
  unsigned flag = 0;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = in[i];
    if (c >= cols) flag = 1u;
    out[i] = static_cast<uint16_t>(c);
  }
  if (flag) atomicOr(bad, flag);
}

__global__ void k_pack16(const uint16_t* __restrict__ col, const uint16_t* __restrict__ val,
                         uint32_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = pack16(col[i], val[i]);
}

// rows [r0, r1) of the stream back to the reference's host encoding (u32 columns, value bits)
template <class M>
__global__ void k_unpack(M mat, uint64_t b, uint64_t n, uint32_t* __restrict__ col,
                         typename M::Val* __restrict__ val) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const auto e = mat.load(b + i);
    col[i] = M::c_of(e);
    val[i] = M::v_of(e);
  }
}

// x staging: dst0 <- src (skipped when they alias), dst1 (the shifted copy, XSource) <- src
__global__ void k_stage_x(const double* __restrict__ src, double* dst0, double* __restrict__ dst1,
                          uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double v = src[i];
    if (dst0 != src) dst0[i] = v;
    if (dst1) dst1[i] = v;
  }
}

__global__ void k_rebase(uint64_t* __restrict__ rp, uint64_t n, uint64_t base) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    rp[i] -= base;
}

int grid_for(uint64_t work_items, int threads, int max_blocks_per_sm) {
  // SM count per device, queried once (not on every launch)
  constexpr int kMaxDev = 64;
  static int sm_of[kMaxDev] = {};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < kMaxDev) {
    if (!sm_of[dev]) {
      int v = 0;
      if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sm_of[dev] = v;
    }
    if (sm_of[dev]) sms = sm_of[dev];
  }
  const uint64_t need = (work_items + threads - 1) / threads;
  const uint64_t cap = static_cast<uint64_t>(sms) * max_blocks_per_sm;
  return static_cast<int>(std::max<uint64_t>(1, std::min(need, cap)));
}

// ------------------------------------------------------------------------------------------
int select_device(int32_t want, int* dev_out) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return DG_ERR_NO_DEVICE;
  }
  int dev = want;
  if (dev < 0) DG_CUDA(cudaGetDevice(&dev));
  if (dev >= n) return DG_ERR_INVALID_CONFIG;
  cudaDeviceProp prop;
  DG_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return DG_ERR_NO_DEVICE;  // built for sm_100a only
  DG_CUDA(cudaSetDevice(dev));
  *dev_out = dev;
  return DG_OK;
}

int check_options(const dg_options* o) {
  if (!o) return DG_OK;
  if (o->struct_size != sizeof(dg_options)) return DG_ERR_INVALID_CONFIG;
  const uint32_t L = o->lane_width;
  if (L < 1 || L > 1024 || (L & (L - 1))) return DG_ERR_INVALID_CONFIG;  // spmv.cpp:40-46
  if (o->accumulation > DG_ACCUM_FP32) return DG_ERR_INVALID_CONFIG;
  if (o->accumulation == DG_ACCUM_FP32 && L != 32) return DG_ERR_INVALID_CONFIG;
  return DG_OK;
}

// ------------------------------------------------------------------------------------------
// Row plan, part 1: non-empty rows of length <= 32 binned by next_pow2(len) (lane_width 32),
// or every non-empty row in one list (other lane widths).  Longer rows: plan_tiles (plan.cu);
// DG_PLAN=warp keeps the v0 warp-per-row bin instead, longest row first.
int build_plan(Handle* h, const std::vector<uint64_t>& lens) {
  std::vector<std::vector<uint32_t>> bins(kNumBins);
  uint64_t nonempty = 0, short_rows = 0;
  for (uint64_t len : lens) {
    nonempty += len > 0;
    short_rows += len > 0 && len <= 32;
  }
  // Few short rows: fold them into the tiles (a warp per row, one fewer launch per bin); many:
  // sub-warp bins, G = next_pow2(len) lanes per row.
  uint64_t short_nnz = 0, all_nnz = 0;
  for (uint64_t len : lens) {
    all_nnz += len;
    if (len <= 32) short_nnz += len;
  }
  h->short_max = (short_rows * 20 < nonempty || short_nnz * 50 < all_nnz) ? 0 : 32;
  if (const char* sm = std::getenv("DG_SHORT_MAX"))
    h->short_max = std::min<uint64_t>(32, std::strtoull(sm, nullptr, 10));
  for (uint64_t r = 0; r < lens.size(); ++r) {
    const uint64_t len = lens[r];
    if (len == 0) continue;
    int b;
    if (h->lane_width != 32) b = kBinGeneral;
    else if (h->use_tiles && len > h->short_max) continue;  // plan_tiles owns it
    else if (len == 1) b = 0;
    else if (len == 2) b = 1;
    else if (len <= 4) b = 2;
    else if (len <= 8) b = 3;
    else if (len <= 16) b = 4;
    else if (len <= 32) b = 5;
    else if (h->use_tiles) continue;
    else b = kBinLong;
    bins[b].push_back(static_cast<uint32_t>(r));
  }
  std::stable_sort(bins[kBinLong].begin(), bins[kBinLong].end(),
                   [&](uint32_t a, uint32_t b) { return lens[a] > lens[b]; });
  h->nonempty_rows = nonempty;
  for (int b = 0; b < kNumBins; ++b) {
    h->bin_count[b] = static_cast<uint32_t>(bins[b].size());
    for (uint32_t r : bins[b]) h->bin_nnz[b] += lens[r];
    if (bins[b].empty()) continue;
    DG_CUDA(cudaMalloc(&h->d_bin[b], bins[b].size() * 4));
    DG_CUDA(cudaMemcpy(h->d_bin[b], bins[b].data(), bins[b].size() * 4, cudaMemcpyHostToDevice));
    h->plan_bytes += bins[b].size() * 4;
  }
  return DG_OK;
}

// ------------------------------------------------------------------------------------------
template <int G, class M, typename Acc>
void launch_group(Handle* h, int b, const char* name, cudaStream_t s, const M& mat, const Acc* x,
                  double* y) {
  const uint32_t cnt = h->bin_count[b];
  if (!cnt) return;
  k_group<G, M, Acc><<<grid_for(static_cast<uint64_t>(cnt) * G, 256), 256, 0, s>>>(
      mat, h->d_row_ptr, x, h->d_bin[b], cnt, y, h->gt);
  h->post(s, name, cnt, h->bin_nnz[b]);
}

// One persistent launch per wave (one CTA per SM): wave k continues the segments whose lane
// partials wave k-1 stored.
template <class M, typename Acc, int kWarps, int kU, int kP = 0, int kNB = 2, bool kCarry = true>
int launch_tiles_cfg(Handle* h, const M& mat, const Acc* x, double* y, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(kNB) * h->window_cols * sizeof(Acc);
  if (!h->tiles_attr) {  // a handle has one (M, Acc, config) and one device
    DG_CUDA(cudaFuncSetAttribute(k_tiles<M, Acc, kWarps, kU, kP, kNB, kCarry>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    h->tiles_attr = true;
  }
  // (after k_dense with programmatic launch, the counters were reset before k_dense: the tile
  //  kernel must be the next operation in the stream)
  if (!h->pdl_next) DG_CUDA(cudaMemsetAsync(h->d_counters, 0, Handle::kMaxWaves * sizeof(uint32_t), s));
  BlockSignal sig{nullptr, nullptr, 0};
  if (h->signal_blocks) {
    DG_CUDA(cudaMemcpyAsync(h->d_blk_left, h->d_blk_left_init, h->n_blocks * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, s));
    sig = {h->d_blk_left, h->d_blk_flag, h->epoch};
  }
  if (h->signal_blocks)  // every row not owned by a tile is final here
    DG_CUDA(cudaEventRecord(h->ev_tiles_start, s));
  static const char* const kWaveName[] = {"tiles[w0]", "tiles[w1]", "tiles[w2]", "tiles[w3]",
                                          "tiles[w4]", "tiles[w5]", "tiles[w6]", "tiles[w7]",
                                          "tiles[w8+]"};
  TileTrace tr{nullptr, nullptr};
  if (h->d_trace) {  // diagnostic timeline of wave 0 (DG_TRACE)
    const uint64_t n = 4ull * h->sm_count + 3ull * h->wave_tiles[0];
    DG_CUDA(cudaMemsetAsync(h->d_trace, 0, n * sizeof(unsigned long long), s));
    tr = {h->d_trace, h->d_trace + 4ull * h->sm_count};
  }
  const Carry<Acc> carry{static_cast<Acc*>(h->d_state)};
  for (uint32_t w = 0; w < h->n_launch_lists(); ++w) {
    if (!h->wave_tiles[w]) continue;
    const int grid = std::min<int>(h->sm_count, static_cast<int>(h->wave_tiles[w]));
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kWarps * 32);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    if (h->pdl_next && w == 0) {  // overlaps the tail of k_dense (launched just before)
      lc.attrs = at;
      lc.numAttrs = 1;
    }
    const XSource<Acc> xsrc{x, std::is_same_v<Acc, double> ? reinterpret_cast<const Acc*>(h->d_x1) : nullptr,
                            h->rep_stride};
    DG_CUDA(cudaLaunchKernelEx(&lc, k_tiles<M, Acc, kWarps, kU, kP, kNB, kCarry>, mat, xsrc,
                               static_cast<const Tile*>(h->d_tiles[w]), h->wave_tiles[w],
                               static_cast<const Segment*>(h->d_segs[w]), carry, y,
                               h->d_counters + w, h->window_cols, sig, h->gt,
                               w == 0 ? tr : TileTrace{nullptr, nullptr}));
    if (h->fused_waves)
      h->post(s, "tiles[fused]", h->fused_rows, h->fused_nnz);
    else
      h->post(s, kWaveName[std::min<uint32_t>(w, 8)], h->wave_rows[w], h->wave_nnz[w]);
  }
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

// Tile-kernel configurations (warps per CTA, batch depth U, L2 prefetch distance P, x-window
// buffers NB).  DG_TILE_CFG selects an alternative for measurement; the default is the measured
// best on C2 (profiles/).  (Rejected in r01 and removed: a per-warp TMA ring for the matrix
// stream, 24 warps x 4 stages of 1 KB -- instruction-bound, C2 4.16 ms.)
int tile_buffers_of(int cfg, bool packed) {
  if (!packed) return 2;
  switch (cfg) {
    case 12: return 3;
    case 13: return 4;
    default: return 2;
  }
}

// Dense rows first (k_dense, rows pulled longest first by warps of 8-warp CTAs): every row it
// owns is final before the tile kernel -- and the row-block completion signals -- start.
template <class M, typename Acc>
int launch_dense(Handle* h, const M& mat, const Acc* x, double* y, cudaStream_t s) {
  h->pdl_next = false;
  DG_TRY(launch_values<Acc>(h, x, y, s, h->n_dense_rows == 0));  // the contiguous rows first
  if (h->dense_slices) return launch_dense_slices<Acc>(h, x, y, s);
  if (!h->n_dense_rows) return DG_OK;
  DG_CUDA(cudaMemsetAsync(h->d_dense_counter, 0, sizeof(uint32_t), s));
  // The tile kernel follows as a programmatic dependent launch (it may start on SMs k_dense has
  // left while k_dense's last rows finish) unless something must sit between the two launches:
  // per-launch profiling events, or the row-block signals of the overlapped host download.
  h->pdl_next = h->pdl && h->n_waves && !h->profiling && !h->signal_blocks && !h->d_trace;
  if (h->pdl_next)
    DG_CUDA(cudaMemsetAsync(h->d_counters, 0, Handle::kMaxWaves * sizeof(uint32_t), s));
  // persistent when followed programmatically: every CTA resident (and triggered) at once
  const int grid = h->pdl_next ? h->sm_count * 4 : grid_for(h->n_dense_rows * 32ull, 256, 8);
  switch (h->dense_cfg) {
    case 1:
      k_dense<M, Acc, 16, 2><<<grid, 256, 0, s>>>(mat, h->d_row_ptr, x, h->d_dense_rows,
                                                  static_cast<uint32_t>(h->n_dense_rows),
                                                  h->d_dense_counter, y, h->gt);
      break;
    case 2:
      k_dense<M, Acc, 8, 8><<<grid, 256, 0, s>>>(mat, h->d_row_ptr, x, h->d_dense_rows,
                                                 static_cast<uint32_t>(h->n_dense_rows),
                                                 h->d_dense_counter, y, h->gt);
      break;
    default:
      k_dense<M, Acc, 8, 4><<<grid, 256, 0, s>>>(mat, h->d_row_ptr, x, h->d_dense_rows,
                                                 static_cast<uint32_t>(h->n_dense_rows),
                                                 h->d_dense_counter, y, h->gt);
  }
  h->post(s, "dense", h->n_dense_rows, h->dense_nnz);
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

template <class M, typename Acc>
int launch_tiles(Handle* h, const M& mat, const Acc* x, double* y, cudaStream_t s,
                 const char* /*name*/) {
  // (measured, rejected: k_dense on a side stream beside a 24-warp tile kernel, one CTA of each
  //  per SM -- C2 3.89 ms vs 2.88 back to back; profiles/README.md)
  // (measured, rejected: the contiguous rows AFTER the tile kernel as its programmatic dependent,
  //  to fill the tile kernel's tail -- C2 1.97 vs 1.75 ms, C3 shard 0.29 vs 0.26: the value
  //  kernel's CTAs then start on SMs still configured for the tile kernel's shared memory, and
  //  it is L1-bound)
  DG_TRY(launch_dense(h, mat, x, y, s));
  if (!h->n_waves) return DG_OK;
  if (h->slices) return launch_slices<Acc>(h, x, y, s);
  constexpr int kP = std::is_same_v<Acc, float> ? 4 : 2;  // measured: prefetch distance
  if constexpr (std::is_same_v<M, Packed16>) {
    switch (h->tile_cfg) {
      case 8: return launch_tiles_cfg<M, Acc, 32, 8, 1>(h, mat, x, y, s);
      case 10: return launch_tiles_cfg<M, Acc, 32, 8, 4>(h, mat, x, y, s);
      case 11: return launch_tiles_cfg<M, Acc, 32, 8, 0>(h, mat, x, y, s);
      case 12: return launch_tiles_cfg<M, Acc, 32, 8, kP, 3>(h, mat, x, y, s);
      case 13: return launch_tiles_cfg<M, Acc, 32, 8, kP, 4>(h, mat, x, y, s);
      // (A/B: narrow batches with P = 4; U = 4, P = 2 is the short-segment default below)
      case 19: return launch_tiles_cfg<M, Acc, 32, 4, 4>(h, mat, x, y, s);
      // (measured, rejected: wider batches U = 12 at 32 / 28 warps, U = 16 at 28 warps --
      //  C2 2.70 / 2.66 / 2.82 ms vs 2.62; profiles/README.md)
      // (measured, rejected: cp.async.bulk.prefetch.L2 by one lane instead of per-line
      //  prefetches, P = 2/4/8 -- C2 2.94-3.00 ms vs 2.80; profiles/README.md)
      default:
        // short segments (mean < 256 nonzeros, C1: 136): 4-chunk batches waste fewer masked
        // chunks at each segment's end (C1 0.157 -> 0.148 ms; C2 would lose: 2.63 -> 3.19)
        if (!h->n_carry_slots && h->short_segments)
          return launch_tiles_cfg<M, Acc, Handle::kTileWarps, 4, 2, 2, false>(h, mat, x, y, s);
        if (!h->n_carry_slots)  // no split rows: the carry code is compiled out
          return launch_tiles_cfg<M, Acc, Handle::kTileWarps, Handle::kTileUnroll, kP, 2, false>(
              h, mat, x, y, s);
        return launch_tiles_cfg<M, Acc, Handle::kTileWarps, Handle::kTileUnroll, kP>(h, mat, x, y, s);
    }
  }
  // SoA elements take two registers each: 24 warps leave room for two U = 8 batches
  if (!h->n_carry_slots)
    return launch_tiles_cfg<M, Acc, 24, Handle::kTileUnroll, kP, 2, false>(h, mat, x, y, s);
  // split rows: 20 warps leave 96 registers, room for the carried-partials peek (C4: 6.70 ms
  // vs 6.80 at 24 warps without the peek, 7.37 at 16 warps)
  switch (h->tile_cfg) {
    case 30: return launch_tiles_cfg<M, Acc, 24, Handle::kTileUnroll, kP>(h, mat, x, y, s);
    // (measured, rejected: 4-chunk batches at 24 / 32 warps -- C4 7.49 / 7.12 ms vs 6.65)
    // (measured, rejected: 18 / 22 warps -- C4 7.02 / 6.88 ms vs 6.65 at 20)
    default: return launch_tiles_cfg<M, Acc, 20, Handle::kTileUnroll, kP>(h, mat, x, y, s);
  }
}

// Bytes of one x-window buffer: two buffers of kWindowBytes, or what is left of the 227 KB of
// shared memory per CTA split in NB buffers, rounded down to 3 KB (whole replicas in slot mode).
uint32_t window_bytes_for(int cfg, bool packed) {
  constexpr size_t kMaxDyn = 232448 - 256;  // cudaDevAttrMaxSharedMemoryPerBlockOptin - static
  const int nb = tile_buffers_of(cfg, packed);
  if (nb == 2) return kWindowBytes;
  return static_cast<uint32_t>(kMaxDyn / nb / 3072 * 3072);
}

template <class M>
int launch_exact(Handle* h, const M& mat, const double* x, double* y, cudaStream_t s) {
  if (h->lane_width == 32) {
    launch_group<1>(h, 0, "group<1>", s, mat, x, y);
    launch_group<2>(h, 1, "group<2>", s, mat, x, y);
    launch_group<4>(h, 2, "group<4>", s, mat, x, y);
    launch_group<8>(h, 3, "group<8>", s, mat, x, y);
    launch_group<16>(h, 4, "group<16>", s, mat, x, y);
    launch_group<32>(h, 5, "group<32>", s, mat, x, y);
    if (h->bin_count[kBinLong]) {
      k_warp<M, double><<<grid_for(32ull * h->bin_count[kBinLong], 256), 256, 0, s>>>(
          mat, h->d_row_ptr, x, h->d_bin[kBinLong], h->bin_count[kBinLong], y, h->gt);
      h->post(s, "warp_v0", h->bin_count[kBinLong], h->bin_nnz[kBinLong]);
    }
    DG_TRY(launch_tiles(h, mat, x, y, s, "tiles"));
  } else {
    switch (h->lane_width) {
      case 1: launch_group<1>(h, kBinGeneral, "group<L=1>", s, mat, x, y); break;
      case 2: launch_group<2>(h, kBinGeneral, "group<L=2>", s, mat, x, y); break;
      case 4: launch_group<4>(h, kBinGeneral, "group<L=4>", s, mat, x, y); break;
      case 8: launch_group<8>(h, kBinGeneral, "group<L=8>", s, mat, x, y); break;
      case 16: launch_group<16>(h, kBinGeneral, "group<L=16>", s, mat, x, y); break;
      default: {
        const int L = static_cast<int>(h->lane_width);
        const uint32_t cnt = h->bin_count[kBinGeneral];
        if (cnt) {
          k_block_exact<M><<<grid_for(cnt, 1, 16), L, L * sizeof(double), s>>>(
              mat, h->d_row_ptr, x, h->d_bin[kBinGeneral], cnt, y, h->gt);
          h->post(s, "block<L>", cnt, h->bin_nnz[kBinGeneral]);
        }
      }
    }
  }
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

template <class M>
int launch_fp32(Handle* h, const M& mat, const float* x, double* y, cudaStream_t s) {
  launch_group<1>(h, 0, "group_f32<1>", s, mat, x, y);
  launch_group<2>(h, 1, "group_f32<2>", s, mat, x, y);
  launch_group<4>(h, 2, "group_f32<4>", s, mat, x, y);
  launch_group<8>(h, 3, "group_f32<8>", s, mat, x, y);
  launch_group<16>(h, 4, "group_f32<16>", s, mat, x, y);
  launch_group<32>(h, 5, "group_f32<32>", s, mat, x, y);
  if (h->bin_count[kBinLong]) {
    k_warp<M, float><<<grid_for(32ull * h->bin_count[kBinLong], 256), 256, 0, s>>>(
        mat, h->d_row_ptr, x, h->d_bin[kBinLong], h->bin_count[kBinLong], y, h->gt);
    h->post(s, "warp_f32_v0", h->bin_count[kBinLong], h->bin_nnz[kBinLong]);
  }
  DG_TRY(launch_tiles(h, mat, x, y, s, "tiles_f32"));
  DG_CUDA(cudaGetLastError());
  return DG_OK;
}

int run_kernels(Handle* h, const double* d_x, double* d_y, cudaStream_t s) {
  h->n_launch = 0;
  // empty rows are +0.0 (spmv.cpp:56): the caller's device d every dose; the handle's own d (host
  // path) once -- no kernel writes an empty row
  if (h->rows && (d_y != h->d_y || !h->dy_zeroed)) {
    DG_CUDA(cudaMemsetAsync(d_y, 0, h->rows * sizeof(double), s));
    if (d_y == h->d_y) h->dy_zeroed = true;
  }
  // fused gather: this shard's rows of every rank's full d start at +0.0 (its empty rows); the
  // kernels then store each finished row into every target over NVLink.  Once per target list:
  // no kernel ever writes an empty row, so later doses find them still +0.0 (the full-d buffers
  // are the library's, read-only to the caller) -- no rows x targets x 8 B of remote zeroes per dose
  if (!h->gt_zeroed) {
    for (uint32_t i = 0; i < h->gt.n && h->rows; ++i)
      DG_CUDA(cudaMemsetAsync(h->gt.t[i] + h->gt.row_off, 0, h->rows * sizeof(double), s));
    h->gt_zeroed = true;
  }
  if (h->profiling) DG_CUDA(cudaEventRecord(h->kev[0], s));
  int st;
  if (h->accumulation == DG_ACCUM_FP32) {
    if (h->cols) {
      k_x_to_f32<<<grid_for(h->cols, 256, 2), 256, 0, s>>>(d_x, h->d_xf, h->cols);
      h->post(s, "x_to_f32", 0, 0);
    }
    st = dispatch_mat(h, [&](const auto& mat) { return launch_fp32(h, mat, h->d_xf, d_y, s); });
  } else {
    st = dispatch_mat(h, [&](const auto& mat) { return launch_exact(h, mat, d_x, d_y, s); });
  }
  h->n_kernels = h->n_launch;
  return st;
}

int finish_create(Handle* h, const std::vector<uint64_t>& lens) {
  // row ids in the plan (bins, segments, dense list) are u32: one handle holds < 2^32 rows
  // (a larger matrix is row-sharded over several handles, dg_options.row_begin / row_end)
  if (h->rows > 0xFFFFFFFFull) return DG_ERR_UNSUPPORTED_FEATURE;
  DG_CUDA(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device));
  const char* plan = std::getenv("DG_PLAN");  // "warp": v0 warp-per-row plan (A/B only)
  h->use_tiles = h->lane_width == 32 && !(plan && std::strcmp(plan, "warp") == 0);
  h->acc_bytes = h->accumulation == DG_ACCUM_FP32 ? 4 : 8;
  // ~8 tiles per SM at least (small matrices), at most 768K nonzeros per tile (C2 sweep: 512K-768K
  // flat, 1M +0.6%, 1.5M +1%, with the rows wider than a window in k_dense; C4 / C5 flat)
  h->tile_nnz = std::max<uint64_t>(16 * 1024, std::min<uint64_t>(768 * 1024,
                                                                  h->nnz / (h->min_tiles_per_sm * h->sm_count)));
  if (const char* tn = std::getenv("DG_TILE_NNZ")) h->tile_nnz = std::strtoull(tn, nullptr, 10);
  if (const char* tp = std::getenv("DG_TILES_PER_SM"))
    h->min_tiles_per_sm = std::max<uint64_t>(1, std::strtoull(tp, nullptr, 10));
  if (const char* tc = std::getenv("DG_TILE_CFG")) h->tile_cfg = std::atoi(tc);
  // small launches (under ~4 full tiles per SM: the C3 shards) end with less guided shrinking
  // (C2's 1/8 shard: 0.2522 -> 0.2501 ms; full C2 would lose, 1.187 -> 1.204 ms of tiles)
  if (h->nnz < 4ull * 768 * 1024 * h->sm_count) {
    h->tile_guide = 1;
    h->tile_guide_min = 32 * 1024;
  }
  if (const char* tg = std::getenv("DG_TILE_GUIDE")) h->tile_guide = std::strtoull(tg, nullptr, 10);
  if (const char* tg = std::getenv("DG_TILE_GUIDE_MIN"))
    h->tile_guide_min = std::strtoull(tg, nullptr, 10);
  if (const char* dk = std::getenv("DG_DENSE")) h->dense_mode = std::atoi(dk) != 0;
  if (const char* dm = std::getenv("DG_DENSE_MIN_LEN")) h->dense_min_len = std::strtoull(dm, nullptr, 10);
  if (const char* dc = std::getenv("DG_DENSE_CFG")) h->dense_cfg = std::atoi(dc);
  if (const char* pd = std::getenv("DG_PDL")) h->pdl = std::atoi(pd) != 0;
  if (const char* gm = std::getenv("DG_GLOBAL_MIN_LEN"))
    h->global_min_len = std::strtoull(gm, nullptr, 10);
  h->window_cols = window_bytes_for(h->tile_cfg, h->packed) / h->acc_bytes;
  // replicated x windows for the sparse segments: exact family, Packed16 stream (DG_REPLICAS=0:
  // column mode only, for A/B)
  h->slot_mode = h->use_tiles && h->value_precision == DG_HALF && h->accumulation == DG_ACCUM_EXACT;
  if (const char* rp = std::getenv("DG_REPLICAS")) h->slot_mode = h->slot_mode && std::atoi(rp) != 0;
  // the slice stream: binary16 values (Packed16 or U32 SoA uploads), k_dense available
  h->slices_wanted = h->use_tiles && h->value_precision == DG_HALF && h->dense_mode != 0;
  if (const char* sl = std::getenv("DG_SLICES")) h->slices_wanted = h->slices_wanted && std::atoi(sl) != 0;
  h->slot_mode = h->slot_mode && (h->packed || h->slices_wanted);
  // x staging before the plan: the slot assignment is launched from plan_tiles
  {
    const uint64_t n = std::max<uint64_t>(h->cols, 1) + 2 * Handle::kXPad + 32;
    DG_CUDA(cudaMalloc(&h->d_x_raw, n * sizeof(double)));
    DG_CUDA(cudaMemset(h->d_x_raw, 0, n * sizeof(double)));
    DG_CUDA(cudaMalloc(&h->d_x1_raw, n * sizeof(double)));
    DG_CUDA(cudaMemset(h->d_x1_raw, 0, n * sizeof(double)));
    h->d_x = h->d_x_raw + Handle::kXPad;
    h->d_x1 = h->d_x1_raw + Handle::kXPad + 1;
  }
  DG_TRY(build_plan(h, lens));
  if (h->use_tiles) DG_TRY(plan_tiles(h, lens));
  DG_TRY(build_slices(h));
  if (std::getenv("DG_TRACE") && h->use_tiles && h->wave_tiles[0]) {
    h->trace_len = 4ull * h->sm_count + 3ull * h->wave_tiles[0];
    DG_CUDA(cudaMalloc(&h->d_trace, h->trace_len * sizeof(unsigned long long)));
  }
  DG_CUDA(cudaMalloc(&h->d_y, std::max<uint64_t>(h->rows, 1) * sizeof(double)));
  if (h->accumulation == DG_ACCUM_FP32) {
    DG_CUDA(cudaMalloc(&h->d_xf, (std::max<uint64_t>(h->cols, 1) + 8) * sizeof(float)));
    DG_CUDA(cudaMemset(h->d_xf, 0, (std::max<uint64_t>(h->cols, 1) + 8) * sizeof(float)));
  }
  for (auto& e : h->ev) DG_CUDA(cudaEventCreate(&e));
  for (auto& e : h->kev) DG_CUDA(cudaEventCreate(&e));
  DG_CUDA(cudaEventCreateWithFlags(&h->ev_tiles_start, cudaEventDisableTiming));
  DG_CUDA(cudaEventCreateWithFlags(&h->ev_d2h_done, cudaEventDisableTiming));
  DG_CUDA(cudaStreamCreateWithFlags(&h->d2h_stream, cudaStreamNonBlocking));
  DG_CUDA(cudaStreamCreateWithFlags(&h->d2h_stream2, cudaStreamNonBlocking));
  DG_CUDA(cudaEventCreateWithFlags(&h->ev_d2h_done2, cudaEventDisableTiming));
  // create-time work (memsets, plan uploads, setup kernels) ran on the legacy stream, which the
  // handle's non-blocking dose streams do not wait on: finish it before the handle is returned
  DG_CUDA(cudaDeviceSynchronize());
  return DG_OK;
}

// cuStreamWaitValue32 through the runtime's driver entry-point query (no libcuda link needed).
bool set_block_sinks(Handle* h, const double* const* dst, const int* dev, uint32_t n) {
  h->sink_ptr.assign(const_cast<double* const*>(dst), const_cast<double* const*>(dst) + n);
  h->sink_dev.assign(dev, dev + n);
  h->sink_remote = false;  // a sink on another device (or a UVA / IPC mapping: assumed remote)
  for (uint32_t i = 0; i < n; ++i) h->sink_remote |= dev[i] < 0 || dev[i] != h->device;
  return true;
}

// rows [r0, r1) of this shard's d (src: device) into every sink: peer copies between devices of
// this process (dg_multi), plain UVA copies for CUDA-IPC mappings (sink_dev < 0)
int copy_to_sinks(Handle* h, const double* src, uint64_t r0, uint64_t r1, cudaStream_t c) {
  if (h->host_sink && r1 > r0)  // dg_multi with host d: this shard's slice of the caller's d
    DG_CUDA(cudaMemcpyAsync(h->host_sink + r0, src + r0, (r1 - r0) * sizeof(double),
                            cudaMemcpyDeviceToHost, c));
  for (size_t i = 0; i < h->sink_ptr.size() && r1 > r0; ++i) {
    if (h->sink_dev[i] >= 0)
      DG_CUDA(cudaMemcpyPeerAsync(h->sink_ptr[i] + r0, h->sink_dev[i], src + r0, h->device,
                                  (r1 - r0) * sizeof(double), c));
    else
      DG_CUDA(cudaMemcpyAsync(h->sink_ptr[i] + r0, src + r0, (r1 - r0) * sizeof(double),
                              cudaMemcpyDefault, c));
  }
  return DG_OK;
}

WaitValueFn wait_value_fn() {
  static const WaitValueFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<WaitValueFn>(nullptr);
    }
    return reinterpret_cast<WaitValueFn>(p);
  }();
  return fn;
}

}  // namespace dg

using dg::Handle;

extern "C" {

int dg_create(const dg_csr_view* v, const dg_options* opts_in, dg_handle** out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!v || !out) return DG_ERR_INVALID_CONFIG;
  *out = nullptr;
  dg_options opts;
  dg_default_options(&opts);
  if (opts_in) opts = *opts_in;
  DG_TRY(dg::check_options(&opts));
  if (v->value_precision > DG_DOUBLE) return DG_ERR_INVALID_CONFIG;
  if (v->index_bytes != 2 && v->index_bytes != 4) return DG_ERR_INVALID_CONFIG;
  if (v->col_storage_bytes != 2 && v->col_storage_bytes != 4) return DG_ERR_INVALID_CONFIG;
  if (v->col_storage_bytes == 2 && v->index_bytes == 4) return DG_ERR_INVALID_CONFIG;
  if (v->index_bytes == 2 && v->cols >= 65536) return DG_ERR_VALIDATION_FAILURE;  // sparse.cpp:232-233
  if (v->cols > 0xFFFFFFFFull) return DG_ERR_INDEX_OVERFLOW;
  const uint64_t r0 = opts.row_begin, r1 = opts.row_end ? opts.row_end : v->rows;
  if (r0 > r1 || r1 > v->rows) return DG_ERR_INVALID_CONFIG;
  if (!v->row_ptr || (v->nnz && (!v->col_indices || !v->values))) return DG_ERR_VALIDATION_FAILURE;
  int dev = 0;
  DG_TRY(dg::select_device(opts.device, &dev));

  // Row pointers of the shard (host copy drives validation + the plan).
  const uint64_t n_rows = r1 - r0;
  std::vector<uint64_t> rp(n_rows + 1);
  if (v->on_device)
    DG_CUDA(cudaMemcpy(rp.data(), v->row_ptr + r0, (n_rows + 1) * 8, cudaMemcpyDeviceToHost));
  else
    std::memcpy(rp.data(), v->row_ptr + r0, (n_rows + 1) * 8);
  uint64_t first = 0, last = 0;
  if (v->on_device) {
    DG_CUDA(cudaMemcpy(&first, v->row_ptr, 8, cudaMemcpyDeviceToHost));
    DG_CUDA(cudaMemcpy(&last, v->row_ptr + v->rows, 8, cudaMemcpyDeviceToHost));
  } else {
    first = v->row_ptr[0];
    last = v->row_ptr[v->rows];
  }
  if (first != 0 || last != v->nnz) return DG_ERR_VALIDATION_FAILURE;  // sparse.cpp:221-229
  std::vector<uint64_t> lens(n_rows);
  for (uint64_t r = 0; r < n_rows; ++r) {
    if (rp[r + 1] < rp[r]) return DG_ERR_VALIDATION_FAILURE;  // sparse.cpp:222-227
    lens[r] = rp[r + 1] - rp[r];
  }
  const uint64_t base = rp[0], shard_nnz = rp[n_rows] - rp[0];

  Handle* h = new (std::nothrow) Handle();
  if (!h) return DG_ERR_OUT_OF_MEMORY;
  h->device = dev;
  h->rows = n_rows;
  h->cols = v->cols;
  h->nnz = shard_nnz;
  h->row_begin = r0;
  h->row_end = r1;
  h->value_precision = v->value_precision;
  h->value_bytes = v->value_precision == DG_HALF ? 2 : v->value_precision == DG_SINGLE ? 4 : 8;
  h->index_bytes = v->index_bytes;
  h->lane_width = opts.lane_width;
  h->accumulation = opts.accumulation;

  auto fail = [&](int s) { dg_destroy(reinterpret_cast<dg_handle*>(h)); return s; };
  auto cu = [&](cudaError_t e) { return e == cudaSuccess ? DG_OK : DG_ERR_CUDA_BASE + (int)e; };
  int st;
  if ((st = cu(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking)))) return fail(st);
  if ((st = cu(cudaMalloc(&h->d_bad, sizeof(unsigned))))) return fail(st);
  if ((st = cu(cudaMemset(h->d_bad, 0, sizeof(unsigned))))) return fail(st);

  // --- one-time upload of the native encoding (no expansion: values stay binary16 bits) ------
  if ((st = cu(cudaMalloc(&h->d_row_ptr, (n_rows + 1) * 8)))) return fail(st);
  if ((st = cu(cudaMemcpy(h->d_row_ptr, rp.data(), (n_rows + 1) * 8, cudaMemcpyHostToDevice))))
    return fail(st);
  if (base) dg::k_rebase<<<dg::grid_for(n_rows + 1, 256), 256>>>(h->d_row_ptr, n_rows + 1, base);
  const uint64_t nz = std::max<uint64_t>(shard_nnz, 1);
  if ((st = cu(cudaMalloc(&h->d_val, nz * h->value_bytes)))) return fail(st);
  if ((st = cu(cudaMalloc(&h->d_col, nz * h->index_bytes)))) return fail(st);
  const cudaMemcpyKind kind = v->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (shard_nnz) {
    const char* vsrc = static_cast<const char*>(v->values) + base * h->value_bytes;
    if ((st = cu(cudaMemcpy(h->d_val, vsrc, shard_nnz * h->value_bytes, kind)))) return fail(st);
    const char* csrc = static_cast<const char*>(v->col_indices) + base * v->col_storage_bytes;
    if (v->col_storage_bytes == h->index_bytes) {
      if ((st = cu(cudaMemcpy(h->d_col, csrc, shard_nnz * h->index_bytes, kind)))) return fail(st);
    } else {  // ddm keeps u32 in memory even when tagged U16 (sparse.hpp:104): narrow on device
      const uint64_t chunk = 64ull << 20;
      uint32_t* stage = nullptr;
      if ((st = cu(cudaMalloc(&stage, std::min(chunk, shard_nnz) * 4)))) return fail(st);
      for (uint64_t off = 0; off < shard_nnz && !st; off += chunk) {
        const uint64_t n = std::min(chunk, shard_nnz - off);
        st = cu(cudaMemcpy(stage, csrc + off * 4, n * 4, kind));
        if (!st)
          dg::k_narrow_u32_u16<<<dg::grid_for(n, 256), 256>>>(
              stage, static_cast<uint16_t*>(h->d_col) + off, n, h->cols, h->d_bad);
      }
      cudaDeviceSynchronize();
      cudaFree(stage);
      if (st) return fail(st);
    }
  }
  // --- ddm::validate's per-entry invariants on the device copy --------------------------------
  st = dg::dispatch_mat(h, [&](const auto& mat) {
    dg::k_validate<<<dg::grid_for(32 * n_rows, 256), 256>>>(mat, h->d_row_ptr, n_rows, h->cols,
                                                            h->d_bad);
    return cu(cudaGetLastError());
  });
  if (st) return fail(st);
  unsigned bad = 0;
  if ((st = cu(cudaMemcpy(&bad, h->d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost)))) return fail(st);
  if (bad) return fail(DG_ERR_VALIDATION_FAILURE);
  // --- (binary16, u16): one packed 32-bit stream, same 4 bytes per nonzero --------------------
  const char* nopack = std::getenv("DG_NO_PACK");
  if (h->value_precision == DG_HALF && h->index_bytes == 2 && !(nopack && *nopack == '1')) {
    // +16 B: the 1-D TMA of the stream rounds a batch up to whole 16-byte granules
    if ((st = cu(cudaMalloc(&h->d_packed, nz * 4 + 16)))) return fail(st);
    dg::k_pack16<<<dg::grid_for(shard_nnz, 256), 256>>>(static_cast<const uint16_t*>(h->d_col),
                                                        static_cast<const uint16_t*>(h->d_val),
                                                        h->d_packed, shard_nnz);
    if ((st = cu(cudaDeviceSynchronize()))) return fail(st);
    cudaFree(h->d_col);
    cudaFree(h->d_val);
    h->d_col = h->d_val = nullptr;
    h->packed = true;
  }
  h->matrix_bytes = (n_rows + 1) * 8 + shard_nnz * (h->value_bytes + h->index_bytes);
  if ((st = dg::finish_create(h, lens))) return fail(st);
  *out = reinterpret_cast<dg_handle*>(h);
  return DG_OK;
}

int dg_destroy(dg_handle* hh) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h) return DG_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  cudaFree(h->d_row_ptr);
  cudaFree(h->d_row_ptr_orig);
  cudaFree(h->d_slices);
  cudaFree(h->d_ranges);
  cudaFree(h->d_sseg);
  cudaFree(h->d_trace);
  cudaFree(h->d_dense_rows);
  cudaFree(h->d_dense_counter);
  cudaFree(h->d_dslices);
  cudaFree(h->d_dranges);
  cudaFree(h->d_dsseg);
  cudaFree(h->d_vrows);
  cudaFree(h->d_vstream);
  cudaFree(h->d_value_counter);
  cudaFree(h->d_col);
  cudaFree(h->d_val);
  cudaFree(h->d_packed);
  cudaFree(h->d_x_raw);
  cudaFree(h->d_x1_raw);
  cudaFree(h->d_xf);
  cudaFree(h->d_y);
  cudaFree(h->d_bad);
  for (auto* b : h->d_bin) cudaFree(b);
  for (uint32_t w = 0; w < Handle::kMaxWaves; ++w) {
    cudaFree(h->d_tiles[w]);
    cudaFree(h->d_segs[w]);
  }
  cudaFree(h->d_state);
  cudaFree(h->d_counters);
  cudaFree(h->d_blk_left);
  cudaFree(h->d_blk_left_init);
  cudaFree(h->d_blk_flag);
  if (h->d2h_stream) {
    cudaStreamSynchronize(h->d2h_stream);
    cudaStreamDestroy(h->d2h_stream);
  }
  if (h->d2h_stream2) {
    cudaStreamSynchronize(h->d2h_stream2);
    cudaStreamDestroy(h->d2h_stream2);
  }
  if (h->ev_d2h_done2) cudaEventDestroy(h->ev_d2h_done2);
  if (h->ev_tiles_start) cudaEventDestroy(h->ev_tiles_start);

  if (h->ev_d2h_done) cudaEventDestroy(h->ev_d2h_done);
  for (auto e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto e : h->kev)
    if (e) cudaEventDestroy(e);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return DG_OK;
}

int dg_dose(dg_handle* hh, const double* x, uint64_t x_len, double* y, uint32_t flags,
            void* stream) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || (!x && h->cols) || (!y && h->rows)) return DG_ERR_INVALID_CONFIG;
  if (x_len != h->cols) return DG_ERR_DIMENSION_MISMATCH;  // spmv.cpp:34-38
  DG_CUDA(cudaSetDevice(h->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : h->stream;
  const bool x_dev = flags & DG_X_ON_DEVICE, y_dev = flags & DG_Y_ON_DEVICE;
  // The exact tile kernels TMA the x window straight from the caller's device x when it is
  // 16-byte aligned with a 16-byte multiple length and no window is replicated; otherwise x is
  // staged in the padded buffers (slot mode also needs the one-element-shifted copy, XSource).
  if (h->slot_tiles) DG_TRY(dg::recode_slots(h, false));
  // (dense slices read x[cols] for their neutral words: a staged +0.0 -- never the caller's x)
  const bool x_direct = x_dev && !h->slot_tiles && !h->dense_slices && !h->n_value_rows &&
                        (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (h->cols % 2 == 0);
  const double* d_x = x_direct ? x : h->d_x;
  double* d_y = y_dev ? y : h->d_y;
  DG_CUDA(cudaEventRecord(h->ev[0], s));
  if (!x_direct && h->cols) {
    if (!x_dev)
      DG_CUDA(cudaMemcpyAsync(h->d_x, x, h->cols * sizeof(double), cudaMemcpyHostToDevice, s));
    if (x_dev || h->slot_tiles) {
      dg::k_stage_x<<<dg::grid_for(h->cols, 256, 2), 256, 0, s>>>(
          x_dev ? x : h->d_x, h->d_x, h->slot_tiles ? h->d_x1 : nullptr, h->cols);
      DG_CUDA(cudaGetLastError());
    }
  }
  DG_CUDA(cudaEventRecord(h->ev[1], s));
  h->profiling = (flags & DG_PROFILE) != 0;
  // Host d: download row block k as soon as the tile kernel publishes its completion, while it
  // still works on later blocks (one wave only: with carried partials the last wave owns rows).
  const char* no_ovl = std::getenv("DG_NO_OVERLAP");
  // (single-wave plans only: with split rows every block's last tiles are in the last waves, so
  //  the blocks complete at the very end -- C4 end to end 7.24 ms overlapped vs 7.16 plain; r02
  //  with the slice kernel: 4.82 vs 4.59 ms, and 4.78-4.83 with wave lags 1 / 2 / 4).
  // (measured, rejected: with pinned host d, running the contiguous rows LAST -- after the block
  //  downloads, storing their rows into the pinned d zero-copy -- C2 end to end 2.10 vs 2.10 ms:
  //  the 64 MB download runs at ~45 GB/s beside the kernels either way, 1.42 ms.  Measured again
  //  in its concurrent form -- the contiguous rows right after the tile kernel, each row stored
  //  into the mapped host d once its block's download is flagged done (cuStreamWriteValue32):
  //  e2e 1.922-1.928 vs 1.930-1.932 ms values-first, 32 / 64 blocks 2.00 / 2.10; the PCIe
  //  download beside the HBM-bound kernels (34-44 GB/s; 53.7 GB/s on an idle GPU,
  //  scripts/micro/pcie_d2h.cu) bounds the end-to-end step either way)
  const bool block_plan = h->rows && h->use_tiles && h->n_waves == 1 && h->n_blocks > 1 &&
                          dg::wait_value_fn() && !(no_ovl && *no_ovl == '1');
  const bool overlap = !y_dev && block_plan;
  // dg_multi PEER gather (device d): each block copied to the other devices' full d as it completes
  // (only toward other devices: copies into this device's own memory would compete with the
  //  kernels for the same HBM -- dg_multi on a virtual device list {0,0,0,0}: 2.12 ms overlapped
  //  vs 1.98 after the kernels; DG_SINK_OVERLAP=1 forces it for tests)
  const char* fs = std::getenv("DG_SINK_OVERLAP");
  const bool force_sink = fs && *fs == '1';
  const bool sinks = !h->sink_ptr.empty() || h->host_sink;
  h->sink_overlap = y_dev && block_plan && sinks && !h->profiling &&
                    (h->sink_remote || h->host_sink || force_sink);
  h->signal_blocks = overlap || h->sink_overlap;
  if (h->signal_blocks) ++h->epoch;
  DG_TRY(dg::run_kernels(h, d_x, d_y, s));
  DG_CUDA(cudaEventRecord(h->ev[2], s));
  // Row blocks out of the device d `src` on two copy streams (blocks alternate: two copy engines;
  // DG_D2H_STREAMS=1 for one): into the host d (host_dst, may be null) and every sink.  Per block,
  // each copy waits for the tile kernel's completion flag of that block (per_block), or the whole
  // d follows the kernels.  The dose's stream waits for both copy streams at the end.
  auto copy_out = [&](const double* src, double* host_dst, bool per_block) -> int {
    static const int n_cs = [] { const char* v = std::getenv("DG_D2H_STREAMS"); return v && *v == '1' ? 1 : 2; }();
    cudaStream_t cs[2] = {h->d2h_stream, n_cs > 1 ? h->d2h_stream2 : h->d2h_stream};
    if (!per_block) DG_CUDA(cudaEventRecord(h->ev_tiles_start, s));  // (after the kernels)
    DG_CUDA(cudaStreamWaitEvent(cs[0], h->ev_tiles_start, 0));
    if (cs[1] != cs[0]) DG_CUDA(cudaStreamWaitEvent(cs[1], h->ev_tiles_start, 0));
    const uint32_t nb = per_block ? h->n_blocks : 1;
    for (uint32_t k = 0; k < nb; ++k) {
      const uint64_t r0 = per_block ? h->blk_row0[k] : 0;
      const uint64_t r1 = per_block ? h->blk_row0[k + 1] : h->rows;
      if (r1 == r0) continue;
      cudaStream_t c = cs[k & 1];
      if (per_block && h->blk_tiles[k]) {
        const CUresult cr = dg::wait_value_fn()(
            reinterpret_cast<CUstream>(c),
            reinterpret_cast<CUdeviceptr>(h->d_blk_flag + k), h->epoch, CU_STREAM_WAIT_VALUE_GEQ);
        if (cr != CUDA_SUCCESS) return DG_ERR_CUDA_BASE + static_cast<int>(cudaErrorUnknown);
      }
      if (host_dst)
        DG_CUDA(cudaMemcpyAsync(host_dst + r0, src + r0, (r1 - r0) * sizeof(double),
                                cudaMemcpyDeviceToHost, c));
      DG_TRY(dg::copy_to_sinks(h, src, r0, r1, c));
    }
    DG_CUDA(cudaEventRecord(h->ev_d2h_done, cs[0]));
    DG_CUDA(cudaStreamWaitEvent(s, h->ev_d2h_done, 0));
    if (cs[1] != cs[0]) {
      DG_CUDA(cudaEventRecord(h->ev_d2h_done2, cs[1]));
      DG_CUDA(cudaStreamWaitEvent(s, h->ev_d2h_done2, 0));
    }
    return DG_OK;
  };
  if (overlap) {  // host d, downloaded block by block while the tile kernel works on later blocks
    DG_TRY(copy_out(h->d_y, y, true));
  } else if (!y_dev && h->rows) {
    DG_CUDA(cudaMemcpyAsync(y, h->d_y, h->rows * sizeof(double), cudaMemcpyDeviceToHost, s));
    DG_TRY(dg::copy_to_sinks(h, h->d_y, 0, h->rows, s));
  } else if (y_dev && h->rows && sinks) {
    // device d with sinks (dg_multi PEER gather / host d, block targets): block k as soon as its
    // last tile is done (sink_overlap), or all of d after the kernels
    DG_TRY(copy_out(y, nullptr, h->sink_overlap));
  }
  DG_CUDA(cudaEventRecord(h->ev[3], s));
  h->timing_valid = false;
  if (!(flags & DG_NO_SYNC) || !x_dev || !y_dev) {
    DG_CUDA(cudaStreamSynchronize(s));
    h->collect_timing();
  }
  return DG_OK;
}

int dg_get_info(const dg_handle* hh, dg_info* info) {
  const Handle* h = reinterpret_cast<const Handle*>(hh);
  if (!h || !info) return DG_ERR_INVALID_CONFIG;
  info->rows = h->rows;
  info->cols = h->cols;
  info->nnz = h->nnz;
  info->row_begin = h->row_begin;
  info->row_end = h->row_end;
  info->value_bytes = h->value_bytes;
  info->index_bytes = h->index_bytes;
  info->lane_width = h->lane_width;
  info->accumulation = h->accumulation;
  info->device_bytes = h->matrix_bytes + h->plan_bytes;
  info->model_bytes = dg_traffic_bytes(h->rows, h->cols, h->nnz, h->value_bytes, h->index_bytes);
  info->nonempty_rows = h->nonempty_rows;
  info->n_kernels = h->n_kernels ? h->n_kernels : h->expected_kernels();
  info->device = h->device;
  info->read_ns = h->read_ns;
  return DG_OK;
}

int dg_last_timing(const dg_handle* hh, dg_timing* t) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  Handle* h = const_cast<Handle*>(reinterpret_cast<const Handle*>(hh));
  if (!h || !t) return DG_ERR_INVALID_CONFIG;
  if (!h->timing_valid) {
    DG_CUDA(cudaSetDevice(h->device));
    DG_CUDA(cudaEventSynchronize(h->ev[3]));
    h->collect_timing();
  }
  *t = h->last;
  return DG_OK;
}

int dg_kernel_times(const dg_handle* hh, dg_kernel_time* out, uint32_t cap, uint32_t* n_out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  Handle* h = const_cast<Handle*>(reinterpret_cast<const Handle*>(hh));
  if (!h || !n_out) return DG_ERR_INVALID_CONFIG;
  *n_out = 0;
  if (!h->profiling) return DG_OK;
  DG_CUDA(cudaSetDevice(h->device));
  const uint32_t n = std::min<uint32_t>(h->n_launch, Handle::kMaxLaunches);
  if (n) DG_CUDA(cudaEventSynchronize(h->kev[n]));
  for (uint32_t i = 0; i < n && i < cap; ++i) {
    float ms = 0;
    DG_CUDA(cudaEventElapsedTime(&ms, h->kev[i], h->kev[i + 1]));
    const auto& l = h->launches[i];
    std::snprintf(out[i].name, sizeof(out[i].name), "%s", l.name);
    out[i].ms = ms;
    out[i].rows = l.rows;
    out[i].nnz = l.nnz;
    out[i].bytes = l.rows ? dg_traffic_bytes(l.rows, h->cols, l.nnz, h->value_bytes, h->index_bytes)
                          : 12ull * h->cols;
    *n_out = i + 1;
  }
  return DG_OK;
}

int dg_debug_trace(const dg_handle* hh, uint64_t* out, uint64_t cap, uint64_t* n_out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  const Handle* h = reinterpret_cast<const Handle*>(hh);
  if (!h || !n_out) return DG_ERR_INVALID_CONFIG;
  *n_out = 0;
  if (!h->d_trace) return DG_OK;
  DG_CUDA(cudaSetDevice(h->device));
  const uint64_t n = std::min<uint64_t>(cap, h->trace_len);
  if (n) DG_CUDA(cudaMemcpy(out, h->d_trace, n * 8, cudaMemcpyDeviceToHost));
  *n_out = n;
  return DG_OK;
}

int dg_copy_row_ptr(const dg_handle* hh, uint64_t r0, uint64_t r1, uint64_t* rp_out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  const Handle* h = reinterpret_cast<const Handle*>(hh);
  if (!h || !rp_out || r0 > r1 || r1 > h->rows) return DG_ERR_INVALID_CONFIG;
  DG_CUDA(cudaSetDevice(h->device));
  DG_CUDA(cudaMemcpy(rp_out, dg::orig_row_ptr(h) + r0, (r1 - r0 + 1) * 8, cudaMemcpyDeviceToHost));
  return DG_OK;
}

int dg_copy_rows(const dg_handle* hh, uint64_t r0, uint64_t r1, uint64_t* rp_out,
                 uint32_t* col_out, void* val_out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  const Handle* h = reinterpret_cast<const Handle*>(hh);
  if (!h || r0 > r1 || r1 > h->rows) return DG_ERR_INVALID_CONFIG;
  DG_CUDA(cudaSetDevice(h->device));
  DG_CUDA(cudaMemcpy(rp_out, dg::orig_row_ptr(h) + r0, (r1 - r0 + 1) * 8, cudaMemcpyDeviceToHost));
  const uint64_t b = rp_out[0], n = rp_out[r1 - r0] - b;
  for (uint64_t i = 0; i <= r1 - r0; ++i) rp_out[i] -= b;
  if (!n) return DG_OK;
  if (h->slices) {  // decode the slice and rest streams back to the row-ordered encoding
    uint32_t* d_col = nullptr;
    uint16_t* d_val = nullptr;
    DG_CUDA(cudaMalloc(&d_col, n * 4));
    cudaError_t e = cudaMalloc(&d_val, n * 2);
    int st = e == cudaSuccess ? dg::decode_rows(h, r0, r1, d_col, d_val) : DG_ERR_CUDA_BASE + (int)e;
    if (st == DG_OK) {
      e = cudaMemcpy(col_out, d_col, n * 4, cudaMemcpyDeviceToHost);
      if (e == cudaSuccess) e = cudaMemcpy(val_out, d_val, n * 2, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) st = DG_ERR_CUDA_BASE + (int)e;
    }
    cudaFree(d_col);
    cudaFree(d_val);
    return st;
  }
  // slot-mode positions back to columns for the copy (the next dose re-encodes them)
  DG_TRY(dg::recode_slots(const_cast<Handle*>(h), true));
  uint32_t* d_col = nullptr;
  void* d_val = nullptr;
  DG_CUDA(cudaMalloc(&d_col, n * 4));
  cudaError_t e = cudaMalloc(&d_val, n * h->value_bytes);
  if (e == cudaSuccess) {
    dg::dispatch_mat(h, [&](const auto& mat) {
      using M = std::decay_t<decltype(mat)>;
      dg::k_unpack<M><<<dg::grid_for(n, 256), 256>>>(mat, b, n, d_col,
                                                     static_cast<typename M::Val*>(d_val));
      return 0;
    });
    e = cudaMemcpy(col_out, d_col, n * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(val_out, d_val, n * h->value_bytes, cudaMemcpyDeviceToHost);
  }
  cudaFree(d_col);
  cudaFree(d_val);
  DG_CUDA(e);
  return DG_OK;
}

int dg_checksum_bits(const double* v, uint64_t n, int on_device, uint64_t* out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  std::vector<double> host;
  const double* p = v;
  if (on_device) {
    host.resize(n);
    if (n) DG_CUDA(cudaMemcpy(host.data(), v, n * 8, cudaMemcpyDeviceToHost));
    p = host.data();
  }
  uint64_t hsh = 14695981039346656037ull;  // checksum.hpp:25-35, LSB first
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t u;
    std::memcpy(&u, p + i, 8);
    for (int k = 0; k < 8; ++k) {
      hsh ^= static_cast<uint8_t>(u >> (8 * k));
      hsh *= 1099511628211ull;
    }
  }
  *out = hsh;
  return DG_OK;
}

}  // extern "C"
