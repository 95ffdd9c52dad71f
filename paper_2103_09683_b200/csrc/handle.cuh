// handle.cuh -- the device-resident state behind a dg_handle.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "dosegpu.h"

namespace dg {

constexpr int kNumBins = 8;
constexpr int kBinLong = 6;     // L = 32: rows with len > 32, warp per row
constexpr int kBinGeneral = 7;  // L != 32: every non-empty row
// Shared memory per tile CTA for the x window (2 CTAs per SM): 13,824 doubles / 27,648 floats.
constexpr uint32_t kTileSmemBytes = 108 * 1024;

struct Handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t rows = 0, cols = 0, nnz = 0, row_begin = 0, row_end = 0;
  uint32_t value_precision = DG_HALF, value_bytes = 2, index_bytes = 2;
  uint32_t lane_width = 32, accumulation = DG_ACCUM_EXACT;

  // native encoding, shard-local (row_ptr rebased to 0)
  uint64_t* d_row_ptr = nullptr;
  void* d_col = nullptr;  // u16 or u32
  void* d_val = nullptr;  // binary16 bits / f32 / f64
  uint64_t matrix_bytes = 0;

  // row plan: short-row bins ...
  uint32_t* d_bin[kNumBins] = {};
  uint32_t bin_count[kNumBins] = {};
  uint64_t plan_bytes = 0, nonempty_rows = 0;
  // ... and column-windowed tiles of row segments, per wave (plan.cu, spmv_tiles.cuh)
  static constexpr uint32_t kMaxWaves = 32;
  static constexpr int kTileWarps = 16;
  uint32_t acc_bytes = 8;                 // shared-memory x element: 8 exact, 4 fp32
  uint32_t window_cols = 0;               // x window capacity per tile (columns)
  uint64_t tile_nnz = 256 * 1024;         // target nonzeros per tile
  uint32_t n_waves = 0;
  uint64_t n_split_rows = 0;
  uint32_t wave_tiles[kMaxWaves] = {};
  uint64_t wave_nnz[kMaxWaves] = {}, wave_rows[kMaxWaves] = {};
  void* d_tiles[kMaxWaves] = {};
  void* d_segs[kMaxWaves] = {};
  void* d_state = nullptr;
  uint32_t* d_counters = nullptr;
  int sm_count = 148;
  bool use_tiles = false;

  // staging for host x / y and the fp32 family
  double* d_x = nullptr;
  double* d_y = nullptr;
  float* d_xf = nullptr;
  unsigned* d_bad = nullptr;

  cudaEvent_t ev[4] = {};
  dg_timing last = {};
  bool timing_valid = false;
  uint32_t n_kernels = 0;

  // per-launch profiling (DG_PROFILE)
  static constexpr int kMaxLaunches = 16;
  uint64_t bin_nnz[kNumBins] = {};
  cudaEvent_t kev[kMaxLaunches + 1] = {};
  struct Launch {
    const char* name;
    uint64_t rows, nnz;
  } launches[kMaxLaunches] = {};
  bool profiling = false;
  uint32_t n_launch = 0;

  // call right after each kernel launch of a dose
  void post(cudaStream_t s, const char* name, uint64_t rows_, uint64_t nnz_) {
    if (n_launch < kMaxLaunches) {
      launches[n_launch] = {name, rows_, nnz_};
      if (profiling) cudaEventRecord(kev[n_launch + 1], s);
    }
    ++n_launch;
  }

  uint32_t expected_kernels() const {
    uint32_t n = accumulation == DG_ACCUM_FP32 ? 1 : 0;
    if (lane_width == 32) {
      for (int b = 0; b < kNumBins; ++b) n += bin_count[b] ? 1 : 0;
      for (uint32_t w = 0; w < n_waves; ++w) n += wave_tiles[w] ? 1 : 0;
    } else {
      n += bin_count[kBinGeneral] ? 1 : 0;
    }
    return n;
  }

  void collect_timing() {
    float a = 0, b = 0, c = 0, t = 0;
    cudaEventElapsedTime(&a, ev[0], ev[1]);
    cudaEventElapsedTime(&b, ev[1], ev[2]);
    cudaEventElapsedTime(&c, ev[2], ev[3]);
    cudaEventElapsedTime(&t, ev[0], ev[3]);
    last = {a, b, c, t};
    timing_valid = true;
  }
};

// shared by dosegpu.cu and generator.cu
int select_device(int32_t want, int* dev_out);
int check_options(const dg_options* o);
int finish_create(Handle* h, const std::vector<uint64_t>& lens);
int plan_tiles(Handle* h, const std::vector<uint64_t>& lens);
int grid_for(uint64_t work_items, int threads, int max_blocks_per_sm = 8);

}  // namespace dg
