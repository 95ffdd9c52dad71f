// handle.cuh -- the device-resident state behind a dg_handle.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"
#include "dosegpu.h"

namespace dg {

struct Tile;
struct Segment;

constexpr int kNumBins = 8;
constexpr int kBinLong = 6;     // v0 plan (DG_PLAN=warp): rows with len > 32, warp per row
constexpr int kBinGeneral = 7;  // L != 32: every non-empty row
// Shared memory of the tile CTA (one per SM): two x-window buffers of 110,592 bytes each,
// i.e. 13,824 doubles (exact) or 27,648 floats (fp32) per window.
constexpr uint32_t kWindowBytes = 108 * 1024;

struct Handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t rows = 0, cols = 0, nnz = 0, row_begin = 0, row_end = 0;
  uint32_t value_precision = DG_HALF, value_bytes = 2, index_bytes = 2;
  uint32_t lane_width = 32, accumulation = DG_ACCUM_EXACT;

  // native encoding, shard-local (row_ptr rebased to 0).  (binary16, u16) matrices are kept as
  // one packed u32 stream (Packed16: column << 16 | value bits); everything else as SoA arrays.
  uint64_t* d_row_ptr = nullptr;
  void* d_col = nullptr;  // u16 or u32 (SoA)
  void* d_val = nullptr;  // binary16 bits / f32 / f64 (SoA)
  uint32_t* d_packed = nullptr;
  bool packed = false;
  uint64_t matrix_bytes = 0;
  uint64_t read_ns = 0;  // dg_create_from_ddm: file sections -> device (dg_info.read_ns)

  // row plan: short-row bins ...
  uint32_t* d_bin[kNumBins] = {};
  uint32_t bin_count[kNumBins] = {};
  uint64_t bin_nnz[kNumBins] = {};
  uint64_t plan_bytes = 0, nonempty_rows = 0;
  // ... and column-windowed tiles of row segments, per wave (plan.cu, spmv_tiles.cuh)
  static constexpr uint32_t kMaxWaves = 64;
  static constexpr int kTileWarps = 32;
  static constexpr int kTileUnroll = 8;
  uint32_t acc_bytes = 8;          // shared-memory x element: 8 exact, 4 fp32
  uint32_t window_cols = 0;        // x window capacity per buffer (columns)
  // replicated x windows (slot mode, spmv_tiles.cuh): exact family on the Packed16 stream
  bool slot_mode = false;          // the plan may build slot-mode tiles (DG_REPLICAS=0: never)
  uint32_t rep_stride = 0;         // elements between replica regions of a window buffer
  uint64_t slot_tiles = 0;         // slot-mode tiles in the plan
  bool slots_encoded = false;      // the stream's slot-mode positions hold slots (else columns)
  // slice stream (spmv_slices.cuh, slices.cu): binary16 matrices under lane_width 32
  static constexpr int kSliceWarps = 28;       // warps per CTA of k_slices (72 registers; r02: 28 / 32 / 24 warps: C2 1.214 / 1.219 / 1.275 ms, C3 shard 0.176 / 0.182, C5 and 100-step C2 -1 to -5%)
  static constexpr int kSliceWarpsShort = 32;  // ... with 4-chunk batches (short segments; C1: 32 / 28 warps 0.0996 / 0.1036 ms)
  static constexpr int kSliceWarpsCarry = 28;  // ... with carried partials (r02 C4: 20 / 24 / 26 / 28 / 32 warps 4.11 / 3.79 / 3.79 / 3.66 / 4.34 ms; 28 = 72 registers)
  bool slices_wanted = false;      // plan for the slice stream (DG_SLICES=0: row-ordered k_tiles)
  bool slices = false;             // the plan has one; d_slices holds it
  static constexpr int kRunsPerWarp = 2;     // runs per tile = kRunsPerWarp x warps (pulled dynamically)
  int slice_warps = 0;
  int slice_runs = 0;
  uint64_t slice_chunks = 0;       // 32-word chunks in the stream
  uint32_t* d_slices = nullptr;
  void* d_ranges = nullptr;        // WarpRange[tiles * runs + 1]
  void* d_sseg = nullptr;          // SliceSeg per segment
  uint64_t n_segments = 0;         // segments of launch list 0
  // with slices the handle's stream (d_packed / d_col / d_val, d_row_ptr) is the REST stream of
  // the rows the tile kernel does not own; d_row_ptr_orig is the upload's row pointer
  uint64_t* d_row_ptr_orig = nullptr;
  uint64_t rest_nnz = 0;
  uint64_t tile_nnz = 768 * 1024;  // target nonzeros per tile (finish_create: the measured sweep)
  uint64_t min_tiles_per_sm = 8;   // tiles <= nnz / (this x SMs) (DG_TILES_PER_SM)
  uint64_t tile_guide = 2;             // guided tail: tiles <= remaining / (guide * SMs) (0: off)
  uint64_t tile_guide_min = 64 * 1024;  // smallest guided tile (nonzeros)
  uint32_t n_waves = 0;
  uint64_t n_split_rows = 0, n_global_rows = 0;
  uint64_t short_max = 32;  // rows with len <= short_max use the sub-warp bins, others the tiles
  uint64_t global_min_len = ~0ull;  // dense rows at least this long read x from global memory
  // dense rows (>= 3/4 of their span) at least dense_min_len long: the k_dense kernel (DG_DENSE)
  int dense_mode = -1;        // DG_DENSE: -1 auto (plan.cu), 0 off, 1 on
  bool dense_kernel = false;
  uint64_t dense_min_len = 4096;  // C2: 2.69 ms (1024: 2.80); its 1/8 shard 0.394 ms (1024: 0.380)
  uint32_t* d_dense_rows = nullptr;  // longest first
  uint32_t* d_dense_counter = nullptr;
  // dense rows over the slice layout (k_dense_slices, spmv_slices.cuh): Packed16 uploads with the
  // slice stream; the rows are then not in the rest stream
  bool dense_slices = false;
  uint32_t* d_dslices = nullptr;   // lane-major 4-chunk blocks, one run per dense row
  void* d_dranges = nullptr;       // WarpRange[n_dense_rows + 1]
  void* d_dsseg = nullptr;         // SliceSeg[n_dense_rows]
  uint64_t dense_chunks = 0;
  uint64_t n_dense_rows = 0, dense_nnz = 0;
  // contiguous rows (columns lo .. lo + len - 1: every dense row of the reference generator's
  // profiles at len >= its locality window) at least dense_min_len long, with the slice stream:
  // streamed as binary16 values only (k_dense_values, spmv_slices.cuh) -- the column of position
  // p is lo + p, so 2 bytes per nonzero instead of 4; not in the rest stream
  std::vector<uint8_t> dense_contig;  // plan -> build_slices: per dense row (longest first)
  uint64_t n_value_rows = 0, value_nnz = 0, value_blocks = 0;
  void* d_vrows = nullptr;            // DenseRow[n_value_rows], longest first
  uint16_t* d_vstream = nullptr;      // lane-major 8-chunk blocks of binary16 values
  uint32_t* d_value_counter = nullptr;
  int dense_cfg = 0;  // DG_DENSE_CFG: (U, P) = (8, 4) default, 1: (16, 2), 2: (8, 8)
  bool pdl = true;       // DG_PDL: tile kernel as a programmatic dependent launch after k_dense
  bool pdl_next = false; // (this dose: the next launch is that dependent launch)
  uint32_t wave_tiles[kMaxWaves] = {};
  uint64_t wave_nnz[kMaxWaves] = {}, wave_rows[kMaxWaves] = {};
  void* d_tiles[kMaxWaves] = {};
  void* d_segs[kMaxWaves] = {};
  void* d_state = nullptr;
  bool fused_waves = false;            // all waves in one launch (wave 0's list)
  bool short_segments = false;         // mean tile segment < 256 nonzeros: 4-chunk batches
  uint64_t n_carry_slots = 0;          // split-row boundaries (32 partials each, Carry)
  uint64_t fused_rows = 0, fused_nnz = 0;
  uint32_t* d_counters = nullptr;
  unsigned long long* d_trace = nullptr;  // DG_TRACE diagnostic timeline (dg_debug_trace)
  uint64_t trace_len = 0;
  int sm_count = 148;
  bool use_tiles = false;
  bool tiles_attr = false;
  int tile_cfg = 0;  // DG_TILE_CFG: alternative (warps, U) configurations for A/B

  // output row blocks (plan.cu): the d download of block k overlaps the kernel's later blocks
  static constexpr uint32_t kMaxBlocks = 64;     // DG_BLOCKS range
  static constexpr uint32_t kDefaultBlocks = 16;  // r02 C2 e2e: 16 blocks 2.12-2.14 ms, 32: 2.19-2.27, 64: 2.44-2.47
  uint32_t n_blocks = 1;
  uint64_t blk_row0[kMaxBlocks + 1] = {};
  uint32_t blk_tiles[kMaxBlocks] = {};
  uint32_t* d_blk_left = nullptr;       // per-dose countdown of unfinished tiles per block
  uint32_t* d_blk_left_init = nullptr;  // the tile counts, copied into d_blk_left per dose
  uint32_t* d_blk_flag = nullptr;       // epoch of the dose that last completed block k
  uint32_t epoch = 0;
  cudaStream_t d2h_stream = nullptr, d2h_stream2 = nullptr;
  cudaEvent_t ev_d2h_done2 = nullptr;
  cudaEvent_t ev_tiles_start = nullptr, ev_d2h_done = nullptr;
  bool signal_blocks = false;  // this dose publishes block completion (host d, overlapped D2H)
  // dg_multi PEER gather: device copies of this shard's rows (other devices' full d at this
  // shard's offset); a device-d dose copies each row block there as soon as the tile kernel
  // publishes it (copy engines, overlapped with the later blocks' tiles)
  std::vector<double*> sink_ptr;
  std::vector<int> sink_dev;
  bool sink_overlap = false;  // (this dose)
  bool sink_remote = false;   // some sink is on another device (overlap pays there)
  double* host_sink = nullptr;  // dg_multi, host d: this dose also downloads its rows here, block by block

  // fused d gather: every finished row also goes to each rank's full-d buffer (peer memory)
  GatherTargets gt = {};
  bool gt_zeroed = false;  // this shard's rows of every target were zero-filled (once per list)

  // staging for host x / y and the fp32 family
  // x staged for the tile kernel (XSource): d_x_raw + kXPad is x (16-byte aligned, 16 readable
  // elements on each side), d_x1_raw + kXPad + 1 the same values one element further on
  static constexpr uint32_t kXPad = 16;
  double* d_x_raw = nullptr;
  double* d_x1_raw = nullptr;
  double* d_x = nullptr;   // = d_x_raw + kXPad
  double* d_x1 = nullptr;  // = d_x1_raw + kXPad + 1
  double* d_y = nullptr;
  bool dy_zeroed = false;  // d_y's empty rows hold +0.0 (zero-filled by the first host-d dose)
  float* d_xf = nullptr;
  unsigned* d_bad = nullptr;

  cudaEvent_t ev[4] = {};
  dg_timing last = {};
  bool timing_valid = false;
  uint32_t n_kernels = 0;

  // per-launch profiling (DG_PROFILE)
  static constexpr int kMaxLaunches = 48;
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

  // tile launch lists: one (all waves fused) or one per wave (n_waves <= kMaxWaves)
  uint32_t n_launch_lists() const { return fused_waves ? 1u : (n_waves < kMaxWaves ? n_waves : kMaxWaves); }

  uint32_t expected_kernels() const {
    uint32_t n = accumulation == DG_ACCUM_FP32 ? 1 : 0;
    if (lane_width == 32) {
      for (int b = 0; b < kNumBins; ++b) n += bin_count[b] ? 1 : 0;
      for (uint32_t w = 0; w < n_launch_lists(); ++w) n += wave_tiles[w] ? 1 : 0;
      n += n_dense_rows ? 1 : 0;
      n += n_value_rows ? 1 : 0;
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

// Call f with the handle's element stream (Packed16 or SoA<V, I>).
template <typename F>
int dispatch_mat(const Handle* h, F&& f) {
  if (h->packed) return f(Packed16{h->d_packed});
  const bool u16 = h->index_bytes == 2;
  switch (h->value_precision) {
    case DG_HALF:
      return u16 ? f(SoA<uint16_t, uint16_t>{static_cast<const uint16_t*>(h->d_col),
                                             static_cast<const uint16_t*>(h->d_val)})
                 : f(SoA<uint16_t, uint32_t>{static_cast<const uint32_t*>(h->d_col),
                                             static_cast<const uint16_t*>(h->d_val)});
    case DG_SINGLE:
      return u16 ? f(SoA<float, uint16_t>{static_cast<const uint16_t*>(h->d_col),
                                          static_cast<const float*>(h->d_val)})
                 : f(SoA<float, uint32_t>{static_cast<const uint32_t*>(h->d_col),
                                          static_cast<const float*>(h->d_val)});
    default:
      return u16 ? f(SoA<double, uint16_t>{static_cast<const uint16_t*>(h->d_col),
                                           static_cast<const double*>(h->d_val)})
                 : f(SoA<double, uint32_t>{static_cast<const uint32_t*>(h->d_col),
                                           static_cast<const double*>(h->d_val)});
  }
}

typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn wait_value_fn();
// dg_multi: register the peer copies of this shard's rows (see sink_ptr); false if unused
bool set_block_sinks(Handle* h, const double* const* dst, const int* dev, uint32_t n);
int copy_to_sinks(Handle* h, const double* src, uint64_t r0, uint64_t r1, cudaStream_t c);

// shared by dosegpu.cu, plan.cu and generator.cu
int select_device(int32_t want, int* dev_out);
int check_options(const dg_options* o);
int finish_create(Handle* h, const std::vector<uint64_t>& lens);
int plan_tiles(Handle* h, const std::vector<uint64_t>& lens);
int recode_slots(Handle* h, bool decode);
int plan_slices(Handle* h, const std::vector<Tile>& tiles, std::vector<Segment>& segs);
int build_slices(Handle* h);
int decode_rows(const Handle* h, uint64_t r0, uint64_t r1, uint32_t* d_col, uint16_t* d_val);
template <typename Acc>
int launch_slices(Handle* h, const Acc* x, double* y, cudaStream_t s);
template <typename Acc>
int launch_dense_slices(Handle* h, const Acc* x, double* y, cudaStream_t s);
template <typename Acc>
int launch_values(Handle* h, const Acc* x, double* y, cudaStream_t s, bool last);
// the upload's row pointer (rows in the reference's order)
inline const uint64_t* orig_row_ptr(const Handle* h) { return h->d_row_ptr_orig ? h->d_row_ptr_orig : h->d_row_ptr; }
int grid_for(uint64_t work_items, int threads, int max_blocks_per_sm = 8);
// a handle created from a shard-only view: record the shard's place in the source matrix
inline void set_shard_rows(Handle* h, uint64_t r0, uint64_t r1) {
  h->row_begin = r0;
  h->row_end = r1;
}

}  // namespace dg
