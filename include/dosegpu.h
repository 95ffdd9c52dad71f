/*
 * dosegpu.h -- C-ABI drop-in boundary for the dose product d = A.x on B200 (sm_100a).
 *
 * The reference (ddmkit, /root/reference/proj) exposes its dose path as C++ free functions
 * (no FFI/plugin registry).  Each entry point below names the reference interface it
 * replaces; INTEGRATION.md shows the C++ adapter and the ctypes binding a maintainer adds.
 *
 *   dg_create          <- the one-time cost hidden inside every ddm::spmv_rowchunk call:
 *                         check_dims/check_rowchunk_config (src/spmv.cpp:34-46), the CsrMatrix
 *                         invariants of ddm::validate (src/sparse.cpp:197-255), plus the device
 *                         upload of the native encoding (sparse.hpp:93-108).
 *   dg_dose            <- ddm::spmv_rowchunk(const CsrMatrix&, const DenseVector&,
 *                         const RowChunkConfig&)  (include/ddm/spmv.hpp:37, src/spmv.cpp:98-111)
 *                         and, with lane_width 1, ddm::spmv_oracle (spmv.hpp:29, spmv.cpp:82-96).
 *   dg_checksum_bits   <- ddm::checksum_bits (include/ddm/checksum.hpp:25-35).  FNV-1a is a
 *                         sequential hash: a device array is copied to the host and hashed there.
 *   dg_traffic_bytes   <- ddm::traffic(dims_of(m), layout_of(m)).total_bytes()
 *                         (src/perf_model.cpp:41-54) -- the algorithmic bytes of one evaluation.
 *   dg_partition_rows  <- replaces parallel_blocks' equal-row-count split (src/spmv.cpp:17-32)
 *                         with nnz-balanced contiguous row shards (one per GPU).
 *   dg_create_generated<- ddm::generate (src/matgen.cpp:128-178) re-designed row-parallel on the
 *                         device (statistically equivalent, not bit-identical).
 *   dg_strerror        <- ddm::errc_name (src/sparse.cpp:22-42).
 *
 * Status codes: 0 = OK; 1 + (int)ddm::Errc for contract errors (include/ddm/error.hpp:8-25, same
 * order); DG_ERR_CUDA_BASE + cudaError_t for CUDA failures; DG_ERR_NO_DEVICE when no usable
 * sm_100 device exists (the library never falls back to the CPU).
 *
 * Ownership: the caller owns every array it passes; dg_create copies what it needs to the device
 * and keeps no host pointer.  The handle owns all device memory.  Threading: one host thread per
 * handle at a time; handles are independent; the matrix is immutable after dg_create.  Every
 * entry point restores the calling thread's current CUDA device before it returns.
 */
#ifndef DOSEGPU_H
#define DOSEGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------------------------- */
enum {
  DG_OK = 0,
  /* 1 + ddm::Errc (error.hpp:8-25) */
  DG_ERR_DUPLICATE_ENTRY = 1,
  DG_ERR_INDEX_OVERFLOW = 2,
  DG_ERR_VALUE_OVERFLOW = 3,
  DG_ERR_NAN_INPUT = 4,
  DG_ERR_DIMENSION_MISMATCH = 5,
  DG_ERR_INVALID_CONFIG = 6,
  DG_ERR_ZERO_TRAFFIC = 7,
  DG_ERR_ZERO_DURATION = 8,
  DG_ERR_BAD_MAGIC = 9,
  DG_ERR_TRUNCATED_FILE = 10,
  DG_ERR_VALIDATION_FAILURE = 11,
  DG_ERR_UNSUPPORTED_VERSION = 12,
  DG_ERR_PARSE_ERROR = 13,
  DG_ERR_UNSUPPORTED_FEATURE = 14,
  DG_ERR_INCONSISTENT_PROFILE = 15,
  DG_ERR_IO_FAILURE = 16,
  /* library-specific */
  DG_ERR_NO_DEVICE = 900,
  DG_ERR_OUT_OF_MEMORY = 901,
  DG_ERR_NO_NCCL = 902,      /* DG_GATHER_NCCL requested, libnccl.so.2 not loadable */
  DG_ERR_CUDA_BASE = 1000,   /* + cudaError_t */
  DG_ERR_NCCL_BASE = 2000    /* + ncclResult_t */
};

/* ---- the native encoding (ddm::CsrMatrix, sparse.hpp:93-108) ----------------------------- */
enum { DG_HALF = 0, DG_SINGLE = 1, DG_DOUBLE = 2 }; /* ddm::ValuePrecision == DDM1 byte 5 */

typedef struct {
  uint64_t rows, cols, nnz;
  uint8_t value_precision;   /* DG_HALF / DG_SINGLE / DG_DOUBLE */
  uint8_t index_bytes;       /* IndexWidth tag: 2 (U16, legal only when cols < 65536) or 4 */
  uint8_t col_storage_bytes; /* element size of col_indices as passed: 4 (ddm's in-memory
                                vector<uint32_t>) or 2 */
  uint8_t on_device;         /* 1: the three arrays are device pointers on opts->device */
  const uint64_t* row_ptr;   /* rows + 1 entries, row_ptr[0] == 0, row_ptr[rows] == nnz */
  const void* col_indices;   /* nnz entries, strictly increasing within each row */
  const void* values;        /* nnz IEEE bit patterns of value_precision */
} dg_csr_view;

/* ---- evaluation options (ddm::RowChunkConfig, spmv.hpp:15-18, plus device knobs) -------- */
enum {
  DG_ACCUM_EXACT = 0, /* fp64 products and sums, lane assignment + stride-halving tree pinned:
                         output bits == ddm::spmv_rowchunk(m, x, {lane_width, any workers}) */
  DG_ACCUM_FP32 = 1   /* fp32 x/products/sums (north_star tolerance 1e-5 * max|d|), L = 32 */
};

typedef struct {
  uint32_t struct_size;   /* sizeof(dg_options) */
  int32_t device;         /* CUDA ordinal; -1 = current device */
  uint32_t lane_width;    /* power of two in [1, 1024] (spmv.cpp:40-46), else InvalidConfig */
  uint32_t accumulation;  /* DG_ACCUM_* */
  uint64_t row_begin;     /* shard of the view to own: rows [row_begin, row_end); */
  uint64_t row_end;       /* row_end == 0 -> all rows */
} dg_options;

typedef struct dg_handle dg_handle;

void dg_default_options(dg_options* o);

/* Validate (ddm::validate invariants), plan and upload once.  Device arrays of the shard are
 * allocated on opts->device; row_ptr is rebased to the shard. */
int dg_create(const dg_csr_view* view, const dg_options* opts, dg_handle** out);

/* ---- row-parallel device generator (ddm::generate re-designed, matgen.cpp:128-178) -------- */
typedef struct {
  uint64_t rows, cols;
  double target_nnz_ratio, empty_row_fraction;
  double row_length_log_mean, row_length_log_sigma;
  uint64_t locality_window, seed;
} dg_profile; /* == ddm::MatrixProfile (matgen.hpp:18-27) */

/* Generate rows [opts->row_begin, opts->row_end) of a matrix directly into device memory (Half
 * values; index width: index_bytes, or the narrowest legal when 0).  With n_beams > 1 the matrix
 * is the column-wise hstack of the beams' matrices (beam b's columns offset by the sum of the
 * earlier beams' cols; all beams must have the same rows) -- the multi-beam plan of config C4.
 * Row r's content is a pure function of (profiles, r), so shards generated on different GPUs
 * compose into exactly the matrix one GPU would generate. */
int dg_create_generated(const dg_profile* beams, uint32_t n_beams, uint32_t index_bytes,
                        const dg_options* opts, dg_handle** out);
/* Row lengths of that matrix for rows [row_begin, row_end) (host array of u32), used to cut
 * nnz-balanced shards before generating them. */
int dg_generated_row_lengths(const dg_profile* beams, uint32_t n_beams, uint64_t row_begin,
                             uint64_t row_end, int32_t device, uint32_t* lengths_out);

/* DDM1 file -> device, streamed (ddm::read_ddm, src/io.cpp:103-168; format io.hpp:10-20).
 * With opts->row_begin / row_end only that shard's byte ranges of the column and value sections
 * are read (pread at the offsets the header fixes): device memory holds the shard, not the file.
 * The header is checked exactly as the reference does (BadMagic, UnsupportedVersion,
 * ValidationFailure for bad precision/index/reserved bytes or implausible sizes, TruncatedFile,
 * ValidationFailure for trailing bytes), row pointers are read to the host, and the column and
 * value sections are streamed in large chunks through pinned double buffers straight into device
 * memory (the on-disk little-endian section layout IS the device SoA layout), then validated,
 * planned and packed like dg_create.  Replaces the reference's element-at-a-time reader
 * (~80 MB/s). */
int dg_create_from_ddm(const char* path, const dg_options* opts, dg_handle** out);

int dg_destroy(dg_handle* h);

/* ---- the dose evaluation ------------------------------------------------------------------ */
enum {
  DG_X_ON_DEVICE = 1u << 0, /* x is a device pointer (else host; pinned host is fastest) */
  DG_Y_ON_DEVICE = 1u << 1, /* y is a device pointer (else host) */
  DG_NO_SYNC = 1u << 2,     /* device x/y only: return without synchronising the stream */
  DG_PROFILE = 1u << 3      /* record a CUDA event after every launch (dg_kernel_times) */
};

/* d = A.x for the handle's rows.  x has `cols` doubles, y receives `shard rows` doubles; empty
 * rows are exactly +0.0.  `stream` is a cudaStream_t (NULL = the handle's own stream). */
int dg_dose(dg_handle* h, const double* x, uint64_t x_len, double* y, uint32_t flags,
            void* stream);

/* ---- fused d gather over NVLink peer memory ------------------------------- */
/* With n targets set, every dg_dose of this (shard) handle also writes its rows straight into
 * each target -- the full-d buffers of all ranks (this rank's included), mapped into this
 * process through CUDA IPC (dg_ipc_*) -- at global row row_begin + r: the dose kernels' epilogues
 * store each finished row to every target (P2P stores over NVLink, overlapped with the rest of
 * the kernel); this shard's row range of every target is zero-filled by the first dose after
 * the call (its empty rows, which no later dose writes: the targets are read-only to callers).
 * When every rank's dose has completed (the caller's barrier), every rank holds the full d: the
 * all-gather costs no separate collective.  targets == NULL / n == 0 disables. */
int dg_set_gather_targets(dg_handle* h, double* const* targets, uint32_t n);

/* The same exchange by the copy engines instead of the kernels' epilogues: with n targets set,
 * every dg_dose copies this shard's d into each target (at global row row_begin + r) row block by
 * row block -- block k as soon as the tile kernel publishes that its last tile is done
 * (cuStreamWaitValue32 on the block's flag), while the kernel works on later blocks -- in
 * coalesced DMA transfers over NVLink / NVSwitch that cost no SM time (plans without row blocks:
 * right after the kernels).  The copies complete before the dose does on its stream.  Replaces
 * the serial join of ddm::spmv_rowchunk's parallel_blocks (src/spmv.cpp:17-32) across GPUs.
 * targets == NULL / n == 0 disables; may be combined with dg_set_gather_targets. */
int dg_set_block_targets(dg_handle* h, double* const* targets, uint32_t n);

/* Minimal CUDA IPC plumbing for the targets (64-byte cudaIpcMemHandle_t). */
int dg_ipc_alloc(uint64_t bytes, int32_t device, void** dptr, void* handle64);
int dg_ipc_open(const void* handle64, int32_t device, void** dptr);
int dg_ipc_close(void* dptr);
int dg_ipc_free(void* dptr);

/* ---- the column-scatter comparator --------------------------------------- */
/* ddm::spmv_scatter_baseline (src/spmv.cpp:113-150) -- the paper's "GPU Baseline" (a CSC column
 * scatter) done atomic-free and deterministic: columns are split into
 * chunk_count static ranges (boundary c = cols*c/chunk_count); one CTA scatters a chunk into its
 * private scratch vector in column-major order (one barrier per column orders the updates of a
 * row), and the scratches are merged in chunk order.  d is bit-identical to the reference engine
 * for the same chunk_count.  The CSC copy is built on the device (stable by row, like
 * ddm::csr_to_csc, sparse.cpp:166-195); nnz must be < 2^31. */
typedef struct dg_scatter dg_scatter;
int dg_scatter_create(const dg_csr_view* view, uint32_t chunk_count, int32_t device,
                      dg_scatter** out);
int dg_scatter_dose(dg_scatter* s, const double* x, uint64_t x_len, double* y, uint32_t flags,
                    void* stream);
int dg_scatter_destroy(dg_scatter* s);

/* ---- introspection ------------------------------------------------------------------------ */
typedef struct {
  uint64_t rows, cols, nnz;          /* of the shard */
  uint64_t row_begin, row_end;       /* in the source matrix */
  uint32_t value_bytes, index_bytes; /* device encoding (native: no expansion) */
  uint32_t lane_width, accumulation;
  uint64_t device_bytes;             /* resident matrix + plan bytes */
  uint64_t model_bytes;              /* dg_traffic_bytes of the shard */
  uint64_t nonempty_rows;
  uint32_t n_kernels;                /* kernels launched per dg_dose (device-resident x/y) */
  int32_t device;
  uint64_t read_ns;                  /* dg_create_from_ddm: wall time reading the file's row_ptr,
                                        column and value sections into device memory (0 else) */
} dg_info;
int dg_get_info(const dg_handle* h, dg_info* info);

typedef struct {
  float ms_h2d, ms_kernels, ms_d2h, ms_total; /* CUDA-event times of the last dg_dose */
} dg_timing;
int dg_last_timing(const dg_handle* h, dg_timing* t);

/* Per-launch breakdown of the last dg_dose issued with DG_PROFILE: for each kernel launched,
 * its name, CUDA-event duration and algorithmic bytes ((vb+ib)*nnz + 16*rows of the rows it
 * covers + 8*cols for x).  Returns the number of launches written (<= cap). */
typedef struct {
  char name[48];
  float ms;
  uint64_t bytes;
  uint64_t rows, nnz;
} dg_kernel_time;
int dg_kernel_times(const dg_handle* h, dg_kernel_time* out, uint32_t cap, uint32_t* n_out);

/* ---- one process, several GPUs --------------------------------------------- */
/* The reference fans one dose out over threads behind a single call (ddm::spmv_rowchunk,
 * include/ddm/spmv.hpp:37 -> parallel_blocks, src/spmv.cpp:17-32, 105-107).  dg_multi does the
 * same over GPUs: the rows are cut into n_devices nnz-balanced contiguous shards
 * (dg_partition_rows), one dg_handle per device holds its shard plus a replicated x, the doses
 * run concurrently (one stream per device) and the d slices are gathered per `gather`:
 *   DG_GATHER_NONE  d stays row-sharded on the devices (the optimiser's sharded-resident d);
 *   DG_GATHER_PEER  allgatherv by peer copies (copy engines over NVLink / NVSwitch): every
 *                   device ends with the full d; each shard's kernels write their rows straight
 *                   into their own device's full d, which the peers then copy from;
 *   DG_GATHER_NCCL  allgatherv as ncclGroupStart + one ncclBroadcast per shard (root = the
 *                   shard's device, into d_full + row offset on every device) + ncclGroupEnd --
 *                   no padding.  NCCL (libnccl.so.2) is loaded on first use; its failures are
 *                   DG_ERR_NCCL_BASE + ncclResult_t.  Needs distinct devices.
 * A device may appear several times in `devices` (virtual shards on one GPU; NONE / PEER). */
enum { DG_MAX_DEVICES = 16 };
enum { DG_GATHER_NONE = 0, DG_GATHER_PEER = 1, DG_GATHER_NCCL = 2 };
typedef struct {
  uint32_t struct_size;              /* sizeof(dg_multi_options) */
  uint32_t n_devices;                /* 1 .. DG_MAX_DEVICES */
  int32_t devices[DG_MAX_DEVICES];   /* CUDA ordinals of the shards, in row order */
  uint32_t lane_width;               /* as dg_options */
  uint32_t accumulation;             /* as dg_options */
  uint32_t gather;                   /* DG_GATHER_* */
} dg_multi_options;
typedef struct dg_multi dg_multi;

void dg_multi_default_options(dg_multi_options* o); /* 1 device (0), L = 32, exact, PEER */
int dg_multi_create(const dg_csr_view* view, const dg_multi_options* opts, dg_multi** out);
int dg_multi_create_generated(const dg_profile* beams, uint32_t n_beams, uint32_t index_bytes,
                              const dg_multi_options* opts, dg_multi** out);
/* d = A.x over every shard.  x: host (H2D on every device concurrently) or, with
 * DG_X_ON_DEVICE, a device pointer on devices[0] (peer-copied to the others).  y: a host array
 * of `rows` doubles receiving the full d (each device downloads its slice concurrently), or NULL
 * with DG_Y_ON_DEVICE (d stays on the devices: dg_multi_device_d).  The gather runs in both
 * cases.  Synchronous. */
int dg_multi_dose(dg_multi* m, const double* x, uint64_t x_len, double* y, uint32_t flags);
/* shard bounds (n_shards + 1 rows) and shard count */
int dg_multi_bounds(const dg_multi* m, uint32_t* n_shards, uint64_t* bounds);
int dg_multi_shard(const dg_multi* m, uint32_t i, dg_handle** shard);
/* device pointers on shard i's device: its full d (rows doubles; filled by PEER / NCCL gathers)
 * and its own slice (= full_d + bounds[i]) */
int dg_multi_device_d(const dg_multi* m, uint32_t i, double** full_d, double** slice_d);
/* CUDA-event times of the last dg_multi_dose, each the max over devices: x upload, the shard's
 * dose kernels, gather (+ host download), total */
int dg_multi_last_timing(const dg_multi* m, dg_timing* t);
int dg_multi_destroy(dg_multi* m);

/* Diagnostics (no reference counterpart): with DG_TRACE set at dg_create, the first tile wave
 * of every dose records a timeline -- per CTA {start ns, end ns, window-wait cycles, warp-cycles}
 * (4 * sm_count words), then per tile {claim ns, finish ns, CTA | segments << 16 | global-x << 62}.
 * Copies up to cap words of the last dose's timeline; *n_out = 0 when tracing is off. */
int dg_debug_trace(const dg_handle* h, uint64_t* out, uint64_t cap, uint64_t* n_out);

/* ddm::seeded_vector (src/bench.cpp:31-36): x[k] = xoshiro256**(seed).next_double53(). */
void dg_seeded_vector(uint64_t n, uint64_t seed, double* out);

/* Copy rows [r0, r1) of the shard (shard-relative) back to host in the reference's in-memory
 * encoding: row_ptr (r1 - r0 + 1, rebased to 0), col as u32, values as bit patterns. */
int dg_copy_rows(const dg_handle* h, uint64_t r0, uint64_t r1, uint64_t* row_ptr_out,
                 uint32_t* col_out, void* values_out);

/* Row pointers [r0, r1] of the shard (r1 - r0 + 1 entries, shard-relative, NOT rebased). */
int dg_copy_row_ptr(const dg_handle* h, uint64_t r0, uint64_t r1, uint64_t* row_ptr_out);

/* FNV-1a-64 over the bit patterns of a device or host double array (checksum.hpp:25-35); a
 * device array is copied to the host first (the hash is sequential). */
int dg_checksum_bits(const double* v, uint64_t n, int on_device, uint64_t* out);

/* Algorithmic bytes of one evaluation (perf_model.cpp:41-54 with layout_of: row_ptr 8 B and
 * vectors 8 B): (value_bytes + index_bytes)*nnz + 16*rows + 8*cols. */
uint64_t dg_traffic_bytes(uint64_t rows, uint64_t cols, uint64_t nnz, uint32_t value_bytes,
                          uint32_t index_bytes);

/* nnz-balanced contiguous row shards: bounds[0] = 0, bounds[parts] = rows, and bounds[g] is the
 * first row r with W(r) >= g*W(rows)/parts, W(r) = sum_{i<r} (bytes_per_nnz*len_i + 16).
 * row_ptr is a host array (rows + 1). */
int dg_partition_rows(const uint64_t* row_ptr, uint64_t rows, uint32_t bytes_per_nnz,
                      uint32_t parts, uint64_t* bounds);
/* Same, from per-row lengths (u32) instead of row pointers. */
int dg_partition_lengths(const uint32_t* lengths, uint64_t rows, uint32_t bytes_per_nnz,
                         uint32_t parts, uint64_t* bounds);

const char* dg_strerror(int status);
const char* dg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DOSEGPU_H */
