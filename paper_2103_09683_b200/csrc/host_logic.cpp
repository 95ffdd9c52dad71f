// host_logic.cpp -- host-side (CPU) pieces of the C ABI that need no device: status strings,
// the perf-model byte count and the nnz-balanced row partitioner.  Kept in a separate TU so the
// CPU test suite can exercise them through the C ABI on a box without a GPU.
#include <cstdint>

#include "dosegpu.h"

extern "C" {

// ddm::errc_name (src/sparse.cpp:22-42), indexed by status - 1.
const char* dg_strerror(int status) {
  static const char* const kErrc[] = {
      "DuplicateEntry", "IndexOverflow",      "ValueOverflow",     "NanInput",
      "DimensionMismatch", "InvalidConfig",   "ZeroTraffic",       "ZeroDuration",
      "BadMagic",       "TruncatedFile",      "ValidationFailure", "UnsupportedVersion",
      "ParseError",     "UnsupportedFeature", "InconsistentProfile", "IoFailure"};
  if (status == DG_OK) return "OK";
  if (status >= 1 && status <= 16) return kErrc[status - 1];
  if (status == DG_ERR_NO_DEVICE) return "NoDevice";
  if (status == DG_ERR_OUT_OF_MEMORY) return "OutOfMemory";
  if (status == DG_ERR_NO_NCCL) return "NoNccl";
  if (status >= DG_ERR_NCCL_BASE) return "NcclError";
  if (status >= DG_ERR_CUDA_BASE) return "CudaError";
  return "Unknown";
}

const char* dg_version(void) { return "dosegpu 0.2 (sm_100a)"; }

void dg_multi_default_options(dg_multi_options* o) {
  if (!o) return;
  *o = dg_multi_options{};
  o->struct_size = sizeof(dg_multi_options);
  o->n_devices = 1;
  o->devices[0] = 0;
  o->lane_width = 32;
  o->accumulation = DG_ACCUM_EXACT;
  o->gather = DG_GATHER_PEER;
}

// ddm::traffic(dims_of(m), layout_of(m)).total_bytes() -- perf_model.cpp:41-54 with
// layout_of's 8-byte row pointers and 8-byte input/output vectors.
uint64_t dg_traffic_bytes(uint64_t rows, uint64_t cols, uint64_t nnz, uint32_t value_bytes,
                          uint32_t index_bytes) {
  return static_cast<uint64_t>(value_bytes + index_bytes) * nnz + 16ull * rows + 8ull * cols;
}

// ddm::seeded_vector (src/bench.cpp:31-36) over xoshiro256** seeded by splitmix64
// (include/ddm/rng.hpp:16-40): the reference benchmark's x.
void dg_seeded_vector(uint64_t n, uint64_t seed, double* out) {
  uint64_t s[4], z = seed;
  for (auto& w : s) {
    z += 0x9E3779B97F4A7C15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    w = x ^ (x >> 31);
  }
  auto rotl = [](uint64_t x, int k) { return (x << k) | (x >> (64 - k)); };
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    out[i] = static_cast<double>(result >> 11) * 0x1.0p-53;
  }
}

void dg_default_options(dg_options* o) {
  o->struct_size = sizeof(dg_options);
  o->device = -1;
  o->lane_width = 32;
  o->accumulation = DG_ACCUM_EXACT;
  o->row_begin = 0;
  o->row_end = 0;
}

}  // extern "C"

namespace {

// bounds[g] = first r with W(r) * parts >= g * W(rows), W(r) = sum_{i<r} (bpn*len_i + 16).
template <typename LenAt>
int partition(uint64_t rows, uint32_t bytes_per_nnz, uint32_t parts, uint64_t* bounds,
              LenAt len_at) {
  if (parts < 1 || bytes_per_nnz < 1) return DG_ERR_INVALID_CONFIG;
  unsigned __int128 total = 0;
  for (uint64_t r = 0; r < rows; ++r)
    total += static_cast<unsigned __int128>(bytes_per_nnz) * len_at(r) + 16u;
  bounds[0] = 0;
  uint32_t g = 1;
  unsigned __int128 w = 0;
  for (uint64_t r = 0; r < rows && g < parts; ++r) {
    while (g < parts && w * parts >= total * g) bounds[g++] = r;
    w += static_cast<unsigned __int128>(bytes_per_nnz) * len_at(r) + 16u;
  }
  while (g < parts) {
    // W(r) * parts >= g * total can first hold at r = rows only when the tail is empty.
    bounds[g++] = rows;
  }
  bounds[parts] = rows;
  return DG_OK;
}

}  // namespace

extern "C" {

int dg_partition_rows(const uint64_t* row_ptr, uint64_t rows, uint32_t bytes_per_nnz,
                      uint32_t parts, uint64_t* bounds) {
  if (!row_ptr || !bounds) return DG_ERR_INVALID_CONFIG;
  for (uint64_t r = 0; r < rows; ++r)
    if (row_ptr[r + 1] < row_ptr[r]) return DG_ERR_VALIDATION_FAILURE;
  return partition(rows, bytes_per_nnz, parts, bounds,
                   [&](uint64_t r) { return row_ptr[r + 1] - row_ptr[r]; });
}

int dg_partition_lengths(const uint32_t* lengths, uint64_t rows, uint32_t bytes_per_nnz,
                         uint32_t parts, uint64_t* bounds) {
  if (!lengths || !bounds) return DG_ERR_INVALID_CONFIG;
  return partition(rows, bytes_per_nnz, parts, bounds,
                   [&](uint64_t r) { return static_cast<uint64_t>(lengths[r]); });
}

}  // extern "C"
