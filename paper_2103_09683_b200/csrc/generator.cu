// generator.cu -- row-parallel synthetic dose-deposition matrices on the device.
//
// Re-design of ddm::generate (src/matgen.cpp:128-178) for billion-nnz matrices: the reference
// draws every row from ONE sequential xoshiro256** stream on the host (C2 would take ~7 min and
// ~60 GB of host RAM).  Here each row owns an independent xoshiro256** stream seeded from
// (profile seed, row), so rows are generated in parallel, and any row range (a GPU's shard) is
// generated without the others.  Per row the draw ORDER and DISTRIBUTIONS follow the reference:
//   empty test (next_double53 < empty_row_fraction)                       matgen.cpp:149
//   len = clip(llround(exp(mu + sigma * normal)), 1, cols)                matgen.cpp:151-155
//   centre = next_below(cols); span = max(window, len); lo clamped         matgen.cpp:157-160
//   a uniform len-subset of [lo, lo+span), ascending                       matgen.cpp:162-167
//   values uniform in [2^-14, 1], rounded to binary16 (RNE)                matgen.cpp:171-172
// The subset is drawn by selection sampling (Knuth's Algorithm S), which emits the columns
// already sorted instead of the reference's partial Fisher-Yates + sort; both give every
// len-subset probability 1/C(span, len).  The output is statistically, not bitwise, equivalent
// (device exp/log1p/cos differ from glibc in the last ulp, and the streams differ); parity of the
// dose path on these matrices is checked row-sampled against the oracle (tests/).
#include <cub/device/device_scan.cuh>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <new>
#include <vector>

#include "common.cuh"
#include "handle.cuh"
#include "spmv_kernels.cuh"

namespace dg {

struct Beam {
  uint64_t cols, window, seed, col_offset;
  double empty, mu, sigma;
};

constexpr int kMaxBeams = 16;
struct Beams {
  Beam b[kMaxBeams];
  int n;
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// xoshiro256** 1.0 (rng.hpp:14-61), one stream per (beam seed, row).
struct Rng {
  uint64_t s0, s1, s2, s3;
  __device__ explicit Rng(uint64_t seed, uint64_t row) {
    uint64_t z = mix64(seed ^ mix64(row + 0x632BE59BD9B4E019ull));
    z += 0x9E3779B97F4A7C15ull; s0 = mix64(z);
    z += 0x9E3779B97F4A7C15ull; s1 = mix64(z);
    z += 0x9E3779B97F4A7C15ull; s2 = mix64(z);
    z += 0x9E3779B97F4A7C15ull; s3 = mix64(z);
  }
  __device__ __forceinline__ static uint64_t rotl(uint64_t x, int k) {
    return (x << k) | (x >> (64 - k));
  }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t result = rotl(s1 * 5, 7) * 9;
    const uint64_t t = s1 << 17;
    s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t;
    s3 = rotl(s3, 45);
    return result;
  }
  __device__ __forceinline__ double next_double53() {
    return static_cast<double>(next() >> 11) * 0x1.0p-53;
  }
  __device__ uint64_t next_below(uint64_t n) {  // Lemire (rng.hpp:43-54)
    uint64_t x = next();
    uint64_t hi = __umul64hi(x, n), lo = x * n;
    if (lo < n) {
      const uint64_t threshold = (0 - n) % n;
      while (lo < threshold) {
        x = next();
        hi = __umul64hi(x, n);
        lo = x * n;
      }
    }
    return hi;
  }
  __device__ double next_normal() {  // Box-Muller, cosine branch (rng.hpp:57-61)
    const double u1 = next_double53();
    const double u2 = next_double53();
    return sqrt(-2.0 * log1p(-u1)) * cos(2.0 * 3.141592653589793 * u2);
  }
};

struct RowDraw {
  uint64_t len, lo, span;
};

__device__ __forceinline__ RowDraw draw_row(const Beam& b, Rng& rng) {
  RowDraw d{0, 0, 0};
  if (rng.next_double53() < b.empty) return d;
  const double raw = exp(b.mu + b.sigma * rng.next_normal());
  uint64_t len = b.cols;
  if (raw < static_cast<double>(b.cols)) len = max(1ll, llround(raw));
  const uint64_t center = rng.next_below(b.cols);
  const uint64_t span = max(b.window, len);
  uint64_t lo = center > span / 2 ? center - span / 2 : 0;
  lo = min(lo, b.cols - span);
  return {len, lo, span};
}

__global__ void k_gen_lengths(Beams beams, uint64_t row0, uint64_t n_rows, uint64_t* out64,
                              uint32_t* out32) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_rows;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t len = 0;
    for (int k = 0; k < beams.n; ++k) {
      Rng rng(beams.b[k].seed, row0 + i);
      len += draw_row(beams.b[k], rng).len;
    }
    if (out64) out64[i] = len;
    if (out32) out32[i] = static_cast<uint32_t>(len);
  }
  if (out64 && blockIdx.x == 0 && threadIdx.x == 0) out64[n_rows] = 0;
}

// Writes SoA (col, val) or, when packed != nullptr, Packed16 words (u16 columns only).
template <typename I>
__global__ void k_gen_fill(Beams beams, uint64_t row0, uint64_t n_rows,
                           const uint64_t* __restrict__ rp, I* __restrict__ col,
                           uint16_t* __restrict__ val, uint32_t* __restrict__ packed) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_rows;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t pos = rp[i];
    for (int k = 0; k < beams.n; ++k) {
      const Beam& b = beams.b[k];
      Rng rng(b.seed, row0 + i);
      const RowDraw d = draw_row(b, rng);
      uint64_t need = d.len;
      for (uint64_t t = 0; need > 0; ++t) {
        // Algorithm S: keep position t with probability need / (span - t).
        if (rng.next_double53() * static_cast<double>(d.span - t) < static_cast<double>(need)) {
          const uint64_t c = b.col_offset + d.lo + t;
          const double v = 0x1p-14 + (1.0 - 0x1p-14) * rng.next_double53();
          const uint16_t hv = __half_as_ushort(__double2half(v));
          if (packed) {
            packed[pos] = pack16(static_cast<uint16_t>(c), hv);
          } else {
            col[pos] = static_cast<I>(c);
            val[pos] = hv;
          }
          ++pos;
          --need;
        }
      }
    }
  }
}

int to_beams(const dg_profile* p, uint32_t n, Beams* out, uint64_t* rows, uint64_t* cols) {
  if (!p || n < 1 || n > kMaxBeams) return DG_ERR_INVALID_CONFIG;
  uint64_t off = 0;
  for (uint32_t k = 0; k < n; ++k) {
    const dg_profile& q = p[k];
    // ddm::validate_profile (matgen.cpp:96-126), same checks, order and Errc: ranges, then the
    // expected-value consistency of the length distribution with the target ratio (+-10%)
    if (q.rows < 1 || q.cols < 1) return DG_ERR_INVALID_CONFIG;
    auto fraction = [](double f) { return f >= 0.0 && f <= 1.0; };
    if (!fraction(q.target_nnz_ratio)) return DG_ERR_INVALID_CONFIG;
    if (!fraction(q.empty_row_fraction)) return DG_ERR_INVALID_CONFIG;
    if (!(q.row_length_log_sigma >= 0.0)) return DG_ERR_INVALID_CONFIG;
    if (q.locality_window < 1 || q.locality_window > q.cols) return DG_ERR_INVALID_CONFIG;
    {
      const double mean_len = std::min(
          static_cast<double>(q.cols),
          std::max(1.0, std::exp(q.row_length_log_mean +
                                 0.5 * q.row_length_log_sigma * q.row_length_log_sigma)));
      const double expected = (1.0 - q.empty_row_fraction) * mean_len / static_cast<double>(q.cols);
      if (q.target_nnz_ratio == 0.0) {
        if (q.empty_row_fraction != 1.0) return DG_ERR_INCONSISTENT_PROFILE;
      } else {
        if (q.empty_row_fraction == 1.0) return DG_ERR_INCONSISTENT_PROFILE;
        if (std::fabs(expected - q.target_nnz_ratio) / q.target_nnz_ratio > 0.10)
          return DG_ERR_INCONSISTENT_PROFILE;
      }
    }
    if (q.rows != p[0].rows) return DG_ERR_DIMENSION_MISMATCH;
    out->b[k] = {q.cols, q.locality_window, q.seed, off, q.empty_row_fraction,
                 q.row_length_log_mean, q.row_length_log_sigma};
    off += q.cols;
  }
  out->n = static_cast<int>(n);
  *rows = p[0].rows;
  *cols = off;
  return off > 0xFFFFFFFFull ? DG_ERR_INDEX_OVERFLOW : DG_OK;
}

}  // namespace dg

using dg::Handle;

extern "C" {

int dg_generated_row_lengths(const dg_profile* p, uint32_t n_beams, uint64_t r0, uint64_t r1,
                             int32_t device, uint32_t* lengths_out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  dg::Beams beams;
  uint64_t rows = 0, cols = 0;
  DG_TRY(dg::to_beams(p, n_beams, &beams, &rows, &cols));
  if (r0 > r1 || r1 > rows || !lengths_out) return DG_ERR_INVALID_CONFIG;
  int dev = 0;
  DG_TRY(dg::select_device(device, &dev));
  const uint64_t n = r1 - r0;
  if (!n) return DG_OK;
  uint32_t* d = nullptr;
  DG_CUDA(cudaMalloc(&d, n * 4));
  dg::k_gen_lengths<<<dg::grid_for(n, 256), 256>>>(beams, r0, n, nullptr, d);
  cudaError_t e = cudaMemcpy(lengths_out, d, n * 4, cudaMemcpyDeviceToHost);
  cudaFree(d);
  DG_CUDA(e);
  return DG_OK;
}

int dg_create_generated(const dg_profile* p, uint32_t n_beams, uint32_t index_bytes,
                        const dg_options* opts_in, dg_handle** out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!out) return DG_ERR_INVALID_CONFIG;
  *out = nullptr;
  dg_options opts;
  dg_default_options(&opts);
  if (opts_in) opts = *opts_in;
  DG_TRY(dg::check_options(&opts));
  dg::Beams beams;
  uint64_t rows = 0, cols = 0;
  DG_TRY(dg::to_beams(p, n_beams, &beams, &rows, &cols));
  if (index_bytes == 0) index_bytes = cols < 65536 ? 2 : 4;  // matgen.cpp:131-132
  if (index_bytes != 2 && index_bytes != 4) return DG_ERR_INVALID_CONFIG;
  if (index_bytes == 2 && cols >= 65536) return DG_ERR_INDEX_OVERFLOW;
  const uint64_t r0 = opts.row_begin, r1 = opts.row_end ? opts.row_end : rows;
  if (r0 > r1 || r1 > rows) return DG_ERR_INVALID_CONFIG;
  int dev = 0;
  DG_TRY(dg::select_device(opts.device, &dev));

  Handle* h = new (std::nothrow) Handle();
  if (!h) return DG_ERR_OUT_OF_MEMORY;
  auto fail = [&](int s) { dg_destroy(reinterpret_cast<dg_handle*>(h)); return s; };
  auto cu = [&](cudaError_t e) { return e == cudaSuccess ? DG_OK : DG_ERR_CUDA_BASE + (int)e; };
  const uint64_t n = r1 - r0;
  h->device = dev;
  h->rows = n;
  h->cols = cols;
  h->row_begin = r0;
  h->row_end = r1;
  h->value_precision = DG_HALF;
  h->value_bytes = 2;
  h->index_bytes = index_bytes;
  h->lane_width = opts.lane_width;
  h->accumulation = opts.accumulation;
  int st;
  if ((st = cu(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking)))) return fail(st);
  if ((st = cu(cudaMalloc(&h->d_bad, sizeof(unsigned))))) return fail(st);
  if ((st = cu(cudaMalloc(&h->d_row_ptr, (n + 1) * 8)))) return fail(st);
  dg::k_gen_lengths<<<dg::grid_for(n + 1, 256), 256>>>(beams, r0, n, h->d_row_ptr, nullptr);
  size_t tmp_bytes = 0;
  if ((st = cu(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, h->d_row_ptr, n + 1)))) return fail(st);
  void* tmp = nullptr;
  if ((st = cu(cudaMalloc(&tmp, tmp_bytes)))) return fail(st);
  st = cu(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, h->d_row_ptr, n + 1));
  cudaFree(tmp);
  if (st) return fail(st);
  std::vector<uint64_t> rp(n + 1);
  if ((st = cu(cudaMemcpy(rp.data(), h->d_row_ptr, (n + 1) * 8, cudaMemcpyDeviceToHost)))) return fail(st);
  h->nnz = rp[n];
  const uint64_t nz = std::max<uint64_t>(h->nnz, 1);
  const char* nopack = std::getenv("DG_NO_PACK");
  if (index_bytes == 2 && !(nopack && *nopack == '1')) {  // (binary16, u16): Packed16 stream
    if ((st = cu(cudaMalloc(&h->d_packed, nz * 4 + 16)))) return fail(st);  // TMA granule pad
    h->packed = true;
    dg::k_gen_fill<uint16_t><<<dg::grid_for(n, 128), 128>>>(beams, r0, n, h->d_row_ptr, nullptr,
                                                           nullptr, h->d_packed);
  } else {
    if ((st = cu(cudaMalloc(&h->d_val, nz * 2)))) return fail(st);
    if ((st = cu(cudaMalloc(&h->d_col, nz * index_bytes)))) return fail(st);
    if (index_bytes == 2)
      dg::k_gen_fill<uint16_t><<<dg::grid_for(n, 128), 128>>>(
          beams, r0, n, h->d_row_ptr, static_cast<uint16_t*>(h->d_col),
          static_cast<uint16_t*>(h->d_val), nullptr);
    else
      dg::k_gen_fill<uint32_t><<<dg::grid_for(n, 128), 128>>>(
          beams, r0, n, h->d_row_ptr, static_cast<uint32_t*>(h->d_col),
          static_cast<uint16_t*>(h->d_val), nullptr);
  }
  if ((st = cu(cudaGetLastError()))) return fail(st);
  // ddm::validate's per-entry invariants on the generated matrix too (the reference validates
  // every CsrMatrix it builds; one pass over the device copy)
  if ((st = cu(cudaMemset(h->d_bad, 0, sizeof(unsigned))))) return fail(st);
  st = dg::dispatch_mat(h, [&](const auto& mat) {
    dg::k_validate<<<dg::grid_for(32 * n, 256), 256>>>(mat, h->d_row_ptr, n, h->cols, h->d_bad);
    return cu(cudaGetLastError());
  });
  if (st) return fail(st);
  if ((st = cu(cudaDeviceSynchronize()))) return fail(st);
  {
    unsigned bad = 0;
    if ((st = cu(cudaMemcpy(&bad, h->d_bad, sizeof(unsigned), cudaMemcpyDeviceToHost)))) return fail(st);
    if (bad) return fail(DG_ERR_VALIDATION_FAILURE);
  }
  h->matrix_bytes = (n + 1) * 8 + h->nnz * (2 + index_bytes);
  std::vector<uint64_t> lens(n);
  for (uint64_t r = 0; r < n; ++r) lens[r] = rp[r + 1] - rp[r];
  if ((st = dg::finish_create(h, lens))) return fail(st);
  *out = reinterpret_cast<dg_handle*>(h);
  return DG_OK;
}

}  // extern "C"
