// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" veneer over the UNMODIFIED reference library (ddmkit, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// the Python tests and bench.py's CPU-baseline leg call the reference's own
// dose path (ddm::spmv_rowchunk / spmv_oracle / run_bench / generate) through
// plain pointers.  Nothing here re-implements reference logic: each function
// copies raw arrays into a ddm::CsrMatrix and calls the reference.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <vector>

#include "ddm/bench.hpp"
#include "ddm/checksum.hpp"
#include "ddm/error.hpp"
#include "ddm/half.hpp"
#include "ddm/io.hpp"
#include "ddm/matgen.hpp"
#include "ddm/sparse.hpp"
#include "ddm/spmv.hpp"
#include "ddm_oracle.h"

namespace {

int code_of(const ddm::Error& e) { return 1 + static_cast<int>(e.code()); }

ddm::CsrMatrix to_ddm(const or_csr* m) {
  ddm::CsrMatrix out;
  out.rows = m->rows;
  out.cols = m->cols;
  out.index_width = m->index_width == OR_U16 ? ddm::IndexWidth::U16 : ddm::IndexWidth::U32;
  out.row_ptr.assign(m->row_ptr, m->row_ptr + m->rows + 1);
  out.col_indices.assign(m->col, m->col + m->nnz);
  switch (m->precision) {
    case OR_HALF: {
      std::vector<ddm::Half> v(m->nnz);
      if (m->nnz) std::memcpy(v.data(), m->values, m->nnz * 2);
      out.values = ddm::ValueStore(std::move(v));
      break;
    }
    case OR_SINGLE: {
      const float* p = static_cast<const float*>(m->values);
      out.values = ddm::ValueStore(std::vector<float>(p, p + m->nnz));
      break;
    }
    default: {
      const double* p = static_cast<const double*>(m->values);
      out.values = ddm::ValueStore(std::vector<double>(p, p + m->nnz));
    }
  }
  return out;
}

ddm::MatrixProfile to_profile(const or_profile* p) {
  ddm::MatrixProfile q;
  q.rows = p->rows;
  q.cols = p->cols;
  q.target_nnz_ratio = p->target_nnz_ratio;
  q.empty_row_fraction = p->empty_row_fraction;
  q.row_length_log_mean = p->row_length_log_mean;
  q.row_length_log_sigma = p->row_length_log_sigma;
  q.locality_window = p->locality_window;
  q.seed = p->seed;
  return q;
}

}  // namespace

extern "C" {

// ddm::generate (matgen.cpp:128-178); arrays malloc'd, release with ref_csr_free.
int ref_generate(const or_profile* p, int precision, int index_width, or_csr* out) {
  std::memset(out, 0, sizeof(*out));
  try {
    std::optional<ddm::IndexWidth> w;
    if (index_width >= 0) w = index_width == OR_U16 ? ddm::IndexWidth::U16 : ddm::IndexWidth::U32;
    const ddm::CsrMatrix m =
        ddm::generate(to_profile(p), static_cast<ddm::ValuePrecision>(precision), w);
    out->rows = m.rows;
    out->cols = m.cols;
    out->nnz = m.nnz();
    out->precision = static_cast<int>(m.precision());
    out->index_width = m.index_width == ddm::IndexWidth::U16 ? OR_U16 : OR_U32;
    out->row_ptr = static_cast<uint64_t*>(std::malloc((m.rows + 1) * 8));
    std::memcpy(out->row_ptr, m.row_ptr.data(), (m.rows + 1) * 8);
    out->col = static_cast<uint32_t*>(std::malloc(m.nnz() * 4 + 4));
    if (m.nnz()) std::memcpy(out->col, m.col_indices.data(), m.nnz() * 4);
    const std::size_t vb = ddm::byte_width(m.precision());
    out->values = std::malloc(m.nnz() * vb + 8);
    std::visit([&](const auto& v) { if (!v.empty()) std::memcpy(out->values, v.data(), v.size() * vb); },
               m.values.data());
    return 0;
  } catch (const ddm::Error& e) {
    return code_of(e);
  }
}

void ref_csr_free(or_csr* m) {
  std::free(m->row_ptr);
  std::free(m->col);
  std::free(m->values);
  std::memset(m, 0, sizeof(*m));
}

// ddm::spmv_rowchunk (spmv.cpp:98-111)
int ref_spmv_rowchunk(const or_csr* m, const double* x, uint64_t x_len, uint64_t lane_width,
                      uint64_t workers, double* y) {
  try {
    const ddm::CsrMatrix mm = to_ddm(m);
    const ddm::DenseVector out = ddm::spmv_rowchunk(
        mm, ddm::DenseVector(x, x + x_len), {.lane_width = lane_width, .workers = workers});
    std::memcpy(y, out.data(), out.size() * 8);
    return 0;
  } catch (const ddm::Error& e) {
    return code_of(e);
  }
}

// ddm::spmv_oracle (spmv.cpp:82-96)
int ref_spmv_oracle(const or_csr* m, const double* x, uint64_t x_len, double* y) {
  try {
    const ddm::CsrMatrix mm = to_ddm(m);
    const ddm::DenseVector out = ddm::spmv_oracle(mm, ddm::DenseVector(x, x + x_len));
    std::memcpy(y, out.data(), out.size() * 8);
    return 0;
  } catch (const ddm::Error& e) {
    return code_of(e);
  }
}

// ddm::validate (sparse.cpp:197-255): 0 when ok, else 1 + ValidationFailure.
int ref_validate(const or_csr* m) {
  const ddm::ValidationReport r = ddm::validate(to_ddm(m));
  return r.ok ? 0 : 1 + static_cast<int>(ddm::Errc::ValidationFailure);
}

// ddm::write_ddm / ddm::read_ddm (src/io.cpp:67-168): the DDM1 container.
int ref_write_ddm(const or_csr* m, const char* path) {
  try {
    ddm::write_ddm(to_ddm(m), std::filesystem::path(path));
    return 0;
  } catch (const ddm::Error& e) {
    return code_of(e);
  }
}

int ref_read_ddm(const char* path, or_csr* out) {
  std::memset(out, 0, sizeof(*out));
  try {
    const ddm::CsrMatrix m = ddm::read_ddm(std::filesystem::path(path));
    out->rows = m.rows;
    out->cols = m.cols;
    out->nnz = m.nnz();
    out->precision = static_cast<int>(m.precision());
    out->index_width = m.index_width == ddm::IndexWidth::U16 ? OR_U16 : OR_U32;
    out->row_ptr = static_cast<uint64_t*>(std::malloc((m.rows + 1) * 8));
    std::memcpy(out->row_ptr, m.row_ptr.data(), (m.rows + 1) * 8);
    out->col = static_cast<uint32_t*>(std::malloc(m.nnz() * 4 + 4));
    if (m.nnz()) std::memcpy(out->col, m.col_indices.data(), m.nnz() * 4);
    const std::size_t vb = ddm::byte_width(m.precision());
    out->values = std::malloc(m.nnz() * vb + 8);
    std::visit([&](const auto& v) { if (!v.empty()) std::memcpy(out->values, v.data(), v.size() * vb); },
               m.values.data());
    return 0;
  } catch (const ddm::Error& e) {
    return code_of(e);
  }
}

uint64_t ref_checksum_bits(const double* v, uint64_t n) {
  return ddm::checksum_bits(std::span<const double>(v, n));
}

double ref_decode_half(uint16_t h) { return ddm::decode_half(ddm::Half{h}); }

int ref_encode_half(double x, uint16_t* out) {
  try {
    *out = ddm::encode_half(x).bits;
    return 0;
  } catch (const ddm::Error& e) {
    return code_of(e);
  }
}

void ref_seeded_vector(uint64_t n, uint64_t seed, double* out) {
  const ddm::DenseVector v = ddm::seeded_vector(n, seed);
  std::memcpy(out, v.data(), n * 8);
}

// ddm::run_bench (bench.cpp:38-103) -- the reference's own CPU timer.
// algorithm: 0 oracle, 1 rowchunk.  out[0..5] = mean_s, min_s, gbps, gflops,
// oi, checksum (as double bits in out_checksum).
int ref_run_bench(const or_csr* m, int algorithm, uint64_t lane_width, uint64_t workers,
                  uint64_t reps, uint64_t warmup, uint64_t vector_seed, double* out,
                  uint64_t* out_checksum) {
  try {
    const ddm::CsrMatrix mm = to_ddm(m);
    ddm::BenchConfig cfg;
    cfg.algorithm = algorithm == 0 ? ddm::Algorithm::Oracle : ddm::Algorithm::RowChunk;
    cfg.lane_width = lane_width;
    cfg.workers = workers;
    cfg.repetitions = reps;
    cfg.warmup = warmup;
    cfg.vector_seed = vector_seed;
    const ddm::BenchReport r = ddm::run_bench(mm, "sample", cfg);
    out[0] = r.mean_seconds;
    out[1] = r.min_seconds;
    out[2] = r.effective_gbps;
    out[3] = r.gflops;
    out[4] = r.operational_intensity;
    *out_checksum = r.output_checksum;
    return 0;
  } catch (const ddm::Error& e) {
    return code_of(e);
  }
}

}  // extern "C"

// ddm::render_csv (bench.cpp:141-153) of one report, for format parity of the GPU rows.
extern "C" int ref_render_csv_row(const char* label, int algorithm, int precision, uint64_t lane,
                                  uint64_t chunks, uint64_t workers, uint64_t reps, double mean,
                                  double mn, double gflops, double gbps, double oi,
                                  uint64_t checksum, char* out, uint64_t cap) {
  ddm::BenchReport r;
  r.matrix_label = label;
  r.algorithm = static_cast<ddm::Algorithm>(algorithm);
  r.precision = static_cast<ddm::ValuePrecision>(precision);
  r.lane_width = lane;
  r.chunk_count = chunks;
  r.workers = workers;
  r.repetitions = reps;
  r.mean_seconds = mean;
  r.min_seconds = mn;
  r.gflops = gflops;
  r.effective_gbps = gbps;
  r.operational_intensity = oi;
  r.output_checksum = checksum;
  const std::string s = ddm::render_csv(std::span<const ddm::BenchReport>(&r, 1));
  if (s.size() + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

// ddm::csr_to_csc + ddm::spmv_scatter_baseline (sparse.cpp:166-195, spmv.cpp:113-150).
extern "C" int ref_spmv_scatter(const or_csr* m, const double* x, uint64_t x_len,
                                uint64_t chunk_count, uint64_t workers, double* y) {
  try {
    const ddm::CscMatrix csc = ddm::csr_to_csc(to_ddm(m));
    const ddm::DenseVector out = ddm::spmv_scatter_baseline(
        csc, ddm::DenseVector(x, x + x_len), {.chunk_count = chunk_count, .workers = workers});
    std::memcpy(y, out.data(), out.size() * 8);
    return 0;
  } catch (const ddm::Error& e) {
    return code_of(e);
  }
}
