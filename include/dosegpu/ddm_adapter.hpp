// ddm_adapter.hpp -- header-only C++ adapter that makes libdosegpu.so a drop-in for the
// reference's dose path.  Include it from code that already includes the reference headers
// (ddm/sparse.hpp, ddm/error.hpp); link with -ldosegpu.
//
//   ddm::spmv_rowchunk(m, x, {32, W})      (include/ddm/spmv.hpp:37)
//   -> ddm_cuda::spmv_rowchunk(m, x, {32, W})   same arguments, same result bits, same errors
//
//   ddm::spmv_oracle(m, x)                 (include/ddm/spmv.hpp:29)
//   -> ddm_cuda::spmv_oracle(m, x)             lane_width 1 on the device, same bits
//
// For the optimisation loop (many doses of one immutable matrix), ddm_cuda::DoseEngine keeps the
// matrix resident on the GPU: construct once, call dose(x) per iteration.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "ddm/error.hpp"
#include "ddm/sparse.hpp"
#include "ddm/spmv.hpp"
#include "dosegpu.h"

namespace ddm_cuda {

struct CudaConfig {
  std::size_t lane_width = 32;  // ddm::RowChunkConfig::lane_width
  std::size_t workers = 1;      // accepted for signature parity; never changes a bit
  int device = -1;              // CUDA ordinal, -1 = current
  bool fp32 = false;            // fp32 family (north_star tolerance) instead of exact fp64
};

// Status -> the reference's error model (include/ddm/error.hpp:8-41): contract codes become
// ddm::Error with the same Errc; device failures become std::runtime_error.
inline void check(int status, const char* where) {
  if (status == DG_OK) return;
  if (status >= 1 && status <= 16)
    ddm::fail(static_cast<ddm::Errc>(status - 1), std::string(where) + ": " + dg_strerror(status));
  throw std::runtime_error(std::string(where) + ": " + dg_strerror(status) + " (" +
                           std::to_string(status) + ")");
}

inline dg_csr_view view_of(const ddm::CsrMatrix& m) {
  dg_csr_view v{};
  v.rows = m.rows;
  v.cols = m.cols;
  v.nnz = m.nnz();
  v.value_precision = static_cast<uint8_t>(m.precision());
  v.index_bytes = m.index_width == ddm::IndexWidth::U16 ? 2 : 4;
  v.col_storage_bytes = 4;  // ddm keeps vector<uint32_t> whatever the tag (sparse.hpp:104)
  v.on_device = 0;
  v.row_ptr = m.row_ptr.data();
  v.col_indices = m.col_indices.data();
  v.values = std::visit([](const auto& vec) -> const void* { return vec.data(); },
                        m.values.data());
  return v;
}

class DoseEngine {
 public:
  DoseEngine(const ddm::CsrMatrix& m, const CudaConfig& cfg = {}) {
    if (cfg.workers < 1) ddm::fail(ddm::Errc::InvalidConfig, "workers must be >= 1");
    dg_options o;
    dg_default_options(&o);
    o.device = cfg.device;
    o.lane_width = static_cast<uint32_t>(cfg.lane_width);
    o.accumulation = cfg.fp32 ? DG_ACCUM_FP32 : DG_ACCUM_EXACT;
    const dg_csr_view v = view_of(m);
    check(dg_create(&v, &o, &h_), "dg_create");
    rows_ = m.rows;
    cols_ = m.cols;
  }
  DoseEngine(const DoseEngine&) = delete;
  DoseEngine& operator=(const DoseEngine&) = delete;
  ~DoseEngine() { dg_destroy(h_); }

  ddm::DenseVector dose(const ddm::DenseVector& x) {
    if (x.size() != cols_)  // spmv.cpp:34-38
      ddm::fail(ddm::Errc::DimensionMismatch, "input vector length " + std::to_string(x.size()) +
                                                  " != matrix columns " + std::to_string(cols_));
    ddm::DenseVector y(rows_, 0.0);
    check(dg_dose(h_, x.data(), x.size(), y.data(), 0, nullptr), "dg_dose");
    return y;
  }

  dg_handle* handle() const { return h_; }

 private:
  dg_handle* h_ = nullptr;
  std::uint64_t rows_ = 0, cols_ = 0;
};

// Several GPUs behind one engine (dg_multi_*): the reference fans one call out over worker
// threads (parallel_blocks, src/spmv.cpp:17-32); this fans it out over devices -- nnz-balanced
// row shards, concurrent doses, the full d gathered on every device (PEER copies or NCCL) and
// returned on the host.  Same bits as DoseEngine / ddm::spmv_rowchunk for any device list.
class MultiDoseEngine {
 public:
  MultiDoseEngine(const ddm::CsrMatrix& m, const std::vector<int>& devices,
                  std::uint32_t gather = DG_GATHER_PEER, const CudaConfig& cfg = {}) {
    if (cfg.workers < 1) ddm::fail(ddm::Errc::InvalidConfig, "workers must be >= 1");
    if (devices.empty() || devices.size() > DG_MAX_DEVICES)
      ddm::fail(ddm::Errc::InvalidConfig, "1.." + std::to_string(DG_MAX_DEVICES) + " devices");
    dg_multi_options o;
    dg_multi_default_options(&o);
    o.n_devices = static_cast<std::uint32_t>(devices.size());
    for (std::size_t i = 0; i < devices.size(); ++i) o.devices[i] = devices[i];
    o.lane_width = static_cast<std::uint32_t>(cfg.lane_width);
    o.accumulation = cfg.fp32 ? DG_ACCUM_FP32 : DG_ACCUM_EXACT;
    o.gather = gather;
    const dg_csr_view v = view_of(m);
    check(dg_multi_create(&v, &o, &m_), "dg_multi_create");
    rows_ = m.rows;
    cols_ = m.cols;
  }
  MultiDoseEngine(const MultiDoseEngine&) = delete;
  MultiDoseEngine& operator=(const MultiDoseEngine&) = delete;
  ~MultiDoseEngine() { dg_multi_destroy(m_); }

  ddm::DenseVector dose(const ddm::DenseVector& x) {
    if (x.size() != cols_)  // spmv.cpp:34-38
      ddm::fail(ddm::Errc::DimensionMismatch, "input vector length " + std::to_string(x.size()) +
                                                  " != matrix columns " + std::to_string(cols_));
    ddm::DenseVector y(rows_, 0.0);
    check(dg_multi_dose(m_, x.data(), x.size(), y.data(), 0), "dg_multi_dose");
    return y;
  }

  dg_multi* handle() const { return m_; }

 private:
  dg_multi* m_ = nullptr;
  std::uint64_t rows_ = 0, cols_ = 0;
};

// Drop-in for ddm::spmv_rowchunk: the reference checks dims before the config (spmv.cpp:99-100).
inline ddm::DenseVector spmv_rowchunk(const ddm::CsrMatrix& m, const ddm::DenseVector& x,
                                      const CudaConfig& cfg = {}) {
  if (x.size() != m.cols)
    ddm::fail(ddm::Errc::DimensionMismatch, "input vector length " + std::to_string(x.size()) +
                                                " != matrix columns " + std::to_string(m.cols));
  DoseEngine e(m, cfg);
  return e.dose(x);
}

inline ddm::DenseVector spmv_rowchunk(const ddm::CsrMatrix& m, const ddm::DenseVector& x,
                                      const ddm::RowChunkConfig& cfg) {
  return spmv_rowchunk(m, x, CudaConfig{cfg.lane_width, cfg.workers, -1, false});
}

inline ddm::DenseVector spmv_oracle(const ddm::CsrMatrix& m, const ddm::DenseVector& x) {
  return spmv_rowchunk(m, x, CudaConfig{1, 1, -1, false});
}

}  // namespace ddm_cuda
