// adapter_test.cpp -- the reference's own dose assertions (proj/tests/test_spmv.cpp,
// acceptance.cpp criterion 4/5) run against the drop-in ddm_cuda adapter, with matrices built by
// the UNMODIFIED reference library (oracle/_ref/libddmref.so).  Built by `make -C oracle adapter`
// into oracle/_ref/adapter_test; run on a GPU box by tests/test_adapter_gpu.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "ddm/bench.hpp"
#include "ddm/checksum.hpp"
#include "ddm/error.hpp"
#include "ddm/matgen.hpp"
#include "ddm/sparse.hpp"
#include "ddm/spmv.hpp"
#include "dosegpu/ddm_adapter.hpp"

namespace {

int g_fail = 0, g_pass = 0;

void check(bool ok, const std::string& what) {
  if (ok) {
    ++g_pass;
  } else {
    ++g_fail;
    std::printf("FAIL: %s\n", what.c_str());
  }
}

bool bit_equal(const ddm::DenseVector& a, const ddm::DenseVector& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * 8) == 0);
}

ddm::CsrMatrix make_csr(std::uint64_t rows, std::uint64_t cols, std::vector<ddm::CooEntry> e,
                        ddm::ValuePrecision p = ddm::ValuePrecision::Double) {
  ddm::CooMatrix coo;
  coo.rows = rows;
  coo.cols = cols;
  coo.entries = std::move(e);
  return ddm::coo_to_csr(coo, p, ddm::IndexWidth::U32);
}

}  // namespace

int main() {
  // criterion 4/5 shape: desk profiles, every lane width, bit-identical to the CPU engine
  for (const auto& prof : {ddm::liver_desk_profile(), ddm::prostate_desk_profile()}) {
    for (const auto prec : {ddm::ValuePrecision::Half, ddm::ValuePrecision::Single,
                            ddm::ValuePrecision::Double}) {
      const ddm::CsrMatrix m = ddm::generate(prof, prec);
      const ddm::DenseVector x = ddm::seeded_vector(m.cols, 42);
      for (std::size_t lane : {1, 2, 4, 8, 16, 32, 64, 256, 1024}) {
        const auto cpu = ddm::spmv_rowchunk(m, x, {lane, 4});
        const auto gpu = ddm_cuda::spmv_rowchunk(m, x, ddm::RowChunkConfig{lane, 4});
        check(bit_equal(cpu, gpu), "rowchunk lane " + std::to_string(lane) + " rows " +
                                       std::to_string(m.rows) + " prec " +
                                       std::to_string(static_cast<int>(prec)));
      }
      check(bit_equal(ddm::spmv_oracle(m, x), ddm_cuda::spmv_oracle(m, x)), "oracle");
      // the optimisation loop: one resident matrix, many x
      ddm_cuda::DoseEngine eng(m);
      for (std::uint64_t seed : {1, 2, 3}) {
        const ddm::DenseVector xs = ddm::seeded_vector(m.cols, seed);
        check(ddm::checksum_bits(eng.dose(xs)) ==
                  ddm::checksum_bits(ddm::spmv_rowchunk(m, xs, {32, 8})),
              "engine seed " + std::to_string(seed));
      }
    }
  }
  // test_spmv.cpp:104-121 pinned tree
  {
    const double p0 = 1.0, p1 = -1.0 + 0x1p-53, p2 = -0x1p-53, p3 = 0x1p-100;
    const auto m = make_csr(1, 4, {{0, 0, p0}, {0, 1, p1}, {0, 2, p2}, {0, 3, p3}});
    const auto y = ddm_cuda::spmv_rowchunk(m, ddm::DenseVector(4, 1.0), ddm::RowChunkConfig{4, 1});
    check(y[0] == 0.0 && !std::signbit(y[0]), "pinned tree");
  }
  // test_spmv.cpp:156-171 error contract, through the adapter
  {
    const auto m = make_csr(4, 4, {{0, 0, 1.0}, {1, 1, 1.0}, {2, 2, 1.0}, {3, 3, 1.0}});
    for (std::size_t lanes : {0, 3, 48, 2048}) {
      bool threw = false;
      try {
        (void)ddm_cuda::spmv_rowchunk(m, ddm::DenseVector(4, 1.0), ddm::RowChunkConfig{lanes, 1});
      } catch (const ddm::Error& e) {
        threw = e.code() == ddm::Errc::InvalidConfig;
      }
      check(threw, "InvalidConfig lane " + std::to_string(lanes));
    }
    bool threw = false;
    try {
      (void)ddm_cuda::spmv_rowchunk(m, ddm::DenseVector(5, 1.0));
    } catch (const ddm::Error& e) {
      threw = e.code() == ddm::Errc::DimensionMismatch;
    }
    check(threw, "DimensionMismatch");
  }
  // the multi-device engine: shards on a device list (virtual shards on one GPU: PEER / NONE
  // gathers), same bits as the CPU engine
  {
    const ddm::CsrMatrix m = ddm::generate(ddm::liver_desk_profile(), ddm::ValuePrecision::Half);
    const ddm::DenseVector x = ddm::seeded_vector(m.cols, 42);
    const auto cpu = ddm::spmv_rowchunk(m, x, {32, 4});
    for (std::uint32_t gather : {DG_GATHER_PEER, DG_GATHER_NONE}) {
      ddm_cuda::MultiDoseEngine eng(m, {0, 0, 0}, gather);
      check(bit_equal(cpu, eng.dose(x)), "multi-device engine gather " + std::to_string(gather));
    }
    bool threw = false;
    try {
      ddm_cuda::MultiDoseEngine eng(m, {0, 0}, DG_GATHER_NCCL);  // one rank per GPU
    } catch (const ddm::Error& e) {
      threw = e.code() == ddm::Errc::InvalidConfig;
    }
    check(threw, "NCCL gather with a repeated device");
  }
  std::printf("adapter_test: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
