// ddm_io.cu -- DDM1 container -> device upload.
//
// The reference reads a DDM1 file element by element through std::istream (get_uint_le per
// value, src/io.cpp:132-159, ~80 MB/s).  The format's sections are already little-endian arrays in
// exactly the SoA layout the device uses (row_ptr u64, col u16/u32, values as bit patterns), so
// here the column and value sections are read with large pread()s into two pinned buffers and
// copied asynchronously to the device while the next chunk is read; dg_create then validates,
// packs and plans the device copy.
//
// Row shards (opts->row_begin / row_end): the section layout is fixed by the header (io.cpp:67-96,
// 103-168), so a rank reads the whole row_ptr section (8 B per row: every row_ptr invariant is
// checked, as read_ddm does) but only the byte ranges [rp[r0], rp[r1]) of the column and value
// sections -- peak device memory is the shard, not the file.  The per-entry invariants
// (ddm::validate: columns in range and increasing, finite values) are checked on the shard's
// entries.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "handle.cuh"

namespace {

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

bool read_all(int fd, void* dst, size_t n, off_t off) {
  char* p = static_cast<char*>(dst);
  while (n) {
    const ssize_t r = pread(fd, p, n, off);
    if (r <= 0) return false;
    p += r;
    off += r;
    n -= static_cast<size_t>(r);
  }
  return true;
}

uint64_t le64(const unsigned char* b) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
  return v;
}

// Stream [off, off + bytes) of the file into device memory through two pinned staging buffers.
int stream_section(int fd, off_t off, uint64_t bytes, char* d_dst, char* pinned[2], size_t chunk,
                   cudaStream_t s, cudaEvent_t done[2]) {
  int buf = 0;
  for (uint64_t pos = 0; pos < bytes; pos += chunk, buf ^= 1) {
    const size_t n = static_cast<size_t>(std::min<uint64_t>(chunk, bytes - pos));
    DG_CUDA(cudaEventSynchronize(done[buf]));  // the copy that last used this buffer finished
    if (!read_all(fd, pinned[buf], n, off + static_cast<off_t>(pos))) return DG_ERR_TRUNCATED_FILE;
    DG_CUDA(cudaMemcpyAsync(d_dst + pos, pinned[buf], n, cudaMemcpyHostToDevice, s));
    DG_CUDA(cudaEventRecord(done[buf], s));
  }
  return DG_OK;
}

}  // namespace

extern "C" int dg_create_from_ddm(const char* path, const dg_options* opts, dg_handle** out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!path || !out) return DG_ERR_INVALID_CONFIG;
  if (opts) DG_TRY(dg::check_options(opts));
  *out = nullptr;
  Fd f;
  f.fd = open(path, O_RDONLY);
  if (f.fd < 0) return DG_ERR_IO_FAILURE;
  struct stat st {};
  if (fstat(f.fd, &st) != 0) return DG_ERR_IO_FAILURE;
  const uint64_t fsize = static_cast<uint64_t>(st.st_size);

  // header: io.hpp:10-20, checks in read_ddm's order (io.cpp:104-130)
  unsigned char h[32];
  const size_t hn = static_cast<size_t>(std::min<uint64_t>(32, fsize));
  if (hn < 4 || !read_all(f.fd, h, hn, 0)) return DG_ERR_TRUNCATED_FILE;
  if (std::memcmp(h, "DDM1", 4) != 0) return DG_ERR_BAD_MAGIC;
  if (hn < 5) return DG_ERR_TRUNCATED_FILE;
  if (h[4] != 1) return DG_ERR_UNSUPPORTED_VERSION;
  if (hn < 6) return DG_ERR_TRUNCATED_FILE;
  if (h[5] > 2) return DG_ERR_VALIDATION_FAILURE;
  if (hn < 7) return DG_ERR_TRUNCATED_FILE;
  if (h[6] != 2 && h[6] != 4) return DG_ERR_VALIDATION_FAILURE;
  if (hn < 8) return DG_ERR_TRUNCATED_FILE;
  if (h[7] != 0) return DG_ERR_VALIDATION_FAILURE;
  if (hn < 32) return DG_ERR_TRUNCATED_FILE;
  const uint64_t rows = le64(h + 8), cols = le64(h + 16), nnz = le64(h + 24);
  if (rows >= (1ull << 53) || nnz >= (1ull << 53)) return DG_ERR_VALIDATION_FAILURE;
  const uint32_t ib = h[6], vb = h[5] == 0 ? 2 : h[5] == 1 ? 4 : 8;
  const uint64_t rp_off = 32, col_off = rp_off + 8 * (rows + 1), val_off = col_off + ib * nnz,
                 end = val_off + vb * nnz;
  if (fsize < end) return DG_ERR_TRUNCATED_FILE;
  if (fsize > end) return DG_ERR_VALIDATION_FAILURE;  // trailing bytes (io.cpp:162-163)

  int dev = 0;
  DG_TRY(dg::select_device(opts ? opts->device : -1, &dev));
  const auto t_read0 = std::chrono::steady_clock::now();
  std::vector<uint64_t> rp(rows + 1);
  if (!read_all(f.fd, rp.data(), 8 * (rows + 1), static_cast<off_t>(rp_off)))
    return DG_ERR_TRUNCATED_FILE;
  // row_ptr invariants of the whole file (sparse.cpp:221-229)
  if (rp[0] != 0 || rp[rows] != nnz) return DG_ERR_VALIDATION_FAILURE;
  for (uint64_t r = 0; r < rows; ++r)
    if (rp[r + 1] < rp[r]) return DG_ERR_VALIDATION_FAILURE;
  const uint64_t r0 = opts ? opts->row_begin : 0;
  const uint64_t r1 = opts && opts->row_end ? opts->row_end : rows;
  if (r0 > r1 || r1 > rows) return DG_ERR_INVALID_CONFIG;
  const uint64_t n_rows = r1 - r0, p0 = rp[r0], snnz = rp[r1] - rp[r0];
  std::vector<uint64_t> srp(n_rows + 1);
  for (uint64_t r = 0; r <= n_rows; ++r) srp[r] = rp[r0 + r] - p0;

  // device staging of the shard's three sections, then the regular create path on a device view
  uint64_t* d_rp = nullptr;
  char *d_col = nullptr, *d_val = nullptr, *pinned[2] = {nullptr, nullptr};
  cudaStream_t s = nullptr;
  cudaEvent_t done[2] = {nullptr, nullptr};
  // 16-MB staging buffers: pinning is paid per call (64 MB buffers took ~80 ms of a C1 read)
  const size_t chunk = 16ull << 20;
  int rc = DG_OK;
  auto cu = [&](cudaError_t e) { if (rc == DG_OK && e != cudaSuccess) rc = DG_ERR_CUDA_BASE + (int)e; };
  cu(cudaMalloc(&d_rp, 8 * (n_rows + 1)));
  cu(cudaMalloc(&d_col, std::max<uint64_t>(ib * snnz, 16)));
  cu(cudaMalloc(&d_val, std::max<uint64_t>(vb * snnz, 16)));
  cu(cudaHostAlloc(&pinned[0], chunk, cudaHostAllocDefault));
  cu(cudaHostAlloc(&pinned[1], chunk, cudaHostAllocDefault));
  cu(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cu(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  cu(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  if (rc == DG_OK) {
    cu(cudaEventRecord(done[0], s));
    cu(cudaEventRecord(done[1], s));
    cu(cudaMemcpyAsync(d_rp, srp.data(), 8 * (n_rows + 1), cudaMemcpyHostToDevice, s));
  }
  if (rc == DG_OK)
    rc = stream_section(f.fd, static_cast<off_t>(col_off + ib * p0), ib * snnz, d_col, pinned, chunk, s, done);
  if (rc == DG_OK)
    rc = stream_section(f.fd, static_cast<off_t>(val_off + vb * p0), vb * snnz, d_val, pinned, chunk, s, done);
  if (rc == DG_OK) cu(cudaStreamSynchronize(s));
  const uint64_t read_ns = static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                                     std::chrono::steady_clock::now() - t_read0).count());
  if (rc == DG_OK) {
    dg_csr_view v{};
    v.rows = n_rows;
    v.cols = cols;
    v.nnz = snnz;
    v.value_precision = h[5];
    v.index_bytes = static_cast<uint8_t>(ib);
    v.col_storage_bytes = static_cast<uint8_t>(ib);
    v.on_device = 1;
    v.row_ptr = d_rp;
    v.col_indices = d_col;
    v.values = d_val;
    dg_options o;
    dg_default_options(&o);
    if (opts) o = *opts;
    o.device = dev;
    o.row_begin = 0;
    o.row_end = 0;
    rc = dg_create(&v, &o, out);
    if (rc == DG_OK) {
      dg::set_shard_rows(reinterpret_cast<dg::Handle*>(*out), r0, r1);
      reinterpret_cast<dg::Handle*>(*out)->read_ns = read_ns;
    }
  }
  if (s) cudaStreamSynchronize(s);
  cudaFree(d_rp);
  cudaFree(d_col);
  cudaFree(d_val);
  cudaFreeHost(pinned[0]);
  cudaFreeHost(pinned[1]);
  for (auto e : done)
    if (e) cudaEventDestroy(e);
  if (s) cudaStreamDestroy(s);
  return rc;
}
