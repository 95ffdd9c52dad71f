// scatter.cu -- the column-scatter comparator: ddm::spmv_scatter_baseline on the
// device, atomic-free and bit-identical (src/spmv.cpp:70-78,113-150).
//
// Reference semantics: columns are split into chunk_count static ranges [b(c), b(c+1)) with
// b(c) = cols * c / chunk_count; chunk c scatters into a private scratch vector (initialised to
// +0.0) in column-major order -- for each column ascending, for each of its rows ascending,
// scratch[row] += x[col] * widen(v) -- and d[i] = sum over chunks in index order, from +0.0.
// Device mapping: one CTA per chunk; a column's rows are distinct, so its updates run in parallel
// with no conflict, and one __syncthreads() per column keeps every row's updates in column
// order.  No atomics anywhere, so the bits are those of the reference for the same chunk_count.
// This is the structure of the paper's "GPU Baseline": a scatter that pays a
// read-modify-write of 8 B of scratch per nonzero, against 4 B of streamed matrix for the gather.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <new>
#include <vector>

#include "common.cuh"
#include "handle.cuh"

struct dg_scatter {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t rows = 0, cols = 0, nnz = 0;
  uint32_t chunks = 1, value_precision = DG_HALF, value_bytes = 2;
  uint64_t* d_col_ptr = nullptr;  // cols + 1
  uint32_t* d_row = nullptr;      // nnz, ascending within each column
  void* d_val = nullptr;          // nnz value bits
  double* d_scratch = nullptr;    // chunks * rows
  double* d_x = nullptr;
  double* d_y = nullptr;
};

namespace dg {

__global__ void k_iota(uint32_t* __restrict__ a, uint64_t n) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    a[i] = static_cast<uint32_t>(i);
}

__global__ void k_row_of(const uint64_t* __restrict__ rp, uint64_t rows, uint32_t* __restrict__ r_of) {
  for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    for (uint64_t j = rp[r]; j < rp[r + 1]; ++j) r_of[j] = static_cast<uint32_t>(r);
}

template <class M>
__global__ void k_col_of(M mat, uint64_t nnz, uint32_t* __restrict__ c_of, uint64_t* __restrict__ counts) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < nnz;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = mat.col_at(j);
    c_of[j] = c;
    atomicAdd(reinterpret_cast<unsigned long long*>(counts + c), 1ull);  // counts only: order-free
  }
}

template <class M>
__global__ void k_gather_csc(M mat, const uint32_t* __restrict__ perm, const uint32_t* __restrict__ r_of,
                             uint64_t nnz, uint32_t* __restrict__ row, typename M::Val* __restrict__ val) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t j = perm[k];
    row[k] = r_of[j];
    val[k] = M::v_of(mat.load(j));
  }
}

template <typename V>
__global__ void __launch_bounds__(1024) k_scatter(const uint64_t* __restrict__ col_ptr,
                                                  const uint32_t* __restrict__ row,
                                                  const V* __restrict__ val,
                                                  const double* __restrict__ x, uint64_t rows,
                                                  uint64_t cols, uint32_t chunks,
                                                  double* __restrict__ scratch) {
  for (uint32_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    // spmv.cpp:120-122: 128-bit boundary so cols * c cannot overflow
    const uint64_t b0 = static_cast<uint64_t>((static_cast<unsigned __int128>(cols) * c) / chunks);
    const uint64_t b1 = static_cast<uint64_t>((static_cast<unsigned __int128>(cols) * (c + 1)) / chunks);
    double* s = scratch + static_cast<uint64_t>(c) * rows;
    for (uint64_t col = b0; col < b1; ++col) {
      const double xc = x[col];
      for (uint64_t j = col_ptr[col] + threadIdx.x; j < col_ptr[col + 1]; j += blockDim.x) {
        const uint32_t r = row[j];
        s[r] = __dadd_rn(s[r], __dmul_rn(xc, widen(val[j])));  // spmv.cpp:76
      }
      __syncthreads();  // the next column's update of a row comes after this one's
    }
  }
}

__global__ void k_merge(const double* __restrict__ scratch, uint64_t rows, uint32_t chunks,
                        double* __restrict__ y) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double acc = 0.0;  // spmv.cpp:143-147
    for (uint32_t c = 0; c < chunks; ++c) acc = __dadd_rn(acc, scratch[static_cast<uint64_t>(c) * rows + i]);
    y[i] = acc;
  }
}

}  // namespace dg

extern "C" {

int dg_scatter_destroy(dg_scatter* s) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!s) return DG_OK;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  cudaFree(s->d_col_ptr);
  cudaFree(s->d_row);
  cudaFree(s->d_val);
  cudaFree(s->d_scratch);
  cudaFree(s->d_x);
  cudaFree(s->d_y);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return DG_OK;
}

int dg_scatter_create(const dg_csr_view* v, uint32_t chunk_count, int32_t device, dg_scatter** out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!v || !out) return DG_ERR_INVALID_CONFIG;
  *out = nullptr;
  if (chunk_count < 1) return DG_ERR_INVALID_CONFIG;  // spmv.cpp:116
  if (v->nnz >= (1ull << 31)) return DG_ERR_UNSUPPORTED_FEATURE;
  // the CSR upload, validation and stream dispatch are dg_create's (exact family, L = 32)
  dg_options o;
  dg_default_options(&o);
  o.device = device;
  dg_handle* hh = nullptr;
  DG_TRY(dg_create(v, &o, &hh));
  dg::Handle* h = reinterpret_cast<dg::Handle*>(hh);
  dg_scatter* s = new (std::nothrow) dg_scatter();
  if (!s) {
    dg_destroy(hh);
    return DG_ERR_OUT_OF_MEMORY;
  }
  s->device = h->device;
  s->rows = h->rows;
  s->cols = h->cols;
  s->nnz = h->nnz;
  s->chunks = chunk_count;
  s->value_precision = h->value_precision;
  s->value_bytes = h->value_bytes;
  int st = DG_OK;
  auto cu = [&](cudaError_t e) { if (st == DG_OK && e != cudaSuccess) st = DG_ERR_CUDA_BASE + (int)e; };
  const uint64_t nz = std::max<uint64_t>(s->nnz, 1);
  uint32_t *r_of = nullptr, *keys = nullptr, *keys_out = nullptr, *idx = nullptr, *perm = nullptr;
  void* tmp = nullptr;
  cu(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  cu(cudaMalloc(&s->d_col_ptr, (s->cols + 1) * 8));
  cu(cudaMalloc(&s->d_row, nz * 4));
  cu(cudaMalloc(&s->d_val, nz * s->value_bytes));
  cu(cudaMalloc(&s->d_scratch, std::max<uint64_t>(1, static_cast<uint64_t>(chunk_count) * s->rows) * 8));
  cu(cudaMalloc(&s->d_x, std::max<uint64_t>(s->cols, 1) * 8));
  cu(cudaMalloc(&s->d_y, std::max<uint64_t>(s->rows, 1) * 8));
  cu(cudaMalloc(&r_of, nz * 4));
  cu(cudaMalloc(&keys, nz * 4));
  cu(cudaMalloc(&keys_out, nz * 4));
  cu(cudaMalloc(&idx, nz * 4));
  cu(cudaMalloc(&perm, nz * 4));
  if (st == DG_OK) st = dg::recode_slots(h, true);  // columns, not slots (the next dose re-encodes)
  // a slice-stream handle: the row-ordered encoding decoded into a (u32 column, binary16) view
  dg::Handle view;
  uint32_t* v_col = nullptr;
  uint16_t* v_val = nullptr;
  if (st == DG_OK && h->slices) {
    cu(cudaMalloc(&v_col, nz * 4));
    cu(cudaMalloc(&v_val, nz * 2));
    if (st == DG_OK) st = dg::decode_rows(h, 0, h->rows, v_col, v_val);
    view.packed = false;
    view.value_precision = DG_HALF;
    view.index_bytes = 4;
    view.d_col = v_col;
    view.d_val = v_val;
    view.d_row_ptr = h->d_row_ptr_orig;
    h = &view;
  }
  if (st == DG_OK) {
    cu(cudaMemset(s->d_col_ptr, 0, (s->cols + 1) * 8));
    dg::k_row_of<<<dg::grid_for(s->rows, 256), 256>>>(h->d_row_ptr, s->rows, r_of);
    st = dg::dispatch_mat(h, [&](const auto& mat) {
      dg::k_col_of<<<dg::grid_for(s->nnz, 256), 256>>>(mat, s->nnz, keys, s->d_col_ptr);
      return 0;
    });
    cu(cudaGetLastError());
  }
  if (st == DG_OK && s->nnz) {
    // identity permutation, then a STABLE radix sort by column: the row-major input order makes
    // the rows ascending inside every column, as ddm::csr_to_csc produces them
    dg::k_iota<<<dg::grid_for(s->nnz, 256), 256>>>(idx, s->nnz);
    size_t tb = 0;
    cu(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_out, idx, perm,
                                       static_cast<int>(s->nnz)));
    cu(cudaMalloc(&tmp, tb));
    cu(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_out, idx, perm,
                                       static_cast<int>(s->nnz)));
    st = st ? st : dg::dispatch_mat(h, [&](const auto& mat) {
      using M = std::decay_t<decltype(mat)>;
      dg::k_gather_csc<M><<<dg::grid_for(s->nnz, 256), 256>>>(
          mat, perm, r_of, s->nnz, s->d_row, static_cast<typename M::Val*>(s->d_val));
      return 0;
    });
    // col_ptr = exclusive scan of the per-column counts (in place, cols + 1 entries)
    size_t sb = 0;
    cu(cub::DeviceScan::ExclusiveSum(nullptr, sb, s->d_col_ptr, s->cols + 1));
    void* stmp = nullptr;
    cu(cudaMalloc(&stmp, sb));
    cu(cub::DeviceScan::ExclusiveSum(stmp, sb, s->d_col_ptr, s->cols + 1));
    cu(cudaDeviceSynchronize());
    cudaFree(stmp);
  }
  cudaFree(tmp);
  cudaFree(r_of);
  cudaFree(keys);
  cudaFree(keys_out);
  cudaFree(idx);
  cudaFree(perm);
  cudaFree(v_col);
  cudaFree(v_val);
  view.d_col = view.d_val = nullptr;
  view.d_row_ptr = nullptr;
  dg_destroy(hh);
  if (st) {
    dg_scatter_destroy(s);
    return st;
  }
  *out = s;
  return DG_OK;
}

int dg_scatter_dose(dg_scatter* s, const double* x, uint64_t x_len, double* y, uint32_t flags,
                    void* stream) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!s || (!x && s->cols) || (!y && s->rows)) return DG_ERR_INVALID_CONFIG;
  if (x_len != s->cols) return DG_ERR_DIMENSION_MISMATCH;
  DG_CUDA(cudaSetDevice(s->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->stream;
  const bool x_dev = flags & DG_X_ON_DEVICE, y_dev = flags & DG_Y_ON_DEVICE;
  const double* d_x = x_dev ? x : s->d_x;
  double* d_y = y_dev ? y : s->d_y;
  if (!x_dev && s->cols)
    DG_CUDA(cudaMemcpyAsync(s->d_x, x, s->cols * 8, cudaMemcpyHostToDevice, st));
  if (s->rows) {
    DG_CUDA(cudaMemsetAsync(s->d_scratch, 0, static_cast<uint64_t>(s->chunks) * s->rows * 8, st));
    const int grid = static_cast<int>(std::min<uint32_t>(s->chunks, 4096));
    switch (s->value_precision) {
      case DG_HALF:
        dg::k_scatter<uint16_t><<<grid, 1024, 0, st>>>(s->d_col_ptr, s->d_row,
            static_cast<const uint16_t*>(s->d_val), d_x, s->rows, s->cols, s->chunks, s->d_scratch);
        break;
      case DG_SINGLE:
        dg::k_scatter<float><<<grid, 1024, 0, st>>>(s->d_col_ptr, s->d_row,
            static_cast<const float*>(s->d_val), d_x, s->rows, s->cols, s->chunks, s->d_scratch);
        break;
      default:
        dg::k_scatter<double><<<grid, 1024, 0, st>>>(s->d_col_ptr, s->d_row,
            static_cast<const double*>(s->d_val), d_x, s->rows, s->cols, s->chunks, s->d_scratch);
    }
    dg::k_merge<<<dg::grid_for(s->rows, 256), 256, 0, st>>>(s->d_scratch, s->rows, s->chunks, d_y);
    DG_CUDA(cudaGetLastError());
  }
  if (!y_dev && s->rows)
    DG_CUDA(cudaMemcpyAsync(y, s->d_y, s->rows * 8, cudaMemcpyDeviceToHost, st));
  if (!(flags & DG_NO_SYNC) || !x_dev || !y_dev) DG_CUDA(cudaStreamSynchronize(st));
  return DG_OK;
}

}  // extern "C"
