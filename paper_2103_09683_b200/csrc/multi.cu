// multi.cu -- one process, several GPUs behind one handle (include/dosegpu.h, dg_multi_*).
//
// The reference's dose call fans out internally: ddm::spmv_rowchunk (include/ddm/spmv.hpp:37)
// runs parallel_blocks (src/spmv.cpp:17-32, 105-107), equal row-count blocks on std::threads.
// Here the rows are cut into nnz-balanced contiguous shards (dg_partition_rows: the rows are
// independent, src/spmv.cpp:53-67, so a shard needs no data from another), one dg_handle per
// device holds its shard and a replicated x, the shards' doses are issued on one stream per device
// without host synchronisation in between (they run concurrently), and the d slices are gathered
// only when asked:
//   * PEER: every shard's kernels write their rows straight into its own device's full-d buffer
//     (y of that dg_dose = full_d + bounds[g]); the other devices' full d receive that range by
//     cudaMemcpyPeerAsync, i.e. the copy engines move it over NVLink / NVSwitch in large
//     coalesced transfers: row block by row block as the tile kernel publishes each block
//     (cuStreamWaitValue32 on its completion flag), overlapped with the shard's later tiles;
//   * NCCL: an allgatherv with no padding -- ncclGroupStart, for every shard g and every rank r
//     ncclBroadcast(full_r + b_g, count nr_g, root g), ncclGroupEnd.
// NCCL is loaded with dlopen on first use, so the library itself keeps no link-time dependency
// on it and the PEER / NONE paths work where NCCL is absent.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "common.cuh"
#include "handle.cuh"

namespace dg {
namespace {

// ---- NCCL through dlopen -------------------------------------------------------------------
struct Nccl {
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return;
    n.comm_init_all = reinterpret_cast<decltype(n.comm_init_all)>(dlsym(lib, "ncclCommInitAll"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(lib, "ncclCommDestroy"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(lib, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(lib, "ncclGroupEnd"));
    n.broadcast = reinterpret_cast<decltype(n.broadcast)>(dlsym(lib, "ncclBroadcast"));
    n.ok = n.comm_init_all && n.comm_destroy && n.group_start && n.group_end && n.broadcast;
  });
  return n;
}

#define DG_NCCL(expr)                                                          \
  do {                                                                         \
    ncclResult_t _r = (expr);                                                  \
    if (_r != ncclSuccess) return DG_ERR_NCCL_BASE + static_cast<int>(_r);     \
  } while (0)

}  // namespace

struct Multi {
  uint32_t n = 0;
  uint32_t gather = DG_GATHER_PEER;
  uint64_t rows = 0, cols = 0;
  std::vector<int> dev;
  std::vector<uint64_t> bounds;      // n + 1
  std::vector<dg_handle*> shard;
  std::vector<cudaStream_t> stream;
  std::vector<double*> x;            // replicated x per device
  std::vector<double*> full;         // full d per device (the shard's slice is full + bounds[g])
  std::vector<ncclComm_t> comm;
  std::vector<cudaEvent_t> ev;       // 4 per device: start, x ready, dose done, gathered
  bool timing = false;
};

namespace {

int check_multi_options(const dg_multi_options* o) {
  if (!o || o->struct_size != sizeof(dg_multi_options)) return DG_ERR_INVALID_CONFIG;
  if (o->n_devices < 1 || o->n_devices > DG_MAX_DEVICES) return DG_ERR_INVALID_CONFIG;
  if (o->gather > DG_GATHER_NCCL) return DG_ERR_INVALID_CONFIG;
  dg_options so;
  dg_default_options(&so);
  so.lane_width = o->lane_width;
  so.accumulation = o->accumulation;
  DG_TRY(check_options(&so));
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return DG_ERR_NO_DEVICE;
  }
  for (uint32_t i = 0; i < o->n_devices; ++i)
    if (o->devices[i] < 0 || o->devices[i] >= count) return DG_ERR_INVALID_CONFIG;
  if (o->gather == DG_GATHER_NCCL)
    for (uint32_t i = 0; i < o->n_devices; ++i)
      for (uint32_t j = i + 1; j < o->n_devices; ++j)
        if (o->devices[i] == o->devices[j]) return DG_ERR_INVALID_CONFIG;  // one rank per GPU
  return DG_OK;
}

void destroy_multi(Multi* m) {
  if (!m) return;
  for (uint32_t g = 0; g < m->stream.size(); ++g)
    if (m->stream[g]) {
      cudaSetDevice(m->dev[g]);
      cudaStreamSynchronize(m->stream[g]);
    }
  for (auto c : m->comm)
    if (c && nccl().ok) nccl().comm_destroy(c);
  for (uint32_t g = 0; g < m->n; ++g) {
    cudaSetDevice(m->dev[g]);
    if (g < m->shard.size()) dg_destroy(m->shard[g]);
    if (g < m->x.size()) cudaFree(m->x[g]);
    if (g < m->full.size()) cudaFree(m->full[g]);
    if (g < m->stream.size() && m->stream[g]) cudaStreamDestroy(m->stream[g]);
    for (int k = 0; k < 4; ++k)
      if (4 * g + k < m->ev.size() && m->ev[4 * g + k]) cudaEventDestroy(m->ev[4 * g + k]);
  }
  delete m;
}

// Everything after the shards exist: per-device buffers, streams, events, peer access, NCCL.
int finish_multi(Multi* m) {
  m->stream.assign(m->n, nullptr);
  m->x.assign(m->n, nullptr);
  m->full.assign(m->n, nullptr);
  m->ev.assign(4 * m->n, nullptr);
  for (uint32_t g = 0; g < m->n; ++g) {
    DG_CUDA(cudaSetDevice(m->dev[g]));
    DG_CUDA(cudaStreamCreateWithFlags(&m->stream[g], cudaStreamNonBlocking));
    DG_CUDA(cudaMalloc(&m->x[g], std::max<uint64_t>(m->cols, 1) * sizeof(double)));
    DG_CUDA(cudaMalloc(&m->full[g], std::max<uint64_t>(m->rows, 1) * sizeof(double)));
    DG_CUDA(cudaMemset(m->full[g], 0, std::max<uint64_t>(m->rows, 1) * sizeof(double)));
    for (int k = 0; k < 4; ++k) DG_CUDA(cudaEventCreate(&m->ev[4 * g + k]));
  }
  // peer access between every pair of distinct devices (NVLink / NVSwitch); where it is not
  // available cudaMemcpyPeerAsync still works, staged through the host
  for (uint32_t a = 0; a < m->n; ++a)
    for (uint32_t b = 0; b < m->n; ++b) {
      if (m->dev[a] == m->dev[b]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, m->dev[a], m->dev[b]);
      if (!can) continue;
      cudaSetDevice(m->dev[a]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(m->dev[b], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return DG_ERR_CUDA_BASE + (int)e;
      cudaGetLastError();
    }
  // PEER: every shard's dose copies each of its row blocks into the other devices' full d as soon
  // as the tile kernel publishes the block (copy engines over NVLink / NVSwitch, overlapped with
  // the shard's later tiles); plans without row blocks copy right after their kernels
  if (m->gather == DG_GATHER_PEER)
    for (uint32_t g = 0; g < m->n; ++g) {
      std::vector<const double*> dst;
      std::vector<int> dv;
      for (uint32_t t = 0; t < m->n; ++t)
        if (t != g && m->full[t] != m->full[g]) {
          dst.push_back(m->full[t] + m->bounds[g]);
          dv.push_back(m->dev[t]);
        }
      set_block_sinks(reinterpret_cast<Handle*>(m->shard[g]), dst.data(), dv.data(),
                      static_cast<uint32_t>(dst.size()));
    }
  if (m->gather == DG_GATHER_NCCL) {
    if (!nccl().ok) return DG_ERR_NO_NCCL;
    m->comm.assign(m->n, nullptr);
    DG_NCCL(nccl().comm_init_all(m->comm.data(), static_cast<int>(m->n), m->dev.data()));
  }
  for (uint32_t g = 0; g < m->n; ++g) {
    DG_CUDA(cudaSetDevice(m->dev[g]));
    DG_CUDA(cudaDeviceSynchronize());
  }
  return DG_OK;
}

// Create the n shards concurrently (one host thread per shard: planning is host work).
template <class MakeShard>
int create_shards(Multi* m, MakeShard&& make) {
  m->shard.assign(m->n, nullptr);
  std::vector<int> st(m->n, DG_OK);
  std::vector<std::thread> th;
  for (uint32_t g = 0; g < m->n; ++g)
    th.emplace_back([&, g] { st[g] = make(g, &m->shard[g]); });
  for (auto& t : th) t.join();
  for (int s : st) DG_TRY(s);
  return DG_OK;
}

dg_options shard_options(const dg_multi_options* o, const Multi* m, uint32_t g) {
  dg_options so;
  dg_default_options(&so);
  so.device = m->dev[g];
  so.lane_width = o->lane_width;
  so.accumulation = o->accumulation;
  so.row_begin = m->bounds[g];
  so.row_end = m->bounds[g + 1];
  return so;
}

int multi_dose(Multi* m, const double* x, uint64_t x_len, double* y, uint32_t flags) {
  if ((!x && m->cols) || (!y && !(flags & DG_Y_ON_DEVICE) && m->rows)) return DG_ERR_INVALID_CONFIG;
  if (x_len != m->cols) return DG_ERR_DIMENSION_MISMATCH;  // spmv.cpp:34-38
  const bool x_dev = flags & DG_X_ON_DEVICE, y_host = !(flags & DG_Y_ON_DEVICE);
  // 1. x on every device
  for (uint32_t g = 0; g < m->n; ++g) {
    DG_CUDA(cudaSetDevice(m->dev[g]));
    DG_CUDA(cudaEventRecord(m->ev[4 * g], m->stream[g]));
    if (m->cols) {
      if (x_dev)
        DG_CUDA(cudaMemcpyPeerAsync(m->x[g], m->dev[g], x, m->dev[0], m->cols * sizeof(double),
                                    m->stream[g]));
      else
        DG_CUDA(cudaMemcpyAsync(m->x[g], x, m->cols * sizeof(double), cudaMemcpyHostToDevice,
                                m->stream[g]));
    }
    DG_CUDA(cudaEventRecord(m->ev[4 * g + 1], m->stream[g]));
  }
  // 2. every shard's dose, issued back to back (no host sync): the devices run concurrently;
  //    rows land in the shard device's full d at their global row
  //    (host d: each shard's dose also downloads its slice of the caller's d row block by row
  //    block as its tile kernel finishes each block -- over every device's own PCIe link,
  //    overlapped with the later blocks)
  //    Pinned host d only: a copy into pageable memory blocks the host thread until its block is
  //    done, which would serialise the devices' launches -- pageable d is downloaded in step 4.
  bool pinned = false;
  if (y_host && m->rows) {
    cudaPointerAttributes pa{};
    pinned = cudaPointerGetAttributes(&pa, y) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
  }
  for (uint32_t g = 0; g < m->n; ++g) {
    Handle* hg = reinterpret_cast<Handle*>(m->shard[g]);
    hg->host_sink = pinned ? y + m->bounds[g] : nullptr;
    const int st = dg_dose(m->shard[g], m->x[g], m->cols, m->full[g] + m->bounds[g],
                           DG_X_ON_DEVICE | DG_Y_ON_DEVICE | DG_NO_SYNC, m->stream[g]);
    hg->host_sink = nullptr;
    DG_TRY(st);
    DG_CUDA(cudaSetDevice(m->dev[g]));
    DG_CUDA(cudaEventRecord(m->ev[4 * g + 2], m->stream[g]));
  }
  // 3. gather
  if (m->gather == DG_GATHER_PEER) {
    // (the shards' doses above issued their copies: block by block, overlapped with their tiles)
    // device t's full d is complete once every shard's copies into it are: each stream waits
    // for the others' copy-done events before its "gathered" mark
    for (uint32_t g = 0; g < m->n; ++g) {
      DG_CUDA(cudaSetDevice(m->dev[g]));
      DG_CUDA(cudaEventRecord(m->ev[4 * g + 3], m->stream[g]));
    }
    for (uint32_t t = 0; t < m->n; ++t) {
      DG_CUDA(cudaSetDevice(m->dev[t]));
      for (uint32_t g = 0; g < m->n; ++g)
        if (g != t) DG_CUDA(cudaStreamWaitEvent(m->stream[t], m->ev[4 * g + 3], 0));
    }
  } else if (m->gather == DG_GATHER_NCCL) {
    DG_NCCL(nccl().group_start());
    for (uint32_t g = 0; g < m->n; ++g) {
      const uint64_t r0 = m->bounds[g], nr = m->bounds[g + 1] - r0;
      if (!nr) continue;
      for (uint32_t r = 0; r < m->n; ++r) {
        // (in place at the root: its send buffer is its receive range)
        const ncclResult_t e = nccl().broadcast(m->full[r] + r0, m->full[r] + r0, nr, ncclFloat64,
                                                static_cast<int>(g), m->comm[r], m->stream[r]);
        if (e != ncclSuccess) {
          nccl().group_end();
          return DG_ERR_NCCL_BASE + static_cast<int>(e);
        }
      }
    }
    DG_NCCL(nccl().group_end());
  }
  // 4. pageable host d: every device downloads its own slice concurrently (pinned host d was
  //    downloaded block by block by the shards' doses in step 2)
  for (uint32_t g = 0; g < m->n; ++g) {
    DG_CUDA(cudaSetDevice(m->dev[g]));
    const uint64_t r0 = m->bounds[g], nr = m->bounds[g + 1] - r0;
    if (y_host && !pinned && nr)
      DG_CUDA(cudaMemcpyAsync(y + r0, m->full[g] + r0, nr * sizeof(double), cudaMemcpyDeviceToHost,
                              m->stream[g]));
    DG_CUDA(cudaEventRecord(m->ev[4 * g + 3], m->stream[g]));
  }
  for (uint32_t g = 0; g < m->n; ++g) {
    DG_CUDA(cudaSetDevice(m->dev[g]));
    DG_CUDA(cudaStreamSynchronize(m->stream[g]));
  }
  m->timing = true;
  return DG_OK;
}

}  // namespace
}  // namespace dg

using dg::Multi;

extern "C" {

int dg_multi_create(const dg_csr_view* v, const dg_multi_options* o, dg_multi** out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!v || !out) return DG_ERR_INVALID_CONFIG;
  *out = nullptr;
  DG_TRY(dg::check_multi_options(o));
  if (!v->row_ptr) return DG_ERR_VALIDATION_FAILURE;
  if (v->value_precision > DG_DOUBLE || (v->index_bytes != 2 && v->index_bytes != 4))
    return DG_ERR_INVALID_CONFIG;
  // nnz-balanced shard bounds from the row pointers (host copy when the view is on a device)
  std::vector<uint64_t> rp(v->rows + 1);
  if (v->on_device) {
    DG_CUDA(cudaSetDevice(o->devices[0]));
    DG_CUDA(cudaMemcpy(rp.data(), v->row_ptr, rp.size() * 8, cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(rp.data(), v->row_ptr, rp.size() * 8);
  }
  for (uint64_t r = 0; r < v->rows; ++r)
    if (rp[r + 1] < rp[r]) return DG_ERR_VALIDATION_FAILURE;  // sparse.cpp:222-227
  Multi* m = new (std::nothrow) Multi();
  if (!m) return DG_ERR_OUT_OF_MEMORY;
  m->n = o->n_devices;
  m->gather = o->gather;
  m->rows = v->rows;
  m->cols = v->cols;
  m->dev.assign(o->devices, o->devices + m->n);
  m->bounds.assign(m->n + 1, 0);
  const uint32_t vb = v->value_precision == DG_HALF ? 2 : v->value_precision == DG_SINGLE ? 4 : 8;
  int st = dg_partition_rows(rp.data(), v->rows, vb + v->index_bytes, m->n, m->bounds.data());
  if (st == DG_OK)
    st = dg::create_shards(m, [&](uint32_t g, dg_handle** h) {
      const dg_options so = dg::shard_options(o, m, g);
      return dg_create(v, &so, h);
    });
  if (st == DG_OK) st = dg::finish_multi(m);
  if (st != DG_OK) {
    dg::destroy_multi(m);
    return st;
  }
  *out = reinterpret_cast<dg_multi*>(m);
  return DG_OK;
}

int dg_multi_create_generated(const dg_profile* beams, uint32_t n_beams, uint32_t index_bytes,
                              const dg_multi_options* o, dg_multi** out) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!beams || !out || n_beams == 0) return DG_ERR_INVALID_CONFIG;
  *out = nullptr;
  DG_TRY(dg::check_multi_options(o));
  const uint64_t rows = beams[0].rows;
  uint64_t cols = 0;
  for (uint32_t b = 0; b < n_beams; ++b) cols += beams[b].cols;
  std::vector<uint32_t> lens(rows);
  DG_TRY(dg_generated_row_lengths(beams, n_beams, 0, rows, o->devices[0], lens.data()));
  Multi* m = new (std::nothrow) Multi();
  if (!m) return DG_ERR_OUT_OF_MEMORY;
  m->n = o->n_devices;
  m->gather = o->gather;
  m->rows = rows;
  m->cols = cols;
  m->dev.assign(o->devices, o->devices + m->n);
  m->bounds.assign(m->n + 1, 0);
  const uint32_t ib = index_bytes ? index_bytes : (cols < 65536 ? 2 : 4);
  int st = dg_partition_lengths(lens.data(), rows, 2 + ib, m->n, m->bounds.data());
  if (st == DG_OK)
    st = dg::create_shards(m, [&](uint32_t g, dg_handle** h) {
      const dg_options so = dg::shard_options(o, m, g);
      return dg_create_generated(beams, n_beams, index_bytes, &so, h);
    });
  if (st == DG_OK) st = dg::finish_multi(m);
  if (st != DG_OK) {
    dg::destroy_multi(m);
    return st;
  }
  *out = reinterpret_cast<dg_multi*>(m);
  return DG_OK;
}

int dg_multi_dose(dg_multi* mm, const double* x, uint64_t x_len, double* y, uint32_t flags) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  Multi* m = reinterpret_cast<Multi*>(mm);
  if (!m) return DG_ERR_INVALID_CONFIG;
  return dg::multi_dose(m, x, x_len, y, flags);
}

int dg_multi_bounds(const dg_multi* mm, uint32_t* n_shards, uint64_t* bounds) {
  const Multi* m = reinterpret_cast<const Multi*>(mm);
  if (!m || !n_shards) return DG_ERR_INVALID_CONFIG;
  *n_shards = m->n;
  if (bounds) std::copy(m->bounds.begin(), m->bounds.end(), bounds);
  return DG_OK;
}

int dg_multi_shard(const dg_multi* mm, uint32_t i, dg_handle** shard) {
  const Multi* m = reinterpret_cast<const Multi*>(mm);
  if (!m || !shard || i >= m->n) return DG_ERR_INVALID_CONFIG;
  *shard = m->shard[i];
  return DG_OK;
}

int dg_multi_device_d(const dg_multi* mm, uint32_t i, double** full_d, double** slice_d) {
  const Multi* m = reinterpret_cast<const Multi*>(mm);
  if (!m || i >= m->n) return DG_ERR_INVALID_CONFIG;
  if (full_d) *full_d = m->full[i];
  if (slice_d) *slice_d = m->full[i] + m->bounds[i];
  return DG_OK;
}

int dg_multi_last_timing(const dg_multi* mm, dg_timing* t) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  const Multi* m = reinterpret_cast<const Multi*>(mm);
  if (!m || !t) return DG_ERR_INVALID_CONFIG;
  *t = dg_timing{};
  if (!m->timing) return DG_OK;
  for (uint32_t g = 0; g < m->n; ++g) {
    DG_CUDA(cudaSetDevice(m->dev[g]));
    float a = 0, b = 0, c = 0, tot = 0;
    const cudaEvent_t* e = &m->ev[4 * g];
    DG_CUDA(cudaEventElapsedTime(&a, e[0], e[1]));
    DG_CUDA(cudaEventElapsedTime(&b, e[1], e[2]));
    DG_CUDA(cudaEventElapsedTime(&c, e[2], e[3]));
    DG_CUDA(cudaEventElapsedTime(&tot, e[0], e[3]));
    t->ms_h2d = std::max(t->ms_h2d, a);
    t->ms_kernels = std::max(t->ms_kernels, b);
    t->ms_d2h = std::max(t->ms_d2h, c);
    t->ms_total = std::max(t->ms_total, tot);
  }
  return DG_OK;
}

int dg_multi_destroy(dg_multi* mm) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  dg::destroy_multi(reinterpret_cast<Multi*>(mm));
  return DG_OK;
}

}  // extern "C"
