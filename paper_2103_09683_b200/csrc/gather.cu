// gather.cu -- fused d gather targets and the CUDA IPC plumbing behind them.
//
// One process per GPU: each rank allocates its full-d buffer with dg_ipc_alloc, the 64-byte IPC
// handles are exchanged by the host (torch.distributed all_gather_object), every rank opens its
// peers' buffers with dg_ipc_open (peer mappings over NVLink / NVSwitch), and hands the list --
// its own buffer included -- to dg_set_gather_targets.  From then on each dg_dose writes its
// rows into every rank's full d from inside the dose kernels (spmv_kernels.cuh / spmv_tiles.cuh
// epilogues), so the "all-gather" overlaps the SpMV instead of following it.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "common.cuh"
#include "handle.cuh"

extern "C" {

int dg_set_gather_targets(dg_handle* hh, double* const* targets, uint32_t n) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  dg::Handle* h = reinterpret_cast<dg::Handle*>(hh);
  if (!h) return DG_ERR_INVALID_CONFIG;
  if (n > dg::kMaxGatherTargets || (n && !targets)) return DG_ERR_INVALID_CONFIG;
  dg::GatherTargets gt{};
  for (uint32_t i = 0; i < n; ++i) {
    if (!targets[i]) return DG_ERR_INVALID_CONFIG;
    gt.t[i] = targets[i];
  }
  gt.n = n;
  gt.row_off = h->row_begin;
  h->gt = gt;
  h->gt_zeroed = false;  // the next dose zero-fills this shard's rows of the new targets
  return DG_OK;
}

int dg_set_block_targets(dg_handle* hh, double* const* targets, uint32_t n) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  dg::Handle* h = reinterpret_cast<dg::Handle*>(hh);
  if (!h) return DG_ERR_INVALID_CONFIG;
  if (n > dg::kMaxGatherTargets || (n && !targets)) return DG_ERR_INVALID_CONFIG;
  std::vector<const double*> dst(n);
  std::vector<int> dev(n, -1);  // UVA copies (IPC mappings, own device)
  for (uint32_t i = 0; i < n; ++i) {
    if (!targets[i]) return DG_ERR_INVALID_CONFIG;
    dst[i] = targets[i] + h->row_begin;
  }
  dg::set_block_sinks(h, dst.data(), dev.data(), n);
  return DG_OK;
}

int dg_ipc_alloc(uint64_t bytes, int32_t device, void** dptr, void* handle64) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!dptr || !handle64) return DG_ERR_INVALID_CONFIG;
  int dev = 0;
  DG_TRY(dg::select_device(device, &dev));
  DG_CUDA(cudaMalloc(dptr, bytes ? bytes : 1));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, *dptr);
  if (e != cudaSuccess) {
    cudaFree(*dptr);
    *dptr = nullptr;
    return DG_ERR_CUDA_BASE + static_cast<int>(e);
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  std::memcpy(handle64, &h, 64);
  return DG_OK;
}

int dg_ipc_open(const void* handle64, int32_t device, void** dptr) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  if (!handle64 || !dptr) return DG_ERR_INVALID_CONFIG;
  int dev = 0;
  DG_TRY(dg::select_device(device, &dev));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  DG_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return DG_OK;
}

int dg_ipc_close(void* dptr) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  DG_CUDA(cudaIpcCloseMemHandle(dptr));
  return DG_OK;
}

int dg_ipc_free(void* dptr) {
  dg::DeviceGuard device_guard;  // the caller's current device is restored on return
  DG_CUDA(cudaFree(dptr));
  return DG_OK;
}

}  // extern "C"
