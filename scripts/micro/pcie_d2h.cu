// PCIe micro-benchmark behind the host-path dose order (scripts/micro, not product code):
//   1. 64 MB pinned D2H in 16 blocks on one / two copy streams, idle GPU;
//   2. the same beside an HBM-bound read kernel (~1.5 ms);
//   3. a scattered zero-copy "patch": n 8-byte stores into pinned host memory at a given row
//      stride (C2's contiguous rows: ~157K rows, ~51 rows apart), one thread per row.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pcie_d2h pcie_d2h.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_read(const uint4* p, size_t n, unsigned long long* sink) {
  uint4 acc = {0, 0, 0, 0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void k_patch(const double* src, const uint32_t* rows, uint32_t n, double* host) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) host[rows[i]] = src[rows[i]];
}

int main() {
  const size_t rows = 8000000, bytes = rows * 8;
  double *d, *h;
  CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(d, 0, bytes));
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
  const size_t big = 12ull << 30;  // 12 GB read by the HBM kernel
  uint4* a;
  CK(cudaMalloc(&a, big));
  CK(cudaMemset(a, 1, big));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  cudaStream_t s0, c[2];
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  for (auto& x : c) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, k1, cd[2];
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&k1);
  for (auto& x : cd) cudaEventCreate(&x);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto d2h = [&](int ns, bool with_kernel, size_t kbytes) -> float {
    float best = 1e9f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0, s0);
      for (int i = 0; i < ns; ++i) cudaStreamWaitEvent(c[i], e0, 0);
      if (with_kernel) k_read<<<sms * 8, 512, 0, s0>>>(a, kbytes / 16, sink);
      cudaEventRecord(k1, s0);
      const size_t blk = bytes / 16;
      for (int k = 0; k < 16; ++k)
        cudaMemcpyAsync((char*)h + k * blk, (char*)d + k * blk, blk, cudaMemcpyDeviceToHost, c[k % ns]);
      for (int i = 0; i < ns; ++i) { cudaEventRecord(cd[i], c[i]); cudaStreamWaitEvent(s0, cd[i], 0); }
      cudaEventRecord(e1, s0);
      cudaEventSynchronize(e1);
      float ms = 0, kms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventElapsedTime(&kms, e0, k1);
      if (rep) best = ms < best ? ms : best;
      if (rep == 5 && with_kernel) printf("   (kernel alone in that run: %.3f ms)\n", kms);
    }
    return best;
  };
  for (int ns = 1; ns <= 2; ++ns) {
    float ms = d2h(ns, false, 0);
    printf("D2H 64 MB, %d stream(s), idle GPU: %.3f ms = %.1f GB/s\n", ns, ms, bytes / ms / 1e6);
  }
  for (int ns = 1; ns <= 2; ++ns) {
    float ms = d2h(ns, true, 10ull << 30);
    printf("D2H 64 MB, %d stream(s), beside a 10-GB read kernel: %.3f ms total\n", ns, ms);
  }
  {  // kernel alone
    float best = 1e9f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0, s0);
      k_read<<<sms * 8, 512, 0, s0>>>(a, (10ull << 30) / 16, sink);
      cudaEventRecord(e1, s0);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) best = ms < best ? ms : best;
    }
    printf("read kernel alone (10 GB): %.3f ms = %.1f GB/s\n", best, (10ull << 30) / best / 1e6);
  }
  for (uint32_t stride : {51u, 8u, 1u}) {
    const uint32_t n = 157000;
    std::vector<uint32_t> r(n);
    for (uint32_t i = 0; i < n; ++i) r[i] = (uint32_t)(((uint64_t)i * stride + (i * 2654435761u) % (stride ? stride : 1)) % rows);
    uint32_t* dr;
    CK(cudaMalloc(&dr, n * 4));
    CK(cudaMemcpy(dr, r.data(), n * 4, cudaMemcpyHostToDevice));
    double* hp;
    CK(cudaHostGetDevicePointer(&hp, h, 0));
    float best = 1e9f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0, s0);
      k_patch<<<(n + 255) / 256, 256, 0, s0>>>(d, dr, n, hp);
      cudaEventRecord(e1, s0);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep) best = ms < best ? ms : best;
    }
    printf("zero-copy patch: %u rows, stride ~%u rows: %.4f ms (host ptr == device ptr: %d)\n", n, stride, best, hp == h);
    cudaFree(dr);
  }
  CK(cudaGetLastError());
  return 0;
}
