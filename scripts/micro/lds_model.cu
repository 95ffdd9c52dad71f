// Microbenchmark: how many shared-memory wavefronts does one LDS.64 (32 lanes, 8-byte words) cost
// for a given bank-pair pattern?  Throughput-bound (32 warps/SM, independent loads): SM cycles per
// warp-instruction ~= wavefronts per instruction.  Decides the bank model used by the replica
// assignment in plan.cu (half-warp phases vs whole-warp scheduling).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_lds(const int* __restrict__ pat, int iters, double* out, long long* cyc) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int a = pat[lane];
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    double v0, v1, v2, v3;
    const unsigned addr = (unsigned)(__cvta_generic_to_shared(s) + a * 8) + ((it & 1) ? 4096u : 0u);
    asm volatile("ld.shared.f64 %0, [%4];\n\tld.shared.f64 %1, [%4+8192];\n\t"
                 "ld.shared.f64 %2, [%4+16384];\n\tld.shared.f64 %3, [%4+24576];"
                 : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3) : "r"(addr) : "memory");
    acc += v0 + v1 + v2 + v3;
  }
  long long t1 = clock64();
  if (acc == -1.0) out[0] = acc;
  if (lane == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

int main() {
  // patterns: element index per lane (bank pair = index % 16); all indices < 1024
  std::vector<std::pair<const char*, std::vector<int>>> pats;
  std::vector<int> p(32);
  for (int l = 0; l < 32; ++l) p[l] = l;                                     pats.push_back({"consecutive (ideal 2)", p});
  for (int l = 0; l < 32; ++l) p[l] = (l % 16) + 16 * (l / 16);               pats.push_back({"halves distinct, same banks (2 either)", p});
  for (int l = 0; l < 32; ++l) p[l] = 0;                                      pats.push_back({"broadcast", p});
  for (int l = 0; l < 16; ++l) p[l] = (l / 2) + 16 * (l % 2);
  for (int l = 16; l < 32; ++l) p[l] = 8 + ((l - 16) / 2) + 16 * (l % 2);   pats.push_back({"D2: half 2-way, whole 2 (half model 4, whole 2)", p});
  for (int l = 0; l < 32; ++l) p[l] = 16 * l;                                 pats.push_back({"all bank pair 0 (32-way)", p});
  for (int l = 0; l < 32; ++l) p[l] = (l < 16) ? 16 * l : (l - 16) + 1;        pats.push_back({"half0 16-way on bp0, half1 distinct bp1..16", p});
  for (int l = 0; l < 32; ++l) p[l] = (l % 2) ? 16 * l : l;                    pats.push_back({"odd lanes bp0 (16-way), even distinct", p});
  for (int l = 0; l < 32; ++l) p[l] = 2 * l;                                  pats.push_back({"stride 2 doubles (bp even only)", p});
  for (int l = 0; l < 32; ++l) p[l] = (l / 2) * 16 + (l % 2);                 pats.push_back({"pairs: lanes 2k,2k+1 adjacent words, 16-way over pairs", p});
  int* d_pat; double* d_out; long long* d_cyc;
  cudaMalloc(&d_pat, 32 * 4); cudaMalloc(&d_out, 8); cudaMalloc(&d_cyc, 8);
  const int iters = 200, warps = 4;
  for (auto& [name, v] : pats) {
    cudaMemcpy(d_pat, v.data(), 32 * 4, cudaMemcpyHostToDevice);
    cudaMemset(d_cyc, 0, 8);
    k_lds<<<1, warps * 32>>>(d_pat, iters, d_out, d_cyc);
    long long c = 0;
    cudaError_t e = cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    printf("%-60s cycles per LDS.64 per SM: %.2f\n", name, double(c) / (iters * 4.0 * warps));
  }
  return 0;
}
