// Microbenchmark: how fast can ONE warp stream a contiguous run (a long row of the slice stream)?
// The dose kernels consume a run in 1-KB batches (two LDG.128 per lane); a run's time is set by
// the bytes a warp keeps in flight.  Variants: D register batches in flight (1 = the kernels'
// double buffer), an L2 prefetch stream P batches ahead (one line per lane 0..7), and a bulk L2
// prefetch (cp.async.bulk.prefetch.L2) of the next K KB issued every 8 batches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_rate scripts/micro/stream_rate.cu
//   /tmp/stream_rate
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t mix(uint32_t a, const uint4& q) {
  // ~ the per-batch arithmetic of the dose kernel (8 words): keep it a dependent chain
  a = a * 3u + q.x; a = a * 3u + q.y; a = a * 3u + q.z; a = a * 3u + q.w;
  return a;
}

// run of nb batches (1 KB each) at base; D in {1, 2, 3}; P: L2 line prefetch distance (batches);
// BULK: KB prefetched by cp.async.bulk.prefetch.L2 every 8 batches, BULK KB ahead
template <int D, int P, int BULK>
__global__ void k_stream(const uint4* __restrict__ buf, uint64_t run_batches, uint32_t runs_per_warp,
                         uint32_t* out, unsigned long long* cyc) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (blockDim.x / 32)) + threadIdx.x / 32;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (uint32_t r = 0; r < runs_per_warp; ++r) {
    const uint4* p = buf + (warp * runs_per_warp + r) * run_batches * 64 + lane;
    const uint64_t nb = run_batches;
    if (BULK && lane == 0) {
      const uint32_t first = (uint32_t)(nb * 1024 < BULK * 1024u ? nb * 1024 : BULK * 1024u);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(first) : "memory");
    }
    if (P > 0)
      for (int k = 1; k <= P; ++k)
        if (lane < 8 && k < (int)nb) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(p - lane + 64 * k) + 128 * lane));
    uint4 q[D][2];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      q[d][0] = d < (int)nb ? ld16(p + 64 * d) : make_uint4(0, 0, 0, 0);
      q[d][1] = d < (int)nb ? ld16(p + 64 * d + 32) : make_uint4(0, 0, 0, 0);
    }
    for (uint64_t b = 0; b < nb; b += D) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const uint64_t bb = b + d;
        if (bb >= nb) break;
        const uint4 c0 = q[d][0], c1 = q[d][1];
        if (bb + D < nb) {
          q[d][0] = ld16(p + 64 * (bb + D));
          q[d][1] = ld16(p + 64 * (bb + D) + 32);
        }
        if (P > 0 && lane < 8 && bb + D + P < nb)
          asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(p - lane + 64 * (bb + D + P)) + 128 * lane));
        if (BULK && lane == 0 && (bb & 7) == 0 && bb + BULK < nb) {
          const uint64_t s = bb + BULK;  // batches (KB) ahead
          const uint32_t len = (uint32_t)(nb - s < 8 ? nb - s : 8) * 1024u;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p - lane + 64 * s), "r"(len) : "memory");
        }
        acc = mix(acc, c0);
        acc = mix(acc, c1);
      }
    }
  }
  const long long t1 = clock64();
  if (acc == 0x12345678u) out[0] = acc;
  if (lane == 0) atomicMax(cyc, (unsigned long long)(t1 - t0));
}

template <int D, int P, int BULK>
void run(const char* name, const uint4* buf, int warps_per_sm, int sms, uint64_t run_kb, uint32_t runs_per_warp,
         uint32_t* out, unsigned long long* cyc) {
  const int block = 32 * warps_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int it = 0; it < 5; ++it) {
    cudaMemset(cyc, 0, 8);
    // a fresh 1-GB region every repetition: no run starts in L2
    cudaEventRecord(a);
    k_stream<D, P, BULK><<<sms, block>>>(buf + (size_t)it * (1ull << 30) / 16, run_kb, runs_per_warp, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double bytes = (double)sms * warps_per_sm * runs_per_warp * run_kb * 1024.0;
  printf("%-28s warps/SM %2d run %4llu KB: %8.1f us  %7.1f GB/s total  %6.2f GB/s per warp\n", name, warps_per_sm,
         (unsigned long long)run_kb, best * 1e3, bytes / best / 1e6,
         (double)runs_per_warp * run_kb * 1024.0 / best / 1e6);
  cudaError_t e = cudaGetLastError();
  if (e) printf("error %s\n", cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 6ull << 30;
  uint4* buf;
  if (cudaMalloc(&buf, bytes)) return 1;
  cudaMemset(buf, 1, bytes);
  uint32_t* out;
  unsigned long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 8);
  // lone warps: 1 warp per SM, a 160-KB run (C2's longest dense row: 40,000 nonzeros x 4 B)
  for (int w : {1, 4}) {
    run<1, 0, 0>("D1 P0", buf, w, sms, 160, 1, out, cyc);
    run<1, 4, 0>("D1 P4 (k_dense)", buf, w, sms, 160, 1, out, cyc);
    run<1, 2, 0>("D1 P2 (k_slices)", buf, w, sms, 160, 1, out, cyc);
    run<2, 4, 0>("D2 P4", buf, w, sms, 160, 1, out, cyc);
    run<3, 4, 0>("D3 P4", buf, w, sms, 160, 1, out, cyc);
    run<1, 0, 16>("D1 bulk16", buf, w, sms, 160, 1, out, cyc);
    run<1, 0, 32>("D1 bulk32", buf, w, sms, 160, 1, out, cyc);
    run<1, 4, 32>("D1 P4 bulk32", buf, w, sms, 160, 1, out, cyc);
    run<2, 4, 32>("D2 P4 bulk32", buf, w, sms, 160, 1, out, cyc);
    run<2, 0, 64>("D2 bulk64", buf, w, sms, 160, 1, out, cyc);
  }
  // throughput: 32 warps per SM, each 4 runs of 40 KB (the whole machine busy)
  for (int w : {16, 32}) {
    run<1, 2, 0>("D1 P2 (k_slices)", buf, w, sms, 40, 4, out, cyc);
    run<1, 4, 0>("D1 P4", buf, w, sms, 40, 4, out, cyc);
    run<2, 2, 0>("D2 P2", buf, w, sms, 40, 4, out, cyc);
    run<1, 0, 16>("D1 bulk16", buf, w, sms, 40, 4, out, cyc);
    run<1, 2, 16>("D1 P2 bulk16", buf, w, sms, 40, 4, out, cyc);
    run<2, 0, 16>("D2 bulk16", buf, w, sms, 40, 4, out, cyc);
  }
  return 0;
}
