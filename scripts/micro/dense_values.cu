// Microbenchmark: dense (contiguous-column) rows streamed as values only (2 B per nonzero, the
// column of position p is lo + p) vs the slice stream's (slot << 16 | half) words (4 B), both with
// x gathered through L1 from global memory (exact family: fp64 x, F2F + DMUL + DADD per element,
// lane l owns positions l, l + 32, ...).  C2-like rows: contiguous, 4,096 .. 40,000 long.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dense_values scripts/micro/dense_values.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ double h2d(uint32_t bits16) {
  double d;
  asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(static_cast<unsigned short>(bits16)));
  return d;
}

struct Row {
  uint64_t off;   // first 16-byte unit of the row's stream (values: 8-chunk blocks; words: 4-chunk)
  uint32_t lo;    // first column
  uint32_t len;
};

// values: lane-major 8-chunk blocks (512 B: lane l's 16 B = its 8 halves); batch = 2 blocks
// AL: x read from the row's 32-element-aligned base (lo & ~31) -- the traffic of a lane grid
// rotated by lo mod 32 (each chunk's 32 x elements in 2 aligned 128-B lines instead of 3)
template <int P, bool AL = false>
__global__ void __launch_bounds__(256) k_values(const uint4* __restrict__ s, const Row* __restrict__ rows,
                                                uint32_t n_rows, const double* __restrict__ x,
                                                uint32_t zero_col, uint32_t* counter, double* y) {
  const uint32_t lane = threadIdx.x & 31;
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(counter, 1u);
    k = __shfl_sync(~0u, k, 0);
    if (k >= n_rows) break;
    const Row R = rows[k];
    const uint32_t nch = (R.len + 31) / 32, nblk = (nch + 7) / 8;
    const uint4* p = s + R.off + lane;
    double acc = 0;
    const uint32_t nb = (nblk + 1) / 2;
    uint4 a0 = ld16(p), a1 = nblk > 1 ? ld16(p + 32) : make_uint4(0, 0, 0, 0), b0, b1;
    for (int j = 1; j <= P; ++j)
      if (lane < 8 && 2 * j + (lane >= 4) < nblk) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(p - lane + 64 * j) + 128 * lane));
    for (uint32_t bi = 0; bi < nb; ++bi) {
      if (bi + 1 < nb) {
        b0 = ld16(p + 64);
        b1 = 2 * bi + 3 < nblk ? ld16(p + 96) : make_uint4(0, 0, 0, 0);
      }
      if (P > 0 && lane < 8 && 2 * (bi + 1 + P) + (lane >= 4) < nblk)
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(p - lane + 64 * (1 + P)) + 128 * lane));
      const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const uint32_t pos0 = bi * 512 + lane;  // chunk 16 bi, this lane
      if (pos0 + 15 * 32 < R.len) {  // interior batch: all 16 positions inside the row
        double xv[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) xv[c] = __ldg(x + (AL ? R.lo & ~31u : R.lo) + pos0 + 32 * c);
#pragma unroll
        for (int c = 0; c < 16; ++c) acc = __dadd_rn(acc, __dmul_rn(h2d(w[c / 2] >> (16 * (c & 1))), xv[c]));
      } else {
        double xv[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const uint32_t pos = pos0 + 32 * c;
          xv[c] = __ldg(x + (pos < R.len ? (AL ? R.lo & ~31u : R.lo) + pos : zero_col));
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) acc = __dadd_rn(acc, __dmul_rn(h2d(w[c / 2] >> (16 * (c & 1))), xv[c]));
      }
      a0 = b0;
      a1 = b1;
      p += 64;
    }
#pragma unroll
    for (int o = 16; o; o /= 2) acc = __dadd_rn(acc, __shfl_down_sync(~0u, acc, o));
    if (lane == 0) y[k] = acc;
  }
}

// words: lane-major 4-chunk blocks (512 B: lane l's 16 B = its 4 words), word = col << 16 | half
// (x indexed by the word's column); batch = 2 blocks = 8 chunks
template <int P>
__global__ void __launch_bounds__(256) k_words(const uint4* __restrict__ s, const Row* __restrict__ rows,
                                               uint32_t n_rows, const double* __restrict__ x,
                                               uint32_t* counter, double* y) {
  const uint32_t lane = threadIdx.x & 31;
  for (;;) {
    uint32_t k = 0;
    if (lane == 0) k = atomicAdd(counter, 1u);
    k = __shfl_sync(~0u, k, 0);
    if (k >= n_rows) break;
    const Row R = rows[k];
    const uint32_t nch = (R.len + 31) / 32, nblk = (nch + 3) / 4;
    const uint4* p = s + R.off + lane;
    double acc = 0;
    const uint32_t nb = (nblk + 1) / 2;
    uint4 a0 = ld16(p), a1 = nblk > 1 ? ld16(p + 32) : make_uint4(0, 0, 0, 0), b0, b1;
    for (int j = 1; j <= P; ++j)
      if (lane < 8 && 2 * j + (lane >= 4) < nblk) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(p - lane + 64 * j) + 128 * lane));
    for (uint32_t bi = 0; bi < nb; ++bi) {
      if (bi + 1 < nb) {
        b0 = ld16(p + 64);
        b1 = 2 * bi + 3 < nblk ? ld16(p + 96) : make_uint4(0, 0, 0, 0);
      }
      if (P > 0 && lane < 8 && 2 * (bi + 1 + P) + (lane >= 4) < nblk)
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(p - lane + 64 * (1 + P)) + 128 * lane));
      const uint32_t w[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      double xv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) xv[c] = __ldg(x + (w[c] >> 16));
#pragma unroll
      for (int c = 0; c < 8; ++c) acc = __dadd_rn(acc, __dmul_rn(h2d(w[c] & 0xFFFF), xv[c]));
      a0 = b0;
      a1 = b1;
      p += 64;
    }
#pragma unroll
    for (int o = 16; o; o /= 2) acc = __dadd_rn(acc, __shfl_down_sync(~0u, acc, o));
    if (lane == 0) y[k] = acc;
  }
}

// word stream of the rows: chunk c, lane l of a row holds column lo + 32 c + l (or a padding word)
__global__ void k_fill_words(uint32_t* s, const Row* rows, uint32_t n_rows) {
  const Row R = rows[blockIdx.x];
  const uint32_t nch = (R.len + 31) / 32, nblk = (nch + 3) / 4;
  for (uint32_t i = threadIdx.x; i < nblk * 128; i += blockDim.x) {
    const uint32_t blk = i / 128, l = (i % 128) / 4, c = blk * 4 + i % 4;
    const uint32_t pos = 32 * c + l;
    s[R.off * 4 + i] = pos < R.len ? ((R.lo + pos) << 16) | 0x3800u : (40000u << 16);
  }
}

int main(int argc, char** argv) {
  const uint32_t cols = 40000;
  // argv[1]: max row length (default 40000); argv[2]: columns the rows' starts are spread over
  // (default: all) -- a narrow spread is a small x footprint per SM (L1 locality experiment)
  const uint32_t max_len = argc > 1 ? (uint32_t)atoi(argv[1]) : 40000;
  const uint32_t lo_span = argc > 2 ? (uint32_t)atoi(argv[2]) : 0;
  // C2's dense rows: ~1.34e9 nonzeros in rows of 4,096 .. 40,000 (longest first, as k_dense pulls)
  std::vector<Row> rows;
  std::vector<uint32_t> lens;
  uint64_t nnz = 0;
  srand(1);
  while (nnz < 1340000000ull) {
    const double u = rand() / (double)RAND_MAX;
    uint32_t len = (uint32_t)(4096 * __builtin_pow(max_len / 4096.0, u * u));
    lens.push_back(len);
    nnz += len;
  }
  std::sort(lens.begin(), lens.end(), [](uint32_t a, uint32_t b) { return a > b; });
  uint64_t off_v = 0, off_w = 0;
  std::vector<Row> rv, rw;
  for (uint32_t len : lens) {
    const uint32_t room = lo_span ? std::min(lo_span, cols - len + 1) : cols - len + 1;
    const uint32_t lo = rand() % room;
    const uint32_t nch = (len + 31) / 32;
    rv.push_back({off_v, lo, len});
    rw.push_back({off_w, lo, len});
    off_v += (nch + 7) / 8 * 32;  // 16-byte units: 8-chunk block = 32 units
    off_w += (nch + 3) / 4 * 32;
  }
  printf("rows %zu nnz %llu values %.2f GB words %.2f GB\n", lens.size(), (unsigned long long)nnz,
         off_v * 16 / 1e9, off_w * 16 / 1e9);
  uint4 *sv, *sw;
  cudaMalloc(&sv, off_v * 16 + 4096);
  cudaMalloc(&sw, off_w * 16 + 4096);
  // values: halves in [0.5, 1); words: column = lo + position (all positions valid for timing)
  cudaMemset(sv, 0x38, off_v * 16);
  Row *drv, *drw;
  cudaMalloc(&drv, rv.size() * sizeof(Row));
  cudaMalloc(&drw, rw.size() * sizeof(Row));
  cudaMemcpy(drv, rv.data(), rv.size() * sizeof(Row), cudaMemcpyHostToDevice);
  cudaMemcpy(drw, rw.data(), rw.size() * sizeof(Row), cudaMemcpyHostToDevice);
  k_fill_words<<<(unsigned)rw.size(), 256>>>((uint32_t*)sw, drw, (uint32_t)rw.size());
  cudaDeviceSynchronize();
  double *x, *y;
  cudaMalloc(&x, (cols + 1) * 8);
  cudaMemset(x, 0, (cols + 1) * 8);
  cudaMalloc(&y, lens.size() * 8);
  uint32_t* cnt;
  cudaMalloc(&cnt, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, auto launch, double bytes) {
    float best = 1e30f;
    for (int it = 0; it < 8; ++it) {
      cudaMemset(cnt, 0, 4);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it > 1 && ms < best) best = ms;
    }
    printf("%-34s %8.3f ms  %6.2f Gnnz/s  stream %7.1f GB/s  model(4 B/nnz) %7.1f GB/s  %s\n", name, best,
           nnz / best / 1e6, bytes / best / 1e6, nnz * 4.0 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  const uint32_t n = (uint32_t)lens.size();
  for (int g : {4}) {
    char nm[64];
    snprintf(nm, sizeof nm, "words (4 B) P4 grid %dxSM", g);
    time(nm, [&] { k_words<4><<<g * sms, 256>>>(sw, drw, n, x, cnt, y); }, off_w * 16.0);
    snprintf(nm, sizeof nm, "values (2 B) P2 grid %dxSM", g);
    time(nm, [&] { k_values<2><<<g * sms, 256>>>(sv, drv, n, x, cols, cnt, y); }, off_v * 16.0);
    snprintf(nm, sizeof nm, "values (2 B) P4 grid %dxSM", g);
    time(nm, [&] { k_values<4><<<g * sms, 256>>>(sv, drv, n, x, cols, cnt, y); }, off_v * 16.0);
    snprintf(nm, sizeof nm, "values aligned-x P2 grid %dxSM", g);
    time(nm, [&] { k_values<2, true><<<g * sms, 256>>>(sv, drv, n, x, cols, cnt, y); }, off_v * 16.0);
    snprintf(nm, sizeof nm, "values (2 B) P2 grid %dxSM", g);
    time(nm, [&] { k_values<2><<<g * sms, 256>>>(sv, drv, n, x, cols, cnt, y); }, off_v * 16.0);
    snprintf(nm, sizeof nm, "values aligned-x P2 grid %dxSM", g);
    time(nm, [&] { k_values<2, true><<<g * sms, 256>>>(sv, drv, n, x, cols, cnt, y); }, off_v * 16.0);
  }
  return 0;
}
