// Microbenchmark for the heap-tier numeric design (diagnostic only):
//   mode 0: __match_any_sync throughput (per-lane random 32-bit keys)
//   mode 1: ordered rounds of global RMW (ld, add, st) on random positions of a
//           per-warp 8 KB region (all warps: 38 MB, L2-resident), __syncwarp between rounds
//   mode 2: mode 1 with U=4 rounds' loads issued before the ordered updates
//   mode 3: same rounds as mode 1 but the values live in shared memory (4 KB/warp)
// Prints ns per round per warp-resident and rounds/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* region, unsigned* out, int rounds) {
  __shared__ double sv[8][512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + warp;
  double* v = region + static_cast<size_t>(gw) * 1024;  // 8 KB per warp: 38 MB total, L2-resident
  unsigned x = (gw * 32 + lane) * 2654435761u + 12345u, acc = 0;
  for (int r = 0; r < rounds; ++r) {
    x = x * 1664525u + 1013904223u;
    if (MODE == 0) {
      acc += __match_any_sync(0xffffffffu, (x >> 20) & 63);
    } else if (MODE == 1) {
      const unsigned p = (x >> 8) & 1023;
      v[p] = v[p] + 1.0;
      __syncwarp();
    } else if (MODE == 2) {
      if ((r & 3) == 0) {
        unsigned p[4];
        double o[4];
        unsigned y = x;
#pragma unroll
        for (int u = 0; u < 4; ++u) { y = y * 1664525u + 1013904223u; p[u] = (y >> 8) & 1023; o[u] = v[p[u]]; }
#pragma unroll
        for (int u = 0; u < 4; ++u) { v[p[u]] = o[u] + 1.0; __syncwarp(); }
      }
    } else {
      const unsigned p = (x >> 8) & 511;
      sv[warp & 7][p] = sv[warp & 7][p] + 1.0;
      __syncwarp();
    }
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int threads = 256, blocks = sms * 4, rounds = 4096;
  double* region;
  unsigned* out;
  cudaMalloc(&region, static_cast<size_t>(blocks) * 8 * 65536 * 8);
  cudaMemset(region, 0, static_cast<size_t>(blocks) * 8 * 65536 * 8);
  cudaMalloc(&out, 4);
  const char* names[] = {"match_any", "global RMW + syncwarp", "global RMW U=4 batched", "smem RMW + syncwarp"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (m) {
        case 0: k<0><<<blocks, threads>>>(region, out, rounds); break;
        case 1: k<1><<<blocks, threads>>>(region, out, rounds); break;
        case 2: k<2><<<blocks, threads>>>(region, out, rounds); break;
        case 3: k<3><<<blocks, threads>>>(region, out, rounds); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double warps = double(blocks) * threads / 32;
      if (rep)
        printf("%-26s %8.3f ms  %.3f warp-rounds/clk/SM  %.0f cycles/round/warp (32 warps/SM)\n", names[m], ms,
               warps * rounds / (ms * 1e-3) / sms / (clk * 1e3), (ms * 1e-3) * clk * 1e3 / rounds);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
