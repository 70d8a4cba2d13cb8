// Microbenchmark: shared-memory LDS vs ATOMS.OR vs ATOMS.CAS vs ATOMS.ADD throughput on
// random addresses (what the symbolic hash/bitmap inserts do). Prints ns and ops/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned* out, int iters, unsigned mask) {
  __shared__ unsigned tab[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x, acc = 0;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    unsigned a = (x >> 7) & mask;
    if (MODE == 0) acc += tab[a];
    else if (MODE == 1) acc += atomicOr(&tab[a], 1u << (x & 31));
    else if (MODE == 2) acc += atomicCAS(&tab[a], 0u, x);
    else if (MODE == 3) acc += atomicAdd(&tab[a], 1u);
    else if (MODE == 4) { unsigned v = tab[a]; if (v == 0) acc += atomicCAS(&tab[a], 0u, x); else acc += v; }
  }
  if (acc == 0x12345) out[0] = acc;
}
int main() {
  unsigned* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"LDS", "ATOMS.OR", "ATOMS.CAS", "ATOMS.ADD", "LDS+CAS-if-empty"};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096, blocks = sms * 8, threads = 256;
  for (int m = 0; m < 5; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (m) { case 0: k<0><<<blocks, threads>>>(d, iters, 8191); break; case 1: k<1><<<blocks, threads>>>(d, iters, 8191); break;
                   case 2: k<2><<<blocks, threads>>>(d, iters, 8191); break; case 3: k<3><<<blocks, threads>>>(d, iters, 8191); break;
                   case 4: k<4><<<blocks, threads>>>(d, iters, 8191); break; }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = double(blocks) * threads * iters;
      if (rep) printf("%-18s %8.3f ms  %.2f Gop/s  %.2f lane-ops/clk/SM (clk %d MHz)\n", names[m], ms, ops / ms / 1e6,
                      ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
