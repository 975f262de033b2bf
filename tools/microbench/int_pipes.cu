// Microbenchmark: INT pipe throughput on B200 (POPC, LOP3, IADD3, IMAD) and
// the masked-XOR-popcount word-op used by the cost kernel. Prints ops/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
template <int MODE>
__global__ void __launch_bounds__(512) bench(uint32_t* out, uint32_t seed, long long* cyc) {
  uint32_t a[8], b[8], m[8], s[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { a[i] = seed * (threadIdx.x + i + 1); b[i] = a[i] ^ 0x9e3779b9u * i; m[i] = ~a[i] + i; s[i] = 0; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (MODE == 0) { s[i] += __popc(a[i] ^ s[i]); }                       // POPC + LOP3 + IADD (dep chain via s)
      if (MODE == 1) { a[i] = (a[i] ^ b[i]) & (m[i] | a[i]); }               // LOP3 only
      if (MODE == 2) { s[i] = s[i] + a[i] + b[i]; a[i] += 3; }               // IADD3
      if (MODE == 3) { uint32_t x = __popc((a[i] ^ b[i]) & m[i]); s[i] += x; b[i] += x; } // word-op
    }
  }
  long long t1 = clock64();
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) r += s[i] + a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int ops_per_inner) {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int blocks = nsm * 4, threads = 512;
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  bench<MODE><<<blocks, threads>>>(out, 7, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<MODE><<<blocks, threads>>>(out, 7, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long hc[4096]; cudaMemcpy(hc, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double avgc = 0; for (int i = 0; i < blocks; i++) avgc += hc[i]; avgc /= blocks;
  double ops = double(blocks) * threads * ITERS * 8 * ops_per_inner;
  // 4 blocks of 512 threads resident per SM -> per-SM ops per cycle from the in-kernel clock
  double per_sm_clk = double(4) * threads * ITERS * 8 * ops_per_inner / avgc;
  printf("%-10s %8.3f ms  %8.1f Gop/s  %6.1f op/clk/SM (clock64)  avg_cyc=%.0f\n", name, ms, ops / ms / 1e6, per_sm_clk, avgc);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs=%d clockRate=%d kHz\n", nsm, clk);
  run<0>("popc", 1);
  run<1>("lop3", 1);
  run<2>("iadd3", 1);
  run<3>("wordop", 1);
  return 0;
}
