// Microbenchmark: practical throughput of the masked-XOR-popcount instruction
// mixes on sm_100a (word-ops per clock per SM), to choose K3's counting scheme.
// Every mix keeps 8 independent cells per thread (like K3's 32 register cells)
// fed from registers that change every iteration, 16 warps per SM (K3's
// occupancy) and 32 warps per SM.
//   direct : per word      1 LOP3 (a^b)&m + POPC + IADD
//   csa1   : per 2 words   2 LOP3 + CSA (xor3 + maj) + POPC + IMAD   (K3 today)
//   csa2   : per 4 words   4 LOP3 + 3 CSA (6 LOP3) + POPC + IMAD
//   lop3   : LOP3 only; popc : POPC only (pipe rates)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o csa_mixes csa_mixes.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int MODE>
__global__ void __launch_bounds__(256) bench(uint32_t* out, uint32_t seed, uint32_t two) {
    uint32_t a[8], m[8], ones[8], twos[8], acc[8];
    uint32_t b = seed * (threadIdx.x + 1), b2 = b ^ 0x9e3779b9u;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        a[i] = seed * (threadIdx.x + 7 * i + 1);
        m[i] = ~a[i] * 3u + i;
        ones[i] = twos[i] = acc[i] = 0;
    }
    for (int it = 0; it < ITERS; it++) {
        // fresh "other view" words each iteration (K3: shared-memory loads)
        const uint32_t b0 = b * (it + 1), b1 = b2 * (it + 3), b3 = b * 5u * it, b4 = b2 * 3u * it;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (MODE == 0) {  // direct
                acc[i] += __popc((a[i] ^ b0) & m[i]);
            } else if (MODE == 1) {  // csa1: 2 words
                const uint32_t q0 = (a[i] ^ b0) & m[i], q1 = (a[i] ^ b1) & m[i];
                const uint32_t o = ones[i];
                const uint32_t t = (o & q0) | (o & q1) | (q0 & q1);
                ones[i] = o ^ q0 ^ q1;
                acc[i] = __popc(t) * two + acc[i];
            } else if (MODE == 2) {  // csa2: 4 words
                const uint32_t q0 = (a[i] ^ b0) & m[i], q1 = (a[i] ^ b1) & m[i];
                const uint32_t q2 = (a[i] ^ b3) & m[i], q3 = (a[i] ^ b4) & m[i];
                uint32_t o = ones[i];
                const uint32_t ta = (o & q0) | (o & q1) | (q0 & q1);
                o = o ^ q0 ^ q1;
                const uint32_t tb = (o & q2) | (o & q3) | (q2 & q3);
                ones[i] = o ^ q2 ^ q3;
                const uint32_t w = twos[i];
                const uint32_t f = (w & ta) | (w & tb) | (ta & tb);
                twos[i] = w ^ ta ^ tb;
                acc[i] = __popc(f) * (2 * two) + acc[i];
            } else if (MODE == 3) {  // LOP3 only
                acc[i] = (acc[i] ^ b0) & (m[i] | acc[i]);
            } else {  // POPC only
                acc[i] += __popc(acc[i] ^ b0);
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) r += acc[i] + ones[i] + twos[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name, double words_per_inner, int ctas_per_sm) {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = nsm * ctas_per_sm, threads = 256;
    uint32_t* out;
    cudaMalloc(&out, size_t(blocks) * threads * 4);
    bench<MODE><<<blocks, threads>>>(out, 7, 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        bench<MODE><<<blocks, threads>>>(out, 7 + r, 2);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = double(blocks) * threads * ITERS * 8 * words_per_inner;
    const double per_clk_sm = ops / (best * 1e-3) / (double(clk) * 1e3) / nsm;
    printf("%-8s warps/SM=%2d  %8.3f ms  %7.1f Gop/s  %6.2f /clk/SM (at max clock %d MHz)\n", name,
           ctas_per_sm * 8, best, ops / best / 1e6, per_clk_sm, clk / 1000);
    cudaFree(out);
}

int main() {
    for (int c : {2, 4}) {
        run<0>("direct", 1, c);
        run<1>("csa1", 2, c);
        run<2>("csa2", 4, c);
        run<3>("lop3", 1, c);
        run<4>("popc", 1, c);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
