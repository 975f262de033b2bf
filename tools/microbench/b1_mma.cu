// Microbenchmark: legacy warp-level binary MMA (mma.sync ... b1 .and.popc /
// .xor.popc) throughput on sm_100a, for deciding whether the masked-Hamming
// cost can run as a banded binary GEMM on the tensor pipe.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int XOR>
__global__ void __launch_bounds__(256) k_b1(uint32_t* out, uint32_t seed, int iters) {
    uint32_t a[4], b[2];
    int c[8][4];
#pragma unroll
    for (int i = 0; i < 4; i++) a[i] = seed * (threadIdx.x + 3 * i + 1);
    b[0] = seed ^ threadIdx.x;
    b[1] = seed * 7 + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; k++)
#pragma unroll
        for (int i = 0; i < 4; i++) c[k][i] = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (XOR)
                asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            else
                asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_i8(uint32_t* out, uint32_t seed, int iters) {
    uint32_t a[4], b[2];
    int c[8][4];
#pragma unroll
    for (int i = 0; i < 4; i++) a[i] = seed * (threadIdx.x + 3 * i + 1);
    b[0] = seed ^ threadIdx.x;
    b[1] = seed * 7 + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; k++)
#pragma unroll
        for (int i = 0; i < 4; i++) c[k][i] = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
void run(const char* name, F launch, double macs_per_mma) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = nsm * 8, threads = 256, iters = 4096;
    uint32_t* out;
    cudaMalloc(&out, blocks * threads * 4);
    launch(blocks, threads, out, iters);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch(blocks, threads, out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    const double mmas = double(blocks) * (threads / 32) * iters * 8;
    printf("%-12s %8.3f ms  %10.2f G mma/s  %10.1f T bit-or-int-MAC/s  (%s)\n", name, ms, mmas / ms / 1e6,
           mmas * macs_per_mma / ms / 1e9, cudaGetErrorString(err));
    cudaFree(out);
}

int main() {
    run("b1.and.popc", [](int b, int t, uint32_t* o, int it) { k_b1<0><<<b, t>>>(o, 7, it); }, 16.0 * 8 * 256);
    run("b1.xor.popc", [](int b, int t, uint32_t* o, int it) { k_b1<1><<<b, t>>>(o, 7, it); }, 16.0 * 8 * 256);
    run("s8 m16n8k32", [](int b, int t, uint32_t* o, int it) { k_i8<<<b, t>>>(o, 7, it); }, 16.0 * 8 * 32);
    return 0;
}
