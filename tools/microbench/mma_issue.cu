// Is a chain of kind::mxf4 MMAs bound by the tensor core, by the dependency
// on one accumulator, or by the issuing warp?  One CTA per SM; the whole warp
// executes the loop and elect.sync picks the issuing lane; descriptors are
// hoisted; 16 MMAs per iteration into `nacc` accumulators round-robin.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I../../paper_1402_2020_b200/csrc -o mma_issue mma_issue.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
namespace {
constexpr int kCostTile = 128, kCostDisp = 64, kCostK = 16, kCostStages = 3;
#include "kern_cost.cuh"
#include "kern_cost_tc.cuh"

__device__ __forceinline__ void mma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
        "@p tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], 1;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(sfa), "r"(sfb)
        : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_addr(bar))
        : "memory");
}

template <int NACC>
__global__ void __launch_bounds__(128, 1) k_issue(int iters, int n, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t psm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(psm + 16384);
    uint32_t* slot = reinterpret_cast<uint32_t*>(psm + 16384 + 8);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(psm)[i] = 0x22222222u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *slot;
    tc_st32_const(tmem + (uint32_t(warp * 32) << 16) + kTcSfCol, 0x7F7F7F7Fu);
    tc_st32_const(tmem + (uint32_t(warp * 32) << 16) + kTcSfCol + 32, 0x7F7F7F7Fu);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        const uint64_t ad = tc_smem_desc(smem_addr(psm)), bd = tc_smem_desc(smem_addr(psm) + 4096);
        const uint32_t id = tc_idesc_mxf4(n);
        const uint32_t sfa = tmem + kTcSfCol, sfb = tmem + kTcSfCol + 32;
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int j = 0; j < 16; ++j) mma_elect(tmem + (j % NACC) * n, ad, bd, id, sfa, sfb);
            if ((i & 3) == 3) {
                commit_elect(bar);
                tc_wait(bar, ph);
                ph ^= 1u;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    uint32_t v[32];
    tc_ld32(tmem + (uint32_t(warp * 32) << 16), v);
    if (v[0] == 0x12345678u) sink[blockIdx.x] = v[1];
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int NACC>
void run(int nsm, int n, uint32_t* sink) {
    const int iters = 4000;
    cudaFuncSetAttribute(k_issue<NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    k_issue<NACC><<<nsm, 128, 20000>>>(8, n, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_issue<NACC><<<nsm, 128, 20000>>>(iters, n, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = double(iters) * 16;
    const double flops = 2.0 * nsm * mmas * 128 * n * 64;
    std::printf("N %3d, %d accumulator(s): %7.1f TFLOP/s, %6.1f ns per MMA  err=%s\n", n, NACC,
                flops / (ms * 1e-3) / 1e12, ms * 1e6 / mmas, cudaGetErrorString(cudaGetLastError()));
}
}  // namespace

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* sink;
    cudaMalloc(&sink, 4096);
    for (int n : {256, 192, 160, 128, 96, 64, 32}) {
        run<1>(nsm, n, sink);
        if (2 * n <= 448) run<2>(nsm, n, sink);
        if (4 * n <= 448) run<4>(nsm, n, sink);
    }
    return 0;
}
