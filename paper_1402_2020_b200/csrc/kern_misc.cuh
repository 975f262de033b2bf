// kern_misc.cuh -- layout converters for the per-stage API and the
// register-only pipe microbenchmarks behind bench.py's roofline.  Part of
// bsm_kernels.cu's single translation unit.
#pragma once

// ---------------------------------------------------------------------------
// Layout converters for the per-stage API (reference AoS u64 <-> device SoA).
// Device field layout (see bsm_kernels.cu): word plane w at w * P, pixel
// (x, y) of a plane at y * Wq + x (Wq = W rounded up to 4, P >= H * Wq).
__global__ void k_aos_to_soa(const uint32_t* __restrict__ src, int W, int H, int NW, int Wq, size_t P,
                             uint32_t* __restrict__ dst) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;  // over (w, p)
    const size_t total = size_t(NW) * P;
    if (i >= total) return;
    const size_t p = i % P;
    const int w = int(i / P);
    const int x = int(p % Wq), y = int(p / Wq);
    dst[i] = (x < W && y < H) ? src[(size_t(y) * W + x) * NW + w] : 0u;
}

__global__ void k_soa_to_aos(const uint32_t* __restrict__ src, int W, int H, int NW, int Wq, size_t P,
                             uint32_t* __restrict__ dst) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;  // over (y, x, w)
    const size_t total = size_t(H) * W * NW;
    if (i >= total) return;
    const int w = int(i % NW);
    const size_t yx = i / NW;
    const int x = int(yx % W), y = int(yx / W);
    dst[i] = src[size_t(w) * P + size_t(y) * Wq + x];
}

// k_soa_to_aos with the pipeline's bit order undone: reference bit k of a
// pixel's string is device bit pos[k].
__global__ void k_soa_to_aos_perm(const uint32_t* __restrict__ src, int W, int H, int NW, int Wq, size_t P,
                                  const int* __restrict__ pos, int n, uint32_t* __restrict__ dst) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;  // over (y, x, w)
    const size_t total = size_t(H) * W * NW;
    if (i >= total) return;
    const int w = int(i % NW);
    const size_t yx = i / NW;
    const int x = int(yx % W), y = int(yx / W);
    uint32_t v = 0;
    for (int b = 0; b < 32 && 32 * w + b < n; ++b) {
        const int j = __ldg(pos + 32 * w + b);
        v |= ((__ldg(src + size_t(j >> 5) * P + size_t(y) * Wq + x) >> (j & 31)) & 1u) << b;
    }
    dst[i] = v;
}

__global__ void k_keys_to_float(const uint32_t* __restrict__ keys, size_t n, float* __restrict__ out) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = float(keys[i] & 0xFFFFu);
}

// Roofline microbenchmarks of the cost kernel's inner loop (register-only,
// 8 independent chains per thread, 2048 threads per SM):
//   k_popc_peak: one word per LOP3 + POPC + IADD (the direct mix);
//   k_csa_peak:  two words per 4 LOP3 + POPC + IMAD (the carry-save mix the
//                kernel uses; balances the ALU and POPC pipes).
__global__ void __launch_bounds__(512) k_popc_peak(uint32_t* out, uint32_t seed, int iters) {
    uint32_t a[8], b[8], m[8], s[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        a[i] = seed * (threadIdx.x + i + 1);
        b[i] = a[i] ^ (0x9e3779b9u * i);
        m[i] = ~a[i] + i;
        s[i] = 0;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint32_t x = __popc((a[i] ^ b[i]) & m[i]);
            s[i] += x;
            b[i] += x;
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) r += s[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void __launch_bounds__(512) k_csa_peak(uint32_t* out, uint32_t seed, int iters, uint32_t two) {
    uint32_t a[8], b[8], m[8], o[8], s[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        a[i] = seed * (threadIdx.x + i + 1);
        b[i] = (seed + 0x9e3779b9u) * (threadIdx.x * 7u + i + 3u);
        m[i] = ~a[i] + i;
        o[i] = 0;
        s[i] = 0;
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint32_t x0 = (a[i] ^ s[i]) & m[i];
            const uint32_t x1 = (b[i] ^ o[i]) & m[i];
            const uint32_t t = (o[i] & x0) | (o[i] & x1) | (x0 & x1);
            o[i] = o[i] ^ x0 ^ x1;
            s[i] = __popc(t) * two + s[i];
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) r += s[i] + o[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
