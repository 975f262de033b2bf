// bsm_kernels.cu -- sm_100a kernels and the C ABI (include/bsm_cuda.h) of the
// Binary Stereo Matching hot path.  See DESIGN.md for the data layout, each
// kernel's roofline, and the reference function (file:line) it replaces.
//
// Device layout (per view, W x H, n bits, NW = 2*ceil(n/64) u32 words):
//   field[(y*NW + w)*Wp + x]   word-major ("bit-plane rows"), Wp = W rounded up
//   to 128, so a row segment of one word is a contiguous, 16-B-aligned span:
//   the cost kernel stages [K words x span] boxes by TMA (one tensor map per
//   field, dims (Wp, NW, rows)) and every shared-memory read is a
//   conflict-free 16-B lane-contiguous LDS.128.
//   u32 word w of a pixel = bits 32w..32w+31 = the low/high half of the
//   reference's u64 word w>>1 (bitstring.hpp:47-51).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/bsm_cuda.h"
#include "bsm_host.h"

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define BSM_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return set_err(BSM_CUDA_ERROR, std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                               " at " #call);                            \
    } while (0)

constexpr int kMaxPairs = 8192;      // mask kernel keeps 2*ceil(n/128) regs/lane of ranks
constexpr int kCostTile = 128;       // pixels per cost CTA
constexpr int kCostDisp = 64;        // disparities per cost CTA
constexpr int kCostK = 16;           // u32 words per pipeline stage
constexpr int kCostStages = 3;

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }

// ---------------------------------------------------------------------------
// K1' -- descriptor, four pixels per thread.  Same contract as k_descriptor.
// A thread owns pixels x..x+3 (x % 4 == 0) of two rows; per pair it reads the
// 4 p-samples and the 4 q-samples as two aligned words each plus one PRMT
// (the byte alignment is the same for every thread, so the selector is
// warp-uniform), compares the 4 unsigned bytes with a borrow-free SWAR test,
// and deposits the 4 result bits into byte lanes; every 32 pairs a 4x4 byte
// transpose turns them into the 4 pixels' words, stored as one 16-B store.
constexpr int kD2TX = 32, kD2TY = 8, kD2Rows = 2;  // CTA: 128 px x 16 rows

__device__ __forceinline__ uint32_t bytes_gt(uint32_t p, uint32_t q) {
    // bit 7 of each byte: p_b > q_b (unsigned).  d = (q|0x80) - (p&0x7F) has no
    // inter-byte borrow; bit 7 of d is [q_lo >= p_lo]; then q >= p <=>
    // (q7 & ~p7) | (~(q7 ^ p7) & d7), and p > q is its complement.
    const uint32_t d = (q | 0x80808080u) - (p & 0x7F7F7F7Fu);
    const uint32_t ge = (q & ~p) | (~(q ^ p) & d);
    return ~ge & 0x80808080u;
}

__global__ void __launch_bounds__(kD2TX* kD2TY)
    k_descriptor4(const uint8_t* __restrict__ img, int W, int H, int ybeg, int rows,
                  const int2* __restrict__ ptab, int n, int half, int TWs, int NW, int Wp,
                  uint32_t* __restrict__ desc) {
    // tile: clamped bytes; t4[i] = bytes i..i+3 of the tile, so the 4 samples
    // of a thread's 4 pixels at any offset are one aligned 32-bit load.
    extern __shared__ __align__(16) uint32_t dsm[];
    const int TH = kD2TY * kD2Rows + 2 * half;
    const int NT = TWs * TH;
    uint32_t* t4 = dsm;
    uint8_t* tile = reinterpret_cast<uint8_t*>(dsm + NT);
    const int tid = threadIdx.y * kD2TX + threadIdx.x;
    const int gx0 = blockIdx.x * (kD2TX * 4) - half;
    const int ly0 = blockIdx.y * kD2TY * kD2Rows;
    const int gy0 = ybeg + ly0 - half;
    for (int idx = tid; idx < NT; idx += kD2TX * kD2TY) {
        const int r = idx / TWs, c = idx - r * TWs;
        const int gx = min(max(gx0 + c, 0), W - 1);
        const int gy = min(max(gy0 + r, 0), H - 1);
        tile[idx] = __ldg(img + size_t(gy) * W + gx);
    }
    tile[NT] = tile[NT + 1] = tile[NT + 2] = 0;  // t4 tail (never sampled)
    __syncthreads();
    // phased layout: t4[ph * S4 + k] = bytes 4k+ph .. 4k+ph+3, so the windows a
    // warp reads for one pair offset are 32 consecutive words (no conflicts)
    const int S4 = NT >> 2;
    for (int idx = tid; idx < NT; idx += kD2TX * kD2TY)
        t4[(idx & 3) * S4 + (idx >> 2)] = uint32_t(tile[idx]) | (uint32_t(tile[idx + 1]) << 8) |
                                          (uint32_t(tile[idx + 2]) << 16) | (uint32_t(tile[idx + 3]) << 24);
    __syncthreads();
    const int xq = blockIdx.x * (kD2TX * 4) + 4 * threadIdx.x;
    const uint32_t* tb = t4 + ((threadIdx.y * kD2Rows + half) * TWs >> 2) + threadIdx.x;
    const int rowW = TWs >> 2;
    const int full = n >> 5;
    // blockIdx.z splits the word range (small images: more CTAs than SMs)
    const int wper = (NW + gridDim.z - 1) / gridDim.z;
    const int wbeg = blockIdx.z * wper, wend = min(NW, wbeg + wper);
    for (int w = wbeg; w < wend; ++w) {
        uint32_t acc[kD2Rows][4];
#pragma unroll
        for (int r = 0; r < kD2Rows; ++r)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[r][b] = 0;
        const int cnt = w < full ? 32 : (w == full ? (n & 31) : 0);
        if (cnt == 32) {
            // fully unrolled: acc[r][k >> 3] stays a static register choice
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int2 e = __ldg(ptab + 32 * w + k);  // tile-relative offsets of p and q
#pragma unroll
                for (int r = 0; r < kD2Rows; ++r) {
                    const uint32_t f = bytes_gt(tb[r * rowW + e.x], tb[r * rowW + e.y]);  // bit 7 of byte j: pixel j
                    // pair k -> bit (k & 7) of byte lane j of acc[k >> 3]
                    acc[r][k >> 3] |= (f >> (7 - (k & 7)));
                }
            }
        } else {
            for (int k = 0; k < cnt; ++k) {
                const int2 e = __ldg(ptab + 32 * w + k);
#pragma unroll
                for (int r = 0; r < kD2Rows; ++r) {
                    const uint32_t v = bytes_gt(tb[r * rowW + e.x], tb[r * rowW + e.y]) >> (7 - (k & 7));
                    switch (k >> 3) {
                        case 0: acc[r][0] |= v; break;
                        case 1: acc[r][1] |= v; break;
                        case 2: acc[r][2] |= v; break;
                        default: acc[r][3] |= v; break;
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < kD2Rows; ++r) {
            // acc[b] byte j = bits 8b..8b+7 of pixel j  ->  4x4 byte transpose
            const uint32_t t0 = __byte_perm(acc[r][0], acc[r][1], 0x5140), t1 = __byte_perm(acc[r][0], acc[r][1], 0x7362);
            const uint32_t t2 = __byte_perm(acc[r][2], acc[r][3], 0x5140), t3 = __byte_perm(acc[r][2], acc[r][3], 0x7362);
            uint4 o;
            o.x = __byte_perm(t0, t2, 0x5410);
            o.y = __byte_perm(t0, t2, 0x7632);
            o.z = __byte_perm(t1, t3, 0x5410);
            o.w = __byte_perm(t1, t3, 0x7632);
            const int ly = ly0 + threadIdx.y * kD2Rows + r;
            if (ly < rows) *reinterpret_cast<uint4*>(desc + (size_t(ly) * NW + w) * Wp + xq) = o;
        }
    }
}

// ---------------------------------------------------------------------------
// K2 -- mask: shared helpers of k_mask4 (one warp per CTA, kM3Px pixels per
// CTA, two pixels per pass).
constexpr int kM3Px = 8;
// rank-gather index tables (u32 byte offsets): P table, then Q table, each
// sized for MCH = 8 chunks (8192 positions)
constexpr int kPqTable = 8192;

__device__ __forceinline__ uint32_t vmax_u16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

__device__ __forceinline__ uint32_t lds_u32(const uint32_t* base, uint32_t byte_off) {
    return *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(base) + byte_off);
}

// ---------------------------------------------------------------------------
// K2'' -- mask on bit planes.  Lane l owns bit positions [S l, S l + S) in
// MCH chunks of 32 (S = 32 MCH; MCH = 1, 2, 4, 8 for n <= 1024 .. 8192; the
// pair at each position comes from the bank-balanced order, so every 32-lane
// rank gather is one shared-memory wavefront); for two pixels per pass it
//   1. gathers a = max(rhoP, rhoQ) of both pixels per pair (one u32 rank-table
//      gather + VIMNMX.U16x2 serves both), packs each pixel's 32 chunk values
//      into eight byte registers,
//   2. transposes them into 8 bit planes held in registers (four 8x8 bit-matrix
//      transposes and a 4x4 byte transpose): plane j, word m of lane l holds
//      bit j of a for positions S l + 32m + t at bit t -- exactly the layout
//      of output word MCH l + m (MCH = 8 forms one pixel's planes at a time),
//   3. selects the k-th smallest a MSB-first on the planes (per bit: LOP3 +
//      POPC per word, one REDUX; the two pixels in lockstep) with the a <= T
//      comparator fused in, and stages one uint4 of output words per lane.
// 8x8 bit-matrix transpose of the 8 bytes (lo: rows 0-3, hi: rows 4-7),
// afterwards byte j bit k = input byte k bit j.  Three delta-swap stages on the
// 32-bit halves (the first two stay inside a half; left shifts as multiplies
// so they can issue on the FMA pipe).
__device__ __forceinline__ void transpose8x8_32(uint32_t& lo, uint32_t& hi) {
    uint32_t t;
    t = (lo ^ (lo >> 7)) & 0x00AA00AAu;
    lo = lo ^ t ^ (t * 128u);
    t = (hi ^ (hi >> 7)) & 0x00AA00AAu;
    hi = hi ^ t ^ (t * 128u);
    t = (lo ^ (lo >> 14)) & 0x0000CCCCu;
    lo = lo ^ t ^ (t * 16384u);
    t = (hi ^ (hi >> 14)) & 0x0000CCCCu;
    hi = hi ^ t ^ (t * 16384u);
    t = (lo ^ (hi * 16u)) & 0xF0F0F0F0u;
    lo ^= t;
    hi ^= t >> 4;
}

// w[0..7]: 32 byte values (value t = byte t%4 of w[t/4]); planes[j] bit t = bit j of value t.
__device__ __forceinline__ void bytes_to_planes(const uint32_t (&w)[8], uint32_t (&pl)[8]) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        lo[b] = w[2 * b];
        hi[b] = w[2 * b + 1];
        transpose8x8_32(lo[b], hi[b]);
    }
    // 4x4 byte transposes: plane j = byte j of block 0..3
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t* s = h ? hi : lo;
        const uint32_t t0 = __byte_perm(s[0], s[1], 0x5140), t1 = __byte_perm(s[0], s[1], 0x7362);
        const uint32_t t2 = __byte_perm(s[2], s[3], 0x5140), t3 = __byte_perm(s[2], s[3], 0x7362);
        pl[4 * h + 0] = __byte_perm(t0, t2, 0x5410);
        pl[4 * h + 1] = __byte_perm(t0, t2, 0x7632);
        pl[4 * h + 2] = __byte_perm(t1, t3, 0x5410);
        pl[4 * h + 3] = __byte_perm(t1, t3, 0x7632);
    }
}


// MSB-first k-th-smallest selection over 8 bit planes (4 words per lane,
// 128 values per lane, 4096 per warp) fused with the comparator: at a bit
// where the threshold takes 1, the still-equal values with a 0 there are
// strictly below it; the output words are (a <= T) = lt | eq.
// Two selects in lockstep (the two pixels of a pass): the REDUX of one
// overlaps the POPCs and the REDUX of the other.
template <int MCH>
__device__ __forceinline__ void select_le2(const uint32_t (&pa)[8][MCH], const uint32_t (&pb)[8][MCH], int k,
                                           uint32_t (&oa)[MCH], uint32_t (&ob)[MCH]) {
    uint32_t ea[MCH], eb[MCH], la[MCH], lb[MCH];
#pragma unroll
    for (int m = 0; m < MCH; ++m) {
        ea[m] = eb[m] = ~0u;
        la[m] = lb[m] = 0u;
    }
    int ka = k, kb = k;
#pragma unroll
    for (int j = 7; j >= 0; --j) {
        uint32_t za[MCH], zb[MCH];
        uint32_t ca = 0, cb = 0;
#pragma unroll
        for (int m = 0; m < MCH; ++m) {
            za[m] = ea[m] & ~pa[j][m];
            zb[m] = eb[m] & ~pb[j][m];
            ca += __popc(za[m]);
            cb += __popc(zb[m]);
        }
        const int zas = int(__reduce_add_sync(0xFFFFFFFFu, ca));
        const int zbs = int(__reduce_add_sync(0xFFFFFFFFu, cb));
        // warp-uniform choices; written as selects so both chains stay branch-free
        const bool ha = zas < ka, hb = zbs < kb;
        ka -= ha ? zas : 0;
        kb -= hb ? zbs : 0;
#pragma unroll
        for (int m = 0; m < MCH; ++m) {
            la[m] |= ha ? za[m] : 0u;
            ea[m] = ha ? (ea[m] & pa[j][m]) : za[m];
            lb[m] |= hb ? zb[m] : 0u;
            eb[m] = hb ? (eb[m] & pb[j][m]) : zb[m];
        }
    }
#pragma unroll
    for (int m = 0; m < MCH; ++m) {
        oa[m] = la[m] | ea[m];
        ob[m] = lb[m] | eb[m];
    }
}

// Stores MCH consecutive words (16-, 8- or 4-byte aligned).
template <int MCH>
__device__ __forceinline__ void store_words(uint32_t* dst, const uint32_t (&w)[MCH]) {
    if constexpr (MCH == 8) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(dst + 4) = make_uint4(w[4], w[5], w[6], w[7]);
    } else if constexpr (MCH == 4) *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    else if constexpr (MCH == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
    else dst[0] = w[0];
}

// One pixel's select (the split variant for MCH = 8, where two pixels' planes
// would not fit the register budget).
template <int MCH>
__device__ __forceinline__ void select_le1(const uint32_t (&pa)[8][MCH], int k, uint32_t (&oa)[MCH]) {
    uint32_t ea[MCH], la[MCH];
#pragma unroll
    for (int m = 0; m < MCH; ++m) {
        ea[m] = ~0u;
        la[m] = 0u;
    }
    int ka = k;
#pragma unroll
    for (int j = 7; j >= 0; --j) {
        uint32_t za[MCH], ca = 0;
#pragma unroll
        for (int m = 0; m < MCH; ++m) {
            za[m] = ea[m] & ~pa[j][m];
            ca += __popc(za[m]);
        }
        const int zas = int(__reduce_add_sync(0xFFFFFFFFu, ca));
        const bool ha = zas < ka;
        ka -= ha ? zas : 0;
#pragma unroll
        for (int m = 0; m < MCH; ++m) {
            la[m] |= ha ? za[m] : 0u;
            ea[m] = ha ? (ea[m] & pa[j][m]) : za[m];
        }
    }
#pragma unroll
    for (int m = 0; m < MCH; ++m) oa[m] = la[m] | ea[m];
}

// Output staging row stride (words) of k_mask4<MCH>: 32 MCH words per pixel +
// 4 of padding (16-B aligned rows, conflict-free read-out).
__host__ __device__ constexpr int mask4_stage_stride(int mch) { return 32 * mch + 4; }

template <int MCH>
__global__ void __launch_bounds__(32, 16)
    k_mask4(const uint8_t* __restrict__ img, int W, int H, int ybeg, int rows, const uint4* __restrict__ p4,
            const uint4* __restrict__ q4, int n, const int32_t* __restrict__ uoff, int u, int rho_words,
            const uint8_t* __restrict__ rank, int half, int TW, int NW, int Wp, uint32_t* __restrict__ mask) {
    extern __shared__ __align__(16) uint32_t dsm[];
    uint32_t* rho = dsm;                                  // rho_words (u + sentinel, padded)
    constexpr int STG = mask4_stage_stride(MCH);
    uint32_t* stage = rho + rho_words;                    // [kM3Px][STG]
    uint8_t* rrows = reinterpret_cast<uint8_t*>(stage + kM3Px * STG);  // 2 x 256
    uint8_t* tile = rrows + 512;                                            // (2h+1) x TW
    const int G = (n + 31) >> 5;
    const int TH = 2 * half + 1;
    const int lane = threadIdx.x;
    const int x0 = blockIdx.x * kM3Px;
    const int ly = blockIdx.y;
    const int y = ybeg + ly;
    // The tile starts at the word-aligned column a0 <= x0 - h; interior tiles of
    // 4-byte-aligned rows load whole words, the rest bytes with clamping.
    const int a0 = (x0 - half) & ~3, ay0 = y - half;
    const int sh = x0 - half - a0;
    if ((W & 3) == 0 && a0 >= 0 && a0 + TW <= W && ay0 >= 0 && ay0 + TH <= H) {
        const int nw = TW >> 2;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(img + size_t(ay0) * W + a0);
#pragma unroll 4
        for (int idx = lane; idx < TH * nw; idx += 32) {
            const int r = idx / nw;
            reinterpret_cast<uint32_t*>(tile)[idx] = __ldg(src + size_t(r) * (W >> 2) + (idx - r * nw));
        }
    } else {
#pragma unroll 4
        for (int idx = lane; idx < TW * TH; idx += 32) {
            const int r = idx / TW, c = idx - r * TW;
            const int gx = min(max(a0 + c, 0), W - 1);
            const int gy = min(max(ay0 + r, 0), H - 1);
            tile[idx] = __ldg(img + size_t(gy) * W + gx);
        }
    }
    if (lane == 0) rho[u] = 0x00FF00FFu;  // sentinel: a = 255 for both pixels
    __syncwarp();

    const int k = max(1, n / 4);
    const int c0 = half * TW + sh + half;  // tile index of pixel x0
    // rank rows of the next pass's two centre pixels, loaded one pass ahead
    uint4 rr = __ldg(reinterpret_cast<const uint4*>(rank + 256 * int(tile[c0 + (lane >> 4)])) + (lane & 15));
#pragma unroll 1
    for (int q = 0; q < kM3Px; q += 2) {
        const int cia = c0 + q, cib = cia + 1;
        reinterpret_cast<uint4*>(rrows)[lane] = rr;
        if (q + 2 < kM3Px)
            rr = __ldg(reinterpret_cast<const uint4*>(rank + 256 * int(tile[cia + 2 + (lane >> 4)])) + (lane & 15));
        __syncwarp();
        for (int j = lane; j < u; j += 32) {
            const int o = __ldg(uoff + j);
            rho[j] = uint32_t(rrows[tile[cia + o]]) | (uint32_t(rrows[256 + tile[cib + o]]) << 16);
        }
        __syncwarp();

        // a = max(rhoP, rhoQ) of 32 positions of chunk m for both pixels, as
        // byte registers wa (pixel A) and wb (pixel B)
        auto gather = [&](int m, uint32_t(&wa)[8], uint32_t(&wb)[8]) {
#pragma unroll
            for (int t4 = 0; t4 < 8; ++t4) {
                const uint4 P = __ldg(p4 + (m * 8 + t4) * 32 + lane);
                const uint4 Q = __ldg(q4 + (m * 8 + t4) * 32 + lane);
                const uint32_t v0 = vmax_u16x2(lds_u32(rho, P.x), lds_u32(rho, Q.x));
                const uint32_t v1 = vmax_u16x2(lds_u32(rho, P.y), lds_u32(rho, Q.y));
                const uint32_t v2 = vmax_u16x2(lds_u32(rho, P.z), lds_u32(rho, Q.z));
                const uint32_t v3 = vmax_u16x2(lds_u32(rho, P.w), lds_u32(rho, Q.w));
                const uint32_t x01 = __byte_perm(v0, v1, 0x6240);  // [A0 A1 B0 B1]
                const uint32_t x23 = __byte_perm(v2, v3, 0x6240);  // [A2 A3 B2 B3]
                wa[t4] = __byte_perm(x01, x23, 0x5410);
                wb[t4] = __byte_perm(x01, x23, 0x7632);
            }
        };
        if constexpr (MCH <= 4) {
            uint32_t pa[8][MCH], pb[8][MCH];
#pragma unroll
            for (int m = 0; m < MCH; ++m) {
                uint32_t wa[8], wb[8], ta[8], tb[8];
                gather(m, wa, wb);
                bytes_to_planes(wa, ta);
                bytes_to_planes(wb, tb);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    pa[j][m] = ta[j];
                    pb[j][m] = tb[j];
                }
            }
            uint32_t oa[MCH], ob[MCH];
            select_le2<MCH>(pa, pb, k, oa, ob);
            store_words<MCH>(stage + q * STG + MCH * lane, oa);
            store_words<MCH>(stage + (q + 1) * STG + MCH * lane, ob);
        } else {
            // one pixel's planes at a time: the gathers run twice
#pragma unroll 1
            for (int side = 0; side < 2; ++side) {
                uint32_t pl[8][MCH];
#pragma unroll
                for (int m = 0; m < MCH; ++m) {
                    uint32_t wa[8], wb[8], t[8];
                    gather(m, wa, wb);
                    bytes_to_planes(side ? wb : wa, t);
#pragma unroll
                    for (int j = 0; j < 8; ++j) pl[j][m] = t[j];
                }
                uint32_t o[MCH];
                select_le1<MCH>(pl, k, o);
                store_words<MCH>(stage + (q + side) * STG + MCH * lane, o);
            }
        }
        __syncwarp();  // rho / rrows are rewritten by the next pass
    }
    __syncwarp();
    // lane = (word offset w % 4, pixel j): 32-B row segments, stage reads
    // independent across iterations; pad bits and pad words are zero
    const int rem = n & 31;
    const uint32_t tail = rem ? (1u << rem) - 1u : ~0u;
    const int jl = lane & (kM3Px - 1), wl = lane / kM3Px;
    uint32_t* dst = mask + (size_t(ly) * NW + wl) * Wp + x0 + jl;
#pragma unroll 4
    for (int w = wl; w < NW; w += 32 / kM3Px, dst += size_t(32 / kM3Px) * Wp) {
        const uint32_t v = stage[jl * STG + w];
        *dst = w < G - 1 ? v : (w == G - 1 ? v & tail : 0u);
    }
}

// ---------------------------------------------------------------------------
// Colour / float-plane path (compute_field on arbitrary GrayImage + LabImage,
// run_pipeline on RGB).  Same contracts as K1/K2 with float planes.
//
// k_rgb_planes: interleaved RGB -> gray (f32) and Lab planes via the
// host-built 2^24-entry conversion tables (bit-identical to the reference's
// to_gray / to_lab, image.hpp:90-140).  Device Lab planes hold one float4
// (L, a, b, 0) per pixel, so a window sample is one 16-byte load.
__global__ void k_rgb_planes(const uint8_t* __restrict__ rgb, size_t n, const float* __restrict__ gtab,
                             const float* __restrict__ ltab, float* __restrict__ gray, float4* __restrict__ lab4) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = (uint32_t(rgb[3 * i]) << 16) | (uint32_t(rgb[3 * i + 1]) << 8) | uint32_t(rgb[3 * i + 2]);
    gray[i] = __ldg(gtab + k);
    lab4[i] = make_float4(__ldg(ltab + 3 * size_t(k)), __ldg(ltab + 3 * size_t(k) + 1), __ldg(ltab + 3 * size_t(k) + 2),
                          0.0f);
}

// Caller Lab planes (3 floats per pixel, the reference's LabImage layout) ->
// device float4 planes.
__global__ void k_lab3_to_lab4(const float* __restrict__ lab, size_t n, float4* __restrict__ lab4) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    lab4[i] = make_float4(lab[3 * i], lab[3 * i + 1], lab[3 * i + 2], 0.0f);
}

// K1f: descriptor bits I(p) > I(q) on a float gray plane (descriptor.hpp:95-105,
// 214-230).  Thread per pixel column x 4 rows; clamped float tile.
constexpr int kDfTX = 32, kDfTY = 8, kDfPY = 4;

__global__ void __launch_bounds__(kDfTX* kDfTY)
    k_descriptor_f32(const float* __restrict__ gray, int W, int H, int ybeg, int rows, const int2* __restrict__ offs,
                     int n, int half, int NW, int Wp, uint32_t* __restrict__ desc) {
    extern __shared__ __align__(16) float ftile[];
    const int TW = kDfTX + 2 * half, TH = kDfTY * kDfPY + 2 * half;
    const int tid = threadIdx.y * kDfTX + threadIdx.x;
    const int gx0 = blockIdx.x * kDfTX - half;
    const int ly0 = blockIdx.y * kDfTY * kDfPY;
    const int gy0 = ybeg + ly0 - half;
    for (int idx = tid; idx < TW * TH; idx += kDfTX * kDfTY) {
        const int r = idx / TW, c = idx - r * TW;
        ftile[idx] = __ldg(gray + size_t(min(max(gy0 + r, 0), H - 1)) * W + min(max(gx0 + c, 0), W - 1));
    }
    __syncthreads();
    const int x = blockIdx.x * kDfTX + threadIdx.x;
    const float* t0 = ftile + (threadIdx.y * kDfPY + half) * TW + threadIdx.x + half;
    for (int w = 0; w < NW; ++w) {
        uint32_t acc[kDfPY] = {0u, 0u, 0u, 0u};
        const int cnt = min(32, max(0, n - 32 * w));
        if (cnt == 32) {
            // fully unrolled: static bit positions (predicated ORs)
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int2 o = __ldg(offs + 32 * w + k);  // tile-relative (py*TW + px) of p and q
#pragma unroll
                for (int j = 0; j < kDfPY; ++j)
                    if (t0[j * TW + o.x] > t0[j * TW + o.y]) acc[j] |= 1u << k;
            }
        } else {
            for (int k = 0; k < cnt; ++k) {
                const int2 o = __ldg(offs + 32 * w + k);
#pragma unroll
                for (int j = 0; j < kDfPY; ++j) acc[j] |= uint32_t(t0[j * TW + o.x] > t0[j * TW + o.y]) << k;
            }
        }
#pragma unroll
        for (int j = 0; j < kDfPY; ++j) {
            const int ly = ly0 + threadIdx.y * kDfPY + j;
            if (ly < rows) desc[(size_t(ly) * NW + w) * Wp + x] = acc[j];
        }
    }
}

// K2f: mask on a float Lab plane (descriptor.hpp:118-154, 64-76).  One warp
// per CTA, kM3Px pixels per CTA, one pixel per pass.  The window SADs t[slot]
// are kept as float bit patterns (non-negative floats order like u32); lane l
// owns pairs S l + 32m + t, forms a = max(t[P], t[Q]) for 32 pairs per chunk,
// transposes the 32 words into bit planes (5-stage in-register 32x32 bit
// transpose) and selects the k-th smallest MSB-first with the a <= T
// comparator fused in -- over key bits 31..8, and over the low byte only when
// the threshold's tie is not a single slot key.
__device__ __forceinline__ void transpose32(uint32_t (&x)[32]) {
    // afterwards x[j] bit t = (original x[t]) bit j
#pragma unroll
    for (int sidx = 0; sidx < 5; ++sidx) {
        const int sh = 16 >> sidx;
        const uint32_t mk = sidx == 0 ? 0x0000FFFFu : sidx == 1 ? 0x00FF00FFu : sidx == 2 ? 0x0F0F0F0Fu
                           : sidx == 3 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            if (i & sh) continue;
            const uint32_t t = ((x[i] >> sh) ^ x[i + sh]) & mk;
            x[i + sh] ^= t;
            x[i] ^= t << sh;
        }
    }
}

template <int MCH>
__global__ void __launch_bounds__(32, 16)
    k_mask_f32(const float4* __restrict__ lab4, int W, int H, int ybeg, int rows, const uint4* __restrict__ p4,
               const uint4* __restrict__ q4, int n, const int32_t* __restrict__ uxy, int u, int rho_words,
               int NW, int Wp, uint32_t* __restrict__ mask, int half) {
    // Lab samples (float4 per pixel) are read through L1 (no shared tile):
    // shared memory holds only the slot keys and 24 rows of bit planes (the
    // low byte's planes reuse the rows of bits 8..15), for occupancy.
    extern __shared__ __align__(16) uint32_t dsm[];
    uint32_t* tv = dsm;                                   // rho_words: SAD bits per slot (+ sentinel)
    uint32_t* planes = tv + rho_words;                    // [24 rows][MCH chunks][32 lanes]
    auto prow = [](int b) { return b >= 8 ? b - 8 : b; };  // plane row of key bit b
    const int G = (n + 31) >> 5;
    const int lane = threadIdx.x;
    const int x0 = blockIdx.x * kM3Px;
    const int ly = blockIdx.y;
    const int y = ybeg + ly;
    if (lane == 0) tv[u] = 0xFFFFFFFFu;  // sentinel: larger than every SAD
    // windows of all kM3Px pixels inside the view: no clamping
    const bool interior = x0 - half >= 0 && x0 + kM3Px - 1 + half < W && y - half >= 0 && y + half < H;
    const int k = max(1, n / 4);
    const unsigned full = 0xFFFFFFFFu;
    const int rem = n & 31;
#pragma unroll 1
    for (int px = 0; px < kM3Px; ++px) {
        const int x = min(x0 + px, W - 1);  // pad columns repeat the last pixel (not stored)
        const float4 cc = __ldg(lab4 + size_t(y) * W + x);
        // lab_sad(centre, window pixel), image.hpp:144-146
        auto sad = [&](const float4 o) {
            return __fadd_rn(__fadd_rn(fabsf(__fsub_rn(cc.x, o.x)), fabsf(__fsub_rn(cc.y, o.y))),
                             fabsf(__fsub_rn(cc.z, o.z)));
        };
        if (interior) {
            const float4* cp = lab4 + size_t(y) * W + x;
#pragma unroll 8
            for (int j = lane; j < u; j += 32) {  // 8 window samples in flight per lane
                const int e = __ldg(uxy + j);  // (dy << 16) | (dx & 0xFFFF)
                tv[j] = __float_as_uint(sad(__ldg(cp + ((e >> 16) * W + int(int16_t(e & 0xFFFF))))));
            }
        } else {
            for (int j = lane; j < u; j += 32) {
                const int e = __ldg(uxy + j);
                const int gx = min(max(x + int(int16_t(e & 0xFFFF)), 0), W - 1);
                const int gy = min(max(y + (e >> 16), 0), H - 1);
                tv[j] = __float_as_uint(sad(__ldg(lab4 + size_t(gy) * W + gx)));
            }
        }
        __syncwarp();
        // a = max(t[P], t[Q]) of 32 positions per chunk, transposed into bit
        // planes: bits 31..8 first (the transposes' low-byte outputs are dead
        // code), bits 7..0 only when the top 24 bits leave the tie unresolved
        auto planes_of = [&](auto store) {
#pragma unroll 1
            for (int m = 0; m < MCH; ++m) {
                uint32_t x[32];
#pragma unroll
                for (int t4 = 0; t4 < 8; ++t4) {
                    uint4 P, Q;
                    if constexpr (MCH <= 4) {  // packed P | Q << 16 (p4 points at the packed table)
                        P = __ldg(p4 + (m * 8 + t4) * 32 + lane);
                        Q = make_uint4(P.x >> 16, P.y >> 16, P.z >> 16, P.w >> 16);
                        P = make_uint4(P.x & 0xFFFFu, P.y & 0xFFFFu, P.z & 0xFFFFu, P.w & 0xFFFFu);
                    } else {
                        P = __ldg(p4 + (m * 8 + t4) * 32 + lane);
                        Q = __ldg(q4 + (m * 8 + t4) * 32 + lane);
                    }
                    x[4 * t4] = max(lds_u32(tv, P.x), lds_u32(tv, Q.x));
                    x[4 * t4 + 1] = max(lds_u32(tv, P.y), lds_u32(tv, Q.y));
                    x[4 * t4 + 2] = max(lds_u32(tv, P.z), lds_u32(tv, Q.z));
                    x[4 * t4 + 3] = max(lds_u32(tv, P.w), lds_u32(tv, Q.w));
                }
                transpose32(x);
                store(m, x);
            }
        };
        planes_of([&](int m, const uint32_t (&x)[32]) {
#pragma unroll
            for (int j = 8; j < 32; ++j) planes[(prow(j) * MCH + m) * 32 + lane] = x[j];
        });
        __syncwarp();
        // MSB-first k-th smallest over 32-bit keys (pads are 0xFFFFFFFF) with
        // the a <= T comparator fused in: where the threshold takes a 1, the
        // still-equal keys with a 0 there are strictly below it.
        uint32_t eq[MCH], lt[MCH];
#pragma unroll
        for (int m = 0; m < MCH; ++m) {
            eq[m] = ~0u;
            lt[m] = 0u;
        }
        int kk = k;
        uint32_t tbits = 0;  // threshold bits decided so far
        auto rounds = [&](int hi, int lo) {
#pragma unroll 1
            for (int j = hi; j >= lo; --j) {
                uint32_t pl[MCH], z[MCH], cnt = 0;
#pragma unroll
                for (int m = 0; m < MCH; ++m) {
                    pl[m] = planes[(prow(j) * MCH + m) * 32 + lane];
                    z[m] = eq[m] & ~pl[m];
                    cnt += __popc(z[m]);
                }
                const int zeros = int(__reduce_add_sync(full, cnt));
                if (zeros >= kk) {
#pragma unroll
                    for (int m = 0; m < MCH; ++m) eq[m] = z[m];
                } else {
                    kk -= zeros;
                    tbits |= 1u << j;
#pragma unroll
                    for (int m = 0; m < MCH; ++m) {
                        lt[m] |= z[m];
                        eq[m] &= pl[m];
                    }
                }
            }
        };
        rounds(31, 8);
        // Every value is a slot key, so the positions still tied (top 24 bits
        // equal to the threshold's) all hold the threshold itself when the
        // slot keys with those top bits are one value: then eq is final.
        // Otherwise (rare) the low byte is resolved on its own planes.
        uint32_t mn = 0xFFFFFFFFu, mx = 0u;
        for (int j = lane; j < u; j += 32) {
            const uint32_t v = tv[j];
            if ((v >> 8) == (tbits >> 8)) {
                mn = min(mn, v);
                mx = max(mx, v);
            }
        }
#ifdef BSM_MASKF_ALWAYS_LOW  // test hook: resolve the low byte for every pixel
        if (true) {
#else
        if (__reduce_min_sync(full, mn) != __reduce_max_sync(full, mx)) {
#endif
            __syncwarp();
            planes_of([&](int m, const uint32_t (&x)[32]) {  // rows of bits 8..15 are dead now
#pragma unroll
                for (int j = 0; j < 8; ++j) planes[(prow(j) * MCH + m) * 32 + lane] = x[j];
            });
            __syncwarp();
            rounds(7, 0);
        }
#pragma unroll
        for (int m = 0; m < MCH; ++m) {
            const int w = MCH * lane + m;
            if (w < NW) {
                uint32_t v = lt[m] | eq[m];
                if (w >= G) v = 0u;
                else if (rem && w == G - 1) v &= (1u << rem) - 1u;
                mask[(size_t(ly) * NW + w) * Wp + x0 + px] = v;
            }
        }
        __syncwarp();
    }
}

// --- TMA staging helpers (cp.async.bulk.tensor + mbarrier) ----------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}
// 3-D box (x, word, row) of a field into shared memory, completing on bar.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int w, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(w), "r"(y), "r"(smem_addr(bar))
        : "memory");
}

// ---------------------------------------------------------------------------
// K3 -- fused masked Hamming cost + winner-take-all.  matcher.hpp:80-113
// (wta), :24-29/bitstring.hpp:73-88 (masked_hamming), :35-38 (other_column),
// :68-75 (ties -> smaller d).  No cost volume is materialised.
// CTA tile: 128 reference pixels of one row x 64 disparities; 8 warps, warp wi
// owns disparities [d0 + 8wi, +8), lane l owns pixels [x0 + 4l, +4): a 4 x 8
// register block of costs, so each staged word feeds 32 word-ops from 5
// LDS.128 (ref desc, ref mask, a 12-word window of the other view).
// Words stream through a 3-stage ring of K = 16 words filled by TMA: one
// thread arms the stage's mbarrier and issues three tensor-box copies
// ([K x 128] desc, [K x 128] mask, [K x 192] other-view span); columns and
// words outside the field arrive zero-filled, so the load path carries no
// per-thread predicates or address arithmetic.  The argmin key is
// (cost << 16) | d (min cost, then smaller d); d-split CTAs merge with
// atomicMin.  Out-of-image correspondences are skipped (matcher.hpp:100).
template <bool RIGHT, bool MASKED>
__global__ void __launch_bounds__(256, 2)
    k_cost_wta(const __grid_constant__ CUtensorMap tm_ref, const __grid_constant__ CUtensorMap tm_mask,
               const __grid_constant__ CUtensorMap tm_oth, int W, int rows, int NW, int D,
               uint32_t* __restrict__ keys, uint32_t two) {
    constexpr int T = kCostTile, DC = kCostDisp, K = kCostK, ST = kCostStages, BW = T + DC;
    constexpr int SA = K * T, SB = K * BW;
    constexpr int STAGE = (MASKED ? 2 * SA : SA) + SB;
    constexpr uint32_t STAGE_BYTES = uint32_t(STAGE) * 4;
    extern __shared__ __align__(128) uint32_t csm[];
    uint32_t* red = csm + ST * STAGE;                                 // [8][T]
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 8 * T);         // [ST] full, then [ST] empty
    uint64_t* empty = bars + ST;

    const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    const int x0 = blockIdx.y * T;
    const int y = blockIdx.z;
    const int d0 = blockIdx.x * DC;
    const int bbase = RIGHT ? x0 + d0 : x0 - d0 - DC;
    const int nchunks = (NW + K - 1) / K;
    const int xhi = min(x0 + T, W) - 1;
    if (d0 >= D || (RIGHT ? x0 + d0 >= W : xhi < d0)) return;

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(bars + s, 1);
            mbar_init(empty + s, 8);  // one arrival per warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto load_stage = [&](int c, int st) {  // thread 0 only
        uint32_t* s = csm + st * STAGE;
        mbar_expect_tx(bars + st, STAGE_BYTES);
        tma_load_3d(s, &tm_ref, x0, c * K, y, bars + st);
        if constexpr (MASKED) tma_load_3d(s + SA, &tm_mask, x0, c * K, y, bars + st);
        tma_load_3d(s + (MASKED ? 2 * SA : SA), &tm_oth, bbase, c * K, y, bars + st);
    };
    if (tid == 0)
        for (int s = 0; s < ST && s < nchunks; ++s) load_stage(s, s);

    uint32_t acc[4][8], ones[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            acc[j][s] = 0;
            ones[j][s] = 0;
        }

    const int xs = lane * 4;
    const int ds = wi * 8;
    const int c0 = RIGHT ? xs + ds : xs - ds + DC - 8;
    const bool busy = d0 + ds < D && (RIGHT ? x0 + d0 + ds < W : xhi >= d0 + ds);

#pragma unroll 1
    for (int c = 0; c < nchunks; ++c) {
        mbar_wait(bars + c % ST, uint32_t(c / ST) & 1u);
        if (busy) {
        const uint32_t* sa = csm + (c % ST) * STAGE;
        const uint32_t* sm = sa + SA;
        const uint32_t* sb = sa + (MASKED ? 2 * SA : SA);
#pragma unroll 1
        for (int w = 0; w < K; w += 2) {
            uint32_t a[2][4], m[2][4], b[2][12];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint4 a4 = *reinterpret_cast<const uint4*>(sa + (w + h) * T + xs);
                uint4 m4 = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
                if constexpr (MASKED) m4 = *reinterpret_cast<const uint4*>(sm + (w + h) * T + xs);
                const uint4 b0 = *reinterpret_cast<const uint4*>(sb + (w + h) * BW + c0);
                const uint4 b1 = *reinterpret_cast<const uint4*>(sb + (w + h) * BW + c0 + 4);
                const uint4 b2 = *reinterpret_cast<const uint4*>(sb + (w + h) * BW + c0 + 8);
                a[h][0] = a4.x; a[h][1] = a4.y; a[h][2] = a4.z; a[h][3] = a4.w;
                m[h][0] = m4.x; m[h][1] = m4.y; m[h][2] = m4.z; m[h][3] = m4.w;
                b[h][0] = b0.x; b[h][1] = b0.y; b[h][2] = b0.z; b[h][3] = b0.w;
                b[h][4] = b1.x; b[h][5] = b1.y; b[h][6] = b1.z; b[h][7] = b1.w;
                b[h][8] = b2.x; b[h][9] = b2.y; b[h][10] = b2.z; b[h][11] = b2.w;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int s = 0; s < 8; ++s) {
                    const int e = RIGHT ? j + s : j - s + 8;
                    uint32_t q0 = a[0][j] ^ b[0][e];
                    uint32_t q1 = a[1][j] ^ b[1][e];
                    if constexpr (MASKED) {
                        q0 &= m[0][j];
                        q1 &= m[1][j];
                    }
                    const uint32_t o = ones[j][s];
                    const uint32_t twos = (o & q0) | (o & q1) | (q0 & q1);
                    ones[j][s] = o ^ q0 ^ q1;
                    acc[j][s] = __popc(twos) * two + acc[j][s];
                }
        }
        }
        // release the slot; thread 0 refills it once all 8 warps are done
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + c % ST);
        if (tid == 0 && c + ST < nchunks) {
            mbar_wait(empty + c % ST, uint32_t(c / ST) & 1u);
            load_stage(c + ST, c % ST);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int s = 0; s < 8; ++s) acc[j][s] += __popc(ones[j][s]);

#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int x = x0 + xs + j;
        uint32_t best = 0xFFFFFFFFu;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int d = d0 + ds + s;
            const int xo = RIGHT ? x + d : x - d;
            const bool ok = d < D && x < W && xo >= 0 && xo < W;
            const uint32_t key = (acc[j][s] << 16) | uint32_t(d);
            if (ok && key < best) best = key;
        }
        red[wi * T + xs + j] = best;
    }
    __syncthreads();
    if (tid < T) {
        uint32_t best = red[tid];
#pragma unroll
        for (int w = 1; w < 8; ++w) best = min(best, red[w * T + tid]);
        const int x = x0 + tid;
        if (x < W && best != 0xFFFFFFFFu) {
            if (gridDim.x == 1) keys[size_t(y) * W + x] = best;
            else atomicMin(&keys[size_t(y) * W + x], best);
        }
    }
}

// ---------------------------------------------------------------------------
// K5 -- left/right check on WTA keys.  refine.hpp:39-54: valid(x) <=>
// xr = lround(x - dL) in [0, W) and |dL - dR(xr)| <= tol (inclusive, double).
// Also emits the (all-valid) WTA maps as float when requested, the band-local
// max_bin of the checked map (refine.hpp:68-72) and the list of invalid
// pixels in the refine band [rb0, rb1).
__global__ void k_lr_check_keys(const uint32_t* __restrict__ kl, const uint32_t* __restrict__ kr, int W,
                                int rows, double tol, float* __restrict__ chk_d, uint8_t* __restrict__ chk_v,
                                float* __restrict__ left_d, float* __restrict__ right_d, int rb0, int rb1,
                                int* __restrict__ counters, int* __restrict__ inv) {
    const size_t total = size_t(rows) * W;
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < total;
    int dl = 0;
    bool ok = false;
    int yy = 0;
    if (in) {
        yy = int(i / W);
        const int x = int(i - size_t(yy) * W);
        dl = int(kl[i] & 0xFFFFu);
        const int xr = x - dl;
        ok = xr >= 0 && xr < W;
        if (ok) ok = fabs(double(dl) - double(kr[size_t(yy) * W + xr] & 0xFFFFu)) <= tol;
        chk_d[i] = float(dl);
        chk_v[i] = ok ? 1 : 0;
        if (left_d) left_d[i] = float(dl);
        if (right_d) right_d[i] = float(kr[i] & 0xFFFFu);
    }
    const unsigned full = 0xFFFFFFFFu;
    const int mb = __reduce_max_sync(full, (in && ok) ? dl : 0);
    const bool need = in && !ok && yy >= rb0 && yy < rb1;
    const unsigned ballot = __ballot_sync(full, need);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) {
        atomicMax(&counters[0], mb);
        if (ballot) base = atomicAdd(&counters[1], __popc(ballot));
    }
    base = __shfl_sync(full, base, 0);
    if (need) inv[base + __popc(ballot & ((1u << lane) - 1u))] = int(i);
}

// lr_check on float maps (per-stage API, refine.hpp:39-54).
__global__ void k_lr_check_float(const float* __restrict__ dl, const float* __restrict__ dr, int W, int H,
                                 double tol, float* __restrict__ od, uint8_t* __restrict__ ov) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= size_t(W) * H) return;
    const int y = int(i / W), x = int(i - size_t(y) * W);
    const float d = dl[i];
    const long long xr = llround(double(x) - double(d));
    bool ok = xr >= 0 && xr < W;
    if (ok) ok = fabs(double(d) - double(dr[size_t(y) * W + xr])) <= tol;
    od[i] = d;
    ov[i] = ok ? 1 : 0;
}

// ---------------------------------------------------------------------------
// K6 -- bilateral voting refinement.  refine.hpp:62-111.  Warp per invalid
// pixel.  Voters of one window row are examined 32 at a time (lane = column);
// their bin lround(d) and weight (exact host table, refine.hpp:30-35) are
// formed in parallel, then folded into the per-warp double bins strictly in
// row-major voter order (the owner lane of a bin performs its adds in
// sequence), so every bin sum is bit-identical to the reference's.  Argmax:
// strict '>' from bin 0 == smallest bin among the maxima.
__global__ void k_vote_refine(const float* __restrict__ cd, const uint8_t* __restrict__ cv,
                              const uint8_t* __restrict__ gray, int W, int rows, int radius,
                              const double* __restrict__ wtab, int ncol, const int16_t* __restrict__ s2col,
                              const int* __restrict__ counters, const int* __restrict__ inv,
                              int nbins_cap, float* __restrict__ od, uint8_t* __restrict__ ov) {
    extern __shared__ __align__(16) double sbins[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    double* bins = sbins + size_t(warp) * nbins_cap;
    const int max_bin = counters[0];
    const int n_inv = counters[1];
    const unsigned full = 0xFFFFFFFFu;
    for (int idx = blockIdx.x * nwarps + warp; idx < n_inv; idx += gridDim.x * nwarps) {
        const int p = inv[idx];
        const int y = p / W, x = p - y * W;
        const int u = gray[p];
        for (int b = lane; b <= max_bin; b += 32) bins[b] = 0.0;
        __syncwarp();
        const int y0 = max(0, y - radius), y1 = min(rows - 1, y + radius);
        const int x0 = max(0, x - radius), x1 = min(W - 1, x + radius);
        bool any = false;
        for (int py = y0; py <= y1; ++py) {
            const int dy2 = (py - y) * (py - y);
            for (int cx = x0; cx <= x1; cx += 32) {
                const int px = cx + lane;
                const size_t j = size_t(py) * W + px;
                const bool valid = px <= x1 && cv[j];
                int bin = 0;
                double wgt = 0.0;
                if (valid) {
                    bin = int(llround(double(cd[j])));
                    const int v = gray[j];
                    const int hi = max(u, v), lo = min(u, v);
                    const int s = (px - x) * (px - x) + dy2;
                    wgt = __ldg(wtab + (size_t(hi * (hi + 1) / 2 + lo) * ncol + s2col[s]));
                }
                unsigned m = __ballot_sync(full, valid);
                any |= m != 0;
                while (m) {
                    const int i = __ffs(m) - 1;
                    m &= m - 1;
                    const int b = __shfl_sync(full, bin, i);
                    const double wv = __shfl_sync(full, wgt, i);
                    if (lane == (b & 31)) bins[b] += wv;
                }
            }
        }
        __syncwarp();
        if (!any) {
            if (lane == 0) {
                od[p] = 0.0f;
                ov[p] = 0;
            }
            continue;
        }
        double bv = -1.0;
        int bb = 0x7FFFFFFF;
        for (int b = lane; b <= max_bin; b += 32)
            if (bins[b] > bv) {
                bv = bins[b];
                bb = b;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov2 = __shfl_xor_sync(full, bv, o);
            const int ob = __shfl_xor_sync(full, bb, o);
            if (ov2 > bv || (ov2 == bv && ob < bb)) {
                bv = ov2;
                bb = ob;
            }
        }
        if (lane == 0) {
            od[p] = float(bb);
            ov[p] = 1;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// K6' -- voting refinement, thread per invalid pixel (refine.hpp:62-111).
// Each thread walks its clipped (2r+1)^2 window in row-major order and adds
// every valid voter's exact weight to its own column of double bins in
// shared memory ([bin][thread]: a lane always hits its own bank pair, so any
// mix of bins is conflict-free).  Per bin the additions happen in the
// reference's voter order, so the sums are bit-identical.  Voter data comes
// pre-packed (k_make_vmap: bin | gray << 16 | valid << 24); the window offset
// (dy, dx) is warp-uniform, so the distance column of the weight table is a
// broadcast.  Used when the bins fit (nbins * 8 B * 32 threads); otherwise
// the warp-per-pixel k_vote_refine runs.
__global__ void k_make_vmap(const float* __restrict__ cd, const uint8_t* __restrict__ cv,
                            const uint8_t* __restrict__ gray, size_t n, uint32_t* __restrict__ vmap) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t g = gray ? uint32_t(gray[i]) << 16 : 0u;
    vmap[i] = cv[i] ? (g | (1u << 24) | uint32_t(llround(double(cd[i])))) : g;
}

// ---------------------------------------------------------------------------
// K6'' -- voting refinement with device-computed weights.  vote_weight
// (refine.hpp:30-35) = exp(-(double(lab_sad)/lc + sqrt(dx^2+dy^2)/le)):
// lab_sad in float (same association), the divisions and the sum in IEEE
// double, and exp by a restatement of glibc's e_exp.c (FMA build) whose
// table and constants come from the host's libm and were validated bit for
// bit against it (bsmh::glibc_exp_params).  sqrt(s)/le depends only on the
// warp-uniform window offset and comes from a small host table.  Thread per
// invalid pixel, own column of double bins in shared memory; per bin the adds
// follow the reference's row-major voter order.
struct ExpDev {
    double invln2N, shift, negln2hiN, negln2loN, c2, c3, c4, c5;
};

__device__ __forceinline__ double exp_glibc(double x, const ExpDev& p, const unsigned long long* tab) {
    // e_exp.c: |x| < 2^-54 -> 1 + x;  |x| >= 1024 -> 0 / inf;  512 <= |x| < 1024
    // -> specialcase (the scale is built with a biased exponent).
    const unsigned long long xb = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned abstop = unsigned(xb >> 52) & 0x7ffu;
    bool special = false;
    if (abstop - 0x3c9u >= 0x3fu) {
        if (int(abstop) - 0x3c9 < 0) return 1.0 + x;
        if (abstop >= 0x409u) return (xb >> 63) ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
        special = true;
    }
    double kd = fma(x, p.invln2N, p.shift);
    const unsigned long long ki = static_cast<unsigned long long>(__double_as_longlong(kd));
    kd -= p.shift;
    const double r = fma(kd, p.negln2loN, fma(kd, p.negln2hiN, x));
    const unsigned idx = 2u * unsigned(ki & 127ull);
    const unsigned long long top = ki << 45;
    const double tail = __longlong_as_double(static_cast<long long>(tab[idx]));
    unsigned long long sbits = tab[idx + 1] + top;
    const double r2 = r * r;
    const double tmp = fma(r2 * r2, fma(r, p.c5, p.c4), fma(fma(r, p.c3, p.c2), r2, tail + r));
    if (!special) {
        const double scale = __longlong_as_double(static_cast<long long>(sbits));
        return fma(scale, tmp, scale);
    }
    if (!(ki & 0x80000000ull)) {  // k > 0 (x >= 512): overflow range
        sbits -= 1009ull << 52;
        const double scale = __longlong_as_double(static_cast<long long>(sbits));
        return 0x1p1009 * __dadd_rn(scale, __dmul_rn(scale, tmp));
    }
    sbits += 1022ull << 52;  // k < 0: subnormal range, rounded once
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    const double st = __dmul_rn(scale, tmp);
    double y = __dadd_rn(scale, st);
    if (y < 1.0) {
        const double hi = __dadd_rn(y, 1.0);
        const double lo = __dadd_rn(__dsub_rn(scale, y), st);
        const double l2 = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo);
        y = __dsub_rn(__dadd_rn(l2, hi), 1.0);
        if (y == 0.0) y = 0.0;
    }
    return __dmul_rn(y, 0x1p-1022);
}

// K6d -- voting refinement, NP invalid pixels per warp (LPP = 32/NP lanes
// each).  Per window row the LPP lanes of a pixel form the bins and weights of
// LPP consecutive voters in parallel (weight from the exact host table, or
// the device exp for Lab planes; the loads of a batch of CB chunks are issued
// together), stage them, then fold them in voter order: lane sl owns the bins
// b with (b % LPP) == sl, finds its entries of the chunk from ballots of the
// valid flag and the residue bits, and walks them in order, keeping its
// current bin's running sum in a register.  Per bin the additions are
// therefore the reference's row-major sequence; the NP pixels fold side by
// side.
template <int NP, bool DEVEXP>
__global__ void __launch_bounds__(256, 1) k_vote_refine_fold(
    const uint32_t* __restrict__ vmap, const float4* __restrict__ lab, const float* __restrict__ lab256, int W,
    int rows, int radius, double lc, const double* __restrict__ e_over_le, ExpDev ep,
    const unsigned long long* __restrict__ etab, const double* __restrict__ wtab, int ncol,
    const int16_t* __restrict__ s2col, const int* __restrict__ counters, const int* __restrict__ inv, int nbins_cap,
    float* __restrict__ od, uint8_t* __restrict__ ov, int* __restrict__ work) {
    constexpr int LPP = 32 / NP;
    extern __shared__ __align__(16) double fsm[];
    unsigned long long* stab = reinterpret_cast<unsigned long long*>(fsm);  // 256 (DEVEXP)
    float* slab = reinterpret_cast<float*>(stab + 256);                     // 768 (DEVEXP, gray)
    const int nwarps = blockDim.x >> 5;
    double* sw_all = reinterpret_cast<double*>(slab + 768);                 // [warps][32] staged weights
    int* sb_all = reinterpret_cast<int*>(sw_all + nwarps * 32);             // [warps][32] staged bins
    double* bins_all = reinterpret_cast<double*>(sb_all + nwarps * 32);     // [warps][NP][nbins_cap]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / LPP, sl = lane % LPP;
    if (DEVEXP) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) stab[i] = etab[i];
        if (!lab)
            for (int i = threadIdx.x; i < 768; i += blockDim.x) slab[i] = lab256[i];
    }
    __syncthreads();
    double* sw = sw_all + warp * 32;
    int* sbn = sb_all + warp * 32;
    double* bins = bins_all + size_t(warp * NP + sub) * nbins_cap;
    const unsigned full = 0xFFFFFFFFu;
    const unsigned submask = (LPP == 32) ? full : (((1u << LPP) - 1u) << (sub * LPP));
    const int max_bin = counters[0];
    const int n_inv = counters[1];
    // groups of NP pixels are taken from a work counter (*work == 0 at
    // launch): the voter count varies per pixel, so a static stride leaves a tail
    auto grab = [&]() {
        int b = 0;
        if (lane == 0) b = atomicAdd(work, NP);
        return __shfl_sync(0xFFFFFFFFu, b, 0);
    };
    for (int base = grab(); base < n_inv; base = grab()) {  // warp-uniform loop
        const int idx = base + sub;
        const bool live = idx < n_inv;
        const int p = live ? inv[idx] : 0;
        const int y = p / W, x = p - y * W;
        const uint32_t e0 = vmap[p];
        const int u = int((e0 >> 16) & 0xFFu);
        float lx0 = 0.f, lx1 = 0.f, lx2 = 0.f;
        if (DEVEXP) {
            if (lab) {
                const float4 c = lab[p];
                lx0 = c.x;
                lx1 = c.y;
                lx2 = c.z;
            } else {
                lx0 = slab[3 * u];
                lx1 = slab[3 * u + 1];
                lx2 = slab[3 * u + 2];
            }
        }
        for (int b = sl; b <= max_bin; b += LPP) bins[b] = 0.0;
        int cur = -1;
        double acc = 0.0;
        bool any = false;
        const int tu = u * (u + 1) / 2;
        // Per window row, the loads of CB chunks (LPP voters each) are issued
        // together (vmap, then the weights), then the chunks fold in order:
        // one L2 round trip per batch instead of one per chunk.
        constexpr int CB = 6;
        const int nch = (2 * radius + LPP) / LPP;  // ceil((2r + 1) / LPP)
        for (int dy = -radius; dy <= radius; ++dy) {
            const int py = y + dy;
            const bool rowok = live && py >= 0 && py < rows;
            const uint32_t* row = vmap + size_t(rowok ? py : 0) * W;
            const int dy2 = dy * dy;
            for (int c0 = 0; c0 < nch; c0 += CB) {
                uint32_t ev[CB];
#pragma unroll
                for (int k = 0; k < CB; ++k) {
                    const int dx = -radius + (c0 + k) * LPP + sl;
                    const int px = x + dx;
                    ev[k] = (rowok && dx <= radius && px >= 0 && px < W) ? __ldg(row + px) : 0u;
                }
                int bv[CB];
                double wv[CB];
#pragma unroll
                for (int k = 0; k < CB; ++k) {
                    const uint32_t e = ev[k];
                    const int dx = -radius + (c0 + k) * LPP + sl;
                    bv[k] = -1;
                    wv[k] = 0.0;
                    if (e & (1u << 24)) {
                        bv[k] = int(e & 0xFFFFu);
                        const int v = int((e >> 16) & 0xFFu);
                        if (DEVEXP) {
                            float l0, l1, l2;
                            if (lab) {
                                const float4 o = __ldg(lab + size_t(py) * W + x + dx);
                                l0 = o.x;
                                l1 = o.y;
                                l2 = o.z;
                            } else {
                                l0 = slab[3 * v];
                                l1 = slab[3 * v + 1];
                                l2 = slab[3 * v + 2];
                            }
                            const float sad = __fadd_rn(__fadd_rn(fabsf(__fsub_rn(lx0, l0)), fabsf(__fsub_rn(lx1, l1))),
                                                        fabsf(__fsub_rn(lx2, l2)));
                            const double arg = -(__ddiv_rn(double(sad), lc) + __ldg(e_over_le + dx * dx + dy2));
                            wv[k] = exp_glibc(arg, ep, stab);
                        } else {
                            const int tri = v >= u ? (v * (v + 1) / 2 + u) : (tu + v);
                            wv[k] = __ldg(wtab + size_t(tri) * ncol + s2col[dx * dx + dy2]);
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < CB; ++k) {
                    if (c0 + k >= nch) break;  // warp-uniform
                    const int bin = bv[k];
                    const double w = wv[k];
                    // owner lane of bin b: b % LPP; the entries each owner
                    // takes come from four ballots (valid + residue bits)
                    const unsigned vb = __ballot_sync(full, bin >= 0) & submask;
                    unsigned mine = vb >> (sub * LPP);
#pragma unroll
                    for (int kb = 0; (1 << kb) < LPP; ++kb) {
                        const unsigned bk = __ballot_sync(full, (bin >> kb) & 1) >> (sub * LPP);
                        mine &= ((sl >> kb) & 1) ? bk : ~bk;
                    }
                    any |= vb != 0u;
                    sbn[lane] = bin;
                    sw[lane] = w;
                    __syncwarp();
                    while (mine) {
                        const int j = sub * LPP + __ffs(mine) - 1;
                        mine &= mine - 1;
                        const int b = sbn[j];
                        if (b != cur) {
                            if (cur >= 0) bins[cur] = acc;
                            cur = b;
                            acc = bins[b];
                        }
                        acc += sw[j];
                    }
                    __syncwarp();
                }
            }
        }
        if (cur >= 0) bins[cur] = acc;
        __syncwarp();
        // argmax: strict '>' from bin 0 == first bin holding the maximum
        double bv = -1.0;
        int bb = 0x7FFFFFFF;
        for (int b = sl; b <= max_bin; b += LPP)
            if (bins[b] > bv) {
                bv = bins[b];
                bb = b;
            }
#pragma unroll
        for (int o = LPP / 2; o > 0; o >>= 1) {
            const double ov2 = __shfl_xor_sync(full, bv, o);
            const int ob = __shfl_xor_sync(full, bb, o);
            if (ov2 > bv || (ov2 == bv && ob < bb)) {
                bv = ov2;
                bb = ob;
            }
        }
        if (live && sl == 0) {
            od[p] = any ? float(bb) : 0.0f;
            ov[p] = any ? 1 : 0;
        }
        __syncwarp();
    }
}

__global__ void k_exp_eval(const double* __restrict__ x, int n, ExpDev ep, const unsigned long long* __restrict__ tab,
                           double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = exp_glibc(x[i], ep, tab);
}

// ---------------------------------------------------------------------------
// Layout converters for the per-stage API (reference AoS u64 <-> device SoA).
__global__ void k_aos_to_soa(const uint32_t* __restrict__ src, int W, int H, int NW, int Wp,
                             uint32_t* __restrict__ dst) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;  // over (y, w, x)
    const size_t total = size_t(H) * NW * Wp;
    if (i >= total) return;
    const int x = int(i % Wp);
    const size_t yw = i / Wp;
    const int w = int(yw % NW), y = int(yw / NW);
    dst[i] = x < W ? src[(size_t(y) * W + x) * NW + w] : 0u;
}

__global__ void k_soa_to_aos(const uint32_t* __restrict__ src, int W, int H, int NW, int Wp,
                             uint32_t* __restrict__ dst) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;  // over (y, x, w)
    const size_t total = size_t(H) * W * NW;
    if (i >= total) return;
    const int w = int(i % NW);
    const size_t yx = i / NW;
    const int x = int(yx % W), y = int(yx / W);
    dst[i] = src[(size_t(y) * NW + w) * Wp + x];
}

// k_soa_to_aos with the pipeline's bit order undone: reference bit k of a
// pixel's string is device bit pos[k].
__global__ void k_soa_to_aos_perm(const uint32_t* __restrict__ src, int W, int H, int NW, int Wp,
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
        v |= ((__ldg(src + (size_t(y) * NW + (j >> 5)) * Wp + x) >> (j & 31)) & 1u) << b;
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

}  // namespace

// ===========================================================================
// Context.
enum Timing { T_H2D, T_DESC, T_MASK, T_WTA_L, T_WTA_R, T_WTA_U, T_LR, T_REFINE, T_D2H, T_COUNT };
static const char* kTimingNames = "h2d,descriptor,mask,wta_left,wta_right,wta_unmasked,lr_check,refine,d2h";

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap) return BSM_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) return set_err(BSM_CUDA_ERROR, std::string("CUDA: cudaMalloc: ") + cudaGetErrorString(e));
        cap = bytes;
        return BSM_OK;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct bsm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sm_count = 0;
    // pattern
    int n = 0, window = 0, half = 0, NW = 0, u = 0;
    int mslots = 0;                 // rank-table slots used by the mask kernels
    std::vector<int> slot_used;     // slot -> used-offset index (-1: empty)
    int mch = 4;                    // k_mask4 / k_mask_f32 chunks of 32 positions per lane (1, 2, 4)
    std::vector<int> order;         // bit position -> pair index (identity unless permuted)
    bool permuted = false;
    DevBuf d_pos;                   // pair index -> bit position (permuted only)
    double slot_cost[2] = {0, 0};   // avg wavefronts per gather before/after placement
    std::vector<int16_t> pairs;
    std::vector<int2> pair_xy;  // (px,py),(qx,qy) packed later per tile width
    std::vector<int16_t> used;  // used offsets as dy*(2h+1)+dx index list (host)
    DevBuf d_desc4, d_pqb, d_uoff, d_uxy;
    DevBuf d_descf, d_rgb_gray, d_rgb_lab, planes;
    int descf_tw = -1;
    bool rgb_ready = false;
    int desc4_tw = -1, uoff_tw = -1;
    // tables
    float gray_lut[256], lab_lut[768];
    DevBuf d_rank;
    DevBuf d_wtab, d_s2col;
    bool exp_ok = false;            // device exp restatement validated against host libm
    int refine_mode = -1;           // -1: auto, 0: scan kernel, 1: smem bins, 2: weight table
    std::string exp_why;
    ExpDev exp_dev{};
    DevBuf d_etab, d_elam, d_lab256;
    double elam_le = 0;
    int elam_radius = -1;
    double wt_lc = 0, wt_le = 0;
    int wt_radius = -1, wt_ncol = 0;
    // scratch
    DevBuf img_l, img_r, fdl, fml, fdr, fmr, keys_l, keys_r, keys_u;
    DevBuf chk_d, chk_v, ref_d, ref_v, lw_d, rw_d, un_d, counters, inv, vmap;
    DevBuf aux0, aux1, aux2, aux3;
    int last_W = 0, last_rows = 0, last_unmasked = 0, last_r0 = 0, last_out0 = 0, last_out_rows = 0;
    // instrumentation
    bool profiling = false;
    static constexpr int kEvPerSlot = 4;  // a stage may run several times per call (two views)
    cudaEvent_t ev[T_COUNT][kEvPerSlot][2] = {};
    int ev_used[T_COUNT] = {};
    int launches = 0;
    DevBuf popc_out;
};

namespace {

struct Scope {  // brackets one pipeline stage with events when profiling
    bsm_ctx* c;
    int t;
    int slot = -1;
    Scope(bsm_ctx* c_, int t_) : c(c_), t(t_) {
        if (c->profiling && c->ev_used[t] < bsm_ctx::kEvPerSlot) {
            slot = c->ev_used[t]++;
            cudaEventRecord(c->ev[t][slot][0], c->stream);
        }
    }
    ~Scope() {
        if (slot >= 0) cudaEventRecord(c->ev[t][slot][1], c->stream);
    }
};

int check_launch(bsm_ctx* c, const char* what) {
    ++c->launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(BSM_CUDA_ERROR, std::string("CUDA: launch ") + what + ": " + cudaGetErrorString(e));
    return BSM_OK;
}

#define BSM_TRY(x)                  \
    do {                            \
        int rc_ = (x);              \
        if (rc_ != BSM_OK) return rc_; \
    } while (0)

// Tile-relative offset tables depend on the staged tile width.
int desc4_tile_width(int half) { return round_up(kD2TX * 4 + 2 * half + 8, 16); }

// k_descriptor4's per-pair table: word offsets of both endpoints in its
// phased 4-byte-window tile, relative to the thread's base word:
// (half + px) % 4 selects the phase plane, py*TWs/4 + (half + px)/4 the word.
int ensure_desc4_table(bsm_ctx* c) {
    const int TWs = desc4_tile_width(c->half);
    if (c->desc4_tw == TWs) return BSM_OK;
    const int G = (c->n + 31) / 32;
    std::vector<int2> t(size_t(G) * 32, make_int2(0, 0));
    for (int i = 0; i < c->n; ++i) {
        const int16_t* p = &c->pairs[4 * size_t(c->order[size_t(i)])];
        const int TH = kD2TY * kD2Rows + 2 * c->half, S4 = TWs * TH / 4;
        auto woff = [&](int px, int py) { return ((c->half + px) & 3) * S4 + py * (TWs / 4) + ((c->half + px) >> 2); };
        t[size_t(i)] = make_int2(woff(p[0], p[1]), woff(p[2], p[3]));
    }
    BSM_TRY(c->d_desc4.ensure(t.size() * sizeof(int2)));
    BSM_CUDA(cudaMemcpy(c->d_desc4.p, t.data(), t.size() * sizeof(int2), cudaMemcpyHostToDevice));
    c->desc4_tw = TWs;
    return BSM_OK;
}


// Row stride of the k_mask4 / k_mask_f32 window tiles: kM3Px + 2h columns plus
// up to 3 of alignment slack, a multiple of 4 (word-wide tile loads).
int mask4_tw(int half) { return round_up(kM3Px + 2 * half + 3, 4); }

int ensure_mask_offsets(bsm_ctx* c, int TW) {
    if (c->uoff_tw == TW) return BSM_OK;
    const int side = 2 * c->half + 1;
    std::vector<int32_t> o(size_t(c->mslots), 0);  // empty slots read the centre (harmless)
    for (int k = 0; k < c->mslots; ++k) {
        const int ui = c->slot_used[size_t(k)];
        if (ui < 0) continue;
        const int dy = c->used[size_t(ui)] / side - c->half, dx = c->used[size_t(ui)] % side - c->half;
        o[size_t(k)] = dy * TW + dx;
    }
    BSM_TRY(c->d_uoff.ensure(std::max<size_t>(4, o.size() * 4)));
    BSM_CUDA(cudaMemcpy(c->d_uoff.p, o.data(), o.size() * 4, cudaMemcpyHostToDevice));
    // the same slots as (dy << 16) | (dx & 0xFFFF) for the float-plane kernel
    std::vector<int32_t> xy(size_t(c->mslots), 0);
    for (int k = 0; k < c->mslots; ++k) {
        const int ui = c->slot_used[size_t(k)];
        if (ui < 0) continue;
        const int dy = c->used[size_t(ui)] / side - c->half, dx = c->used[size_t(ui)] % side - c->half;
        xy[size_t(k)] = int32_t(uint32_t(dy) << 16 | (uint32_t(dx) & 0xFFFFu));
    }
    BSM_TRY(c->d_uxy.ensure(std::max<size_t>(4, xy.size() * 4)));
    BSM_CUDA(cudaMemcpy(c->d_uxy.p, xy.data(), xy.size() * 4, cudaMemcpyHostToDevice));
    c->uoff_tw = TW;
    return BSM_OK;
}

int ensure_weight_table(bsm_ctx* c, double lc, double le, int radius) {
    if (c->wt_radius == radius && c->wt_lc == lc && c->wt_le == le) return BSM_OK;
    std::vector<double> w;
    std::vector<int16_t> s2col;
    int ncol = 0;
    bsmh::vote_weight_table(c->lab_lut, lc, le, radius, w, s2col, ncol);
    BSM_TRY(c->d_wtab.ensure(w.size() * 8));
    BSM_TRY(c->d_s2col.ensure(s2col.size() * 2));
    BSM_CUDA(cudaMemcpy(c->d_wtab.p, w.data(), w.size() * 8, cudaMemcpyHostToDevice));
    BSM_CUDA(cudaMemcpy(c->d_s2col.p, s2col.data(), s2col.size() * 2, cudaMemcpyHostToDevice));
    c->wt_lc = lc;
    c->wt_le = le;
    c->wt_radius = radius;
    c->wt_ncol = ncol;
    return BSM_OK;
}

int check_pattern(bsm_ctx* c) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    if (c->n <= 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: no sampling pattern set (bsm_set_pattern)");
    return BSM_OK;
}



size_t mask4_smem(const bsm_ctx* c) {
    const int TW = mask4_tw(c->half), TH = 2 * c->half + 1;
    return size_t(round_up(c->mslots + 1, 4)) * 4 + size_t(kM3Px) * mask4_stage_stride(c->mch) * 4 + 512 +
           size_t(TW) * TH;
}


// Descriptors + masks of rows [ybeg, ybeg + rows) of a W x H view on device.
int field_device(bsm_ctx* c, const uint8_t* img, int W, int H, int ybeg, int rows, uint32_t* desc, uint32_t* mask) {
    const int Wp = round_up(W, 128);
    BSM_TRY(ensure_mask_offsets(c, mask4_tw(c->half)));
    {
        Scope s(c, T_DESC);
        BSM_TRY(ensure_desc4_table(c));
        const int TWs = desc4_tile_width(c->half);
        const size_t sm = size_t(TWs) * (kD2TY * kD2Rows + 2 * c->half) * 5 + 16;
        dim3 grid(Wp / (kD2TX * 4), (rows + kD2TY * kD2Rows - 1) / (kD2TY * kD2Rows));
        // split the word range over grid.z until there are ~16 CTAs per SM (the
        // tail of a partial last wave dominates otherwise; c2: 759 -> 3036 CTAs)
        grid.z = unsigned(std::max(1, std::min((c->NW + 7) / 8, (16 * c->sm_count + int(grid.x * grid.y) - 1) /
                                                                    int(grid.x * grid.y))));
        BSM_CUDA(cudaFuncSetAttribute(k_descriptor4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        k_descriptor4<<<grid, dim3(kD2TX, kD2TY), sm, c->stream>>>(img, W, H, ybeg, rows, c->d_desc4.as<int2>(),
                                                                    c->n, c->half, TWs, c->NW, Wp, desc);
        BSM_TRY(check_launch(c, "descriptor"));
    }
    {
        Scope s(c, T_MASK);
        const size_t sm4 = mask4_smem(c);
        dim3 grid3(Wp / kM3Px, rows);
        auto launch = [&](auto kern) -> int {
            BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm4)));
            kern<<<grid3, 32, sm4, c->stream>>>(img, W, H, ybeg, rows, c->d_pqb.as<uint4>(),
                                                c->d_pqb.as<uint4>() + kPqTable / 4, c->n, c->d_uoff.as<int32_t>(),
                                                c->mslots, round_up(c->mslots + 1, 4), c->d_rank.as<uint8_t>(),
                                                c->half, mask4_tw(c->half), c->NW, Wp, mask);
            return BSM_OK;
        };
        // chunks of 32 positions per lane: the work scales with n
        BSM_TRY(c->mch == 1   ? launch(k_mask4<1>)
                : c->mch == 2 ? launch(k_mask4<2>)
                : c->mch == 4 ? launch(k_mask4<4>)
                              : launch(k_mask4<8>));
        BSM_TRY(check_launch(c, "mask"));
    }
    return BSM_OK;
}

// WTA keys of rows [0, rows) of device fields (SoA); keys: rows x W.
// Tensor map of a device field [rows][NW][Wp] u32 for TMA boxes of box_x
// columns x kCostK words x 1 row; out-of-range boxes read zeros.
int field_tensor_map(CUtensorMap* map, const uint32_t* field, int W, int NW, int rows, int box_x) {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        BSM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess)
            return set_err(BSM_CUDA_ERROR, "CUDA: cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    const int Wp = round_up(W, 128);
    const cuuint64_t dims[3] = {cuuint64_t(Wp), cuuint64_t(NW), cuuint64_t(std::max(rows, 1))};
    const cuuint64_t strides[2] = {cuuint64_t(Wp) * 4, cuuint64_t(NW) * Wp * 4};
    const cuuint32_t box[3] = {cuuint32_t(box_x), cuuint32_t(kCostK), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(field), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(BSM_CUDA_ERROR, "CUDA: cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return BSM_OK;
}

int wta_device(bsm_ctx* c, const uint32_t* dref, const uint32_t* mref, const uint32_t* doth, int W, int rows,
               int d_max, bool right, bool masked, uint32_t* keys, int timing) {
    Scope s(c, timing);
    const int Wp = round_up(W, 128);
    const int dz = (d_max + kCostDisp - 1) / kCostDisp;
    if (dz > 1) BSM_CUDA(cudaMemsetAsync(keys, 0xFF, size_t(rows) * W * 4, c->stream));
    dim3 grid(dz, Wp / kCostTile, rows);
    const size_t stage_words = size_t(masked ? 2 : 1) * kCostK * kCostTile + size_t(kCostK) * (kCostTile + kCostDisp);
    const size_t sm = (kCostStages * stage_words + 8 * kCostTile) * 4 + kCostStages * 16;  // + full/empty mbarriers
    CUtensorMap tr, tmk, to;
    BSM_TRY(field_tensor_map(&tr, dref, W, c->NW, rows, kCostTile));
    BSM_TRY(field_tensor_map(&tmk, mref ? mref : dref, W, c->NW, rows, kCostTile));
    BSM_TRY(field_tensor_map(&to, doth, W, c->NW, rows, kCostTile + kCostDisp));
    auto launch = [&](auto kern) -> int {
        BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        kern<<<grid, 256, sm, c->stream>>>(tr, tmk, to, W, rows, c->NW, d_max, keys, 2u);
        return BSM_OK;
    };
    if (right) BSM_TRY(masked ? launch(k_cost_wta<true, true>) : launch(k_cost_wta<true, false>));
    else BSM_TRY(masked ? launch(k_cost_wta<false, true>) : launch(k_cost_wta<false, false>));
    return check_launch(c, "cost_wta");
}

int ensure_elam(bsm_ctx* c, double le, int radius) {
    if (c->elam_le == le && c->elam_radius == radius) return BSM_OK;
    std::vector<double> t(size_t(2 * radius * radius) + 1);
    for (size_t k = 0; k < t.size(); ++k) t[k] = std::sqrt(double(k)) / le;  // sqrt(dx*dx + dy*dy) / lambda_e
    BSM_TRY(c->d_elam.ensure(t.size() * 8));
    BSM_CUDA(cudaMemcpy(c->d_elam.p, t.data(), t.size() * 8, cudaMemcpyHostToDevice));
    c->elam_le = le;
    c->elam_radius = radius;
    return BSM_OK;
}

// Refinement of the invalid pixels listed in c->inv (count in counters[1],
// max_bin in counters[0]) into c->ref_d / c->ref_v (pre-filled with the input
// map).  nbins_max bounds max_bin + 1.  lab: per-pixel Lab plane or nullptr
// (grayscale: the gray value indexes the Lab table).
int refine_launch(bsm_ctx* c, const float* cd, const uint8_t* cv, const uint8_t* gray, const float4* lab, int W,
                  int rows, int radius, int nbins_max, double lc, double le) {
    const size_t px = size_t(rows) * W;
    const int nbins = round_up(std::max(nbins_max, 1), 32);
    const int tb = 256;
    int mode = c->refine_mode >= 0 ? c->refine_mode : (lab ? 4 : 3);
    if (lab && mode != 4) mode = 4;  // Lab planes: the weight table only covers gray pairs
    if (mode == 4 && !c->exp_ok) {
        if (lab) return set_err(BSM_UNSUPPORTED, "bsm: colour refine needs the device exp (" + c->exp_why + ")");
        mode = 3;
    }
    if (mode == 3 || mode == 4) {
        const bool devexp = mode == 4;
        const size_t fixed = 256 * 8 + 768 * 4;
        // bins of NP pixels per warp: 4 (default) or 1 for very wide disparity ranges
        const int np = (fixed + 8 * 32 * 12 + size_t(8) * 4 * nbins * 8 <= 200 * 1024) ? 4 : 1;
        const int warps =
            std::min(8, int((200 * 1024 - fixed) / (size_t(32) * 12 + size_t(np) * nbins * 8)));
        if (warps >= 1) {
            if (devexp) BSM_TRY(ensure_elam(c, le, radius));
            else BSM_TRY(ensure_weight_table(c, lc, le, radius));
            BSM_TRY(c->vmap.ensure(px * 4));
            k_make_vmap<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(cd, cv, gray, px, c->vmap.as<uint32_t>());
            BSM_TRY(check_launch(c, "make_vmap"));
            const size_t sm = fixed + size_t(warps) * 32 * 12 + size_t(warps) * np * nbins * 8;
            auto kern = np == 4 ? (devexp ? k_vote_refine_fold<4, true> : k_vote_refine_fold<4, false>)
                                : (devexp ? k_vote_refine_fold<1, true> : k_vote_refine_fold<1, false>);
            BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
            const int per_sm = std::max(1, std::min(4, int((220 * 1024) / sm)));
            BSM_CUDA(cudaMemsetAsync(c->counters.as<int>() + 2, 0, 4, c->stream));  // work counter
            kern<<<c->sm_count * per_sm, warps * 32, sm, c->stream>>>(
                c->vmap.as<uint32_t>(), lab, c->d_lab256.as<float>(), W, rows, radius, lc, c->d_elam.as<double>(),
                c->exp_dev, c->d_etab.as<unsigned long long>(), c->d_wtab.as<double>(), c->wt_ncol,
                c->d_s2col.as<int16_t>(), c->counters.as<int>(), c->inv.as<int>(), nbins, c->ref_d.as<float>(),
                c->ref_v.as<uint8_t>(), c->counters.as<int>() + 2);
            return check_launch(c, "vote_refine_fold");
        }
        if (lab) return set_err(BSM_UNSUPPORTED, "bsm: disparity range too wide for the colour refine bins");
    }
    // mode 2 (or bins too wide for the fold): warp per pixel, exact host weight table
    BSM_TRY(ensure_weight_table(c, lc, le, radius));
    const int warps = std::max(1, std::min(8, int((96 * 1024) / (size_t(nbins) * 8))));
    const size_t sm = size_t(warps) * nbins * 8;
    BSM_CUDA(cudaFuncSetAttribute(k_vote_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    k_vote_refine<<<c->sm_count * 8, warps * 32, sm, c->stream>>>(
        cd, cv, gray, W, rows, radius, c->d_wtab.as<double>(), c->wt_ncol, c->d_s2col.as<int16_t>(),
        c->counters.as<int>(), c->inv.as<int>(), nbins, c->ref_d.as<float>(), c->ref_v.as<uint8_t>());
    return check_launch(c, "vote_refine");
}

int validate_params(const bsm_params* p) {
    if (!p) return set_err(BSM_INVALID_ARGUMENT, "bsm: null params");
    if (p->d_max < 1) return set_err(BSM_INVALID_ARGUMENT, "config: d_max must be set (>= 1)");
    if (p->d_max > 65535) return set_err(BSM_UNSUPPORTED, "bsm: d_max > 65535 is outside this build's envelope");
    if (!(p->lambda_c > 0)) return set_err(BSM_INVALID_ARGUMENT, "config: lambda_c must be > 0");
    if (!(p->lambda_e > 0)) return set_err(BSM_INVALID_ARGUMENT, "config: lambda_e must be > 0");
    if (p->lr_tolerance < 0) return set_err(BSM_INVALID_ARGUMENT, "config: lr_tolerance must be >= 0");
    if (p->vote_radius < 1) return set_err(BSM_INVALID_ARGUMENT, "config: vote_radius must be >= 1");
    if (p->vote_radius > 180) return set_err(BSM_UNSUPPORTED, "bsm: vote_radius > 180 is outside this build's envelope");
    return BSM_OK;
}

// The fused device pipeline.  Views are full W x H device images; the
// refined output covers rows [out0, out0 + out_rows); fields, WTA and the
// check cover the halo-extended rows [r0, r1).
// k_descriptor_f32's per-pair table: tile-relative offsets py*TW + px.
int ensure_descf_table(bsm_ctx* c) {
    const int TW = kDfTX + 2 * c->half;
    if (c->descf_tw == TW) return BSM_OK;
    const int G = (c->n + 31) / 32;
    std::vector<int2> t(size_t(G) * 32, make_int2(0, 0));
    for (int i = 0; i < c->n; ++i) {
        const int16_t* p = &c->pairs[4 * size_t(c->order[size_t(i)])];
        t[size_t(i)] = make_int2(p[1] * TW + p[0], p[3] * TW + p[2]);
    }
    BSM_TRY(c->d_descf.ensure(t.size() * sizeof(int2)));
    BSM_CUDA(cudaMemcpy(c->d_descf.p, t.data(), t.size() * sizeof(int2), cudaMemcpyHostToDevice));
    c->descf_tw = TW;
    return BSM_OK;
}

size_t maskf_smem(const bsm_ctx* c) { return size_t(round_up(c->mslots + 1, 4)) * 4 + size_t(24) * c->mch * 32 * 4; }

// Descriptors + masks of rows [ybeg, ybeg + rows) from float gray / Lab planes.
int field_device_f32(bsm_ctx* c, const float* gray, const float4* lab, int W, int H, int ybeg, int rows,
                     uint32_t* desc, uint32_t* mask) {
    const int Wp = round_up(W, 128);
    BSM_TRY(ensure_descf_table(c));
    BSM_TRY(ensure_mask_offsets(c, mask4_tw(c->half)));
    {
        Scope s(c, T_DESC);
        const int TW = kDfTX + 2 * c->half, TH = kDfTY * kDfPY + 2 * c->half;
        const size_t sm = size_t(TW) * TH * 4;
        dim3 grid(Wp / kDfTX, (rows + kDfTY * kDfPY - 1) / (kDfTY * kDfPY));
        BSM_CUDA(cudaFuncSetAttribute(k_descriptor_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        k_descriptor_f32<<<grid, dim3(kDfTX, kDfTY), sm, c->stream>>>(gray, W, H, ybeg, rows, c->d_descf.as<int2>(),
                                                                      c->n, c->half, c->NW, Wp, desc);
        BSM_TRY(check_launch(c, "descriptor_f32"));
    }
    {
        Scope s(c, T_MASK);
        const size_t sm = maskf_smem(c);
        dim3 grid(Wp / kM3Px, rows);
        auto launch = [&](auto kern) -> int {
            BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
            kern<<<grid, 32, sm, c->stream>>>(lab, W, H, ybeg, rows,
                                              c->d_pqb.as<uint4>() + (c->mch <= 4 ? 2 * kPqTable / 4 : 0),
                                              c->d_pqb.as<uint4>() + kPqTable / 4, c->n, c->d_uxy.as<int32_t>(), c->mslots,
                                              round_up(c->mslots + 1, 4), c->NW, Wp, mask, c->half);
            return BSM_OK;
        };
        BSM_TRY(c->mch == 1   ? launch(k_mask_f32<1>)
                : c->mch == 2 ? launch(k_mask_f32<2>)
                : c->mch == 4 ? launch(k_mask_f32<4>)
                              : launch(k_mask_f32<8>));
        BSM_TRY(check_launch(c, "mask_f32"));
    }
    return BSM_OK;
}

// The 2^24-colour conversion tables on the device (built once per context).
int ensure_rgb_tables(bsm_ctx* c) {
    if (c->rgb_ready) return BSM_OK;
    std::vector<float> g, l;
    bsmh::rgb24_tables(g, l);
    BSM_TRY(c->d_rgb_gray.ensure(g.size() * 4));
    BSM_TRY(c->d_rgb_lab.ensure(l.size() * 4));
    BSM_CUDA(cudaMemcpy(c->d_rgb_gray.p, g.data(), g.size() * 4, cudaMemcpyHostToDevice));
    BSM_CUDA(cudaMemcpy(c->d_rgb_lab.p, l.data(), l.size() * 4, cudaMemcpyHostToDevice));
    c->rgb_ready = true;
    return BSM_OK;
}

// Device views of a pair: grayscale uint8 images, or float gray + Lab planes
// (colour input / arbitrary GrayImage + LabImage).
struct Views {
    const uint8_t* u8l = nullptr;
    const uint8_t* u8r = nullptr;
    const float* gl = nullptr;
    const float4* ll = nullptr;  // Lab planes, float4 (L, a, b, 0) per pixel
    const float* gr = nullptr;
    const float4* lr = nullptr;
};

int pipeline_device(bsm_ctx* c, const Views& v, int W, int H, int out0, int out_rows, const bsm_params* p,
                    bool want_unmasked) {
    BSM_TRY(check_pattern(c));
    BSM_TRY(validate_params(p));
    const int r0 = std::max(0, out0 - p->vote_radius);
    const int r1 = std::min(H, out0 + out_rows + p->vote_radius);
    const int rows = r1 - r0;
    const int Wp = round_up(W, 128);
    const size_t fbytes = size_t(rows) * c->NW * Wp * 4;
    const size_t px = size_t(rows) * W;
    BSM_TRY(c->fdl.ensure(fbytes));
    BSM_TRY(c->fml.ensure(fbytes));
    BSM_TRY(c->fdr.ensure(fbytes));
    BSM_TRY(c->fmr.ensure(fbytes));
    BSM_TRY(c->keys_l.ensure(px * 4));
    BSM_TRY(c->keys_r.ensure(px * 4));
    if (want_unmasked) BSM_TRY(c->keys_u.ensure(px * 4));
    BSM_TRY(c->chk_d.ensure(px * 4));
    BSM_TRY(c->chk_v.ensure(px));
    BSM_TRY(c->ref_d.ensure(px * 4));
    BSM_TRY(c->ref_v.ensure(px));
    BSM_TRY(c->lw_d.ensure(px * 4));
    BSM_TRY(c->rw_d.ensure(px * 4));
    if (want_unmasked) BSM_TRY(c->un_d.ensure(px * 4));
    BSM_TRY(c->counters.ensure(64));
    BSM_TRY(c->inv.ensure(px * 4));

    if (v.u8l) {
        BSM_TRY(field_device(c, v.u8l, W, H, r0, rows, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>()));
        BSM_TRY(field_device(c, v.u8r, W, H, r0, rows, c->fdr.as<uint32_t>(), c->fmr.as<uint32_t>()));
    } else {
        BSM_TRY(field_device_f32(c, v.gl, v.ll, W, H, r0, rows, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>()));
        BSM_TRY(field_device_f32(c, v.gr, v.lr, W, H, r0, rows, c->fdr.as<uint32_t>(), c->fmr.as<uint32_t>()));
    }
    BSM_TRY(wta_device(c, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>(), c->fdr.as<uint32_t>(), W, rows, p->d_max,
                       false, true, c->keys_l.as<uint32_t>(), T_WTA_L));
    BSM_TRY(wta_device(c, c->fdr.as<uint32_t>(), c->fmr.as<uint32_t>(), c->fdl.as<uint32_t>(), W, rows, p->d_max,
                       true, true, c->keys_r.as<uint32_t>(), T_WTA_R));
    if (want_unmasked)
        BSM_TRY(wta_device(c, c->fdl.as<uint32_t>(), nullptr, c->fdr.as<uint32_t>(), W, rows, p->d_max, false, false,
                           c->keys_u.as<uint32_t>(), T_WTA_U));
    {
        Scope s(c, T_LR);
        BSM_CUDA(cudaMemsetAsync(c->counters.p, 0, 64, c->stream));
        const int tb = 256;
        k_lr_check_keys<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(
            c->keys_l.as<uint32_t>(), c->keys_r.as<uint32_t>(), W, rows, p->lr_tolerance, c->chk_d.as<float>(),
            c->chk_v.as<uint8_t>(), c->lw_d.as<float>(), c->rw_d.as<float>(), out0 - r0, out0 - r0 + out_rows,
            c->counters.as<int>(), c->inv.as<int>());
        BSM_TRY(check_launch(c, "lr_check"));
        if (want_unmasked) {
            k_keys_to_float<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(c->keys_u.as<uint32_t>(), px,
                                                                              c->un_d.as<float>());
            BSM_TRY(check_launch(c, "keys_to_float"));
        }
    }
    {
        Scope s(c, T_REFINE);
        BSM_CUDA(cudaMemcpyAsync(c->ref_d.p, c->chk_d.p, px * 4, cudaMemcpyDeviceToDevice, c->stream));
        BSM_CUDA(cudaMemcpyAsync(c->ref_v.p, c->chk_v.p, px, cudaMemcpyDeviceToDevice, c->stream));
        BSM_TRY(refine_launch(c, c->chk_d.as<float>(), c->chk_v.as<uint8_t>(), v.u8l ? v.u8l + size_t(r0) * W : nullptr,
                              v.u8l ? nullptr : v.ll + size_t(r0) * W, W, rows, p->vote_radius, p->d_max,
                              p->lambda_c, p->lambda_e));
    }
    c->last_W = W;
    c->last_rows = rows;
    c->last_r0 = r0;
    c->last_out0 = out0;
    c->last_out_rows = out_rows;
    c->last_unmasked = want_unmasked ? 1 : 0;
    return BSM_OK;
}

Views u8views(const uint8_t* l, const uint8_t* r) {
    Views v;
    v.u8l = l;
    v.u8r = r;
    return v;
}

int fetch(bsm_ctx* c, bsm_maps* o) {
    if (!o) return BSM_OK;
    Scope s(c, T_D2H);
    const int W = c->last_W;
    const size_t all = size_t(c->last_rows) * W;
    const size_t off = size_t(c->last_out0 - c->last_r0) * W;
    const size_t outpx = size_t(c->last_out_rows) * W;
    auto d2h = [&](void* dst, const DevBuf& b, size_t byte_off, size_t bytes) -> int {
        if (!dst) return BSM_OK;
        BSM_CUDA(cudaMemcpyAsync(dst, static_cast<const char*>(b.p) + byte_off, bytes, cudaMemcpyDeviceToHost, c->stream));
        return BSM_OK;
    };
    BSM_TRY(d2h(o->refined_d, c->ref_d, off * 4, outpx * 4));
    BSM_TRY(d2h(o->refined_v, c->ref_v, off, outpx));
    BSM_TRY(d2h(o->left_d, c->lw_d, 0, all * 4));
    BSM_TRY(d2h(o->right_d, c->rw_d, 0, all * 4));
    BSM_TRY(d2h(o->checked_d, c->chk_d, 0, all * 4));
    BSM_TRY(d2h(o->checked_v, c->chk_v, 0, all));
    if (c->last_unmasked) BSM_TRY(d2h(o->unmasked_d, c->un_d, 0, all * 4));
    return BSM_OK;
}

int begin_call(bsm_ctx* c) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    BSM_CUDA(cudaSetDevice(c->device));
    c->launches = 0;
    for (int t = 0; t < T_COUNT; ++t) c->ev_used[t] = 0;
    return BSM_OK;
}

int upload_views(bsm_ctx* c, const uint8_t* left, const uint8_t* right, int W, int H) {
    Scope s(c, T_H2D);
    const size_t n = size_t(W) * H;
    BSM_TRY(c->img_l.ensure(n));
    BSM_TRY(c->img_r.ensure(n));
    BSM_CUDA(cudaMemcpyAsync(c->img_l.p, left, n, cudaMemcpyHostToDevice, c->stream));
    if (right) BSM_CUDA(cudaMemcpyAsync(c->img_r.p, right, n, cudaMemcpyHostToDevice, c->stream));
    return BSM_OK;
}

int sync(bsm_ctx* c) {
    BSM_CUDA(cudaStreamSynchronize(c->stream));
    return BSM_OK;
}

int check_dims(int W, int H) {
    if (W < 1 || H < 1) return set_err(BSM_INVALID_ARGUMENT, "bsm: image dimensions must be >= 1");
    if (int64_t(W) * H > (int64_t(1) << 31) - 1)
        return set_err(BSM_UNSUPPORTED, "bsm: images above 2^31 pixels are outside this build's envelope");
    return BSM_OK;
}

}  // namespace

// ===========================================================================
// C ABI
extern "C" {

const char* bsm_last_error(void) { return g_err.c_str(); }
const char* bsm_version(void) { return "bsm-b200 0.1 (sm_100a)"; }

int bsm_ctx_create(int device, bsm_ctx** out) {
    if (!out) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return set_err(BSM_CUDA_ERROR, std::string("CUDA: no usable device (") + cudaGetErrorString(e) +
                                           "); this library has no CPU fallback");
    if (device < 0 || device >= ndev) return set_err(BSM_INVALID_ARGUMENT, "bsm: device index out of range");
    BSM_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    BSM_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_err(BSM_CUDA_ERROR, std::string("CUDA: built for sm_100a, device is ") + prop.name);
    bsm_ctx* c = new bsm_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return set_err(BSM_CUDA_ERROR, "CUDA: stream creation failed");
    }
    for (int t = 0; t < T_COUNT; ++t)
        for (int s = 0; s < bsm_ctx::kEvPerSlot; ++s) {
            cudaEventCreate(&c->ev[t][s][0]);
            cudaEventCreate(&c->ev[t][s][1]);
        }
    bsmh::gray_lab_lut(c->gray_lut, c->lab_lut);
    for (int v = 1; v < 256; ++v)
        if (!(c->gray_lut[v] > c->gray_lut[v - 1])) {
            bsm_ctx_destroy(c);
            return set_err(BSM_UNSUPPORTED, "bsm: gray conversion table is not strictly increasing");
        }
    {
        bsmh::ExpParams ep;
        c->exp_ok = bsmh::glibc_exp_params(ep, c->exp_why);
        if (c->exp_ok) {
            c->exp_dev = ExpDev{ep.invln2N, ep.shift, ep.negln2hiN, ep.negln2loN, ep.c2, ep.c3, ep.c4, ep.c5};
            if (c->d_etab.ensure(sizeof ep.tab) != BSM_OK ||
                cudaMemcpy(c->d_etab.p, ep.tab, sizeof ep.tab, cudaMemcpyHostToDevice) != cudaSuccess)
                c->exp_ok = false;
        }
        if (c->d_lab256.ensure(sizeof c->lab_lut) != BSM_OK ||
            cudaMemcpy(c->d_lab256.p, c->lab_lut, sizeof c->lab_lut, cudaMemcpyHostToDevice) != cudaSuccess) {
            bsm_ctx_destroy(c);
            return set_err(BSM_CUDA_ERROR, "CUDA: Lab table upload failed");
        }
    }
    std::vector<uint8_t> rank(65536);
    bsmh::sad_rank_table(c->lab_lut, rank.data());
    int rc = c->d_rank.ensure(65536);
    if (rc == BSM_OK && cudaMemcpy(c->d_rank.p, rank.data(), 65536, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = set_err(BSM_CUDA_ERROR, "CUDA: rank table upload failed");
    if (rc != BSM_OK) {
        bsm_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return BSM_OK;
}

int bsm_ctx_destroy(bsm_ctx* c) {
    if (!c) return BSM_OK;
    cudaSetDevice(c->device);
    DevBuf* bufs[] = {&c->d_pos, &c->d_descf, &c->d_rgb_gray, &c->d_rgb_lab, &c->planes, &c->d_desc4, &c->d_pqb, &c->d_uoff, &c->d_uxy, &c->d_rank, &c->d_wtab, &c->d_s2col,
                      &c->img_l, &c->img_r, &c->fdl, &c->fml, &c->fdr, &c->fmr, &c->keys_l, &c->keys_r,
                      &c->keys_u, &c->chk_d, &c->chk_v, &c->ref_d, &c->ref_v, &c->lw_d, &c->rw_d, &c->un_d,
                      &c->counters, &c->inv, &c->vmap, &c->d_etab, &c->d_elam, &c->d_lab256, &c->aux0, &c->aux1, &c->aux2, &c->aux3, &c->popc_out};
    for (DevBuf* b : bufs) b->release();
    for (int t = 0; t < T_COUNT; ++t)
        for (int s = 0; s < bsm_ctx::kEvPerSlot; ++s) {
            if (c->ev[t][s][0]) cudaEventDestroy(c->ev[t][s][0]);
            if (c->ev[t][s][1]) cudaEventDestroy(c->ev[t][s][1]);
        }
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return BSM_OK;
}

int bsm_generate_pattern(int n, int window, double spread, uint64_t seed, int16_t* out) {
    if (!out) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    std::string err;
    if (!bsmh::generate_pattern(n, window, spread, seed, out, err)) return set_err(BSM_INVALID_ARGUMENT, err);
    return BSM_OK;
}

int bsm_gray_lab_lut(float* gray256, float* lab768) {
    if (!gray256 || !lab768) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    bsmh::gray_lab_lut(gray256, lab768);
    return BSM_OK;
}

int bsm_to_gray_lab(const uint8_t* rgb, int W, int H, float* gray, float* lab) {
    if (!rgb) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    if (W < 1 || H < 1) return set_err(BSM_INVALID_ARGUMENT, "bsm: image dimensions must be >= 1");
    bsmh::to_gray_lab(rgb, size_t(W) * size_t(H), gray, lab);
    return BSM_OK;
}

int bsm_set_pattern(bsm_ctx* c, const int16_t* pairs, int n, int window) {
    if (!c || !pairs) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    if (n < 1) return set_err(BSM_INVALID_ARGUMENT, "pattern: n must be >= 1");
    if (window < 2) return set_err(BSM_INVALID_ARGUMENT, "pattern: window must be >= 2");
    if (n > kMaxPairs) return set_err(BSM_UNSUPPORTED, "bsm: n > 8192 is outside this build's envelope");
    if (window > 128) return set_err(BSM_UNSUPPORTED, "bsm: window > 128 is outside this build's envelope");
    const int half = window / 2, side = 2 * half + 1;
    for (int i = 0; i < 4 * n; ++i)
        if (pairs[i] < -half || pairs[i] > half)
            return set_err(BSM_INVALID_ARGUMENT, "pattern: offset outside window");
    BSM_CUDA(cudaSetDevice(c->device));
    c->n = n;
    c->window = window;
    c->half = half;
    c->NW = 2 * ((n + 63) / 64);
    c->pairs.assign(pairs, pairs + 4 * size_t(n));
    // Used window offsets (index into the (2h+1)^2 table, like
    // build_table_indices, descriptor.hpp:157-168) and per-pair endpoint
    // indices into that list.
    std::vector<int> slot(size_t(side) * side, -1);
    c->used.clear();
    std::vector<uint32_t> pq(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        int idx[2];
        for (int e = 0; e < 2; ++e) {
            const int t = (pairs[4 * i + 2 * e + 1] + half) * side + (pairs[4 * i + 2 * e] + half);
            if (slot[size_t(t)] < 0) {
                slot[size_t(t)] = int(c->used.size());
                c->used.push_back(int16_t(t));
            }
            idx[e] = slot[size_t(t)];
        }
        pq[size_t(i)] = uint32_t(idx[0]) | (uint32_t(idx[1]) << 16);
    }
    c->u = int(c->used.size());
    // k_mask4 / k_mask_f32 give each lane MCH chunks of 32 bit positions
    // (lane l: positions 32*MCH*l ..), MCH the smallest of 1, 2, 4, 8 that
    // holds n.  Otherwise the rank-table slots are placed by local search to
    // limit the gathers' bank conflicts.
    // For n = 1024 * MCH a bank-balanced pair order
    // (bsmh::balanced_gather_order) makes every gather conflict-free; the
    // descriptor bits follow the same order (the masked Hamming cost is
    // invariant under a common permutation of descriptor and mask bits) and
    // the per-stage API un-permutes.
    c->mch = n <= 1024 ? 1 : n <= 2048 ? 2 : n <= 4096 ? 4 : 8;
    const int lane_pos = 32 * c->mch;  // positions per lane
    std::vector<int> rslot(size_t(c->u));
    std::vector<uint8_t> flip;
    c->permuted = false;
    {
        int ns = 0;
        if (n == 32 * lane_pos && bsmh::balanced_gather_order(pq.data(), n, c->u, rslot, ns, c->order, flip)) {
            c->permuted = true;
            c->mslots = ns;
            c->slot_cost[0] = c->slot_cost[1] = 1.0;
        } else {
            rslot.assign(size_t(c->u), 0);
            c->mslots = round_up(c->u, 32) + 32;
            bsmh::place_rank_slots(pq.data(), n, c->u, c->mslots, lane_pos, rslot, &c->slot_cost[0],
                                   &c->slot_cost[1]);
        }
    }
    if (!c->permuted) {
        c->order.resize(size_t(n));
        for (int i = 0; i < n; ++i) c->order[size_t(i)] = i;
        flip.assign(size_t(n), 0);
    } else {
        std::vector<int> pos(static_cast<size_t>(n));
        for (int j = 0; j < n; ++j) pos[size_t(c->order[size_t(j)])] = j;
        BSM_TRY(c->d_pos.ensure(pos.size() * 4));
        BSM_CUDA(cudaMemcpy(c->d_pos.p, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice));
    }
    c->slot_used.assign(size_t(c->mslots), -1);
    for (int o = 0; o < c->u; ++o) c->slot_used[size_t(rslot[size_t(o)])] = o;
    // Byte offsets into the u32 rank table of each bit position's two
    // endpoints (k_mask4 / k_mask_f32): P table at [0, kPqTable), Q table at
    // [kPqTable, 2 kPqTable), lane-block order -- lane l, chunk m < MCH, t:
    // bit 32*MCH*l + 32m + t at uint4 [(m*8 + t/4)*32 + l], component t%4.
    // Pads read the sentinel.  For MCH <= 4, k_mask_f32 reads the packed table
    // at [2 kPqTable, 3 kPqTable): P | Q << 16 (mslots <= 2 * 4096 + 64 there,
    // so byte offsets fit 16 bits) -- half the L1 footprint of the gathers.
    if (c->mch <= 4 && 4 * c->mslots > 0xFFFF) return set_err(BSM_UNSUPPORTED, "bsm: rank-table offsets exceed 16 bits");
    std::vector<uint32_t> pqb(3 * kPqTable, uint32_t(4 * c->mslots));
    for (int i = 0; i < kPqTable; ++i) pqb[2 * kPqTable + i] = uint32_t(4 * c->mslots) * 65537u;
    for (int j = 0; j < n; ++j) {
        const int l = j / lane_pos, m = (j >> 5) % c->mch, t = j & 31;
        const size_t at = (size_t(m * 8 + (t >> 2)) * 32 + l) * 4 + (t & 3);
        const uint32_t e = pq[size_t(c->order[size_t(j)])];
        const uint32_t a = flip[size_t(j)] ? e >> 16 : e & 0xFFFFu, b = flip[size_t(j)] ? e & 0xFFFFu : e >> 16;
        pqb[at] = uint32_t(4 * rslot[size_t(a)]);
        pqb[kPqTable + at] = uint32_t(4 * rslot[size_t(b)]);
        pqb[2 * kPqTable + at] = pqb[at] | (pqb[kPqTable + at] << 16);
    }
    BSM_TRY(c->d_pqb.ensure(pqb.size() * 4));
    BSM_CUDA(cudaMemcpy(c->d_pqb.p, pqb.data(), pqb.size() * 4, cudaMemcpyHostToDevice));
    c->desc4_tw = -1;
    c->descf_tw = -1;
    c->uoff_tw = -1;
    if (mask4_smem(c) > 200 * 1024 || maskf_smem(c) > 200 * 1024)
        return set_err(BSM_UNSUPPORTED, "bsm: pattern too large for shared-memory staging");
    return BSM_OK;
}

// Device SoA field -> reference AoS words in c->aux0 (bit order restored).
static int soa_to_aos(bsm_ctx* c, const uint32_t* src, int W, int H) {
    const int Wp = round_up(W, 128), tb = 256;
    const size_t aos = size_t(H) * W * c->NW;
    if (c->permuted)
        k_soa_to_aos_perm<<<unsigned((aos + tb - 1) / tb), tb, 0, c->stream>>>(src, W, H, c->NW, Wp,
                                                                              c->d_pos.as<int>(), c->n,
                                                                              c->aux0.as<uint32_t>());
    else
        k_soa_to_aos<<<unsigned((aos + tb - 1) / tb), tb, 0, c->stream>>>(src, W, H, c->NW, Wp,
                                                                         c->aux0.as<uint32_t>());
    return check_launch(c, "soa_to_aos");
}

int bsm_compute_field_u8(bsm_ctx* c, const uint8_t* img, int W, int H, uint64_t* desc, uint64_t* mask) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    if (!img) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    const int Wp = round_up(W, 128);
    const size_t fbytes = size_t(H) * c->NW * Wp * 4;
    BSM_TRY(upload_views(c, img, nullptr, W, H));
    BSM_TRY(c->fdl.ensure(fbytes));
    BSM_TRY(c->fml.ensure(fbytes));
    BSM_TRY(field_device(c, c->img_l.as<uint8_t>(), W, H, 0, H, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>()));
    const size_t aos = size_t(H) * W * c->NW;
    BSM_TRY(c->aux0.ensure(aos * 4));
    for (int which = 0; which < 2; ++which) {
        uint64_t* dst = which == 0 ? desc : mask;
        if (!dst) continue;
        BSM_TRY(soa_to_aos(c, which == 0 ? c->fdl.as<uint32_t>() : c->fml.as<uint32_t>(), W, H));
        BSM_CUDA(cudaMemcpyAsync(dst, c->aux0.p, aos * 4, cudaMemcpyDeviceToHost, c->stream));
        BSM_TRY(sync(c));
    }
    return sync(c);
}

int bsm_wta(bsm_ctx* c, const uint64_t* desc_ref, const uint64_t* mask_ref, const uint64_t* desc_other, int W,
            int H, int n, int d_max, int right_ref, int use_mask, float* out_d) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_dims(W, H));
    if (!desc_ref || !desc_other || (use_mask && !mask_ref))
        return set_err(BSM_INVALID_ARGUMENT, "bsm: null field");
    if (d_max < 1) return set_err(BSM_INVALID_ARGUMENT, "wta: d_max must be >= 1");
    if (d_max > 65535) return set_err(BSM_UNSUPPORTED, "bsm: d_max > 65535 is outside this build's envelope");
    if (n < 1 || n > kMaxPairs) return set_err(BSM_UNSUPPORTED, "bsm: n outside [1, 8192]");
    const int NW = 2 * ((n + 63) / 64);
    const int savedNW = c->NW;
    c->NW = NW;
    const int Wp = round_up(W, 128);
    const size_t aos = size_t(H) * W * NW, soa = size_t(H) * NW * Wp;
    int rc = BSM_OK;
    do {
        if ((rc = c->aux0.ensure(aos * 4)) != BSM_OK) break;
        if ((rc = c->fdl.ensure(soa * 4)) != BSM_OK) break;
        if ((rc = c->fml.ensure(soa * 4)) != BSM_OK) break;
        if ((rc = c->fdr.ensure(soa * 4)) != BSM_OK) break;
        if ((rc = c->keys_l.ensure(size_t(H) * W * 4)) != BSM_OK) break;
        if ((rc = c->lw_d.ensure(size_t(H) * W * 4)) != BSM_OK) break;
        const int tb = 256;
        const uint64_t* srcs[3] = {desc_ref, use_mask ? mask_ref : nullptr, desc_other};
        DevBuf* dsts[3] = {&c->fdl, &c->fml, &c->fdr};
        for (int k = 0; k < 3 && rc == BSM_OK; ++k) {
            if (!srcs[k]) continue;
            if (cudaMemcpyAsync(c->aux0.p, srcs[k], aos * 4, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
                rc = set_err(BSM_CUDA_ERROR, "CUDA: field upload failed");
                break;
            }
            k_aos_to_soa<<<unsigned((soa + tb - 1) / tb), tb, 0, c->stream>>>(c->aux0.as<uint32_t>(), W, H, NW, Wp,
                                                                            dsts[k]->as<uint32_t>());
            rc = check_launch(c, "aos_to_soa");
            if (rc == BSM_OK) rc = sync(c);  // aux0 is reused by the next upload
        }
        if (rc != BSM_OK) break;
        rc = wta_device(c, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>(), c->fdr.as<uint32_t>(), W, H, d_max,
                        right_ref != 0, use_mask != 0, c->keys_l.as<uint32_t>(), right_ref ? T_WTA_R : T_WTA_L);
        if (rc != BSM_OK) break;
        const size_t px = size_t(H) * W;
        k_keys_to_float<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(c->keys_l.as<uint32_t>(), px,
                                                                          c->lw_d.as<float>());
        if ((rc = check_launch(c, "keys_to_float")) != BSM_OK) break;
        if (out_d && cudaMemcpyAsync(out_d, c->lw_d.p, px * 4, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) {
            rc = set_err(BSM_CUDA_ERROR, "CUDA: download failed");
            break;
        }
        rc = sync(c);
    } while (0);
    c->NW = savedNW;
    return rc;
}

int bsm_lr_check(bsm_ctx* c, const float* left_d, const float* right_d, int W, int H, double tol, float* out_d,
                 uint8_t* out_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_dims(W, H));
    if (!left_d || !right_d) return set_err(BSM_INVALID_ARGUMENT, "bsm: null map");
    const size_t px = size_t(W) * H;
    BSM_TRY(c->aux0.ensure(px * 4));
    BSM_TRY(c->aux1.ensure(px * 4));
    BSM_TRY(c->aux2.ensure(px * 4));
    BSM_TRY(c->aux3.ensure(px));
    BSM_CUDA(cudaMemcpyAsync(c->aux0.p, left_d, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->aux1.p, right_d, px * 4, cudaMemcpyHostToDevice, c->stream));
    const int tb = 256;
    k_lr_check_float<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(c->aux0.as<float>(), c->aux1.as<float>(), W,
                                                                       H, tol, c->aux2.as<float>(),
                                                                       c->aux3.as<uint8_t>());
    BSM_TRY(check_launch(c, "lr_check_float"));
    if (out_d) BSM_CUDA(cudaMemcpyAsync(out_d, c->aux2.p, px * 4, cudaMemcpyDeviceToHost, c->stream));
    if (out_v) BSM_CUDA(cudaMemcpyAsync(out_v, c->aux3.p, px, cudaMemcpyDeviceToHost, c->stream));
    return sync(c);
}

int bsm_vote_refine_u8(bsm_ctx* c, const float* d, const uint8_t* v, const uint8_t* gray_img, int W, int H,
                       double lambda_c, double lambda_e, int vote_radius, float* out_d, uint8_t* out_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_dims(W, H));
    if (!d || !v || !gray_img) return set_err(BSM_INVALID_ARGUMENT, "bsm: null input");
    if (!(lambda_c > 0)) return set_err(BSM_INVALID_ARGUMENT, "refine: lambda_c must be > 0");
    if (!(lambda_e > 0)) return set_err(BSM_INVALID_ARGUMENT, "refine: lambda_e must be > 0");
    if (vote_radius < 1) return set_err(BSM_INVALID_ARGUMENT, "refine: vote_radius must be >= 1");
    if (vote_radius > 180) return set_err(BSM_UNSUPPORTED, "bsm: vote_radius > 180 is outside this build's envelope");
    const size_t px = size_t(W) * H;
    // Host pre-pass over the caller's map: max_bin (refine.hpp:68-72) and the
    // invalid list.  Valid disparities must round to a bin >= 0.
    int max_bin = 0;
    std::vector<int> invalid;
    for (size_t i = 0; i < px; ++i) {
        if (v[i]) {
            const double dv = double(d[i]);
            if (!(dv > -0.5) || !(dv < 1e6)) return set_err(BSM_INVALID_ARGUMENT, "vote_refine: valid disparity out of range");
            max_bin = std::max(max_bin, int(std::lround(dv)));
        } else {
            invalid.push_back(int(i));
        }
    }
    if (max_bin + 1 > 12288) return set_err(BSM_UNSUPPORTED, "bsm: disparity range too large for the refine bins");
    BSM_TRY(c->img_l.ensure(px));
    BSM_TRY(c->chk_d.ensure(px * 4));
    BSM_TRY(c->chk_v.ensure(px));
    BSM_TRY(c->ref_d.ensure(px * 4));
    BSM_TRY(c->ref_v.ensure(px));
    BSM_TRY(c->counters.ensure(64));
    BSM_TRY(c->inv.ensure(std::max<size_t>(4, invalid.size() * 4)));
    BSM_CUDA(cudaMemcpyAsync(c->img_l.p, gray_img, px, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->chk_d.p, d, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->chk_v.p, v, px, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->ref_d.p, d, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->ref_v.p, v, px, cudaMemcpyHostToDevice, c->stream));
    int cnt[2] = {max_bin, int(invalid.size())};
    BSM_CUDA(cudaMemcpyAsync(c->counters.p, cnt, 8, cudaMemcpyHostToDevice, c->stream));
    if (!invalid.empty())
        BSM_CUDA(cudaMemcpyAsync(c->inv.p, invalid.data(), invalid.size() * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_TRY(sync(c));  // host staging buffers (cnt, invalid) go out of scope
    BSM_TRY(refine_launch(c, c->chk_d.as<float>(), c->chk_v.as<uint8_t>(), c->img_l.as<uint8_t>(), nullptr, W, H,
                          vote_radius, max_bin + 1, lambda_c, lambda_e));
    if (out_d) BSM_CUDA(cudaMemcpyAsync(out_d, c->ref_d.p, px * 4, cudaMemcpyDeviceToHost, c->stream));
    if (out_v) BSM_CUDA(cudaMemcpyAsync(out_v, c->ref_v.p, px, cudaMemcpyDeviceToHost, c->stream));
    return sync(c);
}

int bsm_pipeline_u8(bsm_ctx* c, const uint8_t* left, const uint8_t* right, int W, int H, const bsm_params* params,
                    int want_unmasked, bsm_maps* out) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!left || !right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    BSM_TRY(upload_views(c, left, right, W, H));
    BSM_TRY(pipeline_device(c, u8views(c->img_l.as<uint8_t>(), c->img_r.as<uint8_t>()), W, H, 0, H, params,
                            want_unmasked != 0));
    BSM_TRY(fetch(c, out));
    return sync(c);
}

int bsm_pipeline_u8_device(bsm_ctx* c, const uint8_t* d_left, const uint8_t* d_right, int W, int H,
                           const bsm_params* params, int want_unmasked) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    if (!d_left || !d_right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    return pipeline_device(c, u8views(d_left, d_right), W, H, 0, H, params, want_unmasked != 0);
}

int bsm_fetch_maps(bsm_ctx* c, bsm_maps* out) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    if (c->last_W == 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: no pipeline result to fetch");
    BSM_TRY(fetch(c, out));
    return sync(c);
}

int bsm_pipeline_band_u8(bsm_ctx* c, const uint8_t* left, const uint8_t* right, int W, int H, int y0, int y1,
                         const bsm_params* params, float* refined_d, uint8_t* refined_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!left || !right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    if (y0 < 0 || y1 > H || y0 >= y1) return set_err(BSM_INVALID_ARGUMENT, "bsm: band rows out of range");
    BSM_TRY(upload_views(c, left, right, W, H));
    BSM_TRY(pipeline_device(c, u8views(c->img_l.as<uint8_t>(), c->img_r.as<uint8_t>()), W, H, y0, y1 - y0, params,
                            false));
    bsm_maps m = {};
    m.refined_d = refined_d;
    m.refined_v = refined_v;
    BSM_TRY(fetch(c, &m));
    return sync(c);
}

int bsm_device_exp(bsm_ctx* c, const double* x, int n, double* out) {
    BSM_TRY(begin_call(c));
    if (!x || !out || n < 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: bad arguments");
    if (!c->exp_ok) return set_err(BSM_UNSUPPORTED, "bsm: device exp unavailable (" + c->exp_why + ")");
    if (n == 0) return BSM_OK;
    BSM_TRY(c->aux0.ensure(size_t(n) * 8));
    BSM_TRY(c->aux1.ensure(size_t(n) * 8));
    BSM_CUDA(cudaMemcpyAsync(c->aux0.p, x, size_t(n) * 8, cudaMemcpyHostToDevice, c->stream));
    k_exp_eval<<<(n + 255) / 256, 256, 0, c->stream>>>(c->aux0.as<double>(), n, c->exp_dev,
                                                       c->d_etab.as<unsigned long long>(), c->aux1.as<double>());
    BSM_TRY(check_launch(c, "exp_eval"));
    BSM_CUDA(cudaMemcpyAsync(out, c->aux1.p, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    return sync(c);
}

int bsm_vote_refine_lab(bsm_ctx* c, const float* d, const uint8_t* v, const float* lab, int W, int H,
                        double lambda_c, double lambda_e, int vote_radius, float* out_d, uint8_t* out_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_dims(W, H));
    if (!d || !v || !lab) return set_err(BSM_INVALID_ARGUMENT, "bsm: null input");
    if (!(lambda_c > 0)) return set_err(BSM_INVALID_ARGUMENT, "refine: lambda_c must be > 0");
    if (!(lambda_e > 0)) return set_err(BSM_INVALID_ARGUMENT, "refine: lambda_e must be > 0");
    if (vote_radius < 1) return set_err(BSM_INVALID_ARGUMENT, "refine: vote_radius must be >= 1");
    if (vote_radius > 180) return set_err(BSM_UNSUPPORTED, "bsm: vote_radius > 180 is outside this build's envelope");
    const size_t px = size_t(W) * H;
    int max_bin = 0;
    std::vector<int> invalid;
    for (size_t i = 0; i < px; ++i) {
        if (v[i]) {
            const double dv = double(d[i]);
            if (!(dv > -0.5) || !(dv < 65535.0))
                return set_err(BSM_INVALID_ARGUMENT, "vote_refine: valid disparity out of range");
            max_bin = std::max(max_bin, int(std::lround(dv)));
        } else {
            invalid.push_back(int(i));
        }
    }
    BSM_TRY(c->img_l.ensure(px));
    BSM_TRY(c->aux2.ensure(px * 12));
    BSM_TRY(c->aux3.ensure(px * 16));
    BSM_TRY(c->chk_d.ensure(px * 4));
    BSM_TRY(c->chk_v.ensure(px));
    BSM_TRY(c->ref_d.ensure(px * 4));
    BSM_TRY(c->ref_v.ensure(px));
    BSM_TRY(c->counters.ensure(64));
    BSM_TRY(c->inv.ensure(std::max<size_t>(4, invalid.size() * 4)));
    BSM_CUDA(cudaMemsetAsync(c->img_l.p, 0, px, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->aux2.p, lab, px * 12, cudaMemcpyHostToDevice, c->stream));
    k_lab3_to_lab4<<<unsigned((px + 255) / 256), 256, 0, c->stream>>>(c->aux2.as<float>(), px, c->aux3.as<float4>());
    BSM_TRY(check_launch(c, "lab3_to_lab4"));
    BSM_CUDA(cudaMemcpyAsync(c->chk_d.p, d, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->chk_v.p, v, px, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->ref_d.p, d, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->ref_v.p, v, px, cudaMemcpyHostToDevice, c->stream));
    int cnt[2] = {max_bin, int(invalid.size())};
    BSM_CUDA(cudaMemcpyAsync(c->counters.p, cnt, 8, cudaMemcpyHostToDevice, c->stream));
    if (!invalid.empty())
        BSM_CUDA(cudaMemcpyAsync(c->inv.p, invalid.data(), invalid.size() * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_TRY(sync(c));
    BSM_TRY(refine_launch(c, c->chk_d.as<float>(), c->chk_v.as<uint8_t>(), c->img_l.as<uint8_t>(), c->aux3.as<float4>(),
                          W, H, vote_radius, max_bin + 1, lambda_c, lambda_e));
    if (out_d) BSM_CUDA(cudaMemcpyAsync(out_d, c->ref_d.p, px * 4, cudaMemcpyDeviceToHost, c->stream));
    if (out_v) BSM_CUDA(cudaMemcpyAsync(out_v, c->ref_v.p, px, cudaMemcpyDeviceToHost, c->stream));
    return sync(c);
}

int bsm_set_refine_mode(bsm_ctx* c, int mode) {
    if (!c || mode < -1 || mode > 4 || mode == 0 || mode == 1)
        return set_err(BSM_INVALID_ARGUMENT, "bsm: bad refine mode");
    c->refine_mode = mode;
    return BSM_OK;
}

int bsm_pipeline_band_u8_device(bsm_ctx* c, const uint8_t* d_left, const uint8_t* d_right, int W, int H, int y0,
                                 int y1, const bsm_params* params) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!d_left || !d_right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    if (y0 < 0 || y1 > H || y0 >= y1) return set_err(BSM_INVALID_ARGUMENT, "bsm: band rows out of range");
    return pipeline_device(c, u8views(d_left, d_right), W, H, y0, y1 - y0, params, false);
}

int bsm_result_device(bsm_ctx* c, const float** refined_d, const uint8_t** refined_v, int* row0, int* nrows) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    if (c->last_W == 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: no pipeline result");
    const size_t off = size_t(c->last_out0 - c->last_r0) * c->last_W;
    if (refined_d) *refined_d = c->ref_d.as<float>() + off;
    if (refined_v) *refined_v = c->ref_v.as<uint8_t>() + off;
    if (row0) *row0 = c->last_out0;
    if (nrows) *nrows = c->last_out_rows;
    return BSM_OK;
}

int bsm_copy_result_device(bsm_ctx* c, float* dst_d, uint8_t* dst_v) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    if (c->last_W == 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: no pipeline result");
    const size_t off = size_t(c->last_out0 - c->last_r0) * c->last_W;
    const size_t n = size_t(c->last_out_rows) * c->last_W;
    if (dst_d) BSM_CUDA(cudaMemcpyAsync(dst_d, c->ref_d.as<float>() + off, n * 4, cudaMemcpyDeviceToDevice, c->stream));
    if (dst_v) BSM_CUDA(cudaMemcpyAsync(dst_v, c->ref_v.as<uint8_t>() + off, n, cudaMemcpyDeviceToDevice, c->stream));
    return BSM_OK;
}

int bsm_rgb24_tables(float* gray, float* lab) {
    if (!gray || !lab) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    std::vector<float> g, l;
    bsmh::rgb24_tables(g, l);
    std::memcpy(gray, g.data(), g.size() * 4);
    std::memcpy(lab, l.data(), l.size() * 4);
    return BSM_OK;
}

int bsm_compute_field_f32(bsm_ctx* c, const float* gray, const float* lab, int W, int H, uint64_t* desc,
                          uint64_t* mask) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    if (!gray || !lab) return set_err(BSM_INVALID_ARGUMENT, "bsm: null plane");
    const size_t px = size_t(W) * H;
    const int Wp = round_up(W, 128);
    const size_t fbytes = size_t(H) * c->NW * Wp * 4;
    BSM_TRY(c->planes.ensure(px * 32));
    float* g = c->planes.as<float>();
    float* l3 = g + px;
    float4* l = reinterpret_cast<float4*>(g + 4 * px);  // 16-B aligned (planes is cudaMalloc'd)
    BSM_CUDA(cudaMemcpyAsync(g, gray, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(l3, lab, px * 12, cudaMemcpyHostToDevice, c->stream));
    k_lab3_to_lab4<<<unsigned((px + 255) / 256), 256, 0, c->stream>>>(l3, px, l);
    BSM_TRY(check_launch(c, "lab3_to_lab4"));
    BSM_TRY(c->fdl.ensure(fbytes));
    BSM_TRY(c->fml.ensure(fbytes));
    BSM_TRY(field_device_f32(c, g, l, W, H, 0, H, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>()));
    const size_t aos = size_t(H) * W * c->NW;
    BSM_TRY(c->aux0.ensure(aos * 4));
    for (int which = 0; which < 2; ++which) {
        uint64_t* dst = which == 0 ? desc : mask;
        if (!dst) continue;
        BSM_TRY(soa_to_aos(c, which == 0 ? c->fdl.as<uint32_t>() : c->fml.as<uint32_t>(), W, H));
        BSM_CUDA(cudaMemcpyAsync(dst, c->aux0.p, aos * 4, cudaMemcpyDeviceToHost, c->stream));
        BSM_TRY(sync(c));
    }
    return sync(c);
}

// Colour pair already on the device: RGB -> gray/Lab planes, then the fused pipeline.
static int rgb_pipeline(bsm_ctx* c, const uint8_t* d_left, const uint8_t* d_right, int W, int H,
                        const bsm_params* params, bool want_unmasked) {
    BSM_TRY(ensure_rgb_tables(c));
    const size_t px = size_t(W) * H;
    const size_t lab_off = (2 * px + 3) / 4 * 4;  // floats; keeps the float4 planes 16-B aligned
    BSM_TRY(c->planes.ensure((lab_off + 8 * px) * 4));
    Views v;
    float* base = c->planes.as<float>();
    float4* lab4 = reinterpret_cast<float4*>(base + lab_off);
    v.gl = base;
    v.gr = base + px;
    v.ll = lab4;
    v.lr = lab4 + px;
    {
        Scope s(c, T_DESC);  // the conversion is accounted with the descriptor stage
        const int tb = 256;
        k_rgb_planes<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(d_left, px, c->d_rgb_gray.as<float>(),
                                                                      c->d_rgb_lab.as<float>(), base, lab4);
        BSM_TRY(check_launch(c, "rgb_planes"));
        k_rgb_planes<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(d_right, px, c->d_rgb_gray.as<float>(),
                                                                      c->d_rgb_lab.as<float>(), base + px,
                                                                      lab4 + px);
        BSM_TRY(check_launch(c, "rgb_planes"));
    }
    return pipeline_device(c, v, W, H, 0, H, params, want_unmasked);
}

int bsm_pipeline_rgb(bsm_ctx* c, const uint8_t* left, const uint8_t* right, int W, int H, const bsm_params* params,
                     int want_unmasked, bsm_maps* out) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!left || !right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    const size_t px = size_t(W) * H;
    BSM_TRY(c->img_l.ensure(px * 3));
    BSM_TRY(c->img_r.ensure(px * 3));
    {
        Scope s(c, T_H2D);
        BSM_CUDA(cudaMemcpyAsync(c->img_l.p, left, px * 3, cudaMemcpyHostToDevice, c->stream));
        BSM_CUDA(cudaMemcpyAsync(c->img_r.p, right, px * 3, cudaMemcpyHostToDevice, c->stream));
    }
    BSM_TRY(rgb_pipeline(c, c->img_l.as<uint8_t>(), c->img_r.as<uint8_t>(), W, H, params, want_unmasked != 0));
    BSM_TRY(fetch(c, out));
    return sync(c);
}

int bsm_pipeline_rgb_device(bsm_ctx* c, const uint8_t* d_left, const uint8_t* d_right, int W, int H,
                            const bsm_params* params, int want_unmasked) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!d_left || !d_right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    return rgb_pipeline(c, d_left, d_right, W, H, params, want_unmasked != 0);
}

int bsm_stream(bsm_ctx* c, void** stream) {
    if (!c || !stream) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    *stream = c->stream;
    return BSM_OK;
}

int bsm_set_profiling(bsm_ctx* c, int enable) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    c->profiling = enable != 0;
    return BSM_OK;
}

int bsm_last_timings(bsm_ctx* c, float* ms, int max, int* count) {
    if (!c || !ms) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    BSM_CUDA(cudaStreamSynchronize(c->stream));
    const int k = std::min(max, int(T_COUNT));
    for (int t = 0; t < k; ++t) {
        ms[t] = 0.0f;
        for (int s = 0; s < c->ev_used[t]; ++s) {
            float v = 0.0f;
            cudaEventElapsedTime(&v, c->ev[t][s][0], c->ev[t][s][1]);
            ms[t] += v;
        }
    }
    if (count) *count = k;
    return BSM_OK;
}

const char* bsm_timing_names(void) { return kTimingNames; }

int bsm_last_launch_count(bsm_ctx* c, int* count) {
    if (!c || !count) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    *count = c->launches;
    return BSM_OK;
}

int bsm_measure_popc_peak(bsm_ctx* c, double* ops_per_s) {
    return bsm_measure_word_peaks(c, ops_per_s, nullptr);
}

int bsm_measure_word_peaks(bsm_ctx* c, double* popc_words_per_s, double* csa_words_per_s) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    BSM_CUDA(cudaSetDevice(c->device));
    const int blocks = c->sm_count * 4, threads = 512, iters = 8192;
    BSM_TRY(c->popc_out.ensure(size_t(blocks) * threads * 4));
    cudaEvent_t e0, e1;
    BSM_CUDA(cudaEventCreate(&e0));
    BSM_CUDA(cudaEventCreate(&e1));
    for (int kind = 0; kind < 2; ++kind) {
        double* dst = kind == 0 ? popc_words_per_s : csa_words_per_s;
        if (!dst) continue;
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(e0, c->stream);
            if (kind == 0) k_popc_peak<<<blocks, threads, 0, c->stream>>>(c->popc_out.as<uint32_t>(), 7u + r, iters);
            else k_csa_peak<<<blocks, threads, 0, c->stream>>>(c->popc_out.as<uint32_t>(), 7u + r, iters, 2u);
            cudaEventRecord(e1, c->stream);
            BSM_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0) best = std::min(best, ms);
        }
        const double words = double(blocks) * threads * iters * 8 * (kind == 0 ? 1 : 2);
        *dst = words / (double(best) * 1e-3);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return BSM_OK;
}

}  // extern "C"
