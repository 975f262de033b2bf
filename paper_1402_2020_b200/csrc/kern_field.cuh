// kern_field.cuh -- K1/K2: descriptor and mask kernels (gray uint8 and float /
// Lab planes).  Part of bsm_kernels.cu's single translation unit (included
// inside its anonymous namespace; not a standalone header).
#pragma once

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

// The word at byte offset `off` from `base` (the pair table holds byte
// offsets, so a tile address is one add: no per-load shift).
__device__ __forceinline__ uint32_t ld_off(const uint32_t* base, int off) {
    return *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(base) + off);
}

__global__ void __launch_bounds__(kD2TX* kD2TY)
    k_descriptor4(const uint8_t* __restrict__ img, int W, int H, int ybeg, int rows,
                  const int2* __restrict__ ptab, int n, int half, int TWs, int NW, int Wq, size_t P,
                  uint32_t* __restrict__ desc, const uint8_t* __restrict__ img2, uint32_t* __restrict__ desc2,
                  int zsplit) {
    // grid.z = views x zsplit word ranges: both views of a pair in one launch
    // (one tail instead of two)
    const int view = int(blockIdx.z) / zsplit, zz = int(blockIdx.z) - view * zsplit;
    if (view) {
        img = img2;
        desc = desc2;
    }
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
    const int wper = (NW + zsplit - 1) / zsplit;
    const int wbeg = zz * wper, wend = min(NW, wbeg + wper);
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
                    const uint32_t f = bytes_gt(ld_off(tb + r * rowW, e.x), ld_off(tb + r * rowW, e.y));  // bit 7 of byte j: pixel j
                    // pair k -> bit (k & 7) of byte lane j of acc[k >> 3]
                    acc[r][k >> 3] |= (f >> (7 - (k & 7)));
                }
            }
        } else {
            for (int k = 0; k < cnt; ++k) {
                const int2 e = __ldg(ptab + 32 * w + k);
#pragma unroll
                for (int r = 0; r < kD2Rows; ++r) {
                    const uint32_t v = bytes_gt(ld_off(tb + r * rowW, e.x), ld_off(tb + r * rowW, e.y)) >> (7 - (k & 7));
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
            if (ly < rows && xq < Wq) *reinterpret_cast<uint4*>(desc + size_t(w) * P + size_t(ly) * Wq + xq) = o;
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

// src[0..7]: 32 byte values, value t = byte t/8 of src[t%8] (the gather order
// of the index tables for MCH <= 4); afterwards w[j] bit t = bit j of value t.
// Each byte lane
// holds an 8 x 8 bit matrix (row k = w[k]'s byte); three delta-swap stages
// across the words transpose all four at once, and word j of the result is
// plane j (byte lane b = positions 8b..8b+7): 12 swaps, no byte shuffles.
__device__ __forceinline__ void bytes_to_planes_x(const uint32_t (&src)[8], uint32_t (&w)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = src[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // distance 4: bits 4..7 of rows k <-> bits 0..3 of rows k + 4
        const uint32_t t = ((w[k] >> 4) ^ w[k + 4]) & 0x0F0F0F0Fu;
        w[k + 4] ^= t;
        w[k] ^= t * 16u;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {  // distance 2
        if (k & 2) continue;
        const uint32_t t = ((w[k] >> 2) ^ w[k + 2]) & 0x33333333u;
        w[k + 2] ^= t;
        w[k] ^= t * 4u;
    }
#pragma unroll
    for (int k = 0; k < 8; k += 2) {  // distance 1
        const uint32_t t = ((w[k] >> 1) ^ w[k + 1]) & 0x55555555u;
        w[k + 1] ^= t;
        w[k] ^= t * 2u;
    }
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
        // warp-uniform choices taken as uniform branches (no per-word selects)
        const bool ha = zas < ka, hb = zbs < kb;
        if (ha) {
            ka -= zas;
#pragma unroll
            for (int m = 0; m < MCH; ++m) {
                la[m] |= za[m];
                ea[m] &= pa[j][m];
            }
        } else {
#pragma unroll
            for (int m = 0; m < MCH; ++m) ea[m] = za[m];
        }
        if (hb) {
            kb -= zbs;
#pragma unroll
            for (int m = 0; m < MCH; ++m) {
                lb[m] |= zb[m];
                eb[m] &= pb[j][m];
            }
        } else {
#pragma unroll
            for (int m = 0; m < MCH; ++m) eb[m] = zb[m];
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

template <int MCH, bool PACKED = false>
__global__ void __launch_bounds__(32, 16)
    k_mask4(const uint8_t* __restrict__ img, int W, int H, int ybeg, int rows, const uint4* __restrict__ p4,
            const uint4* __restrict__ q4, int n, const uint32_t* __restrict__ ufill, int nfill, int u, int rho_words,
            const uint8_t* __restrict__ rank, int half, int TW, int NW, int Wq, size_t P, uint32_t* __restrict__ mask,
            const uint8_t* __restrict__ img2, uint32_t* __restrict__ mask2) {
    if (blockIdx.z) {  // second view of the pair (grid.z = 2)
        img = img2;
        mask = mask2;
    }
    extern __shared__ __align__(16) uint32_t dsm[];
    uint32_t* rho2 = dsm;                                 // 2 x rho_words (u + sentinel, padded): two passes' tables
    constexpr int STG = mask4_stage_stride(MCH);
    uint32_t* stage = rho2 + 2 * rho_words;               // [kM3Px][STG]
    uint8_t* rrows = reinterpret_cast<uint8_t*>(stage + kM3Px * STG);  // 4 x 256: rank rows of 4 centres
    uint8_t* tile = rrows + 1024;                                           // (2h+1) x TW
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
    if ((W & 3) == 0 && (reinterpret_cast<uintptr_t>(img) & 3) == 0 && a0 >= 0 && a0 + TW <= W && ay0 >= 0 &&
        ay0 + TH <= H) {
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
    if (lane < 2) rho2[lane * rho_words + u] = 0x00FF00FFu;  // sentinels: a = 255 for both pixels
    __syncwarp();

    const int k = max(1, n / 4);
    const int c0 = half * TW + sh + half;  // tile index of pixel x0
    // rank rows of the next two passes' four centre pixels, loaded two passes ahead
    uint4 rr0 = __ldg(reinterpret_cast<const uint4*>(rank + 256 * int(tile[c0 + (lane >> 4)])) + (lane & 15));
    uint4 rr1 = __ldg(reinterpret_cast<const uint4*>(rank + 256 * int(tile[c0 + 2 + (lane >> 4)])) + (lane & 15));
#pragma unroll 1
    for (int q = 0; q < kM3Px; q += 2) {
        uint32_t* rho = rho2 + ((q >> 1) & 1) * rho_words;
        if ((q & 2) == 0) {
            // the tables of passes q and q + 2 (pixels q .. q + 3) in one sweep: entry
            // j = (slot << 16) | (window offset + h TW + h); lane b of every group of
            // 32 writes a slot of bank b, and a group's offsets lie within a few
            // window rows (host fill order), so stores and tile reads stay
            // conflict-free or nearly
            reinterpret_cast<uint4*>(rrows)[lane] = rr0;
            reinterpret_cast<uint4*>(rrows)[32 + lane] = rr1;
            if (q + 4 < kM3Px) {
                rr0 = __ldg(reinterpret_cast<const uint4*>(rank + 256 * int(tile[c0 + q + 4 + (lane >> 4)])) + (lane & 15));
                rr1 = __ldg(reinterpret_cast<const uint4*>(rank + 256 * int(tile[c0 + q + 6 + (lane >> 4)])) + (lane & 15));
            }
            __syncwarp();
            const uint8_t* tq = tile + sh + q;
            for (int j = lane; j < nfill; j += 32) {
                const uint32_t e = __ldg(ufill + j);
                const uint8_t* tp = tq + (e & 0xFFFFu);
                const uint32_t v0 = uint32_t(rrows[tp[0]]) | (uint32_t(rrows[256 + tp[1]]) << 16);
                const uint32_t v1 = uint32_t(rrows[512 + tp[2]]) | (uint32_t(rrows[768 + tp[3]]) << 16);
                rho2[e >> 16] = v0;
                rho2[rho_words + (e >> 16)] = v1;
            }
            __syncwarp();
        }

        // a = max(rhoP, rhoQ) of 32 positions of chunk m for both pixels, as
        // byte registers wa (pixel A) and wb (pixel B)
        auto gather = [&](int m, uint32_t(&wa)[8], uint32_t(&wb)[8]) {
#pragma unroll
            for (int t4 = 0; t4 < 8; ++t4) {
                uint4 P, Q;
                if constexpr (PACKED) {
                    // one load of P | Q << 16 (p4 points at the packed table),
                    // split on the FMA pipe: hi = x >> 16, lo = x - (hi << 16)
                    const uint4 X = __ldg(p4 + (m * 8 + t4) * 32 + lane);
                    Q = make_uint4(__umulhi(X.x, 65536u), __umulhi(X.y, 65536u), __umulhi(X.z, 65536u),
                                   __umulhi(X.w, 65536u));
                    P = make_uint4(X.x - Q.x * 65536u, X.y - Q.y * 65536u, X.z - Q.z * 65536u, X.w - Q.w * 65536u);
                } else {
                    P = __ldg(p4 + (m * 8 + t4) * 32 + lane);
                    Q = __ldg(q4 + (m * 8 + t4) * 32 + lane);
                }
                const uint32_t v0 = vmax_u16x2(lds_u32(rho, P.x), lds_u32(rho, Q.x));
                const uint32_t v1 = vmax_u16x2(lds_u32(rho, P.y), lds_u32(rho, Q.y));
                const uint32_t v2 = vmax_u16x2(lds_u32(rho, P.z), lds_u32(rho, Q.z));
                const uint32_t v3 = vmax_u16x2(lds_u32(rho, P.w), lds_u32(rho, Q.w));
                // v = [A 0 B 0] bytes: v0 + 256 v1 = [A0 A1 B0 B1] (no carries: an
                // add on the FMA pipe instead of a PRMT on the ALU pipe)
                const uint32_t x01 = v1 * 256u + v0;  // [A0 A1 B0 B1]
                const uint32_t x23 = v3 * 256u + v2;  // [A2 A3 B2 B3]
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
                bytes_to_planes_x(wa, ta);
                bytes_to_planes_x(wb, tb);
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
            // one pixel's planes at a time: the gathers run twice (the index
            // tables keep the 4-consecutive-positions order for MCH = 8, see
            // bsm_set_pattern, so the per-8-byte transposes keep register
            // pressure at the 128 budget)
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
    if (x0 + jl >= Wq) return;
    uint32_t* dst = mask + size_t(wl) * P + size_t(ly) * Wq + x0 + jl;
#pragma unroll 4
    for (int w = wl; w < NW; w += 32 / kM3Px, dst += size_t(32 / kM3Px) * P) {
        const uint32_t v = stage[jl * STG + w];
        *dst = w < G - 1 ? v : (w == G - 1 ? v & tail : 0u);
    }
}

// ---------------------------------------------------------------------------
// K2q -- the mask for four pixels per pass: the rank table holds one byte per
// pixel (the ranks are dense ranks of <= 256 distinct distances, so they fit
// u8), so one u32 gather serves four pixels -- half the rank-gather and
// index-load wavefronts per pixel of k_mask4.  The per-byte max runs as two
// VIMNMX.U16x2 on the even / odd byte lanes (masked operands); the four
// pixels' planes (8 x MCH x 4 words) are split over two warps: warp w owns
// chunks [w MCH/2, (w + 1) MCH/2) of every lane, i.e. the same 32-lane gather
// groups of the bank-balanced index tables as k_mask4 (so every gather is still
// one wavefront), and the MSB-first select adds the two warps' counts through
// shared memory with one CTA barrier per bit (the four pixels in lockstep).
// Output words: lane l, chunk m of the MCH -> word MCH l + m, as in k_mask4.
// Four pixels' select, MW chunks per lane in this warp; counts of the other warp
// arrive through xchg (double-buffered by bit parity: the barrier of round j - 1
// separates round j's reads from round j - 2's writes).
// bytes_to_planes_x with the right shifts as multiply-high (FMA pipe): for the
// ALU-bound k_mask_q (3 LOP3 + 2 IMAD per swap instead of SHF + 3 LOP3 + IMAD).
__device__ __forceinline__ void bytes_to_planes_xf(const uint32_t (&src)[8], uint32_t (&w)[8]) {
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = src[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t t = (__umulhi(w[k], 1u << 28) ^ w[k + 4]) & 0x0F0F0F0Fu;
        w[k + 4] ^= t;
        w[k] ^= t * 16u;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k & 2) continue;
        const uint32_t t = (__umulhi(w[k], 1u << 30) ^ w[k + 2]) & 0x33333333u;
        w[k + 2] ^= t;
        w[k] ^= t * 4u;
    }
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        const uint32_t t = (__umulhi(w[k], 1u << 31) ^ w[k + 1]) & 0x55555555u;
        w[k + 1] ^= t;
        w[k] ^= t * 2u;
    }
}

template <int MW>
__device__ __forceinline__ void select_le4x(const uint32_t (&pl)[4][8][MW], int k, uint32_t (&o)[4][MW],
                                            uint32_t* xchg, int warp, int lane) {
    uint32_t e[4][MW], l[4][MW];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int m = 0; m < MW; ++m) {
            e[p][m] = ~0u;
            l[p][m] = 0u;
        }
    int kk[4] = {k, k, k, k};
#pragma unroll
    for (int j = 7; j >= 0; --j) {
        uint32_t z[4][MW];
        int cs[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            uint32_t c = 0;
#pragma unroll
            for (int m = 0; m < MW; ++m) {
                z[p][m] = e[p][m] & ~pl[p][j][m];
                c += __popc(z[p][m]);
            }
            cs[p] = int(__reduce_add_sync(0xFFFFFFFFu, c));
        }
        uint32_t* buf = xchg + (j & 1) * 8;
        if (lane == 0)
            *reinterpret_cast<uint4*>(buf + 4 * warp) = make_uint4(uint32_t(cs[0]), uint32_t(cs[1]), uint32_t(cs[2]),
                                                                   uint32_t(cs[3]));
        __syncthreads();
        const uint4 ot = *reinterpret_cast<const uint4*>(buf + 4 * (warp ^ 1));
        const int tot[4] = {cs[0] + int(ot.x), cs[1] + int(ot.y), cs[2] + int(ot.z), cs[3] + int(ot.w)};
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            if (tot[p] < kk[p]) {  // block-uniform
                kk[p] -= tot[p];
#pragma unroll
                for (int m = 0; m < MW; ++m) {
                    l[p][m] |= z[p][m];
                    e[p][m] &= pl[p][j][m];
                }
            } else {
#pragma unroll
                for (int m = 0; m < MW; ++m) e[p][m] = z[p][m];
            }
        }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int m = 0; m < MW; ++m) o[p][m] = l[p][m] | e[p][m];
}

template <int MW, int PX = kM3Px>
__global__ void __launch_bounds__(64, 8)
    k_mask_q(const uint8_t* __restrict__ img, int W, int H, int ybeg, int rows, const uint4* __restrict__ pq4, int n,
             const uint32_t* __restrict__ ufill, int nfill, int u, int rho_words, const uint8_t* __restrict__ rank,
             int half, int TW, int NW, int Wq, size_t P, uint32_t* __restrict__ mask, const uint8_t* __restrict__ img2,
             uint32_t* __restrict__ mask2) {
    if (blockIdx.z) {  // second view of the pair (grid.z = 2)
        img = img2;
        mask = mask2;
    }
    constexpr int MCH = 2 * MW;
    constexpr int STG = mask4_stage_stride(MCH);
    extern __shared__ __align__(16) uint32_t dsm[];
    uint32_t* rho = dsm;                                   // rho_words: u8 ranks of 4 pixels per slot
    uint32_t* stage = rho + rho_words;                     // [PX][STG]
    uint32_t* xchg = stage + PX * STG;                     // [2][2 warps][4 pixels]
    uint8_t* rrows = reinterpret_cast<uint8_t*>(xchg + 16);  // 4 x 256
    uint8_t* tile = rrows + 1024;                          // (2h+1) x TW
    const int G = (n + 31) >> 5;
    const int TH = 2 * half + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int x0 = blockIdx.x * PX;
    const int ly = blockIdx.y;
    const int y = ybeg + ly;
    const int a0 = (x0 - half) & ~3, ay0 = y - half;
    const int sh = x0 - half - a0;
    if ((W & 3) == 0 && (reinterpret_cast<uintptr_t>(img) & 3) == 0 && a0 >= 0 && a0 + TW <= W && ay0 >= 0 &&
        ay0 + TH <= H) {
        const int nw = TW >> 2;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(img + size_t(ay0) * W + a0);
        for (int idx = tid; idx < TH * nw; idx += 64) {
            const int r = idx / nw;
            reinterpret_cast<uint32_t*>(tile)[idx] = __ldg(src + size_t(r) * (W >> 2) + (idx - r * nw));
        }
    } else {
        for (int idx = tid; idx < TW * TH; idx += 64) {
            const int r = idx / TW, c = idx - r * TW;
            const int gx = min(max(a0 + c, 0), W - 1);
            const int gy = min(max(ay0 + r, 0), H - 1);
            tile[idx] = __ldg(img + size_t(gy) * W + gx);
        }
    }
    if (tid == 0) rho[u] = 0xFFFFFFFFu;  // sentinel: a = 255 for all four pixels
    __syncthreads();

    const int k = max(1, n / 4);
    const int c0 = half * TW + sh + half;  // tile index of pixel x0
    uint4 rr = __ldg(reinterpret_cast<const uint4*>(rank + 256 * int(tile[c0 + (tid >> 4)])) + (tid & 15));
#pragma unroll 1
    for (int q = 0; q < PX; q += 4) {
        reinterpret_cast<uint4*>(rrows)[tid] = rr;  // rank rows of pixels q .. q + 3
        if (q + 4 < PX)
            rr = __ldg(reinterpret_cast<const uint4*>(rank + 256 * int(tile[c0 + q + 4 + (tid >> 4)])) + (tid & 15));
        __syncthreads();
        const uint8_t* tq = tile + sh + q;
        for (int j = tid; j < nfill; j += 64) {  // host fill order (see k_mask4)
            const uint32_t e = __ldg(ufill + j);
            const uint8_t* tp = tq + (e & 0xFFFFu);
            const uint32_t v01 = uint32_t(rrows[tp[0]]) | (uint32_t(rrows[256 + tp[1]]) << 8);
            const uint32_t v23 = uint32_t(rrows[512 + tp[2]]) | (uint32_t(rrows[768 + tp[3]]) << 8);
            rho[e >> 16] = v01 | (v23 << 16);
        }
        __syncthreads();

        uint32_t pl[4][8][MW];
#pragma unroll
        for (int mw = 0; mw < MW; ++mw) {
            const int m = warp * MW + mw;  // chunk of the shared index tables
            uint32_t wa[8], wb[8], wc[8], wd[8];
#pragma unroll
            for (int t4 = 0; t4 < 8; ++t4) {
                // one load of P | Q << 16, split on the FMA pipe (k_mask4)
                const uint4 X = __ldg(pq4 + (m * 8 + t4) * 32 + lane);
                const uint4 Q = make_uint4(__umulhi(X.x, 65536u), __umulhi(X.y, 65536u), __umulhi(X.z, 65536u),
                                           __umulhi(X.w, 65536u));
                const uint4 Pp = make_uint4(X.x - Q.x * 65536u, X.y - Q.y * 65536u, X.z - Q.z * 65536u,
                                            X.w - Q.w * 65536u);
                const uint32_t p0 = lds_u32(rho, Pp.x), q0 = lds_u32(rho, Q.x);
                const uint32_t p1 = lds_u32(rho, Pp.y), q1 = lds_u32(rho, Q.y);
                const uint32_t p2 = lds_u32(rho, Pp.z), q2 = lds_u32(rho, Q.z);
                const uint32_t p3 = lds_u32(rho, Pp.w), q3 = lds_u32(rho, Q.w);
                // The high byte of a u16 max is the max of the high bytes (ties
                // included), so max.u16x2 of the words gives pixels 1, 3 in bytes 1, 3
                // and of the words shifted left by 8 (IMAD, FMA pipe) pixels 0, 2.
                const uint32_t e0 = vmax_u16x2(p0 * 256u, q0 * 256u);  // [. A . C]
                const uint32_t e1 = vmax_u16x2(p1 * 256u, q1 * 256u);
                const uint32_t e2 = vmax_u16x2(p2 * 256u, q2 * 256u);
                const uint32_t e3 = vmax_u16x2(p3 * 256u, q3 * 256u);
                const uint32_t o0 = vmax_u16x2(p0, q0);  // [. B . D]
                const uint32_t o1 = vmax_u16x2(p1, q1);
                const uint32_t o2 = vmax_u16x2(p2, q2);
                const uint32_t o3 = vmax_u16x2(p3, q3);
                const uint32_t x01 = __byte_perm(e0, e1, 0x7351);  // [A0 A1 C0 C1]
                const uint32_t x23 = __byte_perm(e2, e3, 0x7351);  // [A2 A3 C2 C3]
                const uint32_t y01 = __byte_perm(o0, o1, 0x7351);  // [B0 B1 D0 D1]
                const uint32_t y23 = __byte_perm(o2, o3, 0x7351);
                wa[t4] = __byte_perm(x01, x23, 0x5410);
                wc[t4] = __byte_perm(x01, x23, 0x7632);
                wb[t4] = __byte_perm(y01, y23, 0x5410);
                wd[t4] = __byte_perm(y01, y23, 0x7632);
            }
            uint32_t t[8];
            bytes_to_planes_xf(wa, t);
#pragma unroll
            for (int j = 0; j < 8; ++j) pl[0][j][mw] = t[j];
            bytes_to_planes_xf(wb, t);
#pragma unroll
            for (int j = 0; j < 8; ++j) pl[1][j][mw] = t[j];
            bytes_to_planes_xf(wc, t);
#pragma unroll
            for (int j = 0; j < 8; ++j) pl[2][j][mw] = t[j];
            bytes_to_planes_xf(wd, t);
#pragma unroll
            for (int j = 0; j < 8; ++j) pl[3][j][mw] = t[j];
        }
        uint32_t o[4][MW];
        select_le4x<MW>(pl, k, o, xchg, warp, lane);
#pragma unroll
        for (int p = 0; p < 4; ++p) store_words<MW>(stage + (q + p) * STG + MCH * lane + MW * warp, o[p]);
        __syncthreads();  // rho / rrows are rewritten by the next pass
    }
    // thread = (word offset w % 8, pixel j)
    const int rem = n & 31;
    const uint32_t tail = rem ? (1u << rem) - 1u : ~0u;
    const int jl = tid & (PX - 1), wl = tid / PX;
    if (x0 + jl >= Wq) return;
    uint32_t* dst = mask + size_t(wl) * P + size_t(ly) * Wq + x0 + jl;
#pragma unroll 4
    for (int w = wl; w < NW; w += 64 / PX, dst += size_t(64 / PX) * P) {
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

// The float at byte offset `off` from `base` (the pair table holds byte offsets).
__device__ __forceinline__ float ldf_off(const float* base, int off) {
    return *reinterpret_cast<const float*>(reinterpret_cast<const char*>(base) + off);
}

__global__ void __launch_bounds__(kDfTX* kDfTY)
    k_descriptor_f32(const float* __restrict__ gray, int W, int H, int ybeg, int rows, const int2* __restrict__ offs,
                     int n, int half, int NW, int Wq, size_t P, uint32_t* __restrict__ desc) {
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
                    if (ldf_off(t0 + j * TW, o.x) > ldf_off(t0 + j * TW, o.y)) acc[j] |= 1u << k;
            }
        } else {
            for (int k = 0; k < cnt; ++k) {
                const int2 o = __ldg(offs + 32 * w + k);
#pragma unroll
                for (int j = 0; j < kDfPY; ++j)
                    acc[j] |= uint32_t(ldf_off(t0 + j * TW, o.x) > ldf_off(t0 + j * TW, o.y)) << k;
            }
        }
#pragma unroll
        for (int j = 0; j < kDfPY; ++j) {
            const int ly = ly0 + threadIdx.y * kDfPY + j;
            if (ly < rows && x < Wq) desc[size_t(w) * P + size_t(ly) * Wq + x] = acc[j];
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
               int NW, int Wq, size_t P, uint32_t* __restrict__ mask, int half, int force_low) {
    // Lab samples (float4 per pixel) are read through L1 (no shared tile):
    // shared memory holds only the slot keys and 23 rows of bit planes (key
    // bits 30..8: SADs are non-negative floats, so bit 31 is 0 in every key;
    // the low byte's planes reuse the rows of bits 8..15), for occupancy.
    extern __shared__ __align__(16) uint32_t dsm[];
    uint32_t* tv = dsm;                                   // rho_words: SAD bits per slot (+ sentinel)
    uint32_t* planes = tv + rho_words;                    // [23 rows][MCH chunks][32 lanes]
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
                    // positions t4 + 8c (MCH <= 4) or 4 t4 + c (MCH = 8): the
                    // index tables' order (bsm_set_pattern)
                    constexpr int S1 = MCH <= 4 ? 1 : 4, S2 = MCH <= 4 ? 8 : 1;
                    x[S1 * t4] = max(lds_u32(tv, P.x), lds_u32(tv, Q.x));
                    x[S1 * t4 + S2] = max(lds_u32(tv, P.y), lds_u32(tv, Q.y));
                    x[S1 * t4 + 2 * S2] = max(lds_u32(tv, P.z), lds_u32(tv, Q.z));
                    x[S1 * t4 + 3 * S2] = max(lds_u32(tv, P.w), lds_u32(tv, Q.w));
                }
                transpose32(x);
                store(m, x);
            }
        };
        planes_of([&](int m, const uint32_t (&x)[32]) {
#pragma unroll
            for (int j = 8; j < 31; ++j) planes[(prow(j) * MCH + m) * 32 + lane] = x[j];
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
        // bit 31 is 0 for every key; the pads (0xFFFFFFFF) drop out of eq at
        // the first 0 bit of the threshold, which a finite key always has
        rounds(30, 8);
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
        // (force_low: test hook, BSM_MASKF_FORCE_LOW=1 -- resolve the low byte for every pixel)
        if (force_low || __reduce_min_sync(full, mn) != __reduce_max_sync(full, mx)) {
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
            if (w < NW && x0 + px < Wq) {
                uint32_t v = lt[m] | eq[m];
                if (w >= G) v = 0u;
                else if (rem && w == G - 1) v &= (1u << rem) - 1u;
                mask[size_t(w) * P + size_t(ly) * Wq + x0 + px] = v;
            }
        }
        __syncwarp();
    }
}
