// kern_cost.cuh -- K3: TMA staging helpers and the fused masked-Hamming cost +
// winner-take-all kernel.  Part of bsm_kernels.cu's single translation unit.
#pragma once

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
// 2-D box (pixel, word) of a field into shared memory, completing on bar.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int p, int w, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(p), "r"(w), "r"(smem_addr(bar))
        : "memory");
}
// Arrival on a shared-memory counter with CTA-scope acquire-release ordering;
// returns the previous value.
__device__ __forceinline__ uint32_t smem_arrive_count(uint32_t* ctr) {
    uint32_t old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n" : "=r"(old) : "r"(smem_addr(ctr)) : "memory");
    return old;
}

// ---------------------------------------------------------------------------
// K3 -- fused masked Hamming cost + winner-take-all.  matcher.hpp:80-113
// (wta), :24-29/bitstring.hpp:73-88 (masked_hamming), :35-38 (other_column),
// :68-75 (ties -> smaller d).  No cost volume is materialised.
//
// Pixels are tiled over the flat index p = y * Wq + x of the field planes
// (Wq = W rounded up to 4), so a 128-pixel tile may cover the end of one row
// and the start of the next: no lane idles on padding to a tile multiple, and
// a correspondence p -+ d is valid exactly when x -+ d stays inside the row.
// CTA tile: 128 reference pixels x 64 disparities; 8 warps, warp wi owns
// disparities [d0 + 8wi, +8), lane l owns pixels [p0 + 4l, +4) (one row: Wq and
// p0 + 4l are multiples of 4): a 4 x 8 register block of costs, so each staged
// word feeds 32 word-ops from 5 LDS.128 (ref desc, ref mask, a 12-word window
// of the other view).
// Words stream through a 3-stage ring of K = 16 words filled by TMA: one
// thread arms the stage's mbarrier and issues three tensor-box copies
// ([K x 128] desc, [K x 128] mask, [K x 192] other-view span); pixels and
// words outside the field arrive zero-filled, so the load path carries no
// per-thread predicates or address arithmetic.  Each warp, once done with a
// slot, arrives on the slot's counter (acquire-release, CTA scope); the LAST
// of the 8 warps refills it, so no warp waits for the others between stages.
// Warps whose (pixel, d) block has no in-range correspondence skip the
// arithmetic; CTAs with none exit.  The argmin key is (cost << 16) | d (min
// cost, then smaller d); d-split CTAs merge with atomicMin.  Out-of-image
// correspondences are skipped (matcher.hpp:100).
// One launch covers both directions (blockIdx.y = direction x d-block).
template <bool RIGHT, bool MASKED, bool LASTREFILL>
__device__ __forceinline__ void cost_wta_tile(const CUtensorMap* tm_ref, const CUtensorMap* tm_mask,
                                              const CUtensorMap* tm_oth, int W, int Wq, int npix, int NW, int D,
                                              int p0, int d0, bool split, uint32_t* __restrict__ keys, uint32_t two) {
    constexpr int T = kCostTile, DC = kCostDisp, K = kCostK, ST = kCostStages, BW = T + DC;
    constexpr int SA = K * T, SB = K * BW;
    constexpr int STAGE = (MASKED ? 2 * SA : SA) + SB;
    constexpr uint32_t STAGE_BYTES = uint32_t(STAGE) * 4;
    extern __shared__ __align__(128) uint32_t csm[];
    uint32_t* red = csm + ST * STAGE;                                 // [8][T]
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 8 * T);         // [ST] full barriers
    uint64_t* empty = bars + ST;                                       // [ST] empty barriers (!LASTREFILL)
    uint32_t* ctr = reinterpret_cast<uint32_t*>(bars + 2 * ST);        // [ST] slot-release counters

    const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
    const int bbase = RIGHT ? p0 + d0 : p0 - d0 - DC;
    const int nchunks = (NW + K - 1) / K;
    // this lane's 4 pixels: row yl, columns xl .. xl + 3
    const int pl = p0 + lane * 4;
    const int yl = pl / Wq, xl = pl - yl * Wq;
    const bool lane_in = pl < npix && xl < W;
    const int ds = wi * 8, dlo = d0 + ds;
    const bool any = lane_in && dlo < D && (RIGHT ? xl + dlo < W : min(xl + 3, W - 1) >= dlo);
    const bool busy = __any_sync(0xFFFFFFFFu, any);

    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(bars + s, 1);
            mbar_init(empty + s, 8);  // one arrival per warp
            ctr[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (!__syncthreads_or(busy)) return;  // no in-range correspondence in the whole tile
    auto load_stage = [&](int c, int st) {
        uint32_t* s = csm + st * STAGE;
        mbar_expect_tx(bars + st, STAGE_BYTES);
        tma_load_2d(s, tm_ref, p0, c * K, bars + st);
        if constexpr (MASKED) tma_load_2d(s + SA, tm_mask, p0, c * K, bars + st);
        tma_load_2d(s + (MASKED ? 2 * SA : SA), tm_oth, bbase, c * K, bars + st);
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
    const int c0 = RIGHT ? xs + ds : xs - ds + DC - 8;

#pragma unroll 1
    for (int c = 0; c < nchunks; ++c) {
        const int st = c % ST;
        mbar_wait(bars + st, uint32_t(c / ST) & 1u);
        if (busy) {
        // lane pointers into the slot, advanced by two words per iteration
        const uint32_t* pa = csm + st * STAGE + xs;
        const uint32_t* pb = csm + st * STAGE + (MASKED ? 2 * SA : SA) + c0;
#pragma unroll 1
        for (int w = 0; w < K; w += 2, pa += 2 * T, pb += 2 * BW) {
            uint32_t a[2][4], m[2][4], b[2][12];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint4 a4 = *reinterpret_cast<const uint4*>(pa + h * T);
                uint4 m4 = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
                if constexpr (MASKED) m4 = *reinterpret_cast<const uint4*>(pa + SA + h * T);
                const uint4 b0 = *reinterpret_cast<const uint4*>(pb + h * BW);
                const uint4 b1 = *reinterpret_cast<const uint4*>(pb + h * BW + 4);
                const uint4 b2 = *reinterpret_cast<const uint4*>(pb + h * BW + 8);
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
        __syncwarp();
        if constexpr (LASTREFILL) {
            // release the slot; the last of the 8 warps refills it
            if (lane == 0 && c + ST < nchunks && (smem_arrive_count(ctr + st) & 7u) == 7u) load_stage(c + ST, st);
        } else {
            // release the slot; thread 0 refills it once all 8 warps are done
            if (lane == 0) mbar_arrive(empty + st);
            if (tid == 0 && c + ST < nchunks) {
                mbar_wait(empty + st, uint32_t(c / ST) & 1u);
                load_stage(c + ST, st);
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int s = 0; s < 8; ++s) acc[j][s] += __popc(ones[j][s]);

    // the epilogue's pixel coordinates are recomputed here (from a laundered
    // lane index) rather than kept live through the word loop, whose 4 x 8
    // cells already hold 128 registers
    int lane2;
    asm volatile("mov.u32 %0, %1;" : "=r"(lane2) : "r"(lane));
    const int pe = p0 + lane2 * 4;
    const int ye = pe / Wq, xe = pe - ye * Wq;
    const bool lane_ok = pe < npix;
    const int de = d0 + (tid >> 5) * 8;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int x = xe + j;
        uint32_t best = 0xFFFFFFFFu;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int d = de + s;
            const bool ok = lane_ok && x < W && d < D && (RIGHT ? x + d < W : x >= d);
            const uint32_t key = (acc[j][s] << 16) | uint32_t(d);
            if (ok && key < best) best = key;
        }
        red[(tid >> 5) * T + lane2 * 4 + j] = best;
    }
    __syncthreads();
    if (tid < T) {
        uint32_t best = red[tid];
#pragma unroll
        for (int w = 1; w < 8; ++w) best = min(best, red[w * T + tid]);
        const int p = p0 + tid;
        const int y = p / Wq, x = p - y * Wq;
        if (p < npix && x < W && best != 0xFFFFFFFFu) {
            if (!split) keys[size_t(y) * W + x] = best;
            else atomicMin(&keys[size_t(y) * W + x], best);
        }
    }
}

// 1-D grid over (tile, dd), ndd = dz (x 2 when both directions run in this
// launch), in groups of `group` consecutive tiles: inside a group the order is
// d-block-major, across groups tile-major (group = 1: tile-major, the default:
// the d-blocks and both directions of a tile are launch-order neighbours, so
// the tile's words are re-read from L2, not DRAM; group = tiles: d-major).
// dd < dz: d-block dd of direction dir0; dd >= dz: d-block dd - dz of the other direction
// (0 = left reference, x - d; 1 = right reference, x + d).  The left-reference
// maps / keys are l_*, keys_l; the right-reference ones r_*, keys_r.
template <bool MASKED, bool LASTREFILL>
__global__ void __launch_bounds__(256, 2)
    k_cost_wta(const __grid_constant__ CUtensorMap l_ref, const __grid_constant__ CUtensorMap l_mask,
               const __grid_constant__ CUtensorMap l_oth, const __grid_constant__ CUtensorMap r_ref,
               const __grid_constant__ CUtensorMap r_mask, const __grid_constant__ CUtensorMap r_oth, int W, int Wq,
               int rows, int NW, int D, int dz, int ndd, int tiles, int group, int dir0, uint32_t* __restrict__ keys_l,
               uint32_t* __restrict__ keys_r, uint32_t two) {
    const unsigned span = unsigned(group) * unsigned(ndd), g = blockIdx.x / span, r = blockIdx.x % span;
    const unsigned gsz = min(unsigned(group), unsigned(tiles) - g * unsigned(group));  // the last group may be short
    const int tile = int(g * unsigned(group) + r % gsz), dd = int(r / gsz);
    const bool second = dd >= dz;
    const int dir = dir0 ^ (second ? 1 : 0);
    const int d0 = (second ? dd - dz : dd) * kCostDisp;
    const int p0 = tile * kCostTile;
    if (dir)
        cost_wta_tile<true, MASKED, LASTREFILL>(&r_ref, &r_mask, &r_oth, W, Wq, rows * Wq, NW, D, p0, d0, dz > 1,
                                                keys_r, two);
    else
        cost_wta_tile<false, MASKED, LASTREFILL>(&l_ref, &l_mask, &l_oth, W, Wq, rows * Wq, NW, D, p0, d0, dz > 1,
                                                 keys_l, two);
}
