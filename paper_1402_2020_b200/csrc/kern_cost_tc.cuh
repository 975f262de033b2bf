// kern_cost_tc.cuh -- K3 on the tensor cores: the masked Hamming costs of a
// tile of reference pixels against the span of other-view pixels it can match
// as one int8 tcgen05 MMA, fused with the winner-take-all argmin.  Part of
// bsm_kernels.cu's single translation unit (after kern_cost.cuh, whose
// mbarrier / TMA helpers it uses).
//
// The algebra (matcher.hpp:24-29, bitstring.hpp:73-88): for reference bits a,
// mask m and other-view bits b,
//     popc((a ^ b) & m) = popc(a & m) + sum_k b_k * m_k * (1 - 2 a_k),
// so with A[x][k] = m_k (1 - 2 a_k) in {-1, 0, +1} and B[x'][k] = -b_k in
// {-1, 0}, the cost of (x, x') is  base(x) - (A . B^T)[x][x'],  base(x) =
// popc(a & m).  Every product and partial sum is a small integer, so the s32
// accumulation is exact: the keys equal the popcount kernel's bit for bit.
// (Unmasked: m = all ones.)  A permutation of k applied to both operands
// leaves the dot product unchanged; the expansion uses one: u32 word ->
// 32 int8 K-elements, element 4c + j = bit c of byte j (prmt sign replicate).
//
// A tile is M = 128 consecutive reference pixels (flat index, may straddle
// rows, as in k_cost_wta) and one d-block of dc <= 256 disparities.  Its
// correspondences x' = x -+ d lie in a span of 127 + dc other-view pixels
// (128 + dq, dq = dc - 1 rounded up to 4, so that the span starts on a 16-byte
// boundary), so one accumulator of 128 TMEM lanes x ncols (128 + dq rounded up
// to 32) columns holds every cost the tile needs; row r uses columns r + u,
// u in [0, dq].
// Per stage of kTcKS u32 words (kTcKS MMA K-steps of 32 int8):
//   * a loader thread brings the packed words with TMA (2-D boxes of the word
//     planes: reference desc + mask [KS x 128], span [KS x ncols] as two
//     boxes) into a ring of kTcRawStages slots, zero-filled outside the
//     field; ~60 KB per SM in flight covers the DRAM latency of the
//     compulsory misses;
//   * 16 producer warps expand them: the A rows into TMEM (tcgen05.st, ring
//     of kTcStages x 32 columns), the B rows into shared memory (canonical
//     no-swizzle K-major layout, ring of kTcStages slots);
//   * one thread issues the MMAs (N <= 256 each, two per K-step for
//     ncols > 256) and commits the slot back to the producers;
//   * after the last stage, four epilogue warps read their 32 lanes'
//     accumulator columns (tcgen05.ld) and reduce the keys (cost << 16) | d
//     to the per-pixel minimum (ties -> smaller d, matcher.hpp:68-75), then
//     release the accumulator.
// CTAs are persistent (one per SM: the whole 512-column TMEM), walking the
// (tile, direction x d-block) items tile-major like k_cost_wta.
#pragma once

constexpr int kTcRows = 128;                      // MMA M: reference pixels per tile
constexpr int kTcKS = 4;                          // u32 words (MMA K-steps) per stage
constexpr int kTcStages = 3;                      // expanded ring (smem B + TMEM A)
constexpr int kTcRawStages = 6;                   // TMA ring of packed words
constexpr int kTcMaxDc = 256;                     // disparities per d-block
constexpr int kTcMaxCols = 384;                   // accumulator columns (127 + 256 -> 384)
constexpr int kTcAcol = kTcMaxCols;               // first TMEM column of the A ring
constexpr int kTcProdWarps = 16;                  // warp w: TMEM lane quarter w & 3, word w >> 2
constexpr int kTcEpiWarps = 4;
constexpr int kTcMmaWarp = kTcProdWarps + kTcEpiWarps;
constexpr int kTcLoadWarp = kTcMmaWarp + 1;
constexpr int kTcThreads = (kTcLoadWarp + 1) * 32;
static_assert(kTcProdWarps == 4 * kTcKS, "one producer warp per (lane quarter, word of the stage)");
static_assert(kTcAcol + kTcStages * kTcKS * 8 <= 512, "TMEM: accumulator + A ring");

__device__ __forceinline__ uint32_t tc_sign_bytes(uint32_t x) {
    // each byte -> 0xFF if its top bit is set, else 0x00 (prmt sign replicate)
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ uint64_t tc_smem_desc(uint32_t saddr) {
    // K-major, no swizzle: core matrices of 8 rows x 16 B; the two K halves of
    // a row group 128 B apart (LBO), row groups 256 B apart (SBO); version 1.
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
           (uint64_t(1) << 46);
}
__device__ __forceinline__ uint32_t tc_idesc_i8(int n) {
    // D s32, A s8, B s8, both K-major, N = n, M = 128
    return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(kTcRows >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Item `it` of the persistent walk: tile-major over (tile, direction x d-block).
// dq = dc - 1 rounded up to 4: the left span starts at p0 - d0 - dq, a multiple of
// 4 pixels (a TMA box whose first coordinate is not 16-byte aligned traps).
struct TcItem {
    int p0, dir, d0, dc, dq;
};
__device__ __forceinline__ TcItem tc_item(int it, int ndd, int ndir, int dir0, int Dc, int D) {
    const int per = ndd * ndir, tile = it / per, r = it - tile * per;
    const int dir = dir0 ^ (r >= ndd ? 1 : 0);
    const int d0 = (r >= ndd ? r - ndd : r) * Dc;
    const int dc = min(Dc, D - d0);
    return TcItem{tile * kTcRows, dir, d0, dc, (dc + 2) & ~3};
}

// Shared memory carve-up (bytes), shared by the kernel and the host.
struct TcSmem {
    uint32_t sub, stage, raw_a, raw, b_ring, raw_ring, base, bars, total;
    __host__ __device__ TcSmem(int ncols, bool masked) {
        sub = uint32_t(ncols) * 32u;                                      // one K-step of B rows
        stage = sub * kTcKS;                                              // expanded B stage
        raw_a = kTcKS * kTcRows * 4u;                                     // one [KS x 128] word box
        raw = raw_a * (masked ? 2u : 1u) + kTcKS * uint32_t(ncols) * 4u;  // packed words of a stage
        b_ring = 0;
        raw_ring = b_ring + kTcStages * stage;
        base = raw_ring + kTcRawStages * raw;
        bars = base + 2 * kTcKS * kTcRows * 4;
        total = bars + (2 * kTcStages + 2 * kTcRawStages + 6) * 8 + 16;
    }
};

template <bool MASKED>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_cost_wta_tc(const __grid_constant__ CUtensorMap l_ref, const __grid_constant__ CUtensorMap l_mask,
                  const __grid_constant__ CUtensorMap l_oth, const __grid_constant__ CUtensorMap r_ref,
                  const __grid_constant__ CUtensorMap r_mask, const __grid_constant__ CUtensorMap r_oth, int W,
                  int Wq, int npix, int NW, int D, int Dc, int ncols, int ndd, int ndir, int dir0, int items,
                  uint32_t* __restrict__ keys_l, uint32_t* __restrict__ keys_r) {
    extern __shared__ __align__(1024) uint8_t tsm[];
    const TcSmem L(ncols, MASKED);
    uint8_t* sB = tsm + L.b_ring;                                        // [S][KS][ncols rows x 32 B]
    uint32_t* sraw = reinterpret_cast<uint32_t*>(tsm + L.raw_ring);      // [RS][desc | mask | span]
    uint32_t* sbase = reinterpret_cast<uint32_t*>(tsm + L.base);         // [2 tiles][KS words][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(tsm + L.bars);
    uint64_t* full = bars;                               // [S] producers -> MMA (one arrival per warp)
    uint64_t* empty = full + kTcStages;                  // [S] MMA commit -> producers
    uint64_t* raw_full = empty + kTcStages;              // [RS] TMA bytes -> producers
    uint64_t* raw_empty = raw_full + kTcRawStages;       // [RS] producers (one arrival per warp) -> loader
    uint64_t* acc_full = raw_empty + kTcRawStages;       // MMA commit -> epilogue
    uint64_t* acc_empty = acc_full + 1;                  // epilogue (4 warps) -> MMA
    uint64_t* base_full = acc_full + 2;                  // [2] producers -> epilogue
    uint64_t* base_empty = acc_full + 4;                 // [2] epilogue -> producers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 6);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(full + s, kTcProdWarps);
            mbar_init(empty + s, 1);
        }
        for (int s = 0; s < kTcRawStages; ++s) {
            mbar_init(raw_full + s, 1);
            mbar_init(raw_empty + s, kTcProdWarps);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, kTcEpiWarps);
        for (int i = 0; i < 2; ++i) {
            mbar_init(base_full + i, kTcProdWarps);
            mbar_init(base_empty + i, kTcEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kTcMmaWarp) {  // the MMA warp owns the TMEM allocation
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nst = (NW + kTcKS - 1) / kTcKS;  // stages per tile
    const int half = ncols / 2;                // span pixels per TMA box

    if (warp < kTcProdWarps) {
        // ---------------- producers ----------------
        // A: warp w writes TMEM lanes 32 (w & 3) .. +31 (its lane quarter), the 8
        // columns of word w >> 2 of each stage.  B: thread tid expands span row
        // tid (when < ncols), all kTcKS words of the stage.
        const int q = warp & 3, jw = warp >> 2;
        const int arow = q * 32 + lane;
        const uint32_t a_taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(kTcAcol + 8 * jw);
        const bool has_b = tid < ncols;  // warp-uniform (ncols is a multiple of 32)
        const uint32_t boff = uint32_t((tid >> 3) * 256 + (tid & 7) * 16);
        const uint32_t raw_words = L.raw / 4;
        const uint32_t* rd = sraw + jw * kTcRows + arow;                  // desc word of this A row
        const uint32_t* rm = sraw + L.raw_a / 4 + jw * kTcRows + arow;    // mask word
        // span row tid: box 0 holds rows [0, half), box 1 rows [half, ncols), each [KS][half]
        const uint32_t* rb = sraw + (L.raw_a / 4) * (MASKED ? 2 : 1) + (tid < half ? tid : half * kTcKS + tid - half);
        uint32_t g = 0;  // global stage counter
        int t = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++t) {
            uint32_t base = 0;
            for (int st = 0; st < nst; ++st, ++g) {
                const uint32_t r = g % kTcRawStages, s = g % kTcStages;
                mbar_wait(raw_full + r, (g / kTcRawStages) & 1u);
                const uint32_t a = rd[r * raw_words];
                const uint32_t m = MASKED ? rm[r * raw_words] : 0xFFFFFFFFu;
                uint32_t b[kTcKS];
                if (has_b) {
#pragma unroll
                    for (int j = 0; j < kTcKS; ++j) b[j] = rb[r * raw_words + j * half];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(raw_empty + r);
                // A: byte = m ? (a ? -1 : +1) : 0; column c of a word = bit c of each byte
                const uint32_t u = a & m;
                base += __popc(u);
                uint32_t av[8];
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    av[c] = tc_sign_bytes(u << (7 - c)) | (tc_sign_bytes(m << (7 - c)) & 0x01010101u);
                mbar_wait(empty + s, ((g / kTcStages) & 1u) ^ 1u);
                tc_fence_after();
                __syncwarp();
                tc_st8(a_taddr + s * (kTcKS * 8), av);
                if (has_b) {
                    uint8_t* slot = sB + s * L.stage + boff;
#pragma unroll
                    for (int j = 0; j < kTcKS; ++j) {
                        uint32_t bv[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) bv[c] = tc_sign_bytes(b[j] << (7 - c));
                        *reinterpret_cast<uint4*>(slot + j * L.sub) = make_uint4(bv[0], bv[1], bv[2], bv[3]);
                        *reinterpret_cast<uint4*>(slot + j * L.sub + 128) = make_uint4(bv[4], bv[5], bv[6], bv[7]);
                    }
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B rows -> tensor-core reads
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(full + s);
            }
            // popc(a & m) of this tile's pixels (this warp's words), for the epilogue
            const int par = t & 1;
            mbar_wait(base_empty + par, (uint32_t(t >> 1) & 1u) ^ 1u);
            sbase[(par * kTcKS + jw) * kTcRows + arow] = base;
            __syncwarp();
            if (lane == 0) mbar_arrive(base_full + par);
        }
    } else if (warp < kTcMmaWarp) {
        // ---------------- epilogue ----------------
        const int q = warp & 3, r = q * 32 + lane;
        const uint32_t lane_taddr = tmem + (uint32_t(q * 32) << 16);
        int t = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++t) {
            const TcItem w = tc_item(it, ndd, ndir, dir0, Dc, D);
            const int p = w.p0 + r, y = p / Wq, x = p - y * Wq;
            const bool pix_ok = p < npix && x < W;
            // column j of row r is u = j - r: right d = d0 + u, left d = d0 + dq - u.
            // valid u in [ulo, uhi): d in [d0, d0 + dc), left d <= x, right
            // x + d < W (matcher.hpp:100: out-of-image correspondences skipped)
            int ulo, uhi;
            if (w.dir) {
                ulo = 0;
                uhi = min(w.dc, W - x - w.d0);
            } else {
                ulo = w.dq + 1 - min(w.dc, x + 1 - w.d0);
                uhi = w.dq + 1;
            }
            if (!pix_ok || uhi < ulo) uhi = ulo;
            const uint32_t span = uint32_t(uhi - ulo);
            const int par = t & 1;
            mbar_wait(base_full + par, uint32_t(t >> 1) & 1u);
            uint32_t base = 0;
#pragma unroll
            for (int j = 0; j < kTcKS; ++j) base += sbase[(par * kTcKS + j) * kTcRows + r];
            __syncwarp();
            if (lane == 0) mbar_arrive(base_empty + par);
            mbar_wait(acc_full, uint32_t(t) & 1u);
            tc_fence_after();
            uint32_t best = 0xFFFFFFFFu;
            const int cend = q * 32 + 32 + w.dq;  // last column any lane of this warp uses, + 1
            for (int c0 = q * 32; c0 < cend; c0 += 32) {
                uint32_t v[32];
                __syncwarp();
                tc_ld32(lane_taddr + uint32_t(c0), v);
                const int u0 = c0 - r - ulo;  // element i is valid iff (unsigned)(u0 + i) < span
                // key = (base - acc) << 16 | d with u = c0 + i - r
                const uint32_t kb = (base << 16) + uint32_t(w.dir ? w.d0 + c0 - r : w.d0 + w.dq - c0 + r);
                if (w.dir) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const uint32_t key = (kb - (v[i] << 16)) + uint32_t(i);
                        if (uint32_t(u0 + i) < span) best = min(best, key);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const uint32_t key = (kb - (v[i] << 16)) - uint32_t(i);
                        if (uint32_t(u0 + i) < span) best = min(best, key);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
            if (pix_ok && best != 0xFFFFFFFFu) {
                uint32_t* keys = w.dir ? keys_r : keys_l;
                if (ndd == 1) keys[size_t(y) * W + x] = best;
                else atomicMin(&keys[size_t(y) * W + x], best);
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ---------------- MMA issuer (lane 0 issues; the warp waits with it) ----------------
        const int n1 = min(ncols, 256), n2 = ncols - n1;
        const uint32_t id1 = tc_idesc_i8(n1), id2 = tc_idesc_i8(n2 > 0 ? n2 : 16);
        const uint32_t sB_addr = smem_addr(sB);
        uint32_t g = 0;
        int t = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++t) {
            mbar_wait(acc_empty, (uint32_t(t) & 1u) ^ 1u);
            tc_fence_after();
            for (int st = 0; st < nst; ++st, ++g) {
                const uint32_t s = g % kTcStages;
                mbar_wait(full + s, (g / kTcStages) & 1u);
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int j = 0; j < kTcKS; ++j) {
                        const uint32_t a_t = tmem + uint32_t(kTcAcol) + s * (kTcKS * 8) + j * 8;
                        const uint32_t b_addr = sB_addr + s * L.stage + j * L.sub;
                        const uint32_t acc = (st > 0 || j > 0) ? 1u : 0u;
                        tc_mma_i8(tmem, a_t, tc_smem_desc(b_addr), id1, acc);
                        if (n2 > 0)
                            tc_mma_i8(tmem + uint32_t(n1), a_t, tc_smem_desc(b_addr + uint32_t(n1 / 8) * 256u), id2, acc);
                    }
                    tc_commit(empty + s);
                }
                __syncwarp();
            }
            if (lane == 0) tc_commit(acc_full);
            __syncwarp();
        }
    } else {
        // ---------------- TMA loader (lane 0 issues; the warp waits with it) ----------------
        uint32_t g = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            const TcItem w = tc_item(it, ndd, ndir, dir0, Dc, D);
            const int q0 = w.dir ? w.p0 + w.d0 : w.p0 - w.d0 - w.dq;  // span row 0 (a multiple of 4)
            for (int st = 0; st < nst; ++st, ++g) {
                const uint32_t r = g % kTcRawStages;
                mbar_wait(raw_empty + r, ((g / kTcRawStages) & 1u) ^ 1u);
                if (lane == 0) {
                    uint32_t* dst = sraw + r * (L.raw / 4);
                    uint32_t* db = dst + (L.raw_a / 4) * (MASKED ? 2 : 1);
                    // the tensor maps are addressed directly (a runtime-selected pointer
                    // to a __grid_constant__ parameter would be a local copy)
                    auto issue = [&](const CUtensorMap* mr, const CUtensorMap* mm, const CUtensorMap* mo) {
// A span box wholly outside the field is not loaded (a box
                        // starting further left than its width traps): its rows
                        // only meet out-of-image cells, so stale words are harmless.
                        const bool b0 = q0 + half > 0 && q0 < npix, b1 = q0 + 2 * half > 0 && q0 + half < npix;
                        const uint32_t hb = uint32_t(half) * kTcKS * 4;
                        mbar_expect_tx(raw_full + r, L.raw_a * (MASKED ? 2 : 1) + (b0 ? hb : 0) + (b1 ? hb : 0));
                        tma_load_2d(dst, mr, w.p0, st * kTcKS, raw_full + r);
                        if (MASKED) tma_load_2d(dst + L.raw_a / 4, mm, w.p0, st * kTcKS, raw_full + r);
                        if (b0) tma_load_2d(db, mo, q0, st * kTcKS, raw_full + r);
                        if (b1) tma_load_2d(db + half * kTcKS, mo, q0 + half, st * kTcKS, raw_full + r);
                    };
                    if (w.dir) issue(&r_ref, &r_mask, &r_oth);
                    else issue(&l_ref, &l_mask, &l_oth);
                }
                __syncwarp();
            }
        }
    }
    __syncthreads();
    if (warp == kTcMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}
