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
// Per stage of kTcKS (8) u32 words (8 MMA K-steps of 32 int8):
//   * a loader thread brings the span's packed words with TMA (two 2-D boxes
//     [KS x ncols/2] of the other view's word planes) into a ring of as many
//     slots as fit in shared memory (2..8), zero-filled outside the field;
//   * 16 B-producer warps expand them into the B rows of the stage in shared
//     memory (canonical no-swizzle K-major layout, ring of kTcStages slots);
//   * 8 A-producer warps (2 per TMEM lane quarter) load the reference desc and
//     mask words with plain loads, prefetched one stage ahead, and write the A
//     rows into TMEM (tcgen05.st, ring of kTcStages x 64 columns) -- they write
//     no shared memory, so no proxy fence drains their loads;
//   * one thread issues the MMAs (N <= 256 each, two per K-step for
//     ncols > 256) and commits the slot back to the producers;
//   * after the last stage, four epilogue warps read their 32 lanes'
//     accumulator columns (tcgen05.ld) and reduce the keys (cost << 16) | d
//     to the per-pixel minimum (ties -> smaller d, matcher.hpp:68-75), then
//     release the accumulator.
// CTAs are persistent (one per SM: the whole 512-column TMEM), walking the
// (tile, direction x d-block) items tile-major like k_cost_wta.
#pragma once
#ifndef BSM_TC_ABL
#define BSM_TC_ABL 0  // ablation bits for experiments (tools/microbench/tc_probe): 0 in the library
#endif

constexpr int kTcRows = 128;                      // MMA M: reference pixels per tile
constexpr int kTcKS = 8;                          // u32 words (MMA K-steps) per stage
constexpr int kTcStages = 2;                      // expanded ring (smem B + TMEM A)
constexpr int kTcMaxRaw = 8;                      // TMA ring of packed span words (as many as fit)
constexpr int kTcMaxDc = 256;                     // disparities per d-block
constexpr int kTcMaxCols = 384;                   // accumulator columns (128 + 256 -> 384)
constexpr int kTcAcol = kTcMaxCols;               // first TMEM column of the A ring
constexpr uint32_t kTcSmemLimit = 227 * 1024;     // dynamic shared memory per CTA
constexpr int kTcBWarps = 16;                     // B producers: warps 0-15
constexpr int kTcEpiWarps = 4;                    // epilogue: warps 16-19 (lane quarters 0-3)
constexpr int kTcMmaWarp = kTcBWarps + kTcEpiWarps;  // 20; the TMA loader is warp 21
constexpr int kTcAWarp0 = kTcMmaWarp + 2;         // A producers: warps 22-29
constexpr int kTcAHalves = 2;                     // A producer warps per lane quarter
constexpr int kTcAWarps = 4 * kTcAHalves;
constexpr int kTcThreads = (kTcAWarp0 + kTcAWarps) * 32;
constexpr int kTcBTasks = (kTcMaxCols * kTcKS + kTcBWarps * 32 - 1) / (kTcBWarps * 32);  // (row, word) per thread
static_assert(kTcAcol + kTcStages * kTcKS * 8 <= 512, "TMEM: accumulator + A ring");
static_assert(kTcKS % (2 * kTcAHalves) == 0, "A producers store 2 words per tcgen05.st");

__device__ __forceinline__ uint32_t tc_sign_bytes(uint32_t x) {
    // each byte -> 0xFF if its top bit is set, else 0x00 (prmt sign replicate)
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(x));
    return r;
}
// mbarrier wait with a suspend-time hint (ns): the hardware may park the
// thread until the phase completes instead of re-polling (measured: the same
// speed as the plain try_wait loop at 200 ns .. 20 us hints).
__device__ __forceinline__ void tc_wait(uint32_t bar_saddr, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TCW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra TCW_%=;\n"
        "}\n" ::"r"(bar_saddr),
        "r"(parity), "n"(20000)
        : "memory");
}
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity) { tc_wait(smem_addr(bar), parity); }
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

__device__ __forceinline__ void tc_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

// Shared memory carve-up (bytes), shared by the kernel and the host: the
// expanded B ring, the TMA ring of packed span words (as many stages as fit,
// at most kTcMaxRaw), the per-tile popcount bases and the barriers.
struct TcSmem {
    uint32_t sub, stage, raw, nraw, b_ring, raw_ring, base, bars, total;
    __host__ __device__ explicit TcSmem(int ncols) {
        sub = uint32_t(ncols) * 32u;                 // one K-step of B rows
        stage = sub * kTcKS;                         // expanded B stage
        raw = kTcKS * uint32_t(ncols) * 4u;          // packed span words of a stage
        b_ring = 0;
        raw_ring = b_ring + kTcStages * stage;
        const uint32_t fixed = 2 * kTcAHalves * kTcRows * 4 + (2 * kTcStages + 2 * kTcMaxRaw + 6) * 8 + 16;
        const uint32_t room = kTcSmemLimit > raw_ring + fixed ? kTcSmemLimit - raw_ring - fixed : 0;
        nraw = room / raw < uint32_t(kTcMaxRaw) ? room / raw : uint32_t(kTcMaxRaw);
        base = raw_ring + nraw * raw;
        bars = base + 2 * kTcAHalves * kTcRows * 4;
        total = bars + (2 * kTcStages + 2 * kTcMaxRaw + 6) * 8 + 16;
    }
};

template <bool MASKED>
__global__ void __launch_bounds__(kTcThreads, 1)
    k_cost_wta_tc(const __grid_constant__ CUtensorMap l_oth, const __grid_constant__ CUtensorMap r_oth,
                  const uint32_t* __restrict__ l_ref, const uint32_t* __restrict__ l_mask,
                  const uint32_t* __restrict__ r_ref, const uint32_t* __restrict__ r_mask, int W, int Wq, int npix,
                  int P, int NW, int D, int Dc, int ncols, int ndd, int ndir, int dir0, int items,
                  uint32_t* __restrict__ keys_l, uint32_t* __restrict__ keys_r) {
    extern __shared__ __align__(1024) uint8_t tsm[];
    const TcSmem L(ncols);
    uint8_t* sB = tsm + L.b_ring;                                        // [S][KS][ncols rows x 32 B]
    uint32_t* sraw = reinterpret_cast<uint32_t*>(tsm + L.raw_ring);      // [nraw][2 boxes][KS][ncols / 2]
    uint32_t* sbase = reinterpret_cast<uint32_t*>(tsm + L.base);         // [2 tiles][2 halves][128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(tsm + L.bars);
    uint64_t* full = bars;                               // [S] producers -> MMA (one arrival per warp)
    uint64_t* empty = full + kTcStages;                  // [S] MMA commit -> producers
    uint64_t* raw_full = empty + kTcStages;              // [nraw] TMA bytes -> B producers
    uint64_t* raw_empty = raw_full + kTcMaxRaw;          // [nraw] B producers (one arrival per warp) -> loader
    uint64_t* acc_full = raw_empty + kTcMaxRaw;          // MMA commit -> epilogue
    uint64_t* acc_empty = acc_full + 1;                  // epilogue (4 warps) -> MMA
    uint64_t* base_full = acc_full + 2;                  // [2] A producers -> epilogue
    uint64_t* base_empty = acc_full + 4;                 // [2] epilogue -> A producers
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 6);
    const uint32_t nraw = L.nraw;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(full + s, kTcBWarps + kTcAWarps);
            mbar_init(empty + s, 1);
        }
        for (uint32_t s = 0; s < nraw; ++s) {
            mbar_init(raw_full + s, 1);
            mbar_init(raw_empty + s, kTcBWarps);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, kTcEpiWarps);
        for (int i = 0; i < 2; ++i) {
            mbar_init(base_full + i, kTcAWarps);
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

    if (warp < kTcBWarps) {
        // ---------------- B producers ----------------
        // The ncols x KS (row, word) tasks of a stage are dealt round-robin over the
        // 512 threads (a warp's 32 tasks: one word, 32 consecutive rows); each
        // expands one packed word into the row's 32 int8 (-1 / 0) of that K-step.
        const int ntask = ncols * kTcKS;
        uint32_t tsrc[kTcBTasks], tdst[kTcBTasks];  // raw word offset, expanded-slot byte offset
#pragma unroll
        for (int k = 0; k < kTcBTasks; ++k) {
            const int i = min(tid + k * kTcBWarps * 32, ntask - 1);
            const int j = i / ncols, n = i - j * ncols;
            const int box = n < half ? 0 : 1;
            // span box `box` holds rows [box half, +half) as [KS][half]
            tsrc[k] = uint32_t(box * half * kTcKS + j * half + n - box * half);
            tdst[k] = uint32_t(j) * L.sub + uint32_t((n >> 3) * 256 + (n & 7) * 16);
        }
        uint32_t g = 0;  // global stage counter
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            for (int st = 0; st < nst; ++st, ++g) {
                const uint32_t r = g % nraw, s = g % kTcStages;
                tc_wait(raw_full + r, (g / nraw) & 1u);
                const uint32_t* raw = sraw + r * (L.raw / 4);
                uint32_t b[kTcBTasks];
#pragma unroll
                for (int k = 0; k < kTcBTasks; ++k)
                    if (tid + k * kTcBWarps * 32 < ntask) b[k] = raw[tsrc[k]];
                __syncwarp();
                if (lane == 0) mbar_arrive(raw_empty + r);
                tc_wait(empty + s, ((g / kTcStages) & 1u) ^ 1u);
                uint8_t* slot = sB + s * L.stage;
#pragma unroll
                for (int k = 0; k < kTcBTasks; ++k) {
                    if (!(BSM_TC_ABL & 8) && tid + k * kTcBWarps * 32 < ntask) {
                        uint32_t bv[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) bv[c] = tc_sign_bytes(b[k] << (7 - c));
                        *reinterpret_cast<uint4*>(slot + tdst[k]) = make_uint4(bv[0], bv[1], bv[2], bv[3]);
                        *reinterpret_cast<uint4*>(slot + tdst[k] + 128) = make_uint4(bv[4], bv[5], bv[6], bv[7]);
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B rows -> tensor-core reads
                __syncwarp();
                if (lane == 0) mbar_arrive(full + s);
            }
        }
    } else if (warp >= kTcAWarp0) {
        // ---------------- A producers ----------------
        // warp: TMEM lane quarter q = warp & 3 (its rows 32 q .. +31), words
        // [h KS/2, +KS/2) of each stage; packed words by plain loads, prefetched
        // one stage ahead (these warps write only TMEM: no proxy fence drains them).
        const int q = warp & 3, h = (warp - kTcAWarp0) >> 2;
        const int arow = q * 32 + lane;
        constexpr int WH = kTcKS / kTcAHalves;  // words per warp per stage
        const uint32_t a_taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(kTcAcol + 8 * WH * h);
        int t = 0;
        uint32_t g = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++t) {
            const TcItem w = tc_item(it, ndd, ndir, dir0, Dc, D);
            const size_t pix = size_t(min(w.p0 + arow, npix - 1));
            const uint32_t* pa = (w.dir ? r_ref : l_ref) + pix;
            const uint32_t* pm = (w.dir ? r_mask : l_mask) + pix;
            uint32_t na[WH], nm[WH];
            auto load = [&](int st) {
#pragma unroll
                for (int j = 0; j < WH; ++j) {
                    const int k = st * kTcKS + h * WH + j;
                    const size_t o = size_t(min(k, NW - 1)) * size_t(P);
                    const uint32_t km = k < NW ? 0xFFFFFFFFu : 0u;
                    na[j] = __ldg(pa + o) & km;
                    nm[j] = MASKED ? (__ldg(pm + o) & km) : km;
                }
            };
            load(0);
            uint32_t base = 0;
            for (int st = 0; st < nst; ++st, ++g) {
                uint32_t a[WH], m[WH];
#pragma unroll
                for (int j = 0; j < WH; ++j) {
                    a[j] = na[j];
                    m[j] = nm[j];
                }
                if (st + 1 < nst) load(st + 1);
                const uint32_t s = g % kTcStages;
                tc_wait(empty + s, ((g / kTcStages) & 1u) ^ 1u);
                tc_fence_after();
#pragma unroll
                for (int j0 = 0; j0 < WH; j0 += 2) {
                    // A: byte = m ? (a ? -1 : +1) : 0; column c of a word = bit c of each byte
                    uint32_t av[16];
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const uint32_t u = a[j0 + jj] & m[j0 + jj];
                        base += __popc(u);
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            uint32_t v;
                            asm("lop3.b32 %0, %1, %2, 0x01010101, 0xF8;"  // a | (b & c)
                                : "=r"(v)
                                : "r"(tc_sign_bytes(u << (7 - c))), "r"(m[j0 + jj] >> c));
                            av[8 * jj + c] = v;
                        }
                    }
                    __syncwarp();
                    tc_st16(a_taddr + s * (kTcKS * 8) + j0 * 8, av);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(full + s);
            }
            // popc(a & m) of this tile's pixels (this warp's words), for the epilogue
            const int par = t & 1;
            tc_wait(base_empty + par, (uint32_t(t >> 1) & 1u) ^ 1u);
            sbase[(par * kTcAHalves + h) * kTcRows + arow] = base;
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
            tc_wait(base_full + par, uint32_t(t >> 1) & 1u);
            uint32_t base = 0;
#pragma unroll
            for (int j = 0; j < kTcAHalves; ++j) base += sbase[(par * kTcAHalves + j) * kTcRows + r];
            __syncwarp();
            if (lane == 0) mbar_arrive(base_empty + par);
            tc_wait(acc_full, uint32_t(t) & 1u);
            tc_fence_after();
            uint32_t best = 0xFFFFFFFFu;
            const int cend = (BSM_TC_ABL & 32) ? 0 : q * 32 + 32 + w.dq;  // last column this warp uses, + 1
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
            tc_wait(acc_empty, (uint32_t(t) & 1u) ^ 1u);
            tc_fence_after();
            for (int st = 0; st < nst; ++st, ++g) {
                const uint32_t s = g % kTcStages;
                tc_wait(full + s, (g / kTcStages) & 1u);
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int j = 0; j < kTcKS && !(BSM_TC_ABL & 4); ++j) {
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
        // ---------------- TMA loader of the span words (lane 0 issues) ----------------
        uint32_t g = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            const TcItem w = tc_item(it, ndd, ndir, dir0, Dc, D);
            const int q0 = w.dir ? w.p0 + w.d0 : w.p0 - w.d0 - w.dq;  // span row 0 (a multiple of 4)
            // A span box wholly outside the field is not loaded (a box starting
            // further left than its width traps): its rows only meet out-of-image
            // cells, so stale words are harmless.
            const bool b0 = q0 + half > 0 && q0 < npix, b1 = q0 + 2 * half > 0 && q0 + half < npix;
            const uint32_t hb = uint32_t(half) * kTcKS * 4;
            for (int st = 0; st < nst; ++st, ++g) {
                const uint32_t r = g % nraw;
                tc_wait(raw_empty + r, ((g / nraw) & 1u) ^ 1u);
                if (lane == 0) {
                    uint32_t* db = sraw + r * (L.raw / 4);
                    // the tensor maps are addressed directly (a runtime-selected pointer
                    // to a __grid_constant__ parameter would be a local copy)
                    auto issue = [&](const CUtensorMap* mo) {
                        if (BSM_TC_ABL & 16) { mbar_arrive(raw_full + r); return; }
                        mbar_expect_tx(raw_full + r, (b0 ? hb : 0) + (b1 ? hb : 0));
                        if (b0) tma_load_2d(db, mo, q0, st * kTcKS, raw_full + r);
                        if (b1) tma_load_2d(db + half * kTcKS, mo, q0 + half, st * kTcKS, raw_full + r);
                    };
                    if (w.dir) issue(&r_oth);
                    else issue(&l_oth);
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
