// Probe for the tensor-core cost kernel (kern_cost_tc.cuh): random word planes,
// both directions, keys checked against a CPU popcount on every pixel (small
// cases) or on a pixel sample (large cases), and the kernel timed.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I../../paper_1402_2020_b200/csrc -o tc_probe tc_probe.cu -lcuda
//   ./tc_probe W H NW D [masked=1] [reps=5]
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

namespace {
constexpr int kCostTile = 128, kCostDisp = 64, kCostK = 16, kCostStages = 3;
#include "kern_cost.cuh"
#include "kern_cost_tc.cuh"
}  // namespace

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e = (x);                                                                   \
        if (e != cudaSuccess) {                                                                \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            std::exit(1);                                                                      \
        }                                                                                      \
    } while (0)

static uint32_t cpu_key(const std::vector<uint32_t>& ref, const std::vector<uint32_t>& msk,
                        const std::vector<uint32_t>& oth, bool masked, int W, int Wq, size_t P, int NW, int D, int y,
                        int x, int dir) {
    uint32_t best = 0xFFFFFFFFu;
    const size_t p = size_t(y) * Wq + x;
    for (int d = 0; d < D; ++d) {
        const int xo = dir ? x + d : x - d;
        if (xo < 0 || xo >= W) continue;
        const size_t po = size_t(y) * Wq + xo;
        uint32_t c = 0;
        for (int k = 0; k < NW; ++k) {
            uint32_t v = ref[k * P + p] ^ oth[k * P + po];
            if (masked) v &= msk[k * P + p];
            c += __builtin_popcount(v);
        }
        best = std::min(best, (c << 16) | uint32_t(d));
    }
    return best;
}

int main(int argc, char** argv) {
    const int W = argc > 1 ? std::atoi(argv[1]) : 300;
    const int H = argc > 2 ? std::atoi(argv[2]) : 3;
    const int NW = argc > 3 ? std::atoi(argv[3]) : 8;
    const int D = argc > 4 ? std::atoi(argv[4]) : 192;
    const bool masked = argc > 5 ? std::atoi(argv[5]) != 0 : true;
    const int reps = argc > 6 ? std::atoi(argv[6]) : 5;
    const int dirsel = argc > 7 ? std::atoi(argv[7]) : 2;  // 0 left only, 1 right only, 2 both
    const bool at = argc > 8 ? std::atoi(argv[8]) != 0 : true;  // A operand in TMEM
    const int stages = argc > 9 ? std::atoi(argv[9]) : 2;         // operand ring depth (3: A in TMEM only)
    const int Wq = (W + 3) / 4 * 4;
    const int npix = H * Wq;
    const size_t P = (size_t(npix) + 31) / 32 * 32;
    std::mt19937_64 rng(12345);
    auto plane = [&](uint64_t density_bits) {
        std::vector<uint32_t> v(size_t(NW) * P);
        for (auto& w : v) {
            uint32_t r = uint32_t(rng());
            if (density_bits) r &= uint32_t(rng()) | uint32_t(rng());  // ~75% ones for masks
            w = r;
        }
        return v;
    };
    auto dl = plane(0), dr = plane(0), ml = plane(1), mr = plane(1);
    // correlate the views a little so the minima are meaningful: right = left shifted by 7
    for (int k = 0; k < NW; ++k)
        for (int y = 0; y < H; ++y)
            for (int x = 0; x + 7 < W; ++x)
                if ((rng() & 3) != 0) dr[k * P + size_t(y) * Wq + x] = dl[k * P + size_t(y) * Wq + x + 7];
    uint32_t *gdl, *gdr, *gml, *gmr, *kl, *kr;
    const size_t bytes = size_t(NW) * P * 4;
    CK(cudaMalloc(&gdl, bytes));
    CK(cudaMalloc(&gdr, bytes));
    CK(cudaMalloc(&gml, bytes));
    CK(cudaMalloc(&gmr, bytes));
    CK(cudaMalloc(&kl, size_t(W) * H * 4));
    CK(cudaMalloc(&kr, size_t(W) * H * 4));
    CK(cudaMemcpy(gdl, dl.data(), bytes, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(gdr, dr.data(), bytes, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(gml, ml.data(), bytes, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(gmr, mr.data(), bytes, cudaMemcpyHostToDevice));

    const int ndd = (D + kTcMaxDc - 1) / kTcMaxDc;
    const int Dc = ndd == 1 ? D : ((D + ndd - 1) / ndd + 3) / 4 * 4;  // d-blocks start on multiples of 4
    const int ncols = (128 + ((Dc + 2) & ~3) + 31) / 32 * 32;
    const int tiles = (npix + kTcRows - 1) / kTcRows;
    const int ndir = dirsel == 2 ? 2 : 1, dir0 = dirsel == 1 ? 1 : 0;
    const int items = tiles * ndd * ndir;
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const size_t sm = TcSmem(ncols, masked, at, stages).total;
    auto kern = stages == 3 ? (masked ? k_cost_wta_tc<true, true, 3> : k_cost_wta_tc<false, true, 3>)
                : masked ? (at ? k_cost_wta_tc<true, true> : k_cost_wta_tc<true, false>)
                         : (at ? k_cost_wta_tc<false, true> : k_cost_wta_tc<false, false>);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    const int grid = std::min(items, nsm);
    auto tmap = [&](const uint32_t* field, int box_x) {
        CUtensorMap m;
        const cuuint64_t dims[2] = {cuuint64_t(P), cuuint64_t(NW)};
        const cuuint64_t strides[1] = {cuuint64_t(P) * 4};
        const cuuint32_t box[2] = {cuuint32_t(box_x), cuuint32_t(kTcKS)};
        const cuuint32_t estr[2] = {1, 1};
        CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(field), dims,
                                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { std::printf("tensor map failed %d\n", int(r)); std::exit(1); }
        return m;
    };
    const CUtensorMap m_dl = tmap(gdl, kTcRows), m_ml = tmap(gml, kTcRows), m_dr_o = tmap(gdr, ncols / 2);
    const CUtensorMap m_dr = tmap(gdr, kTcRows), m_mr = tmap(gmr, kTcRows), m_dl_o = tmap(gdl, ncols / 2);
    auto run = [&]() {
        if (ndd > 1) {
            CK(cudaMemset(kl, 0xFF, size_t(W) * H * 4));
            CK(cudaMemset(kr, 0xFF, size_t(W) * H * 4));
        }
        kern<<<grid, kTcThreads, sm>>>(m_dl, m_ml, m_dr_o, m_dr, m_mr, m_dl_o, W, Wq, npix, NW, D, Dc, ncols, ndd, ndir, dir0,
                                       items, kl, kr);
    };
    run();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> hl(size_t(W) * H), hr(size_t(W) * H);
    CK(cudaMemcpy(hl.data(), kl, hl.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), kr, hr.size() * 4, cudaMemcpyDeviceToHost));
    // check
    const long long total = (long long)W * H;
    const bool full = total * D * NW <= 400000000LL;
    std::vector<std::pair<int, int>> pts;
    if (full) {
        for (int y = 0; y < H; ++y)
            for (int x = 0; x < W; ++x) pts.push_back({y, x});
    } else {
        for (int i = 0; i < 3000; ++i) pts.push_back({int(rng() % H), int(rng() % W)});
        for (int y : {0, H - 1})
            for (int x : {0, 1, 2, W / 2, W - 3, W - 2, W - 1}) pts.push_back({y, x});
    }
    long long bad = 0;
    for (auto [y, x] : pts)
        for (int dir = 0; dir < 2; ++dir) {
            if (dirsel != 2 && dir != dirsel) continue;
            const uint32_t want = dir ? cpu_key(dr, mr, dl, masked, W, Wq, P, NW, D, y, x, 1)
                                      : cpu_key(dl, ml, dr, masked, W, Wq, P, NW, D, y, x, 0);
            const uint32_t got = (dir ? hr : hl)[size_t(y) * W + x];
            if (got != want) {
                if (bad < 10)
                    std::printf("MISMATCH dir %d (y %d, x %d): got cost %u d %u, want cost %u d %u\n", dir, y, x,
                                got >> 16, got & 0xFFFF, want >> 16, want & 0xFFFF);
                ++bad;
            }
        }
    std::printf("check: %s, %zu pixels x 2 directions, %lld mismatches\n", full ? "all" : "sample", pts.size(), bad);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0));
        run();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    // in-bounds evaluations (both directions)
    double evals = 0;
    for (int x = 0; x < W; ++x) evals += 2.0 * std::min(D, x + 1);
    evals *= H;
    std::printf("W %d H %d NW %d D %d masked %d: ncols %d ndd %d items %d grid %d smem %zu nraw %u: %.3f ms both directions, "
                "%.1f G word-ops/s, %.0f Mdisp-evals/s (cost only, x2 dirs)\n",
                W, H, NW, D, int(masked), ncols, ndd, items, grid, sm, TcSmem(ncols, masked, at, stages).nraw, best, evals * NW / best / 1e6,
                evals / 2 / best / 1e3);
    return bad ? 2 : 0;
}
