// C++ shim test driver: the reference's own test idioms (proj/tests/*.cpp)
// against include/bsm/ (the drop-in C++ API over libbsm_cuda.so).
//   shim_test host                    -- host-side checks, no device needed
//   shim_test gpu L.raw R.raw W H D out.bin
//                                     -- run_pipeline on a grayscale (W*H bytes) or RGB
//                                        (3*W*H bytes) pair, maps to out.bin
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <vector>

#include "bsm/bsm.hpp"

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static int host_checks() {
    using namespace bsm;
    // test_bitstring / test_matcher known answers
    const BitString a = BitString::from_bits("1010"), b = BitString::from_bits("0110");
    CHECK(masked_hamming(a, b, BitString::from_bits("1111")) == 2);
    CHECK(masked_hamming(a, b, BitString::from_bits("1000")) == 1);
    CHECK(masked_hamming(a, b, BitString::from_bits("0000")) == 0);
    CHECK(throws<DimensionMismatch>([&] { masked_hamming(a, BitString(5), a); }));
    CHECK(throws<InvalidArgument>([] { BitString::from_bits("10x"); }));
    // wta_select: ties to the smaller d (test_matcher.cpp:105-110)
    CHECK(wta_select(std::vector<int>{5, 3, 7}) == 1);
    CHECK(wta_select(std::vector<int>{3, 3, 7}) == 0);
    // quarter_threshold (test_descriptor.cpp:64-72)
    CHECK(quarter_threshold(std::vector<float>{1, 2, 3, 4, 5, 6, 7, 8}) == 2.0f);
    CHECK(quarter_threshold(std::vector<float>(8, 5.0f)) == 5.0f);
    CHECK(quarter_threshold(std::vector<float>{9, 3}) == 3.0f);
    // cost sentinel n + 1 (test_matcher.cpp:64-71)
    DescriptorField f(6, 1, 64);
    CHECK(cost(f, f, 3, 0, 5, MatchParams{6, RefView::left}) == 65);
    CHECK(cost(f, f, 5, 0, 4, MatchParams{6, RefView::right}) == 65);
    CHECK(throws<InvalidArgument>([&] { cost(f, f, 3, 0, 6, MatchParams{6, RefView::left}); }));
    // pattern generation: bit-identical generator (checked against the reference in pytest)
    const SamplingPattern p = generate_pattern(128, 8, 2.0, 5);
    CHECK(p.n == 128 && int(p.pairs.size()) == 128);
    for (const PairOffsets& q : p.pairs) CHECK(!(q.px == q.qx && q.py == q.qy));
    CHECK(throws<InvalidArgument>([] { generate_pattern(0, 8, 2.0, 5); }));
    // config validation
    BsmConfig cfg;
    CHECK(throws<InvalidArgument>([&] { cfg.validate(); }));
    cfg.d_max = 4;
    cfg.validate();
    // colour conversion: red (test_image.cpp:49-54)
    RgbImage red(1, 1);
    red.at(0, 0) = {255, 0, 0};
    const Lab l = to_lab(red).at(0, 0);
    CHECK(std::abs(l.l - 53.2408f) < 0.01f && std::abs(l.a - 80.0925f) < 0.01f && std::abs(l.b - 67.2032f) < 0.01f);
    // dimension checks happen before any device work
    CHECK(throws<DimensionMismatch>([] { run_pipeline(RgbImage(4, 4), RgbImage(5, 4), BsmConfig{}); }));
    CHECK(throws<DimensionMismatch>([] { lr_check(DisparityMap(4, 4), DisparityMap(5, 4), 1.0); }));
    // print the default pattern checksum for the pytest side
    const SamplingPattern d = generate_pattern(BsmConfig{});
    uint64_t h = 1469598103934665603ull;
    for (const PairOffsets& q : d.pairs)
        for (int16_t v : {q.px, q.py, q.qx, q.qy}) h = (h ^ uint16_t(v)) * 1099511628211ull;
    std::printf("pattern_fnv %llu\n", (unsigned long long)h);
    return failures;
}

static int gpu_run(const char* lpath, const char* rpath, int W, int H, int D, const char* out) {
    using namespace bsm;
    // a W*H file is a grayscale view, a 3*W*H file interleaved RGB
    std::ifstream lf(lpath, std::ios::binary | std::ios::ate), rf(rpath, std::ios::binary | std::ios::ate);
    const size_t bytes = size_t(lf.tellg());
    const int ch = bytes == size_t(3) * W * H ? 3 : 1;
    std::vector<uint8_t> L(bytes), R(bytes);
    lf.seekg(0);
    rf.seekg(0);
    lf.read(reinterpret_cast<char*>(L.data()), std::streamsize(bytes));
    rf.read(reinterpret_cast<char*>(R.data()), std::streamsize(bytes));
    RgbImage left(W, H), right(W, H);
    for (size_t i = 0; i < size_t(W) * H; ++i) {
        const size_t k = ch * i;
        left.pixels[i] = {L[k], L[k + (ch - 1) / 2], L[k + ch - 1]};
        right.pixels[i] = {R[k], R[k + (ch - 1) / 2], R[k + ch - 1]};
    }
    BsmConfig cfg;
    cfg.d_max = D;
    const PipelineResult res = run_pipeline(left, right, cfg, /*want_unmasked=*/true);
    // per-stage API, chained like proj/tests/acceptance.cpp:274-279
    const SamplingPattern pat = generate_pattern(cfg);
    const DescriptorField fl = compute_field(to_gray(left), to_lab(left), pat);
    const DescriptorField fr = compute_field(to_gray(right), to_lab(right), pat);
    const DisparityMap lw = wta(fl, fr, MatchParams{D, RefView::left});
    const DisparityMap rw = wta(fr, fl, MatchParams{D, RefView::right});
    const DisparityMap chk = lr_check(lw, rw, cfg.lr_tolerance);
    const DisparityMap ref = vote_refine(chk, to_lab(left), RefineParams{});
    CHECK(lw == res.left_wta);
    CHECK(rw == res.right_wta);
    CHECK(chk == res.checked);
    CHECK(ref == res.refined);
    // single-pixel API (descriptor.hpp:174-196, O(n) window tiles) == the field,
    // at corners, borders and the interior
    const GrayImage gl = to_gray(left);
    const LabImage ll = to_lab(left);
    const int px[][2] = {{0, 0}, {W - 1, 0}, {0, H - 1}, {W - 1, H - 1}, {W / 2, H / 2}, {1, H / 2}, {W / 2, 1}, {3, 2}};
    for (const auto& q : px) {
        CHECK(compute_descriptor(gl, pat, q[0], q[1]) == fl.descriptor_at(q[0], q[1]));
        CHECK(compute_mask(ll, pat, q[0], q[1]) == fl.mask_at(q[0], q[1]));
    }
    std::ofstream o(out, std::ios::binary);
    for (const DisparityMap* m : {&res.refined, &res.left_wta, &res.right_wta, &res.checked, &*res.unmasked}) {
        o.write(reinterpret_cast<const char*>(m->disparity.data()), std::streamsize(m->disparity.size() * 4));
        o.write(reinterpret_cast<const char*>(m->valid.data()), std::streamsize(m->valid.size()));
    }
    return failures;
}

int main(int argc, char** argv) {
    try {
        if (argc >= 2 && std::strcmp(argv[1], "host") == 0) return host_checks();
        if (argc >= 8 && std::strcmp(argv[1], "gpu") == 0)
            return gpu_run(argv[2], argv[3], std::atoi(argv[4]), std::atoi(argv[5]), std::atoi(argv[6]), argv[7]);
        if (argc >= 2 && std::strcmp(argv[1], "nodevice") == 0) {
            // with no device, the first device call must throw (no CPU fallback)
            bool threw = false;
            try {
                bsm::BsmConfig cfg;
                cfg.d_max = 4;
                bsm::run_pipeline(bsm::RgbImage(8, 8), bsm::RgbImage(8, 8), cfg);
            } catch (const bsm::Error& e) {
                threw = std::strstr(e.what(), "no CPU fallback") != nullptr;
                std::printf("%s\n", e.what());
            }
            return threw ? 0 : 1;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    std::fprintf(stderr, "usage: shim_test host | nodevice | gpu L.raw R.raw W H D out.bin\n");
    return 2;
}
