// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" driver around the UNMODIFIED reference library headers in
// /root/reference/proj/include/bsm (compiled in place by oracle/Makefile; no
// reference source is copied into this repository).  The resulting
// oracle/_ref/libbsm_ref_*.so is the ground truth the C restatement
// (oracle/bsm_oracle.c) and the CUDA path are checked against, and it is the
// CPU arm timed by `bench.py --impl reference`.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline /
// --impl reference) load it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "bsm/config.hpp"
#include "bsm/descriptor.hpp"
#include "bsm/image.hpp"
#include "bsm/matcher.hpp"
#include "bsm/pattern.hpp"
#include "bsm/pipeline.hpp"
#include "bsm/refine.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const bsm::InvalidArgument*>(&e)) return 1;
    if (dynamic_cast<const bsm::DimensionMismatch*>(&e)) return 2;
    return 9;
}

bsm::SamplingPattern make_pattern(const int16_t* pairs, int n, int window) {
    bsm::SamplingPattern pat;
    pat.n = n;
    pat.window = window;
    pat.spread = 0.0;
    pat.seed = 0;
    pat.pairs.resize(size_t(n));
    for (int i = 0; i < n; ++i)
        pat.pairs[size_t(i)] = {pairs[4 * i], pairs[4 * i + 1], pairs[4 * i + 2], pairs[4 * i + 3]};
    return pat;
}

// A grayscale u8 view enters the library exactly as a gray PGM is loaded
// (image_io.hpp:257-259): r = g = b = v.
bsm::RgbImage rgb_from_gray(const uint8_t* img, int W, int H) {
    bsm::RgbImage out(W, H);
    for (size_t i = 0; i < size_t(W) * size_t(H); ++i) out.pixels[i] = {img[i], img[i], img[i]};
    return out;
}

bsm::RgbImage rgb_from_rgb(const uint8_t* rgb, int W, int H) {
    bsm::RgbImage out(W, H);
    for (size_t i = 0; i < size_t(W) * size_t(H); ++i)
        out.pixels[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
    return out;
}

bsm::DescriptorField field_from_words(const uint64_t* desc, const uint64_t* mask, int W, int H, int n) {
    bsm::DescriptorField f(W, H, n);
    const int words = f.words_per_string();
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const size_t o = (size_t(y) * W + x) * size_t(words);
            std::memcpy(f.descriptor(x, y).data(), desc + o, size_t(words) * 8);
            std::memcpy(f.mask(x, y).data(), mask + o, size_t(words) * 8);
        }
    return f;
}

void field_to_words(const bsm::DescriptorField& f, uint64_t* desc, uint64_t* mask) {
    const int words = f.words_per_string();
    for (int y = 0; y < f.height(); ++y)
        for (int x = 0; x < f.width(); ++x) {
            const size_t o = (size_t(y) * f.width() + x) * size_t(words);
            std::memcpy(desc + o, f.descriptor(x, y).data(), size_t(words) * 8);
            std::memcpy(mask + o, f.mask(x, y).data(), size_t(words) * 8);
        }
}

bsm::DisparityMap map_from(const float* d, const uint8_t* v, int W, int H) {
    bsm::DisparityMap m(W, H);
    std::memcpy(m.disparity.data(), d, size_t(W) * H * 4);
    if (v) std::memcpy(m.valid.data(), v, size_t(W) * H);
    return m;
}

void map_to(const bsm::DisparityMap& m, float* d, uint8_t* v) {
    if (d) std::memcpy(d, m.disparity.data(), m.disparity.size() * 4);
    if (v) std::memcpy(v, m.valid.data(), m.valid.size());
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_generate_pattern(int n, int window, double spread, uint64_t seed, int16_t* out) {
    try {
        const bsm::SamplingPattern p = bsm::generate_pattern(n, window, spread, seed);
        for (int i = 0; i < n; ++i) {
            out[4 * i] = p.pairs[size_t(i)].px;
            out[4 * i + 1] = p.pairs[size_t(i)].py;
            out[4 * i + 2] = p.pairs[size_t(i)].qx;
            out[4 * i + 3] = p.pairs[size_t(i)].qy;
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// gray[v], lab[3v..3v+2] for the gray pixel (v,v,v).
void ref_gray_lab_lut(float* gray256, float* lab768) {
    bsm::RgbImage img(256, 1);
    for (int v = 0; v < 256; ++v) img.pixels[size_t(v)] = {uint8_t(v), uint8_t(v), uint8_t(v)};
    const bsm::GrayImage g = bsm::to_gray(img);
    const bsm::LabImage l = bsm::to_lab(img);
    for (int v = 0; v < 256; ++v) {
        gray256[v] = g.values[size_t(v)];
        lab768[3 * v] = l.values[size_t(v)].l;
        lab768[3 * v + 1] = l.values[size_t(v)].a;
        lab768[3 * v + 2] = l.values[size_t(v)].b;
    }
}

// Per-pixel colour conversion of an interleaved RGB image.
void ref_to_gray_lab(const uint8_t* rgb, int W, int H, float* gray, float* lab) {
    const bsm::RgbImage img = rgb_from_rgb(rgb, W, H);
    const bsm::GrayImage g = bsm::to_gray(img);
    const bsm::LabImage l = bsm::to_lab(img);
    std::memcpy(gray, g.values.data(), g.values.size() * 4);
    std::memcpy(lab, l.values.data(), l.values.size() * 12);
}

// compute_field (descriptor.hpp:200) on float gray/Lab planes.
int ref_compute_field(const float* gray, const float* lab, int W, int H, const int16_t* pairs,
                      int n, int window, int threads, uint64_t* desc, uint64_t* mask) {
    try {
        bsm::GrayImage g(W, H);
        std::memcpy(g.values.data(), gray, size_t(W) * H * 4);
        bsm::LabImage l(W, H);
        std::memcpy(l.values.data(), lab, size_t(W) * H * 12);
        const bsm::DescriptorField f =
            bsm::compute_field(g, l, make_pattern(pairs, n, window), threads);
        field_to_words(f, desc, mask);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// compute_field of a grayscale u8 view, colour conversion included (pipeline.hpp:145-151).
int ref_compute_field_u8(const uint8_t* img, int W, int H, const int16_t* pairs, int n, int window,
                         int threads, uint64_t* desc, uint64_t* mask) {
    try {
        const bsm::RgbImage rgb = rgb_from_gray(img, W, H);
        const bsm::DescriptorField f = bsm::compute_field(bsm::to_gray(rgb), bsm::to_lab(rgb),
                                                          make_pattern(pairs, n, window), threads);
        field_to_words(f, desc, mask);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

float ref_quarter_threshold(const float* w, int n) {
    return bsm::quarter_threshold(std::span<const float>(w, size_t(n)));
}

int ref_masked_hamming_words(const uint64_t* a, const uint64_t* b, const uint64_t* m, int nwords) {
    return bsm::masked_hamming_words(a, b, m, size_t(nwords));
}

// cost (matcher.hpp:45) of one (x, y, d).
int ref_cost(const uint64_t* dref, const uint64_t* mref, const uint64_t* doth, const uint64_t* moth,
             int W, int H, int n, int x, int y, int d, int d_max, int right_ref, int* out) {
    try {
        const bsm::DescriptorField fr = field_from_words(dref, mref, W, H, n);
        const bsm::DescriptorField fo = field_from_words(doth, moth, W, H, n);
        *out = bsm::cost(fr, fo, x, y, d,
                         bsm::MatchParams{d_max, right_ref ? bsm::RefView::right : bsm::RefView::left});
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// wta (matcher.hpp:80).
int ref_wta(const uint64_t* dref, const uint64_t* mref, const uint64_t* doth, int W, int H, int n,
            int d_max, int right_ref, int use_mask, int threads, float* out) {
    try {
        const bsm::DescriptorField fr = field_from_words(dref, mref, W, H, n);
        std::vector<uint64_t> zeros(size_t(W) * H * size_t(bsm::words_for_bits(n)), 0);
        const bsm::DescriptorField fo = field_from_words(doth, zeros.data(), W, H, n);
        const bsm::DisparityMap m =
            bsm::wta(fr, fo, bsm::MatchParams{d_max, right_ref ? bsm::RefView::right : bsm::RefView::left},
                     threads, use_mask != 0);
        map_to(m, out, nullptr);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// lr_check (refine.hpp:39).
int ref_lr_check(const float* dl, const uint8_t* vl, const float* dr, const uint8_t* vr, int W, int H,
                 double tol, float* od, uint8_t* ov) {
    try {
        map_to(bsm::lr_check(map_from(dl, vl, W, H), map_from(dr, vr, W, H), tol), od, ov);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// vote_refine (refine.hpp:62) with a float Lab plane.
int ref_vote_refine(const float* d, const uint8_t* v, const float* lab, int W, int H, double lc,
                    double le, double tol, int radius, int threads, float* od, uint8_t* ov) {
    try {
        bsm::LabImage l(W, H);
        std::memcpy(l.values.data(), lab, size_t(W) * H * 12);
        map_to(bsm::vote_refine(map_from(d, v, W, H), l, bsm::RefineParams{lc, le, tol, radius}, threads),
               od, ov);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

double ref_vote_weight(const float* lab_x, const float* lab_p, int dx, int dy, double lc, double le) {
    return bsm::vote_weight(bsm::Lab{lab_x[0], lab_x[1], lab_x[2]}, bsm::Lab{lab_p[0], lab_p[1], lab_p[2]},
                            dx, dy, lc, le);
}

// run_pipeline (pipeline.hpp:25) on a grayscale (r=g=b) or interleaved-RGB pair.
// Any output pointer may be null.  *seconds = wall time of run_pipeline alone
// (time_pipeline semantics, eval.hpp:144-159: pattern generation excluded).
int ref_pipeline(const uint8_t* left, const uint8_t* right, int channels, int W, int H,
                 const int16_t* pairs, int n, int window, int d_max, double lc, double le, double tol,
                 int radius, int threads, int want_unmasked, float* refined_d, uint8_t* refined_v,
                 float* left_d, float* right_d, float* checked_d, uint8_t* checked_v, float* unmasked_d,
                 double* seconds) {
    try {
        const bsm::RgbImage L = channels == 3 ? rgb_from_rgb(left, W, H) : rgb_from_gray(left, W, H);
        const bsm::RgbImage R = channels == 3 ? rgb_from_rgb(right, W, H) : rgb_from_gray(right, W, H);
        bsm::BsmConfig cfg;
        cfg.n = n;
        cfg.window = window;
        cfg.d_max = d_max;
        cfg.lambda_c = lc;
        cfg.lambda_e = le;
        cfg.lr_tolerance = tol;
        cfg.vote_radius = radius;
        cfg.threads = threads;
        const bsm::SamplingPattern pat = make_pattern(pairs, n, window);
        const auto t0 = std::chrono::steady_clock::now();
        const bsm::PipelineResult res = bsm::run_pipeline(L, R, pat, cfg, want_unmasked != 0);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        map_to(res.refined, refined_d, refined_v);
        map_to(res.left_wta, left_d, nullptr);
        map_to(res.right_wta, right_d, nullptr);
        map_to(res.checked, checked_d, checked_v);
        if (want_unmasked && unmasked_d) map_to(*res.unmasked, unmasked_d, nullptr);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

}  // extern "C"

// The BASELINE synthetic pair generator (paper_1402_2020_b200/csrc/synth.cpp,
// input generation only) compiled into this test library as ref_synth_pair, so
// that the reference arm of bench.py builds its inputs without loading any
// product library.
#define bsm_synth_pair ref_synth_pair
#include "../paper_1402_2020_b200/csrc/synth.cpp"
#undef bsm_synth_pair
