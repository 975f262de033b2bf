// bsm_io_capi.cpp -- C ABI (include/bsm_io.h) of the host-side file and
// evaluation layer either side of the matching path: this repository's C++
// drop-in headers (include/bsm/image_io.hpp, eval.hpp, config.hpp,
// pattern.hpp) are the single implementation; the Python modules io.py and
// evaluation.py bind this library instead of re-implementing the formats.
// The entry points mirror oracle/ref_io_driver.cpp (prefix refio_) one for
// one, so the tests run the reference's own file/eval code and this layer side
// by side.  Status codes: 0 ok, 1 InvalidArgument, 2 DimensionMismatch,
// 9 other, 10 IoError, 11 FormatError, 12 EmptyRegion.
#include "../../include/bsm_io.h"

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "bsm/bsm.hpp"

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const bsm::IoError*>(&e)) return 10;
    if (dynamic_cast<const bsm::FormatError*>(&e)) return 11;
    if (dynamic_cast<const bsm::InvalidArgument*>(&e)) return 1;
    if (dynamic_cast<const bsm::DimensionMismatch*>(&e)) return 2;
    if (dynamic_cast<const bsm::EmptyRegion*>(&e)) return 12;
    return 9;
}

bsm::DisparityMap map_from(const float* d, const uint8_t* v, int W, int H) {
    bsm::DisparityMap m(W, H);
    std::memcpy(m.disparity.data(), d, size_t(W) * H * 4);
    std::memcpy(m.valid.data(), v, size_t(W) * H);
    return m;
}
}  // namespace

extern "C" {

const char* bsmio_last_error() { return g_err.c_str(); }

// The last decoded image / disparity map of this thread, so the two-call
// protocol (dimensions first, then pixels into a caller buffer) decodes once.
thread_local std::string g_img_path, g_gt_path;
thread_local double g_gt_scale = 0;
thread_local bsm::RgbImage g_img;
thread_local bsm::DisparityMap g_gt;

// load_image (image_io.hpp:240-263): dims always; pixels when rgb != nullptr.
int bsmio_load_image(const char* path, int* w, int* h, uint8_t* rgb) {
    try {
        if (!(rgb && g_img_path == path)) {
            g_img_path.clear();
            g_img = bsm::load_image(path);
            g_img_path = path;
        }
        *w = g_img.width;
        *h = g_img.height;
        if (rgb) {
            std::memcpy(rgb, g_img.pixels.data(), g_img.pixels.size() * 3);
            g_img_path.clear();
            g_img = bsm::RgbImage();
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// load_gt_disparity (image_io.hpp:268-314).
int bsmio_load_gt(const char* path, double scale, int* w, int* h, float* d, uint8_t* v) {
    try {
        if (!((d || v) && g_gt_path == path && g_gt_scale == scale)) {
            g_gt_path.clear();
            g_gt = bsm::load_gt_disparity(path, scale);
            g_gt_path = path;
            g_gt_scale = scale;
        }
        *w = g_gt.width;
        *h = g_gt.height;
        if (d) std::memcpy(d, g_gt.disparity.data(), g_gt.disparity.size() * 4);
        if (v) std::memcpy(v, g_gt.valid.data(), g_gt.valid.size());
        if (d || v) {
            g_gt_path.clear();
            g_gt = bsm::DisparityMap();
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// save_disparity (:317-337) or save_disparity_pfm (:340-355).
int bsmio_save_disparity(const char* path, const float* d, const uint8_t* v, int W, int H, double scale, int pfm) {
    try {
        const bsm::DisparityMap m = map_from(d, v, W, H);
        if (pfm) bsm::save_disparity_pfm(m, path);
        else bsm::save_disparity(m, path, scale);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// save_gray_pgm (:358-371) and save_ppm (:373-382).
int bsmio_save_gray_pgm(const char* path, const float* g, int W, int H) {
    try {
        bsm::GrayImage img(W, H);
        std::memcpy(img.values.data(), g, size_t(W) * H * 4);
        bsm::save_gray_pgm(img, path);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int bsmio_save_ppm(const char* path, const uint8_t* rgb, int W, int H) {
    try {
        bsm::RgbImage img(W, H);
        for (size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = {rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]};
        bsm::save_ppm(img, path);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// save_config / load_config (config.hpp:81-110); ints: n S seed d_max radius threads, doubles: spread lc le tol gt_scale.
int bsmio_save_config(const char* path, const int64_t* iv, const double* dv, const char* generator) {
    try {
        bsm::BsmConfig c;
        c.n = int(iv[0]);
        c.window = int(iv[1]);
        c.seed = uint64_t(iv[2]);
        c.d_max = int(iv[3]);
        c.vote_radius = int(iv[4]);
        c.threads = int(iv[5]);
        c.spread = dv[0];
        c.lambda_c = dv[1];
        c.lambda_e = dv[2];
        c.lr_tolerance = dv[3];
        c.gt_scale = dv[4];
        c.generator = generator;
        bsm::save_config(c, path);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int bsmio_load_config(const char* path, int64_t* iv, double* dv, char* generator, int gen_cap) {
    try {
        const bsm::BsmConfig c = bsm::load_config(path);
        iv[0] = c.n;
        iv[1] = c.window;
        iv[2] = int64_t(c.seed);
        iv[3] = c.d_max;
        iv[4] = c.vote_radius;
        iv[5] = c.threads;
        dv[0] = c.spread;
        dv[1] = c.lambda_c;
        dv[2] = c.lambda_e;
        dv[3] = c.lr_tolerance;
        dv[4] = c.gt_scale;
        std::strncpy(generator, c.generator.c_str(), size_t(gen_cap) - 1);
        generator[gen_cap - 1] = 0;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// save_pattern / load_pattern (pattern.hpp:104-160).
int bsmio_save_pattern(const char* path, const int16_t* pairs, int n, int window, double spread, uint64_t seed) {
    try {
        bsm::SamplingPattern p;
        p.n = n;
        p.window = window;
        p.spread = spread;
        p.seed = seed;
        p.pairs.resize(size_t(n));
        for (int i = 0; i < n; ++i)
            p.pairs[size_t(i)] = {pairs[4 * i], pairs[4 * i + 1], pairs[4 * i + 2], pairs[4 * i + 3]};
        bsm::save_pattern(p, path);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int bsmio_load_pattern(const char* path, int* n, int* window, double* spread, uint64_t* seed, int16_t* pairs,
                       int cap) {
    try {
        const bsm::SamplingPattern p = bsm::load_pattern(path);
        *n = p.n;
        *window = p.window;
        *spread = p.spread;
        *seed = p.seed;
        if (pairs)
            for (int i = 0; i < p.n && i < cap; ++i) {
                pairs[4 * i] = p.pairs[size_t(i)].px;
                pairs[4 * i + 1] = p.pairs[size_t(i)].py;
                pairs[4 * i + 2] = p.pairs[size_t(i)].qx;
                pairs[4 * i + 3] = p.pairs[size_t(i)].qy;
            }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// bad_pixel_rate (eval.hpp:31-59); region may be null.
int bsmio_bad_pixel_rate(const float* d, const uint8_t* v, const float* gd, const uint8_t* gv, const float* region,
                         int W, int H, double threshold, double* rate, long* counted, long* bad) {
    try {
        const bsm::DisparityMap r = map_from(d, v, W, H), g = map_from(gd, gv, W, H);
        bsm::GrayImage reg;
        if (region) {
            reg = bsm::GrayImage(W, H);
            std::memcpy(reg.values.data(), region, size_t(W) * H * 4);
        }
        const bsm::ErrorReport rep = bsm::bad_pixel_rate(r, g, region ? &reg : nullptr, threshold);
        *rate = rep.bad_pixel_rate;
        *counted = rep.counted;
        *bad = rep.bad;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int bsmio_linear_fit_r2(const double* xs, const double* ys, int n, double* out) {
    try {
        *out = bsm::linear_fit_r2(std::vector<double>(xs, xs + n), std::vector<double>(ys, ys + n));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int bsmio_write_sweep_csv(const char* path, const int* n, const double* err, const double* secs, int count) {
    try {
        std::vector<bsm::SweepPoint> pts(static_cast<size_t>(count));
        for (int i = 0; i < count; ++i) pts[size_t(i)] = {n[i], err[i], secs[i]};
        bsm::write_sweep_csv(path, pts);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int bsmio_write_radiometric_csv(const char* path, const double* rate9, double* diag, double* off) {
    try {
        bsm::RadiometricMatrix m;
        for (int i = 0; i < 9; ++i) m.rate[size_t(i / 3)][size_t(i % 3)] = rate9[i];
        if (path) bsm::write_radiometric_csv(path, m);
        *diag = m.diagonal_mean();
        *off = m.off_diagonal_mean();
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

}  // extern "C"
