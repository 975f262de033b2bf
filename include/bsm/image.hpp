// bsm/image.hpp -- image value types and colour conversion (reference
// image.hpp:12-150).  Colour conversion stays on the host: it is
// floating-point and FMA-contraction sensitive, so it runs in the library's
// host code (compiled like the reference) through bsm_to_gray_lab; the GPU
// path consumes grayscale views through bit-exact 256-entry tables.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <optional>
#include <utility>
#include <vector>

#include "../bsm_cuda.h"
#include "bsm/detail_cabi.hpp"
#include "bsm/errors.hpp"

namespace bsm {

struct Rgb8 {
    uint8_t r = 0, g = 0, b = 0;
    friend bool operator==(const Rgb8&, const Rgb8&) = default;
};

struct RgbImage {
    int width = 0, height = 0;
    std::vector<Rgb8> pixels;
    RgbImage() = default;
    RgbImage(int w, int h) : width(w), height(h), pixels(std::size_t(w) * std::size_t(h)) {
        if (w < 1 || h < 1) throw InvalidArgument("RgbImage: dimensions must be >= 1");
    }
    Rgb8& at(int x, int y) { return pixels[std::size_t(y) * width + x]; }
    const Rgb8& at(int x, int y) const { return pixels[std::size_t(y) * width + x]; }
};

struct GrayImage {
    int width = 0, height = 0;
    std::vector<float> values;
    GrayImage() = default;
    GrayImage(int w, int h) : width(w), height(h), values(std::size_t(w) * std::size_t(h), 0.0f) {
        if (w < 1 || h < 1) throw InvalidArgument("GrayImage: dimensions must be >= 1");
    }
    float& at(int x, int y) { return values[std::size_t(y) * width + x]; }
    float at(int x, int y) const { return values[std::size_t(y) * width + x]; }
};

struct Lab {
    float l = 0, a = 0, b = 0;
};

struct LabImage {
    int width = 0, height = 0;
    std::vector<Lab> values;
    LabImage() = default;
    LabImage(int w, int h) : width(w), height(h), values(std::size_t(w) * std::size_t(h)) {
        if (w < 1 || h < 1) throw InvalidArgument("LabImage: dimensions must be >= 1");
    }
    Lab& at(int x, int y) { return values[std::size_t(y) * width + x]; }
    const Lab& at(int x, int y) const { return values[std::size_t(y) * width + x]; }
};

struct DisparityMap {
    int width = 0, height = 0;
    std::vector<float> disparity;
    std::vector<uint8_t> valid;
    DisparityMap() = default;
    DisparityMap(int w, int h)
        : width(w), height(h), disparity(std::size_t(w) * std::size_t(h), 0.0f),
          valid(std::size_t(w) * std::size_t(h), 1) {
        if (w < 1 || h < 1) throw InvalidArgument("DisparityMap: dimensions must be >= 1");
    }
    float& d(int x, int y) { return disparity[std::size_t(y) * width + x]; }
    float d(int x, int y) const { return disparity[std::size_t(y) * width + x]; }
    bool is_valid(int x, int y) const { return valid[std::size_t(y) * width + x] != 0; }
    void set_valid(int x, int y, bool v) { valid[std::size_t(y) * width + x] = v ? 1 : 0; }
    friend bool operator==(const DisparityMap&, const DisparityMap&) = default;
};

inline GrayImage to_gray(const RgbImage& img) {
    GrayImage g(img.width, img.height);
    std::vector<float> lab(std::size_t(img.width) * img.height * 3);
    detail::throw_status(bsm_to_gray_lab(reinterpret_cast<const uint8_t*>(img.pixels.data()), img.width,
                                         img.height, g.values.data(), lab.data()));
    return g;
}

inline LabImage to_lab(const RgbImage& img) {
    LabImage l(img.width, img.height);
    std::vector<float> gray(std::size_t(img.width) * img.height);
    detail::throw_status(bsm_to_gray_lab(reinterpret_cast<const uint8_t*>(img.pixels.data()), img.width,
                                         img.height, gray.data(), reinterpret_cast<float*>(l.values.data())));
    return l;
}

inline float lab_sad(const Lab& a, const Lab& b) {
    return std::abs(a.l - b.l) + std::abs(a.a - b.a) + std::abs(a.b - b.b);
}

inline int clamp_coord(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

namespace detail {

// The uint8 view of an r = g = b image, or nullopt for colour input.
inline std::optional<std::vector<uint8_t>> gray_view(const RgbImage& img) {
    std::vector<uint8_t> v(img.pixels.size());
    for (std::size_t i = 0; i < v.size(); ++i) {
        const Rgb8& p = img.pixels[i];
        if (p.r != p.g || p.g != p.b) return std::nullopt;
        v[i] = p.r;
    }
    return v;
}

struct GrayTables {
    float gray[256];
    float lab[768];
    // (L, a, b) bit patterns of the 256 gray Lab values, sorted, with the gray
    // level: a Lab pixel's level by binary search instead of a 256-entry scan
    std::vector<std::pair<std::array<uint32_t, 3>, int>> lab_index;
    GrayTables() {
        throw_status(bsm_gray_lab_lut(gray, lab));
        for (int c = 0; c < 256; ++c) lab_index.push_back({key(&lab[3 * c]), c});
        std::sort(lab_index.begin(), lab_index.end());
    }
    static std::array<uint32_t, 3> key(const float* p) {
        std::array<uint32_t, 3> k;
        std::memcpy(k.data(), p, 12);
        return k;
    }
    int lab_level(const float* p) const {  // smallest gray level with exactly this Lab, or -1
        const auto k = key(p);
        auto it = std::lower_bound(lab_index.begin(), lab_index.end(), std::make_pair(k, -1));
        if (it == lab_index.end() || it->first != k) return -1;
        return it->second;
    }
};

inline const GrayTables& gray_tables() {
    static const GrayTables t;
    return t;
}

// The uint8 view behind gray / Lab planes that came from a grayscale image
// (every pixel equals the conversion of some (v,v,v)), or nullopt.
inline std::optional<std::vector<uint8_t>> u8_from_planes(const GrayImage* gray, const LabImage* lab) {
    const GrayTables& t = gray_tables();
    const std::size_t n = gray ? gray->values.size() : lab->values.size();
    std::vector<uint8_t> v(n);
    for (std::size_t i = 0; i < n; ++i) {
        int k = -1;
        if (gray) {
            const float g = gray->values[i];
            int lo = 0, hi = 255;  // the table is strictly increasing
            while (lo < hi) {
                const int mid = (lo + hi) / 2;
                if (t.gray[mid] < g) lo = mid + 1;
                else hi = mid;
            }
            if (t.gray[lo] != g) return std::nullopt;
            k = lo;
        }
        if (lab) {
            const Lab& p = lab->values[i];
            if (k < 0) {
                const float q[3] = {p.l, p.a, p.b};
                if (q[0] == 0.0f || q[1] == 0.0f || q[2] == 0.0f) {  // -0.0 == 0.0: compare by value
                    for (int c = 0; c < 256 && k < 0; ++c)
                        if (t.lab[3 * c] == p.l && t.lab[3 * c + 1] == p.a && t.lab[3 * c + 2] == p.b) k = c;
                } else {
                    k = t.lab_level(q);
                }
                if (k < 0) return std::nullopt;
            } else if (t.lab[3 * k] != p.l || t.lab[3 * k + 1] != p.a || t.lab[3 * k + 2] != p.b) {
                return std::nullopt;
            }
        }
        v[i] = uint8_t(k);
    }
    return v;
}

}  // namespace detail
}  // namespace bsm
