// bsm/descriptor.hpp -- DescriptorField and the descriptor/mask API
// (reference descriptor.hpp:18-239).  compute_field runs on the GPU
// (bsm_compute_field_u8 / _f32: kernels k_descriptor4 + k_mask4, or
// k_descriptor_f32 + k_mask_f32 for float planes, any n <= 8192).  The
// single-pixel compute_descriptor / compute_mask (descriptor.hpp:174-196) cost
// O(n): the clamped (2h+1)^2 window around the pixel is gathered on the host
// into a tile whose centre samples exactly what the pixel samples, and the
// same kernels run on that tile.
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <vector>

#include "../bsm_cuda.h"
#include "bsm/bitstring.hpp"
#include "bsm/detail_cabi.hpp"
#include "bsm/errors.hpp"
#include "bsm/image.hpp"
#include "bsm/pattern.hpp"

namespace bsm {

class DescriptorField {
public:
    DescriptorField() = default;
    DescriptorField(int width, int height, int n_bits)
        : width_(width), height_(height), n_(n_bits), words_(words_for_bits(n_bits)),
          desc_(std::size_t(width) * height * std::size_t(words_), 0),
          mask_(std::size_t(width) * height * std::size_t(words_), 0) {}

    int width() const { return width_; }
    int height() const { return height_; }
    int bits() const { return n_; }
    int words_per_string() const { return words_; }

    std::span<const uint64_t> descriptor(int x, int y) const { return {&desc_[index(x, y)], std::size_t(words_)}; }
    std::span<const uint64_t> mask(int x, int y) const { return {&mask_[index(x, y)], std::size_t(words_)}; }
    std::span<uint64_t> descriptor(int x, int y) { return {&desc_[index(x, y)], std::size_t(words_)}; }
    std::span<uint64_t> mask(int x, int y) { return {&mask_[index(x, y)], std::size_t(words_)}; }
    BitString descriptor_at(int x, int y) const { return bits_of(descriptor(x, y)); }
    BitString mask_at(int x, int y) const { return bits_of(mask(x, y)); }

    // Flat AoS storage, index ((y*W + x) * words) -- the C ABI's layout.
    uint64_t* descriptor_data() { return desc_.data(); }
    uint64_t* mask_data() { return mask_.data(); }
    const uint64_t* descriptor_data() const { return desc_.data(); }
    const uint64_t* mask_data() const { return mask_.data(); }

private:
    std::size_t index(int x, int y) const { return (std::size_t(y) * width_ + x) * std::size_t(words_); }
    BitString bits_of(std::span<const uint64_t> w) const {
        BitString b(n_);
        std::copy(w.begin(), w.end(), b.words().begin());
        return b;
    }
    int width_ = 0, height_ = 0, n_ = 0, words_ = 0;
    std::vector<uint64_t> desc_, mask_;
};

// The floor(n/4)-th smallest weight, rank from 1 (host scalar helper).
inline float quarter_threshold(std::span<const float> weights, std::vector<float>& scratch) {
    if (weights.empty()) throw InvalidArgument("quarter_threshold: empty weight sequence");
    const std::size_t rank = std::max<std::size_t>(1, weights.size() / 4);
    scratch.assign(weights.begin(), weights.end());
    std::nth_element(scratch.begin(), scratch.begin() + std::ptrdiff_t(rank - 1), scratch.end());
    return scratch[rank - 1];
}

inline float quarter_threshold(std::span<const float> weights) {
    std::vector<float> s;
    return quarter_threshold(weights, s);
}

namespace detail {
inline DescriptorField field_u8(const std::vector<uint8_t>& img, int W, int H, const SamplingPattern& pat) {
    Context& ctx = context();
    ctx.use_pattern(flat_pairs(pat), pat.n, pat.window);
    DescriptorField f(W, H, pat.n);
    throw_status(bsm_compute_field_u8(ctx.get(), img.data(), W, H, f.descriptor_data(), f.mask_data()));
    return f;
}
// Arbitrary float planes (colour views): the float-plane kernels (any n <= 8192).
inline DescriptorField field_f32(const float* gray, const float* lab, int W, int H, const SamplingPattern& pat) {
    static_assert(sizeof(Lab) == 3 * sizeof(float), "Lab must be three packed floats");
    Context& ctx = context();
    ctx.use_pattern(flat_pairs(pat), pat.n, pat.window);
    DescriptorField f(W, H, pat.n);
    throw_status(bsm_compute_field_f32(ctx.get(), gray, lab, W, H, f.descriptor_data(), f.mask_data()));
    return f;
}
}  // namespace detail

inline DescriptorField compute_field(const GrayImage& gray, const LabImage& lab, const SamplingPattern& pat,
                                     int threads = 1) {
    (void)threads;
    if (gray.width != lab.width || gray.height != lab.height)
        throw DimensionMismatch("compute_field: gray/lab dimensions differ");
    const auto u8 = detail::u8_from_planes(&gray, &lab);
    if (!u8)
        return detail::field_f32(gray.values.data(), &lab.values[0].l, gray.width, gray.height, pat);
    return detail::field_u8(*u8, gray.width, gray.height, pat);
}

namespace detail {
// The (2h+1) x (2h+1) window around (x, y) with the reference's border clamp
// (clamp_coord, image.hpp:148-150): tile(u, v) = img(clamp(x-h+u), clamp(y-h+v)).
// Every sample of the tile's centre pixel lies inside the tile, so its
// descriptor and mask equal the pixel's in the full image.
template <typename T>
std::vector<T> window_tile(const std::vector<T>& img, int W, int H, int x, int y, int half) {
    const int side = 2 * half + 1;
    std::vector<T> t(std::size_t(side) * side);
    for (int v = 0; v < side; ++v) {
        const int yy = std::clamp(y - half + v, 0, H - 1);
        for (int u = 0; u < side; ++u) t[std::size_t(v) * side + u] = img[std::size_t(yy) * W + std::clamp(x - half + u, 0, W - 1)];
    }
    return t;
}
}  // namespace detail

inline BitString compute_descriptor(const GrayImage& gray, const SamplingPattern& pat, int x, int y) {
    if (x < 0 || x >= gray.width || y < 0 || y >= gray.height)
        throw InvalidArgument("compute_descriptor: pixel outside image");
    const int h = pat.half_window(), side = 2 * h + 1;
    GrayImage tile(side, side);
    tile.values = detail::window_tile(gray.values, gray.width, gray.height, x, y, h);
    const auto u8 = detail::u8_from_planes(&tile, nullptr);
    if (!u8) {
        const std::vector<float> lab(tile.values.size() * 3, 0.0f);  // the mask is not read
        return detail::field_f32(tile.values.data(), lab.data(), side, side, pat).descriptor_at(h, h);
    }
    return detail::field_u8(*u8, side, side, pat).descriptor_at(h, h);
}

inline BitString compute_mask(const LabImage& lab, const SamplingPattern& pat, int x, int y) {
    if (x < 0 || x >= lab.width || y < 0 || y >= lab.height)
        throw InvalidArgument("compute_mask: pixel outside image");
    const int h = pat.half_window(), side = 2 * h + 1;
    LabImage tile(side, side);
    tile.values = detail::window_tile(lab.values, lab.width, lab.height, x, y, h);
    const auto u8 = detail::u8_from_planes(nullptr, &tile);
    if (!u8) {
        const std::vector<float> gray(tile.values.size(), 0.0f);  // the descriptor is not read
        return detail::field_f32(gray.data(), &tile.values[0].l, side, side, pat).mask_at(h, h);
    }
    return detail::field_u8(*u8, side, side, pat).mask_at(h, h);
}

}  // namespace bsm
