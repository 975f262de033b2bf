// bsm/pattern.hpp -- sampling pattern (reference pattern.hpp:16-103).
// Generation runs in the library's host code (bsm_generate_pattern):
// mt19937_64 + explicit Box-Muller, bit-identical to the reference.
// The JSON sidecar (save/load_pattern) is file I/O and out of scope here.
#pragma once

#include <cstdint>
#include <vector>

#include "../bsm_cuda.h"
#include "bsm/detail_cabi.hpp"
#include "bsm/errors.hpp"

namespace bsm {

inline constexpr const char* kGeneratorName = "mt19937_64-boxmuller-v1";

struct PairOffsets {
    int16_t px = 0, py = 0, qx = 0, qy = 0;
    friend bool operator==(const PairOffsets&, const PairOffsets&) = default;
};

struct SamplingPattern {
    int n = 0;
    int window = 0;
    double spread = 0.0;
    uint64_t seed = 0;
    std::vector<PairOffsets> pairs;
    int half_window() const { return window / 2; }
    friend bool operator==(const SamplingPattern&, const SamplingPattern&) = default;
};

inline SamplingPattern generate_pattern(int n, int window, double spread, uint64_t seed) {
    SamplingPattern p;
    p.n = n;
    p.window = window;
    p.spread = spread;
    p.seed = seed;
    p.pairs.resize(n > 0 ? std::size_t(n) : 0);
    detail::throw_status(bsm_generate_pattern(n, window, spread, seed,
                                              n > 0 ? reinterpret_cast<int16_t*>(p.pairs.data()) : nullptr));
    return p;
}

namespace detail {
inline std::vector<int16_t> flat_pairs(const SamplingPattern& p) {
    std::vector<int16_t> f(std::size_t(p.n) * 4);
    for (int i = 0; i < p.n; ++i) {
        f[4 * std::size_t(i)] = p.pairs[std::size_t(i)].px;
        f[4 * std::size_t(i) + 1] = p.pairs[std::size_t(i)].py;
        f[4 * std::size_t(i) + 2] = p.pairs[std::size_t(i)].qx;
        f[4 * std::size_t(i) + 3] = p.pairs[std::size_t(i)].qy;
    }
    return f;
}
}  // namespace detail

}  // namespace bsm
