// bsm/config.hpp -- BsmConfig (reference config.hpp:16-108).  JSON
// persistence is file I/O and out of scope for the GPU hot path.
#pragma once

#include <cstdint>
#include <string>

#include "bsm/errors.hpp"
#include "bsm/pattern.hpp"

namespace bsm {

struct BsmConfig {
    int n = 4096;
    int window = 26;
    double spread = 4.0;
    uint64_t seed = 42;
    int d_max = 0;
    double lambda_c = 9.0;
    double lambda_e = 16.0;
    double lr_tolerance = 1.0;
    int vote_radius = 20;
    double gt_scale = 16.0;
    int threads = 1;  // accepted; device output is independent of it
    std::string generator = kGeneratorName;

    void validate() const {
        if (n < 1) throw InvalidArgument("config: n must be >= 1");
        if (window < 2) throw InvalidArgument("config: S must be >= 2");
        if (!(spread > 0)) throw InvalidArgument("config: spread must be > 0");
        if (d_max < 1) throw InvalidArgument("config: d_max must be set (>= 1)");
        if (!(lambda_c > 0)) throw InvalidArgument("config: lambda_c must be > 0");
        if (!(lambda_e > 0)) throw InvalidArgument("config: lambda_e must be > 0");
        if (lr_tolerance < 0) throw InvalidArgument("config: lr_tolerance must be >= 0");
        if (vote_radius < 1) throw InvalidArgument("config: vote_radius must be >= 1");
        if (!(gt_scale > 0)) throw InvalidArgument("config: gt_scale must be > 0");
        if (threads < 1) throw InvalidArgument("config: threads must be >= 1");
        if (generator != kGeneratorName)
            throw InvalidArgument("config: unknown generator '" + generator + "', this build provides " +
                                  kGeneratorName);
    }
    friend bool operator==(const BsmConfig&, const BsmConfig&) = default;
};

inline SamplingPattern generate_pattern(const BsmConfig& cfg) {
    if (cfg.generator != kGeneratorName) throw InvalidArgument("config: unknown generator '" + cfg.generator + "'");
    return generate_pattern(cfg.n, cfg.window, cfg.spread, cfg.seed);
}

}  // namespace bsm
