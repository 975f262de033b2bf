// bsm/config.hpp -- BsmConfig (reference config.hpp:16-108) and its JSON
// sidecar (save_config / load_config, byte-identical files).
#pragma once

#include <cstdint>
#include <fstream>
#include <iterator>
#include <map>
#include <string>
#include <type_traits>

#include "bsm/errors.hpp"
#include "bsm/json_sidecar.hpp"
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

// Sidecar written next to every output (config.hpp:81-86).
inline void save_config(const BsmConfig& c, const std::string& path) {
    const std::map<std::string, std::string> m = {
        {"n", std::to_string(c.n)},
        {"S", std::to_string(c.window)},
        {"spread", json::number(c.spread)},
        {"seed", std::to_string(c.seed)},
        {"d_max", std::to_string(c.d_max)},
        {"lambda_c", json::number(c.lambda_c)},
        {"lambda_e", json::number(c.lambda_e)},
        {"lr_tolerance", json::number(c.lr_tolerance)},
        {"vote_radius", std::to_string(c.vote_radius)},
        {"gt_scale", json::number(c.gt_scale)},
        {"threads", std::to_string(c.threads)},
        {"generator", json::quoted(c.generator)},
    };
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open " + path + " for writing");
    out << json::object(m);
    if (!out) throw IoError("write failed on " + path);
}

// Keys that are absent keep their defaults (config.hpp:65-79, 88-101).
inline BsmConfig load_config(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    json::Value j;
    try {
        j = json::Parser(text).document();
    } catch (const FormatError& e) {
        throw FormatError("bad config file " + path + ": " + e.what());
    }
    if (j.kind != json::Value::Object) throw FormatError("bad config file " + path + ": not an object");
    BsmConfig c;
    auto num = [&](const char* key, auto& field) {
        if (const json::Value* v = j.find(key)) {
            if (v->kind != json::Value::Number)
                throw FormatError("bad config file " + path + ": '" + key + "' must be a number");
            using T = std::decay_t<decltype(field)>;
            if constexpr (std::is_same_v<T, uint64_t>) field = v->is_int ? T(v->uval) : T(v->num);
            else if constexpr (std::is_integral_v<T>) field = v->is_int ? T(v->ival) : T(v->num);
            else field = T(v->num);
        }
    };
    num("n", c.n);
    num("S", c.window);
    num("spread", c.spread);
    num("seed", c.seed);
    num("d_max", c.d_max);
    num("lambda_c", c.lambda_c);
    num("lambda_e", c.lambda_e);
    num("lr_tolerance", c.lr_tolerance);
    num("vote_radius", c.vote_radius);
    num("gt_scale", c.gt_scale);
    num("threads", c.threads);
    if (const json::Value* v = j.find("generator")) {
        if (v->kind != json::Value::String)
            throw FormatError("bad config file " + path + ": 'generator' must be a string");
        c.generator = v->str;
    }
    return c;
}

inline SamplingPattern generate_pattern(const BsmConfig& cfg) {
    if (cfg.generator != kGeneratorName) throw InvalidArgument("config: unknown generator '" + cfg.generator + "'");
    return generate_pattern(cfg.n, cfg.window, cfg.spread, cfg.seed);
}

}  // namespace bsm
