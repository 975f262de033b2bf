// bsm/pattern.hpp -- sampling pattern (reference pattern.hpp:16-103).
// Generation runs in the library's host code (bsm_generate_pattern):
// mt19937_64 + explicit Box-Muller, bit-identical to the reference.
// save_pattern / load_pattern keep the reference's JSON sidecar
// (pattern.hpp:104-160), byte-identical files.
#pragma once

#include <cstdint>
#include <fstream>
#include <iterator>
#include <map>
#include <string>
#include <vector>

#include "../bsm_cuda.h"
#include "bsm/detail_cabi.hpp"
#include "bsm/errors.hpp"
#include "bsm/json_sidecar.hpp"

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

// Generator name, generating parameters and the realised offsets, one
// quadruple per line.
inline void save_pattern(const SamplingPattern& p, const std::string& path) {
    std::string pairs = "[\n";
    for (std::size_t i = 0; i < p.pairs.size(); ++i) {
        const PairOffsets& q = p.pairs[i];
        pairs += "\t\t[" + std::to_string(q.px) + "," + std::to_string(q.py) + "," + std::to_string(q.qx) + "," +
                 std::to_string(q.qy) + "]" + (i + 1 < p.pairs.size() ? ",\n" : "\n");
    }
    pairs += "\t]";
    const std::map<std::string, std::string> m = {
        {"generator", json::quoted(kGeneratorName)}, {"n", std::to_string(p.n)},
        {"S", std::to_string(p.window)},             {"spread", json::number(p.spread)},
        {"seed", std::to_string(p.seed)},            {"pairs", pairs},
    };
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open " + path + " for writing");
    out << json::object(m);
    if (!out) throw IoError("write failed on " + path);
}

inline SamplingPattern load_pattern(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open " + path);
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    const std::string bad = "bad pattern file " + path + ": ";
    json::Value j;
    try {
        j = json::Parser(text).document();
    } catch (const FormatError& e) {
        throw FormatError(bad + e.what());
    }
    auto need = [&](const char* key, json::Value::Kind kind) -> const json::Value& {
        const json::Value* v = j.find(key);
        if (!v) throw FormatError(bad + "missing key '" + key + "'");
        if (v->kind != kind) throw FormatError(bad + "wrong type for '" + key + "'");
        return *v;
    };
    const std::string gen = need("generator", json::Value::String).str;
    if (gen != kGeneratorName)
        throw FormatError("pattern file " + path + " uses unknown generator '" + gen + "'");
    SamplingPattern p;
    p.n = int(need("n", json::Value::Number).num);
    p.window = int(need("S", json::Value::Number).num);
    p.spread = need("spread", json::Value::Number).num;
    const json::Value& sd = need("seed", json::Value::Number);
    p.seed = sd.is_int ? sd.uval : uint64_t(sd.num);
    const json::Value& arr = need("pairs", json::Value::Array);
    if (int(arr.arr.size()) != p.n) throw FormatError("pattern file " + path + ": pair count does not match n");
    const int h = p.window / 2;
    for (const json::Value& e : arr.arr) {
        if (e.kind != json::Value::Array || e.arr.size() < 4) throw FormatError(bad + "malformed pair");
        int16_t v[4];
        for (int k = 0; k < 4; ++k) {
            v[k] = int16_t(e.arr[std::size_t(k)].num);
            if (v[k] < -h || v[k] > h) throw FormatError("pattern file " + path + ": offset outside window");
        }
        p.pairs.push_back({v[0], v[1], v[2], v[3]});
    }
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
