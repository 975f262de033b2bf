// synth.cpp -- the BASELINE.json synthetic stereo-pair generator (bench / test
// input only; not part of the matching path).
//
// Restates BASELINE.json configs[0..4] with the builder choices pinned in
// SURVEY.md section 8(d).  The paper's Middlebury / illumination data are not
// in this container; seeded synthetic pairs with the configs' shapes and value
// distributions stand in for them.
//
//  * RNG: std::mt19937_64, unit = (x >> 11) * 2^-53 (the reference's own
//    convention, pattern.hpp:45-46 / synthetic.hpp:17), explicit Box-Muller.
//  * Texture: uint8 uniform floor(unit*256), 3x3 box mean with border clamp,
//    rounded (sum + 4) / 9.
//  * Left-view disparity: background 10; K axis-aligned rectangles, width in
//    [W/8, W/3], height in [H/8, H/3], uniform position inside the frame,
//    painted in draw order, disparity uniform int in [lo, hi]; optional
//    slanted planes d = round(a + b*x) over an extra rectangle each.
//  * Warp: right(x - d, y) = left(x, y) when x - d >= 0, larger d wins;
//    right pixels with no source get fresh uniform noise.
//  * Noise: N(0, sigma^2) added to both views, rounded, clamped to [0, 255].
//  * Radiometric (configs[2]): right = clip(round(255*((1.5 I + 20)/255)^0.8))
//    before its noise (sigma 4); left sigma 2.
//
// Draw order (pinned): texture (W*H uniforms), then per rectangle
// (w, h, x0, y0, d), then per slanted plane (w, h, x0, y0), then the
// right-view hole fill in raster order, then left noise, then right noise.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace {

struct Rng {
    std::mt19937_64 mt;
    bool have_spare = false;
    double spare = 0.0;
    explicit Rng(uint64_t seed) : mt(seed) {}
    double unit() { return double(mt() >> 11) * 0x1.0p-53; }
    int uniform_int(int lo, int hi) { return lo + int(unit() * double(hi - lo + 1)); }  // inclusive
    double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        const double u1 = 1.0 - unit();
        const double u2 = unit();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = r * std::sin(a);
        have_spare = true;
        return r * std::cos(a);
    }
};

uint8_t clamp_round(double v) {
    const double r = std::floor(v + 0.5);
    return uint8_t(r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r));
}

struct Spec {
    int layers, dlo, dhi;
    int planes;           // slanted planes
    double pa[2], pb[2];  // d = pa + pb * x
    double sigma_left, sigma_right;
    bool radiometric;
};

Spec spec_for(int config) {
    switch (config) {
        case 0: return {4, 5, 55, 0, {0, 0}, {0, 0}, 2.0, 2.0, false};
        case 1: return {8, 10, 230, 1, {40.0, 0}, {0.05, 0}, 2.0, 2.0, false};
        case 2: return {4, 5, 55, 0, {0, 0}, {0, 0}, 2.0, 4.0, true};
        case 3: return {6, 10, 180, 0, {0, 0}, {0, 0}, 2.0, 2.0, false};
        default: return {12, 10, 240, 2, {30.0, 200.0}, {0.03, -0.02}, 2.0, 2.0, false};
    }
}

}  // namespace

extern "C" {

// config: 0..4 = BASELINE.json configs[0..4].  left/right: W*H bytes, row-major.
// disp (optional): the left-view ground-truth disparity used for the warp.
int bsm_synth_pair(int config, uint64_t seed, int W, int H, uint8_t* left, uint8_t* right, int32_t* disp) {
    if (W < 8 || H < 8 || config < 0 || config > 4) return 1;
    const Spec s = spec_for(config);
    Rng rng(seed);
    const size_t N = size_t(W) * size_t(H);

    std::vector<uint8_t> raw(N);
    for (size_t i = 0; i < N; ++i) raw[i] = uint8_t(std::min(255, int(rng.unit() * 256.0)));
    std::vector<uint8_t> tex(N);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            int sum = 0;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int yy = std::clamp(y + dy, 0, H - 1), xx = std::clamp(x + dx, 0, W - 1);
                    sum += raw[size_t(yy) * W + xx];
                }
            tex[size_t(y) * W + x] = uint8_t((sum + 4) / 9);
        }

    std::vector<int> d(N, 10);
    auto rect = [&](int& x0, int& y0, int& rw, int& rh) {
        rw = rng.uniform_int(W / 8, W / 3);
        rh = rng.uniform_int(H / 8, H / 3);
        x0 = rng.uniform_int(0, W - rw);
        y0 = rng.uniform_int(0, H - rh);
    };
    for (int k = 0; k < s.layers; ++k) {
        int x0, y0, rw, rh;
        rect(x0, y0, rw, rh);
        const int dv = rng.uniform_int(s.dlo, s.dhi);
        for (int y = y0; y < y0 + rh; ++y)
            for (int x = x0; x < x0 + rw; ++x) d[size_t(y) * W + x] = dv;
    }
    for (int p = 0; p < s.planes; ++p) {
        int x0, y0, rw, rh;
        rect(x0, y0, rw, rh);
        for (int y = y0; y < y0 + rh; ++y)
            for (int x = x0; x < x0 + rw; ++x)
                d[size_t(y) * W + x] = int(std::floor(s.pa[p] + s.pb[p] * double(x) + 0.5));
    }

    // left = texture; right(x - d) = left(x), larger d in front.
    std::vector<int> owner(N, -1);
    std::vector<uint8_t> r(N, 0);
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const int dv = d[size_t(y) * W + x];
            const int xr = x - dv;
            if (xr < 0) continue;
            int& o = owner[size_t(y) * W + xr];
            if (dv > o) {
                o = dv;
                r[size_t(y) * W + xr] = tex[size_t(y) * W + x];
            }
        }
    for (size_t i = 0; i < N; ++i)
        if (owner[i] < 0) r[i] = uint8_t(std::min(255, int(rng.unit() * 256.0)));

    if (s.radiometric)
        for (size_t i = 0; i < N; ++i)
            r[i] = clamp_round(255.0 * std::pow((1.5 * double(r[i]) + 20.0) / 255.0, 0.8));

    for (size_t i = 0; i < N; ++i) left[i] = clamp_round(double(tex[i]) + s.sigma_left * rng.normal());
    for (size_t i = 0; i < N; ++i) right[i] = clamp_round(double(r[i]) + s.sigma_right * rng.normal());
    if (disp)
        for (size_t i = 0; i < N; ++i) disp[i] = d[i];
    return 0;
}

}  // extern "C"
