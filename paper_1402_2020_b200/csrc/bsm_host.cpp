// bsm_host.cpp -- see bsm_host.h.  Everything here is O(pattern) or O(256^2)
// setup work that the reference also does on the host; none of it scales with
// the image.  Compiled with g++ -O2 -march=x86-64-v3 (FMA contraction, like
// the reference's -march=native default) -- the colour tables are checked
// bit-for-bit against the compiled reference in tests/test_host.py.
#include "bsm_host.h"

#include <algorithm>
#include <cmath>
#include <functional>
#include <random>
#include <thread>

namespace bsmh {

// pattern.hpp:24-48 -- mt19937_64 uniform bits, explicit Box-Muller with spare.
namespace {
class Normal {
public:
    explicit Normal(uint64_t seed) : mt_(seed) {}
    double operator()() {
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        const double u1 = 1.0 - unit();
        const double u2 = unit();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double ang = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare_ = rad * std::sin(ang);
        spare_ok_ = true;
        return rad * std::cos(ang);
    }

private:
    double unit() { return double(mt_() >> 11) * 0x1.0p-53; }
    std::mt19937_64 mt_;
    bool spare_ok_ = false;
    double spare_ = 0.0;
};
}  // namespace

bool generate_pattern(int n, int window, double spread, uint64_t seed, int16_t* out, std::string& err) {
    if (n < 1) { err = "pattern: n must be >= 1"; return false; }
    if (window < 2) { err = "pattern: window must be >= 2"; return false; }
    if (!(spread > 0.0)) { err = "pattern: spread must be > 0"; return false; }
    Normal normal(seed);
    const long half = window / 2;
    auto offset = [&]() {
        const long v = std::lround(spread * normal());
        return int16_t(std::clamp(v, -half, half));
    };
    for (int i = 0; i < n; ++i) {
        int16_t* p = out + 4 * i;
        do {  // endpoints drawn px, py, qx, qy; degenerate pairs redrawn
            p[0] = offset();
            p[1] = offset();
            p[2] = offset();
            p[3] = offset();
        } while (p[0] == p[2] && p[1] == p[3]);
    }
    return true;
}

namespace {
// sRGB decode and the CIE f() with its linear toe (image.hpp:101-106).
double decode(double c) { return c <= 0.04045 ? c / 12.92 : std::pow((c + 0.055) / 1.055, 2.4); }
double cie_f(double t) {
    return t > 216.0 / 24389.0 ? std::cbrt(t) : ((24389.0 / 27.0) * t + 16.0) / 116.0;
}
}  // namespace

namespace {
// BT.601 luma in float, same expression shape as image.hpp:95.
float luma(uint8_t r, uint8_t g, uint8_t b) { return 0.299f * float(r) + 0.587f * float(g) + 0.114f * float(b); }

// sRGB -> XYZ (D65) normalised by the matrix row sums (image.hpp:113-115),
// then CIE Lab; r, g, b are the decoded linear channels.
void lab_from_linear(double r, double g, double b, float* out) {
    const double X = (0.4124564 * r + 0.3575761 * g + 0.1804375 * b) / 0.9504700;
    const double Y = 0.2126729 * r + 0.7151522 * g + 0.0721750 * b;
    const double Z = (0.0193339 * r + 0.1191920 * g + 0.9503041 * b) / 1.0888300;
    const double fx = cie_f(X), fy = cie_f(Y), fz = cie_f(Z);
    out[0] = float(std::clamp(116.0 * fy - 16.0, 0.0, 100.0));
    out[1] = float(500.0 * (fx - fy));
    out[2] = float(200.0 * (fy - fz));
}

void lab_of(uint8_t R, uint8_t G, uint8_t B, float* out) {
    lab_from_linear(decode(R / 255.0), decode(G / 255.0), decode(B / 255.0), out);
}
}  // namespace

void gray_lab_lut(float* gray256, float* lab768) {
    for (int v = 0; v < 256; ++v) {
        const uint8_t c = uint8_t(v);
        gray256[v] = luma(c, c, c);
        lab_of(c, c, c, lab768 + 3 * v);
    }
}

void rgb24_tables(std::vector<float>& gray, std::vector<float>& lab) {
    // Every colour through the very loop that converts images (to_gray_lab),
    // so the FP contraction is the same as for per-pixel conversion.
    gray.resize(size_t(1) << 24);
    lab.resize(size_t(3) << 24);
    auto work = [&](int r0, int r1) {
        std::vector<uint8_t> rgb(size_t(3) << 16);
        for (int r = r0; r < r1; ++r) {
            for (int g = 0; g < 256; ++g)
                for (int b = 0; b < 256; ++b) {
                    uint8_t* p = &rgb[3 * ((size_t(g) << 8) | size_t(b))];
                    p[0] = uint8_t(r);
                    p[1] = uint8_t(g);
                    p[2] = uint8_t(b);
                }
            to_gray_lab(rgb.data(), size_t(1) << 16, &gray[size_t(r) << 16], &lab[(size_t(r) << 16) * 3]);
        }
    };
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t) pool.emplace_back(work, int(256 * t / nt), int(256 * (t + 1) / nt));
    for (auto& th : pool) th.join();
}

void to_gray_lab(const uint8_t* rgb, size_t npx, float* gray, float* lab) {
    for (size_t i = 0; i < npx; ++i) {
        const uint8_t* p = rgb + 3 * i;
        if (gray) gray[i] = luma(p[0], p[1], p[2]);
        if (lab) lab_of(p[0], p[1], p[2], lab + 3 * i);
    }
}

namespace {
float sad(const float* a, const float* b) {  // image.hpp:144-146, same association
    return std::fabs(a[0] - b[0]) + std::fabs(a[1] - b[1]) + std::fabs(a[2] - b[2]);
}
}  // namespace

void sad_rank_table(const float* lab, uint8_t* rank) {
    for (int c = 0; c < 256; ++c) {
        float row[256];
        for (int v = 0; v < 256; ++v) row[v] = sad(lab + 3 * c, lab + 3 * v);
        float sorted[256];
        std::copy(row, row + 256, sorted);
        std::sort(sorted, sorted + 256);
        const int distinct = int(std::unique(sorted, sorted + 256) - sorted);
        for (int v = 0; v < 256; ++v)
            rank[c * 256 + v] = uint8_t(std::lower_bound(sorted, sorted + distinct, row[v]) - sorted);
    }
}

void vote_weight_table(const float* lab, double lc, double le, int radius, std::vector<double>& w,
                       std::vector<int16_t>& s2col, int& ncol) {
    const int smax = 2 * radius * radius;
    s2col.assign(size_t(smax) + 1, -1);
    for (int dy = 0; dy <= radius; ++dy)
        for (int dx = 0; dx <= radius; ++dx) s2col[size_t(dx * dx + dy * dy)] = 0;
    std::vector<int> cols;
    for (int s = 0; s <= smax; ++s)
        if (s2col[size_t(s)] == 0) {
            s2col[size_t(s)] = int16_t(cols.size());
            cols.push_back(s);
        }
    ncol = int(cols.size());
    std::vector<double> e(static_cast<size_t>(ncol));
    for (int k = 0; k < ncol; ++k) {
        // sqrt(double(dx)*dx + double(dy)*dy): the sum is an exact integer.
        e[size_t(k)] = std::sqrt(double(cols[size_t(k)]));
    }
    const int npair = 256 * 257 / 2;
    w.assign(size_t(npair) * size_t(ncol), 0.0);
    auto work = [&](int v0, int v1) {
        for (int v = v0; v < v1; ++v)
            for (int u = 0; u <= v; ++u) {
                const double c = double(sad(lab + 3 * v, lab + 3 * u));
                double* row = &w[(size_t(v) * (v + 1) / 2 + u) * size_t(ncol)];
                for (int k = 0; k < ncol; ++k) row[k] = std::exp(-(c / lc + e[size_t(k)] / le));
            }
    };
    // Rows are independent; split by v with balanced triangle areas.
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    int v0 = 0;
    for (unsigned t = 0; t < nt; ++t) {
        const double frac = double(t + 1) / nt;
        const int v1 = t + 1 == nt ? 256 : int(256.0 * std::sqrt(frac));
        if (v1 > v0) pool.emplace_back(work, v0, v1);
        v0 = std::max(v0, v1);
    }
    for (auto& th : pool) th.join();
}

}  // namespace bsmh

namespace bsmh {

namespace {
// Wavefronts of one 32-lane gather of the given slots: the largest number of
// distinct slots requested from one bank (a slot requested twice is one word).
int gather_cost(const int* s) {
    int cnt[32] = {0};
    uint32_t seen_lo[32] = {0};  // per bank: slots (>> 5) already counted, small tables only
    int mx = 0;
    for (int l = 0; l < 32; ++l) {
        const int b = s[l] & 31, row = s[l] >> 5;
        bool dup;
        if (row < 32) {
            dup = (seen_lo[b] >> row) & 1u;
            seen_lo[b] |= 1u << row;
        } else {
            dup = false;
            for (int k = 0; k < l; ++k)
                if (s[k] == s[l]) dup = true;
        }
        if (!dup) mx = std::max(mx, ++cnt[b]);
    }
    return mx;
}
}  // namespace

void place_rank_slots(const uint32_t* pq, int n, int u, int nslots, int lane_pos, std::vector<int>& slot,
                      double* cost_before, double* cost_after) {
    // gathers: 2 endpoints x lane_pos steps, 32 lanes each (pairs >= n: sentinel, excluded)
    const int nsteps = lane_pos;
    std::vector<int> gpair(size_t(2) * nsteps * 32, -1);  // offset index per (gather, lane), -1 = sentinel
    for (int e = 0; e < 2; ++e)
        for (int st = 0; st < nsteps; ++st)
            for (int l = 0; l < 32; ++l) {
                const int i = lane_pos * l + st;  // st = 32m + t
                if (i < n) gpair[(size_t(e) * nsteps + st) * 32 + l] = int(e ? (pq[i] >> 16) : (pq[i] & 0xFFFFu));
            }
    const int ng = 2 * nsteps;
    // offset -> gathers it appears in
    std::vector<std::vector<int>> uses(static_cast<size_t>(u));
    for (int g = 0; g < ng; ++g)
        for (int l = 0; l < 32; ++l) {
            const int o = gpair[size_t(g) * 32 + l];
            if (o >= 0 && (uses[size_t(o)].empty() || uses[size_t(o)].back() != g)) uses[size_t(o)].push_back(g);
        }
    // slot_owner[s] = offset in slot s or -1; the sentinel is handled by the kernel at slot u
    slot.resize(size_t(u));
    std::vector<int> owner(size_t(nslots), -1);
    for (int o = 0; o < u; ++o) {
        slot[size_t(o)] = o;
        owner[size_t(o)] = o;
    }
    const int sentinel_slot = nslots;  // distinct bank pattern irrelevant (pads are rare)
    auto eval = [&](int g) {
        int s[32];
        for (int l = 0; l < 32; ++l) {
            const int o = gpair[size_t(g) * 32 + l];
            s[l] = o >= 0 ? slot[size_t(o)] : sentinel_slot;
        }
        return gather_cost(s);
    };
    std::vector<int> gcost(static_cast<size_t>(ng));
    long total = 0;
    for (int g = 0; g < ng; ++g) total += (gcost[size_t(g)] = eval(g));
    if (cost_before) *cost_before = double(total) / ng;
    std::mt19937_64 rng(12345);
    std::vector<int> touched;
    std::vector<char> mark(static_cast<size_t>(ng), 0);
    const int iters = 40000;
    for (int it = 0; it < iters; ++it) {
        const int o1 = int(rng() % uint64_t(u));
        const int s2 = int(rng() % uint64_t(nslots));
        const int o2 = owner[size_t(s2)];
        if (o2 == o1) continue;
        const int s1 = slot[size_t(o1)];
        touched.clear();
        for (int g : uses[size_t(o1)])
            if (!mark[size_t(g)]) mark[size_t(g)] = 1, touched.push_back(g);
        if (o2 >= 0)
            for (int g : uses[size_t(o2)])
                if (!mark[size_t(g)]) mark[size_t(g)] = 1, touched.push_back(g);
        long before = 0;
        for (int g : touched) before += gcost[size_t(g)];
        // apply
        slot[size_t(o1)] = s2;
        owner[size_t(s2)] = o1;
        owner[size_t(s1)] = o2;
        if (o2 >= 0) slot[size_t(o2)] = s1;
        long after = 0;
        std::vector<int> nc(touched.size());
        for (size_t k = 0; k < touched.size(); ++k) after += (nc[k] = eval(touched[k]));
        if (after <= before) {
            for (size_t k = 0; k < touched.size(); ++k) gcost[size_t(touched[k])] = nc[k];
            total += after - before;
        } else {  // revert
            slot[size_t(o1)] = s1;
            owner[size_t(s1)] = o1;
            owner[size_t(s2)] = o2;
            if (o2 >= 0) slot[size_t(o2)] = s2;
        }
        for (int g : touched) mark[size_t(g)] = 0;
    }
    if (cost_after) *cost_after = double(total) / ng;
}

bool balanced_gather_order(const uint32_t* pq, int n, int u, std::vector<int>& slot, int& nslots,
                           std::vector<int>& order, std::vector<uint8_t>& flip) {
    constexpr int B = 32;
    const int STEPS = n / B;  // positions per lane: 32, 64 or 128
    if ((STEPS != 32 && STEPS != 64 && STEPS != 128 && STEPS != 256) || n != B * STEPS || u < B) return false;
    // (1) offsets -> banks with exactly 2 * STEPS endpoint references per bank
    //     and at most `cap` offsets per bank (rank-table rows).
    std::vector<int> w(size_t(u), 0);
    for (int i = 0; i < n; ++i) {
        ++w[pq[i] & 0xFFFFu];
        ++w[pq[i] >> 16];
    }
    const int target = 2 * STEPS;
    for (int o = 0; o < u; ++o)
        if (w[size_t(o)] > target) return false;
    const int cap = (u + B - 1) / B + 1;
    std::vector<int> ord(static_cast<size_t>(u));
    for (int o = 0; o < u; ++o) ord[size_t(o)] = o;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return w[size_t(a)] > w[size_t(b)]; });
    std::vector<int> bank(size_t(u), -1), sum(B, 0), cnt(B, 0);
    for (int o : ord) {
        int best = -1;
        for (int b = 0; b < B; ++b)
            if (cnt[size_t(b)] < cap && (best < 0 || sum[size_t(b)] < sum[size_t(best)])) best = b;
        if (best < 0) return false;
        bank[size_t(o)] = best;
        sum[size_t(best)] += w[size_t(o)];
        ++cnt[size_t(best)];
    }
    // local search: moves / swaps that reduce sum |sum_b - target|
    std::mt19937_64 rng(777);
    auto dev = [&](int b, int delta) { return std::abs(sum[size_t(b)] + delta - target); };
    for (int it = 0; it < 2000000; ++it) {
        bool done = true;
        for (int b = 0; b < B; ++b)
            if (sum[size_t(b)] != target) done = false;
        if (done) break;
        const int o1 = int(rng() % uint64_t(u)), b1 = bank[size_t(o1)];
        const int b2 = int(rng() % uint64_t(B));
        if (b2 == b1) continue;
        if ((it & 1) && cnt[size_t(b2)] < cap) {  // move o1 -> b2
            const int d0 = dev(b1, 0) + dev(b2, 0), d1 = dev(b1, -w[size_t(o1)]) + dev(b2, w[size_t(o1)]);
            if (d1 < d0 || (d1 == d0 && (rng() & 1))) {
                sum[size_t(b1)] -= w[size_t(o1)], sum[size_t(b2)] += w[size_t(o1)];
                --cnt[size_t(b1)], ++cnt[size_t(b2)];
                bank[size_t(o1)] = b2;
            }
        } else {  // swap o1 with a random offset of b2
            int o2 = int(rng() % uint64_t(u));
            for (int k = 0; k < u && bank[size_t(o2)] != b2; ++k) o2 = (o2 + 1) % u;
            if (bank[size_t(o2)] != b2) continue;
            const int dw = w[size_t(o2)] - w[size_t(o1)];
            const int d0 = dev(b1, 0) + dev(b2, 0), d1 = dev(b1, dw) + dev(b2, -dw);
            if (d1 < d0 || (d1 == d0 && (rng() & 1))) {
                sum[size_t(b1)] += dw, sum[size_t(b2)] -= dw;
                bank[size_t(o1)] = b2, bank[size_t(o2)] = b1;
            }
        }
    }
    for (int b = 0; b < B; ++b)
        if (sum[size_t(b)] != target) return false;
    // (2) Eulerian orientation of the bank multigraph (every degree is even):
    //     closed walks give each bank STEPS outgoing (A) and STEPS incoming (B) ends.
    std::vector<std::vector<int>> adj(B);
    for (int i = 0; i < n; ++i) {
        adj[size_t(bank[pq[i] & 0xFFFFu])].push_back(i);
        adj[size_t(bank[pq[i] >> 16])].push_back(i);
    }
    std::vector<int> ptr(B, 0), from(static_cast<size_t>(n), -1);
    for (int v0 = 0; v0 < B; ++v0) {
        for (;;) {
            int v = v0;
            bool moved = false;
            for (;;) {
                auto& a = adj[size_t(v)];
                while (ptr[size_t(v)] < int(a.size()) && from[size_t(a[size_t(ptr[size_t(v)])])] >= 0) ++ptr[size_t(v)];
                if (ptr[size_t(v)] == int(a.size())) break;
                const int e = a[size_t(ptr[size_t(v)])];
                from[size_t(e)] = v;
                const int bp = bank[pq[e] & 0xFFFFu], bq = bank[pq[e] >> 16];
                v = bp == v ? bq : bp;
                moved = true;
            }
            if (!moved || v != v0) {
                if (v != v0) return false;  // cannot happen with even degrees
                break;
            }
        }
    }
    // (3) split the STEPS-regular bipartite multigraph (A bank -> B bank) into
    //     STEPS perfect matchings; step s, lane = A bank.
    std::vector<std::vector<int>> ab(size_t(B) * B);
    for (int i = 0; i < n; ++i) {
        if (from[size_t(i)] < 0) return false;
        const int bp = bank[pq[i] & 0xFFFFu], bq = bank[pq[i] >> 16];
        const int a = from[size_t(i)], b = bp == a ? bq : bp;
        ab[size_t(a) * B + b].push_back(i);
    }
    order.assign(static_cast<size_t>(n), -1);
    flip.assign(static_cast<size_t>(n), 0);
    for (int st = 0; st < STEPS; ++st) {
        std::vector<int> match_b(B, -1);  // B bank -> A bank
        for (int a = 0; a < B; ++a) {
            std::vector<char> vis(B, 0);
            std::function<bool(int)> aug = [&](int x) -> bool {
                for (int y = 0; y < B; ++y) {
                    if (ab[size_t(x) * B + y].empty() || vis[size_t(y)]) continue;
                    vis[size_t(y)] = 1;
                    if (match_b[size_t(y)] < 0 || aug(match_b[size_t(y)])) {
                        match_b[size_t(y)] = x;
                        return true;
                    }
                }
                return false;
            };
            if (!aug(a)) return false;
        }
        for (int y = 0; y < B; ++y) {
            const int x = match_b[size_t(y)];
            const int i = ab[size_t(x) * B + y].back();
            ab[size_t(x) * B + y].pop_back();
            const int pos = STEPS * x + st;  // lane x, chunk st / 32, bit st % 32
            order[size_t(pos)] = i;
            flip[size_t(pos)] = uint8_t(bank[pq[i] & 0xFFFFu] != x);  // P is not the lane's bank
        }
    }
    // (4) slots: bank b's offsets take rows 0, 1, ... (slot = b + 32 * row)
    slot.assign(static_cast<size_t>(u), -1);
    std::vector<int> row(B, 0);
    int rows = 0;
    for (int o = 0; o < u; ++o) {
        const int b = bank[size_t(o)];
        slot[size_t(o)] = b + B * row[size_t(b)]++;
        rows = std::max(rows, row[size_t(b)]);
    }
    nslots = B * rows;
    return true;
}

}  // namespace bsmh

#include <dlfcn.h>

#include <cstring>
#include <fstream>

namespace bsmh {

double exp_restated(double x, const ExpParams& p) {
    // e_exp.c with the contraction of the FMA build (see the device copy,
    // exp_glibc in bsm_kernels.cu):
    //   kd = fma(x, InvLn2N, Shift); ki = bits(kd); kd -= Shift;
    //   r = fma(kd, NegLn2loN, fma(kd, NegLn2hiN, x));
    //   tmp = fma(r2*r2, fma(r, C5, C4), fma(fma(r, C3, C2), r2, tail + r));
    //   exp = fma(scale, tmp, scale), or specialcase() for 512 <= |x| < 1024.
    uint64_t xb;
    std::memcpy(&xb, &x, 8);
    const uint32_t abstop = uint32_t(xb >> 52) & 0x7ffu;
    bool special = false;
    if (abstop - 0x3c9u >= 0x3fu) {
        if (int(abstop) - 0x3c9 < 0) return 1.0 + x;
        if (abstop >= 0x409u) return (xb >> 63) ? 0.0 : HUGE_VAL;
        special = true;
    }
    double kd = std::fma(x, p.invln2N, p.shift);
    uint64_t ki;
    std::memcpy(&ki, &kd, 8);
    kd -= p.shift;
    const double r = std::fma(kd, p.negln2loN, std::fma(kd, p.negln2hiN, x));
    const uint64_t idx = 2 * (ki & 127);
    const uint64_t top = ki << 45;
    double tail;
    std::memcpy(&tail, &p.tab[idx], 8);
    uint64_t sbits = p.tab[idx + 1] + top;
    const double r2 = r * r;
    const double tmp = std::fma(r2 * r2, std::fma(r, p.c5, p.c4), std::fma(std::fma(r, p.c3, p.c2), r2, tail + r));
    double scale;
    if (!special) {
        std::memcpy(&scale, &sbits, 8);
        return std::fma(scale, tmp, scale);
    }
    if (!(ki & 0x80000000ull)) {
        sbits -= 1009ull << 52;
        std::memcpy(&scale, &sbits, 8);
        volatile double st = scale * tmp;
        return 0x1p1009 * (scale + st);
    }
    sbits += 1022ull << 52;
    std::memcpy(&scale, &sbits, 8);
    volatile double st = scale * tmp;  // not contracted in the library either
    double y = scale + st;
    if (y < 1.0) {
        volatile double hi = y + 1.0;
        volatile double lo = (scale - y) + st;
        volatile double l2 = ((1.0 - hi) + y) + lo;
        y = (l2 + hi) - 1.0;
        if (y == 0.0) y = 0.0;
    }
    return y * 0x1p-1022;
}

bool glibc_exp_params(ExpParams& p, std::string& why) {
    if (!__builtin_cpu_supports("fma") || !__builtin_cpu_supports("avx2")) {
        why = "host CPU lacks FMA/AVX2: libm uses its non-FMA exp";
        return false;
    }
    Dl_info info;
    double (*fexp)(double) = &::exp;
    if (!dladdr(reinterpret_cast<void*>(fexp), &info) || !info.dli_fname) {
        why = "cannot locate libm";
        return false;
    }
    std::ifstream f(info.dli_fname, std::ios::binary);
    std::string bytes((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    // __exp_data starts with InvLn2N = 0x1.71547652b82fep7, Shift = 0x1.8p52.
    const uint64_t sig[2] = {0x40671547652b82feull, 0x4338000000000000ull};
    size_t at = std::string::npos;
    for (size_t i = 0; i + 0xb0 + 2048 <= bytes.size(); i += 8)
        if (std::memcmp(bytes.data() + i, sig, 16) == 0) {
            at = i;
            break;
        }
    if (at == std::string::npos) {
        why = "exp table not found in " + std::string(info.dli_fname);
        return false;
    }
    std::memcpy(&p.invln2N, bytes.data() + at, 8 * 8);
    std::memcpy(p.tab, bytes.data() + at + 0xb0, sizeof p.tab);
    // Validate against the libm this process calls.
    std::mt19937_64 rng(7);
    for (int i = 0; i < 400000; ++i) {
        // mostly the refine range, plus the underflow/special ranges
        const double span = (i & 7) == 0 ? 1100.0 : 40.0;
        const double x = -span * double(rng() >> 11) * 0x1.0p-53 - 0x1.0p-20;
        const double a = std::exp(x), b = exp_restated(x, p);
        if (std::memcmp(&a, &b, 8) != 0) {
            why = "restated exp differs from libm";
            return false;
        }
    }
    return true;
}

}  // namespace bsmh
