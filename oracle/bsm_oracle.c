/*
 * oracle/bsm_oracle.c -- CPU restatement of the Binary Stereo Matching hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load the library built from it (oracle/_build/libbsm_oracle.so).  The
 * product path (paper_1402_2020_b200/csrc) never links or calls it.
 *
 * Parity pinning: every function below is checked in tests/test_oracle.py
 * against (a) the reference library itself, compiled in place from
 * /root/reference/proj/include by oracle/Makefile into oracle/_ref/, and
 * (b) the known-answer values of the reference's own GoogleTest suite
 * (proj/tests/test_matcher.cpp, test_descriptor.cpp, test_refine.cpp,
 * test_image.cpp, test_pattern.cpp), restated in tests/test_oracle.py.
 *
 * Plain C11 (gnu11, so FP contraction follows the reference's default
 * -O3 -march=native build the same way: see DESIGN.md "float parity").
 * Bit layout follows the reference: bit i of a string lives in 64-bit word
 * i>>6 at position i&63 (bitstring.hpp:21-23,47-51); pad bits stay zero.
 * Fields are AoS, index ((y*W + x) * words64) (descriptor.hpp:48-50).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* mt19937_64 (Matsumoto & Nishimura 2004), as used by std::mt19937_64 in    */
/* pattern.hpp:45 (GaussianSource) -- restated from the published algorithm. */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* pattern.hpp:45-46: to_unit = (x >> 11) * 2^-53 */
static double unit53(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

/* Box-Muller normal source with a spare, pattern.hpp:24-48. */
typedef struct {
    mt64 rng;
    int have_spare;
    double spare;
} gauss_src;

static double gauss_next(gauss_src* g) {
    if (g->have_spare) {
        g->have_spare = 0;
        return g->spare;
    }
    const double u1 = 1.0 - unit53(mt64_next(&g->rng));
    const double u2 = unit53(mt64_next(&g->rng));
    const double radius = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
    g->spare = radius * sin(angle);
    g->have_spare = 1;
    return radius * cos(angle);
}

/* generate_pattern, pattern.hpp:74-103.  out = n x {px, py, qx, qy}. */
int oracle_generate_pattern(int n, int window, double spread, uint64_t seed, int16_t* out) {
    if (n < 1 || window < 2 || !(spread > 0.0)) return 1;
    gauss_src g;
    mt64_seed(&g.rng, seed);
    g.have_spare = 0;
    g.spare = 0.0;
    const int half = window / 2;
    for (int i = 0; i < n; ++i) {
        int16_t v[4];
        do {
            for (int k = 0; k < 4; ++k) {
                long r = lround(spread * gauss_next(&g));
                if (r < -half) r = -half;
                if (r > half) r = half;
                v[k] = (int16_t)r;
            }
        } while (v[0] == v[2] && v[1] == v[3]);
        memcpy(out + 4 * i, v, sizeof v);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Colour conversion, image.hpp:90-140.                                      */
static float to_gray1(uint8_t r, uint8_t g, uint8_t b) {
    return 0.299f * (float)r + 0.587f * (float)g + 0.114f * (float)b;
}

static double srgb_lin(double v) { return v <= 0.04045 ? v / 12.92 : pow((v + 0.055) / 1.055, 2.4); }

static double lab_fn(double t) {
    const double eps = 216.0 / 24389.0;
    const double kappa = 24389.0 / 27.0;
    return t > eps ? cbrt(t) : (kappa * t + 16.0) / 116.0;
}

static void to_lab1(uint8_t R, uint8_t G, uint8_t B, float* out) {
    const double r = srgb_lin(R / 255.0);
    const double g = srgb_lin(G / 255.0);
    const double b = srgb_lin(B / 255.0);
    const double x = (0.4124564 * r + 0.3575761 * g + 0.1804375 * b) / 0.9504700;
    const double y = 0.2126729 * r + 0.7151522 * g + 0.0721750 * b;
    const double z = (0.0193339 * r + 0.1191920 * g + 0.9503041 * b) / 1.0888300;
    const double fx = lab_fn(x), fy = lab_fn(y), fz = lab_fn(z);
    double l = 116.0 * fy - 16.0;
    if (l < 0.0) l = 0.0;
    if (l > 100.0) l = 100.0;
    out[0] = (float)l;
    out[1] = (float)(500.0 * (fx - fy));
    out[2] = (float)(200.0 * (fy - fz));
}

void oracle_gray_lab_lut(float* gray256, float* lab768) {
    for (int v = 0; v < 256; ++v) {
        gray256[v] = to_gray1((uint8_t)v, (uint8_t)v, (uint8_t)v);
        to_lab1((uint8_t)v, (uint8_t)v, (uint8_t)v, lab768 + 3 * v);
    }
}

void oracle_to_gray_lab(const uint8_t* rgb, int W, int H, float* gray, float* lab) {
    for (size_t i = 0; i < (size_t)W * (size_t)H; ++i) {
        gray[i] = to_gray1(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
        to_lab1(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], lab + 3 * i);
    }
}

/* lab_sad, image.hpp:144-146: (|dL| + |da|) + |db| in float. */
static float lab_sad(const float* a, const float* b) {
    return fabsf(a[0] - b[0]) + fabsf(a[1] - b[1]) + fabsf(a[2] - b[2]);
}

static int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); } /* image.hpp:148-150 */

/* ------------------------------------------------------------------------ */
/* quarter_threshold, descriptor.hpp:64-76: the max(1, n/4)-th smallest      */
/* weight (rank from 1).  Exact selection; any exact method returns the same  */
/* value as std::nth_element.                                                 */
static int cmp_float(const void* a, const void* b) {
    const float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

float oracle_quarter_threshold(const float* w, int n) {
    float* s = (float*)malloc(sizeof(float) * (size_t)n);
    memcpy(s, w, sizeof(float) * (size_t)n);
    qsort(s, (size_t)n, sizeof(float), cmp_float);
    const int rank = n / 4 > 1 ? n / 4 : 1;
    const float t = s[rank - 1];
    free(s);
    return t;
}

/* compute_field, descriptor.hpp:200-239 (descriptor :95-105 / :226-230,     */
/* mask_at_pixel :118-154).  Every sample coordinate is clamped; the          */
/* reference's interior fast path reads the same values.                      */
int oracle_compute_field(const float* gray, const float* lab, int W, int H, const int16_t* pairs,
                         int n, int window, uint64_t* desc, uint64_t* mask) {
    if (W < 1 || H < 1 || n < 1) return 1;
    const int words = (n + 63) / 64;
    const int half = window / 2;
    const int side = 2 * half + 1;
    float* table = (float*)malloc(sizeof(float) * (size_t)side * side);
    float* wts = (float*)malloc(sizeof(float) * (size_t)n);
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            uint64_t* d = desc + ((size_t)y * W + x) * words;
            uint64_t* m = mask + ((size_t)y * W + x) * words;
            memset(d, 0, sizeof(uint64_t) * words);
            memset(m, 0, sizeof(uint64_t) * words);
            for (int i = 0; i < n; ++i) {
                const int16_t* p = pairs + 4 * i;
                const float ip = gray[(size_t)clampi(y + p[1], H - 1) * W + clampi(x + p[0], W - 1)];
                const float iq = gray[(size_t)clampi(y + p[3], H - 1) * W + clampi(x + p[2], W - 1)];
                if (ip > iq) d[i >> 6] |= 1ULL << (i & 63);
            }
            const float* c = lab + 3 * ((size_t)y * W + x);
            for (int dy = -half; dy <= half; ++dy)
                for (int dx = -half; dx <= half; ++dx)
                    table[(dy + half) * side + (dx + half)] =
                        lab_sad(c, lab + 3 * ((size_t)clampi(y + dy, H - 1) * W + clampi(x + dx, W - 1)));
            for (int i = 0; i < n; ++i) {
                const int16_t* p = pairs + 4 * i;
                const float tp = table[(p[1] + half) * side + (p[0] + half)];
                const float tq = table[(p[3] + half) * side + (p[2] + half)];
                wts[i] = tp > tq ? tp : tq;  /* std::max(tp, tq): tq when equal -- same value */
            }
            const float thr = oracle_quarter_threshold(wts, n);
            for (int i = 0; i < n; ++i)
                if (wts[i] <= thr) m[i >> 6] |= 1ULL << (i & 63);
        }
    }
    free(table);
    free(wts);
    return 0;
}

/* Grayscale u8 view -> gray/Lab planes through the 256-entry conversion. */
static void planes_from_u8(const uint8_t* img, int W, int H, float* gray, float* lab) {
    float g256[256], l768[768];
    oracle_gray_lab_lut(g256, l768);
    for (size_t i = 0; i < (size_t)W * H; ++i) {
        gray[i] = g256[img[i]];
        memcpy(lab + 3 * i, l768 + 3 * img[i], 12);
    }
}

int oracle_compute_field_u8(const uint8_t* img, int W, int H, const int16_t* pairs, int n, int window,
                            uint64_t* desc, uint64_t* mask) {
    float* gray = (float*)malloc(sizeof(float) * (size_t)W * H);
    float* lab = (float*)malloc(sizeof(float) * 3 * (size_t)W * H);
    planes_from_u8(img, W, H, gray, lab);
    const int rc = oracle_compute_field(gray, lab, W, H, pairs, n, window, desc, mask);
    free(gray);
    free(lab);
    return rc;
}

/* masked_hamming_words / hamming_words, bitstring.hpp:73-88. */
int oracle_masked_hamming_words(const uint64_t* a, const uint64_t* b, const uint64_t* m, int nwords) {
    int t = 0;
    for (int i = 0; i < nwords; ++i) t += __builtin_popcountll((a[i] ^ b[i]) & m[i]);
    return t;
}

static int hamming_words(const uint64_t* a, const uint64_t* b, int nwords) {
    int t = 0;
    for (int i = 0; i < nwords; ++i) t += __builtin_popcountll(a[i] ^ b[i]);
    return t;
}

/* wta, matcher.hpp:80-113: streaming argmin over d ascending, strict '<'     */
/* (ties -> smaller d); out-of-image correspondences skipped (:100).          */
int oracle_wta(const uint64_t* dref, const uint64_t* mref, const uint64_t* doth, int W, int H, int n,
               int d_max, int right_ref, int use_mask, float* out) {
    if (d_max < 1) return 1;
    const int words = (n + 63) / 64;
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            const uint64_t* a = dref + ((size_t)y * W + x) * words;
            const uint64_t* m = mref + ((size_t)y * W + x) * words;
            int best_cost = 0x7fffffff, best_d = 0;
            for (int d = 0; d < d_max; ++d) {
                const int xd = right_ref ? x + d : x - d; /* matcher.hpp:35-38 */
                if (xd < 0 || xd >= W) continue;
                const uint64_t* b = doth + ((size_t)y * W + xd) * words;
                const int c = use_mask ? oracle_masked_hamming_words(a, b, m, words) : hamming_words(a, b, words);
                if (c < best_cost) {
                    best_cost = c;
                    best_d = d;
                }
            }
            out[(size_t)y * W + x] = (float)best_d;
        }
    }
    return 0;
}

/* lr_check, refine.hpp:39-54. */
int oracle_lr_check(const float* dl, const float* dr, int W, int H, double tol, float* od, uint8_t* ov) {
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            const size_t i = (size_t)y * W + x;
            const float d = dl[i];
            const int xr = (int)lround((double)x - (double)d);
            int ok = xr >= 0 && xr < W;
            if (ok) ok = fabs((double)d - (double)dr[(size_t)y * W + xr]) <= tol;
            od[i] = d;
            ov[i] = (uint8_t)(ok ? 1 : 0);
        }
    }
    return 0;
}

/* vote_weight, refine.hpp:30-35. */
double oracle_vote_weight(const float* lx, const float* lp, int dx, int dy, double lc, double le) {
    const double c = (double)lab_sad(lx, lp);
    const double e = sqrt((double)dx * dx + (double)dy * dy);
    return exp(-(c / lc + e / le));
}

/* vote_refine, refine.hpp:62-111: voters = valid pixels of the INPUT map in  */
/* the clipped window, accumulated per bin in row-major order; argmax with    */
/* strict '>' from bin 0; no voter -> d = 0, invalid.                         */
int oracle_vote_refine(const float* d, const uint8_t* v, const float* lab, int W, int H, double lc,
                       double le, int radius, float* od, uint8_t* ov) {
    int max_bin = 0;
    for (size_t i = 0; i < (size_t)W * H; ++i)
        if (v[i]) {
            const int b = (int)lround((double)d[i]);
            if (b > max_bin) max_bin = b;
        }
    double* bins = (double*)malloc(sizeof(double) * (size_t)(max_bin + 1));
    memcpy(od, d, sizeof(float) * (size_t)W * H);
    memcpy(ov, v, (size_t)W * H);
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            if (v[(size_t)y * W + x]) continue;
            for (int b = 0; b <= max_bin; ++b) bins[b] = 0.0;
            int any = 0;
            const float* lx = lab + 3 * ((size_t)y * W + x);
            const int y0 = y - radius < 0 ? 0 : y - radius;
            const int y1 = y + radius > H - 1 ? H - 1 : y + radius;
            const int x0 = x - radius < 0 ? 0 : x - radius;
            const int x1 = x + radius > W - 1 ? W - 1 : x + radius;
            for (int py = y0; py <= y1; ++py)
                for (int px = x0; px <= x1; ++px) {
                    const size_t j = (size_t)py * W + px;
                    if (!v[j]) continue;
                    const int bin = (int)lround((double)d[j]);
                    bins[bin] += oracle_vote_weight(lx, lab + 3 * j, px - x, py - y, lc, le);
                    any = 1;
                }
            const size_t i = (size_t)y * W + x;
            if (!any) {
                od[i] = 0.0f;
                ov[i] = 0;
                continue;
            }
            int best = 0;
            for (int b = 1; b <= max_bin; ++b)
                if (bins[b] > bins[best]) best = b;
            od[i] = (float)best;
            ov[i] = 1;
        }
    }
    free(bins);
    return 0;
}

/* run_pipeline, pipeline.hpp:25-56, for grayscale u8 views (r=g=b).  Any     */
/* output pointer may be NULL.                                                */
int oracle_pipeline_u8(const uint8_t* left, const uint8_t* right, int W, int H, const int16_t* pairs,
                       int n, int window, int d_max, double lc, double le, double tol, int radius,
                       float* refined_d, uint8_t* refined_v, float* left_d, float* right_d,
                       float* checked_d, uint8_t* checked_v) {
    if (d_max < 1) return 1;
    const size_t px = (size_t)W * H;
    const int words = (n + 63) / 64;
    float* gl = (float*)malloc(4 * px);
    float* ll = (float*)malloc(12 * px);
    float* gr = (float*)malloc(4 * px);
    float* lr = (float*)malloc(12 * px);
    uint64_t* dl = (uint64_t*)malloc(8 * px * words);
    uint64_t* ml = (uint64_t*)malloc(8 * px * words);
    uint64_t* dr = (uint64_t*)malloc(8 * px * words);
    uint64_t* mr = (uint64_t*)malloc(8 * px * words);
    float* lw = (float*)malloc(4 * px);
    float* rw = (float*)malloc(4 * px);
    float* cd = (float*)malloc(4 * px);
    uint8_t* cv = (uint8_t*)malloc(px);
    float* fd = (float*)malloc(4 * px);
    uint8_t* fv = (uint8_t*)malloc(px);
    planes_from_u8(left, W, H, gl, ll);
    planes_from_u8(right, W, H, gr, lr);
    oracle_compute_field(gl, ll, W, H, pairs, n, window, dl, ml);
    oracle_compute_field(gr, lr, W, H, pairs, n, window, dr, mr);
    oracle_wta(dl, ml, dr, W, H, n, d_max, 0, 1, lw);
    oracle_wta(dr, mr, dl, W, H, n, d_max, 1, 1, rw);
    oracle_lr_check(lw, rw, W, H, tol, cd, cv);
    oracle_vote_refine(cd, cv, ll, W, H, lc, le, radius, fd, fv);
    if (refined_d) memcpy(refined_d, fd, 4 * px);
    if (refined_v) memcpy(refined_v, fv, px);
    if (left_d) memcpy(left_d, lw, 4 * px);
    if (right_d) memcpy(right_d, rw, 4 * px);
    if (checked_d) memcpy(checked_d, cd, 4 * px);
    if (checked_v) memcpy(checked_v, cv, px);
    free(gl); free(ll); free(gr); free(lr);
    free(dl); free(ml); free(dr); free(mr);
    free(lw); free(rw); free(cd); free(cv); free(fd); free(fv);
    return 0;
}
