// kern_refine.cuh -- K5/K6: left/right check, voting refinement and the
// device exp restatement.  Part of bsm_kernels.cu's single translation unit.
#pragma once

// ---------------------------------------------------------------------------
// Peer outputs of the frame-band partition over peer memory (bsm_frame,
// bsm_dist.cuh): K5 and K6 also store the output band's final values straight
// into every rank's full-frame map (own memory and peers' mapped by CUDA IPC),
// so the all-gather is fused into the kernels that produce the band.
constexpr int kMaxPeers = 8;
struct PeerOut {
    float* d[kMaxPeers];
    uint8_t* v[kMaxPeers];
    int n;    // ranks to store to; 0: none
    int W;
    int rb0;  // band-local first output row
    int g0;   // its global row
};

template <bool PEER>
__device__ __forceinline__ void peer_store(const PeerOut& po, int p, float d, uint8_t v) {
    if (!PEER) return;
    const int yy = p / po.W, x = p - yy * po.W;
    const size_t g = size_t(po.g0 + yy - po.rb0) * po.W + x;
    for (int k = 0; k < po.n; ++k) {
        po.d[k][g] = d;
        po.v[k][g] = v;
    }
}

// ---------------------------------------------------------------------------
// K5 -- left/right check on WTA keys.  refine.hpp:39-54: valid(x) <=>
// xr = lround(x - dL) in [0, W) and |dL - dR(xr)| <= tol (inclusive, double).
// Also emits the (all-valid) WTA maps as float when requested, the band-local
// max_bin of the checked map (refine.hpp:68-72) and the list of invalid
// pixels in the refine band [rb0, rb1).
template <bool PEER>
__global__ void k_lr_check_keys(const uint32_t* __restrict__ kl, const uint32_t* __restrict__ kr, int W,
                                int rows, double tol, float* __restrict__ chk_d, uint8_t* __restrict__ chk_v,
                                float* __restrict__ left_d, float* __restrict__ right_d, int rb0, int rb1,
                                int* __restrict__ counters, int* __restrict__ inv, const PeerOut po) {
    const size_t total = size_t(rows) * W;
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < total;
    int dl = 0;
    bool ok = false;
    int yy = 0;
    if (in) {
        yy = int(i / W);
        const int x = int(i - size_t(yy) * W);
        dl = int(kl[i] & 0xFFFFu);
        const int xr = x - dl;
        ok = xr >= 0 && xr < W;
        if (ok) ok = fabs(double(dl) - double(kr[size_t(yy) * W + xr] & 0xFFFFu)) <= tol;
        chk_d[i] = float(dl);
        chk_v[i] = ok ? 1 : 0;
        if (left_d) left_d[i] = float(dl);
        if (right_d) right_d[i] = float(kr[i] & 0xFFFFu);
        if (yy >= rb0 && yy < rb1) peer_store<PEER>(po, int(i), float(dl), ok ? 1 : 0);  // K6 overwrites the invalid ones
    }
    const unsigned full = 0xFFFFFFFFu;
    const int mb = __reduce_max_sync(full, (in && ok) ? dl : 0);
    const bool need = in && !ok && yy >= rb0 && yy < rb1;
    const unsigned ballot = __ballot_sync(full, need);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) {
        atomicMax(&counters[0], mb);
        if (ballot) base = atomicAdd(&counters[1], __popc(ballot));
    }
    base = __shfl_sync(full, base, 0);
    if (need) inv[base + __popc(ballot & ((1u << lane) - 1u))] = int(i);
}

// The per-stage vote_refine's inputs on the device (refine.hpp:64-72): the
// invalid pixels (warp-aggregated list in counters[1] / inv), max over the
// valid pixels of lround(d) (counters[0], refine.hpp:68-72), and counters[3]
// set when a valid disparity is out of range (not in (-0.5, lim), or NaN).
__global__ void k_invalid_list(const float* __restrict__ d, const uint8_t* __restrict__ v, size_t px, double lim,
                               int* __restrict__ counters, int* __restrict__ inv) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool in = i < px;
    const bool valid = in && v[i] != 0;
    int bin = 0;
    bool bad = false;
    if (valid) {
        const double dv = double(d[i]);
        bad = !(dv > -0.5) || !(dv < lim);
        if (!bad) bin = int(llround(dv));
    }
    const unsigned full = 0xFFFFFFFFu;
    const int mb = __reduce_max_sync(full, bin);
    const bool anybad = __any_sync(full, bad);
    const bool need = in && !valid;
    const unsigned ballot = __ballot_sync(full, need);
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) {
        atomicMax(&counters[0], mb);
        if (anybad) atomicExch(&counters[3], 1);
        if (ballot) base = atomicAdd(&counters[1], __popc(ballot));
    }
    base = __shfl_sync(full, base, 0);
    if (need) inv[base + __popc(ballot & ((1u << lane) - 1u))] = int(i);
}

// lr_check on float maps (per-stage API, refine.hpp:39-54).
__global__ void k_lr_check_float(const float* __restrict__ dl, const float* __restrict__ dr, int W, int H,
                                 double tol, float* __restrict__ od, uint8_t* __restrict__ ov) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= size_t(W) * H) return;
    const int y = int(i / W), x = int(i - size_t(y) * W);
    const float d = dl[i];
    const long long xr = llround(double(x) - double(d));
    bool ok = xr >= 0 && xr < W;
    if (ok) ok = fabs(double(d) - double(dr[size_t(y) * W + xr])) <= tol;
    od[i] = d;
    ov[i] = ok ? 1 : 0;
}

// ---------------------------------------------------------------------------
// K6 -- bilateral voting refinement.  refine.hpp:62-111.  Warp per invalid
// pixel.  Voters of one window row are examined 32 at a time (lane = column);
// their bin lround(d) and weight (exact host table, refine.hpp:30-35) are
// formed in parallel, then folded into the per-warp double bins strictly in
// row-major voter order (the owner lane of a bin performs its adds in
// sequence), so every bin sum is bit-identical to the reference's.  Argmax:
// strict '>' from bin 0 == smallest bin among the maxima.
template <bool PEER>
__global__ void k_vote_refine(const float* __restrict__ cd, const uint8_t* __restrict__ cv,
                              const uint8_t* __restrict__ gray, int W, int rows, int radius,
                              const double* __restrict__ wtab, int ncol, const int16_t* __restrict__ s2col,
                              const int* __restrict__ counters, const int* __restrict__ inv,
                              int nbins_cap, float* __restrict__ od, uint8_t* __restrict__ ov, const PeerOut po) {
    extern __shared__ __align__(16) double sbins[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    double* bins = sbins + size_t(warp) * nbins_cap;
    const int max_bin = counters[0];
    const int n_inv = counters[1];
    const unsigned full = 0xFFFFFFFFu;
    for (int idx = blockIdx.x * nwarps + warp; idx < n_inv; idx += gridDim.x * nwarps) {
        const int p = inv[idx];
        const int y = p / W, x = p - y * W;
        const int u = gray[p];
        for (int b = lane; b <= max_bin; b += 32) bins[b] = 0.0;
        __syncwarp();
        const int y0 = max(0, y - radius), y1 = min(rows - 1, y + radius);
        const int x0 = max(0, x - radius), x1 = min(W - 1, x + radius);
        bool any = false;
        for (int py = y0; py <= y1; ++py) {
            const int dy2 = (py - y) * (py - y);
            for (int cx = x0; cx <= x1; cx += 32) {
                const int px = cx + lane;
                const size_t j = size_t(py) * W + px;
                const bool valid = px <= x1 && cv[j];
                int bin = 0;
                double wgt = 0.0;
                if (valid) {
                    bin = int(llround(double(cd[j])));
                    const int v = gray[j];
                    const int hi = max(u, v), lo = min(u, v);
                    const int s = (px - x) * (px - x) + dy2;
                    wgt = __ldg(wtab + (size_t(hi * (hi + 1) / 2 + lo) * ncol + s2col[s]));
                }
                unsigned m = __ballot_sync(full, valid);
                any |= m != 0;
                while (m) {
                    const int i = __ffs(m) - 1;
                    m &= m - 1;
                    const int b = __shfl_sync(full, bin, i);
                    const double wv = __shfl_sync(full, wgt, i);
                    if (lane == (b & 31)) bins[b] += wv;
                }
            }
        }
        __syncwarp();
        if (!any) {
            if (lane == 0) {
                od[p] = 0.0f;
                ov[p] = 0;
                peer_store<PEER>(po, p, 0.0f, 0);
            }
            continue;
        }
        double bv = -1.0;
        int bb = 0x7FFFFFFF;
        for (int b = lane; b <= max_bin; b += 32)
            if (bins[b] > bv) {
                bv = bins[b];
                bb = b;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov2 = __shfl_xor_sync(full, bv, o);
            const int ob = __shfl_xor_sync(full, bb, o);
            if (ov2 > bv || (ov2 == bv && ob < bb)) {
                bv = ov2;
                bb = ob;
            }
        }
        if (lane == 0) {
            od[p] = float(bb);
            ov[p] = 1;
            peer_store<PEER>(po, p, float(bb), 1);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// K6' -- voting refinement, thread per invalid pixel (refine.hpp:62-111).
// Each thread walks its clipped (2r+1)^2 window in row-major order and adds
// every valid voter's exact weight to its own column of double bins in
// shared memory ([bin][thread]: a lane always hits its own bank pair, so any
// mix of bins is conflict-free).  Per bin the additions happen in the
// reference's voter order, so the sums are bit-identical.  Voter data comes
// pre-packed (k_make_vmap: bin | gray << 16 | valid << 24); the window offset
// (dy, dx) is warp-uniform, so the distance column of the weight table is a
// broadcast.  Used when the bins fit (nbins * 8 B * 32 threads); otherwise
// the warp-per-pixel k_vote_refine runs.
__global__ void k_make_vmap(const float* __restrict__ cd, const uint8_t* __restrict__ cv,
                            const uint8_t* __restrict__ gray, size_t n, uint32_t* __restrict__ vmap) {
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t g = gray ? uint32_t(gray[i]) << 16 : 0u;
    vmap[i] = cv[i] ? (g | (1u << 24) | uint32_t(llround(double(cd[i])))) : g;
}

// ---------------------------------------------------------------------------
// K6'' -- voting refinement with device-computed weights.  vote_weight
// (refine.hpp:30-35) = exp(-(double(lab_sad)/lc + sqrt(dx^2+dy^2)/le)):
// lab_sad in float (same association), the divisions and the sum in IEEE
// double, and exp by a restatement of glibc's e_exp.c (FMA build) whose
// table and constants come from the host's libm and were validated bit for
// bit against it (bsmh::glibc_exp_params).  sqrt(s)/le depends only on the
// warp-uniform window offset and comes from a small host table.  Thread per
// invalid pixel, own column of double bins in shared memory; per bin the adds
// follow the reference's row-major voter order.
struct ExpDev {
    double invln2N, shift, negln2hiN, negln2loN, c2, c3, c4, c5;
};

__device__ __forceinline__ double exp_glibc(double x, const ExpDev& p, const unsigned long long* tab) {
    // e_exp.c: |x| < 2^-54 -> 1 + x;  |x| >= 1024 -> 0 / inf;  512 <= |x| < 1024
    // -> specialcase (the scale is built with a biased exponent).
    const unsigned long long xb = static_cast<unsigned long long>(__double_as_longlong(x));
    const unsigned abstop = unsigned(xb >> 52) & 0x7ffu;
    bool special = false;
    if (abstop - 0x3c9u >= 0x3fu) {
        if (int(abstop) - 0x3c9 < 0) return 1.0 + x;
        if (abstop >= 0x409u) return (xb >> 63) ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
        special = true;
    }
    double kd = fma(x, p.invln2N, p.shift);
    const unsigned long long ki = static_cast<unsigned long long>(__double_as_longlong(kd));
    kd -= p.shift;
    const double r = fma(kd, p.negln2loN, fma(kd, p.negln2hiN, x));
    const unsigned idx = 2u * unsigned(ki & 127ull);
    const unsigned long long top = ki << 45;
    const double tail = __longlong_as_double(static_cast<long long>(tab[idx]));
    unsigned long long sbits = tab[idx + 1] + top;
    const double r2 = r * r;
    const double tmp = fma(r2 * r2, fma(r, p.c5, p.c4), fma(fma(r, p.c3, p.c2), r2, tail + r));
    if (!special) {
        const double scale = __longlong_as_double(static_cast<long long>(sbits));
        return fma(scale, tmp, scale);
    }
    if (!(ki & 0x80000000ull)) {  // k > 0 (x >= 512): overflow range
        sbits -= 1009ull << 52;
        const double scale = __longlong_as_double(static_cast<long long>(sbits));
        return 0x1p1009 * __dadd_rn(scale, __dmul_rn(scale, tmp));
    }
    sbits += 1022ull << 52;  // k < 0: subnormal range, rounded once
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    const double st = __dmul_rn(scale, tmp);
    double y = __dadd_rn(scale, st);
    if (y < 1.0) {
        const double hi = __dadd_rn(y, 1.0);
        const double lo = __dadd_rn(__dsub_rn(scale, y), st);
        const double l2 = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo);
        y = __dsub_rn(__dadd_rn(l2, hi), 1.0);
        if (y == 0.0) y = 0.0;
    }
    return __dmul_rn(y, 0x1p-1022);
}

// K6d -- voting refinement, NP invalid pixels per warp (LPP = 32/NP lanes
// each).  Per window row the LPP lanes of a pixel form the bins and weights of
// LPP consecutive voters in parallel (weight from the exact host table, or
// the device exp for Lab planes; the loads of a batch of CB chunks are issued
// together), stage them, then fold them in voter order: lane sl owns the bins
// b with (b % LPP) == sl, finds its entries of the chunk from ballots of the
// valid flag and the residue bits, and walks them in order, keeping its
// current bin's running sum in a register.  Per bin the additions are
// therefore the reference's row-major sequence; the NP pixels fold side by
// side.
template <int NP, bool DEVEXP, bool PEER>
__global__ void __launch_bounds__(256, 1) k_vote_refine_fold(
    const uint32_t* __restrict__ vmap, const float4* __restrict__ lab, const float* __restrict__ lab256, int W,
    int rows, int radius, double lc, const double* __restrict__ e_over_le, ExpDev ep,
    const unsigned long long* __restrict__ etab, const double* __restrict__ wtab, int ncol,
    const int16_t* __restrict__ s2col, const int* __restrict__ counters, const int* __restrict__ inv, int nbins_cap,
    float* __restrict__ od, uint8_t* __restrict__ ov, int* __restrict__ work, const PeerOut po) {
    constexpr int LPP = 32 / NP;
    extern __shared__ __align__(16) double fsm[];
    unsigned long long* stab = reinterpret_cast<unsigned long long*>(fsm);  // 256 (DEVEXP)
    float* slab = reinterpret_cast<float*>(stab + 256);                     // 768 (DEVEXP, gray)
    const int nwarps = blockDim.x >> 5;
    // [warps][32] staged weights; the exp table and gray Lab rows only with DEVEXP
    // (without them a CTA fits four per SM: 32 instead of 24 warps)
    double* sw_all = DEVEXP ? reinterpret_cast<double*>(slab + 768) : fsm;
    int* sb_all = reinterpret_cast<int*>(sw_all + nwarps * 32);             // [warps][32] staged bins
    double* bins_all = reinterpret_cast<double*>(sb_all + nwarps * 32);     // [warps][NP][nbins_cap]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / LPP, sl = lane % LPP;
    if (DEVEXP) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) stab[i] = etab[i];
        if (!lab)
            for (int i = threadIdx.x; i < 768; i += blockDim.x) slab[i] = lab256[i];
    }
    __syncthreads();
    double* sw = sw_all + warp * 32;
    int* sbn = sb_all + warp * 32;
    double* bins = bins_all + size_t(warp * NP + sub) * nbins_cap;
    const unsigned full = 0xFFFFFFFFu;
    const unsigned submask = (LPP == 32) ? full : (((1u << LPP) - 1u) << (sub * LPP));
    const int max_bin = counters[0];
    const int n_inv = counters[1];
    // groups of NP pixels are taken from a work counter (*work == 0 at
    // launch): the voter count varies per pixel, so a static stride leaves a tail
    auto grab = [&]() {
        int b = 0;
        if (lane == 0) b = atomicAdd(work, NP);
        return __shfl_sync(0xFFFFFFFFu, b, 0);
    };
    for (int base = grab(); base < n_inv; base = grab()) {  // warp-uniform loop
        const int idx = base + sub;
        const bool live = idx < n_inv;
        const int p = live ? inv[idx] : 0;
        const int y = p / W, x = p - y * W;
        const uint32_t e0 = vmap[p];
        const int u = int((e0 >> 16) & 0xFFu);
        float lx0 = 0.f, lx1 = 0.f, lx2 = 0.f;
        if (DEVEXP) {
            if (lab) {
                const float4 c = lab[p];
                lx0 = c.x;
                lx1 = c.y;
                lx2 = c.z;
            } else {
                lx0 = slab[3 * u];
                lx1 = slab[3 * u + 1];
                lx2 = slab[3 * u + 2];
            }
        }
        for (int b = sl; b <= max_bin; b += LPP) bins[b] = 0.0;
        int cur = -1;
        double acc = 0.0;
        bool any = false;
        const int tu = u * (u + 1) / 2;
        // Per window row, the loads of CB chunks (LPP voters each) are issued
        // together (vmap, then the weights), then the chunks fold in order:
        // one L2 round trip per batch instead of one per chunk.
        constexpr int CB = 6;
        const int nch = (2 * radius + LPP) / LPP;  // ceil((2r + 1) / LPP)
        for (int dy = -radius; dy <= radius; ++dy) {
            const int py = y + dy;
            const bool rowok = live && py >= 0 && py < rows;
            const uint32_t* row = vmap + size_t(rowok ? py : 0) * W;
            const int dy2 = dy * dy;
            for (int c0 = 0; c0 < nch; c0 += CB) {
                uint32_t ev[CB];
#pragma unroll
                for (int k = 0; k < CB; ++k) {
                    const int dx = -radius + (c0 + k) * LPP + sl;
                    const int px = x + dx;
                    ev[k] = (rowok && dx <= radius && px >= 0 && px < W) ? __ldg(row + px) : 0u;
                }
                int bv[CB];
                double wv[CB];
#pragma unroll
                for (int k = 0; k < CB; ++k) {
                    const uint32_t e = ev[k];
                    const int dx = -radius + (c0 + k) * LPP + sl;
                    bv[k] = -1;
                    wv[k] = 0.0;
                    if (e & (1u << 24)) {
                        bv[k] = int(e & 0xFFFFu);
                        const int v = int((e >> 16) & 0xFFu);
                        if (DEVEXP) {
                            float l0, l1, l2;
                            if (lab) {
                                const float4 o = __ldg(lab + size_t(py) * W + x + dx);
                                l0 = o.x;
                                l1 = o.y;
                                l2 = o.z;
                            } else {
                                l0 = slab[3 * v];
                                l1 = slab[3 * v + 1];
                                l2 = slab[3 * v + 2];
                            }
                            const float sad = __fadd_rn(__fadd_rn(fabsf(__fsub_rn(lx0, l0)), fabsf(__fsub_rn(lx1, l1))),
                                                        fabsf(__fsub_rn(lx2, l2)));
                            const double arg = -(__ddiv_rn(double(sad), lc) + __ldg(e_over_le + dx * dx + dy2));
                            wv[k] = exp_glibc(arg, ep, stab);
                        } else {
                            const int tri = v >= u ? (v * (v + 1) / 2 + u) : (tu + v);
                            wv[k] = __ldg(wtab + size_t(tri) * ncol + s2col[dx * dx + dy2]);
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < CB; ++k) {
                    if (c0 + k >= nch) break;  // warp-uniform
                    const int bin = bv[k];
                    const double w = wv[k];
                    // owner lane of bin b: b % LPP; the entries each owner
                    // takes come from four ballots (valid + residue bits)
                    const unsigned vb = __ballot_sync(full, bin >= 0) & submask;
                    unsigned mine = vb >> (sub * LPP);
#pragma unroll
                    for (int kb = 0; (1 << kb) < LPP; ++kb) {
                        const unsigned bk = __ballot_sync(full, (bin >> kb) & 1) >> (sub * LPP);
                        mine &= ((sl >> kb) & 1) ? bk : ~bk;
                    }
                    any |= vb != 0u;
                    sbn[lane] = bin;
                    sw[lane] = w;
                    __syncwarp();
                    while (mine) {
                        const int j = sub * LPP + __ffs(mine) - 1;
                        mine &= mine - 1;
                        const int b = sbn[j];
                        if (b != cur) {
                            if (cur >= 0) bins[cur] = acc;
                            cur = b;
                            acc = bins[b];
                        }
                        acc += sw[j];
                    }
                    __syncwarp();
                }
            }
        }
        if (cur >= 0) bins[cur] = acc;
        __syncwarp();
        // argmax: strict '>' from bin 0 == first bin holding the maximum
        double bv = -1.0;
        int bb = 0x7FFFFFFF;
        for (int b = sl; b <= max_bin; b += LPP)
            if (bins[b] > bv) {
                bv = bins[b];
                bb = b;
            }
#pragma unroll
        for (int o = LPP / 2; o > 0; o >>= 1) {
            const double ov2 = __shfl_xor_sync(full, bv, o);
            const int ob = __shfl_xor_sync(full, bb, o);
            if (ov2 > bv || (ov2 == bv && ob < bb)) {
                bv = ov2;
                bb = ob;
            }
        }
        if (live && sl == 0) {
            od[p] = any ? float(bb) : 0.0f;
            ov[p] = any ? 1 : 0;
            peer_store<PEER>(po, p, any ? float(bb) : 0.0f, any ? 1 : 0);
        }
        __syncwarp();
    }
}

__global__ void k_exp_eval(const double* __restrict__ x, int n, ExpDev ep, const unsigned long long* __restrict__ tab,
                           double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = exp_glibc(x[i], ep, tab);
}
