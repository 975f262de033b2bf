// bsm_host.h -- host-side pieces of the product library that stay on the CPU
// (SURVEY.md section 8(a) rows R2-R4, R9, R18/R19): the sampling pattern, the
// 256-entry colour-conversion tables, the per-centre rank table the mask
// kernel selects over, and the exact vote-weight table.  Compiled by g++ with
// FP contraction on (bsm_host.cpp), so its floating point matches the
// reference's default -O3 -march=native build.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace bsmh {

// pattern.hpp:74-103.  Returns false (and sets err) on invalid arguments.
bool generate_pattern(int n, int window, double spread, uint64_t seed, int16_t* out, std::string& err);

// image.hpp:90-140 for (v,v,v).
void gray_lab_lut(float* gray256, float* lab768);

// Per-pixel to_gray / to_lab of interleaved RGB (image.hpp:90-140).
void to_gray_lab(const uint8_t* rgb, size_t npx, float* gray, float* lab);

// The same conversions for all 2^24 colours, index (r << 16) | (g << 8) | b
// (gray: 64 MiB, Lab: 192 MiB); multithreaded, built once per context.
void rgb24_tables(std::vector<float>& gray, std::vector<float>& lab);

// rank[c*256 + v] = dense rank of lab_sad(Lab[c], Lab[v]) among the 256 values
// of row c (equal values share a rank).  lab_sad: image.hpp:144-146.
void sad_rank_table(const float* lab768, uint8_t* rank65536);

// Exact refine weights (refine.hpp:30-35) for grayscale views:
//   w[tri(u,v) * ncol + col(s)] = exp(-(double(lab_sad(u,v)) / lc + sqrt(s) / le))
// for every gray pair u <= v (tri(u,v) = v*(v+1)/2 + u) and every distinct
// squared offset s = dx^2 + dy^2 with |dx|,|dy| <= radius.  s2col has
// 2*radius^2 + 1 entries (-1 where s is not a sum of two squares in range).
void vote_weight_table(const float* lab768, double lc, double le, int radius, std::vector<double>& w,
                       std::vector<int16_t>& s2col, int& ncol);

}  // namespace bsmh

namespace bsmh {

// Shared-memory bank placement for the mask kernel's per-warp rank table.
// Pair i's endpoints are used-offset indices P[i], Q[i] (< u).  In k_mask4 lane
// l reads pair 128l + 32m + t at step (m, t); a 32-lane gather costs as many
// shared-memory wavefronts as the largest number of distinct 4-byte slots
// requested from one bank.  Returns slot[o] for every used offset o (slots are
// a permutation of [0, nslots) restricted to u entries, nslots >= u) chosen by
// a deterministic local search that minimises the total wavefront count.
// `cost_before` / `cost_after` receive the average wavefronts per gather.
void place_rank_slots(const uint32_t* pq, int n, int u, int nslots, int lane_pos, std::vector<int>& slot,
                      double* cost_before, double* cost_after);

// Conflict-free gather order for n = 32 S, S in {32, 64, 128, 256} positions per
// lane (k_mask4 / k_mask_f32): offsets are spread over the 32 shared-memory
// banks with exactly 2S endpoint references per bank, the pairs are oriented
// along Eulerian walks of the bank multigraph (each bank: S "A" ends, S "B"
// ends) and the resulting S-regular bipartite multigraph is split into S
// perfect matchings.  Position j = S l + st holds pair order[j]; its A end
// lies in bank l and the B ends of one step st lie in 32 distinct banks, so
// every 32-lane gather is a single wavefront.  flip[j] = 1 when the A end is
// the pair's q.
// Returns false (outputs unspecified) when no such order was found.
bool balanced_gather_order(const uint32_t* pq, int n, int u, std::vector<int>& slot, int& nslots,
                           std::vector<int>& order, std::vector<uint8_t>& flip);

}  // namespace bsmh

namespace bsmh {

// glibc's exp (sysdeps/ieee754/dbl-64/e_exp.c, FMA variant selected on
// x86-64 CPUs with FMA+AVX2), restated so the device can reproduce
// vote_weight's std::exp (refine.hpp:34) bit for bit.  The table and
// constants are read from the libm the process runs with and the restatement
// is validated against that libm's exp before use.
struct ExpParams {
    double invln2N, shift, negln2hiN, negln2loN, c2, c3, c4, c5;
    uint64_t tab[256];
};
// True when the parameters were found and the restatement matched libm's exp
// on every validation argument; `why` explains a false return.
bool glibc_exp_params(ExpParams& p, std::string& why);
// Host restatement (for tests / validation).
double exp_restated(double x, const ExpParams& p);

}  // namespace bsmh
