// bsm/refine.hpp -- left/right check and bilateral voting refinement
// (reference refine.hpp:13-111), both on the GPU (bsm_lr_check,
// bsm_vote_refine_u8).  vote_weight is the scalar host formula.
#pragma once

#include <cmath>

#include "../bsm_cuda.h"
#include "bsm/detail_cabi.hpp"
#include "bsm/errors.hpp"
#include "bsm/image.hpp"

namespace bsm {

struct RefineParams {
    double lambda_c = 9.0;
    double lambda_e = 16.0;
    double lr_tolerance = 1.0;
    int vote_radius = 20;
    void validate() const {
        if (!(lambda_c > 0)) throw InvalidArgument("refine: lambda_c must be > 0");
        if (!(lambda_e > 0)) throw InvalidArgument("refine: lambda_e must be > 0");
        if (lr_tolerance < 0) throw InvalidArgument("refine: lr_tolerance must be >= 0");
        if (vote_radius < 1) throw InvalidArgument("refine: vote_radius must be >= 1");
    }
};

inline double vote_weight(const Lab& at_x, const Lab& at_p, int dx, int dy, double lambda_c, double lambda_e) {
    const double c = double(lab_sad(at_x, at_p));
    const double e = std::sqrt(double(dx) * dx + double(dy) * dy);
    return std::exp(-(c / lambda_c + e / lambda_e));
}

inline DisparityMap lr_check(const DisparityMap& left, const DisparityMap& right, double tol) {
    if (left.width != right.width || left.height != right.height)
        throw DimensionMismatch("lr_check: map dimensions differ");
    DisparityMap out(left.width, left.height);
    detail::throw_status(bsm_lr_check(detail::context().get(), left.disparity.data(), right.disparity.data(),
                                      left.width, left.height, tol, out.disparity.data(), out.valid.data()));
    return out;
}

inline DisparityMap vote_refine(const DisparityMap& map, const LabImage& lab, const RefineParams& params,
                                int threads = 1) {
    (void)threads;
    if (map.width != lab.width || map.height != lab.height)
        throw DimensionMismatch("vote_refine: map/image dimensions differ");
    params.validate();
    const auto u8 = detail::u8_from_planes(nullptr, &lab);
    DisparityMap out(map.width, map.height);
    if (!u8) {
        detail::throw_status(bsm_vote_refine_lab(detail::context().get(), map.disparity.data(), map.valid.data(),
                                                 &lab.values[0].l, map.width, map.height, params.lambda_c,
                                                 params.lambda_e, params.vote_radius, out.disparity.data(),
                                                 out.valid.data()));
        return out;
    }
    detail::throw_status(bsm_vote_refine_u8(detail::context().get(), map.disparity.data(), map.valid.data(),
                                            u8->data(), map.width, map.height, params.lambda_c, params.lambda_e,
                                            params.vote_radius, out.disparity.data(), out.valid.data()));
    return out;
}

}  // namespace bsm
