// bsm/pipeline.hpp -- run_pipeline (reference pipeline.hpp:14-61): the fused
// device pipeline behind one C-ABI call (bsm_pipeline_u8 / bsm_pipeline_rgb).
#pragma once

#include <optional>

#include "../bsm_cuda.h"
#include "bsm/config.hpp"
#include "bsm/descriptor.hpp"
#include "bsm/detail_cabi.hpp"
#include "bsm/errors.hpp"
#include "bsm/image.hpp"
#include "bsm/matcher.hpp"
#include "bsm/refine.hpp"

namespace bsm {

struct PipelineResult {
    DisparityMap refined;
    DisparityMap left_wta;
    DisparityMap right_wta;
    DisparityMap checked;
    std::optional<DisparityMap> unmasked;
};

inline PipelineResult run_pipeline(const RgbImage& left, const RgbImage& right, const SamplingPattern& pattern,
                                   const BsmConfig& cfg, bool want_unmasked = false) {
    if (left.width != right.width || left.height != right.height)
        throw DimensionMismatch("pipeline: left/right dimensions differ");
    cfg.validate();
    const auto L = detail::gray_view(left);
    const auto R = L ? detail::gray_view(right) : std::nullopt;
    detail::Context& ctx = detail::context();
    ctx.use_pattern(detail::flat_pairs(pattern), pattern.n, pattern.window);
    const int W = left.width, H = left.height;
    PipelineResult res{DisparityMap(W, H), DisparityMap(W, H), DisparityMap(W, H), DisparityMap(W, H), {}};
    if (want_unmasked) res.unmasked = DisparityMap(W, H);
    bsm_params p{cfg.d_max, cfg.lambda_c, cfg.lambda_e, cfg.lr_tolerance, cfg.vote_radius};
    bsm_maps m{res.refined.disparity.data(), res.refined.valid.data(), res.left_wta.disparity.data(),
               res.right_wta.disparity.data(), res.checked.disparity.data(), res.checked.valid.data(),
               want_unmasked ? res.unmasked->disparity.data() : nullptr};
    if (L && R) {
        detail::throw_status(bsm_pipeline_u8(ctx.get(), L->data(), R->data(), W, H, &p, want_unmasked ? 1 : 0, &m));
    } else {  // colour: interleaved RGB through the exact 2^24-colour tables
        static_assert(sizeof(Rgb8) == 3, "Rgb8 must be three packed bytes");
        detail::throw_status(bsm_pipeline_rgb(ctx.get(), &left.pixels[0].r, &right.pixels[0].r, W, H, &p,
                                              want_unmasked ? 1 : 0, &m));
    }
    return res;
}

inline PipelineResult run_pipeline(const RgbImage& left, const RgbImage& right, const BsmConfig& cfg,
                                   bool want_unmasked = false) {
    return run_pipeline(left, right, generate_pattern(cfg), cfg, want_unmasked);
}

}  // namespace bsm
