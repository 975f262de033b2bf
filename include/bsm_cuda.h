/*
 * bsm_cuda.h -- C ABI of the B200-native Binary Stereo Matching hot path.
 *
 * The drop-in boundary for the reference library's hot path
 * (/root/reference/proj/include/bsm, a header-only C++20 library with no FFI of
 * its own).  Every entry point below replaces one reference function; the C++
 * shim in include/bsm/ re-exposes them under the reference's own names and
 * signatures, and a ctypes / cgo / JNI binding can bind them directly
 * (INTEGRATION.md).  Plain pointers and sizes only; no torch or CUDA types.
 *
 * Conventions
 *  - Host buffers are caller-owned; any OUTPUT pointer may be NULL to skip it.
 *  - Bit strings use the reference layout: bit i in 64-bit word i>>6 at
 *    position i&63, pad bits zero (bitstring.hpp:21-23,47-51); fields are AoS
 *    with index ((y*W + x) * words64) (descriptor.hpp:48-50).
 *  - Disparity maps are float disparity + uint8 valid (image.hpp:243-263).
 *  - Return value: BSM_OK or an error code; bsm_last_error() holds the
 *    thread-local message (the reference's exception text where one exists).
 *  - Device work runs on the context's own stream; a context is re-entrant
 *    but not shared between threads without external locking.
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    entry point returns BSM_CUDA_ERROR.
 */
#ifndef BSM_CUDA_H
#define BSM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes -> reference exception types (errors.hpp:8-34). */
enum {
    BSM_OK = 0,
    BSM_INVALID_ARGUMENT = 1,   /* bsm::InvalidArgument */
    BSM_DIMENSION_MISMATCH = 2, /* bsm::DimensionMismatch */
    BSM_CUDA_ERROR = 3,         /* device failure / no device */
    BSM_UNSUPPORTED = 4,        /* valid input outside this build's envelope */
    BSM_NCCL_ERROR = 5
};

typedef struct bsm_ctx bsm_ctx;

/* Pipeline parameters: the BsmConfig fields run_pipeline reads
 * (config.hpp:16-28, pipeline.hpp:150-167). */
typedef struct {
    int d_max;            /* hypotheses d in [0, d_max - 1]; no default (config.hpp:14-15) */
    double lambda_c;      /* 9.0 */
    double lambda_e;      /* 16.0 */
    double lr_tolerance;  /* 1.0 */
    int vote_radius;      /* 20 */
} bsm_params;

/* PipelineResult (pipeline.hpp:14-20); every member optional. */
typedef struct {
    float* refined_d;
    uint8_t* refined_v;
    float* left_d;     /* left_wta (all valid) */
    float* right_d;    /* right_wta (all valid) */
    float* checked_d;
    uint8_t* checked_v;
    float* unmasked_d; /* only when want_unmasked */
} bsm_maps;

const char* bsm_last_error(void);
const char* bsm_version(void);

/* Context: owns a device, a stream, the uploaded pattern and scratch. */
int bsm_ctx_create(int device, bsm_ctx** out);
int bsm_ctx_destroy(bsm_ctx* ctx);

/* generate_pattern(n, window, spread, seed) (pattern.hpp:74-103); host-side,
 * out_pairs = n x {px, py, qx, qy}. */
int bsm_generate_pattern(int n, int window, double spread, uint64_t seed, int16_t* out_pairs);

/* Upload a SamplingPattern (pattern.hpp:62-72).  |offset| <= window/2. */
int bsm_set_pattern(bsm_ctx* ctx, const int16_t* pairs, int n, int window);

/* to_gray / to_lab of the gray pixel (v,v,v), v = 0..255 (image.hpp:90-140). */
int bsm_gray_lab_lut(float* gray256, float* lab768);

/* to_gray / to_lab (image.hpp:90-140) of an interleaved RGB image, host-side
 * (floating point compiled like the reference); gray / lab may be NULL. */
int bsm_to_gray_lab(const uint8_t* rgb, int W, int H, float* gray, float* lab);

/* compute_field (descriptor.hpp:200-239) of a grayscale view (r=g=b=img).
 * desc/mask: W*H*words64 uint64 each, AoS. */
int bsm_compute_field_u8(bsm_ctx* ctx, const uint8_t* img, int W, int H, uint64_t* desc, uint64_t* mask);

/* wta (matcher.hpp:80-113) over AoS fields with the context's pattern length n.
 * right_ref = 0: RefView::left (x - d); 1: RefView::right (x + d). */
int bsm_wta(bsm_ctx* ctx, const uint64_t* desc_ref, const uint64_t* mask_ref, const uint64_t* desc_other,
            int W, int H, int n, int d_max, int right_ref, int use_mask, float* out_d);

/* lr_check (refine.hpp:39-54); input validity is ignored, as in the reference. */
int bsm_lr_check(bsm_ctx* ctx, const float* left_d, const float* right_d, int W, int H, double tol,
                 float* out_d, uint8_t* out_v);

/* vote_refine (refine.hpp:62-111) with the Lab image of a grayscale view. */
int bsm_vote_refine_u8(bsm_ctx* ctx, const float* d, const uint8_t* v, const uint8_t* gray_img, int W, int H,
                       double lambda_c, double lambda_e, int vote_radius, float* out_d, uint8_t* out_v);

/* vote_refine (refine.hpp:62-111) with an arbitrary float Lab plane
 * (W*H*3 floats, e.g. from bsm_to_gray_lab of a colour image). */
int bsm_vote_refine_lab(bsm_ctx* ctx, const float* d, const uint8_t* v, const float* lab, int W, int H,
                        double lambda_c, double lambda_e, int vote_radius, float* out_d, uint8_t* out_v);

/* compute_field (descriptor.hpp:200-239) of arbitrary float planes (a
 * GrayImage and a LabImage, e.g. of a colour view). */
int bsm_compute_field_f32(bsm_ctx* ctx, const float* gray, const float* lab, int W, int H, uint64_t* desc,
                          uint64_t* mask);

/* run_pipeline (pipeline.hpp:25-56) of a colour pair: interleaved RGB, 3 bytes
 * per pixel (to_gray / to_lab through exact 2^24-entry tables). */
int bsm_pipeline_rgb(bsm_ctx* ctx, const uint8_t* left_rgb, const uint8_t* right_rgb, int W, int H,
                     const bsm_params* params, int want_unmasked, bsm_maps* out);

/* bsm_pipeline_rgb on device-resident interleaved-RGB views (serving path;
 * results stay on the device: bsm_fetch_maps / bsm_result_device). */
int bsm_pipeline_rgb_device(bsm_ctx* ctx, const uint8_t* d_left_rgb, const uint8_t* d_right_rgb, int W, int H,
                            const bsm_params* params, int want_unmasked);

/* to_gray / to_lab of all 2^24 colours, index (r<<16)|(g<<8)|b (host). */
int bsm_rgb24_tables(float* gray16M, float* lab48M);

/* run_pipeline (pipeline.hpp:25-56) of a grayscale pair (r=g=b), host buffers. */
int bsm_pipeline_u8(bsm_ctx* ctx, const uint8_t* left, const uint8_t* right, int W, int H,
                    const bsm_params* params, int want_unmasked, bsm_maps* out);

/* run_pipeline(...).refined (pipeline.hpp:25-56) of a batch of grayscale pairs
 * (BASELINE configs[3]), host buffers: lefts[i] / rights[i] are W x H views,
 * refined_d[i] / refined_v[i] receive pair i's refined map (either array, or
 * any entry, may be NULL).  Uploads, compute and downloads of consecutive pairs
 * overlap (two device slots, separate copy streams), and each pair's check +
 * refine runs on an internal high-priority stream beside the next pair's
 * descriptor / mask kernels; returns when every map has landed.  Pinned host
 * buffers make the copies asynchronous. */
int bsm_pipeline_batch_u8(bsm_ctx* ctx, int n_pairs, const uint8_t* const* lefts, const uint8_t* const* rights,
                          int W, int H, const bsm_params* params, float* const* refined_d,
                          uint8_t* const* refined_v);
/* Device-resident batch: d_lefts / d_rights / d_refined_* are host arrays of
 * DEVICE pointers; work is queued on bsm_stream() (the internal refine stream
 * is joined back into it before the call returns) and not synchronised. */
int bsm_pipeline_batch_u8_device(bsm_ctx* ctx, int n_pairs, const uint8_t* const* d_lefts,
                                 const uint8_t* const* d_rights, int W, int H, const bsm_params* params,
                                 float* const* d_refined_d, uint8_t* const* d_refined_v);

/* Device-resident variant: left/right are device pointers; results stay on the
 * device in context-owned buffers (read them with bsm_fetch_maps).
 * Device inputs must be complete when the context's stream reaches the call:
 * produce them on bsm_stream(), synchronise, or call bsm_stream_wait() with
 * the producing stream first.  Device pointers must be 4-byte aligned. */
int bsm_pipeline_u8_device(bsm_ctx* ctx, const uint8_t* d_left, const uint8_t* d_right, int W, int H,
                           const bsm_params* params, int want_unmasked);
int bsm_fetch_maps(bsm_ctx* ctx, bsm_maps* out);

/* Multi-GPU row band (c5): compute rows [y0, y1) of the refined map of a
 * W x H pair whose full views are given; the checked map is computed for
 * [y0 - radius, y1 + radius) locally (redundant halo, no exchange).
 * refined_d / refined_v receive (y1 - y0) rows. */
int bsm_pipeline_band_u8(bsm_ctx* ctx, const uint8_t* left, const uint8_t* right, int W, int H, int y0, int y1,
                         const bsm_params* params, float* refined_d, uint8_t* refined_v);

/* Device-resident band: views on the device; read the result with
 * bsm_fetch_maps (refined_d/v only) or bsm_result_device. */
int bsm_pipeline_band_u8_device(bsm_ctx* ctx, const uint8_t* d_left, const uint8_t* d_right, int W, int H, int y0,
                                int y1, const bsm_params* params);
/* Device pointers to the refined rows of the last pipeline/band call (valid
 * until the next call on the context): [row0, row0 + nrows) x W. */
int bsm_result_device(bsm_ctx* ctx, const float** refined_d, const uint8_t** refined_v, int* row0, int* nrows);
/* Stream-ordered device-to-device copy of those rows into caller buffers. */
int bsm_copy_result_device(bsm_ctx* ctx, float* dst_d, uint8_t* dst_v);

/* Multi-GPU partitions over NCCL; one process (and one
 * context) per GPU.  Rank 0 makes an id with bsm_comm_unique_id and hands the
 * 128 bytes to the other ranks out of band (MPI, a file, torch.distributed);
 * every rank then calls bsm_comm_create with its rank.  NCCL is loaded at run
 * time (libnccl.so.2); NCCL failures return BSM_NCCL_ERROR. */
typedef struct bsm_comm bsm_comm;
int bsm_comm_unique_id(uint8_t* id128);
int bsm_comm_create(bsm_ctx* ctx, const uint8_t* id128, int world, int rank, bsm_comm** out);
int bsm_comm_destroy(bsm_comm* comm);
/* One frame (BASELINE configs[4]) partitioned into contiguous row bands:
 * every rank passes the full views, computes its band with a local
 * vote-radius halo (no exchange) and receives the whole refined map through
 * one NCCL all-gather of the bands; bit-identical to run_pipeline(...).refined
 * for every world size (parallel.hpp:12-14). */
int bsm_pipeline_frame_bands_u8(bsm_ctx* ctx, bsm_comm* comm, const uint8_t* left, const uint8_t* right, int W,
                                int H, const bsm_params* params, float* refined_d, uint8_t* refined_v);
/* A batch of pairs (BASELINE configs[3]) sharded by pair: rank r computes the
 * contiguous shard [r*n/world ...) (sizes differ by at most one; only that
 * shard's lefts[i] / rights[i] are read) and the refined maps of ALL pairs
 * land in refined_d[i] / refined_v[i] on rank `root` (ncclSend / ncclRecv;
 * other ranks' output arrays may be NULL). */
int bsm_pipeline_pairs_sharded_u8(bsm_ctx* ctx, bsm_comm* comm, int n_pairs, const uint8_t* const* lefts,
                                  const uint8_t* const* rights, int W, int H, const bsm_params* params, int root,
                                  float* const* refined_d, uint8_t* const* refined_v);

/* One frame over peer memory (configs[4]; the alternative to
 * bsm_pipeline_frame_bands_u8 without a collective launch): each rank creates
 * a full-frame refined map in device memory and exports it (128-byte handle,
 * CUDA IPC); the ranks exchange the handles out of band (rank order) and
 * attach; bsm_pipeline_frame_bands_p2p_u8 computes the rank's row band with
 * its vote-radius halo and its check and refine kernels store the band's
 * final values straight into EVERY rank's map (NVLink P2P stores), returning
 * once this rank's stores have completed.  After a barrier across the ranks
 * (the caller's), bsm_frame_fetch reads the whole refined map on any rank.
 * 1..8 ranks; destroy frames before their context. */
typedef struct bsm_frame bsm_frame;
int bsm_frame_create(bsm_ctx* ctx, int W, int H, int world, int rank, bsm_frame** out, uint8_t* handle128);
int bsm_frame_attach(bsm_frame* frame, const uint8_t* handles /* world x 128 bytes, rank order */);
int bsm_pipeline_frame_bands_p2p_u8(bsm_ctx* ctx, bsm_frame* frame, const uint8_t* left, const uint8_t* right,
                                    const bsm_params* params);
int bsm_frame_fetch(bsm_frame* frame, float* refined_d, uint8_t* refined_v);
int bsm_frame_destroy(bsm_frame* frame);

/* Instrumentation.  bsm_stream returns the cudaStream_t the context launches
 * on.  When profiling is enabled, bsm_last_timings reports the device time (ms)
 * of the last pipeline's kernels, in the order of bsm_timing_names. */
int bsm_stream(bsm_ctx* ctx, void** stream);
/* Order the context's stream after all work queued so far on `stream` (a
 * cudaStream_t of the caller, NULL = the legacy default stream). */
int bsm_stream_wait(bsm_ctx* ctx, void* stream);
int bsm_set_profiling(bsm_ctx* ctx, int enable);
int bsm_last_timings(bsm_ctx* ctx, float* ms, int max, int* count);
const char* bsm_timing_names(void);
/* Test hook: with BSM_GUARD=1 in the environment when the first context is
 * created, every device buffer is bracketed by 4 KiB guards (and its payload
 * pre-filled) with 0xA5; this reports how many guard bytes changed. */
int bsm_debug_check_guards(bsm_ctx* ctx, long long* damaged, int* enabled);
/* Kernel launches issued by the last pipeline call. */
int bsm_last_launch_count(bsm_ctx* ctx, int* count);
/* Measured masked-XOR-popcount word-op throughput of this device (words/s),
 * register-only microbenchmarks of the integer-pipe cost kernel's (K3p,
 * BSM_K3_VARIANT=16) two instruction mixes:
 * direct (LOP3 + POPC + IADD per word) and carry-save (per two words:
 * 4 LOP3 + POPC + IMAD).  Either pointer may be NULL. */
int bsm_measure_popc_peak(bsm_ctx* ctx, double* ops_per_s);
int bsm_measure_word_peaks(bsm_ctx* ctx, double* popc_words_per_s, double* csa_words_per_s);
/* Live dense FP4 tensor peak of this device (tcgen05 kind::mxf4, M128 N256
 * K64, issued back to back), flop/s: the tensor-core cost kernel's roofline. */
int bsm_measure_mma_peak(bsm_ctx* ctx, double* flops_per_s);
/* The device restatement of libm's exp used for refine weights, evaluated on
 * n arguments (validation / tests). */
int bsm_device_exp(bsm_ctx* ctx, const double* x, int n, double* out);
/* Refinement kernel choice (all bit-identical): -1 = auto (3 for grayscale,
 * 4 for Lab planes); 2 = warp per pixel, exact host weight table (grayscale);
 * 3 = four pixels per warp, ordered fold, host weight table (grayscale);
 * 4 = the same fold with the device restatement of libm's exp. */
int bsm_set_refine_mode(bsm_ctx* ctx, int mode);

#ifdef __cplusplus
}
#endif
#endif /* BSM_CUDA_H */
