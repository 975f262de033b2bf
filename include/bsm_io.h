/*
 * bsm_io.h -- C ABI of the host-side file and evaluation layer either side of
 * the matching path: image / disparity files
 * (reference image_io.hpp:238-382), the JSON config and pattern sidecars
 * (config.hpp:81-110, pattern.hpp:104-160) and the evaluation helpers
 * (eval.hpp:31-185).  Implemented once, by this repository's C++ drop-in
 * headers (include/bsm/), in paper_1402_2020_b200/libbsm_io.so; the Python
 * modules io.py / evaluation.py and any other FFI bind these entry points.
 *
 * Status: 0 ok, 1 InvalidArgument, 2 DimensionMismatch, 9 other error,
 * 10 IoError, 11 FormatError, 12 EmptyRegion; bsmio_last_error() holds the
 * thread-local message (the reference's text).  Images are interleaved RGB
 * bytes (gray sources expand to r = g = b); maps are float + uint8 valid.
 * Readers: call once with NULL outputs for the dimensions, then again with
 * buffers (the second call reuses the first call's decode).
 */
#ifndef BSM_IO_H
#define BSM_IO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* bsmio_last_error(void);
int bsmio_load_image(const char* path, int* w, int* h, uint8_t* rgb);
int bsmio_load_gt(const char* path, double scale, int* w, int* h, float* d, uint8_t* v);
int bsmio_save_disparity(const char* path, const float* d, const uint8_t* v, int W, int H, double scale, int pfm);
int bsmio_save_gray_pgm(const char* path, const float* g, int W, int H);
int bsmio_save_ppm(const char* path, const uint8_t* rgb, int W, int H);
/* iv: n, S, seed, d_max, vote_radius, threads; dv: spread, lambda_c, lambda_e, lr_tolerance, gt_scale */
int bsmio_save_config(const char* path, const int64_t* iv, const double* dv, const char* generator);
int bsmio_load_config(const char* path, int64_t* iv, double* dv, char* generator, int gen_cap);
int bsmio_save_pattern(const char* path, const int16_t* pairs, int n, int window, double spread, uint64_t seed);
int bsmio_load_pattern(const char* path, int* n, int* window, double* spread, uint64_t* seed, int16_t* pairs,
                       int cap);
int bsmio_bad_pixel_rate(const float* d, const uint8_t* v, const float* gd, const uint8_t* gv, const float* region,
                         int W, int H, double threshold, double* rate, long* counted, long* bad);
int bsmio_linear_fit_r2(const double* xs, const double* ys, int n, double* out);
int bsmio_write_sweep_csv(const char* path, const int* n, const double* err, const double* secs, int count);
/* rate9: row-major 3x3 bad-pixel rates; path may be NULL (means only) */
int bsmio_write_radiometric_csv(const char* path, const double* rate9, double* diag, double* off);

#ifdef __cplusplus
}
#endif
#endif /* BSM_IO_H */
