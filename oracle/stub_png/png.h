/* oracle/stub_png/png.h -- TEST INFRASTRUCTURE ONLY.
 *
 * libpng is not installed in this image.  This header declares just the
 * simplified-API names the reference's image_io.hpp refers to, so that its
 * PNM/PFM readers and writers can be compiled in place as an oracle.  The
 * matching definitions in oracle/ref_io_driver.cpp always fail, so every PNG
 * path of that oracle throws FormatError; PNG decoding is checked against the
 * reference's own test vectors instead (tests/test_io.py). */
#ifndef BSM_ORACLE_STUB_PNG_H
#define BSM_ORACLE_STUB_PNG_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef struct {
    void* opaque;
    uint32_t version, width, height, format, flags, colormap_entries, warning_or_error;
    char message[64];
} png_image;
typedef png_image* png_imagep;
#define PNG_IMAGE_VERSION 1
#define PNG_FORMAT_GRAY 0u
#define PNG_FORMAT_RGB 2u
#define PNG_IMAGE_SIZE(im) ((size_t)(im).width * (size_t)(im).height * ((im).format == PNG_FORMAT_RGB ? 3u : 1u))
int png_image_begin_read_from_memory(png_imagep image, const void* memory, size_t size);
int png_image_finish_read(png_imagep image, const void* background, void* buffer, int32_t row_stride,
                          void* colormap);
void png_image_free(png_imagep image);
#ifdef __cplusplus
}
#endif
#endif
