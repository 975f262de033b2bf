/* tests/cpp/capi_multi.c -- a plain C client of include/bsm_cuda.h (no C++,
 * no PyTorch): the batch entry point and the NCCL partitions (one rank),
 * as a C / cgo / JNI caller of the drop-in would use them.
 *
 *   capi_multi W H D pairs.raw out.bin
 * pairs.raw: N pairs of (left, right) W*H uint8 views back to back (N from the
 * file size).  out.bin: the batch's N refined maps (float W*H then uint8 W*H
 * each), then the frame-band result of pair 0, then the sharded-pairs result
 * of every pair, then the peer-memory frame-band result of pair 1, in the same
 * format.  Exit status: 0 ok, else the failing
 * call's status. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "bsm_cuda.h"

#define TRY(x)                                                                  \
    do {                                                                        \
        int rc_ = (x);                                                          \
        if (rc_ != BSM_OK) {                                                    \
            fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, bsm_last_error()); \
            return rc_;                                                         \
        }                                                                       \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 6) {
        fprintf(stderr, "usage: capi_multi W H D pairs.raw out.bin\n");
        return 64;
    }
    const int W = atoi(argv[1]), H = atoi(argv[2]), D = atoi(argv[3]);
    const size_t px = (size_t)W * H;
    FILE* f = fopen(argv[4], "rb");
    if (!f) return 65;
    fseek(f, 0, SEEK_END);
    const long bytes = ftell(f);
    fseek(f, 0, SEEK_SET);
    const int n = (int)(bytes / (long)(2 * px));
    uint8_t* views = malloc((size_t)bytes);
    if (fread(views, 1, (size_t)bytes, f) != (size_t)bytes) return 66;
    fclose(f);

    bsm_ctx* ctx = NULL;
    TRY(bsm_ctx_create(0, &ctx));
    int16_t* pairs = malloc(4096 * 4 * sizeof(int16_t));
    TRY(bsm_generate_pattern(4096, 26, 4.0, 42, pairs));
    TRY(bsm_set_pattern(ctx, pairs, 4096, 26));
    bsm_params p = {D, 9.0, 16.0, 1.0, 20};

    const uint8_t** lefts = malloc(sizeof(uint8_t*) * (size_t)n);
    const uint8_t** rights = malloc(sizeof(uint8_t*) * (size_t)n);
    float** od = malloc(sizeof(float*) * (size_t)n);
    uint8_t** ov = malloc(sizeof(uint8_t*) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        lefts[i] = views + (size_t)(2 * i) * px;
        rights[i] = views + (size_t)(2 * i + 1) * px;
        od[i] = malloc(px * 4);
        ov[i] = malloc(px);
    }
    FILE* o = fopen(argv[5], "wb");
    if (!o) return 67;
    TRY(bsm_pipeline_batch_u8(ctx, n, lefts, rights, W, H, &p, od, ov));
    for (int i = 0; i < n; ++i) {
        fwrite(od[i], 4, px, o);
        fwrite(ov[i], 1, px, o);
    }
    uint8_t id[128];
    bsm_comm* comm = NULL;
    TRY(bsm_comm_unique_id(id));
    TRY(bsm_comm_create(ctx, id, 1, 0, &comm));
    TRY(bsm_pipeline_frame_bands_u8(ctx, comm, lefts[0], rights[0], W, H, &p, od[0], ov[0]));
    fwrite(od[0], 4, px, o);
    fwrite(ov[0], 1, px, o);
    TRY(bsm_pipeline_pairs_sharded_u8(ctx, comm, n, lefts, rights, W, H, &p, 0, od, ov));
    for (int i = 0; i < n; ++i) {
        fwrite(od[i], 4, px, o);
        fwrite(ov[i], 1, px, o);
    }
    /* peer-memory frame bands at world 1: the band is the whole frame */
    bsm_frame* frame = NULL;
    uint8_t handle[128];
    TRY(bsm_frame_create(ctx, W, H, 1, 0, &frame, handle));
    TRY(bsm_frame_attach(frame, handle));
    TRY(bsm_pipeline_frame_bands_p2p_u8(ctx, frame, lefts[1], rights[1], &p));
    TRY(bsm_frame_fetch(frame, od[1], ov[1]));
    fwrite(od[1], 4, px, o);
    fwrite(ov[1], 1, px, o);
    TRY(bsm_frame_destroy(frame));
    fclose(o);
    TRY(bsm_comm_destroy(comm));
    TRY(bsm_ctx_destroy(ctx));
    return 0;
}
