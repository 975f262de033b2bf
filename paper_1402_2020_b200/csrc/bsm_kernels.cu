// bsm_kernels.cu -- sm_100a kernels and the C ABI (include/bsm_cuda.h) of the
// Binary Stereo Matching hot path.  See DESIGN.md for the data layout, each
// kernel's roofline, and the reference function (file:line) it replaces.
//
// Device layout (per view, W x H, n bits, NW = 2*ceil(n/64) u32 words):
//   field[w*P + y*Wq + x]   word planes ("bit-plane images"), Wq = W rounded up
//   to 4, P = rows*Wq rounded up to 32: for a fixed word the pixels of all rows
//   are one contiguous run, so the cost kernel tiles pixels over the flat
//   index y*Wq + x (no padding of rows to a tile multiple) and stages
//   [K words x span] boxes by TMA (one 2-D tensor map per field, dims (P, NW));
//   every shared-memory read is a conflict-free 16-B lane-contiguous LDS.128.
//   u32 word w of a pixel = bits 32w..32w+31 = the low/high half of the
//   reference's u64 word w>>1 (bitstring.hpp:47-51).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/bsm_cuda.h"
#include "bsm_host.h"

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define BSM_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return set_err(BSM_CUDA_ERROR, std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                               " at " #call);                            \
    } while (0)

constexpr int kMaxPairs = 8192;      // mask kernel keeps 2*ceil(n/128) regs/lane of ranks
constexpr int kCostTile = 128;       // pixels per cost CTA
constexpr int kCostDisp = 64;        // disparities per cost CTA
constexpr int kCostK = 16;           // u32 words per pipeline stage
constexpr int kCostStages = 3;

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }
// Field plane geometry: row pitch and plane size (u32 words) of `rows` rows.
inline int field_pitch(int W) { return round_up(W, 4); }
inline size_t field_plane(int W, int rows) {
    const size_t p = size_t(std::max(rows, 1)) * size_t(field_pitch(W));
    return (p + 31) / 32 * 32;
}

#include "kern_field.cuh"
#include "kern_cost.cuh"
#include "kern_cost_tc.cuh"
#include "kern_refine.cuh"
#include "kern_misc.cuh"

}  // namespace

// ===========================================================================
// Context.
enum Timing { T_H2D, T_DESC, T_MASK, T_WTA, T_WTA_U, T_LR, T_REFINE, T_D2H, T_COUNT };
static const char* kTimingNames = "h2d,descriptor,mask,wta,wta_unmasked,lr_check,refine,d2h";

// Debug guard mode (environment BSM_GUARD=1 when the first context is
// created; compute-sanitizer is not available on the GPU pool): every device
// buffer gets kGuard bytes of 0xA5 before and after it, and its payload starts
// as 0xA5 too, so out-of-bounds writes show up in bsm_debug_check_guards and
// reads of never-written memory change results against the reference.
constexpr size_t kGuard = 4096;
bool g_guard = false;

struct DevBuf {
    void* p = nullptr;
    void* base = nullptr;
    size_t cap = 0;
    int ensure(size_t bytes) {
        if (bytes <= cap) return BSM_OK;
        release();
        const size_t extra = g_guard ? 2 * kGuard : 0;
        cudaError_t e = cudaMalloc(&base, bytes + extra);
        if (e != cudaSuccess) {
            base = nullptr;
            return set_err(BSM_CUDA_ERROR, std::string("CUDA: cudaMalloc: ") + cudaGetErrorString(e));
        }
        // (the fill runs on the legacy stream, which the context's non-blocking
        // stream does not wait for: complete it before the buffer is handed out)
        if (g_guard && ((e = cudaMemset(base, 0xA5, bytes + extra)) != cudaSuccess ||
                        (e = cudaStreamSynchronize(nullptr)) != cudaSuccess))
            return set_err(BSM_CUDA_ERROR, std::string("CUDA: guard fill: ") + cudaGetErrorString(e));
        p = static_cast<char*>(base) + (g_guard ? kGuard : 0);
        cap = bytes;
        return BSM_OK;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (base) cudaFree(base);
        p = base = nullptr;
        cap = 0;
    }
    // number of guard bytes that no longer hold 0xA5 (0 outside guard mode)
    size_t damaged() const {
        if (!g_guard || !base) return 0;
        std::vector<uint8_t> h(kGuard);
        size_t bad = 0;
        for (int side = 0; side < 2; ++side) {
            const char* g = static_cast<const char*>(base) + (side ? kGuard + cap : 0);
            if (cudaMemcpy(h.data(), g, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return kGuard;
            for (uint8_t v : h) bad += v != 0xA5;
        }
        return bad;
    }
};

struct bsm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sm_count = 0;
    // pattern
    int n = 0, window = 0, half = 0, NW = 0, u = 0;
    int mslots = 0;                 // rank-table slots used by the mask kernels
    int nfill = 0;                  // entries of k_mask4's fill-order table (d_uoff)
    std::vector<int> slot_used;     // slot -> used-offset index (-1: empty)
    int mch = 4;                    // k_mask4 / k_mask_f32 chunks of 32 positions per lane (1, 2, 4)
    std::vector<int> order;         // bit position -> pair index (identity unless permuted)
    bool permuted = false;
    DevBuf d_pos;                   // pair index -> bit position (permuted only)
    double slot_cost[2] = {0, 0};   // avg wavefronts per gather before/after placement
    std::vector<int16_t> pairs;
    std::vector<int2> pair_xy;  // (px,py),(qx,qy) packed later per tile width
    std::vector<int16_t> used;  // used offsets as dy*(2h+1)+dx index list (host)
    DevBuf d_desc4, d_pqb, d_uoff, d_uxy;
    DevBuf d_descf, d_rgb_gray, d_rgb_lab, planes;
    int descf_tw = -1;
    bool rgb_ready = false;
    int desc4_tw = -1, uoff_tw = -1;
    // tables
    float gray_lut[256], lab_lut[768];
    DevBuf d_rank;
    DevBuf d_wtab, d_s2col;
    bool exp_ok = false;            // device exp restatement validated against host libm
    int refine_mode = -1;           // -1: auto, 0: scan kernel, 1: smem bins, 2: weight table
    std::string exp_why;
    ExpDev exp_dev{};
    DevBuf d_etab, d_elam, d_lab256;
    double elam_le = 0;
    int elam_radius = -1;
    double wt_lc = 0, wt_le = 0;
    int wt_radius = -1, wt_ncol = 0;
    // scratch
    DevBuf img_l, img_r, fdl, fml, fdr, fmr, keys_l, keys_r, keys_u;
    DevBuf chk_d, chk_v, ref_d, ref_v, lw_d, rw_d, un_d, counters, inv, vmap;
    DevBuf aux0, aux1, aux2, aux3;
    int last_W = 0, last_rows = 0, last_unmasked = 0, last_r0 = 0, last_out0 = 0, last_out_rows = 0;
    // instrumentation
    bool profiling = false;
    static constexpr int kEvPerSlot = 4;  // a stage may run several times per call (two views)
    cudaEvent_t ev[T_COUNT][kEvPerSlot][2] = {};
    int ev_used[T_COUNT] = {};
    int launches = 0;
    PeerOut peer{};  // peer-memory band outputs during bsm_pipeline_frame_bands_p2p_u8 (n = 0 otherwise)
    int k3_group = 0;    // experiments (BSM_K3_GROUP): tiles per CTA-order group
    int maskf_force_low = 0;  // test hook (BSM_MASKF_FORCE_LOW=1): k_mask_f32 resolves every low byte
    int mq_px = 16;        // pixels per k_mask_q CTA (8, 16 or 32; BSM_MASKQ_PX)
    int mask_variant = 0;  // experiments (BSM_MASK_VARIANT): bit 0 separate P and Q index tables in k_mask4 (implies k_mask4), bit 1 k_mask4 instead of k_mask_q
    int refine_cap = 0;  // experiments (BSM_REFINE_CAP): refine CTAs per SM at most (0: the default rule)
    bool in_batch = false;  // phase B of a batch pair (batch_pair) is being issued
    int k3_variant = 0;  // experiments (BSM_K3_VARIANT): bit 0 thread-0 refill, bit 1 one launch per direction,
                     // bit 2 d-block-major CTA order, bit 3 groups of
                     // 2 x SMs tiles, bit 4 the popcount kernel instead of
                     // the tensor-core one (bits 0-3 apply to the popcount kernel),
                     // bit 5 A in shared memory, bit 7 two operand stages (tensor-core kernel)
    DevBuf popc_out;
    // batch pipelining (bsm_pipeline_batch_u8): two slots of input views and
    // refined maps, an H2D and a D2H copy stream ordered by events
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    DevBuf bimg[2][2], bout_d[2], bout_v[2];
    cudaEvent_t ev_in[2] = {}, ev_free[2] = {}, ev_done[2] = {}, ev_out[2] = {};
    // batches: the check + refine of pair i (phase B) run on s_ref, a
    // high-priority stream, beside the fields of pair i + 1 (phase A) on
    // `stream`; two sets of WTA keys alternate between the phases
    cudaStream_t s_ref = nullptr;
    cudaEvent_t ev_a[2] = {}, ev_b[2] = {};
    DevBuf keys_l2, keys_r2;
};

namespace {

std::vector<DevBuf*> ctx_bufs(bsm_ctx* c) {
    return {&c->d_pos, &c->d_descf, &c->d_rgb_gray, &c->d_rgb_lab, &c->planes, &c->d_desc4, &c->d_pqb, &c->d_uoff,
            &c->d_uxy, &c->d_rank, &c->d_wtab, &c->d_s2col, &c->img_l, &c->img_r, &c->fdl, &c->fml, &c->fdr,
            &c->fmr, &c->keys_l, &c->keys_r, &c->keys_u, &c->chk_d, &c->chk_v, &c->ref_d, &c->ref_v, &c->lw_d,
            &c->rw_d, &c->un_d, &c->counters, &c->inv, &c->vmap, &c->d_etab, &c->d_elam, &c->d_lab256, &c->aux0,
            &c->keys_l2, &c->keys_r2, &c->aux1, &c->aux2, &c->aux3, &c->popc_out, &c->bimg[0][0], &c->bimg[0][1], &c->bimg[1][0],
            &c->bimg[1][1], &c->bout_d[0], &c->bout_d[1], &c->bout_v[0], &c->bout_v[1]};
}

struct Scope {  // brackets one pipeline stage with events when profiling
    bsm_ctx* c;
    int t;
    int slot = -1;
    Scope(bsm_ctx* c_, int t_) : c(c_), t(t_) {
        if (c->profiling && c->ev_used[t] < bsm_ctx::kEvPerSlot) {
            slot = c->ev_used[t]++;
            cudaEventRecord(c->ev[t][slot][0], c->stream);
        }
    }
    ~Scope() {
        if (slot >= 0) cudaEventRecord(c->ev[t][slot][1], c->stream);
    }
};

int check_launch(bsm_ctx* c, const char* what) {
    ++c->launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(BSM_CUDA_ERROR, std::string("CUDA: launch ") + what + ": " + cudaGetErrorString(e));
    return BSM_OK;
}

#define BSM_TRY(x)                  \
    do {                            \
        int rc_ = (x);              \
        if (rc_ != BSM_OK) return rc_; \
    } while (0)

// Tile-relative offset tables depend on the staged tile width.
int desc4_tile_width(int half) { return round_up(kD2TX * 4 + 2 * half + 8, 16); }

// k_descriptor4's per-pair table: byte offsets (4 x word offsets) of both endpoints in its
// phased 4-byte-window tile, relative to the thread's base word:
// (half + px) % 4 selects the phase plane, py*TWs/4 + (half + px)/4 the word.
int ensure_desc4_table(bsm_ctx* c) {
    const int TWs = desc4_tile_width(c->half);
    if (c->desc4_tw == TWs) return BSM_OK;
    const int G = (c->n + 31) / 32;
    std::vector<int2> t(size_t(G) * 32, make_int2(0, 0));
    for (int i = 0; i < c->n; ++i) {
        const int16_t* p = &c->pairs[4 * size_t(c->order[size_t(i)])];
        const int TH = kD2TY * kD2Rows + 2 * c->half, S4 = TWs * TH / 4;
        auto woff = [&](int px, int py) { return ((c->half + px) & 3) * S4 + py * (TWs / 4) + ((c->half + px) >> 2); };
        t[size_t(i)] = make_int2(4 * woff(p[0], p[1]), 4 * woff(p[2], p[3]));  // byte offsets
    }
    BSM_TRY(c->d_desc4.ensure(t.size() * sizeof(int2)));
    BSM_CUDA(cudaMemcpy(c->d_desc4.p, t.data(), t.size() * sizeof(int2), cudaMemcpyHostToDevice));
    c->desc4_tw = TWs;
    return BSM_OK;
}


// Row stride of the k_mask4 / k_mask_f32 window tiles: kM3Px + 2h columns plus
// up to 3 of alignment slack, a multiple of 4 (word-wide tile loads).
int mask4_tw(int half, int px = kM3Px) { return round_up(px + 2 * half + 3, 4); }

int ensure_mask_offsets(bsm_ctx* c, int TW) {
    if (c->uoff_tw == TW) return BSM_OK;
    const int side = 2 * c->half + 1;
    std::vector<int32_t> o(size_t(c->mslots), 0);  // empty slots read the centre (harmless)
    for (int k = 0; k < c->mslots; ++k) {
        const int ui = c->slot_used[size_t(k)];
        if (ui < 0) continue;
        const int dy = c->used[size_t(ui)] / side - c->half, dx = c->used[size_t(ui)] % side - c->half;
        o[size_t(k)] = dy * TW + dx;
    }
    // k_mask4's fill order: groups of 32 slots in which lane b writes a slot of
    // shared-memory bank b (slot % 32 == b: conflict-free stores) and every slot is
    // the g-th of its bank in raster order of its window offset, so one group's
    // tile reads fall within a few window rows (the slot order itself, chosen for
    // the pair gathers, scatters them: 2-3 wavefronts per read, ncu at c4).
    // Entry = (slot << 16) | (offset + h TW + h).  Banks with fewer slots repeat
    // their last one (the same value stored twice).
    {
        std::vector<std::vector<std::pair<int, int>>> bank(32);
        for (int k = 0; k < c->mslots; ++k) bank[size_t(k % 32)].push_back({o[size_t(k)] + c->half * TW + c->half, k});
        size_t groups = 0;
        for (auto& b : bank) {
            std::sort(b.begin(), b.end());
            groups = std::max(groups, b.size());
        }
        std::vector<uint32_t> fill(groups * 32, 0);
        for (size_t g = 0; g < groups; ++g)
            for (int b = 0; b < 32; ++b) {
                if (bank[size_t(b)].empty()) return set_err(BSM_UNSUPPORTED, "bsm: fewer rank-table slots than banks");
                const auto& e = bank[size_t(b)][std::min(g, bank[size_t(b)].size() - 1)];
                if (e.first < 0 || e.first > 0xFFFF || e.second > 0xFFFF)
                    return set_err(BSM_UNSUPPORTED, "bsm: mask window too large for the fill table");
                fill[g * 32 + size_t(b)] = uint32_t(e.second) << 16 | uint32_t(e.first);
            }
        BSM_TRY(c->d_uoff.ensure(std::max<size_t>(4, fill.size() * 4)));
        BSM_CUDA(cudaMemcpy(c->d_uoff.p, fill.data(), fill.size() * 4, cudaMemcpyHostToDevice));
        c->nfill = int(fill.size());
    }
    // the same slots as (dy << 16) | (dx & 0xFFFF) for the float-plane kernel
    std::vector<int32_t> xy(size_t(c->mslots), 0);
    for (int k = 0; k < c->mslots; ++k) {
        const int ui = c->slot_used[size_t(k)];
        if (ui < 0) continue;
        const int dy = c->used[size_t(ui)] / side - c->half, dx = c->used[size_t(ui)] % side - c->half;
        xy[size_t(k)] = int32_t(uint32_t(dy) << 16 | (uint32_t(dx) & 0xFFFFu));
    }
    BSM_TRY(c->d_uxy.ensure(std::max<size_t>(4, xy.size() * 4)));
    BSM_CUDA(cudaMemcpy(c->d_uxy.p, xy.data(), xy.size() * 4, cudaMemcpyHostToDevice));
    c->uoff_tw = TW;
    return BSM_OK;
}

// Bytes of the exact grayscale weight table W[tri(u, v)][col(dx^2 + dy^2)]
// (32,896 gray pairs x distinct squared distances within the radius).
constexpr size_t kWeightTableCap = size_t(256) << 20;
size_t weight_table_bytes(int radius) {
    std::vector<uint8_t> seen(size_t(2) * radius * radius + 1, 0);
    size_t ncol = 0;
    for (int dy = 0; dy <= radius; ++dy)
        for (int dx = 0; dx <= radius; ++dx) {
            uint8_t& f = seen[size_t(dx * dx + dy * dy)];
            ncol += f == 0;
            f = 1;
        }
    return size_t(256 * 257 / 2) * ncol * sizeof(double);
}

int ensure_weight_table(bsm_ctx* c, double lc, double le, int radius) {
    if (c->wt_radius == radius && c->wt_lc == lc && c->wt_le == le) return BSM_OK;
    if (weight_table_bytes(radius) > kWeightTableCap)
        return set_err(BSM_UNSUPPORTED, "bsm: vote_radius " + std::to_string(radius) +
                                            " needs a weight table above 256 MiB and the device exp is unavailable");
    std::vector<double> w;
    std::vector<int16_t> s2col;
    int ncol = 0;
    bsmh::vote_weight_table(c->lab_lut, lc, le, radius, w, s2col, ncol);
    BSM_TRY(c->d_wtab.ensure(w.size() * 8));
    BSM_TRY(c->d_s2col.ensure(s2col.size() * 2));
    BSM_CUDA(cudaMemcpy(c->d_wtab.p, w.data(), w.size() * 8, cudaMemcpyHostToDevice));
    BSM_CUDA(cudaMemcpy(c->d_s2col.p, s2col.data(), s2col.size() * 2, cudaMemcpyHostToDevice));
    c->wt_lc = lc;
    c->wt_le = le;
    c->wt_radius = radius;
    c->wt_ncol = ncol;
    return BSM_OK;
}

int check_pattern(bsm_ctx* c) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    if (c->n <= 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: no sampling pattern set (bsm_set_pattern)");
    return BSM_OK;
}



size_t mask4_smem(const bsm_ctx* c) {
    const int TW = mask4_tw(c->half), TH = 2 * c->half + 1;
    return 2 * size_t(round_up(c->mslots + 1, 4)) * 4 + size_t(kM3Px) * mask4_stage_stride(c->mch) * 4 + 1024 +
           size_t(TW) * TH;
}


// Descriptors + masks of rows [ybeg, ybeg + rows) of a W x H view on device.
// With img2 (desc2, mask2): the second view of a pair in the same launches
// (grid.z), one launch tail per kernel instead of two.
int field_device(bsm_ctx* c, const uint8_t* img, int W, int H, int ybeg, int rows, uint32_t* desc, uint32_t* mask,
                 const uint8_t* img2 = nullptr, uint32_t* desc2 = nullptr, uint32_t* mask2 = nullptr) {
    const int nviews = img2 ? 2 : 1;
    const int Wp = round_up(W, 128), Wq = field_pitch(W);
    const size_t P = field_plane(W, rows);
    // MCH = 2, 4 (1024 < n <= 4096): k_mask_q (its own tile width)
    const bool use_q = (c->mch == 2 || c->mch == 4) && !(c->mask_variant & 3);
    const int mq_px = c->mq_px;
    BSM_TRY(ensure_mask_offsets(c, use_q ? mask4_tw(c->half, mq_px) : mask4_tw(c->half)));
    {
        Scope s(c, T_DESC);
        BSM_TRY(ensure_desc4_table(c));
        const int TWs = desc4_tile_width(c->half);
        const size_t sm = size_t(TWs) * (kD2TY * kD2Rows + 2 * c->half) * 5 + 16;
        dim3 grid(Wp / (kD2TX * 4), (rows + kD2TY * kD2Rows - 1) / (kD2TY * kD2Rows));
        // split the word range over grid.z until there are ~16 CTAs per SM (the
        // tail of a partial last wave dominates otherwise; c2: 759 -> 3036 CTAs)
        const int zsplit = std::max(1, std::min((c->NW + 7) / 8, (16 * c->sm_count + int(grid.x * grid.y) - 1) /
                                                                   int(grid.x * grid.y)));
        grid.z = unsigned(zsplit * nviews);
        BSM_CUDA(cudaFuncSetAttribute(k_descriptor4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        k_descriptor4<<<grid, dim3(kD2TX, kD2TY), sm, c->stream>>>(img, W, H, ybeg, rows, c->d_desc4.as<int2>(),
                                                                    c->n, c->half, TWs, c->NW, Wq, P, desc, img2,
                                                                    desc2, zsplit);
        BSM_TRY(check_launch(c, "descriptor"));
    }
    {
        Scope s(c, T_MASK);
        const size_t sm4 = mask4_smem(c);
        dim3 grid3((Wq + kM3Px - 1) / kM3Px, rows, nviews);
        auto launch = [&](auto kern) -> int {
            BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm4)));
            const bool packed = c->mch <= 4 && !(c->mask_variant & 1);
            kern<<<grid3, 32, sm4, c->stream>>>(img, W, H, ybeg, rows,
                                                c->d_pqb.as<uint4>() + (packed ? 2 * kPqTable / 4 : 0),
                                                c->d_pqb.as<uint4>() + kPqTable / 4, c->n, c->d_uoff.as<uint32_t>(),
                                                c->nfill, c->mslots, round_up(c->mslots + 1, 4), c->d_rank.as<uint8_t>(),
                                                c->half, mask4_tw(c->half), c->NW, Wq, P, mask, img2, mask2);
            return BSM_OK;
        };
        // MCH = 2, 4 (1024 < n <= 4096): four pixels per pass over u8 ranks,
        // two warps per CTA (k_mask_q); BSM_MASK_VARIANT bit 1 keeps k_mask4
        if (use_q) {
            const size_t smq = size_t(round_up(c->mslots + 1, 4)) * 4 + size_t(mq_px) * mask4_stage_stride(c->mch) * 4 +
                               64 + 1024 + size_t(mask4_tw(c->half, mq_px)) * (2 * c->half + 1);
            const dim3 gridq((Wq + mq_px - 1) / mq_px, rows, nviews);
            auto launch_q = [&](auto kern) -> int {
                BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smq)));
                kern<<<gridq, 64, smq, c->stream>>>(img, W, H, ybeg, rows, c->d_pqb.as<uint4>() + 2 * kPqTable / 4,
                                                    c->n, c->d_uoff.as<uint32_t>(), c->nfill, c->mslots,
                                                    round_up(c->mslots + 1, 4), c->d_rank.as<uint8_t>(), c->half,
                                                    mask4_tw(c->half, mq_px), c->NW, Wq, P, mask, img2, mask2);
                return BSM_OK;
            };
            if (mq_px == 32)
                BSM_TRY(c->mch == 2 ? launch_q(k_mask_q<1, 32>) : launch_q(k_mask_q<2, 32>));
            else if (mq_px == 16)
                BSM_TRY(c->mch == 2 ? launch_q(k_mask_q<1, 16>) : launch_q(k_mask_q<2, 16>));
            else
                BSM_TRY(c->mch == 2 ? launch_q(k_mask_q<1>) : launch_q(k_mask_q<2>));
            return check_launch(c, "mask");
        }
        // chunks of 32 positions per lane: the work scales with n
        // MCH <= 4: the packed P | Q << 16 index table (half the index loads;
        // the split runs on the FMA pipe): -3% mask time at c2 / c4
        if (!(c->mask_variant & 1))
            BSM_TRY(c->mch == 1   ? launch(k_mask4<1, true>)
                    : c->mch == 2 ? launch(k_mask4<2, true>)
                    : c->mch == 4 ? launch(k_mask4<4, true>)
                                  : launch(k_mask4<8>));
        else
            BSM_TRY(c->mch == 1   ? launch(k_mask4<1>)
                    : c->mch == 2 ? launch(k_mask4<2>)
                    : c->mch == 4 ? launch(k_mask4<4>)
                                  : launch(k_mask4<8>));
        BSM_TRY(check_launch(c, "mask"));
    }
    return BSM_OK;
}

// WTA keys of rows [0, rows) of device fields (SoA); keys: rows x W.
// Tensor map of a device field [NW][P] u32 for TMA boxes of box_x pixels x
// kCostK words; out-of-range boxes read zeros.
int field_tensor_map(CUtensorMap* map, const uint32_t* field, int W, int NW, int rows, int box_x,
                     int box_w = kCostK) {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        BSM_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess)
            return set_err(BSM_CUDA_ERROR, "CUDA: cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    const size_t P = field_plane(W, rows);
    const cuuint64_t dims[2] = {cuuint64_t(P), cuuint64_t(NW)};
    const cuuint64_t strides[1] = {cuuint64_t(P) * 4};
    const cuuint32_t box[2] = {cuuint32_t(box_x), cuuint32_t(box_w)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(field), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(BSM_CUDA_ERROR, "CUDA: cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return BSM_OK;
}

// K3 over device fields.  Direction 0 (left reference, x - d): ref = (dl, ml),
// other = dr, keys -> keys_l; direction 1 (right reference, x + d): ref =
// (dr, mr), other = dl, keys -> keys_r.  both: one launch for the two
// directions; otherwise only direction `dir`.  ml/mr == nullptr: unmasked.
// Tiles per CTA-order group of the cost kernel (see k_cost_wta).  Tile-major
// (1) by default: measured on B200, it reads less DRAM
// than the tile's words (the two directions and neighbouring d-blocks share
// them through L2: 0.67x the algorithmic bytes at c2 and c4) and is within 2%
// of the fastest order (d-block-major: c2 -1.8% time at 3x the DRAM bytes).
int k3_group(const bsm_ctx* c, int tiles) {
    if (c->k3_variant & 4) return tiles;                               // d-block-major
    if (c->k3_variant & 8) return std::max(1, std::min(tiles, 2 * c->sm_count));  // one wave per d-block pass
    if (c->k3_group > 0) return std::min(tiles, c->k3_group);
    return 1;
}

// K3 on the tensor cores (kern_cost_tc.cuh): persistent CTAs, one per SM.
// d-blocks of at most kTcMaxDc disparities; with several, each starts on a
// multiple of 4 (TMA box alignment) and they merge with atomicMin.
int wta_device_tc(bsm_ctx* c, const uint32_t* dl, const uint32_t* ml, const uint32_t* dr, const uint32_t* mr, int W,
                  int rows, int d_max, bool both, int dir, bool masked, uint32_t* keys_l, uint32_t* keys_r) {
    const int Wq = field_pitch(W);
    const int ndd = (d_max + kTcMaxDc - 1) / kTcMaxDc;
    const int Dc = ndd == 1 ? d_max : round_up((d_max + ndd - 1) / ndd, 4);
    const int ncols = round_up(kTcRows + ((Dc + 2) & ~3), 32);
    const bool use_l = both || dir == 0, use_r = both || dir == 1;
    if (ndd > 1) {
        if (use_l) BSM_CUDA(cudaMemsetAsync(keys_l, 0xFF, size_t(rows) * W * 4, c->stream));
        if (use_r) BSM_CUDA(cudaMemsetAsync(keys_r, 0xFF, size_t(rows) * W * 4, c->stream));
    }
    const long long npix = static_cast<long long>(rows) * Wq;
    const long long tiles = (npix + kTcRows - 1) / kTcRows;
    const int ndir = both ? 2 : 1;
    if (tiles * ndd * ndir > 0x7FFFFFFFLL) return set_err(BSM_UNSUPPORTED, "bsm: image too large for the cost kernel");
    const int items = int(tiles * ndd * ndir);
    CUtensorMap lr, lm, lo, rr, rm, ro;  // unused slots are copies of a valid map
    const uint32_t* ml_ = ml ? ml : dl;
    const uint32_t* mr_ = mr ? mr : dr;
    BSM_TRY(field_tensor_map(&lr, use_l ? dl : dr, W, c->NW, rows, kTcRows, kTcKS));
    BSM_TRY(field_tensor_map(&lm, use_l ? ml_ : mr_, W, c->NW, rows, kTcRows, kTcKS));
    BSM_TRY(field_tensor_map(&lo, use_l ? dr : dl, W, c->NW, rows, ncols / 2, kTcKS));
    BSM_TRY(field_tensor_map(&rr, use_r ? dr : dl, W, c->NW, rows, kTcRows, kTcKS));
    BSM_TRY(field_tensor_map(&rm, use_r ? mr_ : ml_, W, c->NW, rows, kTcRows, kTcKS));
    BSM_TRY(field_tensor_map(&ro, use_r ? dl : dr, W, c->NW, rows, ncols / 2, kTcKS));
    // A operand in TMEM for accumulators up to 320 columns (measured on B200,
    // tools/microbench/tc_probe: c4 -1.1%, c1/c3 -4%; at 384 columns (c2, c5)
    // +0.6%); BSM_K3_VARIANT bit 5 forces A into shared memory
    const bool at = ncols <= 320 && !(c->k3_variant & 32);
    // with A in TMEM the accumulator (<= 320 columns) leaves room for a third
    // operand stage in TMEM and shared memory: c4 -1.9%, c1 -2.5%, c3 -3.6%
    // (tools/microbench/tc_probe); BSM_K3_VARIANT bit 7 keeps two
    const int stages = at && ncols <= tc_acol(3) && !(c->k3_variant & 128) ? 3 : 2;
    const TcSmem L(ncols, masked, at, stages);
    if (L.nraw < 2) return set_err(BSM_UNSUPPORTED, "bsm: cost kernel shared-memory layout");
    const size_t sm = L.total;  // > 114 KB: one CTA per SM (it allocates all 512 TMEM columns)
    const int grid = std::min(items, c->sm_count);
    auto launch = [&](auto kern) -> int {
        BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        kern<<<grid, kTcThreads, sm, c->stream>>>(lr, lm, lo, rr, rm, ro, W, Wq, int(npix), c->NW, d_max, Dc, ncols,
                                                  ndd, ndir, both ? 0 : dir, items, keys_l, keys_r);
        return BSM_OK;
    };
    if (stages == 3) BSM_TRY(masked ? launch(k_cost_wta_tc<true, true, 3>) : launch(k_cost_wta_tc<false, true, 3>));
    else if (at) BSM_TRY(masked ? launch(k_cost_wta_tc<true, true>) : launch(k_cost_wta_tc<false, true>));
    else BSM_TRY(masked ? launch(k_cost_wta_tc<true, false>) : launch(k_cost_wta_tc<false, false>));
    return check_launch(c, "cost_wta_tc");
}

int wta_device(bsm_ctx* c, const uint32_t* dl, const uint32_t* ml, const uint32_t* dr, const uint32_t* mr, int W,
               int rows, int d_max, bool both, int dir, bool masked, uint32_t* keys_l, uint32_t* keys_r, int timing) {
    Scope s(c, timing);
    // default: the tensor-core kernel; BSM_K3_VARIANT bit 4 selects the popcount kernel
    if (!(c->k3_variant & 16)) return wta_device_tc(c, dl, ml, dr, mr, W, rows, d_max, both, dir, masked, keys_l, keys_r);
    const int Wq = field_pitch(W);
    const int dz = (d_max + kCostDisp - 1) / kCostDisp;
    const bool use_l = both || dir == 0, use_r = both || dir == 1;
    if (dz > 1) {
        if (use_l) BSM_CUDA(cudaMemsetAsync(keys_l, 0xFF, size_t(rows) * W * 4, c->stream));
        if (use_r) BSM_CUDA(cudaMemsetAsync(keys_r, 0xFF, size_t(rows) * W * 4, c->stream));
    }
    const long long tiles = (static_cast<long long>(rows) * Wq + kCostTile - 1) / kCostTile;
    const int ndd = dz * (both ? 2 : 1);
    if (tiles * ndd > 0x7FFFFFFFLL) return set_err(BSM_UNSUPPORTED, "bsm: image too large for the cost kernel grid");
    dim3 grid(unsigned(tiles * ndd));
    const size_t stage_words = size_t(masked ? 2 : 1) * kCostK * kCostTile + size_t(kCostK) * (kCostTile + kCostDisp);
    const size_t sm = (kCostStages * stage_words + 8 * kCostTile) * 4 + kCostStages * 16 + kCostStages * 4;
    CUtensorMap lr, lm, lo, rr, rm, ro;  // unused slots are copies of a valid map
    const uint32_t* ml_ = ml ? ml : dl;
    const uint32_t* mr_ = mr ? mr : dr;
    BSM_TRY(field_tensor_map(&lr, use_l ? dl : dr, W, c->NW, rows, kCostTile));
    BSM_TRY(field_tensor_map(&lm, use_l ? ml_ : mr_, W, c->NW, rows, kCostTile));
    BSM_TRY(field_tensor_map(&lo, use_l ? dr : dl, W, c->NW, rows, kCostTile + kCostDisp));
    BSM_TRY(field_tensor_map(&rr, use_r ? dr : dl, W, c->NW, rows, kCostTile));
    BSM_TRY(field_tensor_map(&rm, use_r ? mr_ : ml_, W, c->NW, rows, kCostTile));
    BSM_TRY(field_tensor_map(&ro, use_r ? dl : dr, W, c->NW, rows, kCostTile + kCostDisp));
    auto launch = [&](auto kern) -> int {
        BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        kern<<<grid, 256, sm, c->stream>>>(lr, lm, lo, rr, rm, ro, W, Wq, rows, c->NW, d_max, dz, ndd,
                                           int(tiles), k3_group(c, int(tiles)), both ? 0 : dir,
                                           keys_l, keys_r, 2u);
        return BSM_OK;
    };
    if (c->k3_variant & 1) BSM_TRY(masked ? launch(k_cost_wta<true, false>) : launch(k_cost_wta<false, false>));
    else BSM_TRY(masked ? launch(k_cost_wta<true, true>) : launch(k_cost_wta<false, true>));
    return check_launch(c, "cost_wta");
}

int ensure_elam(bsm_ctx* c, double le, int radius) {
    if (c->elam_le == le && c->elam_radius == radius) return BSM_OK;
    std::vector<double> t(size_t(2 * radius * radius) + 1);
    for (size_t k = 0; k < t.size(); ++k) t[k] = std::sqrt(double(k)) / le;  // sqrt(dx*dx + dy*dy) / lambda_e
    BSM_TRY(c->d_elam.ensure(t.size() * 8));
    BSM_CUDA(cudaMemcpy(c->d_elam.p, t.data(), t.size() * 8, cudaMemcpyHostToDevice));
    c->elam_le = le;
    c->elam_radius = radius;
    return BSM_OK;
}

// Refinement of the invalid pixels listed in c->inv (count in counters[1],
// max_bin in counters[0]) into c->ref_d / c->ref_v (pre-filled with the input
// map).  nbins_max bounds max_bin + 1.  lab: per-pixel Lab plane or nullptr
// (grayscale: the gray value indexes the Lab table).
int refine_launch(bsm_ctx* c, const float* cd, const uint8_t* cv, const uint8_t* gray, const float4* lab, int W,
                  int rows, int radius, int nbins_max, double lc, double le) {
    const size_t px = size_t(rows) * W;
    const int nbins = round_up(std::max(nbins_max, 1), 32);
    const int tb = 256;
    int mode = c->refine_mode >= 0 ? c->refine_mode : (lab ? 4 : 3);
    if (lab && mode != 4) mode = 4;  // Lab planes: the weight table only covers gray pairs
    // large radii: the exact table would exceed 256 MiB (3 GB at radius 180),
    // so the gray path evaluates the weights with the device exp instead
    if (!lab && mode != 4 && c->exp_ok && weight_table_bytes(radius) > kWeightTableCap) mode = 4;
    if (mode == 4 && !c->exp_ok) {
        if (lab) return set_err(BSM_UNSUPPORTED, "bsm: colour refine needs the device exp (" + c->exp_why + ")");
        mode = 3;
    }
    if (mode == 3 || mode == 4) {
        const bool devexp = mode == 4;
        const size_t fixed = devexp ? 256 * 8 + 768 * 4 : 0;  // exp table + gray Lab rows (device exp only)
        // bins of NP pixels per warp: 4 (default) or 1 for very wide disparity ranges
        const int np = (fixed + 8 * 32 * 12 + size_t(8) * 4 * nbins * 8 <= 200 * 1024) ? 4 : 1;
        const int warps =
            std::min(8, int((200 * 1024 - fixed) / (size_t(32) * 12 + size_t(np) * nbins * 8)));
        if (warps >= 1) {
            if (devexp) BSM_TRY(ensure_elam(c, le, radius));
            else BSM_TRY(ensure_weight_table(c, lc, le, radius));
            BSM_TRY(c->vmap.ensure(px * 4));
            k_make_vmap<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(cd, cv, gray, px, c->vmap.as<uint32_t>());
            BSM_TRY(check_launch(c, "make_vmap"));
            const size_t sm = fixed + size_t(warps) * 32 * 12 + size_t(warps) * np * nbins * 8;
            const bool peer = c->peer.n > 0;  // the peer-storing kernels only for bsm_frame bands
            auto kern = peer ? (np == 4 ? (devexp ? k_vote_refine_fold<4, true, true> : k_vote_refine_fold<4, false, true>)
                                        : (devexp ? k_vote_refine_fold<1, true, true> : k_vote_refine_fold<1, false, true>))
                             : (np == 4 ? (devexp ? k_vote_refine_fold<4, true, false> : k_vote_refine_fold<4, false, false>)
                                        : (devexp ? k_vote_refine_fold<1, true, false> : k_vote_refine_fold<1, false, false>));
            BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
            // as many CTAs per SM as fit (4 at c4: 32 warps) when the refine runs
            // alone; in a batch (batch_pair) two, so that the next pair's
            // descriptor / mask CTAs share the SMs: c4 batch 37.8k -> 38.1k
            // Mdisp-evals/s (3: 37.8k, 1: 37.0k) although the refine alone slows
            // from 1.00 to 1.42 ms.  BSM_REFINE_CAP overrides both.
            int per_sm = std::max(1, std::min(4, int((220 * 1024) / sm)));
            const int cap = c->refine_cap > 0 ? c->refine_cap : (c->in_batch ? 2 : 0);
            if (cap > 0) per_sm = std::min(per_sm, cap);
            BSM_CUDA(cudaMemsetAsync(c->counters.as<int>() + 2, 0, 4, c->stream));  // work counter
            kern<<<c->sm_count * per_sm, warps * 32, sm, c->stream>>>(
                c->vmap.as<uint32_t>(), lab, c->d_lab256.as<float>(), W, rows, radius, lc, c->d_elam.as<double>(),
                c->exp_dev, c->d_etab.as<unsigned long long>(), c->d_wtab.as<double>(), c->wt_ncol,
                c->d_s2col.as<int16_t>(), c->counters.as<int>(), c->inv.as<int>(), nbins, c->ref_d.as<float>(),
                c->ref_v.as<uint8_t>(), c->counters.as<int>() + 2, c->peer);
            return check_launch(c, "vote_refine_fold");
        }
        if (lab) return set_err(BSM_UNSUPPORTED, "bsm: disparity range too wide for the colour refine bins");
    }
    // mode 2 (or bins too wide for the fold): warp per pixel, exact host weight table
    BSM_TRY(ensure_weight_table(c, lc, le, radius));
    const int warps = std::max(1, std::min(8, int((96 * 1024) / (size_t(nbins) * 8))));
    const size_t sm = size_t(warps) * nbins * 8;
    auto kvr = c->peer.n > 0 ? k_vote_refine<true> : k_vote_refine<false>;
    BSM_CUDA(cudaFuncSetAttribute(kvr, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
    kvr<<<c->sm_count * 8, warps * 32, sm, c->stream>>>(
        cd, cv, gray, W, rows, radius, c->d_wtab.as<double>(), c->wt_ncol, c->d_s2col.as<int16_t>(),
        c->counters.as<int>(), c->inv.as<int>(), nbins, c->ref_d.as<float>(), c->ref_v.as<uint8_t>(), c->peer);
    return check_launch(c, "vote_refine");
}

int validate_params(const bsm_params* p) {
    if (!p) return set_err(BSM_INVALID_ARGUMENT, "bsm: null params");
    if (p->d_max < 1) return set_err(BSM_INVALID_ARGUMENT, "config: d_max must be set (>= 1)");
    if (p->d_max > 65535) return set_err(BSM_UNSUPPORTED, "bsm: d_max > 65535 is outside this build's envelope");
    if (!(p->lambda_c > 0)) return set_err(BSM_INVALID_ARGUMENT, "config: lambda_c must be > 0");
    if (!(p->lambda_e > 0)) return set_err(BSM_INVALID_ARGUMENT, "config: lambda_e must be > 0");
    if (p->lr_tolerance < 0) return set_err(BSM_INVALID_ARGUMENT, "config: lr_tolerance must be >= 0");
    if (p->vote_radius < 1) return set_err(BSM_INVALID_ARGUMENT, "config: vote_radius must be >= 1");
    if (p->vote_radius > 180) return set_err(BSM_UNSUPPORTED, "bsm: vote_radius > 180 is outside this build's envelope");
    return BSM_OK;
}

// The fused device pipeline.  Views are full W x H device images; the
// refined output covers rows [out0, out0 + out_rows); fields, WTA and the
// check cover the halo-extended rows [r0, r1).
// k_descriptor_f32's per-pair table: tile-relative byte offsets 4 (py*TW + px).
int ensure_descf_table(bsm_ctx* c) {
    const int TW = kDfTX + 2 * c->half;
    if (c->descf_tw == TW) return BSM_OK;
    const int G = (c->n + 31) / 32;
    std::vector<int2> t(size_t(G) * 32, make_int2(0, 0));
    for (int i = 0; i < c->n; ++i) {
        const int16_t* p = &c->pairs[4 * size_t(c->order[size_t(i)])];
        t[size_t(i)] = make_int2(4 * (p[1] * TW + p[0]), 4 * (p[3] * TW + p[2]));  // byte offsets
    }
    BSM_TRY(c->d_descf.ensure(t.size() * sizeof(int2)));
    BSM_CUDA(cudaMemcpy(c->d_descf.p, t.data(), t.size() * sizeof(int2), cudaMemcpyHostToDevice));
    c->descf_tw = TW;
    return BSM_OK;
}

size_t maskf_smem(const bsm_ctx* c) { return size_t(round_up(c->mslots + 1, 4)) * 4 + size_t(23) * c->mch * 32 * 4; }

// Descriptors + masks of rows [ybeg, ybeg + rows) from float gray / Lab planes.
int field_device_f32(bsm_ctx* c, const float* gray, const float4* lab, int W, int H, int ybeg, int rows,
                     uint32_t* desc, uint32_t* mask) {
    const int Wq = field_pitch(W);
    const size_t P = field_plane(W, rows);
    BSM_TRY(ensure_descf_table(c));
    // k_mask_f32 reads only d_uxy, which does not depend on the tile width: keep
    // the gray kernels' fill table as it is (no re-upload between colour and gray calls)
    BSM_TRY(ensure_mask_offsets(c, c->uoff_tw > 0 ? c->uoff_tw : mask4_tw(c->half)));
    {
        Scope s(c, T_DESC);
        const int TW = kDfTX + 2 * c->half, TH = kDfTY * kDfPY + 2 * c->half;
        const size_t sm = size_t(TW) * TH * 4;
        dim3 grid((Wq + kDfTX - 1) / kDfTX, (rows + kDfTY * kDfPY - 1) / (kDfTY * kDfPY));
        BSM_CUDA(cudaFuncSetAttribute(k_descriptor_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        k_descriptor_f32<<<grid, dim3(kDfTX, kDfTY), sm, c->stream>>>(gray, W, H, ybeg, rows, c->d_descf.as<int2>(),
                                                                      c->n, c->half, c->NW, Wq, P, desc);
        BSM_TRY(check_launch(c, "descriptor_f32"));
    }
    {
        Scope s(c, T_MASK);
        const size_t sm = maskf_smem(c);
        dim3 grid((Wq + kM3Px - 1) / kM3Px, rows);
        auto launch = [&](auto kern) -> int {
            BSM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
            kern<<<grid, 32, sm, c->stream>>>(lab, W, H, ybeg, rows,
                                              c->d_pqb.as<uint4>() + (c->mch <= 4 ? 2 * kPqTable / 4 : 0),
                                              c->d_pqb.as<uint4>() + kPqTable / 4, c->n, c->d_uxy.as<int32_t>(), c->mslots,
                                              round_up(c->mslots + 1, 4), c->NW, Wq, P, mask, c->half,
                                              c->maskf_force_low);
            return BSM_OK;
        };
        BSM_TRY(c->mch == 1   ? launch(k_mask_f32<1>)
                : c->mch == 2 ? launch(k_mask_f32<2>)
                : c->mch == 4 ? launch(k_mask_f32<4>)
                              : launch(k_mask_f32<8>));
        BSM_TRY(check_launch(c, "mask_f32"));
    }
    return BSM_OK;
}

// The 2^24-colour conversion tables on the device (built once per context).
int ensure_rgb_tables(bsm_ctx* c) {
    if (c->rgb_ready) return BSM_OK;
    std::vector<float> g, l;
    bsmh::rgb24_tables(g, l);
    BSM_TRY(c->d_rgb_gray.ensure(g.size() * 4));
    BSM_TRY(c->d_rgb_lab.ensure(l.size() * 4));
    BSM_CUDA(cudaMemcpy(c->d_rgb_gray.p, g.data(), g.size() * 4, cudaMemcpyHostToDevice));
    BSM_CUDA(cudaMemcpy(c->d_rgb_lab.p, l.data(), l.size() * 4, cudaMemcpyHostToDevice));
    c->rgb_ready = true;
    return BSM_OK;
}

// Device views of a pair: grayscale uint8 images, or float gray + Lab planes
// (colour input / arbitrary GrayImage + LabImage).
struct Views {
    const uint8_t* u8l = nullptr;
    const uint8_t* u8r = nullptr;
    const float* gl = nullptr;
    const float4* ll = nullptr;  // Lab planes, float4 (L, a, b, 0) per pixel
    const float* gr = nullptr;
    const float4* lr = nullptr;
};

// phases: 1 = fields + WTA (A), 2 = check + refine (B), 3 = both; the WTA
// keys go to keys_l/keys_r, or to the second set with alt_keys (batches).
int pipeline_device(bsm_ctx* c, const Views& v, int W, int H, int out0, int out_rows, const bsm_params* p,
                    bool want_unmasked, int phases = 3, bool alt_keys = false) {
    BSM_TRY(check_pattern(c));
    BSM_TRY(validate_params(p));
    const int r0 = std::max(0, out0 - p->vote_radius);
    const int r1 = std::min(H, out0 + out_rows + p->vote_radius);
    const int rows = r1 - r0;
    const size_t fbytes = field_plane(W, rows) * c->NW * 4;
    const size_t px = size_t(rows) * W;
    BSM_TRY(c->fdl.ensure(fbytes));
    BSM_TRY(c->fml.ensure(fbytes));
    BSM_TRY(c->fdr.ensure(fbytes));
    BSM_TRY(c->fmr.ensure(fbytes));
    BSM_TRY(c->keys_l.ensure(px * 4));
    BSM_TRY(c->keys_r.ensure(px * 4));
    if (want_unmasked) BSM_TRY(c->keys_u.ensure(px * 4));
    BSM_TRY(c->chk_d.ensure(px * 4));
    BSM_TRY(c->chk_v.ensure(px));
    BSM_TRY(c->ref_d.ensure(px * 4));
    BSM_TRY(c->ref_v.ensure(px));
    BSM_TRY(c->lw_d.ensure(px * 4));
    BSM_TRY(c->rw_d.ensure(px * 4));
    if (want_unmasked) BSM_TRY(c->un_d.ensure(px * 4));
    BSM_TRY(c->counters.ensure(64));
    BSM_TRY(c->inv.ensure(px * 4));

    uint32_t* kl = (alt_keys ? c->keys_l2 : c->keys_l).as<uint32_t>();
    uint32_t* kr = (alt_keys ? c->keys_r2 : c->keys_r).as<uint32_t>();
    if (phases & 1) {
    if (v.u8l) {
        BSM_TRY(field_device(c, v.u8l, W, H, r0, rows, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>(), v.u8r,
                             c->fdr.as<uint32_t>(), c->fmr.as<uint32_t>()));
    } else {
        BSM_TRY(field_device_f32(c, v.gl, v.ll, W, H, r0, rows, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>()));
        BSM_TRY(field_device_f32(c, v.gr, v.lr, W, H, r0, rows, c->fdr.as<uint32_t>(), c->fmr.as<uint32_t>()));
    }
    if (c->k3_variant & 2) {  // one launch per direction
        BSM_TRY(wta_device(c, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>(), c->fdr.as<uint32_t>(),
                           c->fmr.as<uint32_t>(), W, rows, p->d_max, false, 0, true, kl, kr, T_WTA));
        BSM_TRY(wta_device(c, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>(), c->fdr.as<uint32_t>(),
                           c->fmr.as<uint32_t>(), W, rows, p->d_max, false, 1, true, kl, kr, T_WTA));
    } else {
        BSM_TRY(wta_device(c, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>(), c->fdr.as<uint32_t>(),
                           c->fmr.as<uint32_t>(), W, rows, p->d_max, true, 0, true, kl, kr, T_WTA));
    }
    if (want_unmasked)
        BSM_TRY(wta_device(c, c->fdl.as<uint32_t>(), nullptr, c->fdr.as<uint32_t>(), nullptr, W, rows, p->d_max, false,
                           0, false, c->keys_u.as<uint32_t>(), nullptr, T_WTA_U));
    }
    if (!(phases & 2)) return BSM_OK;
    {
        Scope s(c, T_LR);
        BSM_CUDA(cudaMemsetAsync(c->counters.p, 0, 64, c->stream));
        const int tb = 256;
        (c->peer.n > 0 ? k_lr_check_keys<true> : k_lr_check_keys<false>)<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(
            kl, kr, W, rows, p->lr_tolerance, c->chk_d.as<float>(),
            c->chk_v.as<uint8_t>(), c->lw_d.as<float>(), c->rw_d.as<float>(), out0 - r0, out0 - r0 + out_rows,
            c->counters.as<int>(), c->inv.as<int>(), c->peer);
        BSM_TRY(check_launch(c, "lr_check"));
        if (want_unmasked) {
            k_keys_to_float<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(c->keys_u.as<uint32_t>(), px,
                                                                              c->un_d.as<float>());
            BSM_TRY(check_launch(c, "keys_to_float"));
        }
    }
    {
        Scope s(c, T_REFINE);
        BSM_CUDA(cudaMemcpyAsync(c->ref_d.p, c->chk_d.p, px * 4, cudaMemcpyDeviceToDevice, c->stream));
        BSM_CUDA(cudaMemcpyAsync(c->ref_v.p, c->chk_v.p, px, cudaMemcpyDeviceToDevice, c->stream));
        BSM_TRY(refine_launch(c, c->chk_d.as<float>(), c->chk_v.as<uint8_t>(), v.u8l ? v.u8l + size_t(r0) * W : nullptr,
                              v.u8l ? nullptr : v.ll + size_t(r0) * W, W, rows, p->vote_radius, p->d_max,
                              p->lambda_c, p->lambda_e));
    }
    c->last_W = W;
    c->last_rows = rows;
    c->last_r0 = r0;
    c->last_out0 = out0;
    c->last_out_rows = out_rows;
    c->last_unmasked = want_unmasked ? 1 : 0;
    return BSM_OK;
}

Views u8views(const uint8_t* l, const uint8_t* r) {
    Views v;
    v.u8l = l;
    v.u8r = r;
    return v;
}

int fetch(bsm_ctx* c, bsm_maps* o) {
    if (!o) return BSM_OK;
    Scope s(c, T_D2H);
    const int W = c->last_W;
    const size_t all = size_t(c->last_rows) * W;
    const size_t off = size_t(c->last_out0 - c->last_r0) * W;
    const size_t outpx = size_t(c->last_out_rows) * W;
    auto d2h = [&](void* dst, const DevBuf& b, size_t byte_off, size_t bytes) -> int {
        if (!dst) return BSM_OK;
        BSM_CUDA(cudaMemcpyAsync(dst, static_cast<const char*>(b.p) + byte_off, bytes, cudaMemcpyDeviceToHost, c->stream));
        return BSM_OK;
    };
    BSM_TRY(d2h(o->refined_d, c->ref_d, off * 4, outpx * 4));
    BSM_TRY(d2h(o->refined_v, c->ref_v, off, outpx));
    BSM_TRY(d2h(o->left_d, c->lw_d, 0, all * 4));
    BSM_TRY(d2h(o->right_d, c->rw_d, 0, all * 4));
    BSM_TRY(d2h(o->checked_d, c->chk_d, 0, all * 4));
    BSM_TRY(d2h(o->checked_v, c->chk_v, 0, all));
    if (c->last_unmasked) BSM_TRY(d2h(o->unmasked_d, c->un_d, 0, all * 4));
    return BSM_OK;
}

int begin_call(bsm_ctx* c) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    BSM_CUDA(cudaSetDevice(c->device));
    c->launches = 0;
    for (int t = 0; t < T_COUNT; ++t) c->ev_used[t] = 0;
    return BSM_OK;
}

int upload_views(bsm_ctx* c, const uint8_t* left, const uint8_t* right, int W, int H) {
    Scope s(c, T_H2D);
    const size_t n = size_t(W) * H;
    BSM_TRY(c->img_l.ensure(n));
    BSM_TRY(c->img_r.ensure(n));
    BSM_CUDA(cudaMemcpyAsync(c->img_l.p, left, n, cudaMemcpyHostToDevice, c->stream));
    if (right) BSM_CUDA(cudaMemcpyAsync(c->img_r.p, right, n, cudaMemcpyHostToDevice, c->stream));
    return BSM_OK;
}

int sync(bsm_ctx* c) {
    BSM_CUDA(cudaStreamSynchronize(c->stream));
    return BSM_OK;
}

// The per-stage vote_refine's pre-pass on the device (c->chk_d / chk_v hold
// the caller's map): invalid list + max_bin into c->counters / c->inv, and
// ref_d / ref_v initialised with the input map; max_bin returned to the host
// (the bin count sizes the refine kernel's shared memory).
int invalid_list(bsm_ctx* c, size_t px, double lim, int& max_bin) {
    BSM_CUDA(cudaMemsetAsync(c->counters.p, 0, 64, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->ref_d.p, c->chk_d.p, px * 4, cudaMemcpyDeviceToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->ref_v.p, c->chk_v.p, px, cudaMemcpyDeviceToDevice, c->stream));
    k_invalid_list<<<unsigned((px + 255) / 256), 256, 0, c->stream>>>(c->chk_d.as<float>(), c->chk_v.as<uint8_t>(), px,
                                                                      lim, c->counters.as<int>(), c->inv.as<int>());
    BSM_TRY(check_launch(c, "invalid_list"));
    int cnt[4];
    BSM_CUDA(cudaMemcpyAsync(cnt, c->counters.p, sizeof cnt, cudaMemcpyDeviceToHost, c->stream));
    BSM_TRY(sync(c));
    if (cnt[3]) return set_err(BSM_INVALID_ARGUMENT, "vote_refine: valid disparity out of range");
    max_bin = cnt[0];
    return BSM_OK;
}

// One pair of a batch in two phases: A (fields + WTA, keys set i % 2) on the
// context stream, then B (check + refine) on the high-priority s_ref, so that
// pair i's latency-bound refine runs beside pair i+1's descriptor / mask
// kernels (the block scheduler serves the higher-priority stream's CTAs as
// SMs free up).  Pair i+2's WTA waits until pair i's check has read that key
// set; phase B's buffers (check, refine, counters) are serial on s_ref.  After
// the call, s_ref holds pair i's remaining work (the caller appends its copies
// there); batch_join orders the context stream after all of it.
int batch_pair(bsm_ctx* c, int i, const Views& v, int W, int H, const bsm_params* params) {
    const int k = i & 1;
    if (i >= 2) BSM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_b[k], 0));  // key set k read by pair i-2
    BSM_TRY(pipeline_device(c, v, W, H, 0, H, params, false, 1, k == 1));
    BSM_CUDA(cudaEventRecord(c->ev_a[k], c->stream));
    BSM_CUDA(cudaStreamWaitEvent(c->s_ref, c->ev_a[k], 0));
    const cudaStream_t main = c->stream;
    c->stream = c->s_ref;
    c->in_batch = true;
    const int rc = pipeline_device(c, v, W, H, 0, H, params, false, 2, k == 1);
    c->in_batch = false;
    c->stream = main;
    BSM_TRY(rc);
    return cudaEventRecord(c->ev_b[k], c->s_ref) == cudaSuccess ? BSM_OK
                                                                : set_err(BSM_CUDA_ERROR, "CUDA: event record failed");
}

int batch_join(bsm_ctx* c) {
    BSM_CUDA(cudaEventRecord(c->ev_a[0], c->s_ref));
    BSM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_a[0], 0));
    return BSM_OK;
}

// Copy streams, events and the two slots of views / refined maps used to
// overlap pair i's compute with pair i+1's upload and pair i-1's download.
// slots: the host-buffer batch's two slots of device views and maps (the
// device batch needs only the streams, events and the second key set).
int ensure_batch(bsm_ctx* c, size_t px, bool slots = true) {
    if (!c->s_h2d) {
        BSM_CUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
        BSM_CUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
        for (int s = 0; s < 2; ++s)
            for (cudaEvent_t* e : {&c->ev_in[s], &c->ev_free[s], &c->ev_done[s], &c->ev_out[s], &c->ev_a[s], &c->ev_b[s]})
                BSM_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        int lo = 0, hi = 0;
        BSM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        BSM_CUDA(cudaStreamCreateWithPriority(&c->s_ref, cudaStreamNonBlocking, hi));
    }
    BSM_TRY(c->keys_l2.ensure(px * 4));
    BSM_TRY(c->keys_r2.ensure(px * 4));
    for (int s = 0; s < 2 && slots; ++s) {
        BSM_TRY(c->bimg[s][0].ensure(px));
        BSM_TRY(c->bimg[s][1].ensure(px));
        BSM_TRY(c->bout_d[s].ensure(px * 4));
        BSM_TRY(c->bout_v[s].ensure(px));
    }
    return BSM_OK;
}

int check_batch_ptrs(int n_pairs, const void* const* a, const void* const* b) {
    if (n_pairs < 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: n_pairs must be >= 0");
    if (n_pairs > 0 && (!a || !b)) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image array");
    for (int i = 0; i < n_pairs; ++i)
        if (!a[i] || !b[i]) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    return BSM_OK;
}

int check_dims(int W, int H) {
    if (W < 1 || H < 1) return set_err(BSM_INVALID_ARGUMENT, "bsm: image dimensions must be >= 1");
    if (int64_t(round_up(W, 128)) * H > (int64_t(1) << 31) - 1)  // field planes index pixels with int
        return set_err(BSM_UNSUPPORTED, "bsm: images above 2^31 pixels are outside this build's envelope");
    if (H > 65535) return set_err(BSM_UNSUPPORTED, "bsm: images taller than 65535 rows are outside this build's envelope");
    return BSM_OK;
}

}  // namespace

// ===========================================================================
// C ABI
extern "C" {

const char* bsm_last_error(void) { return g_err.c_str(); }
const char* bsm_version(void) { return "bsm-b200 0.1 (sm_100a)"; }

int bsm_ctx_create(int device, bsm_ctx** out) {
    if (!out) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return set_err(BSM_CUDA_ERROR, std::string("CUDA: no usable device (") + cudaGetErrorString(e) +
                                           "); this library has no CPU fallback");
    if (device < 0 || device >= ndev) return set_err(BSM_INVALID_ARGUMENT, "bsm: device index out of range");
    BSM_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    BSM_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_err(BSM_CUDA_ERROR, std::string("CUDA: built for sm_100a, device is ") + prop.name);
    {
        const char* g = std::getenv("BSM_GUARD");
        static bool once = (g_guard = g && g[0] == '1', true);
        (void)once;
    }
    bsm_ctx* c = new bsm_ctx();
    c->device = device;
    if (const char* v = std::getenv("BSM_K3_VARIANT")) c->k3_variant = std::atoi(v);
    if (const char* v = std::getenv("BSM_REFINE_CAP")) c->refine_cap = std::atoi(v);
    if (const char* v = std::getenv("BSM_K3_GROUP")) c->k3_group = std::atoi(v);
    if (const char* v = std::getenv("BSM_MASKF_FORCE_LOW")) c->maskf_force_low = std::atoi(v) != 0;
    if (const char* v = std::getenv("BSM_MASK_VARIANT")) c->mask_variant = std::atoi(v);
    if (const char* v = std::getenv("BSM_MASKQ_PX")) c->mq_px = std::atoi(v) == 32 ? 32 : std::atoi(v) == 8 ? 8 : 16;
    c->sm_count = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return set_err(BSM_CUDA_ERROR, "CUDA: stream creation failed");
    }
    for (int t = 0; t < T_COUNT; ++t)
        for (int s = 0; s < bsm_ctx::kEvPerSlot; ++s) {
            cudaEventCreate(&c->ev[t][s][0]);
            cudaEventCreate(&c->ev[t][s][1]);
        }
    bsmh::gray_lab_lut(c->gray_lut, c->lab_lut);
    for (int v = 1; v < 256; ++v)
        if (!(c->gray_lut[v] > c->gray_lut[v - 1])) {
            bsm_ctx_destroy(c);
            return set_err(BSM_UNSUPPORTED, "bsm: gray conversion table is not strictly increasing");
        }
    {
        bsmh::ExpParams ep;
        c->exp_ok = bsmh::glibc_exp_params(ep, c->exp_why);
        if (c->exp_ok) {
            c->exp_dev = ExpDev{ep.invln2N, ep.shift, ep.negln2hiN, ep.negln2loN, ep.c2, ep.c3, ep.c4, ep.c5};
            if (c->d_etab.ensure(sizeof ep.tab) != BSM_OK ||
                cudaMemcpy(c->d_etab.p, ep.tab, sizeof ep.tab, cudaMemcpyHostToDevice) != cudaSuccess)
                c->exp_ok = false;
        }
        if (c->d_lab256.ensure(sizeof c->lab_lut) != BSM_OK ||
            cudaMemcpy(c->d_lab256.p, c->lab_lut, sizeof c->lab_lut, cudaMemcpyHostToDevice) != cudaSuccess) {
            bsm_ctx_destroy(c);
            return set_err(BSM_CUDA_ERROR, "CUDA: Lab table upload failed");
        }
    }
    std::vector<uint8_t> rank(65536);
    bsmh::sad_rank_table(c->lab_lut, rank.data());
    int rc = c->d_rank.ensure(65536);
    if (rc == BSM_OK && cudaMemcpy(c->d_rank.p, rank.data(), 65536, cudaMemcpyHostToDevice) != cudaSuccess)
        rc = set_err(BSM_CUDA_ERROR, "CUDA: rank table upload failed");
    if (rc != BSM_OK) {
        bsm_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return BSM_OK;
}

int bsm_ctx_destroy(bsm_ctx* c) {
    if (!c) return BSM_OK;
    cudaSetDevice(c->device);
    for (DevBuf* b : ctx_bufs(c)) b->release();
    for (int s = 0; s < 2; ++s) {
        for (cudaEvent_t e : {c->ev_in[s], c->ev_free[s], c->ev_done[s], c->ev_out[s], c->ev_a[s], c->ev_b[s]})
            if (e) cudaEventDestroy(e);
    }
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_ref) cudaStreamDestroy(c->s_ref);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    for (int t = 0; t < T_COUNT; ++t)
        for (int s = 0; s < bsm_ctx::kEvPerSlot; ++s) {
            if (c->ev[t][s][0]) cudaEventDestroy(c->ev[t][s][0]);
            if (c->ev[t][s][1]) cudaEventDestroy(c->ev[t][s][1]);
        }
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return BSM_OK;
}

int bsm_generate_pattern(int n, int window, double spread, uint64_t seed, int16_t* out) {
    if (!out) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    std::string err;
    if (!bsmh::generate_pattern(n, window, spread, seed, out, err)) return set_err(BSM_INVALID_ARGUMENT, err);
    return BSM_OK;
}

int bsm_gray_lab_lut(float* gray256, float* lab768) {
    if (!gray256 || !lab768) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    bsmh::gray_lab_lut(gray256, lab768);
    return BSM_OK;
}

int bsm_to_gray_lab(const uint8_t* rgb, int W, int H, float* gray, float* lab) {
    if (!rgb) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    if (W < 1 || H < 1) return set_err(BSM_INVALID_ARGUMENT, "bsm: image dimensions must be >= 1");
    bsmh::to_gray_lab(rgb, size_t(W) * size_t(H), gray, lab);
    return BSM_OK;
}

int bsm_set_pattern(bsm_ctx* c, const int16_t* pairs, int n, int window) {
    if (!c || !pairs) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    if (n < 1) return set_err(BSM_INVALID_ARGUMENT, "pattern: n must be >= 1");
    if (window < 2) return set_err(BSM_INVALID_ARGUMENT, "pattern: window must be >= 2");
    if (n > kMaxPairs) return set_err(BSM_UNSUPPORTED, "bsm: n > 8192 is outside this build's envelope");
    if (window > 128) return set_err(BSM_UNSUPPORTED, "bsm: window > 128 is outside this build's envelope");
    const int half = window / 2, side = 2 * half + 1;
    for (int i = 0; i < 4 * n; ++i)
        if (pairs[i] < -half || pairs[i] > half)
            return set_err(BSM_INVALID_ARGUMENT, "pattern: offset outside window");
    BSM_CUDA(cudaSetDevice(c->device));
    // any failure below leaves the context without a pattern (n = 0), never
    // with a half-updated one; c->n is set last
    c->n = 0;
    c->window = window;
    c->half = half;
    c->NW = 2 * ((n + 63) / 64);
    c->pairs.assign(pairs, pairs + 4 * size_t(n));
    // Used window offsets (index into the (2h+1)^2 table, like
    // build_table_indices, descriptor.hpp:157-168) and per-pair endpoint
    // indices into that list.
    std::vector<int> slot(size_t(side) * side, -1);
    c->used.clear();
    std::vector<uint32_t> pq(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        int idx[2];
        for (int e = 0; e < 2; ++e) {
            const int t = (pairs[4 * i + 2 * e + 1] + half) * side + (pairs[4 * i + 2 * e] + half);
            if (slot[size_t(t)] < 0) {
                slot[size_t(t)] = int(c->used.size());
                c->used.push_back(int16_t(t));
            }
            idx[e] = slot[size_t(t)];
        }
        pq[size_t(i)] = uint32_t(idx[0]) | (uint32_t(idx[1]) << 16);
    }
    c->u = int(c->used.size());
    // k_mask4 / k_mask_f32 give each lane MCH chunks of 32 bit positions
    // (lane l: positions 32*MCH*l ..), MCH the smallest of 1, 2, 4, 8 that
    // holds n.  Otherwise the rank-table slots are placed by local search to
    // limit the gathers' bank conflicts.
    // For n = 1024 * MCH a bank-balanced pair order
    // (bsmh::balanced_gather_order) makes every gather conflict-free; the
    // descriptor bits follow the same order (the masked Hamming cost is
    // invariant under a common permutation of descriptor and mask bits) and
    // the per-stage API un-permutes.
    c->mch = n <= 1024 ? 1 : n <= 2048 ? 2 : n <= 4096 ? 4 : 8;
    const int lane_pos = 32 * c->mch;  // positions per lane
    std::vector<int> rslot(size_t(c->u));
    std::vector<uint8_t> flip;
    c->permuted = false;
    {
        int ns = 0;
        if (n == 32 * lane_pos && bsmh::balanced_gather_order(pq.data(), n, c->u, rslot, ns, c->order, flip)) {
            c->permuted = true;
            c->mslots = ns;
            c->slot_cost[0] = c->slot_cost[1] = 1.0;
        } else {
            rslot.assign(size_t(c->u), 0);
            c->mslots = round_up(c->u, 32) + 32;
            bsmh::place_rank_slots(pq.data(), n, c->u, c->mslots, lane_pos, rslot, &c->slot_cost[0],
                                   &c->slot_cost[1]);
        }
    }
    if (!c->permuted) {
        c->order.resize(size_t(n));
        for (int i = 0; i < n; ++i) c->order[size_t(i)] = i;
        flip.assign(size_t(n), 0);
    } else {
        std::vector<int> pos(static_cast<size_t>(n));
        for (int j = 0; j < n; ++j) pos[size_t(c->order[size_t(j)])] = j;
        BSM_TRY(c->d_pos.ensure(pos.size() * 4));
        BSM_CUDA(cudaMemcpy(c->d_pos.p, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice));
    }
    c->slot_used.assign(size_t(c->mslots), -1);
    for (int o = 0; o < c->u; ++o) c->slot_used[size_t(rslot[size_t(o)])] = o;
    // Byte offsets into the u32 rank table of each bit position's two
    // endpoints (k_mask4 / k_mask_f32): P table at [0, kPqTable), Q table at
    // [kPqTable, 2 kPqTable), lane-block order -- lane l, chunk m < MCH, t:
    // bit 32*MCH*l + 32m + t at uint4 [(m*8 + t%8)*32 + l], component t/8 for
    // MCH <= 4 (the four positions t, t+8, t+16, t+24 of one load land in the
    // four byte lanes of one word, so k_mask4's bit-plane transposes run across
    // words); [(m*8 + t/4)*32 + l], component t%4 for MCH = 8 (whose per-pixel
    // pass keeps the per-8-byte transposes to stay within 128 registers).
    // Pads read the sentinel.  For MCH <= 4, k_mask_f32 reads the packed table
    // at [2 kPqTable, 3 kPqTable): P | Q << 16 (mslots <= 2 * 4096 + 64 there,
    // so byte offsets fit 16 bits) -- half the L1 footprint of the gathers.
    if (c->mch <= 4 && 4 * c->mslots > 0xFFFF) return set_err(BSM_UNSUPPORTED, "bsm: rank-table offsets exceed 16 bits");
    std::vector<uint32_t> pqb(3 * kPqTable, uint32_t(4 * c->mslots));
    for (int i = 0; i < kPqTable; ++i) pqb[2 * kPqTable + i] = uint32_t(4 * c->mslots) * 65537u;
    for (int j = 0; j < n; ++j) {
        const int l = j / lane_pos, m = (j >> 5) % c->mch, t = j & 31;
        const size_t at = c->mch <= 4 ? (size_t(m * 8 + (t & 7)) * 32 + l) * 4 + (t >> 3)
                                      : (size_t(m * 8 + (t >> 2)) * 32 + l) * 4 + (t & 3);
        const uint32_t e = pq[size_t(c->order[size_t(j)])];
        const uint32_t a = flip[size_t(j)] ? e >> 16 : e & 0xFFFFu, b = flip[size_t(j)] ? e & 0xFFFFu : e >> 16;
        pqb[at] = uint32_t(4 * rslot[size_t(a)]);
        pqb[kPqTable + at] = uint32_t(4 * rslot[size_t(b)]);
        pqb[2 * kPqTable + at] = pqb[at] | (pqb[kPqTable + at] << 16);
    }
    BSM_TRY(c->d_pqb.ensure(pqb.size() * 4));
    BSM_CUDA(cudaMemcpy(c->d_pqb.p, pqb.data(), pqb.size() * 4, cudaMemcpyHostToDevice));
    c->desc4_tw = -1;
    c->descf_tw = -1;
    c->uoff_tw = -1;
    if (mask4_smem(c) > 200 * 1024 || maskf_smem(c) > 200 * 1024)
        return set_err(BSM_UNSUPPORTED, "bsm: pattern too large for shared-memory staging");
    c->n = n;  // committed: every table above is consistent with this pattern
    return BSM_OK;
}

// Device SoA field -> reference AoS words in c->aux0 (bit order restored).
static int soa_to_aos(bsm_ctx* c, const uint32_t* src, int W, int H) {
    const int Wq = field_pitch(W), tb = 256;
    const size_t P = field_plane(W, H);
    const size_t aos = size_t(H) * W * c->NW;
    if (c->permuted)
        k_soa_to_aos_perm<<<unsigned((aos + tb - 1) / tb), tb, 0, c->stream>>>(src, W, H, c->NW, Wq, P,
                                                                              c->d_pos.as<int>(), c->n,
                                                                              c->aux0.as<uint32_t>());
    else
        k_soa_to_aos<<<unsigned((aos + tb - 1) / tb), tb, 0, c->stream>>>(src, W, H, c->NW, Wq, P,
                                                                         c->aux0.as<uint32_t>());
    return check_launch(c, "soa_to_aos");
}

int bsm_compute_field_u8(bsm_ctx* c, const uint8_t* img, int W, int H, uint64_t* desc, uint64_t* mask) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    if (!img) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    const size_t fbytes = field_plane(W, H) * c->NW * 4;
    BSM_TRY(upload_views(c, img, nullptr, W, H));
    BSM_TRY(c->fdl.ensure(fbytes));
    BSM_TRY(c->fml.ensure(fbytes));
    BSM_TRY(field_device(c, c->img_l.as<uint8_t>(), W, H, 0, H, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>()));
    const size_t aos = size_t(H) * W * c->NW;
    BSM_TRY(c->aux0.ensure(aos * 4));
    for (int which = 0; which < 2; ++which) {
        uint64_t* dst = which == 0 ? desc : mask;
        if (!dst) continue;
        BSM_TRY(soa_to_aos(c, which == 0 ? c->fdl.as<uint32_t>() : c->fml.as<uint32_t>(), W, H));
        BSM_CUDA(cudaMemcpyAsync(dst, c->aux0.p, aos * 4, cudaMemcpyDeviceToHost, c->stream));
        BSM_TRY(sync(c));
    }
    return sync(c);
}

int bsm_wta(bsm_ctx* c, const uint64_t* desc_ref, const uint64_t* mask_ref, const uint64_t* desc_other, int W,
            int H, int n, int d_max, int right_ref, int use_mask, float* out_d) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_dims(W, H));
    if (!desc_ref || !desc_other || (use_mask && !mask_ref))
        return set_err(BSM_INVALID_ARGUMENT, "bsm: null field");
    if (d_max < 1) return set_err(BSM_INVALID_ARGUMENT, "wta: d_max must be >= 1");
    if (d_max > 65535) return set_err(BSM_UNSUPPORTED, "bsm: d_max > 65535 is outside this build's envelope");
    if (n < 1 || n > kMaxPairs) return set_err(BSM_UNSUPPORTED, "bsm: n outside [1, 8192]");
    const int NW = 2 * ((n + 63) / 64);
    const int savedNW = c->NW;
    c->NW = NW;
    const int Wq = field_pitch(W);
    const size_t P = field_plane(W, H);
    const size_t aos = size_t(H) * W * NW, soa = size_t(NW) * P;
    int rc = BSM_OK;
    do {
        if ((rc = c->aux0.ensure(aos * 4)) != BSM_OK) break;
        if ((rc = c->fdl.ensure(soa * 4)) != BSM_OK) break;
        if ((rc = c->fml.ensure(soa * 4)) != BSM_OK) break;
        if ((rc = c->fdr.ensure(soa * 4)) != BSM_OK) break;
        if ((rc = c->keys_l.ensure(size_t(H) * W * 4)) != BSM_OK) break;
        if ((rc = c->lw_d.ensure(size_t(H) * W * 4)) != BSM_OK) break;
        const int tb = 256;
        const uint64_t* srcs[3] = {desc_ref, use_mask ? mask_ref : nullptr, desc_other};
        DevBuf* dsts[3] = {&c->fdl, &c->fml, &c->fdr};
        for (int k = 0; k < 3 && rc == BSM_OK; ++k) {
            if (!srcs[k]) continue;
            if (cudaMemcpyAsync(c->aux0.p, srcs[k], aos * 4, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
                rc = set_err(BSM_CUDA_ERROR, "CUDA: field upload failed");
                break;
            }
            k_aos_to_soa<<<unsigned((soa + tb - 1) / tb), tb, 0, c->stream>>>(c->aux0.as<uint32_t>(), W, H, NW, Wq, P,
                                                                            dsts[k]->as<uint32_t>());
            rc = check_launch(c, "aos_to_soa");
            if (rc == BSM_OK) rc = sync(c);  // aux0 is reused by the next upload
        }
        if (rc != BSM_OK) break;
        // the reference field is fdl (+ fml) whichever the direction
        rc = right_ref ? wta_device(c, c->fdr.as<uint32_t>(), nullptr, c->fdl.as<uint32_t>(),
                                    use_mask ? c->fml.as<uint32_t>() : nullptr, W, H, d_max, false, 1, use_mask != 0,
                                    nullptr, c->keys_l.as<uint32_t>(), T_WTA)
                       : wta_device(c, c->fdl.as<uint32_t>(), use_mask ? c->fml.as<uint32_t>() : nullptr,
                                    c->fdr.as<uint32_t>(), nullptr, W, H, d_max, false, 0, use_mask != 0,
                                    c->keys_l.as<uint32_t>(), nullptr, T_WTA);
        if (rc != BSM_OK) break;
        const size_t px = size_t(H) * W;
        k_keys_to_float<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(c->keys_l.as<uint32_t>(), px,
                                                                          c->lw_d.as<float>());
        if ((rc = check_launch(c, "keys_to_float")) != BSM_OK) break;
        if (out_d && cudaMemcpyAsync(out_d, c->lw_d.p, px * 4, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) {
            rc = set_err(BSM_CUDA_ERROR, "CUDA: download failed");
            break;
        }
        rc = sync(c);
    } while (0);
    c->NW = savedNW;
    return rc;
}

int bsm_lr_check(bsm_ctx* c, const float* left_d, const float* right_d, int W, int H, double tol, float* out_d,
                 uint8_t* out_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_dims(W, H));
    if (!left_d || !right_d) return set_err(BSM_INVALID_ARGUMENT, "bsm: null map");
    const size_t px = size_t(W) * H;
    BSM_TRY(c->aux0.ensure(px * 4));
    BSM_TRY(c->aux1.ensure(px * 4));
    BSM_TRY(c->aux2.ensure(px * 4));
    BSM_TRY(c->aux3.ensure(px));
    BSM_CUDA(cudaMemcpyAsync(c->aux0.p, left_d, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->aux1.p, right_d, px * 4, cudaMemcpyHostToDevice, c->stream));
    const int tb = 256;
    k_lr_check_float<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(c->aux0.as<float>(), c->aux1.as<float>(), W,
                                                                       H, tol, c->aux2.as<float>(),
                                                                       c->aux3.as<uint8_t>());
    BSM_TRY(check_launch(c, "lr_check_float"));
    if (out_d) BSM_CUDA(cudaMemcpyAsync(out_d, c->aux2.p, px * 4, cudaMemcpyDeviceToHost, c->stream));
    if (out_v) BSM_CUDA(cudaMemcpyAsync(out_v, c->aux3.p, px, cudaMemcpyDeviceToHost, c->stream));
    return sync(c);
}

int bsm_vote_refine_u8(bsm_ctx* c, const float* d, const uint8_t* v, const uint8_t* gray_img, int W, int H,
                       double lambda_c, double lambda_e, int vote_radius, float* out_d, uint8_t* out_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_dims(W, H));
    if (!d || !v || !gray_img) return set_err(BSM_INVALID_ARGUMENT, "bsm: null input");
    if (!(lambda_c > 0)) return set_err(BSM_INVALID_ARGUMENT, "refine: lambda_c must be > 0");
    if (!(lambda_e > 0)) return set_err(BSM_INVALID_ARGUMENT, "refine: lambda_e must be > 0");
    if (vote_radius < 1) return set_err(BSM_INVALID_ARGUMENT, "refine: vote_radius must be >= 1");
    if (vote_radius > 180) return set_err(BSM_UNSUPPORTED, "bsm: vote_radius > 180 is outside this build's envelope");
    const size_t px = size_t(W) * H;
    BSM_TRY(c->img_l.ensure(px));
    BSM_TRY(c->chk_d.ensure(px * 4));
    BSM_TRY(c->chk_v.ensure(px));
    BSM_TRY(c->ref_d.ensure(px * 4));
    BSM_TRY(c->ref_v.ensure(px));
    BSM_TRY(c->counters.ensure(64));
    BSM_TRY(c->inv.ensure(std::max<size_t>(4, px * 4)));
    BSM_CUDA(cudaMemcpyAsync(c->img_l.p, gray_img, px, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->chk_d.p, d, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->chk_v.p, v, px, cudaMemcpyHostToDevice, c->stream));
    int max_bin = 0;
    BSM_TRY(invalid_list(c, px, 1e6, max_bin));
    if (max_bin + 1 > 12288) return set_err(BSM_UNSUPPORTED, "bsm: disparity range too large for the refine bins");
    BSM_TRY(refine_launch(c, c->chk_d.as<float>(), c->chk_v.as<uint8_t>(), c->img_l.as<uint8_t>(), nullptr, W, H,
                          vote_radius, max_bin + 1, lambda_c, lambda_e));
    if (out_d) BSM_CUDA(cudaMemcpyAsync(out_d, c->ref_d.p, px * 4, cudaMemcpyDeviceToHost, c->stream));
    if (out_v) BSM_CUDA(cudaMemcpyAsync(out_v, c->ref_v.p, px, cudaMemcpyDeviceToHost, c->stream));
    return sync(c);
}

int bsm_pipeline_u8(bsm_ctx* c, const uint8_t* left, const uint8_t* right, int W, int H, const bsm_params* params,
                    int want_unmasked, bsm_maps* out) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!left || !right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    BSM_TRY(upload_views(c, left, right, W, H));
    BSM_TRY(pipeline_device(c, u8views(c->img_l.as<uint8_t>(), c->img_r.as<uint8_t>()), W, H, 0, H, params,
                            want_unmasked != 0));
    BSM_TRY(fetch(c, out));
    return sync(c);
}

int bsm_pipeline_u8_device(bsm_ctx* c, const uint8_t* d_left, const uint8_t* d_right, int W, int H,
                           const bsm_params* params, int want_unmasked) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    if (!d_left || !d_right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    return pipeline_device(c, u8views(d_left, d_right), W, H, 0, H, params, want_unmasked != 0);
}

int bsm_fetch_maps(bsm_ctx* c, bsm_maps* out) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    if (c->last_W == 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: no pipeline result to fetch");
    BSM_TRY(fetch(c, out));
    return sync(c);
}

int bsm_pipeline_band_u8(bsm_ctx* c, const uint8_t* left, const uint8_t* right, int W, int H, int y0, int y1,
                         const bsm_params* params, float* refined_d, uint8_t* refined_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!left || !right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    if (y0 < 0 || y1 > H || y0 >= y1) return set_err(BSM_INVALID_ARGUMENT, "bsm: band rows out of range");
    BSM_TRY(upload_views(c, left, right, W, H));
    BSM_TRY(pipeline_device(c, u8views(c->img_l.as<uint8_t>(), c->img_r.as<uint8_t>()), W, H, y0, y1 - y0, params,
                            false));
    bsm_maps m = {};
    m.refined_d = refined_d;
    m.refined_v = refined_v;
    BSM_TRY(fetch(c, &m));
    return sync(c);
}

// run_pipeline(...).refined (pipeline.hpp:25-56) of every pair of a batch
// (BASELINE configs[3]).  Pair i's views are uploaded on the H2D stream while
// pair i-1 computes, and its refined map is downloaded on the D2H stream
// while pair i+1 computes; two slots of device views / maps alternate.
int bsm_pipeline_batch_u8(bsm_ctx* c, int n_pairs, const uint8_t* const* lefts, const uint8_t* const* rights, int W,
                          int H, const bsm_params* params, float* const* refined_d, uint8_t* const* refined_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    BSM_TRY(check_batch_ptrs(n_pairs, reinterpret_cast<const void* const*>(lefts),
                             reinterpret_cast<const void* const*>(rights)));
    if (n_pairs == 0) return BSM_OK;
    const size_t px = size_t(W) * H;
    BSM_TRY(ensure_batch(c, px));
    for (int i = 0; i < n_pairs; ++i) {
        const int s = i & 1;
        if (i >= 2) BSM_CUDA(cudaStreamWaitEvent(c->s_h2d, c->ev_free[s], 0));  // slot views consumed
        BSM_CUDA(cudaMemcpyAsync(c->bimg[s][0].p, lefts[i], px, cudaMemcpyHostToDevice, c->s_h2d));
        BSM_CUDA(cudaMemcpyAsync(c->bimg[s][1].p, rights[i], px, cudaMemcpyHostToDevice, c->s_h2d));
        BSM_CUDA(cudaEventRecord(c->ev_in[s], c->s_h2d));
        BSM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_in[s], 0));
        const Views v = u8views(c->bimg[s][0].as<uint8_t>(), c->bimg[s][1].as<uint8_t>());
        BSM_TRY(batch_pair(c, i, v, W, H, params));  // phase B of pair i on s_ref from here
        BSM_CUDA(cudaEventRecord(c->ev_free[s], c->s_ref));  // views consumed (the refine reads the left one)
        if (i >= 2) BSM_CUDA(cudaStreamWaitEvent(c->s_ref, c->ev_out[s], 0));  // slot map downloaded
        BSM_CUDA(cudaMemcpyAsync(c->bout_d[s].p, c->ref_d.p, px * 4, cudaMemcpyDeviceToDevice, c->s_ref));
        BSM_CUDA(cudaMemcpyAsync(c->bout_v[s].p, c->ref_v.p, px, cudaMemcpyDeviceToDevice, c->s_ref));
        BSM_CUDA(cudaEventRecord(c->ev_done[s], c->s_ref));
        BSM_CUDA(cudaStreamWaitEvent(c->s_d2h, c->ev_done[s], 0));
        if (refined_d && refined_d[i])
            BSM_CUDA(cudaMemcpyAsync(refined_d[i], c->bout_d[s].p, px * 4, cudaMemcpyDeviceToHost, c->s_d2h));
        if (refined_v && refined_v[i])
            BSM_CUDA(cudaMemcpyAsync(refined_v[i], c->bout_v[s].p, px, cudaMemcpyDeviceToHost, c->s_d2h));
        BSM_CUDA(cudaEventRecord(c->ev_out[s], c->s_d2h));
    }
    BSM_TRY(batch_join(c));
    BSM_CUDA(cudaStreamSynchronize(c->s_d2h));
    return sync(c);
}

// Device-resident batch: views and refined maps are device buffers (arrays of
// device pointers held on the host); stream-ordered on bsm_stream(), no sync.
int bsm_pipeline_batch_u8_device(bsm_ctx* c, int n_pairs, const uint8_t* const* d_lefts,
                                 const uint8_t* const* d_rights, int W, int H, const bsm_params* params,
                                 float* const* d_refined_d, uint8_t* const* d_refined_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    BSM_TRY(check_batch_ptrs(n_pairs, reinterpret_cast<const void* const*>(d_lefts),
                             reinterpret_cast<const void* const*>(d_rights)));
    const size_t px = size_t(W) * H;
    if (n_pairs == 0) return BSM_OK;
    BSM_TRY(ensure_batch(c, px, false));
    for (int i = 0; i < n_pairs; ++i) {
        BSM_TRY(batch_pair(c, i, u8views(d_lefts[i], d_rights[i]), W, H, params));
        if (d_refined_d && d_refined_d[i])
            BSM_CUDA(cudaMemcpyAsync(d_refined_d[i], c->ref_d.p, px * 4, cudaMemcpyDeviceToDevice, c->s_ref));
        if (d_refined_v && d_refined_v[i])
            BSM_CUDA(cudaMemcpyAsync(d_refined_v[i], c->ref_v.p, px, cudaMemcpyDeviceToDevice, c->s_ref));
    }
    return batch_join(c);
}

// Guard mode (BSM_GUARD=1): damaged guard bytes over every device buffer of
// the context after its queued work completes; *enabled = guard mode on.
int bsm_debug_check_guards(bsm_ctx* c, long long* damaged, int* enabled) {
    if (!c || !damaged) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    BSM_CUDA(cudaSetDevice(c->device));
    BSM_CUDA(cudaStreamSynchronize(c->stream));
    long long bad = 0;
    for (DevBuf* b : ctx_bufs(c)) bad += (long long)b->damaged();
    *damaged = bad;
    if (enabled) *enabled = g_guard ? 1 : 0;
    return BSM_OK;
}

// Make the context's stream wait for all work queued so far on `stream` (a
// cudaStream_t of the caller, e.g. the one that produced device inputs).
int bsm_stream_wait(bsm_ctx* c, void* stream) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    BSM_CUDA(cudaSetDevice(c->device));
    cudaEvent_t e;
    BSM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaError_t r = cudaEventRecord(e, static_cast<cudaStream_t>(stream));
    if (r == cudaSuccess) r = cudaStreamWaitEvent(c->stream, e, 0);
    cudaEventDestroy(e);
    if (r != cudaSuccess) return set_err(BSM_CUDA_ERROR, std::string("CUDA: stream wait: ") + cudaGetErrorString(r));
    return BSM_OK;
}

int bsm_device_exp(bsm_ctx* c, const double* x, int n, double* out) {
    BSM_TRY(begin_call(c));
    if (!x || !out || n < 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: bad arguments");
    if (!c->exp_ok) return set_err(BSM_UNSUPPORTED, "bsm: device exp unavailable (" + c->exp_why + ")");
    if (n == 0) return BSM_OK;
    BSM_TRY(c->aux0.ensure(size_t(n) * 8));
    BSM_TRY(c->aux1.ensure(size_t(n) * 8));
    BSM_CUDA(cudaMemcpyAsync(c->aux0.p, x, size_t(n) * 8, cudaMemcpyHostToDevice, c->stream));
    k_exp_eval<<<(n + 255) / 256, 256, 0, c->stream>>>(c->aux0.as<double>(), n, c->exp_dev,
                                                       c->d_etab.as<unsigned long long>(), c->aux1.as<double>());
    BSM_TRY(check_launch(c, "exp_eval"));
    BSM_CUDA(cudaMemcpyAsync(out, c->aux1.p, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    return sync(c);
}

int bsm_vote_refine_lab(bsm_ctx* c, const float* d, const uint8_t* v, const float* lab, int W, int H,
                        double lambda_c, double lambda_e, int vote_radius, float* out_d, uint8_t* out_v) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_dims(W, H));
    if (!d || !v || !lab) return set_err(BSM_INVALID_ARGUMENT, "bsm: null input");
    if (!(lambda_c > 0)) return set_err(BSM_INVALID_ARGUMENT, "refine: lambda_c must be > 0");
    if (!(lambda_e > 0)) return set_err(BSM_INVALID_ARGUMENT, "refine: lambda_e must be > 0");
    if (vote_radius < 1) return set_err(BSM_INVALID_ARGUMENT, "refine: vote_radius must be >= 1");
    if (vote_radius > 180) return set_err(BSM_UNSUPPORTED, "bsm: vote_radius > 180 is outside this build's envelope");
    const size_t px = size_t(W) * H;
    BSM_TRY(c->img_l.ensure(px));
    BSM_TRY(c->aux2.ensure(px * 12));
    BSM_TRY(c->aux3.ensure(px * 16));
    BSM_TRY(c->chk_d.ensure(px * 4));
    BSM_TRY(c->chk_v.ensure(px));
    BSM_TRY(c->ref_d.ensure(px * 4));
    BSM_TRY(c->ref_v.ensure(px));
    BSM_TRY(c->counters.ensure(64));
    BSM_TRY(c->inv.ensure(std::max<size_t>(4, px * 4)));
    BSM_CUDA(cudaMemsetAsync(c->img_l.p, 0, px, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->aux2.p, lab, px * 12, cudaMemcpyHostToDevice, c->stream));
    k_lab3_to_lab4<<<unsigned((px + 255) / 256), 256, 0, c->stream>>>(c->aux2.as<float>(), px, c->aux3.as<float4>());
    BSM_TRY(check_launch(c, "lab3_to_lab4"));
    BSM_CUDA(cudaMemcpyAsync(c->chk_d.p, d, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(c->chk_v.p, v, px, cudaMemcpyHostToDevice, c->stream));
    int max_bin = 0;
    BSM_TRY(invalid_list(c, px, 65535.0, max_bin));
    BSM_TRY(refine_launch(c, c->chk_d.as<float>(), c->chk_v.as<uint8_t>(), c->img_l.as<uint8_t>(), c->aux3.as<float4>(),
                          W, H, vote_radius, max_bin + 1, lambda_c, lambda_e));
    if (out_d) BSM_CUDA(cudaMemcpyAsync(out_d, c->ref_d.p, px * 4, cudaMemcpyDeviceToHost, c->stream));
    if (out_v) BSM_CUDA(cudaMemcpyAsync(out_v, c->ref_v.p, px, cudaMemcpyDeviceToHost, c->stream));
    return sync(c);
}

int bsm_set_refine_mode(bsm_ctx* c, int mode) {
    if (!c || mode < -1 || mode > 4 || mode == 0 || mode == 1)
        return set_err(BSM_INVALID_ARGUMENT, "bsm: bad refine mode");
    c->refine_mode = mode;
    return BSM_OK;
}

int bsm_pipeline_band_u8_device(bsm_ctx* c, const uint8_t* d_left, const uint8_t* d_right, int W, int H, int y0,
                                 int y1, const bsm_params* params) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!d_left || !d_right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    if (y0 < 0 || y1 > H || y0 >= y1) return set_err(BSM_INVALID_ARGUMENT, "bsm: band rows out of range");
    return pipeline_device(c, u8views(d_left, d_right), W, H, y0, y1 - y0, params, false);
}

int bsm_result_device(bsm_ctx* c, const float** refined_d, const uint8_t** refined_v, int* row0, int* nrows) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    if (c->last_W == 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: no pipeline result");
    const size_t off = size_t(c->last_out0 - c->last_r0) * c->last_W;
    if (refined_d) *refined_d = c->ref_d.as<float>() + off;
    if (refined_v) *refined_v = c->ref_v.as<uint8_t>() + off;
    if (row0) *row0 = c->last_out0;
    if (nrows) *nrows = c->last_out_rows;
    return BSM_OK;
}

int bsm_copy_result_device(bsm_ctx* c, float* dst_d, uint8_t* dst_v) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    if (c->last_W == 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: no pipeline result");
    const size_t off = size_t(c->last_out0 - c->last_r0) * c->last_W;
    const size_t n = size_t(c->last_out_rows) * c->last_W;
    if (dst_d) BSM_CUDA(cudaMemcpyAsync(dst_d, c->ref_d.as<float>() + off, n * 4, cudaMemcpyDeviceToDevice, c->stream));
    if (dst_v) BSM_CUDA(cudaMemcpyAsync(dst_v, c->ref_v.as<uint8_t>() + off, n, cudaMemcpyDeviceToDevice, c->stream));
    return BSM_OK;
}

int bsm_rgb24_tables(float* gray, float* lab) {
    if (!gray || !lab) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    std::vector<float> g, l;
    bsmh::rgb24_tables(g, l);
    std::memcpy(gray, g.data(), g.size() * 4);
    std::memcpy(lab, l.data(), l.size() * 4);
    return BSM_OK;
}

int bsm_compute_field_f32(bsm_ctx* c, const float* gray, const float* lab, int W, int H, uint64_t* desc,
                          uint64_t* mask) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    if (!gray || !lab) return set_err(BSM_INVALID_ARGUMENT, "bsm: null plane");
    const size_t px = size_t(W) * H;
    const size_t fbytes = field_plane(W, H) * c->NW * 4;
    BSM_TRY(c->planes.ensure(px * 32));
    float* g = c->planes.as<float>();
    float* l3 = g + px;
    float4* l = reinterpret_cast<float4*>(g + 4 * px);  // 16-B aligned (planes is cudaMalloc'd)
    BSM_CUDA(cudaMemcpyAsync(g, gray, px * 4, cudaMemcpyHostToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(l3, lab, px * 12, cudaMemcpyHostToDevice, c->stream));
    k_lab3_to_lab4<<<unsigned((px + 255) / 256), 256, 0, c->stream>>>(l3, px, l);
    BSM_TRY(check_launch(c, "lab3_to_lab4"));
    BSM_TRY(c->fdl.ensure(fbytes));
    BSM_TRY(c->fml.ensure(fbytes));
    BSM_TRY(field_device_f32(c, g, l, W, H, 0, H, c->fdl.as<uint32_t>(), c->fml.as<uint32_t>()));
    const size_t aos = size_t(H) * W * c->NW;
    BSM_TRY(c->aux0.ensure(aos * 4));
    for (int which = 0; which < 2; ++which) {
        uint64_t* dst = which == 0 ? desc : mask;
        if (!dst) continue;
        BSM_TRY(soa_to_aos(c, which == 0 ? c->fdl.as<uint32_t>() : c->fml.as<uint32_t>(), W, H));
        BSM_CUDA(cudaMemcpyAsync(dst, c->aux0.p, aos * 4, cudaMemcpyDeviceToHost, c->stream));
        BSM_TRY(sync(c));
    }
    return sync(c);
}

// Colour pair already on the device: RGB -> gray/Lab planes, then the fused pipeline.
static int rgb_pipeline(bsm_ctx* c, const uint8_t* d_left, const uint8_t* d_right, int W, int H,
                        const bsm_params* params, bool want_unmasked) {
    BSM_TRY(ensure_rgb_tables(c));
    const size_t px = size_t(W) * H;
    const size_t lab_off = (2 * px + 3) / 4 * 4;  // floats; keeps the float4 planes 16-B aligned
    BSM_TRY(c->planes.ensure((lab_off + 8 * px) * 4));
    Views v;
    float* base = c->planes.as<float>();
    float4* lab4 = reinterpret_cast<float4*>(base + lab_off);
    v.gl = base;
    v.gr = base + px;
    v.ll = lab4;
    v.lr = lab4 + px;
    {
        Scope s(c, T_DESC);  // the conversion is accounted with the descriptor stage
        const int tb = 256;
        k_rgb_planes<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(d_left, px, c->d_rgb_gray.as<float>(),
                                                                      c->d_rgb_lab.as<float>(), base, lab4);
        BSM_TRY(check_launch(c, "rgb_planes"));
        k_rgb_planes<<<unsigned((px + tb - 1) / tb), tb, 0, c->stream>>>(d_right, px, c->d_rgb_gray.as<float>(),
                                                                      c->d_rgb_lab.as<float>(), base + px,
                                                                      lab4 + px);
        BSM_TRY(check_launch(c, "rgb_planes"));
    }
    return pipeline_device(c, v, W, H, 0, H, params, want_unmasked);
}

int bsm_pipeline_rgb(bsm_ctx* c, const uint8_t* left, const uint8_t* right, int W, int H, const bsm_params* params,
                     int want_unmasked, bsm_maps* out) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!left || !right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    const size_t px = size_t(W) * H;
    BSM_TRY(c->img_l.ensure(px * 3));
    BSM_TRY(c->img_r.ensure(px * 3));
    {
        Scope s(c, T_H2D);
        BSM_CUDA(cudaMemcpyAsync(c->img_l.p, left, px * 3, cudaMemcpyHostToDevice, c->stream));
        BSM_CUDA(cudaMemcpyAsync(c->img_r.p, right, px * 3, cudaMemcpyHostToDevice, c->stream));
    }
    BSM_TRY(rgb_pipeline(c, c->img_l.as<uint8_t>(), c->img_r.as<uint8_t>(), W, H, params, want_unmasked != 0));
    BSM_TRY(fetch(c, out));
    return sync(c);
}

int bsm_pipeline_rgb_device(bsm_ctx* c, const uint8_t* d_left, const uint8_t* d_right, int W, int H,
                            const bsm_params* params, int want_unmasked) {
    BSM_TRY(begin_call(c));
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!d_left || !d_right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    return rgb_pipeline(c, d_left, d_right, W, H, params, want_unmasked != 0);
}

int bsm_stream(bsm_ctx* c, void** stream) {
    if (!c || !stream) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    *stream = c->stream;
    return BSM_OK;
}

int bsm_set_profiling(bsm_ctx* c, int enable) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null context");
    c->profiling = enable != 0;
    return BSM_OK;
}

int bsm_last_timings(bsm_ctx* c, float* ms, int max, int* count) {
    if (!c || !ms) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    BSM_CUDA(cudaStreamSynchronize(c->stream));
    const int k = std::min(max, int(T_COUNT));
    for (int t = 0; t < k; ++t) {
        ms[t] = 0.0f;
        for (int s = 0; s < c->ev_used[t]; ++s) {
            float v = 0.0f;
            cudaEventElapsedTime(&v, c->ev[t][s][0], c->ev[t][s][1]);
            ms[t] += v;
        }
    }
    if (count) *count = k;
    return BSM_OK;
}

const char* bsm_timing_names(void) { return kTimingNames; }

int bsm_last_launch_count(bsm_ctx* c, int* count) {
    if (!c || !count) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    *count = c->launches;
    return BSM_OK;
}

int bsm_measure_popc_peak(bsm_ctx* c, double* ops_per_s) {
    return bsm_measure_word_peaks(c, ops_per_s, nullptr);
}

int bsm_measure_mma_peak(bsm_ctx* c, double* flops_per_s) {
    if (!c || !flops_per_s) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    BSM_CUDA(cudaSetDevice(c->device));
    const int iters = 65536;
    BSM_TRY(c->popc_out.ensure(size_t(c->sm_count) * 4));
    BSM_CUDA(cudaFuncSetAttribute(k_mxf4_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
    cudaEvent_t e0, e1;
    BSM_CUDA(cudaEventCreate(&e0));
    BSM_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0, c->stream);
        // 120 KB of dynamic shared memory: one CTA (and one TMEM allocation) per SM
        k_mxf4_peak<<<c->sm_count, 128, 120 * 1024, c->stream>>>(iters, c->popc_out.as<uint32_t>());
        cudaEventRecord(e1, c->stream);
        BSM_CUDA(cudaEventSynchronize(e1));
        BSM_CUDA(cudaGetLastError());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0) best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *flops_per_s = 2.0 * 128 * 256 * 64 * double(iters) * c->sm_count / (double(best) * 1e-3);
    return BSM_OK;
}

int bsm_measure_word_peaks(bsm_ctx* c, double* popc_words_per_s, double* csa_words_per_s) {
    if (!c) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    BSM_CUDA(cudaSetDevice(c->device));
    const int blocks = c->sm_count * 4, threads = 512, iters = 8192;
    BSM_TRY(c->popc_out.ensure(size_t(blocks) * threads * 4));
    cudaEvent_t e0, e1;
    BSM_CUDA(cudaEventCreate(&e0));
    BSM_CUDA(cudaEventCreate(&e1));
    for (int kind = 0; kind < 2; ++kind) {
        double* dst = kind == 0 ? popc_words_per_s : csa_words_per_s;
        if (!dst) continue;
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
            cudaEventRecord(e0, c->stream);
            if (kind == 0) k_popc_peak<<<blocks, threads, 0, c->stream>>>(c->popc_out.as<uint32_t>(), 7u + r, iters);
            else k_csa_peak<<<blocks, threads, 0, c->stream>>>(c->popc_out.as<uint32_t>(), 7u + r, iters, 2u);
            cudaEventRecord(e1, c->stream);
            BSM_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0) best = std::min(best, ms);
        }
        const double words = double(blocks) * threads * iters * 8 * (kind == 0 ? 1 : 2);
        *dst = words / (double(best) * 1e-3);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return BSM_OK;
}

}  // extern "C"

#include "bsm_dist.cuh"
