// bsm_dist.cuh -- the multi-GPU partitions of the matching path over NCCL
// (SURVEY.md 8(e)), part of bsm_kernels.cu's translation unit.  C ABI:
// include/bsm_cuda.h "Multi-GPU".
//
//  * one frame, row bands (BASELINE configs[4]): rank r computes rows
//    band_rows(H, world, r) with a local vote-radius halo of redundant rows
//    (no halo exchange), then one ncclAllGather of the padded refined bands;
//  * a batch of pairs (configs[3]): rank r computes shard_units(n, world, r)
//    (independent units, no data-path collective) and the refined maps are
//    gathered to one root rank with ncclSend / ncclRecv.
// The reference parallelises with parallel_for over rows and guarantees that
// the output does not depend on the worker count (parallel.hpp:12-14); both
// partitions keep that: every pixel is computed from the same full-frame
// inputs with the same arithmetic.
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: in a PyTorch process
// the copy torch already mapped), so the core library has no link-time NCCL
// dependency; without it the entry points return BSM_NCCL_ERROR.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
    bool tried = false, ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi a;
    static std::mutex m;
    std::lock_guard<std::mutex> g(m);
    if (a.tried) return a;
    a.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        a.why = std::string("libnccl.so.2 not loadable: ") + (dlerror() ? dlerror() : "?");
        return a;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        all = all && fn != nullptr;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    if (!all) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
}

#define BSM_NCCL(call)                                                                                  \
    do {                                                                                                \
        ncclResult_t r_ = (call);                                                                       \
        if (r_ != ncclSuccess)                                                                          \
            return set_err(BSM_NCCL_ERROR, std::string("NCCL: ") + nccl().GetErrorString(r_) + " at " #call); \
    } while (0)

// Contiguous row band [y0, y1) of `rank` (sizes differ by at most one row);
// the same formula as paper_1402_2020_b200.dist.band_rows.
void band_of(int n, int world, int rank, int& y0, int& y1) {
    const int base = n / world, extra = n % world;
    y0 = rank * base + std::min(rank, extra);
    y1 = y0 + base + (rank < extra ? 1 : 0);
}

}  // namespace

struct bsm_comm {
    bsm_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int device = 0, world = 1, rank = 0;
    DevBuf send_d, send_v, recv_d, recv_v, shard_d, shard_v;
};

extern "C" {

int bsm_comm_unique_id(uint8_t* id) {
    if (!id) return set_err(BSM_INVALID_ARGUMENT, "bsm: null output pointer");
    NcclApi& a = nccl();
    if (!a.ok) return set_err(BSM_NCCL_ERROR, "NCCL: " + a.why);
    ncclUniqueId u;
    BSM_NCCL(a.GetUniqueId(&u));
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return BSM_OK;
}

int bsm_comm_create(bsm_ctx* c, const uint8_t* id, int world, int rank, bsm_comm** out) {
    if (!c || !id || !out) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return set_err(BSM_INVALID_ARGUMENT, "bsm: bad world size or rank");
    NcclApi& a = nccl();
    if (!a.ok) return set_err(BSM_NCCL_ERROR, "NCCL: " + a.why);
    BSM_CUDA(cudaSetDevice(c->device));
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm = nullptr;
    BSM_NCCL(a.CommInitRank(&comm, world, u, rank));
    bsm_comm* m = new bsm_comm();
    m->ctx = c;
    m->device = c->device;
    m->comm = comm;
    m->world = world;
    m->rank = rank;
    *out = m;
    return BSM_OK;
}

int bsm_comm_destroy(bsm_comm* m) {
    if (!m) return BSM_OK;
    cudaSetDevice(m->device);
    for (DevBuf* b : {&m->send_d, &m->send_v, &m->recv_d, &m->recv_v, &m->shard_d, &m->shard_v}) b->release();
    if (m->comm) nccl().CommDestroy(m->comm);
    delete m;
    return BSM_OK;
}

int bsm_pipeline_frame_bands_u8(bsm_ctx* c, bsm_comm* m, const uint8_t* left, const uint8_t* right, int W, int H,
                                const bsm_params* params, float* refined_d, uint8_t* refined_v) {
    BSM_TRY(begin_call(c));
    if (!m || m->ctx != c) return set_err(BSM_INVALID_ARGUMENT, "bsm: communicator does not belong to this context");
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (!left || !right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    if (H < m->world) return set_err(BSM_INVALID_ARGUMENT, "bsm: fewer rows than ranks");
    int y0, y1;
    band_of(H, m->world, m->rank, y0, y1);
    const int rows_max = (H + m->world - 1) / m->world;
    const size_t band_px = size_t(rows_max) * W;
    BSM_TRY(upload_views(c, left, right, W, H));
    BSM_TRY(pipeline_device(c, u8views(c->img_l.as<uint8_t>(), c->img_r.as<uint8_t>()), W, H, y0, y1 - y0, params,
                            false));
    BSM_TRY(m->send_d.ensure(band_px * 4));
    BSM_TRY(m->send_v.ensure(band_px));
    BSM_TRY(m->recv_d.ensure(band_px * 4 * m->world));
    BSM_TRY(m->recv_v.ensure(band_px * m->world));
    const size_t off = size_t(c->last_out0 - c->last_r0) * W, mine = size_t(y1 - y0) * W;
    BSM_CUDA(cudaMemcpyAsync(m->send_d.p, c->ref_d.as<float>() + off, mine * 4, cudaMemcpyDeviceToDevice, c->stream));
    BSM_CUDA(cudaMemcpyAsync(m->send_v.p, c->ref_v.as<uint8_t>() + off, mine, cudaMemcpyDeviceToDevice, c->stream));
    NcclApi& a = nccl();
    BSM_NCCL(a.GroupStart());
    BSM_NCCL(a.AllGather(m->send_d.p, m->recv_d.p, band_px, ncclFloat32, m->comm, c->stream));
    BSM_NCCL(a.AllGather(m->send_v.p, m->recv_v.p, band_px, ncclUint8, m->comm, c->stream));
    BSM_NCCL(a.GroupEnd());
    for (int r = 0; r < m->world; ++r) {  // each rank's band sits at r * band_px in the receive buffer
        int b0, b1;
        band_of(H, m->world, r, b0, b1);
        const size_t n = size_t(b1 - b0) * W;
        if (refined_d)
            BSM_CUDA(cudaMemcpyAsync(refined_d + size_t(b0) * W, m->recv_d.as<float>() + size_t(r) * band_px, n * 4,
                                     cudaMemcpyDeviceToHost, c->stream));
        if (refined_v)
            BSM_CUDA(cudaMemcpyAsync(refined_v + size_t(b0) * W, m->recv_v.as<uint8_t>() + size_t(r) * band_px, n,
                                     cudaMemcpyDeviceToHost, c->stream));
    }
    return sync(c);
}

int bsm_pipeline_pairs_sharded_u8(bsm_ctx* c, bsm_comm* m, int n_pairs, const uint8_t* const* lefts,
                                  const uint8_t* const* rights, int W, int H, const bsm_params* params, int root,
                                  float* const* refined_d, uint8_t* const* refined_v) {
    BSM_TRY(begin_call(c));
    if (!m || m->ctx != c) return set_err(BSM_INVALID_ARGUMENT, "bsm: communicator does not belong to this context");
    BSM_TRY(check_pattern(c));
    BSM_TRY(check_dims(W, H));
    BSM_TRY(validate_params(params));
    if (root < 0 || root >= m->world) return set_err(BSM_INVALID_ARGUMENT, "bsm: root rank out of range");
    if (n_pairs < 0) return set_err(BSM_INVALID_ARGUMENT, "bsm: n_pairs must be >= 0");
    int u0, u1;
    band_of(n_pairs, m->world, m->rank, u0, u1);
    for (int i = u0; i < u1; ++i)
        if (!lefts || !rights || !lefts[i] || !rights[i]) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    const size_t px = size_t(W) * H;
    int per = 0;  // largest shard: the fixed message size of the gather
    for (int r = 0; r < m->world; ++r) {
        int a0, a1;
        band_of(n_pairs, m->world, r, a0, a1);
        per = std::max(per, a1 - a0);
    }
    if (per == 0) return BSM_OK;
    BSM_TRY(m->shard_d.ensure(size_t(per) * px * 4));
    BSM_TRY(m->shard_v.ensure(size_t(per) * px));
    const bool is_root = m->rank == root;
    if (is_root) {
        BSM_TRY(m->recv_d.ensure(size_t(per) * px * 4 * m->world));
        BSM_TRY(m->recv_v.ensure(size_t(per) * px * m->world));
    }
    if (u1 > u0) {
        BSM_TRY(ensure_batch(c, px));
        for (int i = u0; i < u1; ++i) {  // uploads overlap the previous pair's compute
            const int s = (i - u0) & 1;
            if (i - u0 >= 2) BSM_CUDA(cudaStreamWaitEvent(c->s_h2d, c->ev_free[s], 0));
            BSM_CUDA(cudaMemcpyAsync(c->bimg[s][0].p, lefts[i], px, cudaMemcpyHostToDevice, c->s_h2d));
            BSM_CUDA(cudaMemcpyAsync(c->bimg[s][1].p, rights[i], px, cudaMemcpyHostToDevice, c->s_h2d));
            BSM_CUDA(cudaEventRecord(c->ev_in[s], c->s_h2d));
            BSM_CUDA(cudaStreamWaitEvent(c->stream, c->ev_in[s], 0));
            // two phases per pair (batch_pair): this pair's refine beside the next one's fields
            BSM_TRY(batch_pair(c, i - u0, u8views(c->bimg[s][0].as<uint8_t>(), c->bimg[s][1].as<uint8_t>()), W, H,
                               params));
            BSM_CUDA(cudaEventRecord(c->ev_free[s], c->s_ref));
            const size_t k = size_t(i - u0);
            BSM_CUDA(cudaMemcpyAsync(m->shard_d.as<float>() + k * px, c->ref_d.p, px * 4, cudaMemcpyDeviceToDevice,
                                     c->s_ref));
            BSM_CUDA(cudaMemcpyAsync(m->shard_v.as<uint8_t>() + k * px, c->ref_v.p, px, cudaMemcpyDeviceToDevice,
                                     c->s_ref));
        }
        BSM_TRY(batch_join(c));
    }
    NcclApi& a = nccl();
    const float* own_d = m->shard_d.as<float>();
    const uint8_t* own_v = m->shard_v.as<uint8_t>();
    if (!is_root) {
        if (u1 > u0) {
            BSM_NCCL(a.GroupStart());
            BSM_NCCL(a.Send(own_d, size_t(u1 - u0) * px, ncclFloat32, root, m->comm, c->stream));
            BSM_NCCL(a.Send(own_v, size_t(u1 - u0) * px, ncclUint8, root, m->comm, c->stream));
            BSM_NCCL(a.GroupEnd());
        }
        return sync(c);
    }
    BSM_NCCL(a.GroupStart());
    for (int r = 0; r < m->world; ++r) {
        int a0, a1;
        band_of(n_pairs, m->world, r, a0, a1);
        if (r == root || a1 == a0) continue;
        BSM_NCCL(a.Recv(m->recv_d.as<float>() + size_t(r) * per * px, size_t(a1 - a0) * px, ncclFloat32, r, m->comm,
                        c->stream));
        BSM_NCCL(a.Recv(m->recv_v.as<uint8_t>() + size_t(r) * per * px, size_t(a1 - a0) * px, ncclUint8, r, m->comm,
                        c->stream));
    }
    BSM_NCCL(a.GroupEnd());
    for (int r = 0; r < m->world; ++r) {
        int a0, a1;
        band_of(n_pairs, m->world, r, a0, a1);
        const float* src_d = r == root ? own_d : m->recv_d.as<float>() + size_t(r) * per * px;
        const uint8_t* src_v = r == root ? own_v : m->recv_v.as<uint8_t>() + size_t(r) * per * px;
        for (int i = a0; i < a1; ++i) {
            const size_t k = size_t(i - a0);
            if (refined_d && refined_d[i])
                BSM_CUDA(cudaMemcpyAsync(refined_d[i], src_d + k * px, px * 4, cudaMemcpyDeviceToHost, c->stream));
            if (refined_v && refined_v[i])
                BSM_CUDA(cudaMemcpyAsync(refined_v[i], src_v + k * px, px, cudaMemcpyDeviceToHost, c->stream));
        }
    }
    return sync(c);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// One frame over peer memory (BASELINE configs[4], the B200-first variant of
// bsm_pipeline_frame_bands_u8): every rank owns a full-frame refined map in
// device memory, exported with CUDA IPC; the ranks exchange the handles out of
// band and map each other's maps; each rank's left/right check (K5) and
// voting refinement (K6) then store its band's final values straight into
// every rank's map over NVLink (P2P stores), so the all-gather is fused into
// the kernels that produce the band -- no collective launch, no staging
// buffer.  No kernel waits on another rank: the caller's barrier after the
// call orders the stores before any rank reads its map (bsm_frame_fetch).
struct bsm_frame {
    bsm_ctx* ctx = nullptr;
    int device = 0, W = 0, H = 0, world = 1, rank = 0;
    float* d = nullptr;
    uint8_t* v = nullptr;
    float* peer_d[kMaxPeers] = {};
    uint8_t* peer_v[kMaxPeers] = {};
    bool attached = false;
};

extern "C" {

int bsm_frame_create(bsm_ctx* c, int W, int H, int world, int rank, bsm_frame** out, uint8_t* handle) {
    if (!c || !out || !handle) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    *out = nullptr;
    BSM_TRY(check_dims(W, H));
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world)
        return set_err(world > kMaxPeers ? BSM_UNSUPPORTED : BSM_INVALID_ARGUMENT,
                       "bsm: peer-memory frames take 1 to 8 ranks");
    if (H < world) return set_err(BSM_INVALID_ARGUMENT, "bsm: fewer rows than ranks");
    BSM_CUDA(cudaSetDevice(c->device));
    bsm_frame* f = new bsm_frame();
    f->ctx = c;
    f->device = c->device;
    f->W = W;
    f->H = H;
    f->world = world;
    f->rank = rank;
    const size_t px = size_t(W) * H;
    cudaIpcMemHandle_t hd, hv;
    cudaError_t e = cudaMalloc(&f->d, px * 4);
    if (e == cudaSuccess) e = cudaMalloc(&f->v, px);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hd, f->d);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hv, f->v);
    if (e != cudaSuccess) {
        bsm_frame_destroy(f);
        return set_err(BSM_CUDA_ERROR, std::string("CUDA: frame allocation / IPC export: ") + cudaGetErrorString(e));
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    std::memcpy(handle, &hd, 64);
    std::memcpy(handle + 64, &hv, 64);
    *out = f;
    return BSM_OK;
}

int bsm_frame_attach(bsm_frame* f, const uint8_t* handles) {
    if (!f || !handles) return set_err(BSM_INVALID_ARGUMENT, "bsm: null argument");
    if (f->attached) return set_err(BSM_INVALID_ARGUMENT, "bsm: frame already attached");
    BSM_CUDA(cudaSetDevice(f->device));
    for (int r = 0; r < f->world; ++r) {
        if (r == f->rank) {
            f->peer_d[r] = f->d;
            f->peer_v[r] = f->v;
            continue;
        }
        cudaIpcMemHandle_t hd, hv;
        std::memcpy(&hd, handles + size_t(r) * 128, 64);
        std::memcpy(&hv, handles + size_t(r) * 128 + 64, 64);
        void *pd = nullptr, *pv = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&pd, hd, cudaIpcMemLazyEnablePeerAccess);
        if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&pv, hv, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess)
            return set_err(BSM_CUDA_ERROR, std::string("CUDA: opening rank ") + std::to_string(r) +
                                               "'s frame: " + cudaGetErrorString(e));
        f->peer_d[r] = static_cast<float*>(pd);
        f->peer_v[r] = static_cast<uint8_t*>(pv);
    }
    f->attached = true;
    return BSM_OK;
}

int bsm_pipeline_frame_bands_p2p_u8(bsm_ctx* c, bsm_frame* f, const uint8_t* left, const uint8_t* right,
                                    const bsm_params* params) {
    BSM_TRY(begin_call(c));
    if (!f || f->ctx != c) return set_err(BSM_INVALID_ARGUMENT, "bsm: frame does not belong to this context");
    if (!f->attached) return set_err(BSM_INVALID_ARGUMENT, "bsm: frame not attached (bsm_frame_attach)");
    BSM_TRY(check_pattern(c));
    BSM_TRY(validate_params(params));
    if (!left || !right) return set_err(BSM_INVALID_ARGUMENT, "bsm: null image");
    const int W = f->W, H = f->H;
    int y0, y1;
    band_of(H, f->world, f->rank, y0, y1);
    BSM_TRY(upload_views(c, left, right, W, H));
    PeerOut po{};
    for (int r = 0; r < f->world; ++r) {
        po.d[r] = f->peer_d[r];
        po.v[r] = f->peer_v[r];
    }
    po.n = f->world;
    po.W = W;
    po.rb0 = y0 - std::max(0, y0 - params->vote_radius);  // the output band inside the halo band
    po.g0 = y0;
    c->peer = po;
    const int rc = pipeline_device(c, u8views(c->img_l.as<uint8_t>(), c->img_r.as<uint8_t>()), W, H, y0, y1 - y0,
                                   params, false);
    c->peer = PeerOut{};
    BSM_TRY(rc);
    return sync(c);  // this rank's stores into every map have completed
}

int bsm_frame_fetch(bsm_frame* f, float* d, uint8_t* v) {
    if (!f) return set_err(BSM_INVALID_ARGUMENT, "bsm: null frame");
    BSM_CUDA(cudaSetDevice(f->device));
    const size_t px = size_t(f->W) * f->H;
    if (d) BSM_CUDA(cudaMemcpy(d, f->d, px * 4, cudaMemcpyDeviceToHost));
    if (v) BSM_CUDA(cudaMemcpy(v, f->v, px, cudaMemcpyDeviceToHost));
    return BSM_OK;
}

int bsm_frame_destroy(bsm_frame* f) {
    if (!f) return BSM_OK;
    cudaSetDevice(f->device);
    for (int r = 0; r < f->world; ++r)
        if (r != f->rank && f->peer_d[r]) {
            cudaIpcCloseMemHandle(f->peer_d[r]);
            cudaIpcCloseMemHandle(f->peer_v[r]);
        }
    if (f->d) cudaFree(f->d);
    if (f->v) cudaFree(f->v);
    delete f;
    return BSM_OK;
}

}  // extern "C"
