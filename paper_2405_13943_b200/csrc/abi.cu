// C-ABI (include/bsgpu.h): contexts, device buffers, the per-step pipeline and
// the consensus round. Host code only; kernels live in the other .cu files.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "bsg_internal.cuh"

#include <chrono>
#include <thread>

namespace bsg {

namespace {
thread_local std::string g_err;

// NCCL is resolved at run time (dlopen) so that the library never pins a
// libnccl.so.2 of its own: inside a PyTorch process the already-loaded copy
// (RTLD_NOLOAD) is reused, otherwise the system one is loaded on first use.
struct NcclApi {
    bool ready = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*comm_get_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
};

NcclApi& nccl_api() {
    static NcclApi api;
    if (api.ready) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw std::runtime_error(std::string("cannot load libnccl.so.2: ") + dlerror());
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.comm_get_async_error = reinterpret_cast<decltype(api.comm_get_async_error)>(dlsym(h, "ncclCommGetAsyncError"));
    api.comm_abort = reinterpret_cast<decltype(api.comm_abort)>(dlsym(h, "ncclCommAbort"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.comm_destroy || !api.error_string ||
        !api.group_start || !api.group_end || !api.comm_get_async_error || !api.comm_abort)
        throw std::runtime_error("libnccl.so.2 lacks a required symbol");
    api.ready = true;
    return api;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return BSG_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return BSG_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return BSG_ERR_CUDA;
    }
}

void invalid(const std::string& m) { throw Error{BSG_ERR_INVALID_ARGUMENT, m}; }

template <typename T>
void dev_alloc(T** p, size_t count) {
    if (*p) cudaFree(*p);
    *p = nullptr;
    if (count == 0) count = 1;
    BSG_CUDA(cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
}

void use_device(Ctx* c) { BSG_CUDA(cudaSetDevice(c->device)); }

void free_all(Ctx* c) {
    void* ptrs[] = {c->x, c->m, c->v, c->adam_ring, c->rec, c->depth_key, c->tiles, c->g2d, c->g2d_wide,
                    c->vis_mask, c->vis_prefix, c->sh_mask, c->sh_prefix, c->vkey[0], c->vkey[1], c->vrow[0], c->vrow[1], c->poff, c->vis_rows, c->pkey[0],
                    c->pkey[1], c->pval[0], c->pval[1], c->ranges, c->tile_order, c->tile_cnt, c->tile_cur, c->scan_status, c->radix_status, c->radix_hist,
                    c->counters, c->scalars, c->losses_dev, c->out_rgb, c->out_T, c->out_n, c->out_last, c->dl_dc,
                    c->ssim_f, c->gt_stage, c->gt_stage_b, c->gt_u8[0], c->gt_u8[1], c->sh_rows, c->sh_slots, c->sh_first, c->z, c->u, c->zprev, c->zslot,
                    c->in_zprev, c->slot_owners, c->pack, c->qref, c->slot_reset, c->round_scalars};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (float* p : c->view_gt)
        if (p) cudaFree(p);
    if (c->counters_host) cudaFreeHost(c->counters_host);
    if (c->mbox) cudaFreeHost(c->mbox);
    if (c->lb_ticket) cudaFree(c->lb_ticket);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->nccl) nccl_api().comm_destroy(static_cast<ncclComm_t>(c->nccl));
    if (c->host_buf) cudaFreeHost(c->host_buf);
    for (cudaEvent_t e : {c->gt_ready, c->gt_ready_b, c->gt_free[0], c->gt_free[1]})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {c->x_ready, c->round_done, c->round_t0, c->round_t1})
        if (e) cudaEventDestroy(e);
    if (c->round_host) cudaFreeHost(c->round_host);
    if (c->rho_dev) cudaFree(c->rho_dev);
    if (c->rho_state) cudaFree(c->rho_state);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->stream) cudaStreamDestroy(c->stream);
}

void check_camera(const bsg_camera* cam) {
    if (!cam) invalid("null camera");
    if (cam->width == 0 || cam->height == 0) invalid("camera has zero size");
    if (cam->width > 32767 || cam->height > 32767) invalid("camera larger than 32767 px");
}

void alloc_rows(Ctx* c, size_t n) {
    const size_t cap = (std::max<size_t>(n, 1) + 31) / 32 * 32;  // float4-aligned component rows
    dev_alloc(&c->x, row_stride(c->fd) * cap);
    dev_alloc(&c->m, row_stride(c->fd) * cap);
    dev_alloc(&c->v, row_stride(c->fd) * cap);
    alloc_row_scratch(c, cap);
}

// Host FP64 reference layout -> device FP32 rows (row_stride / pslot).
void upload_params(Ctx* c, const double* pos, const double* rot, const double* ls, const double* feat,
                   const double* op) {
    const size_t n = c->n, cap = c->cap;
    const int fd = c->fd;
    std::vector<float> h(static_cast<size_t>(row_stride(fd)) * cap, 0.f);
    for (size_t i = 0; i < n; ++i) {
        for (int k = 0; k < 3; ++k) h[pidx(i, kPos + k, fd)] = static_cast<float>(pos[3 * i + k]);
        for (int k = 0; k < 4; ++k) h[pidx(i, kRot + k, fd)] = static_cast<float>(rot[4 * i + k]);
        for (int k = 0; k < 3; ++k) h[pidx(i, kLs + k, fd)] = static_cast<float>(ls[3 * i + k]);
        for (int k = 0; k < fd; ++k) h[pidx(i, kFeat + k, fd)] = static_cast<float>(feat[i * fd + k]);
        h[pidx(i, op_comp(fd), fd)] = static_cast<float>(op[i]);
    }
    BSG_CUDA(cudaMemcpyAsync(c->x, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    // scene extent of the (FP32-stored) positions: |tight_aabb extent| (trainer.cpp:153-154)
    if (c->n) {
        double lo[3], hi[3];
        for (int k = 0; k < 3; ++k) lo[k] = hi[k] = h[pidx(0, kPos + k, fd)];
        for (size_t i = 0; i < c->n; ++i)
            for (int k = 0; k < 3; ++k) {
                const double v = h[pidx(i, kPos + k, fd)];
                lo[k] = std::min(lo[k], v);
                hi[k] = std::max(hi[k], v);
            }
        const double e0 = hi[0] - lo[0], e1 = hi[1] - lo[1], e2 = hi[2] - lo[2];
        c->scene_extent = std::max(std::sqrt((e0 * e0 + e1 * e1) + e2 * e2), 1e-9);
    }
    BSG_CUDA(cudaStreamSynchronize(c->stream));
}

// Row-layout (reference bundle) FP64 <-> component-major FP32 for n rows.
std::vector<float> rows_to_cm(const double* rows, size_t n, int D) {
    std::vector<float> h(static_cast<size_t>(D) * std::max<size_t>(n, 1), 0.f);
    for (size_t i = 0; i < n; ++i)
        for (int c = 0; c < D; ++c) h[c * n + i] = static_cast<float>(rows[i * D + c]);
    return h;
}

void cm_to_rows(const float* cm, size_t n, int D, double* rows) {
    for (size_t i = 0; i < n; ++i)
        for (int c = 0; c < D; ++c) rows[i * D + c] = cm[c * n + i];
}

// D-component row of the reference bundle order: pos3 rot4 ls3 feat fd op1 —
// identical to the device component order, so a "row" is just D values.

}  // namespace

void set_error(const std::string& msg) { g_err = msg; }

bool pdl_enabled() {
    static const bool on = std::getenv("BSG_NO_PDL") == nullptr;
    return on;
}

void stage_begin(Ctx* c, int stage) {
    if (c->stage_timing) BSG_CUDA(cudaEventRecord(c->ev[stage], c->stream));
}
void stage_end(Ctx* c, int stage) {
    if (c->stage_timing) BSG_CUDA(cudaEventRecord(c->ev[stage + 1], c->stream));
}

void ensure_image_buffers(Ctx* c, int W, int H) {
    const size_t px = static_cast<size_t>(W) * H;
    if (px > c->img_cap) {
        dev_alloc(&c->out_rgb, 3 * px);
        dev_alloc(&c->out_T, px);
        dev_alloc(&c->out_n, px);
        dev_alloc(&c->out_last, px);
        dev_alloc(&c->dl_dc, 3 * px);
        dev_alloc(&c->ssim_f, 9 * px);
        dev_alloc(&c->gt_stage, 3 * px);
        dev_alloc(&c->gt_stage_b, 3 * px);
        c->img_cap = px;
    }
    const size_t ntiles = static_cast<size_t>((W + kTile - 1) / kTile) * ((H + kTile - 1) / kTile);
    if (ntiles > c->ranges_cap) {
        dev_alloc(&c->ranges, ntiles);
        dev_alloc(&c->tile_order, ntiles);
        dev_alloc(&c->tile_cnt, kTileSub * ntiles);
        dev_alloc(&c->tile_cur, kTileSub * ntiles);
        c->ranges_cap = ntiles;
    }
}

// Tile-pair buffers grow geometrically (x2, at least the row count): a
// reallocation frees and allocates device memory under a device-wide sync
// (tens of ms for large buffers), so views with more pairs than seen so far
// must not trigger one each time.
void ensure_pair_capacity(Ctx* c, size_t P) {
    if (P <= c->pcap) return;
    // Headroom of 2x the rows: a view sequence rarely needs a second growth.
    // Stream-ordered: cudaFree would wait for the whole device (a growth in
    // the middle of a run cost ~0.1 s that way) and stall the other streams.
    const size_t cap = std::max({2 * P, 2 * c->pcap, 2 * c->cap, static_cast<size_t>(1) << 20});
    uint32_t** bufs[4] = {&c->pkey[0], &c->pkey[1], &c->pval[0], &c->pval[1]};
    for (uint32_t** p : bufs) {
        if (*p) BSG_CUDA(cudaFreeAsync(*p, c->stream));
        *p = nullptr;
        BSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(p), cap * sizeof(uint32_t), c->stream));
    }
    c->pcap = cap;
}

namespace {

int tile_bits(const DevCam& cam) {
    const uint32_t ntiles = static_cast<uint32_t>(cam.tiles_x * cam.tiles_y);
    int b = 1;
    while ((1u << b) < ntiles) ++b;
    return b;
}

__global__ __launch_bounds__(512) void zero_counters_kernel(StepCounters* __restrict__ cnt,
                                                           uint32_t* __restrict__ tile_cnt, uint32_t ntiles) {
    pdl_prologue();
    uint32_t* w = reinterpret_cast<uint32_t*>(cnt);
    for (uint32_t i = threadIdx.x; i < sizeof(StepCounters) / 4; i += blockDim.x) w[i] = 0;
    for (uint32_t i = threadIdx.x; i < kTileSub * ntiles; i += blockDim.x) tile_cnt[i] = 0;
}

// K1-K5: projection, compaction, depth sort, pair emission, tile sort, ranges.
// No stream synchronisation on the common path: the compaction and the
// pair-offset scan publish V and P to the host-mapped mailbox, and the host
// polls for each while the kernel enqueued behind it (depth histograms, pair
// emission into the current capacity) keeps the GPU busy.
// Global binning (the fallback, and bsg_project's path): stable LSD sort of
// the 32-bit range-normalised depth key + exact FP64 tie fix-up, pair
// emission in depth order, stable tile-key sort, ranges, launch order.
uint32_t bin_global(Ctx* c, const DevCam& cam, uint32_t V, uint32_t kbits) {
    uint32_t* k32[2] = {reinterpret_cast<uint32_t*>(c->vkey[0]), reinterpret_cast<uint32_t*>(c->vkey[1])};
    stage_begin(c, kStDepthSort);
    // (depth, index) order (renderer.cpp:86-89): stable LSD sort of the 32-bit
    // range-normalised depth key over rows in ascending index order, then runs
    // of equal keys sorted by the full FP64 depth. A run longer than 64 that is
    // out of order falls back to all 8 digit passes of the FP64 bits.
    c->depth_sorted = 0;
    if (V > 1) {
        launch_depth_hist(c, k32[0]);  // digit histograms of the 32-bit depth keys
        radix_sort_u32(c, k32, c->vrow, V, 0, static_cast<int>(kbits / 8), &c->counters->depth_hist[0][0], nullptr,
                       &c->depth_sorted);
    }
    depth_tie_fixup(c, k32[c->depth_sorted], c->vrow[c->depth_sorted], c->depth_key, V, &c->counters->overflow);
    stage_end(c, kStDepthSort);
    stage_begin(c, kStPairs);
    uint32_t P = 0;
    if (V) {
        Publish pp;
        pp.val = &c->mbox->P;
        pp.seq_word = &c->mbox->seq_p;
        pp.seq = ++c->mbox_seq;
        pp.extra_src = &c->counters->overflow;
        pp.extra_dst = &c->mbox->overflow;
        scan_exclusive_u32(c, c->tiles, c->vrow[c->depth_sorted], c->poff, V, &c->counters->pairs, pp);
        launch_pairs(c, cam, V);  // into the current capacity; + digit histograms of the tile keys
        wait_mailbox(c, &c->mbox->seq_p, pp.seq);
        P = c->mbox->P;
        bool redo = false;
        if (c->mbox->overflow) {
            // rare: a long out-of-order run of equal 32-bit keys -> full 64-bit sort
            BSG_CUDA(cudaMemsetAsync(c->counters, 0, sizeof(StepCounters), c->stream));
            compact_visible(c, static_cast<uint32_t>(c->n), false);
            BSG_CUDA(cudaMemcpyAsync(c->counters_host, c->counters, offsetof(StepCounters, tile_hist),
                                     cudaMemcpyDeviceToHost, c->stream));
            BSG_CUDA(cudaStreamSynchronize(c->stream));
            radix_sort_u64(c, c->vkey, c->vrow, V, 0, 8, &c->counters->depth_hist[0][0],
                           &c->counters_host->depth_hist[0][0], &c->depth_sorted);
            scan_exclusive_u32(c, c->tiles, c->vrow[c->depth_sorted], c->poff, V, &c->counters->pairs);
            BSG_CUDA(cudaMemcpyAsync(c->counters_host, c->counters, 16, cudaMemcpyDeviceToHost, c->stream));
            BSG_CUDA(cudaStreamSynchronize(c->stream));
            P = c->counters_host->pairs;
            redo = true;
        }
        if (P > c->pcap) {
            ensure_pair_capacity(c, P);
            redo = true;
        }
        if (redo) {  // the emission ran against the old order or capacity
            BSG_CUDA(cudaMemsetAsync(&c->counters->tile_hist[0][0], 0, sizeof(c->counters->tile_hist), c->stream));
            launch_pairs(c, cam, V);
        }
    }
    stage_end(c, kStPairs);
    stage_begin(c, kStTileSort);
    const int passes = (tile_bits(cam) + 7) / 8;
    radix_sort_u32(c, c->pkey, c->pval, P, 0, passes, &c->counters->tile_hist[0][0], nullptr, &c->pairs_sorted);
    stage_end(c, kStTileSort);
    stage_begin(c, kStRanges);
    launch_ranges(c, cam, V, P);
    stage_end(c, kStRanges);
    c->last_binning = 1;
    return P;
}

// K1-K5: projection, compaction, binning into tiles, per-tile depth order,
// ranges. No stream synchronisation on the common path: the compaction and
// the tile scan publish V and P to the host-mapped mailbox, and the host
// polls for them while the kernel enqueued behind (the speculative pair
// emission into the current capacity) keeps the GPU busy.
void project_and_bin(Ctx* c, const DevCam& cam, const DevRender& rc) {
    ensure_image_buffers(c, cam.W, cam.H);
    const uint32_t ntiles = static_cast<uint32_t>(cam.tiles_x * cam.tiles_y);
    launch_pdl(c->stream, 1, 512, 0, zero_counters_kernel, c->counters, c->tile_cnt, ntiles);
    BSG_LAUNCHED(c);
    c->tile_scan_used = false;
    stage_begin(c, kStPreprocess);
    launch_preprocess(c, cam, rc);  // + pairs per tile
    stage_end(c, kStPreprocess);
    stage_begin(c, kStCompact);
    uint32_t V = 0, kbits = 16, P = 0;
    if (c->n == 0) {
        compact_visible(c, 0, true);
        stage_end(c, kStCompact);
        launch_ranges(c, cam, 0, 0);  // empty ranges + launch order
        c->last_binning = 1;
        c->last_counters.visible = 0;
        c->last_counters.pairs = 0;
        return;
    }
    Publish pv;
    pv.val = &c->mbox->V;
    pv.seq_word = &c->mbox->seq_v;
    pv.seq = ++c->mbox_seq;
    pv.extra_src = &c->counters->visible_pre;
    pv.extra_dst = &c->mbox->visible_pre;
    // the previous view's largest tile picks the path up front, so a dense
    // sequence of views does not pay the speculative per-tile emission; the
    // per-tile path compacts from the preprocess's visibility mask (no depth keys)
    const bool global_path = c->global_order || c->last_max_tile > kTileSortCap;
    if (global_path)
        compact_visible(c, static_cast<uint32_t>(c->n), true, pv);
    else
        compact_visible_mask(c, static_cast<uint32_t>(c->n), pv);
    stage_end(c, kStCompact);
    if (global_path) {
        launch_tile_scan(c, cam, ++c->mbox_seq);  // only for the largest-tile count (cheap)
        wait_mailbox(c, &c->mbox->seq_v, pv.seq);
        V = c->mbox->V;
        kbits = static_cast<uint32_t>(depth_key_bits(c->mbox->visible_pre));
        P = bin_global(c, cam, V, kbits);  // its P wait orders the tile scan's mailbox write before this read
        if (c->mbox->pairs_big) throw Error{BSG_ERR_CAPACITY, "view with 2^30 or more tile pairs"};
        c->last_max_tile = c->mbox->max_tile;
    } else {
        stage_begin(c, kStDepthSort);
        uint32_t seq = ++c->mbox_seq;
        launch_tile_scan(c, cam, seq);
        stage_end(c, kStDepthSort);
        stage_begin(c, kStPairs);
        launch_emit_tiles(c, cam);  // speculative: into the current capacity
        wait_mailbox(c, &c->mbox->seq_v, pv.seq);
        V = c->mbox->V;
        kbits = static_cast<uint32_t>(depth_key_bits(c->mbox->visible_pre));
        wait_mailbox(c, &c->mbox->seq_p, seq);
        P = c->mbox->P;
        if (c->mbox->pairs_big) throw Error{BSG_ERR_CAPACITY, "view with 2^30 or more tile pairs"};
        const uint32_t max_tile = c->mbox->max_tile;
        c->last_max_tile = max_tile;
        stage_end(c, kStPairs);
        if (max_tile > kTileSortCap) {
            // a tile too long for the shared-memory sort: the global path, whose
            // depth sort needs the keyed compaction
            compact_visible(c, static_cast<uint32_t>(c->n), true);
            P = bin_global(c, cam, V, kbits);
        } else {
            if (P > c->pcap) {  // the emission ran out of capacity: grow, reset the cursors, emit again
                ensure_pair_capacity(c, P);
                launch_tile_scan(c, cam, ++c->mbox_seq);
                launch_emit_tiles(c, cam);
            }
            stage_begin(c, kStTileSort);
            if (P) launch_tile_sort(c, cam, max_tile);
            stage_end(c, kStTileSort);
            stage_begin(c, kStRanges);  // (ranges and the launch order came from the tile scan)
            stage_end(c, kStRanges);
            c->pairs_sorted = 0;
            c->last_binning = 0;
        }
    }
    c->last_counters.visible = V;
    c->last_counters.pairs = P;
    c->last_ntiles = ntiles;
}

}  // namespace

void project_and_bin_public(Ctx* c, const DevCam& cam, const DevRender& rc) { project_and_bin(c, cam, rc); }

void alloc_row_scratch(Ctx* c, size_t cap) {
    dev_alloc(&c->rec, 3 * cap);
    dev_alloc(&c->depth_key, cap);
    dev_alloc(&c->tiles, cap);
    dev_alloc(&c->g2d, 3 * cap);
    dev_alloc(&c->vis_mask, cap / 32);
    dev_alloc(&c->vis_prefix, cap / 32);
    dev_alloc(&c->sh_mask, cap / 32);
    dev_alloc(&c->sh_prefix, cap / 32);
    dev_alloc(&c->vkey[0], cap);
    dev_alloc(&c->vkey[1], cap);
    dev_alloc(&c->vrow[0], cap);
    dev_alloc(&c->vrow[1], cap);
    dev_alloc(&c->poff, cap);
    dev_alloc(&c->vis_rows, cap);
    c->cap = cap;
}

// Anchor index of a row = its rank among the (ascending) shared rows: 1 bit per
// row + shared rows before each 32-row word (read by the Adam kernels).
void install_shared_masks(Ctx* c) {
    std::vector<uint32_t> mask(c->cap / 32, 0), prefix(c->cap / 32, 0);
    for (uint32_t r : c->sh_rows_host) mask[r / 32] |= 1u << (r % 32);
    uint32_t run = 0;
    for (size_t w = 0; w < mask.size(); ++w) {
        prefix[w] = run;
        run += static_cast<uint32_t>(__builtin_popcount(mask[w]));
    }
    BSG_CUDA(cudaMemcpyAsync(c->sh_mask, mask.data(), mask.size() * 4, cudaMemcpyHostToDevice, c->stream));
    BSG_CUDA(cudaMemcpyAsync(c->sh_prefix, prefix.data(), prefix.size() * 4, cudaMemcpyHostToDevice, c->stream));
}

namespace {

float* upload_gt_f64(Ctx* c, const double* gt, size_t px) {
    std::vector<float> h(3 * px);
    for (size_t i = 0; i < 3 * px; ++i) h[i] = static_cast<float>(gt[i]);
    BSG_CUDA(cudaMemcpyAsync(c->gt_stage, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    BSG_CUDA(cudaStreamSynchronize(c->stream));
    return c->gt_stage;
}

void collect_stage_times(Ctx* c) {
    if (!c->stage_timing) return;
    BSG_CUDA(cudaMemcpyAsync(&c->counters_host->evals, &c->counters->evals, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, c->stream));
    BSG_CUDA(cudaStreamSynchronize(c->stream));
    c->last_evals = c->counters_host->evals;
    for (int s = 0; s < kStCount; ++s) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->ev[s], c->ev[s + 1]) != cudaSuccess) {
            cudaGetLastError();
            ms = 0.f;
        }
        c->stage_ms[s] = ms;
    }
}

AdamStep make_adam_step(Ctx* c) {
    AdamStep st{};
    const bsg_trainer_config& t = c->tcfg;
    const uint64_t step = ++c->adam_t;  // trainer.cpp:267
    st.t = static_cast<uint32_t>(step);
    const double progress = t.iterations > 0 ? static_cast<double>(c->iteration) / static_cast<double>(t.iterations) : 0.0;
    const double lr_pos = t.lr_position * std::pow(t.lr_position_decay, progress);  // trainer.cpp:268-271
    const double bc1 = 1.0 - std::pow(t.beta1, static_cast<double>(step));
    const double bc2 = 1.0 - std::pow(t.beta2, static_cast<double>(step));
    for (int k = 0; k < c->D; ++k) {
        double lr = t.lr_features;
        if (k < kRot) lr = lr_pos;
        else if (k < kLs) lr = t.lr_rotation;
        else if (k < kFeat) lr = t.lr_log_scale;
        else if (k == op_comp(c->fd)) lr = t.lr_opacity;
        st.lr[k] = static_cast<float>(lr);
    }
    st.b1 = static_cast<float>(t.beta1);
    st.b2 = static_cast<float>(t.beta2);
    st.omb1 = static_cast<float>(1.0 - t.beta1);
    st.omb2 = static_cast<float>(1.0 - t.beta2);
    st.eps = static_cast<float>(t.eps);
    st.inv_bc1 = static_cast<float>(1.0 / bc1);
    st.inv_bc2 = static_cast<float>(1.0 / bc2);
    st.has_anchor = (c->anchored && c->n_shared > 0) ? 1 : 0;
    return st;
}

// One train_step (trainer.cpp:249-295) on a device-resident ground truth:
// FP32, or (gt8 non-null) the 8-bit image the loss kernels read directly.
// gt_ready (nullable): event the loss waits on (ground truth still in flight
// on the copy stream while projection, sorting and the forward blend run).
void train_one(Ctx* c, const bsg_camera& view, const float* gt, double* loss_dev, cudaEvent_t gt_ready = nullptr,
               const uint8_t* gt8 = nullptr) {
    c->step_launches = 0;
    const DevCam cam = make_cam(view);
    const DevRender rc = make_render(c->tcfg.render);
    project_and_bin(c, cam, rc);  // (the preprocess zeroes the step scalars)
    stage_begin(c, kStBlendFwd);
    launch_blend_fwd(c, cam, rc);
    stage_end(c, kStBlendFwd);
    stage_begin(c, kStLoss);
    if (gt_ready) BSG_CUDA(cudaStreamWaitEvent(c->stream, gt_ready, 0));
    if (gt8)
        launch_loss(c, cam, rc, gt8);
    else
        launch_loss(c, cam, rc, gt);
    stage_end(c, kStLoss);
    stage_begin(c, kStBlendBwd);
    launch_blend_bwd(c, cam, rc);
    stage_end(c, kStBlendBwd);
    // the fold runs fused with the Adam (fold_adam_kernel), stage "adam"
    stage_begin(c, kStAdam);
    // penalty + Adam need the round's anchor, duals and rho
    if (c->round_pending) BSG_CUDA(cudaStreamWaitEvent(c->stream, c->round_done, 0));
    const AdamStep st = make_adam_step(c);
    launch_adam(c, cam, st, loss_dev, 0);
    stage_end(c, kStAdam);
    launch_finalize_loss(c, cam, rc, loss_dev, st.has_anchor != 0);
    c->iteration++;
    c->last_counters.overflow = 0;
}

void ensure_views_buffers(Ctx* c, size_t n) {
    if (n > c->losses_cap) {
        dev_alloc(&c->losses_dev, 3 * n);
        c->losses_cap = n;
    }
}

// ---- consensus plumbing --------------------------------------------------
void reduce_nccl(Ctx* c, void* buf, size_t count, ncclDataType_t type, ncclRedOp_t op) {
    if (c->host_reduce) {
        // host communicator (bsg_comm_init_host): the buffer goes through pinned
        // host memory and the caller's all-reduce; the round blocks here
        const size_t bytes = count * (type == ncclFloat64 ? 8 : 4);
        if (bytes == 0) return;
        if (bytes > c->host_buf_cap) {
            if (c->host_buf) cudaFreeHost(c->host_buf);
            c->host_buf = nullptr;
            BSG_CUDA(cudaMallocHost(&c->host_buf, bytes));
            c->host_buf_cap = bytes;
        }
        BSG_CUDA(cudaMemcpyAsync(c->host_buf, buf, bytes, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        const int rc = c->host_reduce(c->host_user, c->host_buf, count, type == ncclFloat64 ? 1 : 0,
                                      op == ncclMax ? 1 : 0);
        if (rc != 0) throw Error{BSG_ERR_NCCL, "host all-reduce failed (" + std::to_string(rc) + ")"};
        BSG_CUDA(cudaMemcpyAsync(buf, c->host_buf, bytes, cudaMemcpyHostToDevice, c->stream));
        return;
    }
    if (!c->nccl) return;
    NcclApi& n = nccl_api();
    const ncclResult_t r = n.all_reduce(buf, buf, count, type, op, static_cast<ncclComm_t>(c->nccl), c->stream);
    if (r != ncclSuccess) throw Error{BSG_ERR_NCCL, std::string("ncclAllReduce: ") + n.error_string(r)};
}

__global__ void sum_into_kernel(float* __restrict__ acc, const float* __restrict__ src, size_t n) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) acc[i] += src[i];
}
__global__ void max_into_kernel(float* __restrict__ acc, const float* __restrict__ src, size_t n) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    if (i < n) acc[i] = fmaxf(acc[i], src[i]);
}

// In-order (ascending block id) reduction of one buffer across a local group.
void reduce_group(Ctx* const* ctxs, size_t k, float* Ctx::*field, size_t count, bool max_op) {
    if (k <= 1 || count == 0) return;
    Ctx* c0 = ctxs[0];
    for (size_t b = 0; b < k; ++b) BSG_CUDA(cudaStreamSynchronize(ctxs[b]->stream));
    use_device(c0);
    float* tmp = nullptr;
    BSG_CUDA(cudaMalloc(&tmp, count * sizeof(float)));
    for (size_t b = 1; b < k; ++b) {
        BSG_CUDA(cudaMemcpyPeerAsync(tmp, c0->device, ctxs[b]->*field, ctxs[b]->device, count * sizeof(float),
                                     c0->stream));
        if (max_op)
            max_into_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, c0->stream>>>(c0->*field, tmp, count);
        else
            sum_into_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, c0->stream>>>(c0->*field, tmp, count);
        BSG_LAUNCHED(c0);
    }
    BSG_CUDA(cudaStreamSynchronize(c0->stream));
    BSG_CUDA(cudaFree(tmp));
    for (size_t b = 1; b < k; ++b) {
        use_device(ctxs[b]);
        BSG_CUDA(cudaMemcpyPeerAsync(ctxs[b]->*field, ctxs[b]->device, c0->*field, c0->device, count * sizeof(float),
                                     ctxs[b]->stream));
        BSG_CUDA(cudaStreamSynchronize(ctxs[b]->stream));
    }
}

void check_round_ready(Ctx* c) {
    if (!c->anchored) throw Error{BSG_ERR_STATE, "consensus round before set_anchor"};
}

void upload_resets(Ctx* c, const bsg_round_args* a) {
    if (c->n_slots == 0) return;
    BSG_CUDA(cudaMemsetAsync(c->slot_reset, 0, c->n_slots, c->stream));
    if (a->n_reset == 0) return;
    std::vector<uint8_t> h(c->n_slots, 0);
    for (size_t i = 0; i < a->n_reset; ++i) {
        if (a->reset_slots[i] >= c->n_slots) invalid("reset slot out of range");
        h[a->reset_slots[i]] = 1;
    }
    BSG_CUDA(cudaMemcpyAsync(c->slot_reset, h.data(), h.size(), cudaMemcpyHostToDevice, c->stream));
    BSG_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace

// Exposed for consensus.cu diagnostics.
void round_pack_duals(Ctx* c);
void round_dual_linf(Ctx* c);
void round_pack_minmax(Ctx* c);
void round_spread(Ctx* c);

// n steps on host images, each uploaded on the copy stream into one of two
// device buffers while the previous step computes. `upload(k, b, buf)`
// enqueues step k's image on the copy stream: into the FP32 buffer buf
// (returns null), or into an 8-bit buffer it returns.
template <typename Upload>
void train_steps_from_host(Ctx* c, size_t n, const bsg_camera* cams, double* losses, Upload&& upload) {
    ensure_views_buffers(c, std::max<size_t>(n, 1));
    // every buffer sized for the largest view first: an image-buffer growth
    // must not free a staging buffer with an upload in flight
    for (size_t k = 0; k < n; ++k)
        ensure_image_buffers(c, static_cast<int>(cams[k].width), static_cast<int>(cams[k].height));
    // Step k's image is uploaded while step k-1 computes (issued before step
    // k-1's kernels), so step k waits for it at its start -- a step boundary --
    // and the step's own kernels stay one programmatic-launch chain.
    const uint8_t* gt8[2] = {nullptr, nullptr};
    auto issue = [&](size_t k) {
        const int b = static_cast<int>(k & 1);
        float* buf = b ? c->gt_stage_b : c->gt_stage;
        // step k-2 read this buffer: its loss must be done before the overwrite
        if (k >= 2) BSG_CUDA(cudaStreamWaitEvent(c->copy_stream, c->gt_free[b], 0));
        gt8[b] = upload(k, b, buf);
        BSG_CUDA(cudaEventRecord(b ? c->gt_ready_b : c->gt_ready, c->copy_stream));
    };
    if (n) issue(0);
    for (size_t k = 0; k < n; ++k) {
        const int b = static_cast<int>(k & 1);
        if (k + 1 < n) issue(k + 1);
        BSG_CUDA(cudaStreamWaitEvent(c->stream, b ? c->gt_ready_b : c->gt_ready, 0));
        train_one(c, cams[k], b ? c->gt_stage_b : c->gt_stage, c->losses_dev + 3 * k, nullptr, gt8[b]);
        BSG_CUDA(cudaEventRecord(c->gt_free[b], c->stream));
        maybe_densify(c);
    }
    if (n) {
        std::vector<double> l(3 * n);
        BSG_CUDA(cudaMemcpyAsync(l.data(), c->losses_dev, l.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        if (losses)
            for (size_t k = 0; k < n; ++k) losses[k] = l[3 * k];
    }
    collect_stage_times(c);
}

}  // namespace bsg

using namespace bsg;

extern "C" {

int bsg_abi_version(void) { return BSG_ABI_VERSION; }
const char* bsg_last_error(void) { return g_err.c_str(); }

void bsg_default_render_config(bsg_render_config* o) {
    o->near_plane = 0.01;
    o->dilation = 0.3;
    o->alpha_clamp = 0.99;
    o->transmittance_stop = 1e-4;
    o->sigma_extent = 3.0;
    o->background[0] = o->background[1] = o->background[2] = 0.0;
    o->lambda = 0.2;
}

void bsg_default_trainer_config(bsg_trainer_config* o) {
    o->iterations = 3000;
    o->lr_position = 1.6e-4;
    o->lr_position_decay = 0.01;
    o->lr_rotation = 1e-3;
    o->lr_log_scale = 5e-3;
    o->lr_features = 2.5e-3;
    o->lr_opacity = 5e-2;
    o->beta1 = 0.9;
    o->beta2 = 0.999;
    o->eps = 1e-8;
    bsg_default_render_config(&o->render);
    o->densify.enabled = 1;  // trainer.hpp:43-51
    o->densify.interval = 200;
    o->densify.stop_iteration = 0;
    o->densify.grad_threshold = 2e-4;
    o->densify.prune_opacity = 0.005;
    o->densify.split_scale_fraction = 0.01;
    o->densify.split_shrink = 1.6;
    o->densify.block_id = 0;
    o->densify.global_initial_count = 0;
}

void bsg_default_penalties(bsg_penalties* o) {
    o->rho_p = 1e4;
    o->rho_q = 1e4;
    o->rho_s = 1e4;
    o->rho_f = 1e3;
    o->rho_o = 1e4;
}

int bsg_create(int device, int feature_dim, bsg_ctx** out) {
    return guarded([&] {
        if (!out) invalid("null output");
        if (feature_dim != 3 && feature_dim != 12) invalid("unsupported feature width");
        int count = 0;
        BSG_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) invalid("no such CUDA device");
        cudaDeviceProp prop{};
        BSG_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) throw Error{BSG_ERR_CUDA, "libbsgpu is built for sm_100a (B200); device is sm_" +
                                                            std::to_string(prop.major * 10 + prop.minor)};
        auto* c = new Ctx();
        c->device = device;
        c->fd = feature_dim;
        c->D = 11 + feature_dim;
        try {
            use_device(c);
            BSG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            BSG_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
            BSG_CUDA(cudaEventCreateWithFlags(&c->gt_ready, cudaEventDisableTiming));
            BSG_CUDA(cudaEventCreateWithFlags(&c->gt_ready_b, cudaEventDisableTiming));
            for (auto& e : c->gt_free) BSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            BSG_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
            BSG_CUDA(cudaEventCreateWithFlags(&c->x_ready, cudaEventDisableTiming));
            BSG_CUDA(cudaEventCreateWithFlags(&c->round_done, cudaEventDisableTiming));
            BSG_CUDA(cudaEventCreate(&c->round_t0));
            BSG_CUDA(cudaEventCreate(&c->round_t1));
            BSG_CUDA(cudaMallocHost(&c->round_host, 16 * sizeof(double)));  // 8 round scalars + 5 rho
            dev_alloc(&c->rho_dev, kMaxD);
            dev_alloc(&c->rho_state, 5);
            dev_alloc(&c->adam_ring, kAdamRing);
            dev_alloc(&c->g2d_wide, 9 * static_cast<size_t>(kWideCap));
            BSG_CUDA(cudaMallocHost(&c->counters_host, sizeof(StepCounters)));
            BSG_CUDA(cudaHostAlloc(&c->mbox, sizeof(Mailbox), cudaHostAllocMapped | cudaHostAllocPortable));
            std::memset(c->mbox, 0, sizeof(Mailbox));
            dev_alloc(&c->counters, 1);
            dev_alloc(&c->scalars, 1);
            dev_alloc(&c->radix_hist, 1);
            dev_alloc(&c->round_scalars, 8 + kMaxD);
            dev_alloc(&c->losses_dev, 3);
            c->losses_cap = 1;
            for (auto& e : c->ev) BSG_CUDA(cudaEventCreate(&e));
            bsg_default_trainer_config(&c->tcfg);
            bsg_default_penalties(&c->rho);
            upload_rho(c);
            alloc_rows(c, 1);
        } catch (...) {
            free_all(c);
            delete c;
            throw;
        }
        *out = reinterpret_cast<bsg_ctx*>(c);
    });
}

int bsg_destroy(bsg_ctx* h) {
    return guarded([&] {
        if (!h) return;
        auto* c = reinterpret_cast<Ctx*>(h);
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        free_all(c);
        delete c;
    });
}

int bsg_upload_cloud(bsg_ctx* h, size_t n, const uint64_t* ids, const double* pos, const double* rot, const double* ls,
                     const double* feat, const double* op) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (n > 0 && (!ids || !pos || !rot || !ls || !feat || !op)) invalid("null parameter array");
        for (size_t i = 1; i < n; ++i)
            if (ids[i] <= ids[i - 1]) invalid("initial cloud ids not ascending");
        if (n >= (1u << 30)) invalid("cloud larger than 2^30 rows");
        use_device(c);
        c->n = n;
        c->ids.assign(ids, ids + n);
        alloc_rows(c, n);
        upload_params(c, pos, rot, ls, feat, op);
        BSG_CUDA(cudaMemsetAsync(c->m, 0, row_stride(c->fd) * c->cap * sizeof(float), c->stream));  // (densify stats too)
        BSG_CUDA(cudaMemsetAsync(c->v, 0, row_stride(c->fd) * c->cap * sizeof(float), c->stream));
        BSG_CUDA(cudaMemsetAsync(c->vis_mask, 0, c->cap / 32 * sizeof(uint32_t), c->stream));
        BSG_CUDA(cudaMemsetAsync(c->sh_mask, 0, c->cap / 32 * sizeof(uint32_t), c->stream));
        BSG_CUDA(cudaMemsetAsync(c->sh_prefix, 0, c->cap / 32 * sizeof(uint32_t), c->stream));
        c->adam_t = 0;
        reset_row_meta(c, 0, false);
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        c->iteration = 0;
        c->anchored = false;
        c->n_shared = 0;
        c->n_slots = 0;
    });
}

size_t bsg_cloud_size(const bsg_ctx* h) { return h ? reinterpret_cast<const Ctx*>(h)->n : 0; }

int bsg_download_cloud(bsg_ctx* h, uint64_t* ids, double* pos, double* rot, double* ls, double* feat, double* op) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        const size_t n = c->n, cap = c->cap;
        if (ids) std::copy(c->ids.begin(), c->ids.end(), ids);
        if (!pos && !rot && !ls && !feat && !op) return;  // ids only
        materialize(c);
        const int fd = c->fd;
        std::vector<float> hx(static_cast<size_t>(row_stride(fd)) * cap);
        BSG_CUDA(cudaMemcpyAsync(hx.data(), c->x, hx.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        if (ids) std::copy(c->ids.begin(), c->ids.end(), ids);
        for (size_t i = 0; i < n; ++i) {
            if (pos) for (int k = 0; k < 3; ++k) pos[3 * i + k] = hx[pidx(i, kPos + k, fd)];
            if (rot) for (int k = 0; k < 4; ++k) rot[4 * i + k] = hx[pidx(i, kRot + k, fd)];
            if (ls) for (int k = 0; k < 3; ++k) ls[3 * i + k] = hx[pidx(i, kLs + k, fd)];
            if (feat) for (int k = 0; k < fd; ++k) feat[i * fd + k] = hx[pidx(i, kFeat + k, fd)];
            if (op) op[i] = hx[pidx(i, op_comp(fd), fd)];
        }
    });
}

int bsg_encode_gspl(bsg_ctx* h, uint8_t* out, size_t out_cap, size_t* out_len) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!out_len) invalid("null out_len");
        const size_t n = c->n;
        const size_t floats = static_cast<size_t>(11 + c->fd) * n;
        const size_t len = 8 + 4 + 8 * n + 4 * floats;
        *out_len = len;
        if (!out) return;
        if (out_cap < len) throw Error{BSG_ERR_CAPACITY, "GSPL buffer smaller than the payload"};
        use_device(c);
        const uint64_t count = n;
        const uint32_t fd = static_cast<uint32_t>(c->fd);
        std::memcpy(out, &count, 8);
        std::memcpy(out + 8, &fd, 4);
        if (n) std::memcpy(out + 12, c->ids.data(), 8 * n);
        if (!floats) return;
        // the transposed arrays in a scratch buffer of the call
        float* scratch = nullptr;
        BSG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), 4 * static_cast<size_t>(c->D) * c->cap, c->stream));
        launch_gspl_floats(c, scratch);
        BSG_CUDA(cudaMemcpyAsync(out + 12 + 8 * n, scratch, 4 * floats, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaFreeAsync(scratch, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int bsg_render(bsg_ctx* h, const bsg_camera* cam, const bsg_render_config* cfg, double* out_rgb, double* out_T,
               uint32_t* out_n) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        check_camera(cam);
        bsg_render_config rcfg;
        if (cfg) rcfg = *cfg; else bsg_default_render_config(&rcfg);
        use_device(c);
        c->step_launches = 0;
        const DevCam dc = make_cam(*cam);
        const DevRender rc = make_render(rcfg);
        project_and_bin(c, dc, rc);
        stage_begin(c, kStBlendFwd);
        launch_blend_fwd(c, dc, rc);
        stage_end(c, kStBlendFwd);
        const size_t px = static_cast<size_t>(cam->width) * cam->height;
        std::vector<float> rgb(3 * px), T(px);
        BSG_CUDA(cudaMemcpyAsync(rgb.data(), c->out_rgb, rgb.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaMemcpyAsync(T.data(), c->out_T, T.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        if (out_n) BSG_CUDA(cudaMemcpyAsync(out_n, c->out_n, px * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        collect_stage_times(c);
        if (out_rgb) for (size_t i = 0; i < 3 * px; ++i) out_rgb[i] = rgb[i];
        if (out_T) for (size_t i = 0; i < px; ++i) out_T[i] = T[i];
    });
}

int bsg_evaluate(bsg_ctx* h, size_t n_views, const bsg_camera* cams, const double* const* gt, uint32_t holdout_modulus,
                 const bsg_render_config* cfg, double* per_view_psnr, double* per_view_ssim, size_t* n_scored,
                 double* mean_psnr, double* mean_ssim) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (n_views && (!cams || !gt)) invalid("null views");
        bsg_render_config rcfg;
        if (cfg) rcfg = *cfg; else bsg_default_render_config(&rcfg);
        use_device(c);
        const DevRender rc = make_render(rcfg);
        double* gt_dev = nullptr;
        double* scratch = nullptr;
        size_t gt_cap = 0;
        size_t k = 0;
        double sp = 0, ss = 0;
        try {
            BSG_CUDA(cudaMalloc(&scratch, sizeof(double)));
            for (size_t i = 0; i < n_views; ++i) {
                if (holdout_modulus != 0 && i % holdout_modulus != 0) continue;  // metrics.cpp:34
                check_camera(&cams[i]);
                if (!gt[i]) invalid("null ground truth");
                const DevCam dc = make_cam(cams[i]);
                ensure_image_buffers(c, dc.W, dc.H);
                const size_t n = 3 * static_cast<size_t>(dc.W) * dc.H;
                if (n > gt_cap) {
                    if (gt_dev) cudaFree(gt_dev);
                    BSG_CUDA(cudaMalloc(&gt_dev, n * sizeof(double)));
                    gt_cap = n;
                }
                BSG_CUDA(cudaMemcpyAsync(gt_dev, gt[i], n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
                double r[2];
                eval_view(c, dc, rc, gt_dev, scratch, r);
                if (per_view_psnr) per_view_psnr[k] = r[0];
                if (per_view_ssim) per_view_ssim[k] = r[1];
                sp += r[0];
                ss += r[1];
                ++k;
            }
        } catch (...) {
            if (gt_dev) cudaFree(gt_dev);
            if (scratch) cudaFree(scratch);
            throw;
        }
        if (gt_dev) cudaFree(gt_dev);
        if (scratch) cudaFree(scratch);
        if (k == 0) invalid("empty holdout");  // metrics.cpp:44
        if (n_scored) *n_scored = k;
        if (mean_psnr) *mean_psnr = sp / static_cast<double>(k);
        if (mean_ssim) *mean_ssim = ss / static_cast<double>(k);
    });
}

int bsg_render_backward(bsg_ctx* h, const bsg_camera* cam, const double* gt, const bsg_render_config* cfg,
                        double* out_loss3, double* g_pos, double* g_rot, double* g_ls, double* g_feat, double* g_op,
                        double* sgn, uint8_t* visible, double* out_rendered) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        check_camera(cam);
        if (!gt) invalid("image dimension mismatch");
        bsg_render_config rcfg;
        if (cfg) rcfg = *cfg; else bsg_default_render_config(&rcfg);
        use_device(c);
        c->step_launches = 0;
        const DevCam dc = make_cam(*cam);
        const DevRender rc = make_render(rcfg);
        const size_t px = static_cast<size_t>(cam->width) * cam->height;
        ensure_image_buffers(c, dc.W, dc.H);
        const float* gtd = upload_gt_f64(c, gt, px);
        BSG_CUDA(cudaMemsetAsync(c->scalars, 0, sizeof(StepScalars), c->stream));
        project_and_bin(c, dc, rc);
        stage_begin(c, kStBlendFwd);
        launch_blend_fwd(c, dc, rc);
        stage_end(c, kStBlendFwd);
        stage_begin(c, kStLoss);
        launch_loss(c, dc, rc, gtd);
        stage_end(c, kStLoss);
        stage_begin(c, kStBlendBwd);
        launch_blend_bwd(c, dc, rc);
        stage_end(c, kStBlendBwd);
        ensure_views_buffers(c, 1);
        launch_finalize_loss(c, dc, rc, c->losses_dev, false);
        const size_t n = c->n;
        double* gdev = nullptr;
        double* sdev = nullptr;
        uint8_t* vdev = nullptr;
        BSG_CUDA(cudaMalloc(&gdev, std::max<size_t>(1, c->D * n) * sizeof(double)));
        BSG_CUDA(cudaMalloc(&sdev, std::max<size_t>(1, n) * sizeof(double)));
        BSG_CUDA(cudaMalloc(&vdev, std::max<size_t>(1, n)));
        stage_begin(c, kStFold);
        launch_fold_grads(c, dc, gdev, sdev, vdev);
        stage_end(c, kStFold);
        std::vector<double> g(static_cast<size_t>(c->D) * n);
        double l3[3];
        BSG_CUDA(cudaMemcpyAsync(g.data(), gdev, g.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaMemcpyAsync(l3, c->losses_dev, sizeof(l3), cudaMemcpyDeviceToHost, c->stream));
        if (sgn) BSG_CUDA(cudaMemcpyAsync(sgn, sdev, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (visible) BSG_CUDA(cudaMemcpyAsync(visible, vdev, n, cudaMemcpyDeviceToHost, c->stream));
        std::vector<float> rgb;
        if (out_rendered) {
            rgb.resize(3 * px);
            BSG_CUDA(cudaMemcpyAsync(rgb.data(), c->out_rgb, rgb.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        }
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        cudaFree(gdev);
        cudaFree(sdev);
        cudaFree(vdev);
        collect_stage_times(c);
        if (out_loss3) for (int k = 0; k < 3; ++k) out_loss3[k] = l3[k];
        for (size_t i = 0; i < n; ++i) {
            if (g_pos) for (int k = 0; k < 3; ++k) g_pos[3 * i + k] = g[(kPos + k) * n + i];
            if (g_rot) for (int k = 0; k < 4; ++k) g_rot[4 * i + k] = g[(kRot + k) * n + i];
            if (g_ls) for (int k = 0; k < 3; ++k) g_ls[3 * i + k] = g[(kLs + k) * n + i];
            if (g_feat) for (int k = 0; k < c->fd; ++k) g_feat[i * c->fd + k] = g[(kFeat + k) * n + i];
            if (g_op) g_op[i] = g[op_comp(c->fd) * n + i];
        }
        if (out_rendered) for (size_t i = 0; i < 3 * px; ++i) out_rendered[i] = rgb[i];
    });
}

int bsg_image_loss(bsg_ctx* h, uint32_t width, uint32_t height, const double* rendered, const double* gt,
                   const bsg_render_config* cfg, double* out_loss3, double* out_dl_dc) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!rendered || !gt || width == 0 || height == 0) invalid("image dimension mismatch");
        bsg_render_config rcfg;
        if (cfg) rcfg = *cfg; else bsg_default_render_config(&rcfg);
        use_device(c);
        bsg_camera cam{};
        cam.fx = cam.fy = 1.0;
        cam.R[0] = cam.R[4] = cam.R[8] = 1.0;
        cam.width = width;
        cam.height = height;
        const DevCam dc = make_cam(cam);
        const DevRender rc = make_render(rcfg);
        const size_t px = static_cast<size_t>(width) * height;
        ensure_image_buffers(c, dc.W, dc.H);
        const float* gtd = upload_gt_f64(c, gt, px);
        {
            std::vector<float> r(3 * px);
            for (size_t i = 0; i < 3 * px; ++i) r[i] = static_cast<float>(rendered[i]);
            BSG_CUDA(cudaMemcpyAsync(c->out_rgb, r.data(), r.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
            BSG_CUDA(cudaMemsetAsync(c->scalars, 0, sizeof(StepScalars), c->stream));
            launch_loss(c, dc, rc, gtd);
            ensure_views_buffers(c, 1);
            launch_finalize_loss(c, dc, rc, c->losses_dev, false);
            std::vector<float> g(3 * px);
            double l3[3];
            BSG_CUDA(cudaMemcpyAsync(g.data(), c->dl_dc, g.size() * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
            BSG_CUDA(cudaMemcpyAsync(l3, c->losses_dev, sizeof(l3), cudaMemcpyDeviceToHost, c->stream));
            BSG_CUDA(cudaStreamSynchronize(c->stream));
            if (out_loss3) for (int k = 0; k < 3; ++k) out_loss3[k] = l3[k];
            if (out_dl_dc) for (size_t i = 0; i < 3 * px; ++i) out_dl_dc[i] = g[i];
        }
    });
}

int bsg_project(bsg_ctx* h, const bsg_camera* cam, const bsg_render_config* cfg, uint8_t* out_visible,
                double* out_depth, int32_t* out_rect, uint32_t* out_order, size_t* out_V) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        check_camera(cam);
        bsg_render_config rcfg;
        if (cfg) rcfg = *cfg; else bsg_default_render_config(&rcfg);
        use_device(c);
        const DevCam dc = make_cam(*cam);
        c->global_order = true;  // the depth order of the visible splats is an output here
        try {
            project_and_bin(c, dc, make_render(rcfg));
        } catch (...) {
            c->global_order = false;
            throw;
        }
        c->global_order = false;
        const size_t n = c->n;
        const uint32_t V = c->last_counters.visible;
        std::vector<uint32_t> tiles(n);
        std::vector<uint64_t> keys(n);
        std::vector<float4> rec(3 * n);
        BSG_CUDA(cudaMemcpyAsync(tiles.data(), c->tiles, n * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaMemcpyAsync(keys.data(), c->depth_key, n * 8, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaMemcpyAsync(rec.data(), c->rec, 3 * n * sizeof(float4), cudaMemcpyDeviceToHost, c->stream));
        if (out_order && V)
            BSG_CUDA(cudaMemcpyAsync(out_order, c->vrow[c->depth_sorted], V * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        for (size_t i = 0; i < n; ++i) {
            const bool vis = tiles[i] > 0;
            if (out_visible) out_visible[i] = vis;
            double d = 0;
            uint32_t r01 = 0, r23 = 0;
            if (vis) {
                std::memcpy(&d, &keys[i], 8);
                std::memcpy(&r01, &rec[3 * i + 2].y, 4);
                std::memcpy(&r23, &rec[3 * i + 2].z, 4);
            }
            if (out_depth) out_depth[i] = d;
            if (out_rect) {
                out_rect[4 * i + 0] = vis ? static_cast<int32_t>(r01 & 0xffffu) : 0;
                out_rect[4 * i + 1] = vis ? static_cast<int32_t>(r01 >> 16) : -1;
                out_rect[4 * i + 2] = vis ? static_cast<int32_t>(r23 & 0xffffu) : 0;
                out_rect[4 * i + 3] = vis ? static_cast<int32_t>(r23 >> 16) : -1;
            }
        }
        if (out_V) *out_V = V;
    });
}

int bsg_tile_pairs(bsg_ctx* h, uint32_t* out_tile, uint32_t* out_row, size_t capacity, size_t* out_pairs) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        const size_t P = c->last_counters.pairs;
        if (out_pairs) *out_pairs = P;
        if (!out_tile && !out_row) return;
        if (capacity < P) invalid("pair buffer too small");
        if (P == 0) return;
        if (out_tile && c->last_binning == 1)
            BSG_CUDA(cudaMemcpyAsync(out_tile, c->pkey[c->pairs_sorted], P * 4, cudaMemcpyDeviceToHost, c->stream));
        if (out_tile && c->last_binning == 0) {
            // per-tile binning keeps no tile keys: the ranges give them
            const size_t nt = c->last_ntiles;
            std::vector<uint2> rg(nt);
            BSG_CUDA(cudaMemcpyAsync(rg.data(), c->ranges, nt * sizeof(uint2), cudaMemcpyDeviceToHost, c->stream));
            BSG_CUDA(cudaStreamSynchronize(c->stream));
            for (size_t t = 0; t < nt; ++t)
                for (uint32_t q = rg[t].x; q < rg[t].y && q < P; ++q) out_tile[q] = static_cast<uint32_t>(t);
        }
        if (out_row)
            BSG_CUDA(cudaMemcpyAsync(out_row, c->pval[c->pairs_sorted], P * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int bsg_set_views(bsg_ctx* h, size_t n_views, const bsg_camera* cams, const double* const* gt) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (n_views == 0) invalid("trainer needs at least one view");
        use_device(c);
        for (float* p : c->view_gt)
            if (p) cudaFree(p);
        c->view_gt.clear();
        c->view_cams.assign(cams, cams + n_views);
        for (size_t v = 0; v < n_views; ++v) {
            check_camera(&cams[v]);
            if (!gt || !gt[v]) invalid("view without ground truth");
            const size_t px = static_cast<size_t>(cams[v].width) * cams[v].height;
            std::vector<float> hh(3 * px);
            for (size_t i = 0; i < 3 * px; ++i) hh[i] = static_cast<float>(gt[v][i]);
            float* d = nullptr;
            BSG_CUDA(cudaMalloc(&d, hh.size() * sizeof(float)));
            BSG_CUDA(cudaMemcpyAsync(d, hh.data(), hh.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
            c->view_gt.push_back(d);
            ensure_image_buffers(c, static_cast<int>(cams[v].width), static_cast<int>(cams[v].height));
        }
    });
}

int bsg_trainer_init(bsg_ctx* h, const bsg_trainer_config* cfg) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        materialize(c);  // the parameters current under the previous optimizer state (and its config)
        if (cfg) c->tcfg = *cfg; else bsg_default_trainer_config(&c->tcfg);
        BSG_CUDA(cudaMemsetAsync(c->m, 0, row_stride(c->fd) * c->cap * sizeof(float), c->stream));  // (densify stats too)
        BSG_CUDA(cudaMemsetAsync(c->v, 0, row_stride(c->fd) * c->cap * sizeof(float), c->stream));
        c->adam_t = 0;
        reset_row_meta(c, 0, false);
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        c->iteration = 0;
        bsg_densify_config& d = c->tcfg.densify;
        if (d.stop_iteration == 0) d.stop_iteration = (c->tcfg.iterations * 6) / 10;  // trainer.cpp:148-149
        if (d.enabled && d.interval == 0) invalid("densify interval 0");
        const uint64_t initial = d.global_initial_count ? d.global_initial_count : c->n;
        c->alloc_next = (static_cast<uint64_t>(d.block_id) << 48) + (d.block_id == 0 ? initial : 0);  // trainer.cpp:55-61
        c->alloc_end = (static_cast<uint64_t>(d.block_id) + 1) << 48;
        c->removed_ids.clear();
        c->new_ids.clear();
        c->trainer_ready = true;
    });
}

int bsg_train_steps(bsg_ctx* h, size_t n, const uint32_t* view_seq, double* losses) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!c->trainer_ready) throw Error{BSG_ERR_STATE, "train step before bsg_trainer_init"};
        if (c->view_cams.empty()) throw Error{BSG_ERR_STATE, "train step before bsg_set_views"};
        use_device(c);
        ensure_views_buffers(c, std::max<size_t>(n, 1));
        for (size_t k = 0; k < n; ++k) {
            const uint32_t vi = view_seq[k];
            if (vi >= c->view_cams.size()) invalid("view index out of range");
            train_one(c, c->view_cams[vi], c->view_gt[vi], c->losses_dev + 3 * k);
            maybe_densify(c);
        }
        if (losses && n) {
            std::vector<double> l(3 * n);
            BSG_CUDA(cudaMemcpyAsync(l.data(), c->losses_dev, l.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                     c->stream));
            BSG_CUDA(cudaStreamSynchronize(c->stream));
            for (size_t k = 0; k < n; ++k) losses[k] = l[3 * k];
        }
        collect_stage_times(c);
    });
}

int bsg_train_steps_host(bsg_ctx* h, size_t n, const bsg_camera* cams, const float* const* gts_host,
                         double* losses) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!c->trainer_ready) throw Error{BSG_ERR_STATE, "train step before bsg_trainer_init"};
        if (n && (!cams || !gts_host)) invalid("null views");
        for (size_t k = 0; k < n; ++k) {
            check_camera(&cams[k]);
            if (!gts_host[k]) invalid("null ground truth");
        }
        use_device(c);
        train_steps_from_host(c, n, cams, losses, [&](size_t k, int, float* buf) {
            const size_t px = static_cast<size_t>(cams[k].width) * cams[k].height;
            BSG_CUDA(cudaMemcpyAsync(buf, gts_host[k], 3 * px * sizeof(float), cudaMemcpyHostToDevice,
                                     c->copy_stream));
            return static_cast<const uint8_t*>(nullptr);
        });
    });
}

int bsg_train_steps_host_u8(bsg_ctx* h, size_t n, const bsg_camera* cams, const uint8_t* const* gts_host,
                            double* losses) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!c->trainer_ready) throw Error{BSG_ERR_STATE, "train step before bsg_trainer_init"};
        if (n && (!cams || !gts_host)) invalid("null views");
        size_t need = 0;
        for (size_t k = 0; k < n; ++k) {
            check_camera(&cams[k]);
            if (!gts_host[k]) invalid("null ground truth");
            need = std::max(need, 3 * static_cast<size_t>(cams[k].width) * cams[k].height);
        }
        use_device(c);
        if (need > c->gt_u8_cap) {
            for (auto& p : c->gt_u8) dev_alloc(&p, need);
            c->gt_u8_cap = need;
        }
        train_steps_from_host(c, n, cams, losses, [&](size_t k, int b, float* buf) {
            const size_t bytes = 3 * static_cast<size_t>(cams[k].width) * cams[k].height;
            (void)buf;
            BSG_CUDA(cudaMemcpyAsync(c->gt_u8[b], gts_host[k], bytes, cudaMemcpyHostToDevice, c->copy_stream));
            // the loss kernels read the bytes (v / 255 as the dequantisation of
            // image.cpp): no widening pass competing with the step's kernels
            return static_cast<const uint8_t*>(c->gt_u8[b]);
        });
    });
}

int bsg_train_step_host(bsg_ctx* h, const bsg_camera* cam, const float* gt_host, double* loss) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!c->trainer_ready) throw Error{BSG_ERR_STATE, "train step before bsg_trainer_init"};
        check_camera(cam);
        if (!gt_host) invalid("null ground truth");
        use_device(c);
        ensure_image_buffers(c, static_cast<int>(cam->width), static_cast<int>(cam->height));
        ensure_views_buffers(c, 1);
        const size_t px = static_cast<size_t>(cam->width) * cam->height;
        // the ground-truth upload overlaps the step's projection/sort/forward blend
        BSG_CUDA(cudaMemcpyAsync(c->gt_stage, gt_host, 3 * px * sizeof(float), cudaMemcpyHostToDevice,
                                 c->copy_stream));
        BSG_CUDA(cudaEventRecord(c->gt_ready, c->copy_stream));
        train_one(c, *cam, c->gt_stage, c->losses_dev, c->gt_ready);
        maybe_densify(c);
        double l3[3];
        BSG_CUDA(cudaMemcpyAsync(l3, c->losses_dev, sizeof(l3), cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        if (loss) *loss = l3[0];
        collect_stage_times(c);
    });
}

uint64_t bsg_iteration(const bsg_ctx* h) { return h ? reinterpret_cast<const Ctx*>(h)->iteration : 0; }

int bsg_download_moments(bsg_ctx* h, double* m, double* v) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        materialize(c);
        const size_t n = c->n, cap = c->cap;
        const int fd = c->fd;
        std::vector<float> hm(row_stride(fd) * cap), hv(row_stride(fd) * cap);
        BSG_CUDA(cudaMemcpyAsync(hm.data(), c->m, hm.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaMemcpyAsync(hv.data(), c->v, hv.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        for (int k = 0; k < c->D; ++k)
            for (size_t i = 0; i < n; ++i) {
                if (m) m[k * n + i] = hm[pidx(i, k, fd)];
                if (v) v[k * n + i] = hv[pidx(i, k, fd)];
            }
    });
}

int bsg_upload_moments(bsg_ctx* h, const double* m, const double* v, uint64_t adam_step) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (c->n > 0 && (!m || !v)) invalid("null moment array");
        if (adam_step >= (1ull << 31)) invalid("adam step out of range");
        use_device(c);
        const size_t n = c->n, cap = c->cap;
        const int fd = c->fd;
        for (size_t i = 0; i < static_cast<size_t>(c->D) * n; ++i)
            if (!(v[i] >= 0.0) || !std::isfinite(v[i]) || !std::isfinite(m[i])) invalid("moments not finite or v < 0");
        if (c->round_pending) throw Error{BSG_ERR_STATE, "upload_moments while a consensus round is pending"};
        // the parameters current under the old state first; the rows' metadata
        // slots (densify statistics) kept
        materialize(c);
        std::vector<float> hm(row_stride(fd) * cap), hv(row_stride(fd) * cap);
        BSG_CUDA(cudaMemcpyAsync(hm.data(), c->m, hm.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaMemcpyAsync(hv.data(), c->v, hv.size() * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        for (int k = 0; k < c->D; ++k)
            for (size_t i = 0; i < n; ++i) {
                hm[pidx(i, k, fd)] = static_cast<float>(m[k * n + i]);
                hv[pidx(i, k, fd)] = static_cast<float>(v[k * n + i]);
            }
        BSG_CUDA(cudaMemcpyAsync(c->m, hm.data(), hm.size() * 4, cudaMemcpyHostToDevice, c->stream));
        BSG_CUDA(cudaMemcpyAsync(c->v, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice, c->stream));
        c->adam_t = adam_step;
        reset_row_meta(c, static_cast<uint32_t>(adam_step), false);
        BSG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int bsg_set_adam_sync_interval(bsg_ctx* h, uint32_t every) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (every < 1 || every > kAdamRing / 2) invalid("adam sync interval outside 1..32");
        c->adam_sync = every;
    });
}

int bsg_download_densify_stats(bsg_ctx* h, double* ga, uint32_t* gs) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        // (the rows' metadata slot of m and v, bsg_internal.cuh)
        std::vector<float> a(c->n);
        const size_t pitch = row_stride(c->fd) * sizeof(float);
        if (c->n)
            BSG_CUDA(cudaMemcpy2DAsync(a.data(), 4, c->m + kMetaSlot, pitch, 4, c->n, cudaMemcpyDeviceToHost, c->stream));
        if (gs && c->n)
            BSG_CUDA(cudaMemcpy2DAsync(gs, 4, c->v + kMetaSlot, pitch, 4, c->n, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        if (ga) for (size_t i = 0; i < c->n; ++i) ga[i] = a[i];
    });
}

int bsg_take_removed_ids(bsg_ctx* h, uint64_t* out, size_t capacity, size_t* n) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c || !n) invalid("null argument");
        *n = c->removed_ids.size();
        if (!out) return;
        if (capacity < *n) invalid("capacity too small");
        std::copy(c->removed_ids.begin(), c->removed_ids.end(), out);
        c->removed_ids.clear();
    });
}

int bsg_take_new_ids(bsg_ctx* h, uint64_t* out, size_t capacity, size_t* n) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c || !n) invalid("null argument");
        // trainer.cpp take_new_rows: the added ids still in the cloud, ascending
        std::vector<uint64_t> live;
        std::vector<uint64_t> sorted = c->new_ids;
        std::sort(sorted.begin(), sorted.end());
        for (uint64_t id : sorted)
            if (std::binary_search(c->ids.begin(), c->ids.end(), id)) live.push_back(id);
        *n = live.size();
        if (!out) return;
        if (capacity < *n) invalid("capacity too small");
        std::copy(live.begin(), live.end(), out);
        c->new_ids.clear();
    });
}

int bsg_shared_ids(bsg_ctx* h, uint64_t* out, size_t capacity, size_t* n) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c || !n) invalid("null argument");
        *n = c->sh_rows_host.size();
        if (!out) return;
        if (capacity < *n) invalid("capacity too small");
        for (size_t j = 0; j < *n; ++j) out[j] = c->ids[c->sh_rows_host[j]];
    });
}

int bsg_set_shared(bsg_ctx* h, size_t ns, const uint32_t* rows, const uint32_t* slots, const uint8_t* first,
                   size_t n_slots, const uint32_t* owners) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        materialize(c);  // anchored rows are updated every step: none may be stale
        for (size_t j = 0; j < ns; ++j) {
            if (rows[j] >= c->n) invalid("shared rows missing from cloud");
            if (slots[j] >= n_slots) invalid("slot out of range");
            if (j && rows[j] <= rows[j - 1]) invalid("shared rows not ascending");
        }
        for (size_t s = 0; s < n_slots; ++s)
            if (owners[s] == 0) invalid("slot without owners");
        c->n_shared = ns;
        c->n_slots = n_slots;
        dev_alloc(&c->sh_rows, ns);
        dev_alloc(&c->sh_slots, ns);
        dev_alloc(&c->sh_first, ns);
        dev_alloc(&c->z, c->D * std::max<size_t>(ns, 1));
        dev_alloc(&c->u, c->D * std::max<size_t>(ns, 1));
        dev_alloc(&c->zprev, c->D * std::max<size_t>(n_slots, 1));
        dev_alloc(&c->zslot, c->D * std::max<size_t>(n_slots, 1));
        dev_alloc(&c->in_zprev, n_slots);
        dev_alloc(&c->slot_owners, n_slots);
        dev_alloc(&c->pack, 2 * c->D * std::max<size_t>(n_slots, 1) + n_slots);
        dev_alloc(&c->qref, 4 * std::max<size_t>(n_slots, 1));
        dev_alloc(&c->slot_reset, n_slots);
        if (ns) {
            BSG_CUDA(cudaMemcpyAsync(c->sh_rows, rows, ns * 4, cudaMemcpyHostToDevice, c->stream));
            BSG_CUDA(cudaMemcpyAsync(c->sh_slots, slots, ns * 4, cudaMemcpyHostToDevice, c->stream));
            BSG_CUDA(cudaMemcpyAsync(c->sh_first, first, ns, cudaMemcpyHostToDevice, c->stream));
        }
        if (n_slots) BSG_CUDA(cudaMemcpyAsync(c->slot_owners, owners, n_slots * 4, cudaMemcpyHostToDevice, c->stream));
        c->sh_rows_host.assign(rows, rows + ns);
        c->sh_slots_host.assign(slots, slots + ns);
        c->sh_first_host.assign(first, first + ns);
        install_shared_masks(c);
        BSG_CUDA(cudaMemsetAsync(c->in_zprev, 0, std::max<size_t>(n_slots, 1), c->stream));
        c->anchored = false;
    });
}

int bsg_set_anchor(bsg_ctx* h, const double* z_rows, const double* zprev_slots, const bsg_penalties* rho) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        const std::vector<float> zc = rows_to_cm(z_rows, c->n_shared, c->D);
        if (c->n_shared) {
            BSG_CUDA(cudaMemcpyAsync(c->z, zc.data(), c->D * c->n_shared * 4, cudaMemcpyHostToDevice, c->stream));
            BSG_CUDA(cudaMemsetAsync(c->u, 0, c->D * c->n_shared * 4, c->stream));
        }
        if (c->n_slots) {
            if (zprev_slots) {
                const std::vector<float> zp = rows_to_cm(zprev_slots, c->n_slots, c->D);
                BSG_CUDA(cudaMemcpyAsync(c->zprev, zp.data(), c->D * c->n_slots * 4, cudaMemcpyHostToDevice, c->stream));
                BSG_CUDA(cudaMemsetAsync(c->in_zprev, 1, c->n_slots, c->stream));
            } else {
                BSG_CUDA(cudaMemsetAsync(c->in_zprev, 0, c->n_slots, c->stream));
            }
        }
        if (rho) {
            c->rho = *rho;
            upload_rho(c);
        }
        c->anchored = true;
    });
}

int bsg_set_penalties(bsg_ctx* h, const bsg_penalties* rho) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c || !rho) invalid("null argument");
        if (c->round_pending) throw Error{BSG_ERR_STATE, "set_penalties while a consensus round is pending"};
        use_device(c);
        c->rho = *rho;
        upload_rho(c);
    });
}

int bsg_download_duals(bsg_ctx* h, double* u_rows) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        std::vector<float> hu(c->D * std::max<size_t>(c->n_shared, 1));
        if (c->n_shared) BSG_CUDA(cudaMemcpyAsync(hu.data(), c->u, c->D * c->n_shared * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        cm_to_rows(hu.data(), c->n_shared, c->D, u_rows);
    });
}

int bsg_upload_duals(bsg_ctx* h, const double* u_rows) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!c->anchored) throw Error{BSG_ERR_STATE, "duals before set_anchor"};
        use_device(c);
        const std::vector<float> uc = rows_to_cm(u_rows, c->n_shared, c->D);
        if (c->n_shared) BSG_CUDA(cudaMemcpyAsync(c->u, uc.data(), c->D * c->n_shared * 4, cudaMemcpyHostToDevice, c->stream));
    });
}

int bsg_download_anchor(bsg_ctx* h, double* z_rows) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        std::vector<float> hz(c->D * std::max<size_t>(c->n_shared, 1));
        if (c->n_shared) BSG_CUDA(cudaMemcpyAsync(hz.data(), c->z, c->D * c->n_shared * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        cm_to_rows(hz.data(), c->n_shared, c->D, z_rows);
    });
}

int bsg_download_consensus(bsg_ctx* h, double* z_slots) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        if (c->round_pending) throw Error{BSG_ERR_STATE, "consensus download while a round is pending"};
        round_slots_from_sums(c);
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        std::vector<float> hz(c->D * std::max<size_t>(c->n_slots, 1));
        if (c->n_slots) BSG_CUDA(cudaMemcpyAsync(hz.data(), c->zslot, c->D * c->n_slots * 4, cudaMemcpyDeviceToHost, c->stream));
        BSG_CUDA(cudaStreamSynchronize(c->stream));
        cm_to_rows(hz.data(), c->n_slots, c->D, z_slots);
    });
}

int bsg_apply_broadcast(bsg_ctx* h, const double* z_slots, size_t n_reset, const uint32_t* reset_slots, double alpha,
                        int relax) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        check_round_ready(c);
        use_device(c);
        if (c->n_slots) {
            const std::vector<float> zc = rows_to_cm(z_slots, c->n_slots, c->D);
            BSG_CUDA(cudaMemcpyAsync(c->zslot, zc.data(), c->D * c->n_slots * 4, cudaMemcpyHostToDevice, c->stream));
            c->zslot_from_pack = false;
            BSG_CUDA(cudaMemcpyAsync(c->zprev, zc.data(), c->D * c->n_slots * 4, cudaMemcpyHostToDevice, c->stream));
            BSG_CUDA(cudaMemsetAsync(c->in_zprev, 1, c->n_slots, c->stream));
        }
        bsg_round_args args{};
        args.n_reset = n_reset;
        args.reset_slots = reset_slots;
        upload_resets(c, &args);
        round_apply_broadcast(c, alpha, relax != 0, n_reset > 0);
        BSG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int bsg_nccl_unique_id(uint8_t out_id[128]) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId id;
        NcclApi& n = nccl_api();
        const ncclResult_t r = n.get_unique_id(&id);
        if (r != ncclSuccess) throw Error{BSG_ERR_NCCL, n.error_string(r)};
        std::memcpy(out_id, &id, 128);
    });
}

// Round watchdog (the reference's per-message timeouts,
// runtime.cpp:44-53,98-119): poll the round's event; between polls check the
// NCCL communicator for an asynchronous error, and give up after the round
// timeout (0 = wait forever). Either failure aborts the communicator, so the
// collective cannot hang the process, and surfaces as BSG_ERR_NCCL.
void wait_round(Ctx* c) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        const cudaError_t q = cudaEventQuery(c->round_done);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) BSG_CUDA(q);
        if (c->nccl) {
            NcclApi& napi = nccl_api();
            ncclResult_t ae = ncclSuccess;
            napi.comm_get_async_error(static_cast<ncclComm_t>(c->nccl), &ae);
            if (ae != ncclSuccess && ae != ncclInProgress) {
                napi.comm_abort(static_cast<ncclComm_t>(c->nccl));
                c->nccl = nullptr;
                c->round_pending = false;
                throw Error{BSG_ERR_NCCL, std::string("consensus round: NCCL async error: ") + napi.error_string(ae)};
            }
        }
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (c->round_timeout > 0 && el > c->round_timeout) {
            if (c->nccl) {
                nccl_api().comm_abort(static_cast<ncclComm_t>(c->nccl));
                c->nccl = nullptr;
            }
            c->round_pending = false;
            throw Error{BSG_ERR_NCCL, "consensus round timed out after " + std::to_string(c->round_timeout) + " s"};
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

int bsg_comm_init(bsg_ctx* h, const uint8_t id[128], int nranks, int rank) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (nranks < 1 || rank < 0 || rank >= nranks) invalid("bad rank layout");
        use_device(c);
        c->nranks = nranks;
        c->rank = rank;
        // a one-rank communicator is created too: its AllReduces are local
        // copies, and the NCCL path runs (and is tested) on a single GPU
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        ncclComm_t comm;
        NcclApi& napi = nccl_api();
        const ncclResult_t r = napi.comm_init_rank(&comm, nranks, uid, rank);
        if (r != ncclSuccess) throw Error{BSG_ERR_NCCL, std::string("ncclCommInitRank: ") + napi.error_string(r)};
        c->nccl = comm;
    });
}

int bsg_comm_init_local(bsg_ctx* const* hs, size_t k) {
    return guarded([&] {
        if (!hs || k == 0) invalid("no contexts");
        std::vector<Ctx*> cs(k);
        for (size_t b = 0; b < k; ++b) {
            cs[b] = reinterpret_cast<Ctx*>(hs[b]);
            if (!cs[b]) invalid("null context");
            for (size_t a = 0; a < b; ++a)
                if (cs[a]->device == cs[b]->device) invalid("local NCCL group needs one device per context");
        }
        NcclApi& napi = nccl_api();
        ncclUniqueId uid;
        ncclResult_t r = napi.get_unique_id(&uid);
        if (r != ncclSuccess) throw Error{BSG_ERR_NCCL, std::string("ncclGetUniqueId: ") + napi.error_string(r)};
        std::vector<ncclComm_t> comms(k);
        // one process, k ranks: the inits must be grouped (each blocks until all ranks joined)
        napi.group_start();
        for (size_t b = 0; b < k; ++b) {
            use_device(cs[b]);
            r = napi.comm_init_rank(&comms[b], static_cast<int>(k), uid, static_cast<int>(b));
            if (r != ncclSuccess) {
                napi.group_end();
                throw Error{BSG_ERR_NCCL, std::string("ncclCommInitRank: ") + napi.error_string(r)};
            }
        }
        r = napi.group_end();
        if (r != ncclSuccess) throw Error{BSG_ERR_NCCL, std::string("ncclGroupEnd: ") + napi.error_string(r)};
        for (size_t b = 0; b < k; ++b) {
            cs[b]->nccl = comms[b];
            cs[b]->nranks = static_cast<int>(k);
            cs[b]->rank = static_cast<int>(b);
        }
    });
}

int bsg_comm_init_host(bsg_ctx* h, bsg_host_allreduce fn, void* user, int nranks, int rank) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c || !fn) invalid("null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) invalid("bad rank layout");
        c->host_reduce = fn;
        c->host_user = user;
        c->nranks = nranks;
        c->rank = rank;
    });
}

int bsg_set_round_timeout(bsg_ctx* h, double seconds) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!(seconds >= 0)) invalid("negative timeout");
        c->round_timeout = seconds;
    });
}

// The round on the communication stream (c->stream is swapped for the
// duration of the enqueue so the round_* helpers launch there).
struct CommScope {
    Ctx* c;
    cudaStream_t main;
    explicit CommScope(Ctx* ctx) : c(ctx), main(ctx->stream) { c->stream = c->comm_stream; }
    ~CommScope() { c->stream = main; }
};

int bsg_consensus_round_async(bsg_ctx* h, const bsg_round_args* a, const bsg_adapt_args* adapt) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c || !a) invalid("null argument");
        check_round_ready(c);
        if (c->round_pending) throw Error{BSG_ERR_STATE, "consensus round started before the previous one was waited for"};
        use_device(c);
        BSG_CUDA(cudaEventRecord(c->x_ready, c->stream));  // behind the last parameter update
        CommScope scope(c);
        upload_resets(c, a);
        BSG_CUDA(cudaStreamWaitEvent(c->stream, c->x_ready, 0));
        BSG_CUDA(cudaEventRecord(c->round_t0, c->stream));
        round_pack_q(c);
        reduce_nccl(c, c->qref, 4 * c->n_slots, ncclFloat, ncclSum);
        round_pack_main(c, a->alpha, a->relax != 0);
        reduce_nccl(c, c->pack, (c->D + 1) * c->n_slots, ncclFloat, ncclSum);
        round_unpack(c, a->alpha, a->relax != 0, a->n_reset ? c->slot_reset : nullptr, a->n_reset, a->diagnostics != 0);
        // primal^2, dual^2 (each slot by its lowest owner) and flip-count partials
        // summed over ranks: every rank adapts rho on bit-identical inputs
        reduce_nccl(c, c->round_scalars, 3, ncclFloat64, ncclSum);
        if (adapt) round_adapt(c, *adapt);
        if (a->diagnostics) {
            round_pack_duals(c);
            reduce_nccl(c, c->pack, c->D * c->n_slots, ncclFloat, ncclSum);
            round_dual_linf(c);
            round_pack_minmax(c);
            reduce_nccl(c, c->pack, 2 * c->D * c->n_slots, ncclFloat, ncclMax);
            round_spread(c);
        }
        BSG_CUDA(cudaEventRecord(c->round_t1, c->stream));
        BSG_CUDA(cudaMemcpyAsync(c->round_host, c->round_scalars, 8 * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
        // rho (adapted on the device or not) rides in the same pinned block, so
        // the wait never touches the compute stream
        BSG_CUDA(cudaMemcpyAsync(c->round_host + 8, c->rho_state, 5 * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
        BSG_CUDA(cudaEventRecord(c->round_done, c->stream));
        c->round_pending = true;
        c->round_diag = a->diagnostics != 0;
    });
}

int bsg_consensus_wait(bsg_ctx* h, bsg_round_result* out, bsg_penalties* rho_out) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (!c->round_pending) throw Error{BSG_ERR_STATE, "no consensus round pending"};
        use_device(c);
        wait_round(c);
        c->round_pending = false;
        const double* rs = c->round_host + 8;
        c->rho = bsg_penalties{rs[0], rs[1], rs[2], rs[3], rs[4]};
        if (rho_out) *rho_out = c->rho;
        float ms = 0;
        cudaEventElapsedTime(&ms, c->round_t0, c->round_t1);
        const double* sc = c->round_host;
        if (out) {
            out->primal = std::sqrt(sc[0]);
            out->dual = std::sqrt(sc[1]);
            out->flipped = static_cast<uint64_t>(sc[2]);
            out->dual_mean_linf = c->round_diag ? sc[3] : 0.0;
            out->max_disagreement = c->round_diag ? sc[4] : 0.0;
            out->ms = ms;
        }
    });
}

int bsg_consensus_round(bsg_ctx* h, const bsg_round_args* a, bsg_round_result* out) {
    const int st = bsg_consensus_round_async(h, a, nullptr);
    if (st != BSG_OK) return st;
    return bsg_consensus_wait(h, out, nullptr);
}

int bsg_group_consensus_round(bsg_ctx* const* hs, size_t k, const bsg_round_args* a, bsg_round_result* out) {
    return guarded([&] {
        if (!hs || k == 0 || !a) invalid("no block contributions");
        std::vector<Ctx*> cs(k);
        for (size_t b = 0; b < k; ++b) {
            cs[b] = reinterpret_cast<Ctx*>(hs[b]);
            if (!cs[b]) invalid("null context");
            check_round_ready(cs[b]);
            if (cs[b]->n_slots != cs[0]->n_slots || cs[b]->D != cs[0]->D) invalid("slot layouts differ");
        }
        Ctx* const* cp = cs.data();
        for (Ctx* c : cs) {
            use_device(c);
            upload_resets(c, a);
            round_pack_q(c);
        }
        reduce_group(cp, k, &Ctx::qref, 4 * cs[0]->n_slots, false);
        for (Ctx* c : cs) {
            use_device(c);
            round_pack_main(c, a->alpha, a->relax != 0);
        }
        reduce_group(cp, k, &Ctx::pack, (cs[0]->D + 1) * cs[0]->n_slots, false);
        double primal2 = 0, dual2 = 0, flips = 0;  // per-block partials, summed in block order
        for (size_t b = 0; b < k; ++b) {
            Ctx* c = cs[b];
            use_device(c);
            round_unpack(c, a->alpha, a->relax != 0, a->n_reset ? c->slot_reset : nullptr, a->n_reset,
                         a->diagnostics != 0);
            double sc[8];
            BSG_CUDA(cudaMemcpyAsync(sc, c->round_scalars, sizeof(sc), cudaMemcpyDeviceToHost, c->stream));
            BSG_CUDA(cudaStreamSynchronize(c->stream));
            primal2 += sc[0];
            dual2 += sc[1];
            flips += sc[2];
        }
        double linf = 0, spread = 0;
        if (a->diagnostics) {
            for (Ctx* c : cs) {
                use_device(c);
                round_pack_duals(c);
            }
            reduce_group(cp, k, &Ctx::pack, cs[0]->D * cs[0]->n_slots, false);
            use_device(cs[0]);
            round_dual_linf(cs[0]);
            for (Ctx* c : cs) {
                use_device(c);
                round_pack_minmax(c);
            }
            reduce_group(cp, k, &Ctx::pack, 2 * cs[0]->D * cs[0]->n_slots, true);
            use_device(cs[0]);
            round_spread(cs[0]);
            double sc[8];
            BSG_CUDA(cudaMemcpyAsync(sc, cs[0]->round_scalars, sizeof(sc), cudaMemcpyDeviceToHost, cs[0]->stream));
            BSG_CUDA(cudaStreamSynchronize(cs[0]->stream));
            linf = sc[3];
            spread = sc[4];
        }
        if (out) {
            out->primal = std::sqrt(primal2);
            out->dual = std::sqrt(dual2);
            out->flipped = static_cast<uint64_t>(flips);
            out->dual_mean_linf = linf;
            out->max_disagreement = spread;
            out->ms = 0;
        }
    });
}

int bsg_enable_stage_timing(bsg_ctx* h, int enable) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        c->stage_timing = enable != 0;
    });
}

int bsg_stage_count(void) { return kStCount; }

const char* bsg_stage_name(int i) {
    // bin_scan / bin_emit / bin_sort: tile scan, pair emission, per-tile sort
    // (per-tile binning) or depth sort, pair emission, tile-key sort (global)
    static const char* names[kStCount] = {"preprocess", "compact", "bin_scan", "bin_emit", "bin_sort",
                                          "ranges", "blend_fwd", "loss_ssim", "blend_bwd", "fold", "adam"};
    return (i >= 0 && i < kStCount) ? names[i] : "";
}

int bsg_stage_times(bsg_ctx* h, double* ms) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c || !ms) invalid("null argument");
        for (int s = 0; s < kStCount; ++s) ms[s] = c->stage_ms[s];
    });
}

int bsg_step_counters(bsg_ctx* h, uint64_t* visible, uint64_t* pairs, uint64_t* launches) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        if (visible) *visible = c->last_counters.visible;
        if (pairs) *pairs = c->last_counters.pairs;
        if (launches) *launches = c->step_launches;
    });
}

uint64_t bsg_step_blend_evals(const bsg_ctx* h) { return h ? reinterpret_cast<const Ctx*>(h)->last_evals : 0; }

// ---- checked build probe ---------------------------------------------------

__global__ void checked_probe_kernel(int v) { BSG_DASSERT(v != 1); }

int bsg_checked_build(void) {
#ifdef BSG_CHECKED
    return 1;
#else
    return 0;
#endif
}

int bsg_checked_probe(int device) {
    return guarded([&] {
        BSG_CUDA(cudaSetDevice(device));
        checked_probe_kernel<<<1, 1>>>(1);
        BSG_CUDA(cudaGetLastError());
        BSG_CUDA(cudaDeviceSynchronize());
    });
}

// ---- master-round ownership bookkeeping (owners.cu) ----------------------

int bsg_owners_create(int device, size_t n, const uint64_t* ids, const uint32_t* masks, uint32_t blocks,
                      bsg_owner_table** out) {
    return guarded([&] {
        if (!out || (n && (!ids || !masks))) invalid("null argument");
        if (blocks == 0 || blocks > 32) invalid("owner table: 1..32 blocks");
        for (size_t i = 0; i < n; ++i) {
            if (i && ids[i] <= ids[i - 1]) invalid("owner table ids must be strictly ascending");
            if (__builtin_popcount(masks[i]) < 2 || (blocks < 32 && (masks[i] >> blocks)))
                invalid("owner table rows need >= 2 owners among the blocks");
        }
        auto* t = new OwnerTable;
        t->device = device;
        t->blocks = blocks;
        try {
            BSG_CUDA(cudaSetDevice(device));
            BSG_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
            BSG_CUDA(cudaMalloc(&t->totals_dev, 2 * sizeof(uint32_t)));
            BSG_CUDA(cudaMallocHost(&t->totals_host, 2 * sizeof(uint32_t)));
            owners_alloc(t, n);
            if (n) {
                BSG_CUDA(cudaMemcpyAsync(t->ids[0], ids, n * sizeof(uint64_t), cudaMemcpyHostToDevice, t->stream));
                BSG_CUDA(cudaMemcpyAsync(t->mask[0], masks, n * sizeof(uint32_t), cudaMemcpyHostToDevice, t->stream));
            }
            BSG_CUDA(cudaStreamSynchronize(t->stream));
            t->n = static_cast<uint32_t>(n);
        } catch (...) {
            bsg_owners_destroy(reinterpret_cast<bsg_owner_table*>(t));
            throw;
        }
        *out = reinterpret_cast<bsg_owner_table*>(t);
    });
}

int bsg_owners_destroy(bsg_owner_table* h) {
    auto* t = reinterpret_cast<OwnerTable*>(h);
    if (!t) return BSG_OK;
    cudaSetDevice(t->device);
    void* dev[] = {t->ids[0], t->ids[1], t->mask[0], t->mask[1], t->rm, t->chunk, t->totals_dev, t->t_slot,
                   t->t_class, t->t_mask, t->in_ids, t->in_blk, t->in_found};
    for (void* p : dev)
        if (p) cudaFree(p);
    if (t->totals_host) cudaFreeHost(t->totals_host);
    if (t->stream) cudaStreamDestroy(t->stream);
    delete t;
    return BSG_OK;
}

size_t bsg_owners_size(const bsg_owner_table* h) { return h ? reinterpret_cast<const OwnerTable*>(h)->n : 0; }

int bsg_owners_download(const bsg_owner_table* h, uint64_t* ids, uint32_t* masks) {
    return guarded([&] {
        const auto* t = reinterpret_cast<const OwnerTable*>(h);
        if (!t) invalid("null owner table");
        BSG_CUDA(cudaSetDevice(t->device));
        if (t->n && ids)
            BSG_CUDA(cudaMemcpyAsync(ids, t->ids[t->cur], t->n * sizeof(uint64_t), cudaMemcpyDeviceToHost, t->stream));
        if (t->n && masks)
            BSG_CUDA(cudaMemcpyAsync(masks, t->mask[t->cur], t->n * sizeof(uint32_t), cudaMemcpyDeviceToHost, t->stream));
        BSG_CUDA(cudaStreamSynchronize(t->stream));
    });
}

int bsg_owners_remove(bsg_owner_table* h, const uint64_t* const* removed, const size_t* n_removed, uint32_t* out_slot,
                      uint8_t* out_class, uint32_t* out_mask, size_t cap, size_t* out_touched, uint8_t* out_found) {
    return guarded([&] {
        auto* t = reinterpret_cast<OwnerTable*>(h);
        if (!t || !n_removed || !out_touched) invalid("null argument");
        BSG_CUDA(cudaSetDevice(t->device));
        std::vector<uint64_t> ids;
        std::vector<uint32_t> blk;
        for (uint32_t b = 0; b < t->blocks; ++b) {
            if (n_removed[b] && (!removed || !removed[b])) invalid("null removed list");
            for (size_t i = 0; i < n_removed[b]; ++i) {
                ids.push_back(removed[b][i]);
                blk.push_back(b);
            }
        }
        const size_t m = ids.size();
        if (m > t->in_cap) {
            for (void* p : {static_cast<void*>(t->in_ids), static_cast<void*>(t->in_blk), static_cast<void*>(t->in_found)})
                if (p) cudaFree(p);
            t->in_cap = std::max<size_t>(m, 1024);
            BSG_CUDA(cudaMalloc(&t->in_ids, t->in_cap * sizeof(uint64_t)));
            BSG_CUDA(cudaMalloc(&t->in_blk, t->in_cap * sizeof(uint32_t)));
            BSG_CUDA(cudaMalloc(&t->in_found, t->in_cap));
        }
        if (m) {
            BSG_CUDA(cudaMemcpyAsync(t->in_ids, ids.data(), m * sizeof(uint64_t), cudaMemcpyHostToDevice, t->stream));
            BSG_CUDA(cudaMemcpyAsync(t->in_blk, blk.data(), m * sizeof(uint32_t), cudaMemcpyHostToDevice, t->stream));
        }
        // the removals are marked first; the capacity check happens before the
        // compaction commits, so a too-small output leaves the table unchanged
        const uint32_t n_before = t->n;
        const int cur_before = t->cur;
        const uint32_t touched = owners_round(t, t->in_ids, t->in_blk, static_cast<uint32_t>(m), t->in_found);
        *out_touched = touched;
        if (touched > cap) {
            // undo: the compaction swapped buffers; restore the pre-round table
            // (the removal bits were cleared by the compaction, the masks of the
            // old buffer are untouched)
            t->cur = cur_before;
            t->n = n_before;
            throw Error{BSG_ERR_CAPACITY, "owner round: more touched slots than the output capacity"};
        }
        if (touched) {
            if (!out_slot || !out_class || !out_mask) invalid("null output");
            BSG_CUDA(cudaMemcpyAsync(out_slot, t->t_slot, touched * sizeof(uint32_t), cudaMemcpyDeviceToHost, t->stream));
            BSG_CUDA(cudaMemcpyAsync(out_class, t->t_class, touched, cudaMemcpyDeviceToHost, t->stream));
            BSG_CUDA(cudaMemcpyAsync(out_mask, t->t_mask, touched * sizeof(uint32_t), cudaMemcpyDeviceToHost, t->stream));
        }
        if (out_found && m) BSG_CUDA(cudaMemcpyAsync(out_found, t->in_found, m, cudaMemcpyDeviceToHost, t->stream));
        BSG_CUDA(cudaStreamSynchronize(t->stream));
    });
}

int bsg_last_binning(const bsg_ctx* h) { return h ? reinterpret_cast<const Ctx*>(h)->last_binning : -1; }

uint64_t bsg_launch_count(const bsg_ctx* h) { return h ? reinterpret_cast<const Ctx*>(h)->launches : 0; }

void* bsg_stream(bsg_ctx* h) { return h ? reinterpret_cast<Ctx*>(h)->stream : nullptr; }

int bsg_synchronize(bsg_ctx* h) {
    return guarded([&] {
        auto* c = reinterpret_cast<Ctx*>(h);
        if (!c) invalid("null context");
        use_device(c);
        BSG_CUDA(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"
