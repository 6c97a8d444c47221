// Internal declarations of the B200 (sm_100a) blocksplat hot path.
// Device state is FP32 component-major ([D][cap]); the per-Gaussian
// projection that decides integer footprints and depth order runs in FP64
// (see preprocess.cu).
#pragma once

#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/bsgpu.h"

namespace bsg {

constexpr int kTile = 16;             // 16x16 pixel tiles, one thread per pixel
// Splats whose footprint rect covers at least kWideArea pixels (near-plane
// grazers spanning most of the image) accumulate their image-space gradient
// in FP64 (compact slot per splat): their fold cancels to ~1e-5 of the sum, so
// FP32 atomics in arbitrary order would leave O(10%) run-to-run noise.
constexpr uint32_t kWideArea = 4096;
constexpr uint32_t kWideCap = 65536;  // wide splats per step with an FP64 slot (others stay FP32)
constexpr uint32_t kNoWide = 0xffffffffu;
// rec[3i+2].w: the splat's gradient target -- its row i, or kWideBit | slot
// for a wide footprint's FP64 slot (the backward blend adds to it directly).
constexpr uint32_t kWideBit = 0x80000000u;
constexpr int kTileThreads = kTile * kTile;
// Splat record scale: the factor L of minv (= L^T L) and the affine offsets k
// are stored times sqrt(log2(e) / 2), so |L d|^2 is the exponent of ex2. The
// backward's accumulators then carry kQScale^2 (mean path) and kQScale^4
// (covariance path), removed when the fold reads them.
constexpr double kQScale = 0.84932180028801904272;  // sqrt(0.5 * log2(e))
constexpr double kQScale2 = kQScale * kQScale;
constexpr int kMaxFd = 12;            // SH degree 1 (cloud.hpp:16-17)
constexpr int kMaxD = 11 + kMaxFd;    // pos3 rot4 ls3 feat fd op1
constexpr double kSh0 = 0.28209479177387814;  // cloud.hpp:14
constexpr double kSh1 = 0.4886025119029199;   // cloud.hpp:15

// Component offsets of the [D][cap] parameter matrix.
constexpr int kPos = 0, kRot = 3, kLs = 7, kFeat = 10;
__host__ __device__ inline int op_comp(int fd) { return kFeat + fd; }

// Parameter and Adam-moment storage (x, m, v): row-major, row_stride(fd)
// FP32 per row (64 B at SH degree 0, 128 B at degree 1), slots
//   [pos0 pos1 pos2 ls0 ls1 ls2 op -][rot0 rot1 rot2 rot3 feat0 .. feat(fd-1) -..]
// so the per-step culling read of every row (position + log-scale) is one
// 32-byte sector and a whole row is 2 (4) sectors: the kernels that touch a
// subset of rows (the preprocess's candidates, densification, consensus
// packs) gather whole rows instead of one sector per component.
// Slot 7 (padding of the first sector) carries per-row metadata, so it rides
// along with sectors the kernels read or write whole anyway (a separate 4-byte
// array costs a DRAM read-modify-write per scattered update): in x the Adam
// step the row is current at (lazy Adam, u32 bits), in m the densify gradient
// accumulator and in v the densify visibility count (u32 bits)
// (trainer.cpp:284-289).
__host__ __device__ constexpr int row_stride(int fd) { return fd <= 4 ? 16 : 32; }
constexpr int kMetaSlot = 7;
__host__ __device__ constexpr int pslot(int comp, int fd) {
    return comp < kRot ? comp
                       : (comp < kLs ? 8 + (comp - kRot)
                                     : (comp < kFeat ? 3 + (comp - kLs) : (comp < kFeat + fd ? 12 + (comp - kFeat) : 6)));
}
__host__ __device__ inline size_t pidx(size_t row, int comp, int fd) {
    return row * static_cast<size_t>(row_stride(fd)) + static_cast<size_t>(pslot(comp, fd));
}

// Camera as consumed by kernels (by value).
struct DevCam {
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    double center[3];  // -R^T t (camera.hpp:31)
    int W, H;
    int tiles_x, tiles_y;
};

struct DevRender {
    double near_plane, dilation, alpha_clamp, tstop, sigma_extent;
    float bg[3];
    double lambda;
};

// Per-step counters kept in device memory (read back once per step).
struct StepCounters {
    uint32_t visible;   // V
    uint32_t pairs;     // P
    uint32_t overflow;  // a run of equal 32-bit depth keys too long for the fix-up
    uint32_t visible_pre;  // visible count as seen by the preprocess (sizes the depth key)
    uint32_t wide;         // wide splats given an FP64 gradient slot this step
    uint32_t dens_keep;    // densify: surviving rows
    uint32_t dens_children;// densify: added rows
    uint32_t pad3;
    unsigned long long evals;  // (pixel, contributor) alpha evaluations composited by the forward blend
    unsigned long long zmin_inv;  // ~bits of the smallest visible FP64 depth (atomicMax of the complement)
    unsigned long long zmax;      // bits of the largest visible FP64 depth
    uint32_t depth_hist[8][256];  // digit histograms of the visible depth keys (filled by the compaction)
    uint32_t tile_hist[2][256];   // digit histograms of the tile keys (filled by the pair emission)
    uint32_t order_hist[1024];    // tiles per launch-order bucket (1023 - min(pairs, 1023)), tile scan
    uint32_t order_cur[1024];     // per-bucket placement cursors of the launch order
    uint32_t tile_max;            // largest per-tile pair count
    uint32_t pad4;
    unsigned long long pairs_wide;  // P without 32-bit wrap-around (the 2^30 capacity guard)
};

// Host-mapped pinned mailbox: the compaction and the pair-offset scan write
// their totals here (value, then __threadfence_system, then the sequence
// word), so the host learns V and P by polling instead of a copy + stream
// sync, while the kernel enqueued behind them keeps the GPU busy.
struct Mailbox {
    uint32_t seq_v, V, visible_pre, pad0;
    uint32_t seq_p, P, overflow, max_tile;  // max_tile: largest per-tile pair count (per-tile binning)
    uint32_t pairs_big, pad1, pad2, pad3;   // the view's tile pairs reach kMaxPairs (32-bit offsets, 30-bit look-back counts)
};
constexpr unsigned long long kMaxPairs = 1ull << 30;

// Per-tile binning sorts a tile's pairs by (FP64 depth bits, row) in shared
// memory with a bitonic network; a view with a tile holding more pairs uses
// the global depth sort + stable tile sort. cfg 5 (1080p): a 2048 cap beats
// 1024 at 4M rows (3.60 -> 3.48 ms/iter) and ties 4096 at 8M-16M.
constexpr uint32_t kTileSortCap = 2048;
// Each tile's pair count and emission cursor are split kTileSub ways (by row
// mod kTileSub): the preprocess's counting reductions and the emission's slot
// claims on a busy tile spread over kTileSub addresses instead of
// serialising on one (the tile scan lays the sub-ranges end to end).
constexpr uint32_t kTileSub = 4;

// Device-side invariant checks of the checked build (lib/libbsgpu_checked.so,
// -DBSG_CHECKED; tests/test_gpu_checked.py): a failed check prints its site
// and traps, so the entry point returns BSG_ERR_CUDA. Compiled out otherwise.
#ifdef BSG_CHECKED
#define BSG_DASSERT(cond)                                                                       \
    do {                                                                                      \
        if (!(cond)) {                                                                        \
            printf("BSG_DASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));              \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)
#else
#define BSG_DASSERT(cond) \
    do {                  \
    } while (0)
#endif

// Where a scan's final CTA publishes its total (all null: nowhere).
struct Publish {
    uint32_t* val = nullptr;
    uint32_t* seq_word = nullptr;
    uint32_t seq = 0;
    const uint32_t* extra_src = nullptr;  // copied to extra_dst before the sequence word
    uint32_t* extra_dst = nullptr;
};

// One decoupled look-back launch: status words carry the launch's epoch (no
// zeroing between launches), tile ids come from a monotonic 64-bit ticket.
struct Lookback {
    unsigned long long* ticket;
    unsigned long long base;
    uint32_t epoch;
};

// Scalars reduced on the device every step.
struct StepScalars {
    double l1_sum;
    double ssim_sum;
    double penalty;
    double pad;
};

enum Stage {
    kStPreprocess = 0, kStCompact, kStDepthSort, kStPairs, kStTileSort, kStRanges, kStBlendFwd, kStLoss,
    kStBlendBwd, kStFold, kStAdam, kStCount
};

// Device owner table of the master round (owners.cu): the
// consensus slot table's ids (ascending) and owner bitmasks, ping-pong for
// the compaction, plus the touched-slot outputs of the last round.
struct OwnerTable {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint32_t n = 0, blocks = 0;
    size_t cap = 0;
    int cur = 0;
    uint64_t* ids[2] = {nullptr, nullptr};
    uint32_t* mask[2] = {nullptr, nullptr};
    uint32_t* rm = nullptr;      // this round's removal bits per slot (kept zero between rounds)
    uint2* chunk = nullptr;      // per-chunk (kept, touched) counts -> offsets
    uint32_t* totals_dev = nullptr;
    uint32_t* totals_host = nullptr;  // pinned
    size_t t_cap = 0;
    uint32_t* t_slot = nullptr;  // touched slots (pre-compaction numbering), ascending
    uint8_t* t_class = nullptr;  // 1 reset, 2 unshared, 3 dead
    uint32_t* t_mask = nullptr;  // owner mask after the round
    size_t in_cap = 0;
    uint64_t* in_ids = nullptr;  // removed ids of the round (all blocks)
    uint32_t* in_blk = nullptr;
    uint8_t* in_found = nullptr;
};
void owners_alloc(OwnerTable* t, size_t n);
uint32_t owners_round(OwnerTable* t, const uint64_t* d_in_ids, const uint32_t* d_in_blk, uint32_t m, uint8_t* d_found);

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // host ground-truth uploads (e2e path)
    cudaEvent_t gt_ready = nullptr;
    cudaEvent_t gt_ready_b = nullptr, gt_free[2] = {nullptr, nullptr};  // double-buffered host ground truth
    cudaStream_t comm_stream = nullptr;  // consensus rounds (overlap with the next step)
    cudaEvent_t x_ready = nullptr, round_done = nullptr, round_t0 = nullptr, round_t1 = nullptr;
    bool round_pending = false;
    bool tile_scan_used = false;  // the multi-CTA tile scan ran since this step's counters were zeroed
    bool round_diag = false;
    double* round_host = nullptr;        // pinned copy of round_scalars
    int fd = 3, D = 14;
    size_t n = 0, cap = 0;
    std::vector<uint64_t> ids;

    // parameters and optimizer state, [D][cap]
    float* x = nullptr;
    float* m = nullptr;
    float* v = nullptr;

    // per-row scratch
    float4* rec = nullptr;         // 3 x float4 per row: {l11,l12,l22,k1},{k2,o,r,g},{b,rect01,rect23,target}
    uint64_t* depth_key = nullptr; // FP64 depth bits
    uint32_t* tiles = nullptr;     // tiles touched, 0 = culled
    float4* g2d = nullptr;         // 3 x float4 per row: {gmx,gmy,gc00,gc01},{gc11,gr,gg,gb},{go,-,-,-}
    double* g2d_wide = nullptr;    // [kWideCap][9] FP64 gradients of wide splats (kWideBit | slot in rec[3i+2].w)
    float4* adam_ring = nullptr;   // per Adam step t, at t % kAdamRing: {1/bc1, 1/bc2, lr_pos, -}
    uint32_t* vis_prefix = nullptr;// visible rows before each 32-row word (visible position = prefix + rank in word)
    uint32_t* vis_mask = nullptr;  // 1 bit per row: visible this step (written by the compaction)
    uint32_t* sh_mask = nullptr;   // 1 bit per row: shared (has an anchor)
    uint32_t* sh_prefix = nullptr; // shared rows before each 32-row word (anchor index = prefix + rank in word)

    // compaction + depth sort (ping-pong)
    uint64_t* vkey[2] = {nullptr, nullptr};
    uint32_t* vrow[2] = {nullptr, nullptr};
    uint32_t* poff = nullptr;      // pair offsets (exclusive scan over sorted splats)
    uint32_t* vis_rows = nullptr;  // visible rows in ascending row order (compaction output)
    int depth_sorted = 0;          // which ping-pong buffer holds the sorted result

    // tile pairs (ping-pong)
    size_t pcap = 0;
    uint32_t* pkey[2] = {nullptr, nullptr};
    uint32_t* pval[2] = {nullptr, nullptr};
    int pairs_sorted = 0;
    uint2* ranges = nullptr;
    uint32_t* tile_order = nullptr;  // blend launch order: tiles by descending pair count
    uint32_t* tile_cnt = nullptr;    // pairs per tile (counted by the preprocess)
    uint32_t* tile_cur = nullptr;    // per-tile write cursors of the pair emission
    size_t ranges_cap = 0;
    bool global_order = false;       // bsg_project: global depth sort path (exposes the depth order)
    int last_binning = 0;            // 0: per-tile sort, 1: global sorts (what the pair buffers hold)
    size_t last_ntiles = 0;
    uint32_t last_max_tile = 0;      // largest tile of the previous binning (picks the path up front)

    // radix / scan scratch
    unsigned long long* scan_status = nullptr;   // decoupled look-back status words (epoch-tagged)
    size_t scan_status_cap = 0;
    unsigned long long* radix_status = nullptr;
    size_t radix_status_cap = 0;
    unsigned long long* lb_ticket = nullptr;  // [2] monotonic tile tickets (scan, radix)
    unsigned long long lb_next[2] = {0, 0};   // host mirror of the tickets handed out
    uint32_t lb_epoch = 0;
    Mailbox* mbox = nullptr;                  // host-mapped pinned
    uint32_t mbox_seq = 0;
    uint32_t* radix_hist = nullptr;    // [8 passes][256]
    uint32_t* counters_dev = nullptr;  // tile-id tickets
    StepCounters* counters = nullptr;  // device
    StepCounters* counters_host = nullptr;  // pinned
    StepScalars* scalars = nullptr;         // device
    double* losses_dev = nullptr;           // per-step losses
    size_t losses_cap = 0;

    // images for the current view
    size_t img_cap = 0;  // pixels
    float* out_rgb = nullptr;
    float* out_T = nullptr;
    uint32_t* out_n = nullptr;
    uint32_t* out_last = nullptr;
    float* dl_dc = nullptr;
    float* ssim_f = nullptr;   // 9 planes of the valid window grid
    float* gt_stage = nullptr; // host ground truth staging (e2e path)
    float* gt_stage_b = nullptr;  // second staging buffer (bsg_train_steps_host)
    uint8_t* gt_u8[2] = {nullptr, nullptr};  // 8-bit host images in flight (bsg_train_steps_host_u8)
    size_t gt_u8_cap = 0;

    // resident training views
    std::vector<bsg_camera> view_cams;
    std::vector<float*> view_gt;

    // training
    bool trainer_ready = false;
    bsg_trainer_config tcfg{};
    uint64_t iteration = 0;
    uint64_t adam_t = 0;
    // every row caught up every adam_sync steps (1 = dense Adam; <= kAdamRing / 2). 16: the
    // full replays run as one MUFU-bound kernel, cheaper than the same steps replayed piecemeal
    // for the culling candidates (cfg 3 preprocess + Adam: 355 / 347 / 346 / 349 us at 32 / 16 / 12 / 8)
    uint32_t adam_sync = 16;
    // densification (trainer.cpp:301-385)
    double scene_extent = 1e-9;
    uint64_t alloc_next = 0, alloc_end = 0;  // IdAllocator
    std::vector<uint64_t> removed_ids, new_ids;
    std::vector<uint32_t> sh_rows_host, sh_slots_host;  // host copies of the shared bookkeeping
    std::vector<uint8_t> sh_first_host;

    // consensus (per block)
    size_t n_shared = 0, n_slots = 0;
    uint32_t* sh_rows = nullptr;
    uint32_t* sh_slots = nullptr;
    uint8_t* sh_first = nullptr;
    float* z = nullptr;         // anchor [D][n_shared]
    float* u = nullptr;         // duals  [D][n_shared]
    float* zprev = nullptr;     // [D][n_slots]
    float* zslot = nullptr;     // consensus of the last round [D][n_slots] (materialised on demand)
    bool zslot_from_pack = false;  // zslot is stale; `pack` holds the reduced sums
    uint8_t* in_zprev = nullptr;
    uint32_t* slot_owners = nullptr;
    float* pack = nullptr;      // [D+1][n_slots] (+1 = flip flag)
    float* qref = nullptr;      // [4][n_slots]
    uint8_t* slot_reset = nullptr;
    double* round_scalars = nullptr;  // primal2, dual2, flips, maxdis, linf
    bool anchored = false;
    bsg_penalties rho{};           // host copy; the device copy below is authoritative for Adam
    float* rho_dev = nullptr;      // per-component rho [kMaxD] read by the penalty + Adam
    double* rho_state = nullptr;   // rho_p, rho_q, rho_s, rho_f, rho_o (adapted on the device)
    void* nccl = nullptr;       // ncclComm_t
    bsg_host_allreduce host_reduce = nullptr;  // host communicator (bsg_comm_init_host)
    void* host_user = nullptr;
    void* host_buf = nullptr;   // pinned staging of the host communicator
    size_t host_buf_cap = 0;
    double round_timeout = 0;   // seconds, 0 = none (bsg_set_round_timeout)
    int nranks = 1, rank = 0;

    // measurement
    bool stage_timing = false;
    cudaEvent_t ev[kStCount + 1] = {};
    float stage_ms[kStCount] = {};
    uint64_t launches = 0;
    uint64_t step_launches = 0;
    uint64_t last_evals = 0;  // forward-blend evaluations of the last step (read when stage timing is on)
    StepCounters last_counters{};
};

// ---- error plumbing -----------------------------------------------------
void set_error(const std::string& msg);
struct Error {
    int code;
    std::string msg;
};
#define BSG_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw ::bsg::Error{BSG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
    } while (0)
#define BSG_LAUNCHED(ctx)                                                                  \
    do {                                                                                   \
        (ctx)->launches++;                                                                 \
        (ctx)->step_launches++;                                                            \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess)                                                             \
            throw ::bsg::Error{BSG_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)}; \
    } while (0)

// Programmatic dependent launch (PDL) for the kernels of a step: each one is
// launched with programmatic stream serialisation, so its CTAs are scheduled
// while the previous kernel drains, and starts with pdl_prologue(): wait until
// the previous grid has completed and flushed its writes, then allow the next
// kernel to be scheduled. (Without the launch attribute both are no-ops.)
__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();  // false when BSG_NO_PDL is set (A/B measurements)
constexpr unsigned long long kPdlMaxCtas = 4096;

// Programmatic launch for any grid size (the Adam kernels: streaming, behind
// the fold; measured +0.8% at cfg 2, neutral at cfg 5).
struct PdlAlways {};

template <typename... KArgs, typename... Args>
void launch_pdl_impl(bool always, cudaStream_t stream, dim3 grid, dim3 block, size_t smem, void (*kernel)(KArgs...),
                     Args&&... args);

template <typename... KArgs, typename... Args>
void launch_pdl(PdlAlways, cudaStream_t stream, dim3 grid, dim3 block, size_t smem, void (*kernel)(KArgs...),
                Args&&... args) {
    launch_pdl_impl(true, stream, grid, block, smem, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
void launch_pdl(cudaStream_t stream, dim3 grid, dim3 block, size_t smem, void (*kernel)(KArgs...), Args&&... args) {
    launch_pdl_impl(false, stream, grid, block, smem, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
void launch_pdl_impl(bool always, cudaStream_t stream, dim3 grid, dim3 block, size_t smem, void (*kernel)(KArgs...),
                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // large grids gain nothing from an early launch and measured slower with
    // it (cfg 5, 16M rows: 10.24 vs 9.90 ms/iter); small ones hide the launch gap
    const unsigned long long ctas = static_cast<unsigned long long>(grid.x) * grid.y * grid.z;
    cfg.numAttrs = pdl_enabled() && (always || ctas <= kPdlMaxCtas) ? 1 : 0;
    BSG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Width of the range-normalised depth key for V visible splats: ~6 bits more
// than log2(V), so equal keys (distinct depths in one bucket) stay rare,
// rounded up to whole 8-bit radix digits.
__host__ __device__ inline int depth_key_bits(uint32_t V) {
    int lg = 0;
    while (lg < 32 && (1ull << lg) < V) ++lg;
    const int b = ((lg + 6 + 7) / 8) * 8;
    return b < 16 ? 16 : (b > 32 ? 32 : b);
}

// ---- building blocks (scan.cu, radix.cu) -------------------------------
// Visible rows (ascending) from the preprocess's visibility mask: the
// per-tile binning path's compaction (no depth keys).
void compact_visible_mask(Ctx* c, uint32_t n, const Publish& pub);
// Exclusive scan of n u32 values read through a gather (in[idx ? idx[i] : i]),
// optional predicate compaction. Result in out; total in *total_dev.
void scan_exclusive_u32(Ctx* c, const uint32_t* in, const uint32_t* gather_idx, uint32_t* out, uint32_t n,
                        uint32_t* total_dev, const Publish& pub = Publish{});
// Look-back bookkeeping for one launch of `grid` CTAs (which: 0 scan, 1 radix).
Lookback next_lookback(Ctx* c, int which, uint32_t grid);
// Polls the mailbox until *seq_word == seq (checks the stream for errors while waiting).
void wait_mailbox(Ctx* c, const volatile uint32_t* seq_word, uint32_t seq);
// Stable compaction of rows with tiles[i] > 0: writes keys/rows in row order and V.
// key32: the 32-bit range-normalised depth key (bits(z) - bits(zmin)) >> shift
// into vkey (as u32) with its 4 digit histograms; otherwise the full FP64 bits
// with all 8 digit histograms.
void compact_visible(Ctx* c, uint32_t n, bool key32, const Publish& pub = Publish{});
// Stable LSD radix sort (onesweep) of (u64 key, u32 val) / (u32 key, u32 val)
// over `passes` 8-bit digits from bit 0. d_hist holds the per-pass digit
// counts (produced by the kernel that wrote the keys) and is turned into
// offsets in place; h_hist (nullable) is a host copy used to skip passes
// whose digit is constant. Result lands in buffer *sel.
void radix_sort_u64(Ctx* c, uint64_t* keys[2], uint32_t* vals[2], uint32_t n, int first_pass, int passes,
                    uint32_t* d_hist, const uint32_t* h_hist, int* sel);
void radix_sort_u32(Ctx* c, uint32_t* keys[2], uint32_t* vals[2], uint32_t n, int first_pass, int passes,
                    uint32_t* d_hist, const uint32_t* h_hist, int* sel);
// Digit histograms of the compacted 32-bit depth keys into counters->depth_hist
// (zeroed by the step's counter reset); n and the digit count come from the
// device counters (visible, depth_key_bits(visible_pre)), so it is enqueued
// before the host knows V.
void launch_depth_hist(Ctx* c, const uint32_t* keys);
// Sorts runs of equal 32-bit depth keys by the full FP64 depth bits of their
// rows (stable); sets *long_run if a run exceeds 64 (caller redoes the full sort).
void depth_tie_fixup(Ctx* c, uint32_t* keys, uint32_t* rows, const uint64_t* depth_bits, uint32_t V,
                     uint32_t* long_run);

// ---- rasterizer stages (preprocess.cu, raster.cu, ssim.cu, adam.cu) ----
DevCam make_cam(const bsg_camera& c);
DevRender make_render(const bsg_render_config& r);
void launch_preprocess(Ctx* c, const DevCam& cam, const DevRender& rc);
void launch_pairs(Ctx* c, const DevCam& cam, uint32_t V);
// Per-tile binning: tile ranges / cursors / launch order from the preprocess's
// tile counts (P and the largest count to the mailbox under `seq`), the rows
// placed into their tiles (pval[1]), each tile sorted by (depth, row) into pval[0].
void launch_tile_scan(Ctx* c, const DevCam& cam, uint32_t seq);
void launch_tile_scan_multi(Ctx* c, uint32_t ntiles, uint32_t seq);  // (scan.cu; views over 1024 tiles)
void launch_emit_tiles(Ctx* c, const DevCam& cam);
void launch_tile_sort(Ctx* c, const DevCam& cam, uint32_t max_tile);
// The f32 arrays of the GSPL checkpoint section ((11 + fd) n floats, section order) into out.
void launch_gspl_floats(Ctx* c, float* out);
void launch_ranges(Ctx* c, const DevCam& cam, uint32_t V, uint32_t P);
void launch_blend_fwd(Ctx* c, const DevCam& cam, const DevRender& rc);
void launch_loss(Ctx* c, const DevCam& cam, const DevRender& rc, const float* gt);
void launch_loss(Ctx* c, const DevCam& cam, const DevRender& rc, const uint8_t* gt);  // 8-bit ground truth
void launch_blend_bwd(Ctx* c, const DevCam& cam, const DevRender& rc);
void launch_fold_grads(Ctx* c, const DevCam& cam, double* g_out /*[D][n] f64*/, double* sgn, uint8_t* vis);
struct AdamStep {
    float lr[kMaxD];
    float b1, b2, eps, omb1, omb2;
    float inv_bc1, inv_bc2;
    int has_anchor;
    uint32_t t;  // the step's Adam count (after the increment, trainer.cpp:267)
};

// ---- lazy Adam ------------------------------------------------------------
// The reference's Adam is dense (every row, every step, trainer.cpp:267-281).
// A row whose gradient is zero at a step (not visible, not anchored) evolves
// there as m <- b1 m, v <- b2 v, x <- x - lr m_hat / (sqrt(v_hat) + eps) (then
// the quaternion canonicalisation): a pure function of the row and the step's
// constants. Such rows are left untouched and replayed -- the same FP32
// operations, so bit-identical -- when they are next needed: by the
// preprocess for a culling candidate, by materialize() before any host read
// or densification, and every adam_sync (<= kAdamRing / 2) steps for all rows (the ring of
// per-step constants covers kAdamRing steps). The sparse Adam updates only
// the visible and anchored rows.
constexpr uint32_t kAdamRing = 64;
struct LazyAdam {
    float b1, b2, eps, omb1, omb2;
    float lr[kMaxD];        // lr of the components whose rate does not change (not used for positions)
    const float4* ring;
    uint32_t t;             // Adam steps applied so far (rows whose step stamp is below are stale)
    float drift_pos, drift_ls;  // per-component drift bounds per unit of the geometric staleness factor
    float rho;              // b1 / sqrt(b2): decay of |m_hat / sqrt(v_hat)| over a zero-gradient step
};

// One Adam step of one component (trainer.cpp:120-131); the sqrt and the
// division are the approximate MUFU forms (~2 ulp each on the update term,
// far below the FP32 rounding of x). Every Adam update and every lazy replay
// runs this same function, and every rounding is spelled out (explicit
// _rn intrinsics), so its bits do not depend on the file's --fmad setting:
// the replay in the preprocess (--fmad=false) and in the Adam kernels give
// the dense update's bits exactly (tests/test_gpu_lazy_adam.py).
__device__ __forceinline__ float adam_update_step(float x, float g, float& m, float& v, float lr, float b1, float omb1,
                                                  float b2, float omb2, float inv_bc1, float inv_bc2, float eps) {
    m = __fmaf_rn(b1, m, __fmul_rn(omb1, g));
    v = __fmaf_rn(b2, v, __fmul_rn(__fmul_rn(omb2, g), g));
    float sq;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(__fmul_rn(v, inv_bc2)));
    return __fmaf_rn(-lr, __fdividef(__fmul_rn(m, inv_bc1), __fadd_rn(sq, eps)), x);
}

// canonicalise (cloud.cpp:82-85): normalise, (0,0,0,0) -> (1,0,0,0), w >= 0;
// one reciprocal square root per row, the sign flip folded into the scale
__device__ __forceinline__ void canonicalize(float& qw, float& qx, float& qy, float& qz) {
    const float n2 = __fmaf_rn(qz, qz, __fmaf_rn(qy, qy, __fmaf_rn(qx, qx, __fmul_rn(qw, qw))));
    if (n2 == 0.f) {
        qw = 1.f; qx = 0.f; qy = 0.f; qz = 0.f;
    } else {
        float r;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(n2));
        const float inv = qw < 0.f ? -r : r;
        qw *= inv; qx *= inv; qy *= inv; qz *= inv;
    }
}

// Component stored in a slot of the row layout, -1 for padding (inverse of pslot).
__host__ __device__ constexpr int comp_of_slot(int s, int fd) {
    return s < 3 ? kPos + s
                 : (s < 6 ? kLs + (s - 3)
                          : (s == 6 ? kFeat + fd
                                    : (s == 7 ? -1 : (s < 12 ? kRot + (s - 8) : (s < 12 + fd ? kFeat + (s - 12) : -1)))));
}

// Replays Adam steps t0+1 .. la.t with zero gradient on sector h (slots
// 8h .. 8h+7) of a row, in registers.
template <int fd, int h>
__device__ __forceinline__ void catch_up_sector(float (&xs)[8], float (&ms)[8], float (&vs)[8], uint32_t t0,
                                                const LazyAdam& la) {
    for (uint32_t t = t0 + 1; t <= la.t; ++t) {
        const float4 k = la.ring[t % kAdamRing];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = comp_of_slot(8 * h + j, fd);
            if (c < 0) continue;
            const float lr = c < kRot ? k.z : la.lr[c];
            xs[j] = adam_update_step(xs[j], 0.f, ms[j], vs[j], lr, la.b1, la.omb1, la.b2, la.omb2, k.x, k.y, la.eps);
        }
        if (h == 1) canonicalize(xs[0], xs[1], xs[2], xs[3]);
    }
    if (h == 0) xs[kMetaSlot] = __uint_as_float(la.t);  // the row is current at la.t
}

// Sector h of row i (stale since t0) brought up to la.t in memory.
template <int fd, int h>
__device__ __forceinline__ void catch_up_sector_mem(float* __restrict__ x, float* __restrict__ m, float* __restrict__ v,
                                                    uint32_t i, uint32_t t0, const LazyAdam& la) {
    const size_t off = static_cast<size_t>(i) * row_stride(fd) + 8 * h;
    float xs[8], ms[8], vs[8];
    float4* x4 = reinterpret_cast<float4*>(x + off);
    float4* m4 = reinterpret_cast<float4*>(m + off);
    float4* v4 = reinterpret_cast<float4*>(v + off);
    const float4 xa = x4[0], xb = x4[1], ma = m4[0], mb = m4[1], va = v4[0], vb = v4[1];
    xs[0] = xa.x; xs[1] = xa.y; xs[2] = xa.z; xs[3] = xa.w; xs[4] = xb.x; xs[5] = xb.y; xs[6] = xb.z; xs[7] = xb.w;
    ms[0] = ma.x; ms[1] = ma.y; ms[2] = ma.z; ms[3] = ma.w; ms[4] = mb.x; ms[5] = mb.y; ms[6] = mb.z; ms[7] = mb.w;
    vs[0] = va.x; vs[1] = va.y; vs[2] = va.z; vs[3] = va.w; vs[4] = vb.x; vs[5] = vb.y; vs[6] = vb.z; vs[7] = vb.w;
    catch_up_sector<fd, h>(xs, ms, vs, t0, la);
    x4[0] = make_float4(xs[0], xs[1], xs[2], xs[3]);
    x4[1] = make_float4(xs[4], xs[5], xs[6], xs[7]);
    m4[0] = make_float4(ms[0], ms[1], ms[2], ms[3]);
    m4[1] = make_float4(ms[4], ms[5], ms[6], ms[7]);
    v4[0] = make_float4(vs[0], vs[1], vs[2], vs[3]);
    v4[1] = make_float4(vs[4], vs[5], vs[6], vs[7]);
}

// Brings row i (stale since t0) up to la.t in memory: x, m, v sector by sector.
template <int fd>
__device__ __forceinline__ void catch_up_row(float* __restrict__ x, float* __restrict__ m, float* __restrict__ v,
                                             uint32_t i, uint32_t t0, const LazyAdam& la) {
    constexpr int RS = row_stride(fd), H = fd <= 4 ? 2 : 3;
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const size_t off = static_cast<size_t>(i) * RS + 8 * h;
        float xs[8], ms[8], vs[8];
        float4* x4 = reinterpret_cast<float4*>(x + off);
        float4* m4 = reinterpret_cast<float4*>(m + off);
        float4* v4 = reinterpret_cast<float4*>(v + off);
        const float4 xa = x4[0], xb = x4[1], ma = m4[0], mb = m4[1], va = v4[0], vb = v4[1];
        xs[0] = xa.x; xs[1] = xa.y; xs[2] = xa.z; xs[3] = xa.w; xs[4] = xb.x; xs[5] = xb.y; xs[6] = xb.z; xs[7] = xb.w;
        ms[0] = ma.x; ms[1] = ma.y; ms[2] = ma.z; ms[3] = ma.w; ms[4] = mb.x; ms[5] = mb.y; ms[6] = mb.z; ms[7] = mb.w;
        vs[0] = va.x; vs[1] = va.y; vs[2] = va.z; vs[3] = va.w; vs[4] = vb.x; vs[5] = vb.y; vs[6] = vb.z; vs[7] = vb.w;
        if (h == 0) catch_up_sector<fd, 0>(xs, ms, vs, t0, la);
        else if (h == 1) catch_up_sector<fd, 1>(xs, ms, vs, t0, la);
        else catch_up_sector<fd, 2>(xs, ms, vs, t0, la);
        x4[0] = make_float4(xs[0], xs[1], xs[2], xs[3]);
        x4[1] = make_float4(xs[4], xs[5], xs[6], xs[7]);
        m4[0] = make_float4(ms[0], ms[1], ms[2], ms[3]);
        m4[1] = make_float4(ms[4], ms[5], ms[6], ms[7]);
        v4[0] = make_float4(vs[0], vs[1], vs[2], vs[3]);
        v4[1] = make_float4(vs[4], vs[5], vs[6], vs[7]);
    }
}
LazyAdam make_lazy_adam(const Ctx* c);
void launch_adam(Ctx* c, const DevCam& cam, const AdamStep& st, double* loss_out, int step_index);
void materialize(Ctx* c);
// Every row's step stamp (x slot kMetaSlot) set to `stamp`; with reset_stats
// the densify statistics (m, v slot kMetaSlot) zeroed.
void reset_row_meta(Ctx* c, uint32_t stamp, bool reset_stats);
void launch_finalize_loss(Ctx* c, const DevCam& cam, const DevRender& rc, double* out, bool add_penalty);
bool launch_ssim_windows(Ctx* c, const DevCam& cam, const float* gt);
// K1-K5 for one view (abi.cu), and the evaluation of one holdout view (eval.cu).
void project_and_bin_public(Ctx* c, const DevCam& cam, const DevRender& rc);
void eval_view(Ctx* c, const DevCam& cam, const DevRender& rc, const double* gt_dev, double* scratch, double out[2]);

// ---- densification (densify.cu) ----------------------------------------
// maybe_densify (trainer.cpp:301-385) after the step that made c->iteration.
void maybe_densify(Ctx* c);
// (Re)allocation of the per-row arrays for `cap` rows (x, m, v untouched).
void alloc_row_scratch(Ctx* c, size_t cap);
void install_shared_masks(Ctx* c);

// ---- consensus (consensus.cu) ------------------------------------------
void round_pack_q(Ctx* c);
void round_pack_main(Ctx* c, double alpha, bool relax);
void round_unpack(Ctx* c, double alpha, bool relax, const uint8_t* reset_slots_dev, size_t n_reset, bool diag);
void round_slots_from_sums(Ctx* c);
void round_apply_broadcast(Ctx* c, double alpha, bool relax, bool has_resets);
// adapt_penalties (admm.cpp:200-217) on the device from round_scalars; writes rho_state and rho_dev.
void round_adapt(Ctx* c, const bsg_adapt_args& a);
// rho_state / rho_dev from the host copy c->rho (stream-ordered on c->stream).
void upload_rho(Ctx* c);

// ---- the step ------------------------------------------------------------
void ensure_image_buffers(Ctx* c, int W, int H);
void ensure_pair_capacity(Ctx* c, size_t P);
void stage_begin(Ctx* c, int stage);
void stage_end(Ctx* c, int stage);

}  // namespace bsg
