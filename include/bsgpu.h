/*
 * bsgpu.h — C-ABI drop-in boundary for the blocksplat (DOGS) hot path on
 * NVIDIA B200 (sm_100a).
 *
 * The reference (/root/reference/proj/core) is a C++ library with no plugin
 * registry: its operator boundary is the free-function / class API in
 * renderer.hpp, admm.hpp, trainer.hpp and runtime.hpp. Each entry point below
 * names the reference interface it replaces (file:line). A host adapter that
 * keeps the reference signatures calls these (INTEGRATION.md shows it).
 *
 * Conventions
 *  - Plain pointers and sizes; no C++ or torch types. Host arrays use the
 *    reference's own layouts (GaussianCloud SoA, cloud.hpp:41-46; Image
 *    row-major interleaved RGB, image.hpp:11-25) and FP64, converted at the
 *    boundary. Device-resident parameters and Adam moments are FP32 row-major
 *    (16 floats a row at SH degree 0, 32 at degree 1).
 *  - Every call returns a status (BSG_OK = 0). On failure bsg_last_error()
 *    returns a thread-local message; BSG_ERR_INVALID_ARGUMENT maps to the
 *    reference's blocksplat::InvalidArgument, everything else to
 *    std::runtime_error (errors.hpp:33-36).
 *  - A context owns one block's state on one device (BlockTrainer is
 *    single-owner, trainer.hpp:85-87); calls on one context must come from one
 *    host thread at a time.
 *  - There is no CPU fallback: creating a context without a usable sm_100
 *    device fails with BSG_ERR_CUDA.
 */
#ifndef BSGPU_H
#define BSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSG_ABI_VERSION 1

enum bsg_status {
    BSG_OK = 0,
    BSG_ERR_INVALID_ARGUMENT = 1, /* blocksplat::InvalidArgument */
    BSG_ERR_CUDA = 2,             /* CUDA runtime / launch failure */
    BSG_ERR_NCCL = 3,             /* collective failure */
    BSG_ERR_STATE = 4,            /* call out of order (e.g. step before init) */
    BSG_ERR_CAPACITY = 5,         /* device buffer capacity exceeded */
    BSG_ERR_FORMAT = 6            /* blocksplat::FormatError (container decode); see format_code */
};

/* CameraView (camera.hpp:14-37): x_c = R x_w + t, pixel = (fx X/Z + cx, fy Y/Z + cy).
 * R is the cached row-major matrix of the stored quaternion (camera.hpp:23-26). */
typedef struct bsg_camera {
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    uint32_t width, height;
} bsg_camera;

/* RenderConfig (renderer.hpp:13-21). */
typedef struct bsg_render_config {
    double near_plane;         /* 0.01 */
    double dilation;           /* 0.3 */
    double alpha_clamp;        /* 0.99 */
    double transmittance_stop; /* 1e-4 */
    double sigma_extent;       /* 3.0 */
    double background[3];      /* 0 */
    double lambda;             /* 0.2 */
} bsg_render_config;

/* DensifyConfig (trainer.hpp:43-51) plus the BlockTrainer inputs densification
 * needs: the block id and global initial count of its IdAllocator
 * (trainer.cpp:55-66; block k hands out [k 2^48, (k+1) 2^48), block 0 starting
 * past the initial ids). The scene extent (trainer.cpp:153-154) is taken from
 * the cloud at bsg_trainer_init. */
typedef struct bsg_densify_config {
    int enabled;                  /* 1 */
    uint32_t interval;            /* 200 */
    uint64_t stop_iteration;      /* 0 resolves to 60% of iterations */
    double grad_threshold;        /* 2e-4, mean screen-space gradient norm */
    double prune_opacity;         /* 0.005 */
    double split_scale_fraction;  /* 0.01 of the scene extent: clone below, split above */
    double split_shrink;          /* 1.6 */
    uint32_t block_id;            /* 0 */
    uint64_t global_initial_count;/* 0: the uploaded cloud's size */
} bsg_densify_config;

/* TrainerConfig device subset (trainer.hpp:13-62). */
typedef struct bsg_trainer_config {
    uint64_t iterations;
    double lr_position, lr_position_decay, lr_rotation, lr_log_scale, lr_features, lr_opacity;
    double beta1, beta2, eps;
    bsg_render_config render;
    bsg_densify_config densify;
} bsg_trainer_config;

/* PropertyPenalties (admm.hpp:12-18). */
typedef struct bsg_penalties {
    double rho_p, rho_q, rho_s, rho_f, rho_o;
} bsg_penalties;

typedef struct bsg_ctx bsg_ctx;

/* ---- lifecycle ------------------------------------------------------- */
int bsg_abi_version(void);
const char* bsg_last_error(void);
/* Fills the defaults of renderer.hpp:13-21 / trainer.hpp:13-62 / admm.hpp:12-18. */
void bsg_default_render_config(bsg_render_config* out);
void bsg_default_trainer_config(bsg_trainer_config* out);
void bsg_default_penalties(bsg_penalties* out);
int bsg_create(int device, int feature_dim, bsg_ctx** out);
int bsg_destroy(bsg_ctx* ctx);

/* ---- parameters (GaussianCloud, cloud.hpp:32-102) ---------------------- */
/* Uploads n rows (ids strictly ascending, cloud.cpp:66-74) in the reference
 * FP64 layout: pos 3n, rot 4n (w,x,y,z), log_scale 3n, features fd*n, opacity
 * logits n. Resets optimizer moments and densify statistics. */
int bsg_upload_cloud(bsg_ctx* ctx, size_t n, const uint64_t* ids, const double* pos, const double* rot,
                     const double* log_scale, const double* features, const double* opacity_logit);
size_t bsg_cloud_size(const bsg_ctx* ctx);
int bsg_download_cloud(bsg_ctx* ctx, uint64_t* ids, double* pos, double* rot, double* log_scale, double* features,
                       double* opacity_logit);
/* GSPL checkpoint payload of the context's cloud (scene_io.cpp:48-59): u64
 * count, u32 feature width, u64 ids, then f32 positions 3n, rotations 4n,
 * log-scales 3n, features fd*n, opacity logits n, little-endian. Encoded on
 * the device from the FP32 parameters (narrow_to_f32, scene_io.cpp:230-241,
 * is the identity on them). out == NULL: *out_len receives the byte size;
 * otherwise out_cap must be at least that (BSG_ERR_CAPACITY). */
int bsg_encode_gspl(bsg_ctx* ctx, uint8_t* out, size_t out_cap, size_t* out_len);

/* ---- rendering (renderer.hpp:71-81) ---------------------------------- */
/* render(): out_rgb HxWx3, out_transmittance HxW, out_contributors HxW (any may be NULL). */
int bsg_render(bsg_ctx* ctx, const bsg_camera* cam, const bsg_render_config* cfg, double* out_rgb,
               double* out_transmittance, uint32_t* out_contributors);
/* render_backward(): gt HxWx3. out_loss3 = {loss, l1, ssim}. Gradient arrays
 * have the cloud layouts (culled rows are exactly 0); screen_grad_norm n,
 * visible n. out_rendered (HxWx3) may be NULL. */
int bsg_render_backward(bsg_ctx* ctx, const bsg_camera* cam, const double* gt_rgb, const bsg_render_config* cfg,
                        double* out_loss3, double* g_pos, double* g_rot, double* g_log_scale, double* g_features,
                        double* g_opacity_logit, double* screen_grad_norm, uint8_t* visible, double* out_rendered);

/* The loss and its image gradient of the training step on given images:
 * loss_value (renderer.cpp:185-192) and dL/dC = sign(C - GT) / (3HW) -
 * lambda dSSIM/dC (renderer.cpp:259-272, ssim_with_gradient ssim.cpp:138-185),
 * through the step's own SSIM kernels. rendered, gt: HxWx3; out_loss3 =
 * {loss, l1, ssim}; out_dl_dc HxWx3 (both nullable). */
int bsg_image_loss(bsg_ctx* ctx, uint32_t width, uint32_t height, const double* rendered, const double* gt,
                   const bsg_render_config* cfg, double* out_loss3, double* out_dl_dc);

/* ---- projection / sort introspection (parity of the integer paths) --- */
/* Per row: visible flag, FP64 depth, footprint rect {x0,x1,y0,y1}; and the
 * compositing order (rows of visible splats sorted by (depth, index),
 * renderer.cpp:86-89). out_order must hold n entries; *out_visible_count is V. */
int bsg_project(bsg_ctx* ctx, const bsg_camera* cam, const bsg_render_config* cfg, uint8_t* out_visible,
                double* out_depth, int32_t* out_rect, uint32_t* out_order, size_t* out_visible_count);
/* Tile lists after the tile-key sort: for the last projected camera, the
 * (tile, row) pairs in sorted order. Pass NULL arrays to query *out_pairs. */
int bsg_tile_pairs(bsg_ctx* ctx, uint32_t* out_tile, uint32_t* out_row, size_t capacity, size_t* out_pairs);

/* ---- training (BlockTrainer, trainer.hpp:88-149) ---------------------- */
/* Installs the training views (TrainView, trainer.hpp:80-83): cameras and
 * ground-truth images (HxWx3 FP64 each), kept resident in HBM as FP32. */
int bsg_set_views(bsg_ctx* ctx, size_t n_views, const bsg_camera* cams, const double* const* gt_rgb);
int bsg_trainer_init(bsg_ctx* ctx, const bsg_trainer_config* cfg);
/* n train_step()s (trainer.cpp:249-295) on resident views view_seq[0..n).
 * losses (n, nullable) receives render loss + penalty per step. */
int bsg_train_steps(bsg_ctx* ctx, size_t n, const uint32_t* view_seq, double* losses);
/* One train_step() whose ground truth comes from host memory (HxWx3 FP32,
 * pinned or pageable); the copy is part of the step (end-to-end path). */
int bsg_train_step_host(bsg_ctx* ctx, const bsg_camera* cam, const float* gt_rgb_host, double* loss);
/* n steps on host ground-truth images (BlockTrainer::run_iterations over
 * host-resident views, trainer.hpp:100-104): step k trains on cams[k] against
 * gts_host[k] (HxWx3 FP32, pinned for full overlap). Each image is copied on
 * a copy stream into one of two device buffers while the previous step
 * computes; losses[k] (nullable) receives step k's loss (one read-back of all
 * n at the end of the call). */
int bsg_train_steps_host(bsg_ctx* ctx, size_t n, const bsg_camera* cams, const float* const* gts_host,
                         double* losses);
/* As bsg_train_steps_host with 8-bit RGB images (HxWx3 bytes: the PPM data
 * the reference loads, image.cpp:60-79), widened on the device as
 * dequantize does (byte / 255, image.cpp:21-27): a quarter of the upload. */
int bsg_train_steps_host_u8(bsg_ctx* ctx, size_t n, const bsg_camera* cams, const uint8_t* const* gts_host,
                            double* losses);
uint64_t bsg_iteration(const bsg_ctx* ctx);
/* Optimizer moments, [D][n] component-major FP64 (D = 11 + fd), for parity. */
int bsg_download_moments(bsg_ctx* ctx, double* m, double* v);
/* Restores optimizer state (resume; the inverse of bsg_download_moments):
 * moments [D][n] (v >= 0, finite) and the Adam step count t of
 * OptimizerState (trainer.cpp:267) the bias corrections continue from. Call
 * after bsg_trainer_init (which resets them). */
int bsg_upload_moments(bsg_ctx* ctx, const double* m, const double* v, uint64_t adam_step);
/* Lazy Adam: a row with no gradient and no penalty this step is not touched;
 * the zero-gradient steps it skipped are replayed (the same FP32 operations,
 * bit for bit) when it next becomes a projection candidate, before any host
 * read, and for every row every `every` steps (1..32; default 16). 1 = the
 * reference's dense update (trainer.cpp:120-131) applied to every row every
 * step. The results do not depend on it; only the cost does. */
int bsg_set_adam_sync_interval(bsg_ctx* ctx, uint32_t every);
/* Densify statistics (trainer.cpp:284-289): grad_accum n, grad_seen n. */
int bsg_download_densify_stats(bsg_ctx* ctx, double* grad_accum, uint32_t* grad_seen);
/* take_removed_ids / take_new_rows (trainer.hpp:137-140): ids removed by
 * densification since the last call (pruned rows and split parents, in
 * removal order), and ids of rows it added that are still in the cloud
 * (ascending); both lists are cleared. Query sizes with a null output. */
int bsg_take_removed_ids(bsg_ctx* ctx, uint64_t* out, size_t capacity, size_t* n);
int bsg_take_new_ids(bsg_ctx* ctx, uint64_t* out, size_t capacity, size_t* n);
/* Shared ids of this block after densification pruned some (ascending). */
int bsg_shared_ids(bsg_ctx* ctx, uint64_t* out, size_t capacity, size_t* n);

/* evaluate (metrics.cpp:28-51) of the uploaded cloud: renders every view with
 * index % holdout_modulus == 0 (0: every view) and scores it against gt[i]
 * (HxWx3 FP64, reference Image layout): PSNR = min(99, 10 log10(1 / mse))
 * over all channels from an FP64 squared error (metrics.cpp:14-26), and mean
 * SSIM (ssim.cpp). per_view_* (nullable, capacity n_views) receive the scored
 * views in order; BSG_ERR_INVALID_ARGUMENT "empty holdout" when none qualifies. */
int bsg_evaluate(bsg_ctx* ctx, size_t n_views, const bsg_camera* cams, const double* const* gt,
                 uint32_t holdout_modulus, const bsg_render_config* cfg, double* per_view_psnr, double* per_view_ssim,
                 size_t* n_scored, double* mean_psnr, double* mean_ssim);

/* ---- consensus (admm.hpp:47-89, trainer.cpp:161-223, runtime.cpp:482-611) */
/* Shared rows of this block: anchor j is cloud row rows[j] (ascending ids),
 * consensus slot slots[j] in [0, n_slots). slot_owners[s] = number of blocks
 * owning slot s; first_owner[j] = 1 if this block is the lowest owner of
 * slots[j] (admm.cpp:56-67 visits owners in ascending block id). */
int bsg_set_shared(bsg_ctx* ctx, size_t n_shared, const uint32_t* rows, const uint32_t* slots,
                   const uint8_t* first_owner, size_t n_slots, const uint32_t* slot_owners);
/* set_anchor (trainer.cpp:161-166): z for this block's shared rows (n_shared
 * x D, reference row layout), duals := 0, and z_prev for every slot
 * (n_slots x D) as the master's z_prev (runtime.cpp:465). */
int bsg_set_anchor(bsg_ctx* ctx, const double* z_rows, const double* z_prev_slots, const bsg_penalties* rho);
int bsg_set_penalties(bsg_ctx* ctx, const bsg_penalties* rho);
int bsg_download_duals(bsg_ctx* ctx, double* u_rows);
int bsg_download_anchor(bsg_ctx* ctx, double* z_rows);
/* Restores duals (n_shared x D rows), e.g. after the shared set shrinks. */
int bsg_upload_duals(bsg_ctx* ctx, const double* u_rows);
/* apply_broadcast (trainer.cpp:168-223) with a z computed elsewhere (e.g. a
 * master process, runtime.cpp:567-570): z_slots is n_slots x D rows; the
 * relaxed local x_hat uses the current anchor, u += x_hat - z, listed slots are
 * reset, anchor := z. */
int bsg_apply_broadcast(bsg_ctx* ctx, const double* z_slots, size_t n_reset, const uint32_t* reset_slots, double alpha,
                        int relax);
/* Consensus z over all slots (n_slots x D) after the last round. */
int bsg_download_consensus(bsg_ctx* ctx, double* z_slots);

typedef struct bsg_round_args {
    double alpha;          /* over-relaxation (admm.hpp:25) */
    int relax;             /* enabled && alpha != 1 && !final (runtime.cpp:530) */
    size_t n_reset;        /* extra reset slots from ownership edits (runtime.cpp:506-512) */
    const uint32_t* reset_slots;
    int diagnostics;       /* also compute max_disagreement and dual-mean L-inf */
} bsg_round_args;

typedef struct bsg_round_result {
    double primal;          /* admm.cpp:147-198 */
    double dual;
    double max_disagreement;/* admm.cpp:219-243 (diagnostics only) */
    double dual_mean_linf;  /* runtime.cpp:572-606 (diagnostics only) */
    uint64_t flipped;       /* slots whose quaternion needed a sign flip */
    double ms;              /* device time of the round on this block */
} bsg_round_result;

/* Multi-process / multi-GPU collective (one rank per block, NCCL over NVLink). */
int bsg_nccl_unique_id(uint8_t out_id[128]);
int bsg_comm_init(bsg_ctx* ctx, const uint8_t id[128], int nranks, int rank);
int bsg_consensus_round(bsg_ctx* ctx, const bsg_round_args* args, bsg_round_result* out);

/* Penalty adaptation (adapt_penalties, admm.cpp:200-217) applied on the device
 * at the end of an asynchronous round: `iteration` is the round's iteration t. */
typedef struct bsg_adapt_args {
    double mu, tau_inc, tau_dec;   /* ConsensusConfig (admm.hpp:20-29) */
    uint64_t freeze_iteration;
    int adaptive;
    uint64_t iteration;
} bsg_adapt_args;

/* One process driving k contexts on k distinct devices (run_simulated with
 * one GPU per block): one NCCL communicator per context, initialised as a
 * group (ncclGroupStart / CommInitRank x k / GroupEnd); rank = position. */
int bsg_comm_init_local(bsg_ctx* const* ctxs, size_t k);
/* Host communicator: the round's all-reduces go through pinned host memory
 * and fn (in place on buf: count elements, dtype 0 = f32 / 1 = f64, op 0 =
 * sum / 1 = max; nonzero return = failure -> BSG_ERR_NCCL). For ranks that
 * cannot share an NCCL communicator (several blocks on one GPU, the
 * in-process threaded driver; processes joined by another transport, e.g. a
 * gloo group in tests). A round on a host communicator blocks its caller
 * until the reductions are done; the unpack still runs on the comm stream. */
typedef int (*bsg_host_allreduce)(void* user, void* buf, size_t count, int dtype, int op);
int bsg_comm_init_host(bsg_ctx* ctx, bsg_host_allreduce fn, void* user, int nranks, int rank);
/* Round watchdog: bsg_consensus_wait gives up after `seconds` (0 = never,
 * the default) and checks the NCCL communicator for asynchronous errors while
 * it waits; either aborts the communicator and returns BSG_ERR_NCCL (the
 * reference's per-message timeouts, runtime.cpp:44-53,98-119). */
int bsg_set_round_timeout(bsg_ctx* ctx, double seconds);

/* Asynchronous round (the overlap of SURVEY §8(e)): enqueued on the block's
 * communication stream behind the last parameter update, returns at once.
 * The next bsg_train_steps runs projection, sorting, both blends and the fold
 * while the round's reductions are in flight; only its penalty + Adam waits
 * for the round, and reads the (possibly adapted) rho from device memory, so
 * the exact iteration order of Alg. 2 is kept with no host round trip.
 * adapt (nullable): adapt rho on the device from the reduced residuals (every
 * rank decides on identical reduced values). Collective: all ranks call it in
 * the same order. bsg_consensus_wait blocks for the pending round and returns
 * its result and the rho now in force (rho_out nullable). The pending round
 * must be waited for before the next one is started. A bsg_train_steps that
 * crosses a densification iteration while a round is pending blocks for the
 * round before densifying (densification rewrites the anchor and dual rows
 * the round writes); the round's result stays pending for bsg_consensus_wait. */
int bsg_consensus_round_async(bsg_ctx* ctx, const bsg_round_args* args, const bsg_adapt_args* adapt);
int bsg_consensus_wait(bsg_ctx* ctx, bsg_round_result* out, bsg_penalties* rho_out);

/* Single-process group: k contexts (any devices) reduced in ascending block
 * order without NCCL; runs one round for all of them. */
int bsg_group_consensus_round(bsg_ctx* const* ctxs, size_t k, const bsg_round_args* args, bsg_round_result* out);

/* ---- block planner (host, splitter.cpp:48-201; runtime.cpp:265-305) ---
 * Recursive median bipartition along the longer ground axis into k cells,
 * expansion by `scale` about each cell centre on the ground axes (vertical
 * axis spans everything), closed-box assignment with nearest-box fallback.
 * The points are the Gaussian positions (plan_cluster). Shared ids (two or
 * more owners) get consensus slots in ascending id order. Host-only: no GPU. */
typedef struct bsg_plan bsg_plan;
const char* bsg_plan_last_error(void);
int bsg_plan_create(size_t n, const uint64_t* ids, const double* pos, size_t n_views, const double* view_centers,
                    uint32_t k, double scale, int vertical_axis, int midpoint_plane, bsg_plan** out);
void bsg_plan_destroy(bsg_plan* plan);
int bsg_plan_block_sizes(const bsg_plan* plan, uint32_t block, size_t* n_gaussians, size_t* n_views);
int bsg_plan_block(const bsg_plan* plan, uint32_t block, uint64_t* ids, uint32_t* views);
int bsg_plan_boxes(const bsg_plan* plan, double* core_min, double* core_max, double* exp_min, double* exp_max);
size_t bsg_plan_shared_count(const bsg_plan* plan);
int bsg_plan_shared(const bsg_plan* plan, uint64_t* ids, uint32_t* owner_count, uint32_t* first_owner);
int bsg_plan_block_shared(const bsg_plan* plan, uint32_t block, size_t* n_out, uint32_t* rows, uint32_t* slots,
                          uint8_t* first_owner);

/* ---- K-block driver (run_simulated, runtime.cpp:623-671) --------------- */
/* plan_cluster + BlockTrainers + consensus rounds, implemented by the C++
 * host layer (include/blocksplat_gpu.hpp) in this library. */
typedef struct bsg_session_options {
    uint64_t total_iterations;  /* SessionOptions::total_iterations */
    uint32_t interval;          /* ConsensusConfig (admm.hpp:20-29) */
    double alpha, mu, tau_inc, tau_dec;
    uint64_t freeze_iteration;
    int adaptive, enabled;
    bsg_penalties rho;
    uint64_t seed;              /* TrainerConfig::seed */
    uint32_t blocks;            /* plan_cluster arguments (runtime.hpp:101-103) */
    double expand_scale;
    uint32_t holdout;
} bsg_session_options;

typedef struct bsg_round_diag {  /* RoundDiagnostics (runtime.hpp:61-71) */
    uint64_t iteration;
    double primal, dual;
    bsg_penalties rho;
    double max_disagreement, dual_mean_linf, mean_loss;
    uint64_t shared_count, global_count;
    double consensus_ms;
} bsg_round_diag;

const char* bsg_driver_last_error(void);
/* The view sequence of BlockTrainer::train_step (trainer.cpp:116-118,250-252)
 * for seed / block id: the host trainer's own Fisher-Yates code path
 * (errors via bsg_driver_last_error). */
int bsg_view_sequence(uint64_t seed, uint32_t block_id, size_t n_views, size_t n_steps, uint32_t* out);
int bsg_run_simulated(int feature_dim, size_t n, const uint64_t* ids, const double* pos, const double* rot,
                      const double* log_scale, const double* features, const double* opacity_logit, size_t n_views,
                      const bsg_camera* cams, const double* const* gt_rgb, const bsg_trainer_config* trainer,
                      const bsg_session_options* session, size_t n_devices, const int* devices,
                      size_t model_capacity, uint64_t* out_ids, double* out_pos, double* out_rot,
                      double* out_log_scale, double* out_features, double* out_opacity_logit, size_t* out_n,
                      bsg_round_diag* rounds, size_t max_rounds, size_t* n_rounds, double* wall_seconds);
/* The out_* arrays hold up to model_capacity rows of the assembled model
 * (densification changes its size; *out_n receives it, BSG_ERR_CAPACITY when
 * it exceeds the capacity). */

/* ---- checkpoint files (DOGS container, scene_io.cpp) ------------------- */
/* model.dogs (main.cpp:353-357): a DOGS v1 container with empty CAMS / PNTS
 * sections and the GSPL section of the f32-narrowed model. */
int bsg_save_model(const char* path, int feature_dim, size_t n, const uint64_t* ids, const double* pos,
                   const double* rot, const double* log_scale, const double* features, const double* opacity_logit);
/* The GSPL checkpoint of a DOGS container file (the plan_cluster checkpoint
 * path, runtime.cpp:273-275). ids == NULL: only *out_n and *out_fd. On a
 * decode error returns BSG_ERR_FORMAT with *format_code = the
 * FormatErrorCode (errors.hpp:10-19, 0 = BadMagic ... 7 = BadHeader);
 * a container without a checkpoint gives BSG_ERR_INVALID_ARGUMENT. */
int bsg_load_checkpoint(const char* path, size_t capacity, uint64_t* ids, double* pos, double* rot,
                        double* log_scale, double* features, double* opacity_logit, size_t* out_n, int* out_fd,
                        int* format_code);
/* Same, from bytes in memory (decode_scene, scene_io.cpp:134-176). */
int bsg_decode_checkpoint(const uint8_t* data, size_t size, size_t capacity, uint64_t* ids, double* pos,
                          double* rot, double* log_scale, double* features, double* opacity_logit, size_t* out_n,
                          int* out_fd, int* format_code);

/* ---- checked build ------------------------------------------------------ */
/* 1 in lib/libbsgpu_checked.so (device invariant checks compiled in), else 0. */
int bsg_checked_build(void);
/* Launches one kernel whose check fails on purpose: BSG_ERR_CUDA (and a
 * corrupted CUDA context -- run it in a throwaway process) in the checked
 * build, BSG_OK otherwise. Proves the checks are live. */
int bsg_checked_probe(int device);

/* ---- master-round ownership bookkeeping (device) ------------------------ */
/* The owner table of the consensus slot table on one device (
 * replaces the master's std::map of owners, runtime.cpp:490-518): n_slots
 * shared ids (ascending) with a bitmask of their owning blocks (K <= 32,
 * >= 2 bits set). Non-shared ids never enter it: they have one owner, so a
 * removal kills them, and new rows are born single-owner. */
typedef struct bsg_owner_table bsg_owner_table;
int bsg_owners_create(int device, size_t n_slots, const uint64_t* slot_ids, const uint32_t* owner_masks,
                      uint32_t blocks, bsg_owner_table** out);
int bsg_owners_destroy(bsg_owner_table* t);
size_t bsg_owners_size(const bsg_owner_table* t);
/* Current table (n = bsg_owners_size): ids ascending, owner masks. */
int bsg_owners_download(const bsg_owner_table* t, uint64_t* slot_ids, uint32_t* owner_masks);
/* One round's removals: removed[b] (n_removed[b] ids) taken from block b.
 * Clears the owners, classifies every touched slot (1 reset: >= 2 owners
 * remain; 2 unshared: one remains; 3 dead: none) and drops the slots left
 * with fewer than 2 owners from the table. Writes the touched slots in
 * ascending order -- their index in the table before this call, class and
 * new owner mask -- (capacity cap; BSG_ERR_CAPACITY with *out_touched set
 * when too small, the table unchanged) and, per removed id in block order,
 * whether it was in the table (found; nullable). */
int bsg_owners_remove(bsg_owner_table* t, const uint64_t* const* removed, const size_t* n_removed,
                      uint32_t* out_slot, uint8_t* out_class, uint32_t* out_mask, size_t cap, size_t* out_touched,
                      uint8_t* out_found);

/* ---- measurement ------------------------------------------------------ */
/* Per-stage device times of the most recent step (CUDA events on the
 * context's stream), milliseconds, in the order of bsg_stage_name(i). */
int bsg_enable_stage_timing(bsg_ctx* ctx, int enable);
int bsg_stage_count(void);
const char* bsg_stage_name(int i);
int bsg_stage_times(bsg_ctx* ctx, double* ms);
/* Counters of the most recent step: visible splats V, tile pairs P, kernels launched. */
int bsg_step_counters(bsg_ctx* ctx, uint64_t* visible, uint64_t* pairs, uint64_t* launches);
/* (pixel, contributor) pairs the forward blend composited in the last step
 * (read only while stage timing is enabled; the FP32 work measure of the
 * blend rooflines). */
uint64_t bsg_step_blend_evals(const bsg_ctx* ctx);
/* Binning path of the most recent projection: 0 = per-tile shared-memory
 * sort (every tile <= 2048 pairs), 1 = global depth sort + stable tile-key
 * sort (bsg_project, or a view with a longer tile). Both give the order of
 * renderer.cpp:86-117; the parity tests assert which one they exercised. */
int bsg_last_binning(const bsg_ctx* ctx);
/* Kernel launches since context creation (all entry points). */
uint64_t bsg_launch_count(const bsg_ctx* ctx);
/* Opaque cudaStream_t of the context (for event timing by the caller). */
void* bsg_stream(bsg_ctx* ctx);
int bsg_synchronize(bsg_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* BSGPU_H */
