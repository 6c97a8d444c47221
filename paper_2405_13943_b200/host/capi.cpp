// C entry point of the K-block driver (run_simulated over the C++ host
// layer), for hosts that bind C (Python ctypes, the bench, tests).
#include <algorithm>
#include <cstring>
#include <string>

#include "../../include/blocksplat_gpu.hpp"

namespace {
thread_local std::string g_drv_err;
}

namespace {

template <typename Decode>
int checkpoint_out(Decode&& decode, size_t cap, uint64_t* ids, double* pos, double* rot, double* ls, double* feat,
                   double* op, size_t* out_n, int* out_fd, int* format_code) {
    using namespace blocksplat;
    try {
        const SceneDataset d = decode();
        if (!d.has_checkpoint) throw InvalidArgument("container has no GSPL checkpoint");
        const GaussianCloud& c = d.checkpoint;
        const size_t n = c.size();
        const int fd = c.feature_dim();
        if (out_n) *out_n = n;
        if (out_fd) *out_fd = fd;
        if (!ids) return BSG_OK;
        if (n > cap) {
            g_drv_err = "checkpoint has more rows than the capacity";
            return BSG_ERR_CAPACITY;
        }
        std::copy(c.ids.begin(), c.ids.end(), ids);
        if (pos) std::copy(c.positions.begin(), c.positions.end(), pos);
        if (rot) std::copy(c.rotations.begin(), c.rotations.end(), rot);
        if (ls) std::copy(c.log_scales.begin(), c.log_scales.end(), ls);
        if (feat) std::copy(c.features.begin(), c.features.end(), feat);
        if (op) std::copy(c.opacity_logits.begin(), c.opacity_logits.end(), op);
        return BSG_OK;
    } catch (const FormatError& e) {
        g_drv_err = e.what();
        if (format_code) *format_code = static_cast<int>(e.code());
        return BSG_ERR_FORMAT;
    } catch (const InvalidArgument& e) {
        g_drv_err = e.what();
        return BSG_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_drv_err = e.what();
        return BSG_ERR_STATE;
    }
}
}  // namespace

extern "C" {

const char* bsg_driver_last_error(void) { return g_drv_err.c_str(); }

int bsg_view_sequence(uint64_t seed, uint32_t block_id, size_t n_views, size_t n_steps, uint32_t* out) {
    try {
        if (!out && n_steps) throw blocksplat::InvalidArgument("null output");
        const std::vector<uint32_t> seq = blocksplat::view_sequence(seed, block_id, n_views, n_steps);
        std::copy(seq.begin(), seq.end(), out);
        return BSG_OK;
    } catch (const blocksplat::InvalidArgument& e) {
        g_drv_err = e.what();
        return BSG_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_drv_err = e.what();
        return BSG_ERR_STATE;
    }
}

int bsg_run_simulated(int fd, size_t n, const uint64_t* ids, const double* pos, const double* rot, const double* ls,
                      const double* feat, const double* op, size_t n_views, const bsg_camera* cams,
                      const double* const* gts, const bsg_trainer_config* tc, const bsg_session_options* so,
                      size_t n_devices, const int* devices, size_t model_capacity, uint64_t* out_ids,
                      double* out_pos, double* out_rot, double* out_ls, double* out_feat, double* out_op,
                      size_t* out_n, bsg_round_diag* rounds, size_t max_rounds, size_t* n_rounds,
                      double* wall_seconds) {
    using namespace blocksplat;
    try {
        GaussianCloud init(fd);
        init.ids.assign(ids, ids + n);
        init.positions.assign(pos, pos + 3 * n);
        init.rotations.assign(rot, rot + 4 * n);
        init.log_scales.assign(ls, ls + 3 * n);
        init.features.assign(feat, feat + n * fd);
        init.opacity_logits.assign(op, op + n);
        std::vector<CameraView> views(n_views);
        std::vector<Image> images(n_views);
        for (size_t v = 0; v < n_views; ++v) {
            CameraView& c = views[v];
            c.view_id = v;
            c.fx = cams[v].fx; c.fy = cams[v].fy; c.cx = cams[v].cx; c.cy = cams[v].cy;
            for (int k = 0; k < 9; ++k) c.rotation[k] = cams[v].R[k];
            for (int k = 0; k < 3; ++k) c.translation[k] = cams[v].t[k];
            c.width = cams[v].width;
            c.height = cams[v].height;
            images[v] = Image(c.width, c.height);
            std::memcpy(images[v].data.data(), gts[v], images[v].data.size() * sizeof(double));
        }
        TrainerConfig t;
        t.iterations = tc->iterations;
        t.seed = so->seed;
        t.lr = LearningRates{tc->lr_position, tc->lr_position_decay, tc->lr_rotation, tc->lr_log_scale,
                             tc->lr_features, tc->lr_opacity};
        t.adam = AdamParams{tc->beta1, tc->beta2, tc->eps};
        t.render.near_plane = tc->render.near_plane;
        t.render.dilation = tc->render.dilation;
        t.render.alpha_clamp = tc->render.alpha_clamp;
        t.render.transmittance_stop = tc->render.transmittance_stop;
        t.render.sigma_extent = tc->render.sigma_extent;
        for (int k = 0; k < 3; ++k) t.render.background[k] = tc->render.background[k];
        t.render.lambda = tc->render.lambda;
        t.densify.enabled = tc->densify.enabled != 0;
        t.densify.interval = tc->densify.interval;
        t.densify.stop_iteration = tc->densify.stop_iteration;
        t.densify.grad_threshold = tc->densify.grad_threshold;
        t.densify.prune_opacity = tc->densify.prune_opacity;
        t.densify.split_scale_fraction = tc->densify.split_scale_fraction;
        t.densify.split_shrink = tc->densify.split_shrink;
        SessionOptions opt;
        opt.total_iterations = so->total_iterations;
        opt.consensus.interval = so->interval;
        opt.consensus.alpha = so->alpha;
        opt.consensus.mu = so->mu;
        opt.consensus.tau_inc = so->tau_inc;
        opt.consensus.tau_dec = so->tau_dec;
        opt.consensus.freeze_iteration = so->freeze_iteration;
        opt.consensus.adaptive = so->adaptive != 0;
        opt.consensus.enabled = so->enabled != 0;
        opt.rho = PropertyPenalties{so->rho.rho_p, so->rho.rho_q, so->rho.rho_s, so->rho.rho_f, so->rho.rho_o};
        const ClusterPlan plan = plan_cluster(init, views, images, so->blocks, so->expand_scale, so->holdout);
        std::vector<int> devs(devices, devices + n_devices);
        if (devs.empty()) devs.push_back(0);
        const RunResult r = run_simulated(plan, t, opt, {}, devs);
        const size_t nm = r.model.size();
        if (out_n) *out_n = nm;
        if (nm > model_capacity) {
            g_drv_err = "model larger than the output capacity";
            return BSG_ERR_CAPACITY;
        }
        if (out_ids) std::copy(r.model.ids.begin(), r.model.ids.end(), out_ids);
        for (size_t i = 0; i < nm; ++i) {
            for (int k = 0; k < 3; ++k) out_pos[3 * i + k] = r.model.positions[3 * i + k];
            for (int k = 0; k < 4; ++k) out_rot[4 * i + k] = r.model.rotations[4 * i + k];
            for (int k = 0; k < 3; ++k) out_ls[3 * i + k] = r.model.log_scales[3 * i + k];
            for (int k = 0; k < fd; ++k) out_feat[i * fd + k] = r.model.features[i * fd + k];
            out_op[i] = r.model.opacity_logits[i];
        }
        const size_t nr = std::min(max_rounds, r.rounds.size());
        for (size_t j = 0; j < nr; ++j) {
            const RoundDiagnostics& d = r.rounds[j];
            rounds[j].iteration = d.iteration;
            rounds[j].primal = d.primal_residual;
            rounds[j].dual = d.dual_residual;
            rounds[j].rho = bsg_penalties{d.rho.rho_p, d.rho.rho_q, d.rho.rho_s, d.rho.rho_f, d.rho.rho_o};
            rounds[j].max_disagreement = d.max_disagreement;
            rounds[j].dual_mean_linf = d.dual_mean_linf;
            rounds[j].mean_loss = d.mean_loss;
            rounds[j].shared_count = d.shared_count;
            rounds[j].global_count = d.global_count;
            rounds[j].consensus_ms = d.consensus_ms;
        }
        if (n_rounds) *n_rounds = r.rounds.size();
        if (wall_seconds) *wall_seconds = r.wall_seconds;
        return BSG_OK;
    } catch (const InvalidArgument& e) {
        g_drv_err = e.what();
        return BSG_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_drv_err = e.what();
        return BSG_ERR_STATE;
    }
}

int bsg_save_model(const char* path, int fd, size_t n, const uint64_t* ids, const double* pos, const double* rot,
                   const double* ls, const double* feat, const double* op) {
    using namespace blocksplat;
    try {
        if (!path) throw InvalidArgument("null path");
        if (fd != kFeatureDimDeg0 && fd != kFeatureDimDeg1) throw InvalidArgument("feature width must be 3 or 12");
        if (n && (!ids || !pos || !rot || !ls || !feat || !op)) throw InvalidArgument("null model array");
        GaussianCloud m(fd);
        if (n) {
            m.ids.assign(ids, ids + n);
            m.positions.assign(pos, pos + 3 * n);
            m.rotations.assign(rot, rot + 4 * n);
            m.log_scales.assign(ls, ls + 3 * n);
            m.features.assign(feat, feat + n * fd);
            m.opacity_logits.assign(op, op + n);
        }
        save_model(path, m);
        return BSG_OK;
    } catch (const InvalidArgument& e) {
        g_drv_err = e.what();
        return BSG_ERR_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_drv_err = e.what();
        return BSG_ERR_STATE;
    }
}


int bsg_load_checkpoint(const char* path, size_t cap, uint64_t* ids, double* pos, double* rot, double* ls,
                        double* feat, double* op, size_t* out_n, int* out_fd, int* format_code) {
    if (!path) {
        g_drv_err = "null path";
        return BSG_ERR_INVALID_ARGUMENT;
    }
    return checkpoint_out([&] { return blocksplat::load_scene(path); }, cap, ids, pos, rot, ls, feat, op, out_n,
                          out_fd, format_code);
}

int bsg_decode_checkpoint(const uint8_t* data, size_t size, size_t cap, uint64_t* ids, double* pos, double* rot,
                          double* ls, double* feat, double* op, size_t* out_n, int* out_fd, int* format_code) {
    if (!data && size) {
        g_drv_err = "null data";
        return BSG_ERR_INVALID_ARGUMENT;
    }
    return checkpoint_out([&] { return blocksplat::decode_scene(data, size); }, cap, ids, pos, rot, ls, feat, op,
                          out_n, out_fd, format_code);
}

}  // extern "C"
