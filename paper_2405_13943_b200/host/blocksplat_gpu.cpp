// C++ host layer (include/blocksplat_gpu.hpp): the reference's blocksplat API
// (renderer.hpp, trainer.hpp, runtime.hpp) implemented over the C-ABI in
// bsgpu.h. Host bookkeeping only; every FLOP of the hot path runs in
// libbsgpu's sm_100a kernels.
#include "../../include/blocksplat_gpu.hpp"

#include <algorithm>
#include <cstring>
#include <mutex>
#include <condition_variable>
#include <chrono>
#include <cmath>
#include <exception>
#include <memory>
#include <random>
#include <set>
#include <thread>

namespace blocksplat {

namespace {

void check(int status) {
    if (status == BSG_OK) return;
    const std::string msg = bsg_last_error();
    if (status == BSG_ERR_INVALID_ARGUMENT) throw InvalidArgument(msg);
    throw std::runtime_error(msg);
}

bsg_camera to_dev(const CameraView& c) {
    bsg_camera d{};
    d.fx = c.fx; d.fy = c.fy; d.cx = c.cx; d.cy = c.cy;
    for (int k = 0; k < 9; ++k) d.R[k] = c.rotation[k];
    for (int k = 0; k < 3; ++k) d.t[k] = c.translation[k];
    d.width = c.width;
    d.height = c.height;
    return d;
}

bsg_render_config to_dev(const RenderConfig& r) {
    bsg_render_config d{};
    d.near_plane = r.near_plane;
    d.dilation = r.dilation;
    d.alpha_clamp = r.alpha_clamp;
    d.transmittance_stop = r.transmittance_stop;
    d.sigma_extent = r.sigma_extent;
    for (int k = 0; k < 3; ++k) d.background[k] = r.background[k];
    d.lambda = r.lambda;
    return d;
}

bsg_penalties to_dev(const PropertyPenalties& p) { return bsg_penalties{p.rho_p, p.rho_q, p.rho_s, p.rho_f, p.rho_o}; }

bsg_trainer_config to_dev(const TrainerConfig& t) {
    bsg_trainer_config d{};
    d.iterations = t.iterations;
    d.lr_position = t.lr.position;
    d.lr_position_decay = t.lr.position_decay;
    d.lr_rotation = t.lr.rotation;
    d.lr_log_scale = t.lr.log_scale;
    d.lr_features = t.lr.features;
    d.lr_opacity = t.lr.opacity;
    d.beta1 = t.adam.beta1;
    d.beta2 = t.adam.beta2;
    d.eps = t.adam.eps;
    d.render = to_dev(t.render);
    d.densify.enabled = t.densify.enabled ? 1 : 0;  // trainer.hpp:43-51
    d.densify.interval = t.densify.interval;
    d.densify.stop_iteration = t.densify.stop_iteration;
    d.densify.grad_threshold = t.densify.grad_threshold;
    d.densify.prune_opacity = t.densify.prune_opacity;
    d.densify.split_scale_fraction = t.densify.split_scale_fraction;
    d.densify.split_shrink = t.densify.split_shrink;
    return d;
}

void upload(bsg_ctx* ctx, const GaussianCloud& c) {
    check(bsg_upload_cloud(ctx, c.size(), c.ids.data(), c.positions.data(), c.rotations.data(), c.log_scales.data(),
                           c.features.data(), c.opacity_logits.data()));
}

GaussianCloud download(bsg_ctx* ctx, int fd) {
    GaussianCloud c(fd);
    const size_t n = bsg_cloud_size(ctx);
    c.ids.resize(n);
    c.positions.resize(3 * n);
    c.rotations.resize(4 * n);
    c.log_scales.resize(3 * n);
    c.features.resize(n * fd);
    c.opacity_logits.resize(n);
    check(bsg_download_cloud(ctx, c.ids.data(), c.positions.data(), c.rotations.data(), c.log_scales.data(),
                             c.features.data(), c.opacity_logits.data()));
    return c;
}

// D-wide rows in the bundle order pos3 rot4 ls3 feat op1.
std::vector<double> rows_of(const GaussianCloud& c, const std::vector<size_t>& idx) {
    const int fd = c.feature_dim(), D = 11 + fd;
    std::vector<double> out(idx.size() * D);
    for (size_t j = 0; j < idx.size(); ++j) {
        const size_t i = idx[j];
        double* r = &out[j * D];
        for (int k = 0; k < 3; ++k) r[k] = c.positions[3 * i + k];
        for (int k = 0; k < 4; ++k) r[3 + k] = c.rotations[4 * i + k];
        for (int k = 0; k < 3; ++k) r[7 + k] = c.log_scales[3 * i + k];
        for (int k = 0; k < fd; ++k) r[10 + k] = c.features[i * fd + k];
        r[10 + fd] = c.opacity_logits[i];
    }
    return out;
}

GaussianCloud bundle_of(const std::vector<uint64_t>& ids, const std::vector<double>& rows, int fd) {
    const int D = 11 + fd;
    GaussianCloud c(fd);
    c.ids = ids;
    for (size_t j = 0; j < ids.size(); ++j) {
        const double* r = &rows[j * D];
        c.positions.insert(c.positions.end(), r, r + 3);
        c.rotations.insert(c.rotations.end(), r + 3, r + 7);
        c.log_scales.insert(c.log_scales.end(), r + 7, r + 10);
        c.features.insert(c.features.end(), r + 10, r + 10 + fd);
        c.opacity_logits.push_back(r[10 + fd]);
    }
    return c;
}

std::vector<size_t> find_all(const GaussianCloud& c, const std::vector<uint64_t>& ids, const char* what) {
    std::vector<size_t> idx(ids.size());
    for (size_t j = 0; j < ids.size(); ++j) {
        idx[j] = c.find(ids[j]);
        if (idx[j] == GaussianCloud::npos) throw InvalidArgument(what);
    }
    return idx;
}

// math.hpp:88-97,123-129: mt19937_64 + rejection uniform_index + Fisher-Yates.
uint64_t uniform_index(std::mt19937_64& g, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v;
    do {
        v = g();
    } while (v >= limit);
    return v % n;
}

// trainer.cpp:250-252: a fresh Fisher-Yates shuffle of the view order at the
// start of every pass, then the views in that order.
void draw_views(std::mt19937_64& g, std::vector<size_t>& order, size_t& cursor, uint32_t* seq, uint64_t n) {
    for (uint64_t s = 0; s < n; ++s) {
        if (cursor == 0)
            for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[uniform_index(g, i)]);
        seq[s] = static_cast<uint32_t>(order[cursor]);
        cursor = (cursor + 1) % order.size();
    }
}

// derive_seed (trainer.cpp:116-118)
uint64_t derive_seed(uint64_t seed, uint32_t block_id) {
    return seed ^ (0x9e3779b97f4a7c15ull * (static_cast<uint64_t>(block_id) + 1));
}

Mat3 quat_to_rotation(const Vec4& q) {  // math.hpp:37-44
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    return {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
            2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
            2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
}

struct CtxCache {
    std::map<std::pair<int, int>, bsg_ctx*> ctxs;
    ~CtxCache() {
        for (auto& kv : ctxs) bsg_destroy(kv.second);
    }
    bsg_ctx* get(int device, int fd) {
        auto& c = ctxs[{device, fd}];
        if (!c) check(bsg_create(device, fd, &c));
        return c;
    }
};
thread_local CtxCache t_ctx;

}  // namespace

// ------------------------------------------------------------ cloud / camera
size_t GaussianCloud::find(uint64_t id) const {
    auto it = std::lower_bound(ids.begin(), ids.end(), id);
    if (it == ids.end() || *it != id) return npos;
    return static_cast<size_t>(it - ids.begin());
}

bool GaussianCloud::check_invariants() const {
    const size_t n = ids.size();
    if (positions.size() != 3 * n || rotations.size() != 4 * n || log_scales.size() != 3 * n ||
        features.size() != n * static_cast<size_t>(feature_dim_) || opacity_logits.size() != n)
        return false;
    for (size_t i = 1; i < n; ++i)
        if (ids[i] <= ids[i - 1]) return false;
    return true;
}

GaussianCloud slice_by_ids(const GaussianCloud& cloud, const std::vector<uint64_t>& ids) {
    std::vector<size_t> idx;
    std::vector<uint64_t> kept;
    for (uint64_t id : ids) {
        const size_t i = cloud.find(id);
        if (i != GaussianCloud::npos) {
            idx.push_back(i);
            kept.push_back(id);
        }
    }
    return bundle_of(kept, rows_of(cloud, idx), cloud.feature_dim());
}

void CameraView::set_rotation_quat(const Vec4& q) {
    rotation_q = q;
    rotation = quat_to_rotation(q);
}

Vec3 CameraView::center() const {  // camera.hpp:31
    Vec3 c;
    for (int i = 0; i < 3; ++i)
        c[i] = -((rotation[i] * translation[0] + rotation[3 + i] * translation[1]) + rotation[6 + i] * translation[2]);
    return c;
}

CameraView look_at(const Vec3& position, const Vec3& target, const Vec3& world_up, double fx, double fy, double cx,
                   double cy, uint32_t width, uint32_t height) {  // camera.hpp:42-58, math.hpp:48-69
    auto norm = [](const Vec3& v) {
        const double n = std::sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
        return Vec3{v[0] / n, v[1] / n, v[2] / n};
    };
    auto cross = [](const Vec3& a, const Vec3& b) {
        return Vec3{a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    };
    const Vec3 forward = norm(Vec3{target[0] - position[0], target[1] - position[1], target[2] - position[2]});
    const Vec3 right = norm(cross(forward, world_up));
    const Vec3 down = cross(forward, right);
    const double r[9] = {right[0], right[1], right[2], down[0], down[1], down[2], forward[0], forward[1], forward[2]};
    auto R = [&](int i, int j) { return r[3 * i + j]; };
    const double t = (R(0, 0) + R(1, 1)) + R(2, 2);
    Vec4 q;
    if (t > 0.0) {
        const double s = std::sqrt(t + 1.0) * 2.0;
        q = {0.25 * s, (R(2, 1) - R(1, 2)) / s, (R(0, 2) - R(2, 0)) / s, (R(1, 0) - R(0, 1)) / s};
    } else if (R(0, 0) > R(1, 1) && R(0, 0) > R(2, 2)) {
        const double s = std::sqrt(1.0 + R(0, 0) - R(1, 1) - R(2, 2)) * 2.0;
        q = {(R(2, 1) - R(1, 2)) / s, 0.25 * s, (R(0, 1) + R(1, 0)) / s, (R(0, 2) + R(2, 0)) / s};
    } else if (R(1, 1) > R(2, 2)) {
        const double s = std::sqrt(1.0 + R(1, 1) - R(0, 0) - R(2, 2)) * 2.0;
        q = {(R(0, 2) - R(2, 0)) / s, (R(0, 1) + R(1, 0)) / s, 0.25 * s, (R(1, 2) + R(2, 1)) / s};
    } else {
        const double s = std::sqrt(1.0 + R(2, 2) - R(0, 0) - R(1, 1)) * 2.0;
        q = {(R(1, 0) - R(0, 1)) / s, (R(0, 2) + R(2, 0)) / s, (R(1, 2) + R(2, 1)) / s, 0.25 * s};
    }
    const double n = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    if (n == 0.0) q = {1, 0, 0, 0};
    else q = {q[0] / n, q[1] / n, q[2] / n, q[3] / n};
    if (q[0] < 0.0) q = {-q[0], -q[1], -q[2], -q[3]};
    CameraView cam;
    cam.set_rotation_quat(q);
    for (int i = 0; i < 3; ++i)
        cam.translation[i] = -((cam.rotation[3 * i] * position[0] + cam.rotation[3 * i + 1] * position[1]) +
                               cam.rotation[3 * i + 2] * position[2]);
    cam.fx = fx; cam.fy = fy; cam.cx = cx; cam.cy = cy;
    cam.width = width;
    cam.height = height;
    return cam;
}

// ------------------------------------------------------------------ renderer
RenderOutput render(const GaussianCloud& cloud, const CameraView& cam, const RenderConfig& cfg, int device) {
    bsg_ctx* ctx = t_ctx.get(device, cloud.feature_dim());
    upload(ctx, cloud);
    RenderOutput out;
    out.color = Image(cam.width, cam.height);
    out.transmittance.resize(out.color.pixel_count());
    out.contributors.resize(out.color.pixel_count());
    const bsg_camera dc = to_dev(cam);
    const bsg_render_config rc = to_dev(cfg);
    check(bsg_render(ctx, &dc, &rc, out.color.data.data(), out.transmittance.data(), out.contributors.data()));
    return out;
}

double psnr(const Image& a, const Image& b) {  // metrics.cpp:14-26
    if (a.width != b.width || a.height != b.height) throw InvalidArgument("image dimensions differ");
    if (a.data.empty()) throw InvalidArgument("empty image");
    double acc = 0;
    for (size_t i = 0; i < a.data.size(); ++i) {
        const double d = a.data[i] - b.data[i];
        acc += d * d;
    }
    const double mse = acc / static_cast<double>(a.data.size());
    if (mse <= 0) return 99.0;
    return std::min(99.0, 10.0 * std::log10(1.0 / mse));
}

MetricsReport evaluate(const GaussianCloud& model, const std::vector<CameraView>& views,
                       const std::vector<Image>& images, uint32_t holdout_modulus, const RenderConfig& rc,
                       int device) {  // metrics.cpp:28-51
    if (views.size() != images.size()) throw InvalidArgument("image dimension mismatch");
    bsg_ctx* ctx = t_ctx.get(device, model.feature_dim());
    upload(ctx, model);
    std::vector<bsg_camera> cams(views.size());
    std::vector<const double*> gts(views.size());
    for (size_t i = 0; i < views.size(); ++i) {
        if (images[i].width != views[i].width || images[i].height != views[i].height)
            throw InvalidArgument("image dimension mismatch");
        cams[i] = to_dev(views[i]);
        gts[i] = images[i].data.data();
    }
    const bsg_render_config dc = to_dev(rc);
    std::vector<double> p(views.size() + 1), q(views.size() + 1);
    size_t k = 0;
    MetricsReport report;
    check(bsg_evaluate(ctx, views.size(), cams.data(), gts.data(), holdout_modulus, &dc, p.data(), q.data(), &k,
                       &report.mean_psnr, &report.mean_ssim));
    size_t j = 0;
    for (size_t i = 0; i < views.size(); ++i) {
        if (holdout_modulus != 0 && i % holdout_modulus != 0) continue;
        report.per_view.push_back(ViewMetrics{views[i].view_id, p[j], q[j]});
        ++j;
    }
    report.gaussian_count = model.size();
    return report;
}

BackwardOutput render_backward(const GaussianCloud& cloud, const CameraView& cam, const Image& gt,
                               const RenderConfig& cfg, int device) {
    if (gt.width != cam.width || gt.height != cam.height) throw InvalidArgument("image dimension mismatch");
    bsg_ctx* ctx = t_ctx.get(device, cloud.feature_dim());
    upload(ctx, cloud);
    BackwardOutput out;
    const size_t n = cloud.size();
    out.grads.positions.resize(3 * n);
    out.grads.rotations.resize(4 * n);
    out.grads.log_scales.resize(3 * n);
    out.grads.features.resize(n * cloud.feature_dim());
    out.grads.opacity_logits.resize(n);
    out.screen_grad_norm.resize(n);
    out.visible.resize(n);
    out.rendered = Image(cam.width, cam.height);
    const bsg_camera dc = to_dev(cam);
    const bsg_render_config rc = to_dev(cfg);
    double l3[3];
    check(bsg_render_backward(ctx, &dc, gt.data.data(), &rc, l3, out.grads.positions.data(), out.grads.rotations.data(),
                              out.grads.log_scales.data(), out.grads.features.data(), out.grads.opacity_logits.data(),
                              out.screen_grad_norm.data(), out.visible.data(), out.rendered.data.data()));
    out.loss = l3[0];
    out.l1 = l3[1];
    out.ssim = l3[2];
    return out;
}

PropertyPenalties adapt_penalties(const PropertyPenalties& rho, double primal, double dual, const ConsensusConfig& cfg,
                                  uint64_t iteration) {  // admm.cpp:200-217
    if (!cfg.adaptive || iteration > cfg.freeze_iteration) return rho;
    PropertyPenalties out = rho;
    auto scale_all = [&out](double f) {
        out.rho_p *= f; out.rho_q *= f; out.rho_s *= f; out.rho_f *= f; out.rho_o *= f;
    };
    if (primal > cfg.mu * dual)
        scale_all(cfg.tau_inc);
    else if (dual > cfg.mu * primal)
        scale_all(1.0 / cfg.tau_dec);
    return out;
}

// -------------------------------------------------------------- BlockTrainer
BlockTrainer::BlockTrainer(uint32_t block_id, GaussianCloud initial, std::vector<TrainView> views,
                           std::vector<uint64_t> shared_ids, uint64_t global_initial_count, const TrainerConfig& cfg,
                           int device)
    : block_id_(block_id), cfg_(cfg), fd_(initial.feature_dim()), views_(std::move(views)),
      shared_ids_(std::move(shared_ids)) {
    if (views_.empty()) throw InvalidArgument("trainer needs at least one view");
    if (!initial.check_invariants()) throw InvalidArgument("initial cloud ids not ascending");
    check(bsg_create(device, fd_, &ctx_));
    ids_ = initial.ids;
    upload(ctx_, initial);
    std::vector<bsg_camera> cams;
    std::vector<const double*> gts;
    for (const TrainView& v : views_) {
        if (!v.image) throw InvalidArgument("view without ground truth");
        if (v.image->width != v.camera.width || v.image->height != v.camera.height)
            throw InvalidArgument("image dimension mismatch");
        cams.push_back(to_dev(v.camera));
        gts.push_back(v.image->data.data());
    }
    check(bsg_set_views(ctx_, cams.size(), cams.data(), gts.data()));
    bsg_trainer_config tc = to_dev(cfg_);
    tc.densify.block_id = block_id;  // IdAllocator::for_block (trainer.cpp:55-61)
    tc.densify.global_initial_count = global_initial_count;
    check(bsg_trainer_init(ctx_, &tc));
    // trainer.cpp:116-118,135-159
    rng_ = new std::mt19937_64(derive_seed(cfg_.seed, block_id));
    view_order_.resize(views_.size());
    for (size_t i = 0; i < view_order_.size(); ++i) view_order_[i] = i;
    for (uint64_t id : shared_ids_)
        if (std::find(ids_.begin(), ids_.end(), id) == ids_.end()) throw InvalidArgument("shared rows missing from cloud");
    // the device needs the shared set before any anchor: densification buds
    // shared rows instead of splitting them (trainer.cpp:333-340)
    if (!shared_ids_.empty()) install_shared();
}

BlockTrainer::BlockTrainer(BlockTrainer&& o) noexcept
    : block_id_(o.block_id_), cfg_(o.cfg_), ctx_(o.ctx_), ids_(std::move(o.ids_)), fd_(o.fd_),
      views_(std::move(o.views_)), shared_ids_(std::move(o.shared_ids_)), slots_(std::move(o.slots_)),
      slot_owners_(std::move(o.slot_owners_)), first_(std::move(o.first_)), have_anchor_(o.have_anchor_),
      rng_state_seed_(o.rng_state_seed_), view_order_(std::move(o.view_order_)), view_cursor_(o.view_cursor_),
      last_loss_(o.last_loss_), rng_(o.rng_) {
    o.ctx_ = nullptr;
    o.rng_ = nullptr;
}

BlockTrainer::~BlockTrainer() {
    if (ctx_) bsg_destroy(ctx_);
    delete static_cast<std::mt19937_64*>(rng_);
}

double BlockTrainer::train_step() {
    run_iterations(1);
    return last_loss_;
}

void BlockTrainer::run_iterations(uint64_t n) {
    if (n == 0) return;
    auto& g = *static_cast<std::mt19937_64*>(rng_);
    std::vector<uint32_t> seq(n);
    draw_views(g, view_order_, view_cursor_, seq.data(), n);
    const uint64_t it0 = bsg_iteration(ctx_);
    std::vector<double> losses(n);
    check(bsg_train_steps(ctx_, n, seq.data(), losses.data()));
    last_loss_ = losses.back();
    // densification points (trainer.cpp:303-304) crossed by this batch
    const uint64_t stop = cfg_.densify.stop_iteration ? cfg_.densify.stop_iteration : (cfg_.iterations * 6) / 10;
    const uint64_t it1 = std::min<uint64_t>(it0 + n, stop), iv = cfg_.densify.interval;
    if (cfg_.densify.enabled && iv && it1 / iv > it0 / iv) refresh_ids();
}

// Densification on the device changes rows and ids (trainer.cpp:301-385):
// re-read the id column and the shared ids that survived.
void BlockTrainer::refresh_ids() {
    const size_t n = bsg_cloud_size(ctx_);
    ids_.resize(n);
    check(bsg_download_cloud(ctx_, ids_.data(), nullptr, nullptr, nullptr, nullptr, nullptr));
    size_t ns = 0;
    check(bsg_shared_ids(ctx_, nullptr, 0, &ns));
    shared_ids_.resize(ns);
    check(bsg_shared_ids(ctx_, shared_ids_.data(), ns, &ns));
    if (slots_.size() != shared_ids_.size()) slots_.clear();
}

std::vector<uint64_t> BlockTrainer::take_removed_ids() {  // trainer.cpp take_removed_ids
    size_t n = 0;
    check(bsg_take_removed_ids(ctx_, nullptr, 0, &n));
    std::vector<uint64_t> out(n);
    check(bsg_take_removed_ids(ctx_, out.data(), n, &n));
    return out;
}

GaussianCloud BlockTrainer::take_new_rows() {  // trainer.cpp take_new_rows
    size_t n = 0;
    check(bsg_take_new_ids(ctx_, nullptr, 0, &n));
    std::vector<uint64_t> ids(n);
    check(bsg_take_new_ids(ctx_, ids.data(), n, &n));
    return slice_by_ids(cloud(), ids);
}

void BlockTrainer::install_shared() {
    std::vector<uint32_t> rows(shared_ids_.size());
    for (size_t j = 0; j < shared_ids_.size(); ++j)
        rows[j] = static_cast<uint32_t>(std::lower_bound(ids_.begin(), ids_.end(), shared_ids_[j]) - ids_.begin());
    if (slots_.empty() || slots_.size() != shared_ids_.size()) {
        // standalone: block-local slots, one owner each
        slots_.resize(shared_ids_.size());
        for (size_t j = 0; j < slots_.size(); ++j) slots_[j] = static_cast<uint32_t>(j);
        first_.assign(shared_ids_.size(), 1);
        slot_owners_.assign(shared_ids_.size(), 1);
    }
    check(bsg_set_shared(ctx_, rows.size(), rows.data(), slots_.data(), first_.data(), slot_owners_.size(),
                         slot_owners_.data()));
}

void BlockTrainer::bind_slots(const std::vector<uint32_t>& slots, const std::vector<uint8_t>& first_owner,
                              const std::vector<uint32_t>& slot_owners) {
    if (slots.size() != shared_ids_.size() || first_owner.size() != shared_ids_.size())
        throw InvalidArgument("id misalignment");
    slots_ = slots;
    first_ = first_owner;
    slot_owners_ = slot_owners;
    install_shared();
}

void BlockTrainer::rebind_slots(const std::vector<uint64_t>& keep_ids, const std::vector<uint32_t>& slots,
                                const std::vector<uint8_t>& first_owner, const std::vector<uint32_t>& slot_owners,
                                const std::vector<double>& zprev_slots, const PropertyPenalties& rho) {
    const GaussianCloud a_old = anchor(), u_old = duals();
    const std::vector<double> ar = rows_of(a_old, find_all(a_old, keep_ids, "anchor misses kept ids")),
                              ur = rows_of(u_old, find_all(u_old, keep_ids, "duals miss kept ids"));
    shared_ids_ = keep_ids;
    bind_slots(slots, first_owner, slot_owners);
    const bsg_penalties p = to_dev(rho);
    check(bsg_set_anchor(ctx_, ar.data(), zprev_slots.empty() ? nullptr : zprev_slots.data(), &p));
    check(bsg_upload_duals(ctx_, ur.data()));
    have_anchor_ = true;
}

void BlockTrainer::set_anchor(const GaussianCloud& z, const PropertyPenalties& rho) {  // trainer.cpp:161-166
    if (slots_.size() != shared_ids_.size()) install_shared();
    const std::vector<double> zr = rows_of(z, find_all(z, shared_ids_, "broadcast misses shared ids"));
    // z_prev over the slot table: standalone slots are this block's own rows
    std::vector<double> zp;
    if (slot_owners_.size() == shared_ids_.size()) zp = zr;
    const bsg_penalties p = to_dev(rho);
    check(bsg_set_anchor(ctx_, zr.data(), zp.empty() ? nullptr : zp.data(), &p));
    have_anchor_ = true;
}

void BlockTrainer::apply_broadcast(const GaussianCloud& z, const std::vector<uint64_t>& reset_ids,
                                   const std::vector<uint64_t>& unshared_ids, const PropertyPenalties& rho,
                                   double alpha, bool over_relaxed) {  // trainer.cpp:168-223
    if (!have_anchor_) {
        set_anchor(z, rho);
        return;
    }
    if (slot_owners_.size() != shared_ids_.size())
        throw InvalidArgument("apply_broadcast needs block-local slots; group runs use the device consensus round");
    if (!unshared_ids.empty()) {
        // ids that stopped being shared leave first, with their anchor/dual rows
        const GaussianCloud u_old = duals(), a_old = anchor();
        std::vector<uint64_t> keep;
        std::set_difference(shared_ids_.begin(), shared_ids_.end(), unshared_ids.begin(), unshared_ids.end(),
                            std::back_inserter(keep));
        shared_ids_ = keep;
        slots_.clear();
        install_shared();
        const std::vector<double> ar = rows_of(a_old, find_all(a_old, keep, "anchor")),
                                  ur = rows_of(u_old, find_all(u_old, keep, "duals"));
        const bsg_penalties p = to_dev(rho);
        check(bsg_set_anchor(ctx_, ar.data(), ar.data(), &p));
        check(bsg_upload_duals(ctx_, ur.data()));
    }
    const std::vector<double> zr = rows_of(z, find_all(z, shared_ids_, "broadcast misses shared ids"));
    std::vector<uint32_t> resets;
    for (uint64_t id : reset_ids) {
        auto it = std::lower_bound(shared_ids_.begin(), shared_ids_.end(), id);
        if (it != shared_ids_.end() && *it == id) resets.push_back(static_cast<uint32_t>(it - shared_ids_.begin()));
    }
    check(bsg_apply_broadcast(ctx_, zr.data(), resets.size(), resets.empty() ? nullptr : resets.data(), alpha,
                              over_relaxed ? 1 : 0));
    const bsg_penalties p = to_dev(rho);
    check(bsg_set_penalties(ctx_, &p));
}

GaussianCloud BlockTrainer::cloud() const { return download(ctx_, fd_); }

GaussianCloud BlockTrainer::shared_slice() const { return slice_by_ids(cloud(), shared_ids_); }

GaussianCloud BlockTrainer::duals() const {
    std::vector<double> r(shared_ids_.size() * (11 + fd_));
    if (have_anchor_) check(bsg_download_duals(ctx_, r.data()));
    return bundle_of(shared_ids_, r, fd_);
}

GaussianCloud BlockTrainer::anchor() const {
    std::vector<double> r(shared_ids_.size() * (11 + fd_));
    if (have_anchor_) check(bsg_download_anchor(ctx_, r.data()));
    return bundle_of(have_anchor_ ? shared_ids_ : std::vector<uint64_t>{}, have_anchor_ ? r : std::vector<double>{},
                     fd_);
}

uint64_t BlockTrainer::iteration() const { return bsg_iteration(ctx_); }

// ------------------------------------------------------------------- runtime
std::vector<uint64_t> consensus_schedule(uint64_t total, uint32_t interval) {  // runtime.cpp:256-263
    if (total == 0) throw InvalidArgument("zero training iterations");
    if (interval == 0) throw InvalidArgument("zero consensus interval");
    std::vector<uint64_t> out;
    for (uint64_t t = interval; t < total; t += interval) out.push_back(t);
    out.push_back(total);
    return out;
}

ClusterPlan plan_cluster(const GaussianCloud& init, const std::vector<CameraView>& views,
                         const std::vector<Image>& images, uint32_t blocks, double expand_scale,
                         uint32_t holdout) {  // runtime.cpp:265-305
    if (views.empty()) throw InvalidArgument("scene has no views");
    if (images.size() != views.size()) throw InvalidArgument("one image per view required");
    if (!init.check_invariants()) throw InvalidArgument("initial cloud ill-formed");
    std::vector<double> centers(3 * views.size());
    for (size_t v = 0; v < views.size(); ++v) {
        const Vec3 c = views[v].center();
        for (int k = 0; k < 3; ++k) centers[3 * v + k] = c[k];
    }
    bsg_plan* p = nullptr;
    const int st = bsg_plan_create(init.size(), init.ids.data(), init.positions.data(), views.size(), centers.data(),
                                   blocks, expand_scale, 1, 0, &p);
    if (st != BSG_OK) {
        const std::string msg = bsg_plan_last_error();
        if (st == BSG_ERR_INVALID_ARGUMENT) throw InvalidArgument(msg);
        throw std::runtime_error(msg);
    }
    std::unique_ptr<bsg_plan, void (*)(bsg_plan*)> guard(p, bsg_plan_destroy);
    ClusterPlan plan;
    plan.init_cloud = init;
    const size_t S = bsg_plan_shared_count(p);
    plan.shared_ids.resize(S);
    plan.shared_owner_count.resize(S);
    plan.shared_first_owner.resize(S);
    bsg_plan_shared(p, plan.shared_ids.data(), plan.shared_owner_count.data(), plan.shared_first_owner.data());
    plan.shards.resize(blocks);
    for (uint32_t b = 0; b < blocks; ++b) {
        size_t ng = 0, nv = 0;
        bsg_plan_block_sizes(p, b, &ng, &nv);
        std::vector<uint64_t> ids(ng);
        std::vector<uint32_t> vs(nv);
        bsg_plan_block(p, b, ids.data(), vs.data());
        for (uint64_t id : ids) plan.owners[id].push_back(b);
        ShardSpec& s = plan.shards[b];
        s.block_id = b;
        s.global_initial_count = init.size();
        s.initial = slice_by_ids(init, ids);
        std::set_intersection(ids.begin(), ids.end(), plan.shared_ids.begin(), plan.shared_ids.end(),
                              std::back_inserter(s.shared_ids));
        for (uint32_t vi : vs) {
            if (holdout != 0 && vi % holdout == 0) continue;
            s.views.push_back(TrainView{views[vi], &images[vi]});
        }
        if (s.views.empty()) throw std::runtime_error("block " + std::to_string(b) + " has no training views");
    }
    return plan;
}

std::vector<uint32_t> view_sequence(uint64_t seed, uint32_t block_id, size_t n_views, size_t n_steps) {
    if (n_views == 0) throw InvalidArgument("block has no training views");  // trainer.cpp:147
    std::mt19937_64 g(derive_seed(seed, block_id));
    std::vector<size_t> order(n_views);
    for (size_t i = 0; i < n_views; ++i) order[i] = i;
    size_t cursor = 0;
    std::vector<uint32_t> seq(n_steps);
    draw_views(g, order, cursor, seq.data(), n_steps);
    return seq;
}

namespace {

// Generation barrier of the driver's threads; abort() releases every waiter
// with an exception (a failing block must not leave the others blocked).
class Barrier {
public:
    explicit Barrier(size_t n) : n_(n) {}
    void wait() {
        std::unique_lock<std::mutex> lk(m_);
        if (aborted_) throw std::runtime_error("run aborted by another block");
        const uint64_t gen = gen_;
        if (++count_ == n_) {
            count_ = 0;
            ++gen_;
            cv_.notify_all();
            return;
        }
        cv_.wait(lk, [&] { return gen_ != gen || aborted_; });
        if (gen_ == gen) throw std::runtime_error("run aborted by another block");
    }
    void abort() {
        std::lock_guard<std::mutex> lk(m_);
        aborted_ = true;
        cv_.notify_all();
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    size_t n_, count_ = 0;
    uint64_t gen_ = 0;
    bool aborted_ = false;
};

// In-process all-reduce among the K block threads (bsg_comm_init_host), for
// blocks that share a GPU (an NCCL communicator needs one device per rank):
// rank 0 reduces in ascending block order, every rank copies the result.
class HostGroup {
public:
    explicit HostGroup(size_t k) : k_(k), bar_(k), bufs_(k, nullptr) {}
    struct Member {
        HostGroup* g;
        size_t rank;
    };
    static int allreduce(void* user, void* buf, size_t count, int dtype, int op) {
        auto* m = static_cast<Member*>(user);
        try {
            m->g->run(m->rank, buf, count, dtype, op);
            return 0;
        } catch (...) {
            return 1;
        }
    }
    void abort() { bar_.abort(); }

private:
    template <typename T>
    void reduce(size_t count, int op) {
        T* acc = static_cast<T*>(bufs_[0]);
        for (size_t r = 1; r < k_; ++r) {
            const T* src = static_cast<const T*>(bufs_[r]);
            if (op == 1)
                for (size_t i = 0; i < count; ++i) acc[i] = std::max(acc[i], src[i]);
            else
                for (size_t i = 0; i < count; ++i) acc[i] += src[i];
        }
    }
    void run(size_t rank, void* buf, size_t count, int dtype, int op) {
        bufs_[rank] = buf;
        bar_.wait();
        if (rank == 0) {
            if (dtype == 1)
                reduce<double>(count, op);
            else
                reduce<float>(count, op);
        }
        bar_.wait();
        if (rank != 0) std::memcpy(buf, bufs_[0], count * (dtype == 1 ? 8 : 4));
        bar_.wait();
    }
    size_t k_;
    Barrier bar_;
    std::vector<void*> bufs_;
};

struct OwnerTableHandle {
    bsg_owner_table* t = nullptr;
    ~OwnerTableHandle() { bsg_owners_destroy(t); }
};

}  // namespace

RunResult run_simulated(const ClusterPlan& plan, const TrainerConfig& trainer, const SessionOptions& opt,
                        const std::function<void(const RoundDiagnostics&)>& observer,
                        const std::vector<int>& devices) {  // runtime.cpp:427-671
    const auto t0 = std::chrono::steady_clock::now();
    if (opt.total_iterations != trainer.iterations) throw InvalidArgument("session and trainer iteration counts differ");
    const auto K = static_cast<uint32_t>(plan.shards.size());
    if (K == 0) throw InvalidArgument("plan has no shards");
    if (K > 32) throw InvalidArgument("at most 32 blocks (owner bitmasks)");
    if (devices.empty()) throw InvalidArgument("no devices");
    const int fd = plan.init_cloud.feature_dim(), D = 11 + fd;
    std::vector<BlockTrainer> tr;
    tr.reserve(K);
    for (uint32_t b = 0; b < K; ++b) {
        const ShardSpec& s = plan.shards[b];
        tr.emplace_back(s.block_id, s.initial, s.views, s.shared_ids, s.global_initial_count, trainer,
                        devices[b % devices.size()]);
    }
    // Global slots, their owners (the device owner table on block 0's GPU) and
    // the round-0 anchor (runtime.cpp:465-477, trainer.cpp:161-166).
    std::vector<uint64_t> S = plan.shared_ids;  // the current consensus slot table (ascending ids)
    std::vector<uint32_t> slot_cnt = plan.shared_owner_count, slot_first = plan.shared_first_owner;
    OwnerTableHandle owners;
    {
        std::vector<uint32_t> masks(S.size(), 0);
        for (size_t k = 0; k < S.size(); ++k)
            for (uint32_t b : plan.owners.at(S[k])) masks[k] |= 1u << b;
        check(bsg_owners_create(devices[0], S.size(), S.data(), masks.data(), K, &owners.t));
    }
    const GaussianCloud z0 = slice_by_ids(plan.init_cloud, S);
    const std::vector<double> z0_rows = rows_of(z0, find_all(z0, S, "initial cloud ill-formed"));
    PropertyPenalties rho = opt.rho;
    const PropertyPenalties zero_rho{0, 0, 0, 0, 0};
    for (uint32_t b = 0; b < K; ++b) {
        const ShardSpec& s = plan.shards[b];
        std::vector<uint32_t> slots(s.shared_ids.size());
        std::vector<uint8_t> first(s.shared_ids.size());
        std::vector<double> zr(s.shared_ids.size() * D);
        for (size_t j = 0; j < s.shared_ids.size(); ++j) {
            slots[j] = static_cast<uint32_t>(std::lower_bound(S.begin(), S.end(), s.shared_ids[j]) - S.begin());
            first[j] = slot_first[slots[j]] == b ? 1 : 0;
            std::copy(&z0_rows[slots[j] * D], &z0_rows[slots[j] * D] + D, &zr[j * D]);
        }
        tr[b].bind_slots(slots, first, slot_cnt);
        // consensus disabled: blocks train independently (zero penalty), z is still reported
        const bsg_penalties p = to_dev(opt.consensus.enabled ? rho : zero_rho);
        check(bsg_set_anchor(tr[b].context(), zr.data(), z0_rows.data(), &p));
    }
    std::vector<bsg_ctx*> ctxs(K);
    for (uint32_t b = 0; b < K; ++b) ctxs[b] = tr[b].context();
    // Communicators: one NCCL rank per GPU when every block has its own
    // device (the 8xB200 layout), else the in-process host all-reduce.
    bool distinct = K > 1;
    for (uint32_t a = 0; a < K && distinct; ++a)
        for (uint32_t b = 0; b < a; ++b)
            if (devices[a % devices.size()] == devices[b % devices.size()]) distinct = false;
    HostGroup hg(K);
    std::vector<HostGroup::Member> members(K);
    if (K > 1) {
        if (distinct) {
            check(bsg_comm_init_local(ctxs.data(), K));
        } else {
            for (uint32_t b = 0; b < K; ++b) {
                members[b] = HostGroup::Member{&hg, b};
                check(bsg_comm_init_host(ctxs[b], &HostGroup::allreduce, &members[b], static_cast<int>(K),
                                         static_cast<int>(b)));
            }
        }
    }
    uint64_t global_count = plan.init_cloud.size();
    std::vector<uint64_t> alloc_start(K), newest(K, UINT64_MAX);  // IdAllocator ranges (trainer.cpp:55-61)
    for (uint32_t b = 0; b < K; ++b)
        alloc_start[b] = (static_cast<uint64_t>(plan.shards[b].block_id) << 48) +
                         (plan.shards[b].block_id == 0 ? plan.shards[b].global_initial_count : 0);
    bool have_z = false;  // a round has produced z (else the slot rebind starts from z0)

    // One host thread per block runs its iterations, reports its densify
    // changes, and -- after the master's bookkeeping -- starts its consensus
    // round asynchronously: the round's reductions and unpack run on the
    // block's communication stream while the block's next iterations
    // project, sort, blend and fold; only their first Adam waits for it
    // (SURVEY §8(e)). The master (this thread) collects the rounds' results
    // when the blocks wait for them at the next consensus point.
    struct Report {
        double loss = 0;
        std::vector<uint64_t> removed, added;
        bsg_round_result res{};
        bsg_penalties rho{};
    };
    std::vector<Report> rep(K);
    std::vector<std::vector<uint32_t>> resets(K);
    std::vector<bsg_round_args> args(K);
    bsg_adapt_args adapt{};
    adapt.mu = opt.consensus.mu;
    adapt.tau_inc = opt.consensus.tau_inc;
    adapt.tau_dec = opt.consensus.tau_dec;
    adapt.freeze_iteration = opt.consensus.freeze_iteration;
    adapt.adaptive = opt.consensus.adaptive ? 1 : 0;
    Barrier ready(K + 1), go(K + 1);
    std::vector<std::exception_ptr> errs(K + 1);
    auto fail_all = [&] {
        ready.abort();
        go.abort();
        hg.abort();
    };
    const std::vector<uint64_t> schedule = consensus_schedule(opt.total_iterations, opt.consensus.interval);
    std::vector<std::thread> workers;
    for (uint32_t b = 0; b < K; ++b)
        workers.emplace_back([&, b] {
            try {
                uint64_t done = 0;
                bool pending = false;
                for (size_t j = 0; j < schedule.size(); ++j) {
                    tr[b].run_iterations(schedule[j] - done);
                    done = schedule[j];
                    Report& r = rep[b];
                    if (pending) {
                        check(bsg_consensus_wait(tr[b].context(), &r.res, &r.rho));
                        pending = false;
                    }
                    r.loss = tr[b].last_loss();
                    r.removed = tr[b].take_removed_ids();
                    r.added = tr[b].take_new_rows().ids;
                    ready.wait();  // master: ownership bookkeeping, slot rebinds
                    go.wait();
                    check(bsg_consensus_round_async(tr[b].context(), &args[b],
                                                    opt.consensus.enabled ? &adapt : nullptr));
                    pending = true;
                }
                if (pending) check(bsg_consensus_wait(tr[b].context(), &rep[b].res, &rep[b].rho));
                ready.wait();
            } catch (...) {
                errs[b] = std::current_exception();
                fail_all();
            }
        });

    RunResult result;
    RoundDiagnostics pending_diag;
    auto emit = [&](RoundDiagnostics d) {  // the round's device results, collected by the blocks' waits
        const bsg_round_result& r = rep[0].res;
        d.primal_residual = r.primal;
        d.dual_residual = r.dual;
        d.max_disagreement = r.max_disagreement;
        d.dual_mean_linf = r.dual_mean_linf;
        d.consensus_ms = r.ms;
        if (opt.consensus.enabled) {
            const bsg_penalties& p = rep[0].rho;
            rho = PropertyPenalties{p.rho_p, p.rho_q, p.rho_s, p.rho_f, p.rho_o};
        }
        d.rho = rho;
        result.rounds.push_back(d);
        if (observer) observer(d);
    };
    try {
        for (size_t j = 0; j < schedule.size(); ++j) {
            const uint64_t t = schedule[j];
            const bool final_round = t == opt.total_iterations;
            ready.wait();
            if (j > 0) emit(pending_diag);
            // ownership changes from densification (runtime.cpp:490-518), on the device
            std::vector<const uint64_t*> rl(K);
            std::vector<size_t> rn(K);
            size_t n_removed = 0, n_added = 0;
            for (uint32_t b = 0; b < K; ++b) {
                rl[b] = rep[b].removed.data();
                rn[b] = rep[b].removed.size();
                n_removed += rn[b];
                n_added += rep[b].added.size();
            }
            std::vector<uint32_t> t_slot(S.size() + 1), t_mask(S.size() + 1);
            std::vector<uint8_t> t_class(S.size() + 1), found(std::max<size_t>(n_removed, 1));
            size_t touched = 0;
            check(bsg_owners_remove(owners.t, rl.data(), rn.data(), t_slot.data(), t_class.data(), t_mask.data(),
                                    t_slot.size(), &touched, found.data()));
            // a removed id outside the table had one owner and dies -- unless it
            // was born and pruned within this interval (never reported as new,
            // so never in the global model; runtime.cpp:498-499 skips it):
            // ids are allocated in increasing order per block (IdAllocator,
            // trainer.cpp:55-66), so such an id lies past the block's newest
            // reported one
            size_t dead = 0;
            for (uint32_t b = 0, i = 0; b < K; ++b)
                for (size_t q = 0; q < rn[b]; ++q, ++i) {
                    if (found[i]) continue;
                    const uint64_t id = rl[b][q];
                    const bool fresh = id >= alloc_start[b] && (newest[b] == UINT64_MAX || id > newest[b]);
                    dead += fresh ? 0 : 1;
                }
            for (uint32_t b = 0; b < K; ++b)
                for (uint64_t id : rep[b].added) newest[b] = newest[b] == UINT64_MAX ? id : std::max(newest[b], id);
            std::vector<uint64_t> reset_ids;
            std::vector<uint32_t> lost;  // slots that leave the table (now < 2 owners)
            for (size_t k = 0; k < touched; ++k) {
                if (t_class[k] == 3) ++dead;
                if (t_class[k] == 1) {
                    reset_ids.push_back(S[t_slot[k]]);
                    slot_cnt[t_slot[k]] = static_cast<uint32_t>(__builtin_popcount(t_mask[k]));
                    slot_first[t_slot[k]] = static_cast<uint32_t>(__builtin_ctz(t_mask[k]));
                } else {
                    lost.push_back(t_slot[k]);
                }
            }
            global_count = global_count + n_added - dead;
            if (!lost.empty()) {
                // new slot table: the kept slots in order; every block keeps its
                // anchor / duals for the ids that stay shared, z_prev from the
                // last consensus (all of it was shared before)
                std::vector<double> zp_old(S.size() * D);
                if (have_z && !S.empty())
                    check(bsg_download_consensus(ctxs[0], zp_old.data()));
                else
                    std::copy(z0_rows.begin(), z0_rows.end(), zp_old.begin());
                std::vector<uint64_t> S_new;
                std::vector<uint32_t> cnt_new, first_new;
                std::vector<double> zp_new;
                std::vector<uint32_t> new_of(S.size(), UINT32_MAX);
                size_t li = 0;
                for (size_t k = 0; k < S.size(); ++k) {
                    if (li < lost.size() && lost[li] == k) {
                        ++li;
                        continue;
                    }
                    new_of[k] = static_cast<uint32_t>(S_new.size());
                    S_new.push_back(S[k]);
                    cnt_new.push_back(slot_cnt[k]);
                    first_new.push_back(slot_first[k]);
                    zp_new.insert(zp_new.end(), &zp_old[k * D], &zp_old[k * D] + D);
                }
                for (uint32_t b = 0; b < K; ++b) {
                    std::vector<uint64_t> keep;
                    std::vector<uint32_t> slots;
                    std::vector<uint8_t> first;
                    for (uint64_t id : tr[b].shared_ids()) {
                        auto it = std::lower_bound(S.begin(), S.end(), id);
                        if (it == S.end() || *it != id) continue;
                        const uint32_t ns = new_of[it - S.begin()];
                        if (ns == UINT32_MAX) continue;
                        keep.push_back(id);
                        slots.push_back(ns);
                        first.push_back(first_new[ns] == b ? 1 : 0);
                    }
                    tr[b].rebind_slots(keep, slots, first, cnt_new, zp_new, opt.consensus.enabled ? rho : zero_rho);
                }
                S = std::move(S_new);
                slot_cnt = std::move(cnt_new);
                slot_first = std::move(first_new);
            }
            std::vector<uint32_t> reset_slots;
            for (uint64_t id : reset_ids) {
                auto it = std::lower_bound(S.begin(), S.end(), id);
                if (it != S.end() && *it == id) reset_slots.push_back(static_cast<uint32_t>(it - S.begin()));
            }
            // this round's arguments (runtime.cpp:529-548, trainer.cpp:168-223)
            adapt.iteration = t;
            for (uint32_t b = 0; b < K; ++b) {
                resets[b] = reset_slots;
                args[b] = bsg_round_args{};
                args[b].alpha = opt.consensus.alpha;
                args[b].relax = opt.consensus.enabled && opt.consensus.alpha != 1.0 && !final_round;
                args[b].diagnostics = 1;
                args[b].n_reset = resets[b].size();
                args[b].reset_slots = resets[b].empty() ? nullptr : resets[b].data();
            }
            pending_diag = RoundDiagnostics{};
            pending_diag.iteration = t;
            for (uint32_t b = 0; b < K; ++b) pending_diag.mean_loss += rep[b].loss;
            pending_diag.mean_loss /= K;
            pending_diag.shared_count = S.size();
            pending_diag.global_count = global_count;
            have_z = true;
            go.wait();
        }
        ready.wait();
        emit(pending_diag);
    } catch (...) {
        errs[K] = std::current_exception();
        fail_all();
    }
    for (auto& w : workers) w.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);

    // Global model (runtime.cpp:550-565): shared rows = normalised z, every
    // other row from the one block that holds it (a non-shared id has a single
    // owner: the others removed it).
    std::vector<double> zs(S.size() * D);
    if (!S.empty()) check(bsg_download_consensus(ctxs[0], zs.data()));
    std::vector<GaussianCloud> finals;
    finals.reserve(K);
    std::vector<uint64_t> all_ids(S.begin(), S.end());
    for (uint32_t b = 0; b < K; ++b) {
        finals.push_back(tr[b].cloud());
        for (uint64_t id : finals.back().ids)
            if (!std::binary_search(S.begin(), S.end(), id)) all_ids.push_back(id);
    }
    std::sort(all_ids.begin(), all_ids.end());
    all_ids.erase(std::unique(all_ids.begin(), all_ids.end()), all_ids.end());
    GaussianCloud model(fd);
    model.ids = all_ids;
    model.positions.resize(3 * model.size());
    model.rotations.resize(4 * model.size());
    model.log_scales.resize(3 * model.size());
    model.features.resize(static_cast<size_t>(fd) * model.size());
    model.opacity_logits.resize(model.size());
    auto row_of = [&](uint64_t id) {
        return static_cast<size_t>(std::lower_bound(model.ids.begin(), model.ids.end(), id) - model.ids.begin());
    };
    auto put = [&](size_t i, const double* row) {
        for (int k = 0; k < 3; ++k) model.positions[3 * i + k] = row[k];
        for (int k = 0; k < 4; ++k) model.rotations[4 * i + k] = row[3 + k];
        for (int k = 0; k < 3; ++k) model.log_scales[3 * i + k] = row[7 + k];
        for (int k = 0; k < fd; ++k) model.features[i * fd + k] = row[10 + k];
        model.opacity_logits[i] = row[10 + fd];
    };
    // shared rows: the consensus z with unit quaternions (runtime.cpp:578-581)
    for (size_t k = 0; k < S.size(); ++k) {
        double row[11 + kFeatureDimDeg1];
        std::copy(&zs[k * D], &zs[k * D] + D, row);
        const double qn = std::sqrt(((row[3] * row[3] + row[4] * row[4]) + row[5] * row[5]) + row[6] * row[6]);
        if (qn == 0.0) {
            row[3] = 1; row[4] = 0; row[5] = 0; row[6] = 0;
        } else {
            for (int q = 3; q < 7; ++q) row[q] /= qn;
        }
        put(row_of(S[k]), row);
    }
    for (uint32_t b = 0; b < K; ++b) {
        const GaussianCloud& c = finals[b];
        for (size_t j = 0; j < c.size(); ++j) {
            const uint64_t id = c.ids[j];
            if (std::binary_search(S.begin(), S.end(), id)) continue;
            double row[11 + kFeatureDimDeg1];
            for (int k = 0; k < 3; ++k) row[k] = c.positions[3 * j + k];
            for (int k = 0; k < 4; ++k) row[3 + k] = c.rotations[4 * j + k];
            for (int k = 0; k < 3; ++k) row[7 + k] = c.log_scales[3 * j + k];
            for (int k = 0; k < fd; ++k) row[10 + k] = c.features[j * fd + k];
            row[10 + fd] = c.opacity_logits[j];
            put(row_of(id), row);
        }
    }
    result.model = std::move(model);
    result.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return result;
}

}  // namespace blocksplat
