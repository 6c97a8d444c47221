// C++ host layer (include/blocksplat_gpu.hpp): the reference's blocksplat API
// (renderer.hpp, trainer.hpp, runtime.hpp) implemented over the C-ABI in
// bsgpu.h. Host bookkeeping only; every FLOP of the hot path runs in
// libbsgpu's sm_100a kernels.
#include "../../include/blocksplat_gpu.hpp"

#include <algorithm>
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

RunResult run_simulated(const ClusterPlan& plan, const TrainerConfig& trainer, const SessionOptions& opt,
                        const std::function<void(const RoundDiagnostics&)>& observer,
                        const std::vector<int>& devices) {  // runtime.cpp:427-671
    const auto t0 = std::chrono::steady_clock::now();
    if (opt.total_iterations != trainer.iterations) throw InvalidArgument("session and trainer iteration counts differ");
    const auto K = static_cast<uint32_t>(plan.shards.size());
    if (K == 0) throw InvalidArgument("plan has no shards");
    if (devices.empty()) throw InvalidArgument("no devices");
    const int fd = plan.init_cloud.feature_dim(), D = 11 + fd;
    std::vector<BlockTrainer> tr;
    tr.reserve(K);
    for (uint32_t b = 0; b < K; ++b) {
        const ShardSpec& s = plan.shards[b];
        tr.emplace_back(s.block_id, s.initial, s.views, s.shared_ids, s.global_initial_count, trainer,
                        devices[b % devices.size()]);
    }
    // Global slots and the round-0 anchor (runtime.cpp:465-477, trainer.cpp:161-166).
    std::vector<uint64_t> S = plan.shared_ids;  // the current consensus slot table (ascending ids)
    std::map<uint64_t, std::vector<uint32_t>> owners = plan.owners;
    std::set<uint64_t> global_ids(plan.init_cloud.ids.begin(), plan.init_cloud.ids.end());
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
            first[j] = plan.shared_first_owner[slots[j]] == b ? 1 : 0;
            std::copy(&z0_rows[slots[j] * D], &z0_rows[slots[j] * D] + D, &zr[j * D]);
        }
        tr[b].bind_slots(slots, first, plan.shared_owner_count);
        // consensus disabled: blocks train independently (zero penalty), z is still reported
        const bsg_penalties p = to_dev(opt.consensus.enabled ? rho : zero_rho);
        check(bsg_set_anchor(tr[b].context(), zr.data(), z0_rows.data(), &p));
    }
    std::vector<bsg_ctx*> ctxs(K);
    for (uint32_t b = 0; b < K; ++b) ctxs[b] = tr[b].context();

    RunResult result;
    const std::vector<uint64_t> schedule = consensus_schedule(opt.total_iterations, opt.consensus.interval);
    uint64_t done = 0;
    for (uint64_t t : schedule) {
        const bool final_round = t == opt.total_iterations;
        // worker halves in parallel, one host thread per block (runtime.cpp:641-656)
        std::vector<std::exception_ptr> errs(K);
        std::vector<std::thread> th;
        for (uint32_t b = 0; b < K; ++b)
            th.emplace_back([&, b] {
                try {
                    tr[b].run_iterations(t - done);
                } catch (...) {
                    errs[b] = std::current_exception();
                }
            });
        for (auto& x : th) x.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        done = t;
        // ownership changes from densification (runtime.cpp:490-518)
        std::map<uint64_t, size_t> prev_owner_count;
        for (uint32_t b = 0; b < K; ++b)
            for (uint64_t id : tr[b].take_removed_ids()) {
                auto it = owners.find(id);
                if (it == owners.end()) continue;
                prev_owner_count.emplace(id, it->second.size());
                auto& list = it->second;
                list.erase(std::remove(list.begin(), list.end(), b), list.end());
            }
        std::vector<uint64_t> reset_ids, dead_ids;
        for (const auto& [id, prev] : prev_owner_count) {
            const auto& list = owners.at(id);
            if (list.empty())
                dead_ids.push_back(id);
            else if (prev >= 2 && list.size() >= 2)
                reset_ids.push_back(id);  // (prev >= 2, now 1 owner: unshared, leaves the slot table)
        }
        for (uint64_t id : dead_ids) {
            owners.erase(id);
            global_ids.erase(id);
        }
        for (uint32_t b = 0; b < K; ++b)
            for (uint64_t id : tr[b].take_new_rows().ids) {
                owners[id] = {b};
                global_ids.insert(id);
            }
        // The shared set only shrinks (new rows have one owner; removals drop
        // owners), so it is S minus the ids that fell below two owners: a
        // merge over S and the (sorted) changed ids instead of a scan of the
        // whole owner map every round.
        std::vector<uint64_t> lost;
        for (const auto& [id, prev] : prev_owner_count) {
            (void)prev;
            auto it = owners.find(id);
            if (it == owners.end() || it->second.size() < 2) lost.push_back(id);
        }
        std::vector<uint64_t> shared_now;
        if (!lost.empty()) {
            shared_now.reserve(S.size());
            std::set_difference(S.begin(), S.end(), lost.begin(), lost.end(), std::back_inserter(shared_now));
        }
        if (!lost.empty() && shared_now.size() != S.size()) {
            // new slot table; every block keeps its anchor / duals for the ids
            // that stay shared, z_prev comes from the last consensus (all of
            // shared_now was shared before: new rows start single-owner)
            std::vector<double> zp_old(S.size() * D), zp_new(shared_now.size() * D);
            if (!S.empty()) check(bsg_download_consensus(ctxs[0], zp_old.data()));
            if (done == schedule.front()) std::copy(z0_rows.begin(), z0_rows.end(), zp_old.begin());
            std::vector<uint32_t> cnt(shared_now.size()), first_owner(shared_now.size());
            for (size_t k = 0; k < shared_now.size(); ++k) {
                const size_t old = std::lower_bound(S.begin(), S.end(), shared_now[k]) - S.begin();
                std::copy(&zp_old[old * D], &zp_old[old * D] + D, &zp_new[k * D]);
                const auto& list = owners.at(shared_now[k]);
                cnt[k] = static_cast<uint32_t>(list.size());
                first_owner[k] = *std::min_element(list.begin(), list.end());
            }
            for (uint32_t b = 0; b < K; ++b) {
                std::vector<uint64_t> keep;
                std::vector<uint32_t> slots;
                std::vector<uint8_t> first;
                for (uint64_t id : tr[b].shared_ids()) {
                    auto it = std::lower_bound(shared_now.begin(), shared_now.end(), id);
                    if (it == shared_now.end() || *it != id) continue;
                    keep.push_back(id);
                    slots.push_back(static_cast<uint32_t>(it - shared_now.begin()));
                    first.push_back(first_owner[slots.back()] == b ? 1 : 0);
                }
                tr[b].rebind_slots(keep, slots, first, cnt, zp_new, opt.consensus.enabled ? rho : zero_rho);
                ctxs[b] = tr[b].context();
            }
            S = shared_now;
        }
        std::vector<uint32_t> reset_slots;
        for (uint64_t id : reset_ids) {
            auto it = std::lower_bound(S.begin(), S.end(), id);
            if (it != S.end() && *it == id) reset_slots.push_back(static_cast<uint32_t>(it - S.begin()));
        }
        // consensus round on the device (runtime.cpp:529-548, trainer.cpp:168-223)
        bsg_round_args args{};
        args.alpha = opt.consensus.alpha;
        args.relax = opt.consensus.enabled && opt.consensus.alpha != 1.0 && !final_round;
        args.diagnostics = 1;
        args.n_reset = reset_slots.size();
        args.reset_slots = reset_slots.empty() ? nullptr : reset_slots.data();
        bsg_round_result r{};
        const auto r0 = std::chrono::steady_clock::now();
        check(bsg_group_consensus_round(ctxs.data(), K, &args, &r));
        const double round_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - r0).count();
        if (opt.consensus.enabled) {
            rho = adapt_penalties(rho, r.primal, r.dual, opt.consensus, t);
            const bsg_penalties p = to_dev(rho);
            for (auto* c : ctxs) check(bsg_set_penalties(c, &p));
        }
        RoundDiagnostics d;
        d.iteration = t;
        d.primal_residual = r.primal;
        d.dual_residual = r.dual;
        d.rho = rho;
        d.max_disagreement = r.max_disagreement;
        d.dual_mean_linf = r.dual_mean_linf;
        for (auto& x : tr) d.mean_loss += x.last_loss();
        d.mean_loss /= K;
        d.shared_count = S.size();
        d.global_count = global_ids.size();
        d.consensus_ms = round_ms;
        result.rounds.push_back(d);
        if (observer) observer(d);
    }
    // Global model (runtime.cpp:550-565): shared rows = normalised z, the rest
    // from their single owner's final cloud.
    GaussianCloud model(fd);
    model.ids.assign(global_ids.begin(), global_ids.end());
    model.positions.resize(3 * model.size());
    model.rotations.resize(4 * model.size());
    model.log_scales.resize(3 * model.size());
    model.features.resize(static_cast<size_t>(fd) * model.size());
    model.opacity_logits.resize(model.size());
    std::vector<double> zs(S.size() * D);
    if (!S.empty()) check(bsg_download_consensus(ctxs[0], zs.data()));
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
    // every other row from its single owner's final cloud, one pass per block
    for (uint32_t b = 0; b < K; ++b) {
        const GaussianCloud c = tr[b].cloud();
        for (size_t j = 0; j < c.size(); ++j) {
            const uint64_t id = c.ids[j];
            if (std::binary_search(S.begin(), S.end(), id)) continue;
            auto it = owners.find(id);
            if (it == owners.end() || it->second.front() != b) continue;
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
