// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU FP64 restatement of the reference `blocksplat` hot path
// (/root/reference/proj/core). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load or call this code,
// and only as the checker or the timed CPU baseline. The product path
// (paper_2405_13943_b200/) never links, imports or falls back to it.
//
// Why a restatement and not the reference itself: the reference needs Eigen3
// (core/CMakeLists.txt:1, math.hpp:8-9), doctest and CLI11, none of which are
// present and there is no network, so it is unbuildable here.
// Every function cites the reference file:line it restates. Small fixed-size
// algebra that the reference writes with Eigen expressions is spelled out with
// a fixed, documented evaluation order (left-to-right sums); integer outputs
// (footprint rects, culling, depth order, block assignment) are pinned to this
// restatement, floating outputs to the reference's own known-answer tests
// (tests/test_oracle_kat.py cites each one).
// ============================================================================
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// cloud.hpp:14-17
inline constexpr double kSh0 = 0.28209479177387814;
inline constexpr double kSh1 = 0.4886025119029199;
inline constexpr int kFeatureDimDeg0 = 3;
inline constexpr int kFeatureDimDeg1 = 12;

// errors.hpp:33-36
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

struct V2 { double x = 0, y = 0; };
struct V3 {
    double v[3] = {0, 0, 0};
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
};
struct V4 {
    double v[4] = {0, 0, 0, 0};
    double& operator[](int i) { return v[i]; }
    double operator[](int i) const { return v[i]; }
};
struct M3 {
    double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double& operator()(int r, int c) { return m[r][c]; }
    double operator()(int r, int c) const { return m[r][c]; }
};
struct M2 {
    double m[2][2] = {{0, 0}, {0, 0}};
    double& operator()(int r, int c) { return m[r][c]; }
    double operator()(int r, int c) const { return m[r][c]; }
};

// ---- math.hpp ---------------------------------------------------------------
inline double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }     // math.hpp:20
inline double logit(double p) { return std::log(p / (1.0 - p)); }          // math.hpp:22
double norm4(const V4& q);
double norm3(const V3& v);
V4 quat_normalized(const V4& q);        // math.hpp:25-29
V4 quat_canonical(const V4& q);         // math.hpp:32-34
M3 quat_to_rotation(const V4& q);       // math.hpp:37-44
V4 rotation_to_quat(const M3& r);       // math.hpp:48-69

// math.hpp:74-135 — mt19937_64 with hand-rolled distributions.
class Rng {
public:
    explicit Rng(uint64_t seed) : gen_(seed) {}
    uint64_t next_u64() { return gen_(); }
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    uint64_t uniform_index(uint64_t n);
    double normal();
    V4 random_unit_quat();
    template <typename T>
    void shuffle(std::vector<T>& v) {
        for (size_t i = v.size(); i > 1; --i) {
            size_t j = static_cast<size_t>(uniform_index(i));
            std::swap(v[i - 1], v[j]);
        }
    }

private:
    std::mt19937_64 gen_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

uint64_t fnv1a64(const void* data, size_t n, uint64_t seed = 0xcbf29ce484222325ull);

// ---- camera.hpp -------------------------------------------------------------
struct Camera {
    uint64_t view_id = 0;
    double fx = 0, fy = 0, cx = 0, cy = 0;
    V4 q{{1, 0, 0, 0}};
    M3 R{{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
    V3 t;
    uint32_t width = 0, height = 0;
    void set_rotation_quat(const V4& qq) { q = qq; R = quat_to_rotation(qq); }   // camera.hpp:23-26
    V3 to_camera(const V3& p) const;                                           // camera.hpp:28
    V3 center() const;                                                         // camera.hpp:31
    V2 project(const V3& pc) const;                                            // camera.hpp:34-36
};
Camera look_at(const V3& position, const V3& target, const V3& world_up, double fx, double fy,
               double cx, double cy, uint32_t w, uint32_t h);                   // camera.hpp:42-58

// ---- cloud.hpp --------------------------------------------------------------
struct Cloud {
    int fd = kFeatureDimDeg0;
    std::vector<uint64_t> ids;
    std::vector<double> pos, rot, ls, feat, op;
    Cloud() = default;
    explicit Cloud(int f) : fd(f) {}
    size_t size() const { return ids.size(); }
    static constexpr size_t npos = static_cast<size_t>(-1);
    size_t find(uint64_t id) const;                         // cloud.cpp:76-80
    bool check_invariants() const;                          // cloud.cpp:66-74
    void canonicalize_rotations();                          // cloud.cpp:82-85
    void push_row(const Cloud& src, size_t i);
    Cloud subset(const std::vector<size_t>& idx) const;     // cloud.cpp:87-92
    void remove_indices(const std::vector<size_t>& idx);    // cloud.cpp:33-57
    void sort_by_id();                                      // cloud.cpp:59-64
    V3 position(size_t i) const { return V3{{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]}}; }
    V4 rotation(size_t i) const { return V4{{rot[4 * i], rot[4 * i + 1], rot[4 * i + 2], rot[4 * i + 3]}}; }
    V3 log_scale(size_t i) const { return V3{{ls[3 * i], ls[3 * i + 1], ls[3 * i + 2]}}; }
    double opacity(size_t i) const { return sigmoid(op[i]); }
};
Cloud slice_by_ids(const Cloud& c, const std::vector<uint64_t>& ids);   // cloud.cpp:94-102
size_t overwrite_by_ids(Cloud& dst, const Cloud& src);                  // cloud.cpp:104-120
void erase_by_ids(Cloud& dst, const std::vector<uint64_t>& ids);        // cloud.cpp:122-129
void insert_rows(Cloud& dst, const Cloud& rows);                        // cloud.cpp:131-138
Cloud zero_bundle(const std::vector<uint64_t>& ids, int fd);            // cloud.cpp:140-149
uint64_t cloud_checksum(const Cloud& c);                                // cloud.cpp:151-160
M3 covariance_from_params(const V4& q, const V3& log_scale);            // cloud.cpp:162-167
V3 sh_color(const double* f, int fd, const V3& view_dir);               // cloud.cpp:180-193

// ---- renderer.hpp -----------------------------------------------------------
struct RenderConfig {                                                   // renderer.hpp:13-21
    double near_plane = 0.01, dilation = 0.3, alpha_clamp = 0.99, transmittance_stop = 1e-4;
    double sigma_extent = 3.0;
    V3 background;
    double lambda = 0.2;
};

struct Image {                                                          // image.hpp:11-25
    uint32_t width = 0, height = 0;
    std::vector<double> data;
    Image() = default;
    Image(uint32_t w, uint32_t h, double fill = 0.0) : width(w), height(h), data(size_t(3) * w * h, fill) {}
    double& at(uint32_t x, uint32_t y, int c) { return data[3 * (size_t(y) * width + x) + c]; }
    double at(uint32_t x, uint32_t y, int c) const { return data[3 * (size_t(y) * width + x) + c]; }
    size_t pixel_count() const { return size_t(width) * height; }
};

struct PixelRect { int x0, x1, y0, y1; };

// Per-Gaussian projection record (renderer.cpp:43-49 Splat, plus the
// culled flag so tests can compare every row).
struct Projected {
    bool visible = false;
    V2 mean2d;
    M2 cov2d;
    double depth = 0;
    M2 minv;
    V3 color;
    double opacity = 0;
    PixelRect rect{0, -1, 0, -1};
};

Projected project_row(const Cloud& c, size_t i, const Camera& cam, const RenderConfig& cfg);
// Surviving rows in compositing order, renderer.cpp:63-91.
std::vector<size_t> depth_order(const std::vector<Projected>& pr);

struct RenderOut {
    Image color;
    std::vector<double> transmittance;
    std::vector<uint32_t> contributors;
};
RenderOut render(const Cloud& c, const Camera& cam, const RenderConfig& cfg);   // renderer.cpp:150-183
double loss_value(const Image& r, const Image& gt, double lambda);             // renderer.cpp:185-192

struct Grads {
    std::vector<double> pos, rot, ls, feat, op;
    void resize_for(const Cloud& c);                                          // renderer.cpp:142-148
};
struct BackwardOut {
    double loss = 0, l1 = 0, ssim = 0;
    Grads grads;
    std::vector<double> screen_grad_norm;
    std::vector<uint8_t> visible;
    Image rendered;
    Image dl_dc;                       // exposed for parity of the loss kernel
    // per surviving splat (compositing order) image-space gradients, for parity
    std::vector<size_t> order;
    std::vector<double> g_mean, g_cov, g_color, g_opacity;  // 2,4,3,1 per splat
};
BackwardOut render_backward(const Cloud& c, const Camera& cam, const Image& gt,
                            const RenderConfig& cfg);                          // renderer.cpp:217-406

// ---- ssim.hpp ---------------------------------------------------------------
inline constexpr int kSsimWindow = 11;
std::vector<double> ssim_window_1d();                                          // ssim.cpp:112-122
double ssim(const Image& x, const Image& y);                                   // ssim.cpp:124-136
double ssim_with_gradient(const Image& x, const Image& y, Image& dx);          // ssim.cpp:138-185

// ---- admm.hpp ---------------------------------------------------------------
struct Penalties { double rho_p = 1e4, rho_q = 1e4, rho_s = 1e4, rho_f = 1e3, rho_o = 1e4; };  // admm.hpp:12-18
struct ConsensusConfig {                                                     // admm.hpp:20-29
    uint32_t interval = 100;
    double mu = 10.0, tau_inc = 2.0, tau_dec = 2.0, alpha = 1.6;
    uint64_t freeze_iteration = 2000;
    bool adaptive = true, enabled = true;
};
inline double relaxed_value(double x, double z_prev, double alpha) {         // admm.hpp:38-41
    if (alpha == 1.0) return x;
    return alpha * x + (1.0 - alpha) * z_prev;
}
double penalty_loss_and_grad(const Cloud& c, const std::vector<size_t>& idx, const Cloud& z,
                             const Cloud& u, const Penalties& rho, Grads& g);  // admm.cpp:11-45
struct Contribution { uint32_t block_id; const Cloud* params; };
Cloud consensus_average(const std::vector<Contribution>& locals, bool over_relaxed,
                        const Cloud& z_prev, double alpha, std::vector<uint64_t>* flipped);  // admm.cpp:71-127
void dual_update(Cloud& u, const Cloud& x_hat, const Cloud& z);                // admm.cpp:129-145
struct Residuals { double primal = 0, dual = 0; };
Residuals residuals(const std::vector<Contribution>& locals, const Cloud& z_new,
                    const Cloud& z_prev, const Penalties& rho);                // admm.cpp:147-198
Penalties adapt_penalties(const Penalties& rho, double primal, double dual,
                          const ConsensusConfig& cfg, uint64_t iteration);     // admm.cpp:200-217
double max_disagreement(const std::vector<Contribution>& locals);             // admm.cpp:219-243

// ---- trainer.hpp ------------------------------------------------------------
struct LearningRates { double position = 1.6e-4, position_decay = 0.01, rotation = 1e-3,
                       log_scale = 5e-3, features = 2.5e-3, opacity = 5e-2; };   // trainer.hpp:13-20
struct AdamParams { double beta1 = 0.9, beta2 = 0.999, eps = 1e-8; };          // trainer.hpp:22-26
struct DensifyConfig {                                                          // trainer.hpp:43-51
    bool enabled = true;
    uint32_t interval = 200;
    uint64_t stop_iteration = 0;
    double grad_threshold = 2e-4, prune_opacity = 0.005, split_scale_fraction = 0.01, split_shrink = 1.6;
};
struct TrainerConfig {                                                          // trainer.hpp:53-62
    uint64_t iterations = 3000, seed = 0;
    int sh_degree = 0;
    double init_opacity = 0.1;
    LearningRates lr;
    AdamParams adam;
    DensifyConfig densify;
    RenderConfig render;
};
struct TrainView { Camera camera; const Image* image = nullptr; };             // trainer.hpp:80-83

struct ScenePoint { float p[3] = {0, 0, 0}; uint8_t rgb[3] = {0, 0, 0}; };     // scene.hpp:15-18
Cloud init_cloud_from_points(const std::vector<ScenePoint>& pts, int sh_degree, double init_opacity);  // trainer.cpp:68-112
uint64_t derive_seed(uint64_t seed, uint32_t block_id);                        // trainer.cpp:116-118

struct Aabb {                                                                   // splitter.hpp:13-28
    V3 min, max;
    bool contains(const V3& p) const;
    V3 center() const;
    V3 extent() const;
    double distance(const V3& p) const;
};
Aabb tight_aabb(const std::vector<V3>& pts);                                    // splitter.cpp:8-17

class BlockTrainer {                                                            // trainer.hpp:88-149
public:
    BlockTrainer(uint32_t block_id, Cloud initial, std::vector<TrainView> views,
                 std::vector<uint64_t> shared_ids, uint64_t global_initial_count,
                 const TrainerConfig& cfg);
    double train_step();
    void run_iterations(uint64_t n) { for (uint64_t i = 0; i < n; ++i) train_step(); }
    void set_anchor(const Cloud& z, const Penalties& rho);
    void apply_broadcast(const Cloud& z, const std::vector<uint64_t>& reset_ids,
                         const std::vector<uint64_t>& unshared_ids, const Penalties& rho,
                         double alpha, bool over_relaxed);
    const Cloud& cloud() const { return cloud_; }
    Cloud shared_slice() const { return slice_by_ids(cloud_, shared_ids_); }
    Cloud nonshared_slice() const;
    const Cloud& duals() const { return duals_; }
    const Cloud& anchor() const { return anchor_; }
    const std::vector<uint64_t>& shared_ids() const { return shared_ids_; }
    uint64_t iteration() const { return iteration_; }
    double last_loss() const { return last_loss_; }
    uint32_t block_id() const { return block_id_; }
    std::vector<uint64_t> take_removed_ids();
    Cloud take_new_rows();
    // Bookkeeping exposed for parity tests (trainer.cpp:145-146 state).
    const std::vector<double>& grad_accum() const { return grad_accum_; }
    const std::vector<uint32_t>& grad_seen() const { return grad_seen_; }
    const std::vector<size_t>& view_order() const { return view_order_; }
    size_t view_cursor() const { return view_cursor_; }
    // Moments in the [component][row] order of the device layout, for parity.
    std::vector<double> moments(int which) const;
    uint64_t adam_steps() const { return steps_; }
    size_t last_view() const { return last_view_; }

private:
    void maybe_densify();
    uint32_t block_id_;
    TrainerConfig cfg_;
    Cloud cloud_;
    std::vector<TrainView> views_;
    std::vector<uint64_t> shared_ids_;
    Cloud anchor_, duals_;
    Penalties rho_;
    bool have_anchor_ = false;
    std::vector<double> m_pos_, v_pos_, m_rot_, v_rot_, m_ls_, v_ls_, m_feat_, v_feat_, m_op_, v_op_;
    uint64_t steps_ = 0;
    uint64_t alloc_next_ = 0, alloc_end_ = 0;
    Rng rng_;
    std::vector<size_t> view_order_;
    size_t view_cursor_ = 0, last_view_ = 0;
    uint64_t iteration_ = 0;
    double last_loss_ = 0;
    double scene_extent_ = 1.0;
    std::vector<double> grad_accum_;
    std::vector<uint32_t> grad_seen_;
    std::vector<uint64_t> removed_ids_, new_ids_;
};

// ---- splitter.hpp -----------------------------------------------------------
struct SplitOptions { int vertical_axis = 1; bool midpoint_plane = false; };
struct CoreBlock { Aabb box; std::vector<size_t> point_indices; };
std::vector<CoreBlock> split_recursive(const std::vector<V3>& pts, uint32_t k, const SplitOptions& o);  // splitter.cpp:48-96
struct BlockPartition {
    uint32_t k = 0;
    std::vector<Aabb> core, expanded;
    std::vector<std::vector<size_t>> block_points, block_views;
    std::vector<std::vector<uint64_t>> block_gaussians;
    std::map<uint64_t, std::vector<uint32_t>> shared;
};
BlockPartition expand_and_assign(const std::vector<CoreBlock>& blocks, const std::vector<V3>& pts,
                                 const std::vector<Camera>& views, const Cloud& g, double scale,
                                 const SplitOptions& o);                                              // splitter.cpp:98-201

// ---- synth / runtime --------------------------------------------------------
struct SynthConfig { uint64_t seed = 0; uint32_t gaussians = 200, cameras = 24, image_size = 96;
                     double extent = 10.0; int sh_degree = 0; RenderConfig render; };   // synth.hpp:14-22
struct Scene {
    std::vector<ScenePoint> points;
    std::vector<Camera> views;
    std::vector<Image> images;
    bool has_checkpoint = false;
    Cloud checkpoint;
    Cloud ground_truth;
};
Scene generate_scene(const SynthConfig& cfg);
// Master-round ownership changes (runtime.cpp:490-518 + current_shared):
// owners updated in place; reset (before the flipped ids join), unshared,
// dead ids and the shared set after the round, all ascending.
struct OwnershipRound { std::vector<uint64_t> reset, unshared, dead, shared_now; };
OwnershipRound master_ownership_round(std::map<uint64_t, std::vector<uint32_t>>& owners,
                                      const std::vector<std::vector<uint64_t>>& removed,
                                      const std::vector<std::vector<uint64_t>>& added);                                  // synth.cpp:13-77

struct ShardSpec { uint32_t block_id = 0; Cloud initial; std::vector<TrainView> views;
                   std::vector<size_t> view_indices; std::vector<uint64_t> shared_ids;
                   uint64_t global_initial_count = 0; };
struct ClusterPlan { Cloud init_cloud; std::map<uint64_t, std::vector<uint32_t>> owners;
                     std::vector<ShardSpec> shards; BlockPartition partition; };
ClusterPlan plan_cluster(const Scene& scene, uint32_t blocks, double expand_scale,
                         uint32_t holdout, const TrainerConfig& tc, const SplitOptions& so);  // runtime.cpp:265-305
std::vector<uint64_t> consensus_schedule(uint64_t total, uint32_t interval);  // runtime.cpp:256-263

struct SessionOptions { ConsensusConfig consensus; Penalties rho; uint64_t total_iterations = 3000;
                        uint32_t nonshared_refresh = 10; };                     // runtime.hpp:109-115
struct RoundDiagnostics {                                                       // runtime.hpp:61-71
    uint64_t iteration = 0;
    double primal_residual = 0, dual_residual = 0;
    Penalties rho;
    double max_disagreement = 0, dual_mean_linf = 0, mean_loss = 0;
    size_t shared_count = 0, global_count = 0;
};
struct RunResult { Cloud model; std::vector<RoundDiagnostics> rounds; std::vector<Cloud> block_clouds; };
// run_simulated with the master session (runtime.cpp:427-621) executed
// in-line on one thread: workers are stepped in block order between barriers,
// which is observationally identical because blocks share no state.
RunResult run_simulated(const ClusterPlan& plan, const TrainerConfig& tc, const SessionOptions& opt);

double psnr(const Image& a, const Image& b);                                    // metrics.cpp:14-26

}  // namespace orc
