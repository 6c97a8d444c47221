// blocksplat_gpu.hpp — C++ host API mirroring the reference's blocksplat
// headers (renderer.hpp, admm.hpp, trainer.hpp, runtime.hpp) on top of the
// B200 C-ABI (bsgpu.h). Same class / function names and argument meaning, so
// reference call sites recompile against it; the work runs on sm_100a.
//
// Differences from the reference, by design:
//  - No Eigen: small vectors are std::array (Vec3/Vec4), CameraView::rotation
//    is a row-major std::array<double, 9>.
//  - BlockTrainer owns a device context; cloud()/duals()/anchor() download.
//  - Densification (trainer.cpp:301-385) runs on the device; run_simulated
//    keeps the master's id / owner bookkeeping (runtime.cpp:490-518) on the host.
//  - FP32 device state: results match the FP64 reference within the
//    tolerances stated in tests/ (integer paths bit-exact).
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "bsgpu.h"

namespace blocksplat {

using Vec3 = std::array<double, 3>;
using Vec4 = std::array<double, 4>;
using Mat3 = std::array<double, 9>;  // row-major

inline constexpr double kSh0 = 0.28209479177387814;  // cloud.hpp:14
inline constexpr double kSh1 = 0.4886025119029199;   // cloud.hpp:15
inline constexpr int kFeatureDimDeg0 = 3;
inline constexpr int kFeatureDimDeg1 = 12;

class InvalidArgument : public std::invalid_argument {  // errors.hpp:33-36
public:
    using std::invalid_argument::invalid_argument;
};

// cloud.hpp:32-102 (SoA, ids ascending)
class GaussianCloud {
public:
    GaussianCloud() = default;
    explicit GaussianCloud(int feature_dim) : feature_dim_(feature_dim) {}
    int feature_dim() const { return feature_dim_; }
    size_t size() const { return ids.size(); }
    bool empty() const { return ids.empty(); }
    std::vector<uint64_t> ids;
    std::vector<double> positions, rotations, log_scales, features, opacity_logits;
    static constexpr size_t npos = static_cast<size_t>(-1);
    size_t find(uint64_t id) const;
    bool check_invariants() const;

private:
    int feature_dim_ = kFeatureDimDeg0;
};
GaussianCloud slice_by_ids(const GaussianCloud& cloud, const std::vector<uint64_t>& ids);  // cloud.cpp:94-102

// camera.hpp:14-58
struct CameraView {
    uint64_t view_id = 0;
    double fx = 0, fy = 0, cx = 0, cy = 0;
    Vec4 rotation_q{1, 0, 0, 0};
    Mat3 rotation{1, 0, 0, 0, 1, 0, 0, 0, 1};
    Vec3 translation{0, 0, 0};
    uint32_t width = 0, height = 0;
    std::string image_path;
    void set_rotation_quat(const Vec4& q);
    Vec3 center() const;
};
CameraView look_at(const Vec3& position, const Vec3& target, const Vec3& world_up, double fx, double fy, double cx,
                   double cy, uint32_t width, uint32_t height);

// errors.hpp:10-31: container / wire decode errors, matched on the code.
enum class FormatErrorCode {
    BadMagic,
    UnsupportedVersion,
    TruncatedSection,
    UnknownSection,
    TruncatedBuffer,
    CountOverflow,
    NonMonotoneIds,
    BadHeader,
};
class FormatError : public std::runtime_error {
public:
    FormatError(FormatErrorCode code, const std::string& message) : std::runtime_error(message), code_(code) {}
    FormatErrorCode code() const noexcept { return code_; }

private:
    FormatErrorCode code_;
};

struct Image {  // image.hpp:11-25
    uint32_t width = 0, height = 0;
    std::vector<double> data;
    Image() = default;
    Image(uint32_t w, uint32_t h, double fill = 0.0) : width(w), height(h), data(size_t(3) * w * h, fill) {}
    size_t pixel_count() const { return size_t(width) * height; }
};

struct RenderConfig {  // renderer.hpp:13-21
    double near_plane = 0.01, dilation = 0.3, alpha_clamp = 0.99, transmittance_stop = 1e-4, sigma_extent = 3.0;
    Vec3 background{0, 0, 0};
    double lambda = 0.2;
};

struct RenderOutput {  // renderer.hpp:39-43
    Image color;
    std::vector<double> transmittance;
    std::vector<uint32_t> contributors;
};

struct ParamGradients {  // renderer.hpp:46-54
    std::vector<double> positions, rotations, log_scales, features, opacity_logits;
};

struct BackwardOutput {  // renderer.hpp:56-67
    double loss = 0, l1 = 0, ssim = 0;
    ParamGradients grads;
    std::vector<double> screen_grad_norm;
    std::vector<uint8_t> visible;
    Image rendered;
};

// renderer.hpp:71-81 (device 0 unless given)
RenderOutput render(const GaussianCloud& cloud, const CameraView& cam, const RenderConfig& cfg = {}, int device = 0);
BackwardOutput render_backward(const GaussianCloud& cloud, const CameraView& cam, const Image& gt,
                               const RenderConfig& cfg = {}, int device = 0);

// metrics.hpp:15-36. psnr is the reference's host formula; evaluate renders
// and scores on the device (bsg_evaluate). The reference takes a LoadedScene;
// here its views and images are passed directly (same holdout rule).
double psnr(const Image& a, const Image& b);
struct ViewMetrics {
    uint64_t view_id = 0;
    double psnr = 0;
    double ssim = 0;
};
struct MetricsReport {
    std::vector<ViewMetrics> per_view;
    double mean_psnr = 0;
    double mean_ssim = 0;
    size_t gaussian_count = 0;
};
MetricsReport evaluate(const GaussianCloud& model, const std::vector<CameraView>& views,
                       const std::vector<Image>& images, uint32_t holdout_modulus, const RenderConfig& rc = {},
                       int device = 0);

// trainer.hpp:13-62
struct LearningRates {
    double position = 1.6e-4, position_decay = 0.01, rotation = 1e-3, log_scale = 5e-3, features = 2.5e-3,
           opacity = 5e-2;
};
struct AdamParams {
    double beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
};
struct DensifyConfig {
    bool enabled = true;  // on the device (csrc/densify.cu); run_simulated tracks ownership on the device (csrc/owners.cu)
    uint32_t interval = 200;
    uint64_t stop_iteration = 0;
    double grad_threshold = 2e-4, prune_opacity = 0.005, split_scale_fraction = 0.01, split_shrink = 1.6;
};
struct TrainerConfig {
    uint64_t iterations = 3000;
    uint64_t seed = 0;
    int sh_degree = 0;
    double init_opacity = 0.1;
    LearningRates lr;
    AdamParams adam;
    DensifyConfig densify;
    RenderConfig render;
};
struct TrainView {  // trainer.hpp:80-83
    CameraView camera;
    const Image* image = nullptr;
};

struct PropertyPenalties {  // admm.hpp:12-18
    double rho_p = 1e4, rho_q = 1e4, rho_s = 1e4, rho_f = 1e3, rho_o = 1e4;
};
struct ConsensusConfig {  // admm.hpp:20-29
    uint32_t interval = 100;
    double mu = 10.0, tau_inc = 2.0, tau_dec = 2.0, alpha = 1.6;
    uint64_t freeze_iteration = 2000;
    bool adaptive = true, enabled = true;
};
PropertyPenalties adapt_penalties(const PropertyPenalties& rho, double primal_norm, double dual_norm,
                                  const ConsensusConfig& cfg, uint64_t iteration);  // admm.cpp:200-217

// trainer.hpp:88-149, one device context per block.
class BlockTrainer {
public:
    BlockTrainer(uint32_t block_id, GaussianCloud initial, std::vector<TrainView> views,
                 std::vector<uint64_t> shared_ids, uint64_t global_initial_count, const TrainerConfig& cfg,
                 int device = 0);
    ~BlockTrainer();
    BlockTrainer(const BlockTrainer&) = delete;
    BlockTrainer& operator=(const BlockTrainer&) = delete;
    BlockTrainer(BlockTrainer&&) noexcept;

    double train_step();
    void run_iterations(uint64_t n);
    void set_anchor(const GaussianCloud& z, const PropertyPenalties& rho);
    void apply_broadcast(const GaussianCloud& z, const std::vector<uint64_t>& reset_ids,
                         const std::vector<uint64_t>& unshared_ids, const PropertyPenalties& rho, double alpha,
                         bool over_relaxed);

    GaussianCloud cloud() const;
    GaussianCloud shared_slice() const;
    GaussianCloud duals() const;
    GaussianCloud anchor() const;
    const std::vector<uint64_t>& shared_ids() const { return shared_ids_; }
    // trainer.hpp:137-140: ids removed by densification since the last call, and
    // the rows it added that are still in the cloud (ascending ids).
    std::vector<uint64_t> take_removed_ids();
    GaussianCloud take_new_rows();
    uint64_t iteration() const;
    double last_loss() const { return last_loss_; }
    uint32_t block_id() const { return block_id_; }
    bsg_ctx* context() const { return ctx_; }
    // Global consensus slots (used by run_simulated): rows of this block's
    // shared ids in the group-wide slot table.
    void bind_slots(const std::vector<uint32_t>& slots, const std::vector<uint8_t>& first_owner,
                    const std::vector<uint32_t>& slot_owners);
    // The group's shared set changed (densification, runtime.cpp:490-518): keep
    // only `keep_ids` (ascending) on new slots, carrying their anchor and duals;
    // zprev_slots = the master's z_prev for the new slot table (rows x D).
    void rebind_slots(const std::vector<uint64_t>& keep_ids, const std::vector<uint32_t>& slots,
                      const std::vector<uint8_t>& first_owner, const std::vector<uint32_t>& slot_owners,
                      const std::vector<double>& zprev_slots, const PropertyPenalties& rho);

private:
    void install_shared();
    void refresh_ids();
    uint32_t block_id_;
    TrainerConfig cfg_;
    bsg_ctx* ctx_ = nullptr;
    std::vector<uint64_t> ids_;
    int fd_;
    std::vector<TrainView> views_;
    std::vector<uint64_t> shared_ids_;
    std::vector<uint32_t> slots_, slot_owners_;
    std::vector<uint8_t> first_;
    bool have_anchor_ = false;
    uint64_t rng_state_seed_;
    std::vector<size_t> view_order_;
    size_t view_cursor_ = 0;
    double last_loss_ = 0;
    void* rng_ = nullptr;  // std::mt19937_64
};

// runtime.hpp:61-115
struct RoundDiagnostics {
    uint64_t iteration = 0;
    double primal_residual = 0, dual_residual = 0;
    PropertyPenalties rho;
    double max_disagreement = 0, dual_mean_linf = 0, mean_loss = 0;
    size_t shared_count = 0, global_count = 0;
    double consensus_ms = 0;
};
struct RunResult {
    GaussianCloud model;
    std::vector<RoundDiagnostics> rounds;
    double wall_seconds = 0;
};
struct ShardSpec {
    uint32_t block_id = 0;
    GaussianCloud initial;
    std::vector<TrainView> views;
    std::vector<uint64_t> shared_ids;
    uint64_t global_initial_count = 0;
};
struct ClusterPlan {
    GaussianCloud init_cloud;
    std::map<uint64_t, std::vector<uint32_t>> owners;
    std::vector<ShardSpec> shards;
    std::vector<uint64_t> shared_ids;        // consensus slots, ascending
    std::vector<uint32_t> shared_owner_count;
    std::vector<uint32_t> shared_first_owner;
};
// plan_cluster (runtime.cpp:265-305) from an initial cloud (the checkpoint
// path, runtime.cpp:273-275) and the scene's views + images.
ClusterPlan plan_cluster(const GaussianCloud& init_cloud, const std::vector<CameraView>& views,
                         const std::vector<Image>& images, uint32_t blocks, double expand_scale,
                         uint32_t holdout_modulus);
std::vector<uint64_t> consensus_schedule(uint64_t total_iterations, uint32_t interval);  // runtime.cpp:256-263

struct SessionOptions {  // runtime.hpp:109-115
    ConsensusConfig consensus;
    PropertyPenalties rho;
    uint64_t total_iterations = 3000;
    uint32_t nonshared_refresh = 10;
};
// run_simulated (runtime.cpp:623-671): K blocks in one process, one host
// thread per block, each starting its consensus round asynchronously so the
// round overlaps its next iterations; the all-reduces go over NCCL (one rank
// per GPU) when every block has its own device, else through an in-process
// host all-reduce (blocks sharing a GPU). The master's ownership bookkeeping
// (runtime.cpp:490-518) runs on the device owner table (bsg_owners_*).
// devices[b % devices.size()] hosts block b.
// The view order BlockTrainer::train_step draws (trainer.cpp:116-118,250-252:
// derive_seed, then a Fisher-Yates shuffle with rejection-sampled indices on
// mt19937_64 at the start of every pass) -- the same code path.
std::vector<uint32_t> view_sequence(uint64_t seed, uint32_t block_id, size_t n_views, size_t n_steps);

RunResult run_simulated(const ClusterPlan& plan, const TrainerConfig& trainer, const SessionOptions& opt,
                        const std::function<void(const RoundDiagnostics&)>& observer = {},
                        const std::vector<int>& devices = {0});

// scene.hpp:15-50 / scene_io.cpp: the DOGS container (little-endian, magic
// "DOGS", version u32, tagged sections CAMS / PNTS / GSPL, each a 4-byte tag,
// a u64 length and the payload). GSPL is the f32 Gaussian checkpoint; the
// trained model is written as a container holding only it (main.cpp:353-357).
struct ScenePoint {
    std::array<float, 3> position{0, 0, 0};
    std::array<uint8_t, 3> rgb{0, 0, 0};
};
struct SceneDataset {
    std::vector<ScenePoint> points;
    std::vector<CameraView> views;
    bool has_checkpoint = false;
    GaussianCloud checkpoint;
};
inline constexpr uint32_t kSceneFormatVersion = 1;
std::vector<uint8_t> encode_scene(const SceneDataset& scene);
SceneDataset decode_scene(const uint8_t* data, size_t size);
void save_scene(const std::string& path, const SceneDataset& scene);
SceneDataset load_scene(const std::string& path);
GaussianCloud narrow_to_f32(const GaussianCloud& cloud);
// The GSPL payload of a block's device cloud, encoded on the device
// (bsg_encode_gspl): byte-identical to the GSPL section encode_scene writes
// for that cloud (the device parameters are already f32).
std::vector<uint8_t> encode_gspl_device(bsg_ctx* ctx);
// model.dogs (main.cpp:353-357): a container holding only the narrowed model.
void save_model(const std::string& path, const GaussianCloud& model);

}  // namespace blocksplat
