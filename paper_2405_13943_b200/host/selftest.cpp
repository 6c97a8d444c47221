// C++ self-test of the reference-shaped host API (include/blocksplat_gpu.hpp),
// mirroring a few of the reference's own unit tests (test_renderer.cpp,
// test_trainer.cpp) so that a reference call site is shown to compile and run
// unchanged against the device implementation. Exit code = failures.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "../../include/blocksplat_gpu.hpp"

using namespace blocksplat;

static int failures = 0;
#define CHECK(cond)                                                         \
    do {                                                                    \
        if (!(cond)) {                                                      \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                     \
        }                                                                   \
    } while (0)

static double logit(double p) { return std::log(p / (1.0 - p)); }

static CameraView axis_camera(double f, double c, uint32_t size) {  // test_renderer.cpp:18-24
    CameraView cam;
    cam.fx = cam.fy = f;
    cam.cx = cam.cy = c;
    cam.width = cam.height = size;
    return cam;
}

static void push(GaussianCloud& c, uint64_t id, Vec3 pos, Vec3 rgb, double opacity, double ls = -1.0) {
    c.ids.push_back(id);
    c.positions.insert(c.positions.end(), pos.begin(), pos.end());
    c.rotations.insert(c.rotations.end(), {1, 0, 0, 0});
    c.log_scales.insert(c.log_scales.end(), {ls, ls, ls});
    for (double v : rgb) c.features.push_back(v / kSh0);
    c.opacity_logits.push_back(logit(opacity));
}

// test_trainer.cpp:45-70 fixtures
static GaussianCloud spread_cloud(int n, double log_scale, double opacity0 = 0.5) {
    GaussianCloud c(kFeatureDimDeg0);
    for (int i = 0; i < n; ++i) {
        c.ids.push_back(static_cast<uint64_t>(i));
        c.positions.insert(c.positions.end(), {i * 5.0 - 2.5 * (n - 1), 0, 5});
        c.rotations.insert(c.rotations.end(), {1, 0, 0, 0});
        c.log_scales.insert(c.log_scales.end(), {log_scale, log_scale, log_scale});
        c.features.insert(c.features.end(), {1.5, 1.0, 0.5});
        c.opacity_logits.push_back(logit(i == 0 ? opacity0 : 0.5));
    }
    return c;
}

struct ViewHolder {
    Image img;
    std::vector<TrainView> views;
    ViewHolder(uint32_t size, double fill, double f, const Vec3& from) : img(size, size, fill) {
        const CameraView cam = look_at(from, {0, 0, 5}, {0, 1, 0}, f, f, size / 2.0, size / 2.0, size, size);
        views.push_back({cam, &img});
    }
};

int main() {
    {  // test_renderer.cpp:204-216 single centred splat
        GaussianCloud c(kFeatureDimDeg0);
        push(c, 1, {0, 0, 5}, {0.9, 0.5, 0.25}, 0.8);
        RenderOutput out = render(c, axis_camera(100, 8, 17));
        const size_t px = 8 * 17 + 8;
        CHECK(std::abs(out.color.data[3 * px] - 0.72) < 1e-6);
        CHECK(std::abs(out.transmittance[px] - 0.2) < 1e-6);
        CHECK(out.contributors[px] >= 1);
    }
    {  // test_renderer.cpp:272-282 early stop
        GaussianCloud c(kFeatureDimDeg0);
        for (int i = 0; i < 10; ++i) push(c, i + 1, {0, 0, 4 + 0.2 * i}, {0.5, 0.5, 0.5}, 0.9999);
        RenderOutput out = render(c, axis_camera(100, 8, 17));
        CHECK(out.contributors[8 * 17 + 8] == 3);
    }
    {  // test_metrics.cpp shape: psnr identities and evaluate's holdout rule on the device
        GaussianCloud c(kFeatureDimDeg0);
        push(c, 1, {0, 0, 5}, {0.9, 0.5, 0.25}, 0.8);
        const CameraView cam = axis_camera(100, 8, 17);
        const Image rendered = render(c, cam).color;
        CHECK(psnr(rendered, rendered) == 99.0);
        Image off = rendered;
        for (double& v : off.data) v += 0.1;
        CHECK(std::abs(psnr(rendered, off) - 20.0) < 1e-9);
        const MetricsReport m = evaluate(c, {cam, cam, cam}, {rendered, off, rendered}, 2);
        CHECK(m.per_view.size() == 2);  // views 0 and 2
        CHECK(m.per_view[0].psnr == 99.0 && m.per_view[1].psnr == 99.0);
        const MetricsReport all = evaluate(c, {cam, cam}, {rendered, off}, 0);
        CHECK(all.per_view.size() == 2 && std::abs(all.per_view[1].psnr - 20.0) < 1e-3);
    }
    {  // test_renderer.cpp:373-387 culled rows
        GaussianCloud c(kFeatureDimDeg0);
        push(c, 1, {0, 0, 5}, {0.5, 0.5, 0.5}, 0.7);
        push(c, 2, {0, 0, -5}, {0.5, 0.5, 0.5}, 0.7);
        BackwardOutput bw = render_backward(c, axis_camera(100, 8, 17), Image(17, 17, 0.9));
        CHECK(bw.visible[0] == 1 && bw.visible[1] == 0);
        CHECK(bw.grads.opacity_logits[1] == 0.0 && bw.grads.opacity_logits[0] != 0.0);
        bool threw = false;
        try {
            render_backward(c, axis_camera(100, 8, 17), Image(16, 17, 0.9));
        } catch (const InvalidArgument&) {
            threw = true;
        }
        CHECK(threw);
    }
    {  // test_trainer.cpp:275-306 anchor + broadcast bookkeeping
        GaussianCloud c(kFeatureDimDeg0);
        for (int i = 0; i < 3; ++i) push(c, i, {i * 5.0 - 5.0, 0, 5}, {0.5, 0.3, 0.2}, 0.5, -2.0);
        Image img(8, 8, 0.0);
        CameraView cam = look_at({0, 0, -5}, {0, 0, 5}, {0, 1, 0}, 10, 10, 4, 4, 8, 8);
        TrainerConfig cfg;
        cfg.iterations = 100;
        BlockTrainer t(0, c, {TrainView{cam, &img}}, {0, 1}, 3, cfg);
        PropertyPenalties rho;
        GaussianCloud z0 = slice_by_ids(c, {0, 1});
        for (double& v : z0.opacity_logits) v += 0.25;
        t.set_anchor(z0, rho);
        CHECK(t.anchor().ids == (std::vector<uint64_t>{0, 1}));
        for (double v : t.duals().opacity_logits) CHECK(v == 0.0);
        GaussianCloud z1 = slice_by_ids(c, {0});
        for (double& v : z1.opacity_logits) v -= 0.5;
        t.apply_broadcast(z1, {}, {1}, rho, 1.0, false);
        CHECK(t.shared_ids() == (std::vector<uint64_t>{0}));
        CHECK(std::abs(t.duals().opacity_logits[0] - 0.5) < 1e-6);
        t.apply_broadcast(z1, {0}, {}, rho, 1.0, false);
        CHECK(t.duals().opacity_logits[0] == 0.0);
        const double l0 = t.train_step();
        t.run_iterations(9);
        CHECK(t.iteration() == 10);
        CHECK(std::isfinite(l0) && std::isfinite(t.last_loss()));
    }
    // test_trainer.cpp:185-273: the reference's densification unit tests
    // through the device path (csrc/densify.cu)
    {  // densify prunes transparent gaussians
        GaussianCloud c = spread_cloud(2, -3.0, 0.001);
        ViewHolder vh(16, 0.0, 14, {0, 0, -4});
        TrainerConfig cfg;
        cfg.iterations = 100;
        cfg.densify.interval = 5;
        cfg.densify.grad_threshold = 1e9;  // isolate pruning
        BlockTrainer t(0, c, vh.views, {}, 2, cfg);
        t.run_iterations(5);
        CHECK(t.cloud().size() == 1);
        CHECK(t.cloud().ids == std::vector<uint64_t>{1});
        CHECK(t.take_removed_ids() == std::vector<uint64_t>{0});
        CHECK(t.take_new_rows().empty());
    }
    {  // densify clones small high-gradient gaussians
        GaussianCloud c = spread_cloud(2, -6.0);
        ViewHolder vh(16, 0.9, 14, {0, 0, -4});
        TrainerConfig cfg;
        cfg.iterations = 100;
        cfg.densify.interval = 4;
        cfg.densify.grad_threshold = 0.0;
        BlockTrainer t(0, c, vh.views, {}, 2, cfg);
        t.run_iterations(4);
        CHECK(t.cloud().size() == 4);
        CHECK(t.take_removed_ids().empty());
        CHECK(t.take_new_rows().ids == (std::vector<uint64_t>{2, 3}));
        CHECK(t.cloud().find(0) != GaussianCloud::npos && t.cloud().find(1) != GaussianCloud::npos);
    }
    {  // densify splits large gaussians and replaces the parent
        GaussianCloud c = spread_cloud(2, 0.0);
        ViewHolder vh(16, 0.9, 14, {0, 0, -4});
        TrainerConfig cfg;
        cfg.iterations = 100;
        cfg.lr.log_scale = 0.0;  // freeze scales so the shrink factor is exact
        cfg.densify.interval = 4;
        cfg.densify.grad_threshold = 0.0;
        BlockTrainer t(0, c, vh.views, {}, 2, cfg);
        t.run_iterations(4);
        CHECK(t.cloud().size() == 4);
        CHECK(t.take_removed_ids() == (std::vector<uint64_t>{0, 1}));
        CHECK(t.take_new_rows().ids == (std::vector<uint64_t>{2, 3, 4, 5}));
        const GaussianCloud m = t.cloud();
        for (size_t i = 0; i < m.size(); ++i)
            CHECK(std::abs(m.log_scales[3 * i] - (0.0 - std::log(1.6))) < 1e-6);  // FP32 storage
    }
    {  // shared gaussians bud a child and keep their id
        GaussianCloud c = spread_cloud(2, 0.0);
        ViewHolder vh(16, 0.9, 14, {0, 0, -4});
        TrainerConfig cfg;
        cfg.iterations = 100;
        cfg.densify.interval = 4;
        cfg.densify.grad_threshold = 0.0;
        BlockTrainer t(0, c, vh.views, {0}, 2, cfg);
        t.run_iterations(4);
        CHECK(t.cloud().size() == 4);
        CHECK(t.cloud().find(0) != GaussianCloud::npos);
        CHECK(t.cloud().find(1) == GaussianCloud::npos);
        CHECK(t.take_removed_ids() == std::vector<uint64_t>{1});
        CHECK(t.take_new_rows().size() == 3);
        CHECK(t.shared_ids() == std::vector<uint64_t>{0});
    }
    {  // pruning a shared gaussian also drops its consensus rows
        GaussianCloud c = spread_cloud(2, -3.0, 0.001);
        ViewHolder vh(16, 0.0, 14, {0, 0, -4});
        TrainerConfig cfg;
        cfg.iterations = 100;
        cfg.densify.interval = 5;
        cfg.densify.grad_threshold = 1e9;
        BlockTrainer t(0, c, vh.views, {0, 1}, 2, cfg);
        PropertyPenalties rho;
        t.set_anchor(slice_by_ids(c, {0, 1}), rho);
        CHECK(t.anchor().size() == 2);
        t.run_iterations(5);
        CHECK(t.shared_ids() == std::vector<uint64_t>{1});
        CHECK(t.anchor().ids == std::vector<uint64_t>{1});
        CHECK(t.duals().ids == std::vector<uint64_t>{1});
    }
    {  // scene container (test_image_scene.cpp:127-250): round trip, narrowing, error codes
        SceneDataset d;
        CameraView v = look_at({0, 2, -5}, {0, 0, 0}, {0, 1, 0}, 40, 40, 16, 12, 32, 24);
        v.view_id = 7;
        v.image_path = "gt/view_00007.ppm";
        d.views.push_back(v);
        d.points.push_back(ScenePoint{{0.5f, -1.0f, 2.0f}, {1, 2, 3}});
        d.has_checkpoint = true;
        d.checkpoint = spread_cloud(3, -1.5);
        d.checkpoint.positions[0] = 0.1;  // not representable in f32
        const std::vector<uint8_t> bytes = encode_scene(d);
        const SceneDataset back = decode_scene(bytes.data(), bytes.size());
        CHECK(back.views.size() == 1 && back.views[0].view_id == 7 && back.views[0].image_path == v.image_path);
        CHECK(back.views[0].fx == v.fx && back.views[0].translation == v.translation);
        CHECK(back.points.size() == 1 && back.points[0].rgb[2] == 3);
        CHECK(back.has_checkpoint && back.checkpoint.ids == d.checkpoint.ids);
        CHECK(back.checkpoint.positions == narrow_to_f32(d.checkpoint).positions);
        CHECK(encode_scene(back) == bytes);  // narrowing is idempotent
        auto code_of = [](std::vector<uint8_t> b) {
            try {
                decode_scene(b.data(), b.size());
            } catch (const FormatError& e) {
                return static_cast<int>(e.code());
            }
            return -1;
        };
        std::vector<uint8_t> bad = bytes;
        bad[0] = 'X';
        CHECK(code_of(bad) == static_cast<int>(FormatErrorCode::BadMagic));
        bad = bytes;
        bad.resize(bad.size() - 3);
        CHECK(code_of(bad) == static_cast<int>(FormatErrorCode::TruncatedSection));
        bad = bytes;
        bad.push_back(0);
        CHECK(code_of(bad) == static_cast<int>(FormatErrorCode::TruncatedBuffer));
        // the device encoder writes the same GSPL section as the host codec
        bsg_ctx* ctx = nullptr;
        CHECK(bsg_create(0, 3, &ctx) == BSG_OK);
        const GaussianCloud& c = d.checkpoint;
        CHECK(bsg_upload_cloud(ctx, c.size(), c.ids.data(), c.positions.data(), c.rotations.data(),
                               c.log_scales.data(), c.features.data(), c.opacity_logits.data()) == BSG_OK);
        const std::vector<uint8_t> dev = encode_gspl_device(ctx);
        CHECK(dev.size() > 12 && std::equal(dev.begin(), dev.end(), bytes.end() - static_cast<long>(dev.size())));
        bsg_destroy(ctx);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures;
}
