// ORACLE — TEST INFRASTRUCTURE ONLY. pybind11 bindings of the CPU FP64
// restatement (orc.hpp) for tests/, smoke() and bench.py's CPU baseline leg.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <chrono>

#include "orc.hpp"

namespace py = pybind11;
using namespace orc;

namespace {

template <typename T>
py::array_t<T> to_np(const std::vector<T>& v, std::vector<ssize_t> shape) {
    py::array_t<T> a(shape);
    std::memcpy(a.mutable_data(), v.data(), v.size() * sizeof(T));
    return a;
}

template <typename T>
std::vector<T> from_np(py::array_t<T, py::array::c_style | py::array::forcecast> a) {
    return std::vector<T>(a.data(), a.data() + a.size());
}

Cloud make_cloud(py::array_t<uint64_t, py::array::c_style | py::array::forcecast> ids,
                 py::array_t<double, py::array::c_style | py::array::forcecast> pos,
                 py::array_t<double, py::array::c_style | py::array::forcecast> rot,
                 py::array_t<double, py::array::c_style | py::array::forcecast> ls,
                 py::array_t<double, py::array::c_style | py::array::forcecast> feat,
                 py::array_t<double, py::array::c_style | py::array::forcecast> op) {
    const size_t n = static_cast<size_t>(ids.size());
    const int fd = n ? static_cast<int>(feat.size() / n) : (feat.ndim() == 2 ? static_cast<int>(feat.shape(1)) : 3);
    Cloud c(fd);
    c.ids = from_np<uint64_t>(ids);
    c.pos = from_np<double>(pos);
    c.rot = from_np<double>(rot);
    c.ls = from_np<double>(ls);
    c.feat = from_np<double>(feat);
    c.op = from_np<double>(op);
    if (!c.check_invariants() && n > 0) {
        // shapes are validated; ordering is the caller's business (trainer checks it)
        if (c.pos.size() != 3 * n || c.rot.size() != 4 * n || c.ls.size() != 3 * n || c.op.size() != n)
            throw InvalidArgument("cloud array shapes inconsistent");
    }
    return c;
}

py::dict cloud_dict(const Cloud& c) {
    py::dict d;
    const ssize_t n = static_cast<ssize_t>(c.size());
    d["ids"] = to_np(c.ids, {n});
    d["pos"] = to_np(c.pos, {n, 3});
    d["rot"] = to_np(c.rot, {n, 4});
    d["ls"] = to_np(c.ls, {n, 3});
    d["feat"] = to_np(c.feat, {n, c.fd});
    d["op"] = to_np(c.op, {n});
    return d;
}

Image make_image(py::array_t<double, py::array::c_style | py::array::forcecast> a) {
    if (a.ndim() != 3 || a.shape(2) != 3) throw InvalidArgument("image must be HxWx3");
    Image im(static_cast<uint32_t>(a.shape(1)), static_cast<uint32_t>(a.shape(0)));
    im.data = from_np<double>(a);
    return im;
}

py::array_t<double> image_np(const Image& im) {
    return to_np(im.data, {static_cast<ssize_t>(im.height), static_cast<ssize_t>(im.width), 3});
}

}  // namespace

PYBIND11_MODULE(_oracle, m) {
    m.doc() = "ORACLE (test infrastructure only): CPU FP64 restatement of the blocksplat reference";
    py::register_exception<InvalidArgument>(m, "InvalidArgument", PyExc_ValueError);

    py::class_<Cloud>(m, "Cloud")
        .def(py::init(&make_cloud))
        .def_readonly("fd", &Cloud::fd)
        .def("size", &Cloud::size)
        .def("dict", &cloud_dict)
        .def("find", &Cloud::find)
        .def("checksum", [](const Cloud& c) { return cloud_checksum(c); });

    py::class_<Camera>(m, "Camera")
        .def(py::init<>())
        .def_readwrite("view_id", &Camera::view_id)
        .def_readwrite("fx", &Camera::fx).def_readwrite("fy", &Camera::fy)
        .def_readwrite("cx", &Camera::cx).def_readwrite("cy", &Camera::cy)
        .def_readwrite("width", &Camera::width).def_readwrite("height", &Camera::height)
        .def("set_rotation_quat", [](Camera& c, std::array<double, 4> q) { c.set_rotation_quat(V4{{q[0], q[1], q[2], q[3]}}); })
        .def_property("t", [](const Camera& c) { return std::array<double, 3>{c.t[0], c.t[1], c.t[2]}; },
                      [](Camera& c, std::array<double, 3> t) { for (int i = 0; i < 3; ++i) c.t[i] = t[i]; })
        .def_property_readonly("q", [](const Camera& c) { return std::array<double, 4>{c.q[0], c.q[1], c.q[2], c.q[3]}; })
        .def_property_readonly("R", [](const Camera& c) {
            std::vector<double> r(9);
            for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r[3 * i + j] = c.R(i, j);
            return to_np(r, {3, 3});
        })
        .def("center", [](const Camera& c) { V3 v = c.center(); return std::array<double, 3>{v[0], v[1], v[2]}; });

    m.def("look_at", [](std::array<double, 3> p, std::array<double, 3> t, std::array<double, 3> up, double fx, double fy,
                        double cx, double cy, uint32_t w, uint32_t h) {
        return look_at(V3{{p[0], p[1], p[2]}}, V3{{t[0], t[1], t[2]}}, V3{{up[0], up[1], up[2]}}, fx, fy, cx, cy, w, h);
    });
    m.def("quat_to_rotation", [](std::array<double, 4> q) {
        M3 r = quat_to_rotation(V4{{q[0], q[1], q[2], q[3]}});
        std::vector<double> v(9);
        for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) v[3 * i + j] = r(i, j);
        return to_np(v, {3, 3});
    });

    py::class_<RenderConfig>(m, "RenderConfig")
        .def(py::init<>())
        .def_readwrite("near_plane", &RenderConfig::near_plane)
        .def_readwrite("dilation", &RenderConfig::dilation)
        .def_readwrite("alpha_clamp", &RenderConfig::alpha_clamp)
        .def_readwrite("transmittance_stop", &RenderConfig::transmittance_stop)
        .def_readwrite("sigma_extent", &RenderConfig::sigma_extent)
        .def_readwrite("lambda_", &RenderConfig::lambda)
        .def_property("background", [](const RenderConfig& c) { return std::array<double, 3>{c.background[0], c.background[1], c.background[2]}; },
                      [](RenderConfig& c, std::array<double, 3> b) { for (int i = 0; i < 3; ++i) c.background[i] = b[i]; });

    m.def("project", [](const Cloud& c, const Camera& cam, const RenderConfig& cfg) {
        const ssize_t n = static_cast<ssize_t>(c.size());
        std::vector<uint8_t> vis(n);
        std::vector<double> depth(n), mean(2 * n), cov(4 * n), minv(4 * n), color(3 * n), opac(n);
        std::vector<int32_t> rect(4 * n);
        std::vector<Projected> pr(n);
        for (ssize_t i = 0; i < n; ++i) {
            const Projected p = project_row(c, i, cam, cfg);
            pr[i] = p;
            vis[i] = p.visible;
            depth[i] = p.depth;
            mean[2 * i] = p.mean2d.x; mean[2 * i + 1] = p.mean2d.y;
            for (int a = 0; a < 2; ++a) for (int b = 0; b < 2; ++b) {
                cov[4 * i + 2 * a + b] = p.cov2d(a, b);
                minv[4 * i + 2 * a + b] = p.minv(a, b);
            }
            for (int k = 0; k < 3; ++k) color[3 * i + k] = p.color[k];
            opac[i] = p.opacity;
            rect[4 * i] = p.rect.x0; rect[4 * i + 1] = p.rect.x1; rect[4 * i + 2] = p.rect.y0; rect[4 * i + 3] = p.rect.y1;
        }
        std::vector<size_t> order = depth_order(pr);
        std::vector<int64_t> ord(order.begin(), order.end());
        py::dict d;
        d["visible"] = to_np(vis, {n});
        d["depth"] = to_np(depth, {n});
        d["mean2d"] = to_np(mean, {n, 2});
        d["cov2d"] = to_np(cov, {n, 2, 2});
        d["minv"] = to_np(minv, {n, 2, 2});
        d["color"] = to_np(color, {n, 3});
        d["opacity"] = to_np(opac, {n});
        d["rect"] = to_np(rect, {n, 4});
        d["order"] = to_np(ord, {static_cast<ssize_t>(ord.size())});
        return d;
    });

    m.def("render", [](const Cloud& c, const Camera& cam, const RenderConfig& cfg) {
        RenderOut o;
        {
            py::gil_scoped_release rel;  // pure function: fixture renders may run on threads
            o = render(c, cam, cfg);
        }
        const ssize_t h = cam.height, w = cam.width;
        return py::make_tuple(image_np(o.color), to_np(o.transmittance, {h, w}), to_np(o.contributors, {h, w}));
    });

    m.def("render_backward", [](const Cloud& c, const Camera& cam, py::array_t<double> gt, const RenderConfig& cfg) {
        BackwardOut o = render_backward(c, cam, make_image(gt), cfg);
        const ssize_t n = static_cast<ssize_t>(c.size());
        const ssize_t ns = static_cast<ssize_t>(o.order.size());
        py::dict d;
        d["loss"] = o.loss; d["l1"] = o.l1; d["ssim"] = o.ssim;
        d["g_pos"] = to_np(o.grads.pos, {n, 3});
        d["g_rot"] = to_np(o.grads.rot, {n, 4});
        d["g_ls"] = to_np(o.grads.ls, {n, 3});
        d["g_feat"] = to_np(o.grads.feat, {n, c.fd});
        d["g_op"] = to_np(o.grads.op, {n});
        d["screen_grad_norm"] = to_np(o.screen_grad_norm, {n});
        d["visible"] = to_np(o.visible, {n});
        d["rendered"] = image_np(o.rendered);
        d["dl_dc"] = image_np(o.dl_dc);
        std::vector<int64_t> ord(o.order.begin(), o.order.end());
        d["order"] = to_np(ord, {ns});
        d["s_mean"] = to_np(o.g_mean, {ns, 2});
        d["s_cov"] = to_np(o.g_cov, {ns, 2, 2});
        d["s_color"] = to_np(o.g_color, {ns, 3});
        d["s_opacity"] = to_np(o.g_opacity, {ns});
        return d;
    });

    m.def("ssim", [](py::array_t<double> x, py::array_t<double> y) { return ssim(make_image(x), make_image(y)); });
    m.def("ssim_with_gradient", [](py::array_t<double> x, py::array_t<double> y) {
        Image dx;
        double s = ssim_with_gradient(make_image(x), make_image(y), dx);
        return py::make_tuple(s, image_np(dx));
    });
    m.def("ssim_window_1d", &ssim_window_1d);
    m.def("loss_value", [](py::array_t<double> r, py::array_t<double> g, double lam) { return loss_value(make_image(r), make_image(g), lam); });
    m.def("psnr", [](py::array_t<double> a, py::array_t<double> b) { return psnr(make_image(a), make_image(b)); });

    py::class_<Penalties>(m, "Penalties")
        .def(py::init<>())
        .def_readwrite("rho_p", &Penalties::rho_p).def_readwrite("rho_q", &Penalties::rho_q)
        .def_readwrite("rho_s", &Penalties::rho_s).def_readwrite("rho_f", &Penalties::rho_f)
        .def_readwrite("rho_o", &Penalties::rho_o);
    py::class_<ConsensusConfig>(m, "ConsensusConfig")
        .def(py::init<>())
        .def_readwrite("interval", &ConsensusConfig::interval).def_readwrite("mu", &ConsensusConfig::mu)
        .def_readwrite("tau_inc", &ConsensusConfig::tau_inc).def_readwrite("tau_dec", &ConsensusConfig::tau_dec)
        .def_readwrite("alpha", &ConsensusConfig::alpha).def_readwrite("freeze_iteration", &ConsensusConfig::freeze_iteration)
        .def_readwrite("adaptive", &ConsensusConfig::adaptive).def_readwrite("enabled", &ConsensusConfig::enabled);

    m.def("penalty_loss_and_grad", [](const Cloud& c, std::vector<size_t> idx, const Cloud& z, const Cloud& u, const Penalties& rho) {
        Grads g;
        g.resize_for(c);
        double loss = penalty_loss_and_grad(c, idx, z, u, rho, g);
        const ssize_t n = static_cast<ssize_t>(c.size());
        py::dict d;
        d["loss"] = loss;
        d["g_pos"] = to_np(g.pos, {n, 3}); d["g_rot"] = to_np(g.rot, {n, 4}); d["g_ls"] = to_np(g.ls, {n, 3});
        d["g_feat"] = to_np(g.feat, {n, c.fd}); d["g_op"] = to_np(g.op, {n});
        return d;
    });
    m.def("consensus_average", [](std::vector<std::pair<uint32_t, Cloud>> locals, bool relax, const Cloud& z_prev, double alpha) {
        std::vector<Contribution> cs;
        for (auto& [b, c] : locals) cs.push_back(Contribution{b, &c});
        std::vector<uint64_t> flipped;
        Cloud z = consensus_average(cs, relax, z_prev, alpha, &flipped);
        return py::make_tuple(z, flipped);
    });
    m.def("dual_update", [](Cloud u, const Cloud& x_hat, const Cloud& z) { dual_update(u, x_hat, z); return u; });
    m.def("residuals", [](std::vector<std::pair<uint32_t, Cloud>> locals, const Cloud& zn, const Cloud& zp, const Penalties& rho) {
        std::vector<Contribution> cs;
        for (auto& [b, c] : locals) cs.push_back(Contribution{b, &c});
        Residuals r = residuals(cs, zn, zp, rho);
        return py::make_tuple(r.primal, r.dual);
    });
    m.def("adapt_penalties", &adapt_penalties);
    m.def("max_disagreement", [](std::vector<std::pair<uint32_t, Cloud>> locals) {
        std::vector<Contribution> cs;
        for (auto& [b, c] : locals) cs.push_back(Contribution{b, &c});
        return max_disagreement(cs);
    });
    m.def("slice_by_ids", &slice_by_ids);
    m.def("zero_bundle", &zero_bundle);

    py::class_<TrainerConfig>(m, "TrainerConfig")
        .def(py::init<>())
        .def_readwrite("iterations", &TrainerConfig::iterations).def_readwrite("seed", &TrainerConfig::seed)
        .def_readwrite("sh_degree", &TrainerConfig::sh_degree).def_readwrite("init_opacity", &TrainerConfig::init_opacity)
        .def_property("densify_enabled", [](const TrainerConfig& c) { return c.densify.enabled; },
                      [](TrainerConfig& c, bool v) { c.densify.enabled = v; })
        .def_property("densify_interval", [](const TrainerConfig& c) { return c.densify.interval; },
                      [](TrainerConfig& c, uint32_t v) { c.densify.interval = v; })
        .def_property("densify_stop_iteration", [](const TrainerConfig& c) { return c.densify.stop_iteration; },
                      [](TrainerConfig& c, uint64_t v) { c.densify.stop_iteration = v; })
        .def_property("densify_grad_threshold", [](const TrainerConfig& c) { return c.densify.grad_threshold; },
                      [](TrainerConfig& c, double v) { c.densify.grad_threshold = v; })
        .def_property("densify_prune_opacity", [](const TrainerConfig& c) { return c.densify.prune_opacity; },
                      [](TrainerConfig& c, double v) { c.densify.prune_opacity = v; })
        .def_property("densify_split_scale_fraction", [](const TrainerConfig& c) { return c.densify.split_scale_fraction; },
                      [](TrainerConfig& c, double v) { c.densify.split_scale_fraction = v; })
        .def_property("densify_split_shrink", [](const TrainerConfig& c) { return c.densify.split_shrink; },
                      [](TrainerConfig& c, double v) { c.densify.split_shrink = v; })
        .def_property("lr", [](const TrainerConfig& c) {
            return std::array<double, 6>{c.lr.position, c.lr.position_decay, c.lr.rotation, c.lr.log_scale, c.lr.features, c.lr.opacity}; },
                      [](TrainerConfig& c, std::array<double, 6> v) {
            c.lr.position = v[0]; c.lr.position_decay = v[1]; c.lr.rotation = v[2]; c.lr.log_scale = v[3]; c.lr.features = v[4]; c.lr.opacity = v[5]; })
        .def_readwrite("render", &TrainerConfig::render);

    // Trainer with its ground-truth images owned by the Python wrapper.
    struct PyTrainer {
        std::vector<Image> images;
        std::unique_ptr<BlockTrainer> t;
    };
    py::class_<PyTrainer>(m, "BlockTrainer")
        .def(py::init([](uint32_t block_id, const Cloud& init, std::vector<Camera> cams, std::vector<py::array_t<double>> gts,
                         std::vector<uint64_t> shared, uint64_t global_count, const TrainerConfig& cfg) {
            auto p = std::make_unique<PyTrainer>();
            p->images.reserve(gts.size());
            for (auto& g : gts) p->images.push_back(make_image(g));
            std::vector<TrainView> views;
            for (size_t i = 0; i < cams.size(); ++i) views.push_back(TrainView{cams[i], &p->images[i]});
            p->t = std::make_unique<BlockTrainer>(block_id, init, views, shared, global_count, cfg);
            return p;
        }))
        .def("train_step", [](PyTrainer& p) { return p.t->train_step(); })
        .def("run_iterations", [](PyTrainer& p, uint64_t n) { p.t->run_iterations(n); })
        .def("set_anchor", [](PyTrainer& p, const Cloud& z, const Penalties& rho) { p.t->set_anchor(z, rho); })
        .def("apply_broadcast", [](PyTrainer& p, const Cloud& z, std::vector<uint64_t> reset, std::vector<uint64_t> unshared,
                                   const Penalties& rho, double alpha, bool relax) { p.t->apply_broadcast(z, reset, unshared, rho, alpha, relax); })
        .def("cloud", [](PyTrainer& p) { return p.t->cloud(); })
        .def("duals", [](PyTrainer& p) { return p.t->duals(); })
        .def("anchor", [](PyTrainer& p) { return p.t->anchor(); })
        .def("shared_ids", [](PyTrainer& p) { return p.t->shared_ids(); })
        .def("shared_slice", [](PyTrainer& p) { return p.t->shared_slice(); })
        .def("iteration", [](PyTrainer& p) { return p.t->iteration(); })
        .def("last_loss", [](PyTrainer& p) { return p.t->last_loss(); })
        .def("last_view", [](PyTrainer& p) { return p.t->last_view(); })
        .def("view_order", [](PyTrainer& p) { return p.t->view_order(); })
        .def("grad_accum", [](PyTrainer& p) { return p.t->grad_accum(); })
        .def("grad_seen", [](PyTrainer& p) { return p.t->grad_seen(); })
        .def("moments", [](PyTrainer& p, int which) { return p.t->moments(which); })
        .def("adam_steps", [](PyTrainer& p) { return p.t->adam_steps(); })
        .def("take_removed_ids", [](PyTrainer& p) { return p.t->take_removed_ids(); })
        .def("take_new_rows", [](PyTrainer& p) { return p.t->take_new_rows(); });

    // View order exactly as BlockTrainer draws it (trainer.cpp:250-252).
    m.def("view_sequence", [](uint64_t seed, uint32_t block_id, size_t n_views, size_t n_steps) {
        Rng rng(derive_seed(seed, block_id));
        std::vector<size_t> order(n_views);
        std::iota(order.begin(), order.end(), size_t{0});
        std::vector<size_t> seq;
        size_t cursor = 0;
        for (size_t s = 0; s < n_steps; ++s) {
            if (cursor == 0) rng.shuffle(order);
            seq.push_back(order[cursor]);
            cursor = (cursor + 1) % n_views;
        }
        return seq;
    });

    py::class_<Rng>(m, "Rng")
        .def(py::init<uint64_t>())
        .def("uniform", py::overload_cast<>(&Rng::uniform))
        .def("uniform_range", py::overload_cast<double, double>(&Rng::uniform))
        .def("uniform_index", &Rng::uniform_index)
        .def("normal", &Rng::normal)
        .def("next_u64", &Rng::next_u64)
        .def("random_unit_quat", [](Rng& r) { V4 q = r.random_unit_quat(); return std::array<double, 4>{q[0], q[1], q[2], q[3]}; });

    py::class_<SynthConfig>(m, "SynthConfig")
        .def(py::init<>())
        .def_readwrite("seed", &SynthConfig::seed).def_readwrite("gaussians", &SynthConfig::gaussians)
        .def_readwrite("cameras", &SynthConfig::cameras).def_readwrite("image_size", &SynthConfig::image_size)
        .def_readwrite("extent", &SynthConfig::extent).def_readwrite("sh_degree", &SynthConfig::sh_degree);
    py::class_<Scene>(m, "Scene")
        .def(py::init<>())
        .def_readwrite("views", &Scene::views)
        .def_readwrite("has_checkpoint", &Scene::has_checkpoint)
        .def_readwrite("checkpoint", &Scene::checkpoint)
        .def_readonly("ground_truth", &Scene::ground_truth)
        .def("images", [](const Scene& s) { py::list l; for (auto& im : s.images) l.append(image_np(im)); return l; })
        .def("set_images", [](Scene& s, std::vector<py::array_t<double>> ims) {
            s.images.clear(); for (auto& a : ims) s.images.push_back(make_image(a)); })
        .def("points", [](const Scene& s) {
            std::vector<float> p; std::vector<uint8_t> c;
            for (auto& q : s.points) { p.insert(p.end(), q.p, q.p + 3); c.insert(c.end(), q.rgb, q.rgb + 3); }
            const ssize_t n = static_cast<ssize_t>(s.points.size());
            return py::make_tuple(to_np(p, {n, 3}), to_np(c, {n, 3}));
        })
        .def("set_points", [](Scene& s, py::array_t<float, py::array::c_style | py::array::forcecast> p,
                              py::array_t<uint8_t, py::array::c_style | py::array::forcecast> c) {
            s.points.resize(p.shape(0));
            for (ssize_t i = 0; i < p.shape(0); ++i)
                for (int k = 0; k < 3; ++k) { s.points[i].p[k] = p.data()[3 * i + k]; s.points[i].rgb[k] = c.data()[3 * i + k]; }
        });
    m.def("generate_scene", &generate_scene);
    m.def("init_cloud_from_points", [](py::array_t<float, py::array::c_style | py::array::forcecast> p,
                                       py::array_t<uint8_t, py::array::c_style | py::array::forcecast> c, int sh, double op) {
        std::vector<ScenePoint> pts(p.shape(0));
        for (ssize_t i = 0; i < p.shape(0); ++i)
            for (int k = 0; k < 3; ++k) { pts[i].p[k] = p.data()[3 * i + k]; pts[i].rgb[k] = c.data()[3 * i + k]; }
        py::gil_scoped_release rel;
        return init_cloud_from_points(pts, sh, op);
    });

    m.def("split_and_assign", [](py::array_t<double, py::array::c_style | py::array::forcecast> pts, uint32_t k,
                                 std::vector<Camera> views, const Cloud& g, double scale, int vertical_axis, bool midpoint) {
        std::vector<V3> p(pts.shape(0));
        for (ssize_t i = 0; i < pts.shape(0); ++i) p[i] = V3{{pts.data()[3 * i], pts.data()[3 * i + 1], pts.data()[3 * i + 2]}};
        SplitOptions o{vertical_axis, midpoint};
        auto cores = split_recursive(p, k, o);
        BlockPartition part = expand_and_assign(cores, p, views, g, scale, o);
        py::dict d;
        auto boxes = [](const std::vector<Aabb>& bs) {
            std::vector<double> v;
            for (auto& b : bs) for (int a = 0; a < 3; ++a) { v.push_back(b.min[a]); }
            for (auto& b : bs) for (int a = 0; a < 3; ++a) { v.push_back(b.max[a]); }
            return v;
        };
        const ssize_t kk = static_cast<ssize_t>(k);
        auto core = boxes(part.core), exp = boxes(part.expanded);
        d["core_min"] = to_np(std::vector<double>(core.begin(), core.begin() + 3 * k), {kk, 3});
        d["core_max"] = to_np(std::vector<double>(core.begin() + 3 * k, core.end()), {kk, 3});
        d["exp_min"] = to_np(std::vector<double>(exp.begin(), exp.begin() + 3 * k), {kk, 3});
        d["exp_max"] = to_np(std::vector<double>(exp.begin() + 3 * k, exp.end()), {kk, 3});
        std::vector<std::vector<size_t>> core_pts;
        for (auto& c : cores) core_pts.push_back(c.point_indices);
        d["core_points"] = core_pts;
        d["block_points"] = part.block_points;
        d["block_views"] = part.block_views;
        d["block_gaussians"] = part.block_gaussians;
        d["shared"] = part.shared;
        return d;
    });

    py::class_<SessionOptions>(m, "SessionOptions")
        .def(py::init<>())
        .def_readwrite("consensus", &SessionOptions::consensus)
        .def_readwrite("rho", &SessionOptions::rho)
        .def_readwrite("total_iterations", &SessionOptions::total_iterations)
        .def_readwrite("nonshared_refresh", &SessionOptions::nonshared_refresh);
    py::class_<RoundDiagnostics>(m, "RoundDiagnostics")
        .def_readonly("iteration", &RoundDiagnostics::iteration)
        .def_readonly("primal_residual", &RoundDiagnostics::primal_residual)
        .def_readonly("dual_residual", &RoundDiagnostics::dual_residual)
        .def_readonly("rho", &RoundDiagnostics::rho)
        .def_readonly("max_disagreement", &RoundDiagnostics::max_disagreement)
        .def_readonly("dual_mean_linf", &RoundDiagnostics::dual_mean_linf)
        .def_readonly("mean_loss", &RoundDiagnostics::mean_loss)
        .def_readonly("shared_count", &RoundDiagnostics::shared_count)
        .def_readonly("global_count", &RoundDiagnostics::global_count);
    py::class_<ClusterPlan>(m, "ClusterPlan")
        .def_readonly("init_cloud", &ClusterPlan::init_cloud)
        .def_readonly("owners", &ClusterPlan::owners)
        .def("shard_ids", [](const ClusterPlan& p, uint32_t b) { return p.shards[b].initial.ids; })
        .def("shard_shared", [](const ClusterPlan& p, uint32_t b) { return p.shards[b].shared_ids; })
        .def("shard_views", [](const ClusterPlan& p, uint32_t b) { return p.shards[b].view_indices; })
        .def("blocks", [](const ClusterPlan& p) { return p.shards.size(); });
    // The plan keeps pointers into the scene's images: keep_alive ties them.
    m.def("plan_cluster", [](const Scene& s, uint32_t blocks, double scale, uint32_t holdout, const TrainerConfig& tc) {
        return plan_cluster(s, blocks, scale, holdout, tc, SplitOptions{});
    }, py::keep_alive<0, 1>());
    py::class_<RunResult>(m, "RunResult")
        .def_readonly("model", &RunResult::model)
        .def_readonly("rounds", &RunResult::rounds)
        .def_readonly("block_clouds", &RunResult::block_clouds);
    m.def("run_simulated", [](const ClusterPlan& plan, const TrainerConfig& tc, const SessionOptions& opt) {
        py::gil_scoped_release rel;
        return run_simulated(plan, tc, opt);
    });
    m.def("consensus_schedule", &consensus_schedule);
    m.def("master_ownership_round", [](std::map<uint64_t, std::vector<uint32_t>> owners,
                                       std::vector<std::vector<uint64_t>> removed,
                                       std::vector<std::vector<uint64_t>> added) {
        OwnershipRound r = master_ownership_round(owners, removed, added);
        py::dict d;
        d["reset"] = r.reset;
        d["unshared"] = r.unshared;
        d["dead"] = r.dead;
        d["shared_now"] = r.shared_now;
        d["owners"] = owners;
        return d;
    });
}
