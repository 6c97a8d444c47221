// ORACLE — TEST INFRASTRUCTURE ONLY (see orc.hpp). CPU FP64 restatement of
// /root/reference/proj/core/src/*.cpp. Compiled with -ffp-contract=off so the
// evaluation order written here is the one executed.
//
// Evaluation-order convention for the reference's Eigen expressions:
//   3-term dot products / matrix-vector rows: (a0*b0 + a1*b1) + a2*b2
//   quaternion norm: sqrt(((w*w + x*x) + y*y) + z*z)
//   matrix products: left-to-right over k.
#include "orc.hpp"

#include <atomic>
#include <thread>

#include <algorithm>
#include <numeric>

namespace orc {

// ---------------------------------------------------------------- math.hpp
double norm4(const V4& q) { return std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]); }
double norm3(const V3& v) { return std::sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]); }

V4 quat_normalized(const V4& q) {  // math.hpp:25-29
    const double n = norm4(q);
    if (n == 0.0) return V4{{1, 0, 0, 0}};
    return V4{{q[0] / n, q[1] / n, q[2] / n, q[3] / n}};
}

V4 quat_canonical(const V4& q) {  // math.hpp:32-34
    return q[0] < 0.0 ? V4{{-q[0], -q[1], -q[2], -q[3]}} : q;
}

M3 quat_to_rotation(const V4& q) {  // math.hpp:37-44
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    M3 r;
    r(0, 0) = 1 - 2 * (y * y + z * z); r(0, 1) = 2 * (x * y - w * z); r(0, 2) = 2 * (x * z + w * y);
    r(1, 0) = 2 * (x * y + w * z); r(1, 1) = 1 - 2 * (x * x + z * z); r(1, 2) = 2 * (y * z - w * x);
    r(2, 0) = 2 * (x * z - w * y); r(2, 1) = 2 * (y * z + w * x); r(2, 2) = 1 - 2 * (x * x + y * y);
    return r;
}

V4 rotation_to_quat(const M3& r) {  // math.hpp:48-69
    const double t = (r(0, 0) + r(1, 1)) + r(2, 2);
    V4 q;
    if (t > 0.0) {
        double s = std::sqrt(t + 1.0) * 2.0;
        q = V4{{0.25 * s, (r(2, 1) - r(1, 2)) / s, (r(0, 2) - r(2, 0)) / s, (r(1, 0) - r(0, 1)) / s}};
    } else if (r(0, 0) > r(1, 1) && r(0, 0) > r(2, 2)) {
        double s = std::sqrt(1.0 + r(0, 0) - r(1, 1) - r(2, 2)) * 2.0;
        q = V4{{(r(2, 1) - r(1, 2)) / s, 0.25 * s, (r(0, 1) + r(1, 0)) / s, (r(0, 2) + r(2, 0)) / s}};
    } else if (r(1, 1) > r(2, 2)) {
        double s = std::sqrt(1.0 + r(1, 1) - r(0, 0) - r(2, 2)) * 2.0;
        q = V4{{(r(0, 2) - r(2, 0)) / s, (r(0, 1) + r(1, 0)) / s, 0.25 * s, (r(1, 2) + r(2, 1)) / s}};
    } else {
        double s = std::sqrt(1.0 + r(2, 2) - r(0, 0) - r(1, 1)) * 2.0;
        q = V4{{(r(1, 0) - r(0, 1)) / s, (r(0, 2) + r(2, 0)) / s, (r(1, 2) + r(2, 1)) / s, 0.25 * s}};
    }
    return quat_canonical(quat_normalized(q));
}

uint64_t Rng::uniform_index(uint64_t n) {  // math.hpp:88-97
    uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v;
    do {
        v = gen_();
    } while (v >= limit);
    return v % n;
}

double Rng::normal() {  // math.hpp:100-114
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    double u1, u2;
    do {
        u1 = uniform();
    } while (u1 <= 0.0);
    u2 = uniform();
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = 2.0 * M_PI * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
}

V4 Rng::random_unit_quat() {  // math.hpp:116-119
    // Vec4(normal(), normal(), normal(), normal()): GCC 13 on x86-64
    // evaluates constructor arguments right to left (checked with this
    // container's g++), so the last component is drawn first.
    const double d = normal();
    const double c = normal();
    const double b = normal();
    const double a = normal();
    return quat_canonical(quat_normalized(V4{{a, b, c, d}}));
}

uint64_t fnv1a64(const void* data, size_t n, uint64_t seed) {  // math.hpp:138-146
    const auto* p = static_cast<const uint8_t*>(data);
    uint64_t h = seed;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

// -------------------------------------------------------------- camera.hpp
V3 Camera::to_camera(const V3& p) const {  // camera.hpp:28
    V3 o;
    for (int i = 0; i < 3; ++i) o[i] = ((R(i, 0) * p[0] + R(i, 1) * p[1]) + R(i, 2) * p[2]) + t[i];
    return o;
}

V3 Camera::center() const {  // camera.hpp:31
    V3 o;
    for (int i = 0; i < 3; ++i) o[i] = -((R(0, i) * t[0] + R(1, i) * t[1]) + R(2, i) * t[2]);
    return o;
}

V2 Camera::project(const V3& pc) const {  // camera.hpp:34-36
    return V2{fx * pc[0] / pc[2] + cx, fy * pc[1] / pc[2] + cy};
}

static V3 cross(const V3& a, const V3& b) {
    return V3{{a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]}};
}
static V3 normalized3(const V3& v) {
    const double n = norm3(v);
    return V3{{v[0] / n, v[1] / n, v[2] / n}};
}

Camera look_at(const V3& position, const V3& target, const V3& world_up, double fx, double fy,
               double cx, double cy, uint32_t w, uint32_t h) {  // camera.hpp:42-58
    const V3 forward = normalized3(V3{{target[0] - position[0], target[1] - position[1], target[2] - position[2]}});
    const V3 right = normalized3(cross(forward, world_up));
    const V3 down = cross(forward, right);
    M3 r;
    for (int k = 0; k < 3; ++k) {
        r(0, k) = right[k];
        r(1, k) = down[k];
        r(2, k) = forward[k];
    }
    Camera cam;
    cam.set_rotation_quat(rotation_to_quat(r));
    for (int i = 0; i < 3; ++i)
        cam.t[i] = -((cam.R(i, 0) * position[0] + cam.R(i, 1) * position[1]) + cam.R(i, 2) * position[2]);
    cam.fx = fx; cam.fy = fy; cam.cx = cx; cam.cy = cy;
    cam.width = w; cam.height = h;
    return cam;
}

// ---------------------------------------------------------------- cloud.cpp
size_t Cloud::find(uint64_t id) const {
    auto it = std::lower_bound(ids.begin(), ids.end(), id);
    if (it == ids.end() || *it != id) return npos;
    return static_cast<size_t>(it - ids.begin());
}

bool Cloud::check_invariants() const {
    const size_t n = ids.size();
    if (pos.size() != 3 * n || rot.size() != 4 * n || ls.size() != 3 * n ||
        feat.size() != n * static_cast<size_t>(fd) || op.size() != n)
        return false;
    for (size_t i = 1; i < n; ++i)
        if (ids[i] <= ids[i - 1]) return false;
    return true;
}

void Cloud::canonicalize_rotations() {  // cloud.cpp:82-85
    for (size_t i = 0; i < size(); ++i) {
        const V4 q = quat_canonical(quat_normalized(rotation(i)));
        for (int k = 0; k < 4; ++k) rot[4 * i + k] = q[k];
    }
}

void Cloud::push_row(const Cloud& s, size_t i) {
    ids.push_back(s.ids[i]);
    pos.insert(pos.end(), s.pos.begin() + 3 * i, s.pos.begin() + 3 * i + 3);
    rot.insert(rot.end(), s.rot.begin() + 4 * i, s.rot.begin() + 4 * i + 4);
    ls.insert(ls.end(), s.ls.begin() + 3 * i, s.ls.begin() + 3 * i + 3);
    feat.insert(feat.end(), s.feat.begin() + i * s.fd, s.feat.begin() + (i + 1) * s.fd);
    op.push_back(s.op[i]);
}

Cloud Cloud::subset(const std::vector<size_t>& idx) const {
    Cloud out(fd);
    for (size_t i : idx) out.push_row(*this, i);
    return out;
}

void Cloud::remove_indices(const std::vector<size_t>& idx) {  // cloud.cpp:33-57
    if (idx.empty()) return;
    std::vector<char> drop(size(), 0);
    for (size_t i : idx) drop[i] = 1;
    std::vector<size_t> keep;
    for (size_t r = 0; r < size(); ++r)
        if (!drop[r]) keep.push_back(r);
    *this = subset(keep);
}

void Cloud::sort_by_id() {
    std::vector<size_t> order(size());
    std::iota(order.begin(), order.end(), size_t{0});
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return ids[a] < ids[b]; });
    *this = subset(order);
}

Cloud slice_by_ids(const Cloud& c, const std::vector<uint64_t>& ids) {
    std::vector<size_t> idx;
    for (uint64_t id : ids) {
        const size_t i = c.find(id);
        if (i != Cloud::npos) idx.push_back(i);
    }
    return c.subset(idx);
}

size_t overwrite_by_ids(Cloud& dst, const Cloud& src) {
    if (dst.fd != src.fd) throw InvalidArgument("feature vector width mismatch");
    const int fd = dst.fd;
    size_t written = 0;
    for (size_t j = 0; j < src.size(); ++j) {
        const size_t i = dst.find(src.ids[j]);
        if (i == Cloud::npos) continue;
        for (int k = 0; k < 3; ++k) dst.pos[3 * i + k] = src.pos[3 * j + k];
        for (int k = 0; k < 4; ++k) dst.rot[4 * i + k] = src.rot[4 * j + k];
        for (int k = 0; k < 3; ++k) dst.ls[3 * i + k] = src.ls[3 * j + k];
        for (int k = 0; k < fd; ++k) dst.feat[i * fd + k] = src.feat[j * fd + k];
        dst.op[i] = src.op[j];
        ++written;
    }
    return written;
}

void erase_by_ids(Cloud& dst, const std::vector<uint64_t>& ids) {
    std::vector<size_t> idx;
    for (uint64_t id : ids) {
        const size_t i = dst.find(id);
        if (i != Cloud::npos) idx.push_back(i);
    }
    dst.remove_indices(idx);
}

void insert_rows(Cloud& dst, const Cloud& rows) {
    for (size_t j = 0; j < rows.size(); ++j) {
        if (dst.find(rows.ids[j]) != Cloud::npos) throw InvalidArgument("duplicate id on insert");
        dst.push_row(rows, j);
    }
    dst.sort_by_id();
}

Cloud zero_bundle(const std::vector<uint64_t>& ids, int fd) {
    Cloud c(fd);
    c.ids = ids;
    c.pos.assign(3 * ids.size(), 0.0);
    c.rot.assign(4 * ids.size(), 0.0);
    c.ls.assign(3 * ids.size(), 0.0);
    c.feat.assign(ids.size() * fd, 0.0);
    c.op.assign(ids.size(), 0.0);
    return c;
}

uint64_t cloud_checksum(const Cloud& c) {  // cloud.cpp:151-160
    uint64_t h = fnv1a64(c.ids.data(), c.ids.size() * sizeof(uint64_t));
    auto fold = [&h](const std::vector<double>& v) { h = fnv1a64(v.data(), v.size() * sizeof(double), h); };
    fold(c.pos);
    fold(c.rot);
    fold(c.ls);
    fold(c.feat);
    fold(c.op);
    return h;
}

M3 covariance_from_params(const V4& q, const V3& log_scale) {  // cloud.cpp:162-167
    const M3 r = quat_to_rotation(quat_normalized(q));
    const double s[3] = {std::exp(log_scale[0]), std::exp(log_scale[1]), std::exp(log_scale[2])};
    M3 m;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m(i, j) = r(i, j) * s[j];
    M3 sigma;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) sigma(i, j) = (m(i, 0) * m(j, 0) + m(i, 1) * m(j, 1)) + m(i, 2) * m(j, 2);
    return sigma;
}

V3 sh_color(const double* f, int fd, const V3& view_dir) {  // cloud.cpp:180-193
    V3 c{{kSh0 * f[0], kSh0 * f[1], kSh0 * f[2]}};
    if (fd >= kFeatureDimDeg1) {
        const V3 d = normalized3(view_dir);
        const double b0 = -kSh1 * d[1];
        const double b1 = kSh1 * d[2];
        const double b2 = -kSh1 * d[0];
        for (int ch = 0; ch < 3; ++ch) c[ch] += b0 * f[3 + 3 * ch] + b1 * f[4 + 3 * ch] + b2 * f[5 + 3 * ch];
    }
    return c;
}

// ------------------------------------------------------------- renderer.cpp
namespace {

// Integer conversion with the out-of-range case pinned (the reference's
// static_cast<int> of an out-of-range double is UB; both this oracle and the
// device kernel clamp to +-2^30 first, identical for every in-range value).
inline int to_int_clamped(double v) {
    if (v < -1073741824.0) return -1073741824;
    if (v > 1073741824.0) return 1073741824;
    return static_cast<int>(v);
}

PixelRect footprint(const V2& mean, double radius, uint32_t w, uint32_t h) {  // renderer.cpp:33-40
    PixelRect r;
    r.x0 = std::max(0, to_int_clamped(std::ceil(mean.x - radius)));
    r.x1 = std::min(static_cast<int>(w) - 1, to_int_clamped(std::floor(mean.x + radius)));
    r.y0 = std::max(0, to_int_clamped(std::ceil(mean.y - radius)));
    r.y1 = std::min(static_cast<int>(h) - 1, to_int_clamped(std::floor(mean.y + radius)));
    return r;
}

double max_eigenvalue_2x2(const M2& m) {  // renderer.cpp:22-26
    const double mid = 0.5 * (m(0, 0) + m(1, 1));
    const double det = m(0, 0) * m(1, 1) - m(0, 1) * m(1, 0);
    return mid + std::sqrt(std::max(0.0, mid * mid - det));
}

// renderer.cpp:14-20
void projection_jacobian(const Camera& cam, const V3& p, double j[2][3]) {
    const double z = p[2], iz = 1.0 / z, iz2 = iz * iz;
    j[0][0] = cam.fx * iz; j[0][1] = 0; j[0][2] = -cam.fx * p[0] * iz2;
    j[1][0] = 0; j[1][1] = cam.fy * iz; j[1][2] = -cam.fy * p[1] * iz2;
}

}  // namespace

// project_gaussian (renderer.cpp:121-134) + the Splat fields of
// project_cloud (renderer.cpp:73-83).
Projected project_row(const Cloud& c, size_t i, const Camera& cam, const RenderConfig& cfg) {
    Projected out;
    const V3 pos = c.position(i);
    const M3 sigma = covariance_from_params(c.rotation(i), c.log_scale(i));
    const V3 pc = cam.to_camera(pos);
    if (pc[2] <= cfg.near_plane) return out;
    out.depth = pc[2];
    out.mean2d = cam.project(pc);
    double j[2][3];
    projection_jacobian(cam, pc, j);
    double a[2][3], tt[2][3];
    for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k) a[r][k] = (j[r][0] * cam.R(0, k) + j[r][1] * cam.R(1, k)) + j[r][2] * cam.R(2, k);
    for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k) tt[r][k] = (a[r][0] * sigma(0, k) + a[r][1] * sigma(1, k)) + a[r][2] * sigma(2, k);
    for (int r = 0; r < 2; ++r)
        for (int s = 0; s < 2; ++s) {
            const double v = (tt[r][0] * a[s][0] + tt[r][1] * a[s][1]) + tt[r][2] * a[s][2];
            out.cov2d(r, s) = v + (r == s ? cfg.dilation : cfg.dilation * 0.0);
        }
    const double radius = cfg.sigma_extent * std::sqrt(max_eigenvalue_2x2(out.cov2d));
    out.rect = footprint(out.mean2d, radius, cam.width, cam.height);
    if (out.rect.x0 > out.rect.x1 || out.rect.y0 > out.rect.y1) return out;
    out.visible = true;
    const M2& cv = out.cov2d;
    const double det = cv(0, 0) * cv(1, 1) - cv(0, 1) * cv(1, 0);
    out.minv(0, 0) = cv(1, 1) / det;
    out.minv(0, 1) = -cv(0, 1) / det;
    out.minv(1, 0) = -cv(1, 0) / det;
    out.minv(1, 1) = cv(0, 0) / det;
    const V3 cc = cam.center();
    const V3 dir{{pos[0] - cc[0], pos[1] - cc[1], pos[2] - cc[2]}};
    out.color = sh_color(c.feat.data() + i * c.fd, c.fd, dir);
    out.opacity = c.opacity(i);
    return out;
}

std::vector<size_t> depth_order(const std::vector<Projected>& pr) {  // renderer.cpp:86-89
    std::vector<size_t> order;
    for (size_t i = 0; i < pr.size(); ++i)
        if (pr[i].visible) order.push_back(i);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        if (pr[a].depth != pr[b].depth) return pr[a].depth < pr[b].depth;
        return a < b;
    });
    return order;
}

namespace {

struct Bins { std::vector<uint32_t> offsets, entries; };

// renderer.cpp:99-117; entries hold positions in `order`.
Bins bin_splats(const std::vector<Projected>& pr, const std::vector<size_t>& order, uint32_t w, uint32_t h) {
    Bins b;
    const size_t pixels = size_t(w) * h;
    b.offsets.assign(pixels + 1, 0);
    for (size_t si : order) {
        const PixelRect& r = pr[si].rect;
        for (int y = r.y0; y <= r.y1; ++y)
            for (int x = r.x0; x <= r.x1; ++x) ++b.offsets[size_t(y) * w + x + 1];
    }
    for (size_t i = 1; i < b.offsets.size(); ++i) b.offsets[i] += b.offsets[i - 1];
    b.entries.resize(b.offsets.back());
    std::vector<uint32_t> cursor(b.offsets.begin(), b.offsets.end() - 1);
    for (uint32_t k = 0; k < order.size(); ++k) {
        const PixelRect& r = pr[order[k]].rect;
        for (int y = r.y0; y <= r.y1; ++y)
            for (int x = r.x0; x <= r.x1; ++x) b.entries[cursor[size_t(y) * w + x]++] = k;
    }
    return b;
}

// renderer.cpp:53-59
inline double splat_weight(const Projected& s, int px, int py, V2& d) {
    d = V2{px - s.mean2d.x, py - s.mean2d.y};
    const double q = d.x * (s.minv(0, 0) * d.x + s.minv(0, 1) * d.y) + d.y * (s.minv(1, 0) * d.x + s.minv(1, 1) * d.y);
    return std::exp(-0.5 * q);
}

}  // namespace

RenderOut render(const Cloud& c, const Camera& cam, const RenderConfig& cfg) {  // renderer.cpp:150-183
    RenderOut out;
    out.color = Image(cam.width, cam.height);
    const size_t pixels = out.color.pixel_count();
    out.transmittance.assign(pixels, 1.0);
    out.contributors.assign(pixels, 0);
    std::vector<Projected> pr(c.size());
    for (size_t i = 0; i < c.size(); ++i) pr[i] = project_row(c, i, cam, cfg);
    const std::vector<size_t> order = depth_order(pr);
    const Bins bins = bin_splats(pr, order, cam.width, cam.height);
    for (uint32_t y = 0; y < cam.height; ++y)
        for (uint32_t x = 0; x < cam.width; ++x) {
            const size_t px = size_t(y) * cam.width + x;
            double t = 1.0;
            double col[3] = {0, 0, 0};
            uint32_t n = 0;
            for (uint32_t e = bins.offsets[px]; e < bins.offsets[px + 1]; ++e) {
                if (t < cfg.transmittance_stop) break;
                const Projected& s = pr[order[bins.entries[e]]];
                V2 d;
                const double g = splat_weight(s, int(x), int(y), d);
                const double alpha = std::min(s.opacity * g, cfg.alpha_clamp);
                for (int ch = 0; ch < 3; ++ch) col[ch] += s.color[ch] * (alpha * t);
                t *= 1.0 - alpha;
                ++n;
            }
            for (int ch = 0; ch < 3; ++ch) out.color.at(x, y, ch) = col[ch] + t * cfg.background[ch];
            out.transmittance[px] = t;
            out.contributors[px] = n;
        }
    return out;
}

double loss_value(const Image& r, const Image& gt, double lambda) {  // renderer.cpp:185-192
    if (r.width != gt.width || r.height != gt.height) throw InvalidArgument("image dimension mismatch");
    double l1 = 0;
    for (size_t i = 0; i < r.data.size(); ++i) l1 += std::abs(r.data[i] - gt.data[i]);
    l1 /= static_cast<double>(r.data.size());
    return l1 + lambda * (1.0 - ssim(r, gt));
}

void Grads::resize_for(const Cloud& c) {
    pos.assign(3 * c.size(), 0.0);
    rot.assign(4 * c.size(), 0.0);
    ls.assign(3 * c.size(), 0.0);
    feat.assign(c.size() * c.fd, 0.0);
    op.assign(c.size(), 0.0);
}

namespace {
void rotation_quat_jacobian(const V4& q, M3 dr[4]) {  // renderer.cpp:198-213
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double d0[9] = {0, -z, y, z, 0, -x, -y, x, 0};
    const double d1[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
    const double d2[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
    const double d3[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
    const double* src[4] = {d0, d1, d2, d3};
    for (int k = 0; k < 4; ++k)
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) dr[k](i, j) = src[k][3 * i + j] * 2.0;
}
}  // namespace

BackwardOut render_backward(const Cloud& c, const Camera& cam, const Image& gt, const RenderConfig& cfg) {
    if (gt.width != cam.width || gt.height != cam.height) throw InvalidArgument("image dimension mismatch");
    BackwardOut out;
    out.grads.resize_for(c);
    out.screen_grad_norm.assign(c.size(), 0.0);
    out.visible.assign(c.size(), 0);

    std::vector<Projected> pr(c.size());
    for (size_t i = 0; i < c.size(); ++i) pr[i] = project_row(c, i, cam, cfg);
    const std::vector<size_t> order = depth_order(pr);
    const Bins bins = bin_splats(pr, order, cam.width, cam.height);
    const size_t pixels = size_t(cam.width) * cam.height;

    // renderer.cpp:233-257
    out.rendered = Image(cam.width, cam.height);
    std::vector<double> t_final(pixels, 1.0);
    std::vector<uint32_t> processed(pixels, 0);
    for (uint32_t y = 0; y < cam.height; ++y)
        for (uint32_t x = 0; x < cam.width; ++x) {
            const size_t px = size_t(y) * cam.width + x;
            double t = 1.0;
            double col[3] = {0, 0, 0};
            uint32_t n = 0;
            for (uint32_t e = bins.offsets[px]; e < bins.offsets[px + 1]; ++e) {
                if (t < cfg.transmittance_stop) break;
                const Projected& s = pr[order[bins.entries[e]]];
                V2 d;
                const double g = splat_weight(s, int(x), int(y), d);
                const double alpha = std::min(s.opacity * g, cfg.alpha_clamp);
                for (int ch = 0; ch < 3; ++ch) col[ch] += s.color[ch] * (alpha * t);
                t *= 1.0 - alpha;
                ++n;
            }
            for (int ch = 0; ch < 3; ++ch) out.rendered.at(x, y, ch) = col[ch] + t * cfg.background[ch];
            t_final[px] = t;
            processed[px] = n;
        }

    // renderer.cpp:259-272
    Image dssim_dx;
    out.ssim = ssim_with_gradient(out.rendered, gt, dssim_dx);
    double l1 = 0;
    out.dl_dc = Image(cam.width, cam.height);
    const double inv_count = 1.0 / static_cast<double>(out.rendered.data.size());
    for (size_t i = 0; i < out.rendered.data.size(); ++i) {
        const double diff = out.rendered.data[i] - gt.data[i];
        l1 += std::abs(diff);
        const double sign = diff > 0 ? 1.0 : (diff < 0 ? -1.0 : 0.0);
        out.dl_dc.data[i] = sign * inv_count - cfg.lambda * dssim_dx.data[i];
    }
    out.l1 = l1 * inv_count;
    out.loss = out.l1 + cfg.lambda * (1.0 - out.ssim);

    // renderer.cpp:274-311
    const size_t ns = order.size();
    out.order = order;
    out.g_mean.assign(2 * ns, 0.0);
    out.g_cov.assign(4 * ns, 0.0);
    out.g_color.assign(3 * ns, 0.0);
    out.g_opacity.assign(ns, 0.0);
    for (uint32_t y = 0; y < cam.height; ++y)
        for (uint32_t x = 0; x < cam.width; ++x) {
            const size_t px = size_t(y) * cam.width + x;
            const uint32_t n = processed[px];
            if (n == 0) continue;
            const double dldc[3] = {out.dl_dc.at(x, y, 0), out.dl_dc.at(x, y, 1), out.dl_dc.at(x, y, 2)};
            double t_run = t_final[px];
            double suffix[3] = {t_run * cfg.background[0], t_run * cfg.background[1], t_run * cfg.background[2]};
            const uint32_t base = bins.offsets[px];
            for (uint32_t k = n; k-- > 0;) {
                const uint32_t si = bins.entries[base + k];
                const Projected& s = pr[order[si]];
                V2 d;
                const double g = splat_weight(s, int(x), int(y), d);
                const double alpha = std::min(s.opacity * g, cfg.alpha_clamp);
                const double t_before = t_run / (1.0 - alpha);
                for (int ch = 0; ch < 3; ++ch) out.g_color[3 * si + ch] += dldc[ch] * (alpha * t_before);
                double dl_dalpha = 0;
                {
                    double terms[3];
                    for (int ch = 0; ch < 3; ++ch) terms[ch] = dldc[ch] * (s.color[ch] * t_before - suffix[ch] / (1.0 - alpha));
                    dl_dalpha = (terms[0] + terms[1]) + terms[2];
                }
                if (s.opacity * g < cfg.alpha_clamp) {
                    const double dl_dg = dl_dalpha * s.opacity;
                    const double md[2] = {s.minv(0, 0) * d.x + s.minv(0, 1) * d.y, s.minv(1, 0) * d.x + s.minv(1, 1) * d.y};
                    out.g_mean[2 * si] += dl_dg * g * md[0];
                    out.g_mean[2 * si + 1] += dl_dg * g * md[1];
                    const double h = 0.5 * dl_dg * g;
                    out.g_cov[4 * si + 0] += h * (md[0] * md[0]);
                    out.g_cov[4 * si + 1] += h * (md[0] * md[1]);
                    out.g_cov[4 * si + 2] += h * (md[1] * md[0]);
                    out.g_cov[4 * si + 3] += h * (md[1] * md[1]);
                    out.g_opacity[si] += dl_dalpha * g;
                }
                for (int ch = 0; ch < 3; ++ch) suffix[ch] += s.color[ch] * (alpha * t_before);
                t_run = t_before;
            }
        }

    // renderer.cpp:313-403 — fold to the parameter arrays.
    const V3 cc = cam.center();
    const int fdim = c.fd;
    for (size_t si = 0; si < ns; ++si) {
        const Projected& s = pr[order[si]];
        const size_t i = order[si];
        out.visible[i] = 1;
        const V3 pos = c.position(i);
        const V3 pcam = cam.to_camera(pos);
        const double z = pcam[2], iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;

        const double o = s.opacity;
        out.grads.op[i] += out.g_opacity[si] * o * (1.0 - o);

        const double* gc = &out.g_color[3 * si];
        for (int ch = 0; ch < 3; ++ch) out.grads.feat[i * fdim + ch] += kSh0 * gc[ch];
        double g_pos_dir[3] = {0, 0, 0};
        if (fdim >= kFeatureDimDeg1) {
            const V3 u{{pos[0] - cc[0], pos[1] - cc[1], pos[2] - cc[2]}};
            const double un = norm3(u);
            const double dir[3] = {u[0] / un, u[1] / un, u[2] / un};
            const double b0 = -kSh1 * dir[1], b1 = kSh1 * dir[2], b2 = -kSh1 * dir[0];
            double g_dir[3] = {0, 0, 0};
            const double* f = c.feat.data() + i * fdim;
            for (int ch = 0; ch < 3; ++ch) {
                out.grads.feat[i * fdim + 3 + 3 * ch] += b0 * gc[ch];
                out.grads.feat[i * fdim + 4 + 3 * ch] += b1 * gc[ch];
                out.grads.feat[i * fdim + 5 + 3 * ch] += b2 * gc[ch];
                g_dir[0] += gc[ch] * (f[5 + 3 * ch] * -kSh1);
                g_dir[1] += gc[ch] * (f[3 + 3 * ch] * -kSh1);
                g_dir[2] += gc[ch] * (f[4 + 3 * ch] * kSh1);
            }
            const double dd = dir[0] * g_dir[0] + dir[1] * g_dir[1] + dir[2] * g_dir[2];
            for (int k = 0; k < 3; ++k) g_pos_dir[k] = (g_dir[k] - dir[k] * dd) / un;
        }

        const double gm[2] = {out.g_mean[2 * si], out.g_mean[2 * si + 1]};
        out.screen_grad_norm[i] += std::sqrt((gm[0] * cam.width * 0.5) * (gm[0] * cam.width * 0.5) +
                                             (gm[1] * cam.height * 0.5) * (gm[1] * cam.height * 0.5));

        double g_pcam[3] = {gm[0] * cam.fx * iz, gm[1] * cam.fy * iz,
                            -gm[0] * cam.fx * pcam[0] * iz2 - gm[1] * cam.fy * pcam[1] * iz2};

        double gcov[2][2] = {{out.g_cov[4 * si], out.g_cov[4 * si + 1]}, {out.g_cov[4 * si + 2], out.g_cov[4 * si + 3]}};
        double j[2][3], a[2][3];
        projection_jacobian(cam, pcam, j);
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k) a[r][k] = (j[r][0] * cam.R(0, k) + j[r][1] * cam.R(1, k)) + j[r][2] * cam.R(2, k);
        const M3 sigma = covariance_from_params(c.rotation(i), c.log_scale(i));
        // g_sigma = a^T gcov a
        double at_g[3][2];
        for (int r = 0; r < 3; ++r)
            for (int s2 = 0; s2 < 2; ++s2) at_g[r][s2] = a[0][r] * gcov[0][s2] + a[1][r] * gcov[1][s2];
        M3 g_sigma;
        for (int r = 0; r < 3; ++r)
            for (int k = 0; k < 3; ++k) g_sigma(r, k) = at_g[r][0] * a[0][k] + at_g[r][1] * a[1][k];
        // g_a = 2 gcov a sigma
        double ga0[2][3], g_a[2][3], g_j[2][3];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k) ga0[r][k] = 2.0 * (gcov[r][0] * a[0][k] + gcov[r][1] * a[1][k]);
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k) g_a[r][k] = (ga0[r][0] * sigma(0, k) + ga0[r][1] * sigma(1, k)) + ga0[r][2] * sigma(2, k);
        // g_j = g_a R^T
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k) g_j[r][k] = (g_a[r][0] * cam.R(k, 0) + g_a[r][1] * cam.R(k, 1)) + g_a[r][2] * cam.R(k, 2);

        g_pcam[0] += g_j[0][2] * (-cam.fx * iz2);
        g_pcam[1] += g_j[1][2] * (-cam.fy * iz2);
        g_pcam[2] += g_j[0][0] * (-cam.fx * iz2) + g_j[1][1] * (-cam.fy * iz2) +
                     g_j[0][2] * (2.0 * cam.fx * pcam[0] * iz3) + g_j[1][2] * (2.0 * cam.fy * pcam[1] * iz3);

        for (int k = 0; k < 3; ++k)
            out.grads.pos[3 * i + k] += ((cam.R(0, k) * g_pcam[0] + cam.R(1, k) * g_pcam[1]) + cam.R(2, k) * g_pcam[2]) + g_pos_dir[k];

        const V4 q_raw = c.rotation(i);
        const V4 q_hat = quat_normalized(q_raw);
        const M3 r = quat_to_rotation(q_hat);
        const V3 lsc = c.log_scale(i);
        const double sc[3] = {std::exp(lsc[0]), std::exp(lsc[1]), std::exp(lsc[2])};
        M3 m, g_m, g_r;
        for (int a1 = 0; a1 < 3; ++a1)
            for (int b1 = 0; b1 < 3; ++b1) m(a1, b1) = r(a1, b1) * sc[b1];
        for (int a1 = 0; a1 < 3; ++a1)
            for (int b1 = 0; b1 < 3; ++b1)
                g_m(a1, b1) = 2.0 * ((g_sigma(a1, 0) * m(0, b1) + g_sigma(a1, 1) * m(1, b1)) + g_sigma(a1, 2) * m(2, b1));
        for (int a1 = 0; a1 < 3; ++a1)
            for (int b1 = 0; b1 < 3; ++b1) g_r(a1, b1) = g_m(a1, b1) * sc[b1];
        for (int k = 0; k < 3; ++k) {
            const double rt_gm_kk = (r(0, k) * g_m(0, k) + r(1, k) * g_m(1, k)) + r(2, k) * g_m(2, k);
            out.grads.ls[3 * i + k] += rt_gm_kk * sc[k];
        }
        M3 dr[4];
        rotation_quat_jacobian(q_hat, dr);
        double g_qhat[4];
        for (int k = 0; k < 4; ++k) {
            double acc = 0;
            for (int a1 = 0; a1 < 3; ++a1)
                for (int b1 = 0; b1 < 3; ++b1) acc += g_r(a1, b1) * dr[k](a1, b1);
            g_qhat[k] = acc;
        }
        const double qn = norm4(q_raw);
        const double proj = ((q_hat[0] * g_qhat[0] + q_hat[1] * g_qhat[1]) + q_hat[2] * g_qhat[2]) + q_hat[3] * g_qhat[3];
        for (int k = 0; k < 4; ++k) out.grads.rot[4 * i + k] += (g_qhat[k] - q_hat[k] * proj) / qn;
    }
    return out;
}

// ----------------------------------------------------------------- ssim.cpp
namespace {
constexpr double kC1 = 0.01 * 0.01;
constexpr double kC2 = 0.03 * 0.03;
constexpr int kHalf = kSsimWindow / 2;

struct Plane {
    uint32_t w = 0, h = 0;
    std::vector<double> v;
    Plane() = default;
    Plane(uint32_t w_, uint32_t h_) : w(w_), h(h_), v(size_t(w_) * h_, 0.0) {}
    double& at(uint32_t x, uint32_t y) { return v[size_t(y) * w + x]; }
    double at(uint32_t x, uint32_t y) const { return v[size_t(y) * w + x]; }
};

Plane channel_plane(const Image& img, int c) {
    Plane p(img.width, img.height);
    for (uint32_t y = 0; y < img.height; ++y)
        for (uint32_t x = 0; x < img.width; ++x) p.at(x, y) = img.at(x, y, c);
    return p;
}

Plane blur_valid(const Plane& in, const std::vector<double>& k) {  // ssim.cpp:34-50
    Plane horiz(in.w - 2 * kHalf, in.h);
    for (uint32_t y = 0; y < in.h; ++y)
        for (uint32_t x = 0; x < horiz.w; ++x) {
            double s = 0;
            for (int t = 0; t < kSsimWindow; ++t) s += k[t] * in.at(x + t, y);
            horiz.at(x, y) = s;
        }
    Plane out(horiz.w, in.h - 2 * kHalf);
    for (uint32_t y = 0; y < out.h; ++y)
        for (uint32_t x = 0; x < out.w; ++x) {
            double s = 0;
            for (int t = 0; t < kSsimWindow; ++t) s += k[t] * horiz.at(x, y + t);
            out.at(x, y) = s;
        }
    return out;
}

Plane spread_full(const Plane& in, const std::vector<double>& k, uint32_t fw, uint32_t fh) {  // ssim.cpp:54-69
    Plane vert(in.w, fh);
    for (uint32_t y = 0; y < in.h; ++y)
        for (uint32_t x = 0; x < in.w; ++x) {
            const double v = in.at(x, y);
            for (int t = 0; t < kSsimWindow; ++t) vert.at(x, y + t) += k[t] * v;
        }
    Plane out(fw, fh);
    for (uint32_t y = 0; y < fh; ++y)
        for (uint32_t x = 0; x < in.w; ++x) {
            const double v = vert.at(x, y);
            for (int t = 0; t < kSsimWindow; ++t) out.at(x + t, y) += k[t] * v;
        }
    return out;
}

struct ChannelStats { Plane mu_x, mu_y, sx2, sy2, sxy, map; };

ChannelStats channel_ssim(const Plane& x, const Plane& y, const std::vector<double>& k) {  // ssim.cpp:75-103
    ChannelStats s;
    s.mu_x = blur_valid(x, k);
    s.mu_y = blur_valid(y, k);
    Plane x2(x.w, x.h), y2(x.w, x.h), xy(x.w, x.h);
    for (size_t i = 0; i < x.v.size(); ++i) {
        x2.v[i] = x.v[i] * x.v[i];
        y2.v[i] = y.v[i] * y.v[i];
        xy.v[i] = x.v[i] * y.v[i];
    }
    s.sx2 = blur_valid(x2, k);
    s.sy2 = blur_valid(y2, k);
    s.sxy = blur_valid(xy, k);
    s.map = Plane(s.mu_x.w, s.mu_x.h);
    for (size_t i = 0; i < s.map.v.size(); ++i) {
        const double mx = s.mu_x.v[i], my = s.mu_y.v[i];
        const double vx = s.sx2.v[i] - mx * mx, vy = s.sy2.v[i] - my * my, cxy = s.sxy.v[i] - mx * my;
        s.sx2.v[i] = vx;
        s.sy2.v[i] = vy;
        s.sxy.v[i] = cxy;
        const double n1 = 2 * mx * my + kC1, n2 = 2 * cxy + kC2;
        const double d1 = mx * mx + my * my + kC1, d2 = vx + vy + kC2;
        s.map.v[i] = (n1 * n2) / (d1 * d2);
    }
    return s;
}

void check_dims(const Image& x, const Image& y) {
    if (x.width != y.width || x.height != y.height) throw InvalidArgument("image dimension mismatch");
}
}  // namespace

std::vector<double> ssim_window_1d() {  // ssim.cpp:112-122
    std::vector<double> k(kSsimWindow);
    double sum = 0;
    for (int i = 0; i < kSsimWindow; ++i) {
        const double d = i - kHalf;
        k[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
        sum += k[i];
    }
    for (double& v : k) v /= sum;
    return k;
}

double ssim(const Image& x, const Image& y) {  // ssim.cpp:124-136
    check_dims(x, y);
    if (x.width < kSsimWindow || x.height < kSsimWindow) return 1.0;
    const auto k = ssim_window_1d();
    double total = 0;
    size_t count = 0;
    for (int c = 0; c < 3; ++c) {
        const ChannelStats s = channel_ssim(channel_plane(x, c), channel_plane(y, c), k);
        for (double v : s.map.v) total += v;
        count += s.map.v.size();
    }
    return total / static_cast<double>(count);
}

double ssim_with_gradient(const Image& x, const Image& y, Image& dx) {  // ssim.cpp:138-185
    check_dims(x, y);
    dx = Image(x.width, x.height, 0.0);
    if (x.width < kSsimWindow || x.height < kSsimWindow) return 1.0;
    const auto k = ssim_window_1d();
    double total = 0;
    size_t count = 0;
    for (int c = 0; c < 3; ++c) {
        const Plane px = channel_plane(x, c), py = channel_plane(y, c);
        const ChannelStats s = channel_ssim(px, py, k);
        const size_t n = s.map.v.size();
        for (double v : s.map.v) total += v;
        count += n;
        Plane f1(s.map.w, s.map.h), f2(s.map.w, s.map.h), f3(s.map.w, s.map.h);
        for (size_t i = 0; i < n; ++i) {
            const double mx = s.mu_x.v[i], my = s.mu_y.v[i];
            const double vx = s.sx2.v[i], vy = s.sy2.v[i], cxy = s.sxy.v[i];
            const double n1 = 2 * mx * my + kC1, n2 = 2 * cxy + kC2;
            const double d1 = mx * mx + my * my + kC1, d2 = vx + vy + kC2;
            const double denom = d1 * d2;
            const double sv = (n1 * n2) / denom;
            const double a = 2 * my * n2 / denom - sv * 2 * mx / d1;
            const double b = -sv / d2;
            const double cc = 2 * n1 / denom;
            f1.v[i] = a - 2 * mx * b - my * cc;
            f2.v[i] = 2 * b;
            f3.v[i] = cc;
        }
        const Plane g1 = spread_full(f1, k, x.width, x.height);
        const Plane g2 = spread_full(f2, k, x.width, x.height);
        const Plane g3 = spread_full(f3, k, x.width, x.height);
        for (uint32_t yy = 0; yy < x.height; ++yy)
            for (uint32_t xx = 0; xx < x.width; ++xx)
                dx.at(xx, yy, c) = g1.at(xx, yy) + px.at(xx, yy) * g2.at(xx, yy) + py.at(xx, yy) * g3.at(xx, yy);
    }
    const double inv = 1.0 / static_cast<double>(count);
    for (double& v : dx.data) v *= inv;
    return total * inv;
}

// ----------------------------------------------------------------- admm.cpp
double penalty_loss_and_grad(const Cloud& c, const std::vector<size_t>& idx, const Cloud& z,
                             const Cloud& u, const Penalties& rho, Grads& g) {
    if (z.size() != idx.size() || u.size() != idx.size()) throw InvalidArgument("id misalignment");
    if (z.fd != c.fd || u.fd != c.fd) throw InvalidArgument("feature vector width mismatch");
    const int fd = c.fd;
    double loss = 0;
    for (size_t j = 0; j < idx.size(); ++j) {
        const size_t i = idx[j];
        if (c.ids[i] != z.ids[j] || z.ids[j] != u.ids[j]) throw InvalidArgument("id misalignment");
        auto acc = [&loss](double r, double x, double zv, double uv, double* gg) {
            const double d = x - zv + uv;
            loss += 0.5 * r * d * d;
            *gg += r * d;
        };
        for (int k = 0; k < 3; ++k) acc(rho.rho_p, c.pos[3 * i + k], z.pos[3 * j + k], u.pos[3 * j + k], &g.pos[3 * i + k]);
        for (int k = 0; k < 4; ++k) acc(rho.rho_q, c.rot[4 * i + k], z.rot[4 * j + k], u.rot[4 * j + k], &g.rot[4 * i + k]);
        for (int k = 0; k < 3; ++k) acc(rho.rho_s, c.ls[3 * i + k], z.ls[3 * j + k], u.ls[3 * j + k], &g.ls[3 * i + k]);
        for (int k = 0; k < fd; ++k) acc(rho.rho_f, c.feat[i * fd + k], z.feat[j * fd + k], u.feat[j * fd + k], &g.feat[i * fd + k]);
        acc(rho.rho_o, c.op[i], z.op[j], u.op[j], &g.op[i]);
    }
    return loss;
}

namespace {
struct Contributor { uint32_t block_id; const Cloud* cloud; size_t row; };
std::map<uint64_t, std::vector<Contributor>> gather(const std::vector<Contribution>& locals) {  // admm.cpp:56-67
    std::vector<Contribution> ordered = locals;
    std::sort(ordered.begin(), ordered.end(), [](const Contribution& a, const Contribution& b) { return a.block_id < b.block_id; });
    std::map<uint64_t, std::vector<Contributor>> owners;
    for (const Contribution& bc : ordered)
        for (size_t r = 0; r < bc.params->size(); ++r) owners[bc.params->ids[r]].push_back({bc.block_id, bc.params, r});
    return owners;
}
}  // namespace

Cloud consensus_average(const std::vector<Contribution>& locals, bool over_relaxed, const Cloud& z_prev,
                        double alpha, std::vector<uint64_t>* flipped_ids) {  // admm.cpp:71-127
    if (locals.empty()) throw InvalidArgument("no block contributions");
    const int fd = locals[0].params->fd;
    for (const Contribution& bc : locals)
        if (bc.params->fd != fd) throw InvalidArgument("feature vector width mismatch");
    const double a = over_relaxed ? alpha : 1.0;
    const auto owners = gather(locals);
    Cloud z(fd);
    std::vector<double> fs(fd);
    for (const auto& [id, who] : owners) {
        const size_t zp = z_prev.find(id);
        const bool blend = zp != Cloud::npos;
        auto rv = [&](double x, double prev) { return blend ? relaxed_value(x, prev, a) : x; };
        double pos[3] = {0, 0, 0}, ls[3] = {0, 0, 0}, rot[4] = {0, 0, 0, 0}, op = 0;
        std::fill(fs.begin(), fs.end(), 0.0);
        V4 q_ref;
        bool flipped = false;
        for (size_t c = 0; c < who.size(); ++c) {
            const Cloud& src = *who[c].cloud;
            const size_t r = who[c].row;
            V4 q = src.rotation(r);
            if (c == 0) {
                q_ref = q;
            } else {
                const double dot = ((q[0] * q_ref[0] + q[1] * q_ref[1]) + q[2] * q_ref[2]) + q[3] * q_ref[3];
                if (dot < 0.0) {
                    for (int k = 0; k < 4; ++k) q[k] = -q[k];
                    flipped = true;
                }
            }
            for (int k = 0; k < 3; ++k) {
                pos[k] += rv(src.pos[3 * r + k], blend ? z_prev.pos[3 * zp + k] : 0.0);
                ls[k] += rv(src.ls[3 * r + k], blend ? z_prev.ls[3 * zp + k] : 0.0);
            }
            for (int k = 0; k < 4; ++k) rot[k] += rv(q[k], blend ? z_prev.rot[4 * zp + k] : 0.0);
            for (int k = 0; k < fd; ++k) fs[k] += rv(src.feat[r * fd + k], blend ? z_prev.feat[zp * fd + k] : 0.0);
            op += rv(src.op[r], blend ? z_prev.op[zp] : 0.0);
        }
        const double inv = 1.0 / static_cast<double>(who.size());
        z.ids.push_back(id);
        for (int k = 0; k < 3; ++k) z.pos.push_back(pos[k] * inv);
        for (int k = 0; k < 4; ++k) z.rot.push_back(rot[k] * inv);
        for (int k = 0; k < 3; ++k) z.ls.push_back(ls[k] * inv);
        for (int k = 0; k < fd; ++k) z.feat.push_back(fs[k] * inv);
        z.op.push_back(op * inv);
        if (flipped && flipped_ids) flipped_ids->push_back(id);
    }
    return z;
}

void dual_update(Cloud& u, const Cloud& x_hat, const Cloud& z) {  // admm.cpp:129-145
    if (u.ids != x_hat.ids) throw InvalidArgument("id misalignment");
    const int fd = u.fd;
    for (size_t j = 0; j < u.size(); ++j) {
        const size_t zi = z.find(u.ids[j]);
        if (zi == Cloud::npos) throw InvalidArgument("id missing from consensus model");
        for (int k = 0; k < 3; ++k) {
            u.pos[3 * j + k] += x_hat.pos[3 * j + k] - z.pos[3 * zi + k];
            u.ls[3 * j + k] += x_hat.ls[3 * j + k] - z.ls[3 * zi + k];
        }
        for (int k = 0; k < 4; ++k) u.rot[4 * j + k] += x_hat.rot[4 * j + k] - z.rot[4 * zi + k];
        for (int k = 0; k < fd; ++k) u.feat[j * fd + k] += x_hat.feat[j * fd + k] - z.feat[zi * fd + k];
        u.op[j] += x_hat.op[j] - z.op[zi];
    }
}

Residuals residuals(const std::vector<Contribution>& locals, const Cloud& z_new, const Cloud& z_prev,
                    const Penalties& rho) {  // admm.cpp:147-198
    Residuals out;
    const int fd = z_new.fd;
    double p2 = 0;
    for (const Contribution& bc : locals) {
        const Cloud& x = *bc.params;
        for (size_t r = 0; r < x.size(); ++r) {
            const size_t zi = z_new.find(x.ids[r]);
            if (zi == Cloud::npos) throw InvalidArgument("id missing from consensus model");
            for (int k = 0; k < 3; ++k) {
                const double dp = x.pos[3 * r + k] - z_new.pos[3 * zi + k];
                const double ds = x.ls[3 * r + k] - z_new.ls[3 * zi + k];
                p2 += dp * dp + ds * ds;
            }
            for (int k = 0; k < 4; ++k) {
                const double d = x.rot[4 * r + k] - z_new.rot[4 * zi + k];
                p2 += d * d;
            }
            for (int k = 0; k < fd; ++k) {
                const double d = x.feat[r * fd + k] - z_new.feat[zi * fd + k];
                p2 += d * d;
            }
            const double d = x.op[r] - z_new.op[zi];
            p2 += d * d;
        }
    }
    double d2 = 0;
    for (size_t i = 0; i < z_new.size(); ++i) {
        const size_t j = z_prev.find(z_new.ids[i]);
        if (j == Cloud::npos) continue;
        for (int k = 0; k < 3; ++k) {
            const double dp = rho.rho_p * (z_new.pos[3 * i + k] - z_prev.pos[3 * j + k]);
            const double ds = rho.rho_s * (z_new.ls[3 * i + k] - z_prev.ls[3 * j + k]);
            d2 += dp * dp + ds * ds;
        }
        for (int k = 0; k < 4; ++k) {
            const double d = rho.rho_q * (z_new.rot[4 * i + k] - z_prev.rot[4 * j + k]);
            d2 += d * d;
        }
        for (int k = 0; k < fd; ++k) {
            const double d = rho.rho_f * (z_new.feat[i * fd + k] - z_prev.feat[j * fd + k]);
            d2 += d * d;
        }
        const double d = rho.rho_o * (z_new.op[i] - z_prev.op[j]);
        d2 += d * d;
    }
    out.primal = std::sqrt(p2);
    out.dual = std::sqrt(d2);
    return out;
}

Penalties adapt_penalties(const Penalties& rho, double primal, double dual, const ConsensusConfig& cfg,
                          uint64_t iteration) {  // admm.cpp:200-217
    if (!cfg.adaptive || iteration > cfg.freeze_iteration) return rho;
    Penalties out = rho;
    auto scale_all = [&out](double f) {
        out.rho_p *= f; out.rho_q *= f; out.rho_s *= f; out.rho_f *= f; out.rho_o *= f;
    };
    if (primal > cfg.mu * dual)
        scale_all(cfg.tau_inc);
    else if (dual > cfg.mu * primal)
        scale_all(1.0 / cfg.tau_dec);
    return out;
}

double max_disagreement(const std::vector<Contribution>& locals) {  // admm.cpp:219-243
    const auto owners = gather(locals);
    double worst = 0;
    for (const auto& [id, who] : owners) {
        if (who.size() < 2) continue;
        const int fd = who[0].cloud->fd;
        auto spread = [&](auto getter, int count) {
            for (int k = 0; k < count; ++k) {
                double lo = getter(*who[0].cloud, who[0].row, k), hi = lo;
                for (size_t c = 1; c < who.size(); ++c) {
                    const double v = getter(*who[c].cloud, who[c].row, k);
                    lo = std::min(lo, v);
                    hi = std::max(hi, v);
                }
                worst = std::max(worst, hi - lo);
            }
        };
        spread([](const Cloud& c, size_t r, int k) { return c.pos[3 * r + k]; }, 3);
        spread([](const Cloud& c, size_t r, int k) { return c.rot[4 * r + k]; }, 4);
        spread([](const Cloud& c, size_t r, int k) { return c.ls[3 * r + k]; }, 3);
        spread([fd](const Cloud& c, size_t r, int k) { return c.feat[r * fd + k]; }, fd);
        spread([](const Cloud& c, size_t r, int) { return c.op[r]; }, 1);
    }
    return worst;
}

// -------------------------------------------------------------- splitter.cpp
bool Aabb::contains(const V3& p) const {
    for (int a = 0; a < 3; ++a)
        if (!(p[a] >= min[a])) return false;
    for (int a = 0; a < 3; ++a)
        if (!(p[a] <= max[a])) return false;
    return true;
}
V3 Aabb::center() const { return V3{{0.5 * (min[0] + max[0]), 0.5 * (min[1] + max[1]), 0.5 * (min[2] + max[2])}}; }
V3 Aabb::extent() const { return V3{{max[0] - min[0], max[1] - min[1], max[2] - min[2]}}; }
double Aabb::distance(const V3& p) const {
    V3 d;
    for (int a = 0; a < 3; ++a) d[a] = std::max(std::max(min[a] - p[a], p[a] - max[a]), 0.0);
    return norm3(d);
}

Aabb tight_aabb(const std::vector<V3>& pts) {  // splitter.cpp:8-17
    if (pts.empty()) throw InvalidArgument("empty point set");
    Aabb box{pts[0], pts[0]};
    for (const V3& p : pts)
        for (int a = 0; a < 3; ++a) {
            box.min[a] = std::min(box.min[a], p[a]);
            box.max[a] = std::max(box.max[a], p[a]);
        }
    return box;
}

namespace {
Aabb tight_aabb_indexed(const std::vector<V3>& pts, const std::vector<size_t>& idx) {
    Aabb box{pts[idx[0]], pts[idx[0]]};
    for (size_t i : idx)
        for (int a = 0; a < 3; ++a) {
            box.min[a] = std::min(box.min[a], pts[i][a]);
            box.max[a] = std::max(box.max[a], pts[i][a]);
        }
    return box;
}
int pick_axis(const Aabb& box, int va) {  // splitter.cpp:32-44
    int best = -1;
    double best_len = -1.0;
    for (int a = 0; a < 3; ++a) {
        if (a == va) continue;
        const double len = box.max[a] - box.min[a];
        if (len > best_len) {
            best_len = len;
            best = a;
        }
    }
    return best;
}
}  // namespace

std::vector<CoreBlock> split_recursive(const std::vector<V3>& pts, uint32_t k, const SplitOptions& o) {
    if (k < 1) throw InvalidArgument("k must be at least 1");
    if (pts.empty()) throw InvalidArgument("empty point set");
    if (k > pts.size()) throw InvalidArgument("over-partitioned");
    std::vector<CoreBlock> cells(1);
    cells[0].point_indices.resize(pts.size());
    std::iota(cells[0].point_indices.begin(), cells[0].point_indices.end(), size_t{0});
    cells[0].box = tight_aabb(pts);
    while (cells.size() < k) {
        size_t target = 0;
        for (size_t c = 1; c < cells.size(); ++c)
            if (cells[c].point_indices.size() > cells[target].point_indices.size()) target = c;
        CoreBlock cell = std::move(cells[target]);
        const int axis = pick_axis(cell.box, o.vertical_axis);
        std::vector<size_t>& idx = cell.point_indices;
        std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
            if (pts[a][axis] != pts[b][axis]) return pts[a][axis] < pts[b][axis];
            return a < b;
        });
        size_t cut;
        if (o.midpoint_plane) {
            const double plane = 0.5 * (cell.box.min[axis] + cell.box.max[axis]);
            cut = static_cast<size_t>(std::lower_bound(idx.begin(), idx.end(), plane,
                                                       [&](size_t a, double v) { return pts[a][axis] < v; }) -
                                      idx.begin());
            cut = std::clamp<size_t>(cut, 1, idx.size() - 1);
        } else {
            cut = idx.size() / 2;
        }
        CoreBlock left, right;
        left.point_indices.assign(idx.begin(), idx.begin() + static_cast<ptrdiff_t>(cut));
        right.point_indices.assign(idx.begin() + static_cast<ptrdiff_t>(cut), idx.end());
        left.box = tight_aabb_indexed(pts, left.point_indices);
        right.box = tight_aabb_indexed(pts, right.point_indices);
        cells[target] = std::move(left);
        cells.push_back(std::move(right));
    }
    for (CoreBlock& c : cells) std::sort(c.point_indices.begin(), c.point_indices.end());
    return cells;
}

BlockPartition expand_and_assign(const std::vector<CoreBlock>& blocks, const std::vector<V3>& pts,
                                 const std::vector<Camera>& views, const Cloud& g, double scale,
                                 const SplitOptions& o) {  // splitter.cpp:98-201
    if (scale < 1.0) throw InvalidArgument("expansion scale must be >= 1");
    BlockPartition part;
    part.k = static_cast<uint32_t>(blocks.size());
    for (const CoreBlock& b : blocks) part.core.push_back(b.box);
    const int va = o.vertical_axis;
    double vmin = std::numeric_limits<double>::infinity(), vmax = -vmin;
    for (const V3& p : pts) {
        vmin = std::min(vmin, p[va]);
        vmax = std::max(vmax, p[va]);
    }
    for (size_t i = 0; i < g.size(); ++i) {
        const V3 p = g.position(i);
        vmin = std::min(vmin, p[va]);
        vmax = std::max(vmax, p[va]);
    }
    for (const CoreBlock& b : blocks) {
        Aabb e = b.box;
        for (int a = 0; a < 3; ++a) {
            if (a == va) continue;
            const double c = 0.5 * (b.box.min[a] + b.box.max[a]);
            const double half = 0.5 * (b.box.max[a] - b.box.min[a]) * scale;
            e.min[a] = std::min(b.box.min[a], c - half);
            e.max[a] = std::max(b.box.max[a], c + half);
        }
        e.min[va] = vmin;
        e.max[va] = vmax;
        part.expanded.push_back(e);
    }
    const uint32_t k = part.k;
    part.block_points.resize(k);
    part.block_views.resize(k);
    part.block_gaussians.resize(k);
    for (size_t i = 0; i < pts.size(); ++i)
        for (uint32_t b = 0; b < k; ++b)
            if (part.expanded[b].contains(pts[i])) part.block_points[b].push_back(i);
    for (size_t i = 0; i < g.size(); ++i) {
        const V3 p = g.position(i);
        uint32_t owners = 0;
        for (uint32_t b = 0; b < k; ++b)
            if (part.expanded[b].contains(p)) {
                part.block_gaussians[b].push_back(g.ids[i]);
                ++owners;
            }
        if (owners == 0) {
            uint32_t best = 0;
            double best_d = part.expanded[0].distance(p);
            for (uint32_t b = 1; b < k; ++b) {
                const double d = part.expanded[b].distance(p);
                if (d < best_d) {
                    best_d = d;
                    best = b;
                }
            }
            part.block_gaussians[best].push_back(g.ids[i]);
            owners = 1;
        }
        if (owners >= 2) {
            std::vector<uint32_t>& who = part.shared[g.ids[i]];
            for (uint32_t b = 0; b < k; ++b)
                if (part.expanded[b].contains(p)) who.push_back(b);
        }
    }
    for (size_t v = 0; v < views.size(); ++v) {
        const V3 c = views[v].center();
        bool placed = false;
        for (uint32_t b = 0; b < k; ++b)
            if (part.expanded[b].contains(c)) {
                part.block_views[b].push_back(v);
                placed = true;
            }
        if (!placed) {
            uint32_t best = 0;
            auto d2 = [&](uint32_t b) {
                const V3 e = part.expanded[b].center();
                const double dx = e[0] - c[0], dy = e[1] - c[1], dz = e[2] - c[2];
                return (dx * dx + dy * dy) + dz * dz;
            };
            double best_d = d2(0);
            for (uint32_t b = 1; b < k; ++b) {
                const double d = d2(b);
                if (d < best_d) {
                    best_d = d;
                    best = b;
                }
            }
            part.block_views[best].push_back(v);
        }
    }
    return part;
}

// -------------------------------------------------------------- trainer.cpp
uint64_t derive_seed(uint64_t seed, uint32_t block_id) {  // trainer.cpp:116-118
    return seed ^ (0x9e3779b97f4a7c15ull * (static_cast<uint64_t>(block_id) + 1));
}

Cloud init_cloud_from_points(const std::vector<ScenePoint>& pts, int sh_degree, double init_opacity) {
    if (pts.empty()) throw InvalidArgument("empty point set");
    const int fd = sh_degree >= 1 ? kFeatureDimDeg1 : kFeatureDimDeg0;
    const size_t n = pts.size();
    Cloud cloud(fd);
    // trainer.cpp:76-97: squared distances from f32 differences (Eigen
    // Vector3f arithmetic), summed in float then widened.
    std::vector<double> mean_dist(n, 0.1);
    for (size_t i = 0; i < n; ++i) {
        double best[3] = {1e300, 1e300, 1e300};
        const float* pi = pts[i].p;
        for (size_t j = 0; j < n; ++j) {
            if (j == i) continue;
            const float dx = pts[j].p[0] - pi[0], dy = pts[j].p[1] - pi[1], dz = pts[j].p[2] - pi[2];
            const double d2 = static_cast<double>((dx * dx + dy * dy) + dz * dz);
            if (d2 < best[2]) {
                best[2] = d2;
                if (best[2] < best[1]) std::swap(best[1], best[2]);
                if (best[1] < best[0]) std::swap(best[0], best[1]);
            }
        }
        double sum = 0;
        int cnt = 0;
        for (double b : best)
            if (b < 1e300) {
                sum += std::sqrt(b);
                ++cnt;
            }
        if (cnt > 0) mean_dist[i] = std::max(sum / cnt, 1e-6);
    }
    const double op_logit = logit(init_opacity);
    for (size_t i = 0; i < n; ++i) {
        cloud.ids.push_back(i);
        for (int k = 0; k < 3; ++k) cloud.pos.push_back(static_cast<double>(pts[i].p[k]));
        cloud.rot.insert(cloud.rot.end(), {1.0, 0.0, 0.0, 0.0});
        const double l = std::log(mean_dist[i]);
        cloud.ls.insert(cloud.ls.end(), {l, l, l});
        for (int k = 0; k < fd; ++k) cloud.feat.push_back(k < 3 ? (pts[i].rgb[k] / 255.0) / kSh0 : 0.0);
        cloud.op.push_back(op_logit);
    }
    return cloud;
}

namespace {
void adam_step(double* x, const double* g, double* m, double* v, size_t n, double lr, uint64_t t,
               const AdamParams& p) {  // trainer.cpp:120-131
    const double bc1 = 1.0 - std::pow(p.beta1, static_cast<double>(t));
    const double bc2 = 1.0 - std::pow(p.beta2, static_cast<double>(t));
    for (size_t i = 0; i < n; ++i) {
        m[i] = p.beta1 * m[i] + (1.0 - p.beta1) * g[i];
        v[i] = p.beta2 * v[i] + (1.0 - p.beta2) * g[i] * g[i];
        const double mh = m[i] / bc1;
        const double vh = v[i] / bc2;
        x[i] -= lr * mh / (std::sqrt(vh) + p.eps);
    }
}

void edit_array(std::vector<double>& v, const std::vector<char>& drop, size_t width, size_t added) {
    size_t w = 0;
    for (size_t r = 0; r < drop.size(); ++r) {
        if (drop[r]) continue;
        if (w != r)
            for (size_t k = 0; k < width; ++k) v[w * width + k] = v[r * width + k];
        ++w;
    }
    v.resize(w * width);
    v.insert(v.end(), added * width, 0.0);
}
}  // namespace

BlockTrainer::BlockTrainer(uint32_t block_id, Cloud initial, std::vector<TrainView> views,
                           std::vector<uint64_t> shared_ids, uint64_t global_initial_count,
                           const TrainerConfig& cfg)  // trainer.cpp:135-159
    : block_id_(block_id), cfg_(cfg), cloud_(std::move(initial)), views_(std::move(views)),
      shared_ids_(std::move(shared_ids)), anchor_(cloud_.fd), duals_(cloud_.fd),
      rng_(derive_seed(cfg.seed, block_id)) {
    if (views_.empty()) throw InvalidArgument("trainer needs at least one view");
    if (!cloud_.check_invariants()) throw InvalidArgument("initial cloud ids not ascending");
    alloc_next_ = (uint64_t(block_id) << 48) + (block_id == 0 ? global_initial_count : 0);
    alloc_end_ = (uint64_t(block_id) + 1) << 48;
    if (cfg_.densify.stop_iteration == 0) cfg_.densify.stop_iteration = (cfg_.iterations * 6) / 10;
    std::vector<V3> pts(cloud_.size());
    for (size_t i = 0; i < cloud_.size(); ++i) pts[i] = cloud_.position(i);
    if (!pts.empty()) scene_extent_ = std::max(norm3(tight_aabb(pts).extent()), 1e-9);
    const size_t n = cloud_.size();
    m_pos_.assign(3 * n, 0); v_pos_.assign(3 * n, 0);
    m_rot_.assign(4 * n, 0); v_rot_.assign(4 * n, 0);
    m_ls_.assign(3 * n, 0); v_ls_.assign(3 * n, 0);
    m_feat_.assign(n * cloud_.fd, 0); v_feat_.assign(n * cloud_.fd, 0);
    m_op_.assign(n, 0); v_op_.assign(n, 0);
    grad_accum_.assign(n, 0.0);
    grad_seen_.assign(n, 0);
    view_order_.resize(views_.size());
    std::iota(view_order_.begin(), view_order_.end(), size_t{0});
}

void BlockTrainer::set_anchor(const Cloud& z, const Penalties& rho) {  // trainer.cpp:161-166
    anchor_ = slice_by_ids(z, shared_ids_);
    duals_ = zero_bundle(anchor_.ids, cloud_.fd);
    rho_ = rho;
    have_anchor_ = true;
}

void BlockTrainer::apply_broadcast(const Cloud& z, const std::vector<uint64_t>& reset_ids,
                                   const std::vector<uint64_t>& unshared_ids, const Penalties& rho,
                                   double alpha, bool over_relaxed) {  // trainer.cpp:168-223
    if (!have_anchor_) {
        set_anchor(z, rho);
        return;
    }
    if (!unshared_ids.empty()) {
        erase_by_ids(duals_, unshared_ids);
        erase_by_ids(anchor_, unshared_ids);
        std::vector<uint64_t> keep;
        std::set_difference(shared_ids_.begin(), shared_ids_.end(), unshared_ids.begin(), unshared_ids.end(),
                            std::back_inserter(keep));
        shared_ids_ = std::move(keep);
    }
    Cloud x_hat = slice_by_ids(cloud_, anchor_.ids);
    if (x_hat.ids != anchor_.ids) throw InvalidArgument("shared rows missing from cloud");
    if (over_relaxed) {
        const int fd = x_hat.fd;
        for (size_t j = 0; j < x_hat.size(); ++j) {
            for (int k = 0; k < 3; ++k) {
                x_hat.pos[3 * j + k] = relaxed_value(x_hat.pos[3 * j + k], anchor_.pos[3 * j + k], alpha);
                x_hat.ls[3 * j + k] = relaxed_value(x_hat.ls[3 * j + k], anchor_.ls[3 * j + k], alpha);
            }
            for (int k = 0; k < 4; ++k) x_hat.rot[4 * j + k] = relaxed_value(x_hat.rot[4 * j + k], anchor_.rot[4 * j + k], alpha);
            for (int k = 0; k < fd; ++k)
                x_hat.feat[j * fd + k] = relaxed_value(x_hat.feat[j * fd + k], anchor_.feat[j * fd + k], alpha);
            x_hat.op[j] = relaxed_value(x_hat.op[j], anchor_.op[j], alpha);
        }
    }
    dual_update(duals_, x_hat, z);
    for (uint64_t id : reset_ids) {
        const size_t j = duals_.find(id);
        if (j == Cloud::npos) continue;
        const int fd = duals_.fd;
        for (int k = 0; k < 3; ++k) duals_.pos[3 * j + k] = 0.0;
        for (int k = 0; k < 4; ++k) duals_.rot[4 * j + k] = 0.0;
        for (int k = 0; k < 3; ++k) duals_.ls[3 * j + k] = 0.0;
        for (int k = 0; k < fd; ++k) duals_.feat[j * fd + k] = 0.0;
        duals_.op[j] = 0.0;
    }
    anchor_ = slice_by_ids(z, shared_ids_);
    if (anchor_.ids != duals_.ids) throw InvalidArgument("broadcast misses shared ids");
    rho_ = rho;
}

Cloud BlockTrainer::nonshared_slice() const {
    std::vector<size_t> idx;
    for (size_t i = 0; i < cloud_.size(); ++i)
        if (!std::binary_search(shared_ids_.begin(), shared_ids_.end(), cloud_.ids[i])) idx.push_back(i);
    return cloud_.subset(idx);
}

std::vector<uint64_t> BlockTrainer::take_removed_ids() {
    std::vector<uint64_t> out = std::move(removed_ids_);
    removed_ids_.clear();
    std::sort(out.begin(), out.end());
    return out;
}

Cloud BlockTrainer::take_new_rows() {
    std::sort(new_ids_.begin(), new_ids_.end());
    Cloud rows = slice_by_ids(cloud_, new_ids_);
    new_ids_.clear();
    return rows;
}

std::vector<double> BlockTrainer::moments(int which) const {
    // which: 0 = m, 1 = v; [component][row] with components pos3 rot4 ls3 feat fd op1.
    const size_t n = cloud_.size();
    const int fd = cloud_.fd;
    const int D = 11 + fd;
    std::vector<double> out(size_t(D) * n);
    const std::vector<double>* arr[5] = {which ? &v_pos_ : &m_pos_, which ? &v_rot_ : &m_rot_, which ? &v_ls_ : &m_ls_,
                                         which ? &v_feat_ : &m_feat_, which ? &v_op_ : &m_op_};
    const int widths[5] = {3, 4, 3, fd, 1};
    int comp = 0;
    for (int g = 0; g < 5; ++g)
        for (int k = 0; k < widths[g]; ++k, ++comp)
            for (size_t i = 0; i < n; ++i) out[size_t(comp) * n + i] = (*arr[g])[i * widths[g] + k];
    return out;
}

double BlockTrainer::train_step() {  // trainer.cpp:249-295
    if (view_cursor_ == 0) rng_.shuffle(view_order_);
    last_view_ = view_order_[view_cursor_];
    const TrainView& view = views_[last_view_];
    view_cursor_ = (view_cursor_ + 1) % views_.size();

    BackwardOut bw = render_backward(cloud_, view.camera, *view.image, cfg_.render);
    double loss = bw.loss;
    if (have_anchor_ && !anchor_.ids.empty()) {
        std::vector<size_t> idx(anchor_.ids.size());
        for (size_t j = 0; j < anchor_.ids.size(); ++j) {
            idx[j] = cloud_.find(anchor_.ids[j]);
            if (idx[j] == Cloud::npos) throw InvalidArgument("shared rows missing from cloud");
        }
        loss += penalty_loss_and_grad(cloud_, idx, anchor_, duals_, rho_, bw.grads);
    }
    const uint64_t t = ++steps_;
    const double progress = cfg_.iterations > 0 ? double(iteration_) / double(cfg_.iterations) : 0.0;
    const double lr_pos = cfg_.lr.position * std::pow(cfg_.lr.position_decay, progress);
    adam_step(cloud_.pos.data(), bw.grads.pos.data(), m_pos_.data(), v_pos_.data(), cloud_.pos.size(), lr_pos, t, cfg_.adam);
    adam_step(cloud_.rot.data(), bw.grads.rot.data(), m_rot_.data(), v_rot_.data(), cloud_.rot.size(), cfg_.lr.rotation, t, cfg_.adam);
    adam_step(cloud_.ls.data(), bw.grads.ls.data(), m_ls_.data(), v_ls_.data(), cloud_.ls.size(), cfg_.lr.log_scale, t, cfg_.adam);
    adam_step(cloud_.feat.data(), bw.grads.feat.data(), m_feat_.data(), v_feat_.data(), cloud_.feat.size(), cfg_.lr.features, t, cfg_.adam);
    adam_step(cloud_.op.data(), bw.grads.op.data(), m_op_.data(), v_op_.data(), cloud_.op.size(), cfg_.lr.opacity, t, cfg_.adam);
    cloud_.canonicalize_rotations();
    for (size_t i = 0; i < cloud_.size(); ++i)
        if (bw.visible[i]) {
            grad_accum_[i] += bw.screen_grad_norm[i];
            ++grad_seen_[i];
        }
    ++iteration_;
    maybe_densify();
    last_loss_ = loss;
    return loss;
}

void BlockTrainer::maybe_densify() {  // trainer.cpp:301-385
    const DensifyConfig& d = cfg_.densify;
    if (!d.enabled || iteration_ == 0) return;
    if (iteration_ % d.interval != 0 || iteration_ > d.stop_iteration) return;
    const double split_scale = d.split_scale_fraction * scene_extent_;
    std::vector<size_t> drop;
    Cloud children(cloud_.fd);
    auto allocate = [this]() {
        if (alloc_next_ >= alloc_end_) throw std::runtime_error("id allocator exhausted");
        return alloc_next_++;
    };
    for (size_t i = 0; i < cloud_.size(); ++i) {
        const uint64_t id = cloud_.ids[i];
        const bool is_shared = std::binary_search(shared_ids_.begin(), shared_ids_.end(), id);
        if (cloud_.opacity(i) < d.prune_opacity) {
            drop.push_back(i);
            removed_ids_.push_back(id);
            continue;
        }
        if (grad_seen_[i] == 0) continue;
        const double mean_grad = grad_accum_[i] / grad_seen_[i];
        if (mean_grad < d.grad_threshold) continue;
        const V3 lsv = cloud_.log_scale(i);
        const double scales[3] = {std::exp(lsv[0]), std::exp(lsv[1]), std::exp(lsv[2])};
        int axis = 0;
        for (int a = 1; a < 3; ++a)
            if (scales[a] > scales[axis]) axis = a;
        const M3 r = quat_to_rotation(quat_normalized(cloud_.rotation(i)));
        const double off[3] = {r(0, axis) * (0.5 * scales[axis]), r(1, axis) * (0.5 * scales[axis]), r(2, axis) * (0.5 * scales[axis])};
        Cloud parent = cloud_.subset({i});
        if (scales[axis] >= split_scale) {
            Cloud child = parent;
            for (int k = 0; k < 3; ++k) child.ls[k] = parent.ls[k] - std::log(d.split_shrink);
            if (is_shared) {
                child.ids[0] = allocate();
                for (int k = 0; k < 3; ++k) child.pos[k] = parent.pos[k] + off[k];
                children.push_row(child, 0);
                new_ids_.push_back(child.ids[0]);
            } else {
                drop.push_back(i);
                removed_ids_.push_back(id);
                for (int s = 0; s < 2; ++s) {
                    child.ids[0] = allocate();
                    for (int k = 0; k < 3; ++k) child.pos[k] = parent.pos[k] + (s == 0 ? off[k] : -off[k]);
                    children.push_row(child, 0);
                    new_ids_.push_back(child.ids[0]);
                }
            }
        } else {
            Cloud clone = parent;
            clone.ids[0] = allocate();
            children.push_row(clone, 0);
            new_ids_.push_back(clone.ids[0]);
        }
    }
    if (drop.empty() && children.size() == 0) {
        std::fill(grad_accum_.begin(), grad_accum_.end(), 0.0);
        std::fill(grad_seen_.begin(), grad_seen_.end(), 0);
        return;
    }
    if (!removed_ids_.empty() && !shared_ids_.empty()) {
        std::vector<uint64_t> gone = removed_ids_;
        std::sort(gone.begin(), gone.end());
        std::vector<uint64_t> keep;
        std::set_difference(shared_ids_.begin(), shared_ids_.end(), gone.begin(), gone.end(), std::back_inserter(keep));
        if (keep.size() != shared_ids_.size()) {
            shared_ids_ = std::move(keep);
            erase_by_ids(anchor_, gone);
            erase_by_ids(duals_, gone);
        }
    }
    cloud_.remove_indices(drop);
    std::vector<char> dropmask(m_op_.size(), 0);
    for (size_t i : drop) dropmask[i] = 1;
    const size_t added = children.size();
    edit_array(m_pos_, dropmask, 3, added); edit_array(v_pos_, dropmask, 3, added);
    edit_array(m_rot_, dropmask, 4, added); edit_array(v_rot_, dropmask, 4, added);
    edit_array(m_ls_, dropmask, 3, added); edit_array(v_ls_, dropmask, 3, added);
    edit_array(m_feat_, dropmask, cloud_.fd, added); edit_array(v_feat_, dropmask, cloud_.fd, added);
    edit_array(m_op_, dropmask, 1, added); edit_array(v_op_, dropmask, 1, added);
    for (size_t j = 0; j < children.size(); ++j) cloud_.push_row(children, j);
    if (!cloud_.check_invariants()) throw std::runtime_error("cloud invariant broken by densify");
    grad_accum_.assign(cloud_.size(), 0.0);
    grad_seen_.assign(cloud_.size(), 0);
}

// ---------------------------------------------------------------- synth.cpp
Scene generate_scene(const SynthConfig& cfg) {  // synth.cpp:13-77
    if (cfg.gaussians == 0) throw InvalidArgument("zero gaussians");
    if (cfg.cameras == 0) throw InvalidArgument("zero cameras");
    Rng rng(cfg.seed);
    const int fd = cfg.sh_degree >= 1 ? kFeatureDimDeg1 : kFeatureDimDeg0;
    const double half = 0.5 * cfg.extent;
    Scene out;
    Cloud& gt = out.ground_truth;
    gt = Cloud(fd);
    for (uint32_t i = 0; i < cfg.gaussians; ++i) {
        gt.ids.push_back(i);
        // Vec3(a, b, c) of three rng calls: GCC evaluates constructor
        // arguments right to left (see Rng::random_unit_quat).
        const double pz = rng.uniform(-half, half);
        const double py = rng.uniform(-half / 5.0, half / 5.0);
        const double px = rng.uniform(-half, half);
        gt.pos.insert(gt.pos.end(), {px, py, pz});
        const V4 q = rng.random_unit_quat();
        gt.rot.insert(gt.rot.end(), {q[0], q[1], q[2], q[3]});
        const double radius = cfg.extent * rng.uniform(0.015, 0.05);
        const double l = std::log(radius);
        gt.ls.insert(gt.ls.end(), {l, l, l});
        std::vector<double> f(fd, 0.0);
        for (int c = 0; c < 3; ++c) f[c] = rng.uniform(0.05, 0.95) / kSh0;
        if (fd > kFeatureDimDeg0)
            for (int k = kFeatureDimDeg0; k < fd; ++k) f[k] = 0.1 * rng.normal();
        gt.feat.insert(gt.feat.end(), f.begin(), f.end());
        gt.op.push_back(logit(rng.uniform(0.4, 0.9)));
    }
    const double orbit_radius = 0.8 * cfg.extent;
    const double orbit_height = 0.5 * cfg.extent;
    const double focal = 0.8 * cfg.image_size;
    const double center = 0.5 * cfg.image_size;
    for (uint32_t i = 0; i < cfg.cameras; ++i) {
        const double angle = 2.0 * M_PI * static_cast<double>(i) / cfg.cameras;
        const V3 position{{orbit_radius * std::cos(angle), orbit_height, orbit_radius * std::sin(angle)}};
        Camera cam = look_at(position, V3{{0, 0, 0}}, V3{{0, 1, 0}}, focal, focal, center, center,
                             cfg.image_size, cfg.image_size);
        cam.view_id = i;
        out.views.push_back(cam);
    }
    // The views' renders are independent pure functions of (gt, cam): drawn
    // on worker threads (test-fixture setup time only; each image is the
    // same sequential per-pixel loop, so the bytes do not change).
    out.images.resize(out.views.size());
    {
        const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32u));
        std::atomic<size_t> next{0};
        std::vector<std::thread> pool;
        for (unsigned w = 0; w < nt; ++w)
            pool.emplace_back([&] {
                for (size_t i; (i = next.fetch_add(1)) < out.views.size();)
                    out.images[i] = render(gt, out.views[i], cfg.render).color;
            });
        for (auto& t : pool) t.join();
    }
    std::vector<size_t> order(cfg.gaussians);
    std::iota(order.begin(), order.end(), size_t{0});
    rng.shuffle(order);
    const size_t keep = (cfg.gaussians + 1) / 2;
    order.resize(keep);
    std::sort(order.begin(), order.end());
    const double jitter = 0.02 * cfg.extent;
    for (size_t idx : order) {
        ScenePoint p;
        const double n2 = rng.normal();  // right-to-left, as above
        const double n1 = rng.normal();
        const double n0 = rng.normal();
        const double nz[3] = {n0, n1, n2};
        for (int k = 0; k < 3; ++k) p.p[k] = static_cast<float>(gt.pos[3 * idx + k] + jitter * nz[k]);
        for (int c = 0; c < 3; ++c) {
            const double v = std::clamp(kSh0 * gt.feat[idx * fd + c], 0.0, 1.0);
            p.rgb[c] = static_cast<uint8_t>(std::lround(255.0 * v));
        }
        out.points.push_back(p);
    }
    return out;
}

// -------------------------------------------------------------- runtime.cpp
std::vector<uint64_t> consensus_schedule(uint64_t total, uint32_t interval) {  // runtime.cpp:256-263
    if (total == 0) throw InvalidArgument("zero training iterations");
    if (interval == 0) throw InvalidArgument("zero consensus interval");
    std::vector<uint64_t> out;
    for (uint64_t t = interval; t < total; t += interval) out.push_back(t);
    out.push_back(total);
    return out;
}

ClusterPlan plan_cluster(const Scene& scene, uint32_t blocks, double expand_scale, uint32_t holdout,
                         const TrainerConfig& tc, const SplitOptions& so) {  // runtime.cpp:265-305
    if (scene.views.empty()) throw InvalidArgument("scene has no views");
    if (scene.images.size() != scene.views.size()) throw InvalidArgument("one image per view required");
    ClusterPlan plan;
    plan.init_cloud = scene.has_checkpoint ? scene.checkpoint
                                           : init_cloud_from_points(scene.points, tc.sh_degree, tc.init_opacity);
    if (!plan.init_cloud.check_invariants()) throw InvalidArgument("initial cloud ill-formed");
    std::vector<V3> positions(plan.init_cloud.size());
    for (size_t i = 0; i < positions.size(); ++i) positions[i] = plan.init_cloud.position(i);
    const std::vector<CoreBlock> cores = split_recursive(positions, blocks, so);
    plan.partition = expand_and_assign(cores, positions, scene.views, plan.init_cloud, expand_scale, so);
    for (uint32_t b = 0; b < blocks; ++b)
        for (uint64_t id : plan.partition.block_gaussians[b]) plan.owners[id].push_back(b);
    plan.shards.resize(blocks);
    for (uint32_t b = 0; b < blocks; ++b) {
        ShardSpec& shard = plan.shards[b];
        shard.block_id = b;
        shard.global_initial_count = plan.init_cloud.size();
        shard.initial = slice_by_ids(plan.init_cloud, plan.partition.block_gaussians[b]);
        for (const auto& [id, owner_list] : plan.partition.shared)
            if (std::binary_search(owner_list.begin(), owner_list.end(), b)) shard.shared_ids.push_back(id);
        for (size_t vi : plan.partition.block_views[b]) {
            if (holdout != 0 && vi % holdout == 0) continue;
            shard.views.push_back(TrainView{scene.views[vi], &scene.images[vi]});
            shard.view_indices.push_back(vi);
        }
        if (shard.views.empty()) throw std::runtime_error("block " + std::to_string(b) + " has no training views");
    }
    return plan;
}

OwnershipRound master_ownership_round(std::map<uint64_t, std::vector<uint32_t>>& owners,
                                      const std::vector<std::vector<uint64_t>>& removed,
                                      const std::vector<std::vector<uint64_t>>& added) {  // runtime.cpp:490-518
    std::map<uint64_t, size_t> prev_owner_count;
    for (uint32_t b = 0; b < removed.size(); ++b)
        for (uint64_t id : removed[b]) {
            auto it = owners.find(id);
            if (it == owners.end()) continue;
            prev_owner_count.emplace(id, it->second.size());
            auto& list = it->second;
            list.erase(std::remove(list.begin(), list.end(), b), list.end());
        }
    OwnershipRound r;
    for (const auto& [id, prev] : prev_owner_count) {
        const auto& list = owners.at(id);
        if (list.empty()) r.dead.push_back(id);
        else if (prev >= 2 && list.size() == 1) r.unshared.push_back(id);
        else if (prev >= 2) r.reset.push_back(id);
    }
    for (uint64_t id : r.dead) owners.erase(id);
    for (uint32_t b = 0; b < added.size(); ++b)
        for (uint64_t id : added[b]) owners[id] = {b};
    for (const auto& [id, list] : owners)  // current_shared (runtime.cpp:520)
        if (list.size() >= 2) r.shared_now.push_back(id);
    return r;
}

RunResult run_simulated(const ClusterPlan& plan, const TrainerConfig& tc, const SessionOptions& opt) {
    if (opt.total_iterations != tc.iterations) throw InvalidArgument("session and trainer iteration counts differ");
    const auto blocks = static_cast<uint32_t>(plan.shards.size());
    if (blocks == 0) throw InvalidArgument("plan has no shards");
    std::vector<BlockTrainer> trainers;
    trainers.reserve(blocks);
    for (uint32_t b = 0; b < blocks; ++b) {
        const ShardSpec& s = plan.shards[b];
        trainers.emplace_back(s.block_id, s.initial, s.views, s.shared_ids, s.global_initial_count, tc);
    }
    // run_master_session (runtime.cpp:427-611) with the worker halves
    // (runtime.cpp:363-425) inlined at each barrier.
    auto owners = plan.owners;
    Cloud global = plan.init_cloud;
    Penalties rho = opt.rho;
    auto current_shared = [&owners] {
        std::vector<uint64_t> out;
        for (const auto& [id, list] : owners)
            if (list.size() >= 2) out.push_back(id);
        return out;
    };
    std::vector<uint64_t> shared_now = current_shared();
    Cloud z_prev = slice_by_ids(global, shared_now);
    if (opt.consensus.enabled)
        for (auto& t : trainers) t.set_anchor(z_prev, rho);

    RunResult result;
    const std::vector<uint64_t> schedule = consensus_schedule(opt.total_iterations, opt.consensus.interval);
    uint64_t done = 0;
    for (size_t j = 0; j < schedule.size(); ++j) {
        const uint64_t t = schedule[j];
        const bool final_round = t == opt.total_iterations;
        struct Up { double loss; Cloud new_rows, shared, nonshared; std::vector<uint64_t> removed; bool has_nonshared; };
        std::vector<Up> ups(blocks);
        for (uint32_t b = 0; b < blocks; ++b) {
            trainers[b].run_iterations(t - done);
            ups[b].loss = trainers[b].last_loss();
            ups[b].new_rows = trainers[b].take_new_rows();
            ups[b].shared = trainers[b].shared_slice();
            ups[b].removed = trainers[b].take_removed_ids();
            ups[b].has_nonshared = final_round || (opt.nonshared_refresh != 0 && (j + 1) % opt.nonshared_refresh == 0);
            if (ups[b].has_nonshared) ups[b].nonshared = trainers[b].nonshared_slice();
        }
        done = t;
        std::vector<std::vector<uint64_t>> removed(blocks), added(blocks);
        for (uint32_t b = 0; b < blocks; ++b) {
            removed[b] = ups[b].removed;
            added[b] = ups[b].new_rows.ids;
        }
        OwnershipRound own = master_ownership_round(owners, removed, added);
        std::vector<uint64_t> reset_ids = own.reset, unshared_ids = own.unshared;
        erase_by_ids(global, own.dead);
        for (uint32_t b = 0; b < blocks; ++b)
            if (ups[b].new_rows.size() != 0) insert_rows(global, ups[b].new_rows);
        shared_now = own.shared_now;
        std::vector<Cloud> slices(blocks);
        std::vector<Contribution> contribs;
        for (uint32_t b = 0; b < blocks; ++b) {
            slices[b] = slice_by_ids(ups[b].shared, shared_now);
            contribs.push_back(Contribution{b, &slices[b]});
        }
        std::vector<uint64_t> flipped;
        const bool relax = opt.consensus.enabled && opt.consensus.alpha != 1.0 && !final_round;
        const Cloud z = consensus_average(contribs, relax, z_prev, opt.consensus.alpha, &flipped);
        reset_ids.insert(reset_ids.end(), flipped.begin(), flipped.end());
        std::sort(reset_ids.begin(), reset_ids.end());
        reset_ids.erase(std::unique(reset_ids.begin(), reset_ids.end()), reset_ids.end());
        const Residuals norms = residuals(contribs, z, z_prev, rho);
        if (opt.consensus.enabled) rho = adapt_penalties(rho, norms.primal, norms.dual, opt.consensus, t);
        RoundDiagnostics diag;
        diag.iteration = t;
        diag.primal_residual = norms.primal;
        diag.dual_residual = norms.dual;
        diag.rho = rho;
        diag.max_disagreement = max_disagreement(contribs);
        for (uint32_t b = 0; b < blocks; ++b) diag.mean_loss += ups[b].loss;
        diag.mean_loss /= blocks;
        Cloud z_model = z;
        for (size_t i = 0; i < z_model.size(); ++i) {
            const V4 q = quat_normalized(z_model.rotation(i));
            for (int k = 0; k < 4; ++k) z_model.rot[4 * i + k] = q[k];
        }
        overwrite_by_ids(global, z_model);
        for (uint64_t id : unshared_ids) {
            const uint32_t owner = owners.at(id).front();
            overwrite_by_ids(global, slice_by_ids(ups[owner].shared, {id}));
        }
        for (uint32_t b = 0; b < blocks; ++b)
            if (ups[b].has_nonshared) overwrite_by_ids(global, ups[b].nonshared);
        z_prev = z;
        // Worker apply_broadcast (runtime.cpp:409-417).
        if (opt.consensus.enabled) {
            const bool wrelax = opt.consensus.alpha != 1.0 && !final_round;
            for (auto& tr : trainers) tr.apply_broadcast(z, reset_ids, unshared_ids, rho, opt.consensus.alpha, wrelax);
        }
        // Dual-mean diagnostic (runtime.cpp:572-606).
        Cloud accum = zero_bundle(shared_now, global.fd);
        std::vector<uint32_t> counts(shared_now.size(), 0);
        for (uint32_t b = 0; b < blocks; ++b) {
            const Cloud& du = trainers[b].duals();
            const int fd = accum.fd;
            for (size_t i = 0; i < du.size(); ++i) {
                const size_t row = accum.find(du.ids[i]);
                if (row == Cloud::npos) continue;
                for (int k = 0; k < 3; ++k) accum.pos[3 * row + k] += du.pos[3 * i + k];
                for (int k = 0; k < 4; ++k) accum.rot[4 * row + k] += du.rot[4 * i + k];
                for (int k = 0; k < 3; ++k) accum.ls[3 * row + k] += du.ls[3 * i + k];
                for (int k = 0; k < fd; ++k) accum.feat[row * fd + k] += du.feat[i * fd + k];
                accum.op[row] += du.op[i];
                ++counts[row];
            }
        }
        double linf = 0;
        const int fd = accum.fd;
        for (size_t row = 0; row < accum.size(); ++row) {
            if (counts[row] == 0) continue;
            const double inv = 1.0 / counts[row];
            auto upd = [&linf, inv](double v) { linf = std::max(linf, std::abs(v * inv)); };
            for (int k = 0; k < 3; ++k) upd(accum.pos[3 * row + k]);
            for (int k = 0; k < 4; ++k) upd(accum.rot[4 * row + k]);
            for (int k = 0; k < 3; ++k) upd(accum.ls[3 * row + k]);
            for (int k = 0; k < fd; ++k) upd(accum.feat[row * fd + k]);
            upd(accum.op[row]);
        }
        diag.dual_mean_linf = linf;
        diag.shared_count = shared_now.size();
        diag.global_count = global.size();
        result.rounds.push_back(diag);
    }
    result.model = global;
    for (auto& tr : trainers) result.block_clouds.push_back(tr.cloud());
    return result;
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

}  // namespace orc
