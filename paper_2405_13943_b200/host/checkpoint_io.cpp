// DOGS container and GSPL checkpoint codec (scene.hpp:15-50, scene_io.cpp),
// plus the model.dogs writer of main.cpp:353-357. Host byte work: the only
// device piece is encode_gspl_device, which asks the block's context for the
// GSPL payload of its cloud (csrc/checkpoint.cu) instead of downloading FP64
// rows and narrowing them on the host.
#include <cstdio>
#include <cstring>

#include "../../include/blocksplat_gpu.hpp"

namespace blocksplat {
namespace {

// Little-endian byte sink (the host is little-endian; values are copied bytewise).
class Sink {
public:
    template <typename T>
    void put(T v) {
        uint8_t b[sizeof(T)];
        std::memcpy(b, &v, sizeof(T));
        buf_.insert(buf_.end(), b, b + sizeof(T));
    }
    void raw(const void* p, size_t n) {
        const auto* b = static_cast<const uint8_t*>(p);
        buf_.insert(buf_.end(), b, b + n);
    }
    std::vector<uint8_t>& bytes() { return buf_; }

private:
    std::vector<uint8_t> buf_;
};

// Bounded reader: running past the end is a FormatError with the code the
// reader was made with (TruncatedBuffer for the container, TruncatedSection
// inside a section), as serial::Reader in the reference.
class Source {
public:
    Source(const uint8_t* p, size_t n, FormatErrorCode code) : p_(p), n_(n), code_(code) {}
    template <typename T>
    T get() {
        T v;
        take(&v, sizeof(T));
        return v;
    }
    void take(void* dst, size_t k) {
        need(k);
        if (k) std::memcpy(dst, p_ + at_, k);
        at_ += k;
    }
    void skip(size_t k) {
        need(k);
        at_ += k;
    }
    size_t left() const { return n_ - at_; }
    size_t pos() const { return at_; }
    bool done() const { return at_ == n_; }

private:
    void need(size_t k) const {
        if (k > n_ - at_) throw FormatError(code_, "payload ends early");
    }
    const uint8_t* p_;
    size_t n_, at_ = 0;
    FormatErrorCode code_;
};

// A count read from the payload must fit in what is left (per item bytes)
// before anything is allocated for it.
size_t bounded_count(const Source& r, uint64_t count, uint64_t item_bytes) {
    if (count > r.left() / item_bytes) throw FormatError(FormatErrorCode::CountOverflow, "declared count needs more bytes than the section holds");
    return static_cast<size_t>(count);
}

void put_section(Sink& out, const char* tag, const std::vector<uint8_t>& payload) {
    out.raw(tag, 4);
    out.put<uint64_t>(payload.size());
    out.raw(payload.data(), payload.size());
}

// CAMS: u64 count, per view u64 id, f64 fx fy cx cy, u32 w h, f64 q[4], f64 t[3], u32 len + path.
std::vector<uint8_t> cams_payload(const std::vector<CameraView>& views) {
    Sink s;
    s.put<uint64_t>(views.size());
    for (const CameraView& v : views) {
        s.put<uint64_t>(v.view_id);
        for (double d : {v.fx, v.fy, v.cx, v.cy}) s.put<double>(d);
        s.put<uint32_t>(v.width);
        s.put<uint32_t>(v.height);
        for (double d : v.rotation_q) s.put<double>(d);
        for (double d : v.translation) s.put<double>(d);
        s.put<uint32_t>(static_cast<uint32_t>(v.image_path.size()));
        s.raw(v.image_path.data(), v.image_path.size());
    }
    return std::move(s.bytes());
}

// PNTS: u64 count, per point f32 position[3], u8 rgb[3].
std::vector<uint8_t> pnts_payload(const std::vector<ScenePoint>& points) {
    Sink s;
    s.put<uint64_t>(points.size());
    for (const ScenePoint& p : points) {
        for (float f : p.position) s.put<float>(f);
        s.raw(p.rgb.data(), 3);
    }
    return std::move(s.bytes());
}

// GSPL: u64 count, u32 feature width, u64 ids, then the f32 arrays positions,
// rotations, log-scales, features, opacity logits (each row-interleaved).
std::vector<uint8_t> gspl_payload(const GaussianCloud& c) {
    Sink s;
    s.put<uint64_t>(c.size());
    s.put<uint32_t>(static_cast<uint32_t>(c.feature_dim()));
    for (uint64_t id : c.ids) s.put<uint64_t>(id);
    for (const auto* arr : {&c.positions, &c.rotations, &c.log_scales, &c.features, &c.opacity_logits})
        for (double v : *arr) s.put<float>(static_cast<float>(v));
    return std::move(s.bytes());
}

std::vector<CameraView> read_cams(Source& r) {
    const size_t n = bounded_count(r, r.get<uint64_t>(), 77);  // fixed bytes per view before the path
    std::vector<CameraView> views(n);
    for (CameraView& v : views) {
        v.view_id = r.get<uint64_t>();
        v.fx = r.get<double>();
        v.fy = r.get<double>();
        v.cx = r.get<double>();
        v.cy = r.get<double>();
        v.width = r.get<uint32_t>();
        v.height = r.get<uint32_t>();
        Vec4 q;
        for (double& d : q) d = r.get<double>();
        v.set_rotation_quat(q);
        for (double& d : v.translation) d = r.get<double>();
        const uint32_t len = r.get<uint32_t>();
        v.image_path.resize(len);
        r.take(v.image_path.data(), len);
    }
    return views;
}

std::vector<ScenePoint> read_pnts(Source& r) {
    const size_t n = bounded_count(r, r.get<uint64_t>(), 15);
    std::vector<ScenePoint> points(n);
    for (ScenePoint& p : points) {
        for (float& f : p.position) f = r.get<float>();
        r.take(p.rgb.data(), 3);
    }
    return points;
}

GaussianCloud read_gspl(Source& r) {
    const uint64_t count = r.get<uint64_t>();
    const uint32_t fd = r.get<uint32_t>();
    if (fd != static_cast<uint32_t>(kFeatureDimDeg0) && fd != static_cast<uint32_t>(kFeatureDimDeg1))
        throw FormatError(FormatErrorCode::BadHeader, "GSPL feature width is neither 3 nor 12");
    const size_t n = bounded_count(r, count, 8 + 4 * (11 + static_cast<uint64_t>(fd)));
    GaussianCloud c(static_cast<int>(fd));
    c.ids.resize(n);
    c.positions.resize(3 * n);
    c.rotations.resize(4 * n);
    c.log_scales.resize(3 * n);
    c.features.resize(n * fd);
    c.opacity_logits.resize(n);
    for (uint64_t& id : c.ids) id = r.get<uint64_t>();
    for (auto* arr : {&c.positions, &c.rotations, &c.log_scales, &c.features, &c.opacity_logits})
        for (double& v : *arr) v = r.get<float>();
    for (size_t i = 1; i < n; ++i)
        if (c.ids[i] <= c.ids[i - 1]) throw FormatError(FormatErrorCode::NonMonotoneIds, "GSPL ids must increase strictly");
    return c;
}

void check_status(int st) {
    if (st != BSG_OK) throw std::runtime_error(bsg_last_error());
}

}  // namespace

std::vector<uint8_t> encode_scene(const SceneDataset& scene) {  // scene_io.cpp:124-132
    Sink out;
    out.raw("DOGS", 4);
    out.put<uint32_t>(kSceneFormatVersion);
    put_section(out, "CAMS", cams_payload(scene.views));
    put_section(out, "PNTS", pnts_payload(scene.points));
    if (scene.has_checkpoint) put_section(out, "GSPL", gspl_payload(scene.checkpoint));
    return std::move(out.bytes());
}

SceneDataset decode_scene(const uint8_t* data, size_t size) {  // scene_io.cpp:134-176
    Source top(data, size, FormatErrorCode::TruncatedBuffer);
    char magic[4];
    top.take(magic, 4);
    if (std::memcmp(magic, "DOGS", 4) != 0) throw FormatError(FormatErrorCode::BadMagic, "missing DOGS magic");
    const uint32_t version = top.get<uint32_t>();
    if (version != kSceneFormatVersion)
        throw FormatError(FormatErrorCode::UnsupportedVersion, "DOGS version " + std::to_string(version));
    SceneDataset scene;
    bool cams = false, pnts = false, gspl = false;
    while (!top.done()) {
        char tag[4];
        top.take(tag, 4);
        const uint64_t len = top.get<uint64_t>();
        if (len > top.left()) throw FormatError(FormatErrorCode::TruncatedSection, "section length runs past the container");
        Source sec(data + top.pos(), static_cast<size_t>(len), FormatErrorCode::TruncatedSection);
        top.skip(static_cast<size_t>(len));
        auto once = [&](bool& seen, const char* name) {
            if (seen) throw FormatError(FormatErrorCode::BadHeader, std::string(name) + " section appears twice");
            seen = true;
        };
        if (std::memcmp(tag, "CAMS", 4) == 0) {
            once(cams, "CAMS");
            scene.views = read_cams(sec);
        } else if (std::memcmp(tag, "PNTS", 4) == 0) {
            once(pnts, "PNTS");
            scene.points = read_pnts(sec);
        } else if (std::memcmp(tag, "GSPL", 4) == 0) {
            once(gspl, "GSPL");
            scene.checkpoint = read_gspl(sec);
            scene.has_checkpoint = true;
        } else {
            throw FormatError(FormatErrorCode::UnknownSection, "section tag " + std::string(tag, 4) + " is not CAMS / PNTS / GSPL");
        }
        if (!sec.done()) throw FormatError(FormatErrorCode::TruncatedSection, "section payload longer than its contents");
    }
    return scene;
}

void save_scene(const std::string& path, const SceneDataset& scene) {
    const std::vector<uint8_t> bytes = encode_scene(scene);
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("save_scene: cannot create " + path);
    const size_t wrote = std::fwrite(bytes.data(), 1, bytes.size(), f);
    const bool ok = std::fclose(f) == 0 && wrote == bytes.size();
    if (!ok) throw std::runtime_error("save_scene: short write to " + path);
}

SceneDataset load_scene(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("load_scene: cannot open " + path);
    std::vector<uint8_t> bytes;
    uint8_t chunk[1 << 16];
    size_t got = 0;
    while ((got = std::fread(chunk, 1, sizeof(chunk), f)) > 0) bytes.insert(bytes.end(), chunk, chunk + got);
    const bool err = std::ferror(f) != 0;
    std::fclose(f);
    if (err) throw std::runtime_error("load_scene: read error on " + path);
    return decode_scene(bytes.data(), bytes.size());
}

GaussianCloud narrow_to_f32(const GaussianCloud& cloud) {  // scene_io.cpp:230-241
    GaussianCloud out = cloud;
    for (auto* arr : {&out.positions, &out.rotations, &out.log_scales, &out.features, &out.opacity_logits})
        for (double& v : *arr) v = static_cast<float>(v);
    return out;
}

std::vector<uint8_t> encode_gspl_device(bsg_ctx* ctx) {
    size_t len = 0;
    check_status(bsg_encode_gspl(ctx, nullptr, 0, &len));
    std::vector<uint8_t> out(len);
    check_status(bsg_encode_gspl(ctx, out.data(), out.size(), &len));
    return out;
}

void save_model(const std::string& path, const GaussianCloud& model) {  // main.cpp:353-357
    SceneDataset d;
    d.has_checkpoint = true;
    d.checkpoint = narrow_to_f32(model);
    save_scene(path, d);
}

}  // namespace blocksplat
