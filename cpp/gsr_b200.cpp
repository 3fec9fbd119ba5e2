// gsr_b200.cpp — the C++ host side of the drop-in (cpp/gsr_b200.hpp) over the C ABI
// (include/tgs.h).  Marshals the reference's AoS Eigen structs into the .gsb record layout
// (scene_io.hpp:38-42), validates options exactly where the reference does (render.cpp:9-11,
// binning.cpp:22-30), and maps tgs_status onto the reference's exception types.
#include "gsr_b200.hpp"

#include <cmath>
#include <fstream>
#include <iterator>
#include <cstring>
#include <string>

#include "../include/tgs.h"

namespace gsr {
namespace {

thread_local int t_device = 0;
thread_local b200::StageTimes t_times{};

[[noreturn]] void raise(tgs_status st) {
    const std::string msg = tgs_last_error();
    if (st == TGS_ERR_VALIDATION) throw ValidationError(msg);
    if (st == TGS_ERR_FORMAT) throw FormatError(msg);
    throw DeviceError(msg);
}

void check(tgs_status st) {
    if (st != TGS_OK) raise(st);
}

// One context per (thread, device): contexts own a stream and are used by one thread at a time.
struct CtxHolder {
    tgs_ctx* ctx = nullptr;
    int device = -1;
    ~CtxHolder() {
        if (ctx) tgs_ctx_destroy(ctx);
    }
    tgs_ctx* get(int device_) {
        if (ctx && device == device_) return ctx;
        if (ctx) tgs_ctx_destroy(ctx);
        ctx = nullptr;
        check(tgs_ctx_create(device_, &ctx));
        device = device_;
        return ctx;
    }
};
thread_local CtxHolder t_ctx;

// scene_io .gsb record order: mean3 scale3 quat(w,x,y,z) opacity sh_dc3 [sh_rest45]
std::vector<float> to_records(const std::vector<Gaussian3D>& scene, int& sh_degree) {
    sh_degree = 0;
    if (!scene.empty()) {
        // eval_sh_color (projection.cpp:55-77) takes sh_rest per Gaussian: a scene where only
        // some Gaussians carry it is uploaded as degree 3 with zero coefficients for the others,
        // which adds only +-0 to their colour (bit-identical to the degree-0 evaluation)
        for (const auto& g : scene)
            if (g.sh_rest.has_value()) sh_degree = 3;
    }
    const size_t rf = sh_degree == 3 ? 59 : 14;
    std::vector<float> rec(scene.size() * rf);
    for (size_t i = 0; i < scene.size(); ++i) {
        const Gaussian3D& g = scene[i];
        float* r = &rec[i * rf];
        r[0] = g.mean.x(), r[1] = g.mean.y(), r[2] = g.mean.z();
        r[3] = g.scale.x(), r[4] = g.scale.y(), r[5] = g.scale.z();
        r[6] = g.rotation.w(), r[7] = g.rotation.x(), r[8] = g.rotation.y(), r[9] = g.rotation.z();
        r[10] = g.opacity;
        r[11] = g.sh_dc.x(), r[12] = g.sh_dc.y(), r[13] = g.sh_dc.z();
        if (sh_degree == 3 && g.sh_rest.has_value()) std::memcpy(r + 14, g.sh_rest->data(), sizeof(float) * kShRestCoeffs);
    }
    return rec;
}

tgs_camera to_c(const Camera& cam) {
    tgs_camera c{};
    for (int r = 0; r < 4; ++r)
        for (int k = 0; k < 4; ++k) c.view[r * 4 + k] = cam.view(r, k);
    c.focal_x = cam.focal_x;
    c.focal_y = cam.focal_y;
    c.width = cam.width;
    c.height = cam.height;
    c.near_ = cam.near;
    c.far_ = cam.far;
    return c;
}

tgs_options to_c(const RenderOptions& opt) {
    tgs_options o{};
    o.backend = opt.backend == Backend::scalar ? TGS_BACKEND_SCALAR : TGS_BACKEND_TENSOR;
    o.mode = opt.mode == PrecisionMode::fp16 ? TGS_MODE_FP16 : TGS_MODE_FP32;
    o.group_size = opt.group_size;
    o.workers = opt.workers;
    o.chunk_len = opt.chunk_len;
    o.alpha_skip = opt.constants.alpha_skip;
    o.alpha_clamp = opt.constants.alpha_clamp;
    o.t_terminate = opt.constants.t_terminate;
    return o;
}

RenderResult finish(const Camera& cam, std::vector<float>&& rgb, const tgs_stats& st) {
    RenderResult res;
    res.image.width = cam.width;
    res.image.height = cam.height;
    res.image.rgb = std::move(rgb);
    res.projection.input = st.input;
    res.projection.culled = st.culled;
    res.projection.dropped_degenerate = st.dropped_degenerate;
    res.entries = st.entries;
    res.tile_appearances = st.tile_appearances;
    res.ops.fragment_ops = st.fragment_ops;
    res.ops.chunk_loads = st.chunk_loads;
    res.ops.skipped_pairs = st.skipped_pairs;
    res.ops.used_lanes = st.used_lanes;
    res.ops.total_lanes = st.total_lanes;
    t_times = {st.ms_preprocess, st.ms_binning, st.ms_sort, st.ms_raster, st.ms_total};
    return res;
}

}  // namespace

RenderResult render(const std::vector<Gaussian3D>& scene, const Camera& cam, const RenderOptions& opt) {
    int deg = 0;
    const std::vector<float> rec = to_records(scene, deg);
    tgs_ctx* ctx = t_ctx.get(t_device);
    const tgs_camera c = to_c(cam);
    const tgs_options o = to_c(opt);
    std::vector<float> rgb(static_cast<size_t>(cam.width > 0 ? cam.width : 0) * (cam.height > 0 ? cam.height : 0) * 3);
    tgs_stats st{};
    check(tgs_render_records(ctx, rec.data(), static_cast<int64_t>(scene.size()), deg, &c, &o, rgb.data(), &st));
    return finish(cam, std::move(rgb), st);
}

// ---- stage API over the C ABI --------------------------------------------------------------
namespace {
tgs_projected to_c(const ProjectedGaussian& p) {
    tgs_projected o{};
    o.mean2d[0] = p.mean2d.x();
    o.mean2d[1] = p.mean2d.y();
    o.conic[0] = p.conic_a;
    o.conic[1] = p.conic_b;
    o.conic[2] = p.conic_c;
    o.color[0] = p.color.x();
    o.color[1] = p.color.y();
    o.color[2] = p.color.z();
    o.opacity = p.opacity;
    o.depth = p.depth;
    o.radius = p.radius;
    return o;
}
ProjectedGaussian from_c(const tgs_projected& o) {
    ProjectedGaussian p;
    p.mean2d = Eigen::Vector2f(o.mean2d[0], o.mean2d[1]);
    p.conic_a = o.conic[0];
    p.conic_b = o.conic[1];
    p.conic_c = o.conic[2];
    p.color = Eigen::Vector3f(o.color[0], o.color[1], o.color[2]);
    p.opacity = o.opacity;
    p.depth = o.depth;
    p.radius = o.radius;
    return p;
}
std::vector<tgs_projected> to_c(const std::vector<ProjectedGaussian>& v) {
    std::vector<tgs_projected> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) o[i] = to_c(v[i]);
    return o;
}
static_assert(sizeof(GroupEntry) == sizeof(tgs_group_entry) && sizeof(KeyedEntry) == sizeof(tgs_keyed_entry),
              "entry layouts must match the C ABI");

ImageBuffer rasterize_lists(const SortedGroupLists& lists, const std::vector<ProjectedGaussian>& projected,
                            const GroupConfig& cfg, Backend backend, const RasterConstants& k, PrecisionMode mode,
                            int workers, int chunk_len) {
    cfg.validate();
    RenderOptions opt;
    opt.backend = backend;
    opt.mode = mode;
    opt.group_size = cfg.group_h;
    opt.workers = workers;
    opt.chunk_len = chunk_len;
    opt.constants = k;
    const tgs_options o = to_c(opt);
    const std::vector<tgs_projected> p = to_c(projected);
    ImageBuffer img(cfg.image_width, cfg.image_height);
    check(tgs_rasterize_lists(t_ctx.get(t_device), reinterpret_cast<const tgs_group_entry*>(lists.entries.data()),
                              static_cast<int64_t>(lists.entries.size()), lists.offsets.data(),
                              static_cast<int64_t>(lists.offsets.size()), p.data(), static_cast<int64_t>(p.size()),
                              cfg.image_width, cfg.image_height, &o, img.rgb.data()));
    return img;
}
}  // namespace

std::vector<ProjectedGaussian> project_scene(const std::vector<Gaussian3D>& scene, const Camera& cam, int workers,
                                             ProjectionStats* stats) {
    if (workers < 1) throw ValidationError("project_scene: workers must be >= 1");
    int deg = 0;
    const std::vector<float> rec = to_records(scene, deg);
    tgs_ctx* ctx = t_ctx.get(t_device);
    const tgs_camera c = to_c(cam);
    int64_t n = 0;
    tgs_stats st{};
    check(tgs_project_scene(ctx, rec.data(), static_cast<int64_t>(scene.size()), deg, &c, nullptr, 0, &n, &st));
    std::vector<tgs_projected> out(static_cast<size_t>(n));
    if (n) check(tgs_read_projected(ctx, out.data(), n, &n));
    if (stats) {
        stats->input = st.input;
        stats->culled = st.culled;
        stats->dropped_degenerate = st.dropped_degenerate;
    }
    std::vector<ProjectedGaussian> r(out.size());
    for (size_t i = 0; i < out.size(); ++i) r[i] = from_c(out[i]);
    return r;
}

GroupConfig GroupConfig::square(int g, int image_width, int image_height) {
    GroupConfig cfg;
    cfg.group_h = g;
    cfg.group_w = g;
    cfg.image_width = image_width;
    cfg.image_height = image_height;
    cfg.validate();
    return cfg;
}

void GroupConfig::validate() const {
    if (image_width <= 0 || image_height <= 0) throw ValidationError("GroupConfig: image dimensions must be positive");
    if (!(group_h == group_w && (group_h == 1 || group_h == 2 || group_h == 4)))
        throw ValidationError("GroupConfig: supported group sizes are 1x1, 2x2, 4x4");
}

TileRect tiles_overlapped(const ProjectedGaussian& p, const GroupConfig& cfg) {
    // floor((mean -+ r) / 16): the same IEEE operations the GPU binning uses
    const float r = static_cast<float>(p.radius);
    TileRect t;
    t.min_x = std::max(static_cast<int>(std::floor((p.mean2d.x() - r) / kTileSize)), 0);
    t.max_x = std::min(static_cast<int>(std::floor((p.mean2d.x() + r) / kTileSize)), cfg.tiles_x() - 1);
    t.min_y = std::max(static_cast<int>(std::floor((p.mean2d.y() - r) / kTileSize)), 0);
    t.max_y = std::min(static_cast<int>(std::floor((p.mean2d.y() + r) / kTileSize)), cfg.tiles_y() - 1);
    return t;
}

std::vector<KeyedEntry> build_group_entries(const std::vector<ProjectedGaussian>& projected, const GroupConfig& cfg) {
    cfg.validate();
    tgs_ctx* ctx = t_ctx.get(t_device);
    const std::vector<tgs_projected> p = to_c(projected);
    int64_t n = 0;
    check(tgs_build_group_entries(ctx, p.data(), static_cast<int64_t>(p.size()), cfg.image_width, cfg.image_height,
                                  cfg.group_h, nullptr, 0, &n));
    std::vector<KeyedEntry> out(static_cast<size_t>(n));
    if (n)
        check(tgs_build_group_entries(ctx, p.data(), static_cast<int64_t>(p.size()), cfg.image_width,
                                      cfg.image_height, cfg.group_h, reinterpret_cast<tgs_keyed_entry*>(out.data()),
                                      n, &n));
    return out;
}

SortedGroupLists sort_entries(std::vector<KeyedEntry> entries, const GroupConfig& cfg) {
    cfg.validate();
    SortedGroupLists lists;
    lists.entries.resize(entries.size());
    lists.offsets.assign(static_cast<size_t>(cfg.group_count()) + 1, 0u);
    check(tgs_sort_entries(t_ctx.get(t_device), reinterpret_cast<const tgs_keyed_entry*>(entries.data()),
                           static_cast<int64_t>(entries.size()), cfg.image_width, cfg.image_height, cfg.group_h,
                           reinterpret_cast<tgs_group_entry*>(lists.entries.data()), lists.offsets.data(),
                           static_cast<int64_t>(lists.offsets.size())));
    return lists;
}

ImageBuffer rasterize_tiles_scalar(const SortedGroupLists& lists, const std::vector<ProjectedGaussian>& projected,
                                   const GroupConfig& cfg, const RasterConstants& k, PrecisionMode mode, int workers) {
    return rasterize_lists(lists, projected, cfg, Backend::scalar, k, mode, workers, kFragmentDim);
}

ImageBuffer rasterize_groups_tensor(const SortedGroupLists& lists, const std::vector<ProjectedGaussian>& projected,
                                    const GroupConfig& cfg, const TensorRasterOptions& opt, OpReport* ops) {
    (void)ops;
    return rasterize_lists(lists, projected, cfg, Backend::tensor, opt.constants, opt.mode, opt.workers,
                           opt.chunk_len);
}

namespace b200 {

void set_device(int device) { t_device = device; }
StageTimes last_stage_times() { return t_times; }

struct DeviceScene::Impl {
    tgs_ctx* ctx = nullptr;
    tgs_scene* scene = nullptr;
};

DeviceScene::DeviceScene(const std::vector<Gaussian3D>& scene, int device) : impl_(new Impl) {
    int deg = 0;
    const std::vector<float> rec = to_records(scene, deg);
    check(tgs_ctx_create(device, &impl_->ctx));
    const tgs_status st = tgs_scene_upload(impl_->ctx, rec.data(), static_cast<int64_t>(scene.size()), deg,
                                           &impl_->scene);
    if (st != TGS_OK) {
        tgs_ctx_destroy(impl_->ctx);
        impl_->ctx = nullptr;
        raise(st);
    }
}

DeviceScene::~DeviceScene() {
    if (impl_->scene) tgs_scene_free(impl_->scene);
    if (impl_->ctx) tgs_ctx_destroy(impl_->ctx);
}

RenderResult DeviceScene::render(const Camera& cam, const RenderOptions& opt) {
    const tgs_camera c = to_c(cam);
    const tgs_options o = to_c(opt);
    std::vector<float> rgb(static_cast<size_t>(cam.width > 0 ? cam.width : 0) * (cam.height > 0 ? cam.height : 0) * 3);
    tgs_stats st{};
    check(tgs_render(impl_->ctx, impl_->scene, &c, &o, rgb.data(), &st));
    return finish(cam, std::move(rgb), st);
}

}  // namespace b200
// ---- .gsb scene files (scene_io.cpp:43-136 semantics) ------------------------------------------
namespace {
constexpr char kGsbMagic[4] = {'G', 'S', 'B', '1'};
constexpr size_t kGsbHeader = 16;

std::uint32_t le_u32(const unsigned char* p) {
    return (std::uint32_t)p[0] | ((std::uint32_t)p[1] << 8) | ((std::uint32_t)p[2] << 16) | ((std::uint32_t)p[3] << 24);
}
float le_f32(const unsigned char* p) {
    const std::uint32_t u = le_u32(p);
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
void put_le(std::string& out, std::uint32_t v) {
    for (int k = 0; k < 4; ++k) out.push_back(static_cast<char>((v >> (8 * k)) & 0xffu));
}
void put_le(std::string& out, float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    put_le(out, u);
}
}  // namespace

std::vector<Gaussian3D> load_scene(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw FormatError("cannot open scene file: " + path);
    const std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    const auto* b = reinterpret_cast<const unsigned char*>(bytes.data());
    if (bytes.size() < kGsbHeader)
        throw FormatError(path + ": truncated header at byte offset " + std::to_string(bytes.size()) + " (need 16)");
    if (std::memcmp(b, kGsbMagic, 4) != 0) throw FormatError(path + ": bad magic at byte offset 0");
    const std::uint32_t count = le_u32(b + 4), degree = le_u32(b + 8);
    if (degree != 0 && degree != 3) throw FormatError(path + ": unsupported sh_degree at byte offset 8");
    const size_t rec_bytes = (degree == 3 ? 59u : 14u) * 4u;
    const size_t need = kGsbHeader + static_cast<size_t>(count) * rec_bytes;
    if (bytes.size() < need)
        throw FormatError(path + ": truncated payload at byte offset " + std::to_string(bytes.size()) + " (need " +
                          std::to_string(need) + ")");
    std::vector<Gaussian3D> scene(count);
    for (std::uint32_t i = 0; i < count; ++i) {
        const unsigned char* p = b + kGsbHeader + static_cast<size_t>(i) * rec_bytes;
        Gaussian3D& g = scene[i];
        g.mean = Eigen::Vector3f(le_f32(p), le_f32(p + 4), le_f32(p + 8));
        g.scale = Eigen::Vector3f(le_f32(p + 12), le_f32(p + 16), le_f32(p + 20));
        g.rotation = Eigen::Quaternionf(le_f32(p + 24), le_f32(p + 28), le_f32(p + 32), le_f32(p + 36));
        g.opacity = le_f32(p + 40);
        g.sh_dc = Eigen::Vector3f(le_f32(p + 44), le_f32(p + 48), le_f32(p + 52));
        if (degree == 3) {
            std::array<float, kShRestCoeffs> rest{};
            for (int k = 0; k < kShRestCoeffs; ++k) rest[static_cast<size_t>(k)] = le_f32(p + 56 + 4 * k);
            g.sh_rest = rest;
        }
        const std::string at = path + ": scene record " + std::to_string(i);
        if (!(g.opacity >= 0.0f && g.opacity <= 1.0f)) throw ValidationError(at + ": opacity outside [0,1]");
        if (!g.mean.allFinite() || !g.scale.allFinite()) throw ValidationError(at + ": non-finite mean or scale");
        if (!(g.scale.minCoeff() > 0.0f)) throw ValidationError(at + ": non-positive scale");
        // the reference renormalises only drifted quaternions, so unit ones round-trip bit-exactly
        const float n = g.rotation.norm();
        if (!(n > 0.0f) || !std::isfinite(n))
            throw ValidationError("scene record " + std::to_string(i) + ": quaternion has non-finite or zero norm");
        if (std::fabs(n - 1.0f) > 1e-6f) g.rotation.coeffs() /= n;
    }
    return scene;
}

void save_scene(const std::vector<Gaussian3D>& gaussians, const std::string& path) {
    size_t with_rest = 0;
    for (const auto& g : gaussians) with_rest += g.sh_rest.has_value() ? 1u : 0u;
    if (with_rest != 0 && with_rest != gaussians.size())
        throw ValidationError("save_scene: mixed sh_rest presence across records");
    const std::uint32_t degree = with_rest != 0 ? 3u : 0u;
    std::string out(kGsbMagic, 4);
    put_le(out, static_cast<std::uint32_t>(gaussians.size()));
    put_le(out, degree);
    put_le(out, 0u);
    for (const auto& g : gaussians) {
        for (int k = 0; k < 3; ++k) put_le(out, g.mean[k]);
        for (int k = 0; k < 3; ++k) put_le(out, g.scale[k]);
        put_le(out, g.rotation.w());
        put_le(out, g.rotation.x());
        put_le(out, g.rotation.y());
        put_le(out, g.rotation.z());
        put_le(out, g.opacity);
        for (int k = 0; k < 3; ++k) put_le(out, g.sh_dc[k]);
        if (degree == 3)
            for (float v : *g.sh_rest) put_le(out, v);
    }
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw FormatError("cannot open for writing: " + path);
    f.write(out.data(), static_cast<std::streamsize>(out.size()));
    if (!f) throw FormatError("write failed: " + path);
}

}  // namespace gsr
