// gsr_b200.cpp — the C++ host side of the drop-in (cpp/gsr_b200.hpp) over the C ABI
// (include/tgs.h).  Marshals the reference's AoS Eigen structs into the .gsb record layout
// (scene_io.hpp:38-42), validates options exactly where the reference does (render.cpp:9-11,
// binning.cpp:22-30), and maps tgs_status onto the reference's exception types.
#include "gsr_b200.hpp"

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
        const bool first = scene.front().sh_rest.has_value();
        for (const auto& g : scene)
            if (g.sh_rest.has_value() != first)
                throw ValidationError("render: mixed sh_rest presence across Gaussians");
        sh_degree = first ? 3 : 0;
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
        if (sh_degree == 3) std::memcpy(r + 14, g.sh_rest->data(), sizeof(float) * kShRestCoeffs);
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
}  // namespace gsr
