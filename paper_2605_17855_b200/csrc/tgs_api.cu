// libtgs host runtime and C ABI (include/tgs.h): contexts, device scenes, the per-frame
// pipeline (preprocess -> depth presort -> entry scan -> emission -> group sort -> ranges ->
// raster), capacity management, readback and error mapping.
//
// Reference entry point: proj/src/render.cpp:7-35 (gsr::render).  Validation mirrors it:
// scalar backend requires G == 1 (render.cpp:9-10), workers >= 1 (:11), GroupConfig limits
// (binning.cpp:22-30), non-positive scales of visible splats (projection.cpp:37) and
// non-finite/negative depths of binned splats (binning.cpp:78-83) -> TGS_ERR_VALIDATION.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

namespace tgs {

namespace err_state {
thread_local std::string g_err;
}
using err_state::g_err;

tgs_status set_err(tgs_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

tgs_status cuda_fail(cudaError_t e, const char* expr, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                  cudaGetErrorString(e), file, line, expr);
    return set_err(e == cudaErrorMemoryAllocation ? TGS_ERR_OOM : TGS_ERR_CUDA, buf);
}

// Grow-only device buffer.
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t n) {
        if (n <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, n);
        if (e == cudaSuccess) bytes = n;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

}  // namespace tgs

using namespace tgs;

struct tgs_scene;
struct tgs_ctx;
constexpr int kBatchLanes = 3;  // frames in flight in tgs_render_batch

struct tgs_scene {
    tgs_ctx* ctx = nullptr;
    int device = 0;
    int64_t n = 0;
    int sh_degree = 0;
    DBuf planes;  // pos_op | quat | scale_dcr | dc_gb | sh_rest
    DevScene dev() const {
        DevScene s;
        char* b = planes.as<char>();
        const size_t n4 = (size_t)n * sizeof(float4);
        s.pos_op = reinterpret_cast<const float4*>(b);
        s.quat = reinterpret_cast<const float4*>(b + n4);
        s.scale_dcr = reinterpret_cast<const float4*>(b + 2 * n4);
        s.dc_gb = reinterpret_cast<const float2*>(b + 3 * n4);
        s.sh_rest = sh_degree == 3 ? reinterpret_cast<const float4*>(b + 3 * n4 + (size_t)n * sizeof(float2)) : nullptr;
        s.n = (int)n;
        s.sh_degree = sh_degree;
        return s;
    }
};

struct tgs_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[6] = {};
    // per-frame buffers
    DBuf fc;            // FrameCounters
    DBuf proj;          // mc | co | col (capacity n)
    DBuf pre_keys[2], pre_vals[2];
    DBuf rect, rrect;   // tile rect per compacted splat / per rank
    DBuf list;          // sorted group lists (splat indices)
    DBuf rowlist;       // group-row lists (binning level 1): splat-index plane, column-range plane
    DBuf hist, bsum;    // counting-sort [group][chunk] matrix and its scan block sums
    DBuf ghist, offsets, order;
    DBuf ucost;         // per unit, list entries the last frame walked (schedule feedback)
    uint64_t ucost_key = 0;  // geometry the feedback belongs to (0: none)
    // level-1 binning chunks: sized from the group-row entries of the last synced frame of the
    // same geometry (rc_key), so a block's share of them fits its shared-memory stage
    uint64_t rc_key = 0, rc_pending_key = 0;
    uint64_t rc_entries = 0;
    int row_chunks = 0;
    DBuf image;
    DBuf scratch_records;
    DBuf stg[8];  // stage-API scratch (tgs_build_group_entries / tgs_sort_entries / tgs_rasterize_lists)
    FrameCounters* h_fc = nullptr;  // pinned
    uint32_t capacity = 0;          // entry capacity
    int64_t proj_cap = 0;
    // last frame
    const tgs_scene* last_scene = nullptr;
    tgs_camera last_cam{};
    tgs_options last_opt{};
    GroupGeom last_gg{};
    int last_band0 = 0, last_band1 = 0;
    int image_rows = 0;
    bool pending = false;
    // camera-batch lanes: extra contexts (own stream and buffers) on the same device that render
    // the parent's scenes, so frames of a batch overlap (tgs_render_batch)
    tgs_ctx* lanes[kBatchLanes - 1] = {};
    tgs_ctx* parent = nullptr;
    int tile_cull = 1;  // tgs_set_tile_cull
    // CUDA graph of the per-frame launch sequence (tgs_set_graphs): captured on the second frame
    // of an unchanged configuration, replayed with the camera argument of preprocess updated
    int graphs = 1;
    int exact = 0;  // tgs_set_exact_emulation: fp32 frames through the exact-emulation rasteriser
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t ggraph = nullptr;
    cudaGraphNode_t gpre = nullptr;   // preprocess kernel node
    PreprocessArgs gpa{};             // its captured arguments (camera replaced per launch)
    std::string gkey;                 // configuration the graph was captured for
    std::string pkey;                 // configuration of the previous frame
    uint32_t acked_overflow = 0, acked_invalid = 0;  // sticky frame-failure counters already reported
    tgs_scene* scratch_scene = nullptr;
};

namespace tgs {
namespace api {

int ceil_log2(int n) {
    int b = 0;
    while ((1 << b) < n) ++b;
    return b;
}

tgs_status validate_options(const tgs_camera* cam, const tgs_options* opt) {
    if (!cam || !opt) return set_err(TGS_ERR_VALIDATION, "render: null camera or options");
    if (opt->backend != TGS_BACKEND_SCALAR && opt->backend != TGS_BACKEND_TENSOR)
        return set_err(TGS_ERR_VALIDATION, "render: unknown backend");
    if (opt->backend == TGS_BACKEND_SCALAR && opt->group_size != 1)
        return set_err(TGS_ERR_VALIDATION, "render: the scalar backend requires group size 1");
    if (opt->workers < 1) return set_err(TGS_ERR_VALIDATION, "render: workers must be >= 1");
    if (cam->width <= 0 || cam->height <= 0)
        return set_err(TGS_ERR_VALIDATION, "GroupConfig: image dimensions must be positive");
    if (!(opt->group_size == 1 || opt->group_size == 2 || opt->group_size == 4))
        return set_err(TGS_ERR_VALIDATION, "GroupConfig: supported group sizes are 1x1, 2x2, 4x4");
    return TGS_OK;
}

GroupGeom make_geom(int g, int w, int h, int band0, int band1) {
    GroupGeom gg;
    gg.g = g;
    gg.width = w;
    gg.height = h;
    gg.tiles_x = (w + kTile - 1) / kTile;
    gg.tiles_y = (h + kTile - 1) / kTile;
    gg.groups_x = (gg.tiles_x + g - 1) / g;
    gg.groups_y = (gg.tiles_y + g - 1) / g;
    gg.band_gy0 = band0;
    gg.band_gy1 = band1;
    gg.n_groups_band = gg.groups_x * (band1 - band0);
    return gg;
}

DevCamera make_dev_camera(const tgs_camera* c) {
    DevCamera d;
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) d.r[i][j] = c->view[i * 4 + j];
        d.t[i] = c->view[i * 4 + 3];
    }
    d.fx = c->focal_x;
    d.fy = c->focal_y;
    d.width = c->width;
    d.height = c->height;
    d.near_ = c->near_;
    d.far_ = c->far_;
    return d;
}

DevProjected dev_proj(tgs_ctx* ctx) {
    DevProjected p;
    float4* b = ctx->proj.as<float4>();
    p.mc = b;
    p.co = b + ctx->proj_cap;
    p.col = b + 2 * ctx->proj_cap;
    return p;
}

tgs_status record_frame(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam, const tgs_options* opt,
                        const GroupGeom& gg, bool feedback, int row0, size_t h1, size_t h2, int n_alloc,
                        int units_per_group);

// Stage events: recorded as event-record nodes when the frame is captured into a graph (a plain
// cudaEventRecord on a capturing stream only expresses a dependency and leaves the event unset).
cudaError_t record_event(cudaEvent_t ev, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t e = cudaStreamIsCapturing(s, &cs);
    if (e != cudaSuccess) return e;
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal)
                                               : cudaEventRecord(ev, s);
}

// Enqueue one frame (or band) on ctx->stream.
tgs_status enqueue_frame(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam,
                         const tgs_options* opt, int band0, int band1) {
    tgs_status st = validate_options(cam, opt);
    if (st != TGS_OK) return st;
    if (!scene || (scene->ctx != ctx && scene->ctx != ctx->parent))
        return set_err(TGS_ERR_VALIDATION, "render: scene belongs to another context");
    const GroupGeom full = make_geom(opt->group_size, cam->width, cam->height, 0, 0);
    if (band1 <= 0) {
        band0 = 0;
        band1 = full.groups_y;
    }
    if (band0 < 0 || band1 > full.groups_y || band0 >= band1)
        return set_err(TGS_ERR_VALIDATION, "render_band: group-row band out of range");
    const GroupGeom gg = make_geom(opt->group_size, cam->width, cam->height, band0, band1);
    const int n_groups = gg.n_groups_band;
    if (n_groups > 49152)
        return set_err(TGS_ERR_VALIDATION, "render: more than 49152 groups in one frame/band; use bands");
    // binning lanes own group columns / band rows lane + 32k, k < 16 (tgs_binning.cu)
    if (gg.groups_x > 512)
        return set_err(TGS_ERR_VALIDATION, "render: more than 512 group columns (image wider than 8192 px at "
                                           "G=1); use a larger group size");
    if (band1 - band0 > 512)
        return set_err(TGS_ERR_VALIDATION, "render: more than 512 group rows in one frame/band; use bands");
    cudaStream_t s = ctx->stream;
    const int64_t n = scene->n;
    const int n_alloc = (int)std::max<int64_t>(n, 1);

    // ---- buffers ----
    if (ctx->proj_cap < n_alloc) {
        TGS_CUDA_OK(ctx->proj.ensure((size_t)n_alloc * 3 * sizeof(float4)));
        ctx->proj_cap = n_alloc;
    }
    for (int i = 0; i < 2; ++i) {
        TGS_CUDA_OK(ctx->pre_keys[i].ensure((size_t)n_alloc * 4));
        TGS_CUDA_OK(ctx->pre_vals[i].ensure((size_t)n_alloc * 4));
    }
    TGS_CUDA_OK(ctx->rect.ensure((size_t)n_alloc * sizeof(uint2)));
    TGS_CUDA_OK(ctx->rrect.ensure((size_t)n_alloc * sizeof(uint2)));
    const uint32_t cap = std::max<uint32_t>(ctx->capacity, 1u);
    TGS_CUDA_OK(ctx->list.ensure((size_t)cap * 4));
    // the previous frame's measured walks schedule this one when it had the same unit geometry
    // (same image, group size, band and backend): a camera path changes slowly
    const uint64_t ukey = ((uint64_t)(uint32_t)cam->width << 40) ^ ((uint64_t)(uint32_t)cam->height << 20) ^
                          ((uint64_t)band0 << 8) ^ ((uint64_t)band1 << 28) ^ ((uint64_t)gg.g << 4) ^
                          (uint64_t)opt->backend ^ (1ull << 63);
    ctx->row_chunks = bin_row_chunks(gg, ctx->rc_key == (ukey ^ (uint64_t)(uintptr_t)scene) ? ctx->rc_entries : 0u);
    ctx->rc_pending_key = ukey ^ (uint64_t)(uintptr_t)scene;
    const size_t h1 = bin_hist1_elems(gg, ctx->row_chunks), h2 = bin_hist2_elems(gg, cap), hm = bin_meta_elems(gg);
    TGS_CUDA_OK(ctx->hist.ensure((h1 + h2 + hm + bin_segmap_elems(gg, cap) + bin_slicecum_elems(gg, cap)) * 4));
    TGS_CUDA_OK(ctx->rowlist.ensure((size_t)cap * sizeof(uint2)));
    TGS_CUDA_OK(ctx->bsum.ensure(
        std::max({scan_tmp_elems(h1), scan_tmp_elems(h2), scan_tmp_elems(sort_scratch_elems((size_t)n_alloc))}) * 4));
    TGS_CUDA_OK(ctx->ghist.ensure(sort_scratch_elems((size_t)n_alloc) * 4));
    TGS_CUDA_OK(ctx->offsets.ensure((size_t)(n_groups + 1) * 4));
    // raster work units: the tensor path splits G=4 groups into 2x2-tile quarters
    const int units_per_group = opt->backend == TGS_BACKEND_TENSOR ? raster_units_per_group(gg.g) : 1;
    const size_t n_units = (size_t)std::max(1, n_groups * units_per_group);
    TGS_CUDA_OK(ctx->order.ensure(n_units * 4));
    TGS_CUDA_OK(ctx->ucost.ensure(n_units * 4));
    const int row0 = band0 * gg.g * kTile;
    const int row1 = std::min(cam->height, band1 * gg.g * kTile);
    TGS_CUDA_OK(ctx->image.ensure((size_t)(row1 - row0) * cam->width * 3 * sizeof(float)));

    const bool feedback = ctx->ucost_key == ukey;
    ctx->ucost_key = ukey;
    // everything the launch sequence depends on except the camera pose / intrinsics
    char kbuf[640];
    int kl = std::snprintf(kbuf, sizeof(kbuf), "%p %lld %d %d %d %d %d %d %d %a %a %a %d %d %u %lld %d", (const void*)scene,
                           (long long)scene->n, cam->width, cam->height, opt->backend, opt->mode, opt->group_size,
                           band0, band1,
                           opt->alpha_skip, opt->alpha_clamp, opt->t_terminate, ctx->tile_cull * 2 + ctx->exact,
                           feedback ? 1 : 0,
                           ctx->capacity, (long long)ctx->proj_cap, ctx->row_chunks);
    // ... and every buffer address the captured launches bake in (buffers only ever grow)
    // (the scene's device planes too: a scene freed and another uploaded at the same host address
    // must not replay launches that point at the old planes)
    kl += std::snprintf(kbuf + kl, sizeof(kbuf) - (size_t)kl, " %p %d", scene->planes.p, scene->sh_degree);
    const DBuf* fbufs[] = {&ctx->proj, &ctx->pre_keys[0], &ctx->pre_keys[1], &ctx->pre_vals[0], &ctx->pre_vals[1],
                           &ctx->rect, &ctx->rrect, &ctx->list, &ctx->rowlist, &ctx->hist, &ctx->bsum, &ctx->ghist,
                           &ctx->offsets, &ctx->order, &ctx->ucost, &ctx->image};
    for (const DBuf* b : fbufs) kl += std::snprintf(kbuf + kl, sizeof(kbuf) - (size_t)kl, " %p", b->p);
    const std::string key(kbuf);
    const bool same_as_prev = key == ctx->pkey;
    ctx->pkey = key;
    if (ctx->graphs && ctx->gexec && key == ctx->gkey) {
        // replay: only the camera changes
        PreprocessArgs pa = ctx->gpa;
        pa.cam = make_dev_camera(cam);
        cudaKernelNodeParams kp;
        TGS_CUDA_OK(cudaGraphKernelNodeGetParams(ctx->gpre, &kp));
        void* args[1] = {&pa};
        kp.kernelParams = args;
        kp.extra = nullptr;
        TGS_CUDA_OK(cudaGraphExecKernelNodeSetParams(ctx->gexec, ctx->gpre, &kp));
        TGS_CUDA_OK(cudaGraphLaunch(ctx->gexec, s));
    } else if (ctx->graphs && same_as_prev) {
        // the configuration repeated: capture the launch sequence once, then replay it
        cudaGraph_t graph = nullptr;
        TGS_CUDA_OK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        const tgs_status rs = record_frame(ctx, scene, cam, opt, gg, feedback, row0, h1, h2, n_alloc, units_per_group);
        const cudaError_t ce = cudaStreamEndCapture(s, &graph);
        if (rs != TGS_OK) {
            if (graph) cudaGraphDestroy(graph);
            return rs;
        }
        TGS_CUDA_OK(ce);
        if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
        ctx->gexec = nullptr;
        ctx->gpre = nullptr;
        cudaError_t e = cudaGraphInstantiate(&ctx->gexec, graph, 0);
        if (e == cudaSuccess) {
            size_t nn = 0;
            cudaGraphGetNodes(graph, nullptr, &nn);
            std::vector<cudaGraphNode_t> nodes(nn);
            cudaGraphGetNodes(graph, nodes.data(), &nn);
            for (cudaGraphNode_t nd : nodes) {
                cudaGraphNodeType ty;
                cudaKernelNodeParams kp;
                if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel &&
                    cudaGraphKernelNodeGetParams(nd, &kp) == cudaSuccess && kp.func == preprocess_kernel_fn()) {
                    ctx->gpre = nd;
                    ctx->gpa = *static_cast<const PreprocessArgs*>(kp.kernelParams[0]);
                }
            }
            if (!ctx->gpre) e = cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) {
            if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
            ctx->gexec = nullptr;
            cudaGraphDestroy(graph);
            return cuda_fail(e, "frame graph capture", __FILE__, __LINE__);
        }
        // the executable graph references kernel nodes by the (kept) graph's node handles
        ctx->gkey = key;
        if (ctx->ggraph) cudaGraphDestroy(ctx->ggraph);
        ctx->ggraph = graph;
        TGS_CUDA_OK(cudaGraphLaunch(ctx->gexec, s));
    } else {
        const tgs_status rs = record_frame(ctx, scene, cam, opt, gg, feedback, row0, h1, h2, n_alloc, units_per_group);
        if (rs != TGS_OK) return rs;
    }

    ctx->last_scene = scene;
    ctx->last_cam = *cam;
    ctx->last_opt = *opt;
    ctx->last_gg = gg;
    ctx->last_band0 = band0;
    ctx->last_band1 = band1;
    ctx->image_rows = row1 - row0;
    ctx->pending = true;
    return TGS_OK;
}

// The stream operations of one frame (eager, or recorded into the frame graph).
tgs_status record_frame(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam, const tgs_options* opt,
                        const GroupGeom& gg, bool feedback, int row0, size_t h1, size_t h2, int n_alloc,
                        int units_per_group) {
    cudaStream_t s = ctx->stream;
    const int n_groups = gg.n_groups_band;
    FrameCounters* fc = ctx->fc.as<FrameCounters>();
    const DevProjected proj = dev_proj(ctx);

    TGS_CUDA_OK(record_event(ctx->ev[0], s));
    // the sticky counters at the end of FrameCounters survive across frames (tgs_sync checks them)
    TGS_CUDA_OK(cudaMemsetAsync(fc, 0, offsetof(FrameCounters, sticky_overflow), s));

    // 1. preprocess + compaction
    PreprocessArgs pa;
    pa.scene = scene->dev();
    pa.cam = make_dev_camera(cam);
    pa.out = proj;
    pa.depth_keys = ctx->pre_keys[0].as<uint32_t>();
    pa.rect = ctx->rect.as<uint2>();
    pa.gg = gg;
    pa.fc = fc;
    pa.alpha_skip = opt->alpha_skip;
    launch_preprocess(pa, s);
    TGS_CUDA_OK(cudaGetLastError());
    TGS_CUDA_OK(record_event(ctx->ev[1], s));

    // 2. depth presort (keys: depth bits, values: project_scene index)
    SortBuffers pb;
    pb.keys[0] = ctx->pre_keys[0].as<uint32_t>();
    pb.keys[1] = ctx->pre_keys[1].as<uint32_t>();
    pb.vals[0] = ctx->pre_vals[0].as<uint32_t>();
    pb.vals[1] = ctx->pre_vals[1].as<uint32_t>();
    pb.ghist = ctx->ghist.as<uint32_t>();
    pb.scan_tmp = ctx->bsum.as<uint32_t>();
    pb.result_sel = ctx->ghist.as<uint32_t>() + sort_result_sel_offset();
    // pass 1 covers all n splats and drops the culled ones (key kCulledKey); later passes the kept
    radix_sort(pb, &fc->n_input, &fc->visible, 32, true, false, (size_t)n_alloc, s, &fc->key_min_inv, true);
    TGS_CUDA_OK(cudaGetLastError());

    TGS_CUDA_OK(record_event(ctx->ev[2], s));

    // 3. binning: stable counting sort of (group, rank) entries -> lists + per-group offsets
    BinArgs ba;
    ba.visible = &fc->visible;
    ba.sval[0] = pb.vals[0];
    ba.sval[1] = pb.vals[1];
    ba.sval_sel = pb.result_sel;
    ba.rect = ctx->rect.as<uint2>();
    ba.rrect = ctx->rrect.as<uint2>();
    ba.gg = gg;
    ba.row_chunks = ctx->row_chunks;
    ba.hist1 = ctx->hist.as<uint32_t>();
    ba.hist2 = ba.hist1 + h1;
    ba.meta = ba.hist2 + h2;
    ba.segmap = ba.meta + bin_meta_elems(gg);
    ba.slicecum = ba.segmap + bin_segmap_elems(gg, std::max<uint32_t>(ctx->capacity, 1u));
    ba.rowidx = ctx->rowlist.as<uint32_t>();
    ba.rowxp = ba.rowidx + std::max<uint32_t>(ctx->capacity, 1u);  // the buffer holds 2 x max(capacity, 1) words
    ba.bsum = ctx->bsum.as<uint32_t>();
    ba.offsets = ctx->offsets.as<uint32_t>();
    ba.list = ctx->list.as<uint32_t>();
    ba.fc = fc;
    ba.capacity = ctx->capacity;
    launch_binning(ba, n_alloc, s);
    {
        // tensor G=4 groups are rasterised as 2x2-tile quarters; the CUDA-core baseline walks whole
        // lists.  With feedback the previous frame's measured walks order the units.
        const int per = units_per_group;
        const uint32_t* fb = feedback ? ctx->ucost.as<uint32_t>() : nullptr;
        launch_unit_order(ctx->offsets.as<uint32_t>(), fb, n_groups * per, per, ctx->order.as<int>(), fc, s);
    }
    TGS_CUDA_OK(cudaGetLastError());
    TGS_CUDA_OK(record_event(ctx->ev[3], s));

    // 6. raster
    RasterArgs ra;
    ra.proj = proj;
    ra.list = ctx->list.as<uint32_t>();
    ra.offsets = ctx->offsets.as<uint32_t>();
    ra.order = ctx->order.as<int>();
    ra.gg = gg;
    ra.image = ctx->image.as<float>();
    ra.image_row0 = row0;
    ra.alpha_skip = opt->alpha_skip;
    ra.alpha_clamp = opt->alpha_clamp;
    ra.t_terminate = opt->t_terminate;
    ra.fc = fc;
    ra.tile_trip = nullptr;
    ra.unit_cost = ctx->ucost.as<uint32_t>();
    ra.tile_cull = ctx->tile_cull;
    if (opt->mode == TGS_MODE_FP16 || ctx->exact)
        launch_raster_exact(ra, opt->mode == TGS_MODE_FP16, s);
    else if (opt->backend == TGS_BACKEND_SCALAR)
        launch_raster_scalar(ra, s);
    else
        launch_raster_tensor(ra, ctx->num_sms, s);
    TGS_CUDA_OK(cudaGetLastError());
    TGS_CUDA_OK(record_event(ctx->ev[4], s));
    TGS_CUDA_OK(cudaMemcpyAsync(ctx->h_fc, fc, sizeof(FrameCounters), cudaMemcpyDeviceToHost, s));
    (void)scene;
    return TGS_OK;
}

tgs_status finish_frame(tgs_ctx* ctx, tgs_stats* stats) {
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    ctx->pending = false;
    const FrameCounters& f = *ctx->h_fc;
    {
        // frames enqueued since the last sync that overflowed their entry buffers or failed
        // validation: only the last one is recovered (re-rendered / reported) below, an earlier
        // one left an invalid image behind, so the whole sequence fails
        const uint32_t of = f.sticky_overflow - ctx->acked_overflow, bad = f.sticky_invalid - ctx->acked_invalid;
        ctx->acked_overflow = f.sticky_overflow;
        ctx->acked_invalid = f.sticky_invalid;
        if (of > (f.overflow ? 1u : 0u))
            return set_err(TGS_ERR_OOM, "render: a frame enqueued before the last tgs_sync exceeded the entry "
                                        "capacity (its lists were not built); size the context on every camera first");
        if (bad > (f.err_validation ? 1u : 0u))
            return set_err(TGS_ERR_VALIDATION, "render: a frame enqueued before the last tgs_sync failed validation "
                                               "(non-positive scale or bad depth)");
    }
    if (f.overflow) {
        // entry buffers too small: grow (25% headroom) and re-render this frame
        const uint64_t need = (uint64_t)f.n_entries + f.n_entries / 4 + 1024;
        if (need > 0xFFFFFFF0ull) return set_err(TGS_ERR_OOM, "render: more than 2^32 entries in one frame");
        ctx->capacity = (uint32_t)need;
        tgs_camera cam = ctx->last_cam;
        tgs_options opt = ctx->last_opt;
        tgs_status st = enqueue_frame(ctx, ctx->last_scene, &cam, &opt, ctx->last_band0, ctx->last_band1);
        if (st != TGS_OK) return st;
        TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
        ctx->pending = false;
        ctx->acked_overflow = ctx->h_fc->sticky_overflow;
        ctx->acked_invalid = ctx->h_fc->sticky_invalid;
        if (ctx->h_fc->overflow) return set_err(TGS_ERR_OOM, "render: entry capacity overflow after growth");
    }
    const FrameCounters& g = *ctx->h_fc;
    ctx->rc_key = ctx->rc_pending_key;  // the last enqueued frame's geometry and group-row entries
    ctx->rc_entries = g.row_entries;
    if (g.err_validation & 1u) return set_err(TGS_ERR_VALIDATION, "compute_cov3d: non-positive scale");
    if (g.err_validation & 2u)
        return set_err(TGS_ERR_VALIDATION, "sort_entries: an entry has non-finite or negative depth");
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->input = (uint64_t)ctx->last_scene->n;
        stats->culled = g.culled;
        stats->dropped_degenerate = g.dropped;
        stats->entries = g.n_entries;
        stats->tile_appearances = g.appearances;
        stats->visible = g.visible;
        float ms = 0;
        cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
        stats->ms_preprocess = ms;
        cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]);
        stats->ms_sort = ms;  // depth presort (radix)
        cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
        stats->ms_binning = ms;  // counting sort into group lists + ranges
        cudaEventElapsedTime(&ms, ctx->ev[3], ctx->ev[4]);
        stats->ms_raster = ms;
        cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[4]);
        stats->ms_total = ms;
        (void)cudaGetLastError();  // a timing query must never poison the next frame's error check
        stats->chunk_loads = g.op_chunks;
        stats->fragment_ops = 16ull * g.op_mmas;
        stats->skipped_pairs = g.op_skipped;
        stats->used_lanes = g.op_mma_rows * 128ull * 12ull;
        stats->total_lanes = stats->fragment_ops * 16ull * 16ull * 16ull;
    }
    return TGS_OK;
}

__global__ void records_to_planes(const float* __restrict__ rec, int64_t n, int rf, float4* pos_op,
                                  float4* quat, float4* scale_dcr, float2* dc_gb, float4* sh) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float* p = rec + i * rf;
        pos_op[i] = make_float4(p[0], p[1], p[2], p[10]);
        quat[i] = make_float4(p[6], p[7], p[8], p[9]);
        scale_dcr[i] = make_float4(p[3], p[4], p[5], p[11]);
        dc_gb[i] = make_float2(p[12], p[13]);
        if (sh) {
            for (int k = 0; k < 12; ++k) {
                float v[4];
                for (int c = 0; c < 4; ++c) v[c] = (4 * k + c < 45) ? p[14 + 4 * k + c] : 0.0f;
                sh[(size_t)k * n + i] = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
    }
}

tgs_status upload_into(tgs_ctx* ctx, tgs_scene* sc, const float* records, int64_t count, int deg) {
    if (count < 0 || count > (int64_t)0x7fffffff) return set_err(TGS_ERR_VALIDATION, "scene: bad count");
    if (deg != 0 && deg != 3) return set_err(TGS_ERR_FORMAT, "scene: unsupported sh_degree");
    const int rf = deg == 3 ? 59 : 14;
    const int64_t n = count;
    const size_t n_alloc = (size_t)std::max<int64_t>(n, 1);
    const size_t bytes = n_alloc * (3 * sizeof(float4) + sizeof(float2)) + (deg == 3 ? n_alloc * 12 * sizeof(float4) : 0);
    TGS_CUDA_OK(cudaSetDevice(ctx->device));
    TGS_CUDA_OK(sc->planes.ensure(bytes));
    sc->ctx = ctx;
    sc->device = ctx->device;
    sc->n = n;
    sc->sh_degree = deg;
    if (n == 0) return TGS_OK;
    TGS_CUDA_OK(ctx->scratch_records.ensure((size_t)n * rf * sizeof(float)));
    TGS_CUDA_OK(cudaMemcpyAsync(ctx->scratch_records.p, records, (size_t)n * rf * sizeof(float),
                                cudaMemcpyHostToDevice, ctx->stream));
    const DevScene d = sc->dev();
    records_to_planes<<<148 * 8, 256, 0, ctx->stream>>>(ctx->scratch_records.as<float>(), n, rf,
                                                         const_cast<float4*>(d.pos_op), const_cast<float4*>(d.quat),
                                                         const_cast<float4*>(d.scale_dcr), const_cast<float2*>(d.dc_gb),
                                                         const_cast<float4*>(d.sh_rest));
    TGS_CUDA_OK(cudaGetLastError());
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    return TGS_OK;
}

tgs_status copy_image_to_host(tgs_ctx* ctx, float* out) {
    const size_t bytes = (size_t)ctx->image_rows * ctx->last_cam.width * 3 * sizeof(float);
    TGS_CUDA_OK(cudaMemcpyAsync(out, ctx->image.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    return TGS_OK;
}

}  // namespace api
}  // namespace tgs

using namespace tgs::api;

extern "C" {

const char* tgs_last_error(void) { return g_err.c_str(); }
int tgs_abi_version(void) { return TGS_ABI_VERSION; }

tgs_status tgs_ctx_create(int device, tgs_ctx** out) {
    if (!out) return set_err(TGS_ERR_VALIDATION, "ctx_create: null out");
    *out = nullptr;
    int ndev = 0;
    TGS_CUDA_OK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return set_err(TGS_ERR_CUDA, "ctx_create: no such CUDA device");
    cudaDeviceProp prop;
    TGS_CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_err(TGS_ERR_CUDA, std::string("ctx_create: libtgs is built for sm_100a; device is ") + prop.name);
    TGS_CUDA_OK(cudaSetDevice(device));
    tgs_ctx* c = new tgs_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    for (int i = 0; e == cudaSuccess && i < 6; ++i) e = cudaEventCreate(&c->ev[i]);
    if (e == cudaSuccess) e = c->fc.ensure(sizeof(FrameCounters));
    // the sticky failure counters at the end of FrameCounters start at zero (never memset per frame)
    if (e == cudaSuccess) e = cudaMemset(c->fc.p, 0, sizeof(FrameCounters));
    if (e == cudaSuccess) e = cudaMallocHost(&c->h_fc, sizeof(FrameCounters));
    if (e != cudaSuccess) {
        tgs_ctx_destroy(c);
        return cuda_fail(e, "ctx_create", __FILE__, __LINE__);
    }
    *out = c;
    return TGS_OK;
}

void tgs_ctx_destroy(tgs_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->scratch_scene) tgs_scene_free(c->scratch_scene);
    for (tgs_ctx*& l : c->lanes)
        if (l) {
            tgs_ctx_destroy(l);
            l = nullptr;
        }
    DBuf* bufs[] = {&c->fc, &c->proj, &c->pre_keys[0], &c->pre_keys[1], &c->pre_vals[0],
                    &c->pre_vals[1], &c->rect, &c->rrect, &c->list, &c->rowlist, &c->hist, &c->bsum, &c->ghist,
                    &c->offsets, &c->order, &c->ucost, &c->image, &c->scratch_records};
    for (DBuf* b : bufs) b->release();
    for (DBuf& b : c->stg) b.release();
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->ggraph) cudaGraphDestroy(c->ggraph);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->h_fc) cudaFreeHost(c->h_fc);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

void* tgs_ctx_stream(tgs_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

tgs_status tgs_set_tile_cull(tgs_ctx* ctx, int on) {
    if (!ctx) return set_err(TGS_ERR_VALIDATION, "set_tile_cull: null context");
    ctx->tile_cull = on ? 1 : 0;
    for (tgs_ctx* l : ctx->lanes)
        if (l) l->tile_cull = ctx->tile_cull;
    return TGS_OK;
}

tgs_status tgs_set_exact_emulation(tgs_ctx* ctx, int on) {
    if (!ctx) return set_err(TGS_ERR_VALIDATION, "set_exact_emulation: null context");
    ctx->exact = on ? 1 : 0;
    for (tgs_ctx* l : ctx->lanes)
        if (l) l->exact = ctx->exact;
    return TGS_OK;
}

tgs_status tgs_set_graphs(tgs_ctx* ctx, int on) {
    if (!ctx) return set_err(TGS_ERR_VALIDATION, "set_graphs: null context");
    ctx->graphs = on ? 1 : 0;
    for (tgs_ctx* l : ctx->lanes)
        if (l) l->graphs = ctx->graphs;
    return TGS_OK;
}

tgs_status tgs_scene_upload(tgs_ctx* ctx, const float* records, int64_t count, int sh_degree, tgs_scene** out) {
    if (!ctx || !out || (count > 0 && !records)) return set_err(TGS_ERR_VALIDATION, "scene_upload: null argument");
    tgs_scene* sc = new tgs_scene();
    tgs_status st = upload_into(ctx, sc, records, count, sh_degree);
    if (st != TGS_OK) {
        sc->planes.release();
        delete sc;
        *out = nullptr;
        return st;
    }
    *out = sc;
    return TGS_OK;
}

void tgs_scene_free(tgs_scene* sc) {
    if (!sc) return;
    cudaSetDevice(sc->device);
    sc->planes.release();
    delete sc;
}

tgs_status tgs_render_enqueue(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam, const tgs_options* opt) {
    if (!ctx) return set_err(TGS_ERR_VALIDATION, "render: null context");
    cudaSetDevice(ctx->device);
    return enqueue_frame(ctx, scene, cam, opt, 0, 0);
}

tgs_status tgs_sync(tgs_ctx* ctx, tgs_stats* stats) {
    if (!ctx) return set_err(TGS_ERR_VALIDATION, "sync: null context");
    if (!ctx->pending) {
        TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
        return TGS_OK;
    }
    return finish_frame(ctx, stats);
}

const float* tgs_image_device(tgs_ctx* ctx) { return ctx ? ctx->image.as<float>() : nullptr; }

tgs_status tgs_render(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam, const tgs_options* opt,
                      float* out_rgb, tgs_stats* stats) {
    tgs_status st = tgs_render_enqueue(ctx, scene, cam, opt);
    if (st != TGS_OK) return st;
    st = finish_frame(ctx, stats);
    if (st != TGS_OK) return st;
    return out_rgb ? copy_image_to_host(ctx, out_rgb) : TGS_OK;
}

tgs_status tgs_render_records(tgs_ctx* ctx, const float* records, int64_t count, int sh_degree,
                              const tgs_camera* cam, const tgs_options* opt, float* out_rgb, tgs_stats* stats) {
    if (!ctx) return set_err(TGS_ERR_VALIDATION, "render: null context");
    tgs_status st = validate_options(cam, opt);
    if (st != TGS_OK) return st;
    if (!ctx->scratch_scene) ctx->scratch_scene = new tgs_scene();
    st = upload_into(ctx, ctx->scratch_scene, records, count, sh_degree);
    if (st != TGS_OK) return st;
    return tgs_render(ctx, ctx->scratch_scene, cam, opt, out_rgb, stats);
}

tgs_status tgs_render_band(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam, const tgs_options* opt,
                           int group_row0, int group_row1, float* out_rgb, tgs_stats* stats) {
    if (!ctx) return set_err(TGS_ERR_VALIDATION, "render_band: null context");
    if (group_row1 <= group_row0) return set_err(TGS_ERR_VALIDATION, "render_band: empty band");
    cudaSetDevice(ctx->device);
    tgs_status st = enqueue_frame(ctx, scene, cam, opt, group_row0, group_row1);
    if (st != TGS_OK) return st;
    st = finish_frame(ctx, stats);
    if (st != TGS_OK) return st;
    return out_rgb ? copy_image_to_host(ctx, out_rgb) : TGS_OK;
}

tgs_status tgs_group_row_entries(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam, const tgs_options* opt,
                                 uint64_t* counts, int64_t cap, int64_t* n_rows) {
    if (!ctx || !n_rows) return set_err(TGS_ERR_VALIDATION, "group_row_entries: null argument");
    tgs_status st = validate_options(cam, opt);
    if (st != TGS_OK) return st;
    if (!scene || (scene->ctx != ctx && scene->ctx != ctx->parent))
        return set_err(TGS_ERR_VALIDATION, "group_row_entries: scene belongs to another context");
    cudaSetDevice(ctx->device);
    const GroupGeom full = make_geom(opt->group_size, cam->width, cam->height, 0, 0);
    const GroupGeom gg = make_geom(opt->group_size, cam->width, cam->height, 0, full.groups_y);
    *n_rows = gg.groups_y;
    if (!counts || cap < gg.groups_y) return TGS_OK;
    const int64_t na = std::max<int64_t>(scene->n, 1);
    if (ctx->proj_cap < na) {
        TGS_CUDA_OK(ctx->proj.ensure((size_t)na * 3 * sizeof(float4)));
        ctx->proj_cap = na;
    }
    TGS_CUDA_OK(ctx->pre_keys[0].ensure((size_t)na * 4));
    TGS_CUDA_OK(ctx->rect.ensure((size_t)na * sizeof(uint2)));
    TGS_CUDA_OK(ctx->stg[6].ensure((size_t)gg.groups_y * sizeof(unsigned long long)));
    FrameCounters* fc = ctx->fc.as<FrameCounters>();
    TGS_CUDA_OK(cudaMemsetAsync(fc, 0, offsetof(FrameCounters, sticky_overflow), ctx->stream));
    PreprocessArgs pa;
    pa.scene = scene->dev();
    pa.cam = make_dev_camera(cam);
    pa.out = dev_proj(ctx);
    pa.depth_keys = ctx->pre_keys[0].as<uint32_t>();
    pa.rect = ctx->rect.as<uint2>();
    pa.gg = gg;
    pa.fc = fc;
    pa.alpha_skip = opt->alpha_skip;
    launch_preprocess(pa, ctx->stream);
    launch_row_entries(ctx->rect.as<uint2>(), &fc->n_input, gg, ctx->stg[6].as<unsigned long long>(), ctx->stream);
    TGS_CUDA_OK(cudaGetLastError());
    TGS_CUDA_OK(cudaMemcpyAsync(counts, ctx->stg[6].p, (size_t)gg.groups_y * 8, cudaMemcpyDeviceToHost, ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    return TGS_OK;
}

tgs_status tgs_render_batch(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cams, int n,
                            const tgs_options* opt, float* out_rgb, tgs_stats* stats) {
    if (!ctx || !cams || n < 0) return set_err(TGS_ERR_VALIDATION, "render_batch: bad arguments");
    for (int i = 0; i < n; ++i)
        if (cams[i].width != cams[0].width || cams[i].height != cams[0].height)
            return set_err(TGS_ERR_VALIDATION, "render_batch: all cameras must share width/height");
    cudaSetDevice(ctx->device);
    // round-robin over up to kBatchLanes contexts: frame i is enqueued on lane i % L once the lane's
    // previous frame (i - L) is retired and its image copied out, so the copies and one frame's
    // latency-bound raster overlap other frames' preprocess/sort/binning
    const int L = std::max(1, std::min(n, kBatchLanes));
    tgs_ctx* lane[kBatchLanes] = {ctx};
    for (int k = 1; k < L; ++k) {
        if (!ctx->lanes[k - 1]) {
            tgs_status st = tgs_ctx_create(ctx->device, &ctx->lanes[k - 1]);
            if (st != TGS_OK) return st;
            ctx->lanes[k - 1]->parent = ctx;
            ctx->lanes[k - 1]->tile_cull = ctx->tile_cull;
            ctx->lanes[k - 1]->graphs = ctx->graphs;
        }
        lane[k] = ctx->lanes[k - 1];
    }
    tgs_stats acc{};
    const size_t px = n ? (size_t)cams[0].width * cams[0].height * 3 : 0;
    for (int i = 0; i < n + L; ++i) {
        if (i >= L) {
            const int j = i - L;
            tgs_ctx* c = lane[j % L];
            tgs_stats one{};
            tgs_status st = finish_frame(c, &one);
            if (st == TGS_OK && out_rgb) st = copy_image_to_host(c, out_rgb + px * j);
            if (st != TGS_OK) {
                for (int k = 0; k < L; ++k) cudaStreamSynchronize(lane[k]->stream), lane[k]->pending = false;
                return st;
            }
            acc.input += one.input;
            acc.culled += one.culled;
            acc.dropped_degenerate += one.dropped_degenerate;
            acc.entries += one.entries;
            acc.tile_appearances += one.tile_appearances;
            acc.visible += one.visible;
            acc.ms_preprocess += one.ms_preprocess;
            acc.ms_binning += one.ms_binning;
            acc.ms_sort += one.ms_sort;
            acc.ms_raster += one.ms_raster;
            acc.ms_total += one.ms_total;
            acc.fragment_ops += one.fragment_ops;
            acc.chunk_loads += one.chunk_loads;
            acc.skipped_pairs += one.skipped_pairs;
            acc.used_lanes += one.used_lanes;
            acc.total_lanes += one.total_lanes;
        }
        if (i < n) {
            tgs_status st = validate_options(&cams[i], opt);
            if (st == TGS_OK) st = enqueue_frame(lane[i % L], scene, &cams[i], opt, 0, 0);
            if (st != TGS_OK) {
                for (int k = 0; k < L; ++k) cudaStreamSynchronize(lane[k]->stream), lane[k]->pending = false;
                return st;
            }
        }
    }
    if (stats) *stats = acc;
    return TGS_OK;
}

namespace tgs {
namespace api {
// project_scene's compacted order (projection.cpp:131-139): kept[i] and the compacted index of
// every input splat, from the per-splat rect words (kCulledRect = not projected).
tgs_status compaction_map(tgs_ctx* ctx, std::vector<int64_t>& cidx, int64_t& visible) {
    const int64_t n = ctx->last_scene->n;
    std::vector<uint2> rect((size_t)n);
    if (n) TGS_CUDA_OK(cudaMemcpy(rect.data(), ctx->rect.p, (size_t)n * sizeof(uint2), cudaMemcpyDeviceToHost));
    cidx.assign((size_t)n, -1);
    visible = 0;
    for (int64_t i = 0; i < n; ++i)
        if (!(rect[i].x == kCulledRect && rect[i].y == kCulledRect)) cidx[i] = visible++;
    return TGS_OK;
}
}  // namespace api
}  // namespace tgs

tgs_status tgs_read_projected(tgs_ctx* ctx, tgs_projected* out, int64_t cap, int64_t* n) {
    if (!ctx || !n) return set_err(TGS_ERR_VALIDATION, "read_projected: null argument");
    if (!ctx->last_scene) return set_err(TGS_ERR_VALIDATION, "read_projected: no frame rendered yet");
    const int64_t v = ctx->h_fc->visible;
    *n = v;
    if (!out || cap < v || v == 0) return TGS_OK;
    std::vector<int64_t> cidx;
    int64_t vis = 0;
    tgs_status st = compaction_map(ctx, cidx, vis);
    if (st != TGS_OK) return st;
    const int64_t N = ctx->last_scene->n;
    std::vector<float4> h((size_t)N * 3);
    const DevProjected p = dev_proj(ctx);
    TGS_CUDA_OK(cudaMemcpy(h.data(), p.mc, (size_t)N * sizeof(float4), cudaMemcpyDeviceToHost));
    TGS_CUDA_OK(cudaMemcpy(h.data() + N, p.co, (size_t)N * sizeof(float4), cudaMemcpyDeviceToHost));
    TGS_CUDA_OK(cudaMemcpy(h.data() + 2 * N, p.col, (size_t)N * sizeof(float4), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < N; ++i) {
        if (cidx[i] < 0) continue;
        const float4 mc = h[i], co = h[N + i], col = h[2 * N + i];
        tgs_projected& o = out[cidx[i]];
        o.mean2d[0] = mc.x;
        o.mean2d[1] = mc.y;
        o.conic[0] = mc.z;
        o.conic[1] = mc.w;
        o.conic[2] = co.x;
        o.opacity = co.y;
        o.depth = co.z;
        std::memcpy(&o.radius, &co.w, 4);
        o.color[0] = col.x;
        o.color[1] = col.y;
        o.color[2] = col.z;
    }
    return TGS_OK;
}

tgs_status tgs_read_lists(tgs_ctx* ctx, tgs_group_entry* out, int64_t cap, uint32_t* offsets,
                          int64_t offsets_cap, int64_t* n) {
    if (!ctx || !n) return set_err(TGS_ERR_VALIDATION, "read_lists: null argument");
    if (!ctx->last_scene) return set_err(TGS_ERR_VALIDATION, "read_lists: no frame rendered yet");
    const int64_t m = ctx->h_fc->n_entries;
    const int ng = ctx->last_gg.n_groups_band;
    *n = m;
    if (!out || cap < m || !offsets || offsets_cap < ng + 1) return TGS_OK;
    TGS_CUDA_OK(cudaMemcpy(offsets, ctx->offsets.p, (size_t)(ng + 1) * 4, cudaMemcpyDeviceToHost));
    if (m == 0) return TGS_OK;
    DBuf tmp;
    TGS_CUDA_OK(tmp.ensure((size_t)m * sizeof(tgs_group_entry)));
    launch_lists_readback(ctx->list.as<uint32_t>(), ctx->offsets.as<uint32_t>(), ng,
                          dev_proj(ctx), ctx->last_gg, tmp.as<tgs_group_entry>(), ctx->stream);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, tmp.p, (size_t)m * sizeof(tgs_group_entry), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    tmp.release();
    if (e != cudaSuccess) return cuda_fail(e, "read_lists", __FILE__, __LINE__);
    // entries reference input indices on the device; the reference's GroupEntry holds the
    // project_scene (compacted) index
    std::vector<int64_t> cidx;
    int64_t vis = 0;
    tgs_status st = compaction_map(ctx, cidx, vis);
    if (st != TGS_OK) return st;
    for (int64_t k = 0; k < m; ++k) out[k].gaussian_index = (uint32_t)cidx[out[k].gaussian_index];
    return TGS_OK;
}

tgs_status tgs_tile_trips(tgs_ctx* ctx, uint32_t* trips, int64_t cap, int64_t* n) {
    if (!ctx || !n) return set_err(TGS_ERR_VALIDATION, "tile_trips: null argument");
    if (!ctx->last_scene) return set_err(TGS_ERR_VALIDATION, "tile_trips: no frame rendered yet");
    const GroupGeom& gg = ctx->last_gg;
    const int tiles = gg.tiles_x * (gg.band_gy1 - gg.band_gy0) * gg.g;
    *n = tiles;
    if (!trips || cap < tiles) return TGS_OK;
    DBuf tmp;
    TGS_CUDA_OK(tmp.ensure((size_t)tiles * 4));
    FrameCounters* fc = ctx->fc.as<FrameCounters>();
    RasterArgs ra;
    ra.proj = dev_proj(ctx);
    ra.list = ctx->list.as<uint32_t>();
    ra.offsets = ctx->offsets.as<uint32_t>();
    ra.order = nullptr;
    ra.gg = gg;
    ra.image = nullptr;
    ra.image_row0 = 0;
    ra.alpha_skip = ctx->last_opt.alpha_skip;
    ra.alpha_clamp = ctx->last_opt.alpha_clamp;
    ra.t_terminate = ctx->last_opt.t_terminate;
    ra.fc = fc;
    ra.tile_trip = tmp.as<uint32_t>();
    ra.unit_cost = nullptr;
    ra.tile_cull = 0;
    launch_count_pairs(ra, ctx->stream);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(trips, tmp.p, (size_t)tiles * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    tmp.release();
    if (e != cudaSuccess) return cuda_fail(e, "tile_trips", __FILE__, __LINE__);
    return TGS_OK;
}

tgs_status tgs_reuse_report(tgs_ctx* ctx, uint64_t* n_group, uint64_t* n_total, double* load_reduction,
                            uint64_t hist[17]) {
    if (!ctx || !n_group || !n_total || !load_reduction || !hist)
        return set_err(TGS_ERR_VALIDATION, "reuse_report: null argument");
    if (!ctx->last_scene) return set_err(TGS_ERR_VALIDATION, "reuse_report: no frame rendered yet");
    cudaSetDevice(ctx->device);
    DBuf tmp;
    TGS_CUDA_OK(tmp.ensure(17 * sizeof(unsigned long long)));
    launch_reuse_hist(ctx->fc.as<FrameCounters>(), ctx->rect.as<uint2>(), ctx->last_gg,
                      (int)std::max<int64_t>(1, ctx->last_scene->n), tmp.as<unsigned long long>(), ctx->stream);
    cudaError_t e = cudaGetLastError();
    unsigned long long h[17];
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, tmp.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    tmp.release();
    if (e != cudaSuccess) return cuda_fail(e, "reuse_report", __FILE__, __LINE__);
    uint64_t ng = 0, nt = 0;
    for (int p = 0; p < 17; ++p) {
        hist[p] = h[p];
        ng += h[p];
        nt += (uint64_t)p * h[p];
    }
    if (ng == 0) return set_err(TGS_ERR_VALIDATION, "load_reduction: empty entry list has an undefined ratio");
    *n_group = ng;
    *n_total = nt;
    *load_reduction = 1.0 - (double)ng / (double)nt;
    return TGS_OK;
}

tgs_status tgs_count_pairs(tgs_ctx* ctx, uint64_t* walked, uint64_t* blended) {
    if (!ctx || !walked || !blended) return set_err(TGS_ERR_VALIDATION, "count_pairs: null argument");
    if (!ctx->last_scene) return set_err(TGS_ERR_VALIDATION, "count_pairs: no frame rendered yet");
    FrameCounters* fc = ctx->fc.as<FrameCounters>();
    TGS_CUDA_OK(cudaMemsetAsync(&fc->walked, 0, 2 * sizeof(unsigned long long), ctx->stream));
    RasterArgs ra;
    ra.proj = dev_proj(ctx);
    ra.list = ctx->list.as<uint32_t>();
    ra.offsets = ctx->offsets.as<uint32_t>();
    ra.order = nullptr;
    ra.gg = ctx->last_gg;
    ra.image = nullptr;
    ra.image_row0 = 0;
    ra.alpha_skip = ctx->last_opt.alpha_skip;
    ra.alpha_clamp = ctx->last_opt.alpha_clamp;
    ra.t_terminate = ctx->last_opt.t_terminate;
    ra.fc = fc;
    ra.tile_trip = nullptr;
    ra.unit_cost = nullptr;
    ra.tile_cull = 0;
    launch_count_pairs(ra, ctx->stream);
    TGS_CUDA_OK(cudaGetLastError());
    unsigned long long h[2];
    TGS_CUDA_OK(cudaMemcpyAsync(h, &fc->walked, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    *walked = h[0];
    *blended = h[1];
    return TGS_OK;
}

tgs_status tgs_encode_u8(tgs_ctx* ctx, const float* rgb_device, int64_t n, uint8_t* out_host) {
    if (!ctx || !rgb_device || !out_host || n < 0) return set_err(TGS_ERR_VALIDATION, "encode_u8: bad arguments");
    DBuf tmp;
    TGS_CUDA_OK(tmp.ensure((size_t)std::max<int64_t>(n, 1)));
    launch_encode_u8(rgb_device, n, tmp.as<uint8_t>(), ctx->stream);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_host, tmp.p, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    tmp.release();
    if (e != cudaSuccess) return cuda_fail(e, "encode_u8", __FILE__, __LINE__);
    return TGS_OK;
}

}  // extern "C"

// ---- stage API on caller-provided data ------------------------------------------------------
namespace tgs {
namespace api {

tgs_status validate_group_config(int g, int width, int height) {  // GroupConfig::validate (binning.cpp:22-30)
    if (width <= 0 || height <= 0) return set_err(TGS_ERR_VALIDATION, "GroupConfig: image dimensions must be positive");
    if (!(g == 1 || g == 2 || g == 4))
        return set_err(TGS_ERR_VALIDATION, "GroupConfig: supported group sizes are 1x1, 2x2, 4x4");
    return TGS_OK;
}

// Host -> device copy of n items into scratch buffer k (grown as needed).
template <class T>
tgs_status upload(tgs_ctx* ctx, int k, const T* host, size_t n, T** dev) {
    TGS_CUDA_OK(ctx->stg[k].ensure(std::max<size_t>(n, 1) * sizeof(T)));
    if (n) TGS_CUDA_OK(cudaMemcpyAsync(ctx->stg[k].p, host, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    *dev = ctx->stg[k].as<T>();
    return TGS_OK;
}

}  // namespace api
}  // namespace tgs

extern "C" {

tgs_status tgs_project_scene(tgs_ctx* ctx, const float* records, int64_t count, int sh_degree, const tgs_camera* cam,
                             tgs_projected* out, int64_t cap, int64_t* n, tgs_stats* stats) {
    if (!ctx || !cam || !n || (count > 0 && !records)) return set_err(TGS_ERR_VALIDATION, "project_scene: null argument");
    cudaSetDevice(ctx->device);
    if (!ctx->scratch_scene) ctx->scratch_scene = new tgs_scene();
    tgs_status st = upload_into(ctx, ctx->scratch_scene, records, count, sh_degree);
    if (st != TGS_OK) return st;
    const int64_t na = std::max<int64_t>(count, 1);
    if (ctx->proj_cap < na) {
        TGS_CUDA_OK(ctx->proj.ensure((size_t)na * 3 * sizeof(float4)));
        ctx->proj_cap = na;
    }
    TGS_CUDA_OK(ctx->pre_keys[0].ensure((size_t)na * 4));
    TGS_CUDA_OK(ctx->rect.ensure((size_t)na * sizeof(uint2)));
    const int w = std::max(cam->width, 1), h = std::max(cam->height, 1);
    const GroupGeom gg = make_geom(1, w, h, 0, (h + kTile - 1) / kTile);
    FrameCounters* fc = ctx->fc.as<FrameCounters>();
    TGS_CUDA_OK(cudaMemsetAsync(fc, 0, offsetof(FrameCounters, sticky_overflow), ctx->stream));
    PreprocessArgs pa;
    pa.scene = ctx->scratch_scene->dev();
    pa.cam = make_dev_camera(cam);
    pa.out = dev_proj(ctx);
    pa.depth_keys = ctx->pre_keys[0].as<uint32_t>();
    pa.rect = ctx->rect.as<uint2>();
    pa.gg = gg;
    pa.fc = fc;
    pa.alpha_skip = 1.0f / 255.0f;
    launch_preprocess(pa, ctx->stream);
    TGS_CUDA_OK(cudaGetLastError());
    TGS_CUDA_OK(cudaMemcpyAsync(ctx->h_fc, fc, sizeof(FrameCounters), cudaMemcpyDeviceToHost, ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    ctx->acked_overflow = ctx->h_fc->sticky_overflow;
    ctx->acked_invalid = ctx->h_fc->sticky_invalid;
    if (ctx->h_fc->err_validation & 1u) return set_err(TGS_ERR_VALIDATION, "compute_cov3d: non-positive scale");
    // the readback below reads the frame state of this call
    ctx->last_scene = ctx->scratch_scene;
    ctx->last_cam = *cam;
    ctx->last_gg = gg;
    if (stats) {
        std::memset(stats, 0, sizeof(*stats));
        stats->input = (uint64_t)count;
        stats->culled = ctx->h_fc->culled;
        stats->dropped_degenerate = ctx->h_fc->dropped;
        stats->visible = ctx->h_fc->visible;
    }
    return tgs_read_projected(ctx, out, cap, n);
}

tgs_status tgs_build_group_entries(tgs_ctx* ctx, const tgs_projected* proj, int64_t n, int width, int height,
                                   int group_size, tgs_keyed_entry* out, int64_t cap, int64_t* n_out) {
    if (!ctx || !n_out || n < 0 || (n > 0 && !proj)) return set_err(TGS_ERR_VALIDATION, "build_group_entries: bad arguments");
    tgs_status st = validate_group_config(group_size, width, height);
    if (st != TGS_OK) return st;
    cudaSetDevice(ctx->device);
    const GroupGeom gg = make_geom(group_size, width, height, 0, 0);
    tgs_projected* dp = nullptr;
    st = upload(ctx, 0, proj, (size_t)n, &dp);
    if (st != TGS_OK) return st;
    TGS_CUDA_OK(ctx->stg[1].ensure((size_t)(n + 1) * 4));
    uint32_t* counts = ctx->stg[1].as<uint32_t>();
    TGS_CUDA_OK(ctx->stg[2].ensure(scan_tmp_elems((size_t)n + 1) * 4));
    TGS_CUDA_OK(cudaMemsetAsync(counts, 0, (size_t)(n + 1) * 4, ctx->stream));
    launch_entries_count(dp, n, gg, counts, ctx->stream);
    launch_exclusive_scan(counts, (size_t)n + 1, ctx->stg[2].as<uint32_t>(), ctx->stream);
    TGS_CUDA_OK(cudaGetLastError());
    uint32_t total = 0;
    TGS_CUDA_OK(cudaMemcpyAsync(&total, counts + n, 4, cudaMemcpyDeviceToHost, ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    *n_out = total;
    if (!out || cap < (int64_t)total || total == 0) return TGS_OK;
    TGS_CUDA_OK(ctx->stg[3].ensure((size_t)total * sizeof(tgs_keyed_entry)));
    launch_entries_emit(dp, n, gg, counts, ctx->stg[3].as<tgs_keyed_entry>(), ctx->stream);
    TGS_CUDA_OK(cudaGetLastError());
    TGS_CUDA_OK(cudaMemcpyAsync(out, ctx->stg[3].p, (size_t)total * sizeof(tgs_keyed_entry), cudaMemcpyDeviceToHost,
                                ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    return TGS_OK;
}

tgs_status tgs_sort_entries(tgs_ctx* ctx, const tgs_keyed_entry* entries, int64_t n, int width, int height,
                            int group_size, tgs_group_entry* out, uint32_t* offsets, int64_t offsets_cap) {
    if (!ctx || n < 0 || (n > 0 && (!entries || !out)) || !offsets)
        return set_err(TGS_ERR_VALIDATION, "sort_entries: bad arguments");
    if (n > 0x7fffffffll) return set_err(TGS_ERR_VALIDATION, "sort_entries: more than 2^31 entries");
    tgs_status st = validate_group_config(group_size, width, height);
    if (st != TGS_OK) return st;
    const GroupGeom gg = make_geom(group_size, width, height, 0, 0);
    const uint32_t n_groups = (uint32_t)(gg.groups_x * gg.groups_y);
    if (offsets_cap < (int64_t)n_groups + 1) return set_err(TGS_ERR_VALIDATION, "sort_entries: offsets too small");
    cudaSetDevice(ctx->device);
    const uint32_t m = (uint32_t)n;
    tgs_keyed_entry* de = nullptr;
    st = upload(ctx, 0, entries, (size_t)m, &de);
    if (st != TGS_OK) return st;
    const size_t cap = ((size_t)std::max<uint32_t>(m, 1) + 31) & ~(size_t)31;  // 16-byte aligned sub-arrays (vector loads)
    // stg[1]: keys a | keys b | vals a | vals b | gids | flags+count ; stg[2]: sort scratch ; stg[3]: scan tmp
    TGS_CUDA_OK(ctx->stg[1].ensure((5 * cap + 4) * 4));
    uint32_t* u = ctx->stg[1].as<uint32_t>();
    uint32_t *ka = u, *kb = u + cap, *va = u + 2 * cap, *vb = u + 3 * cap, *gid = u + 4 * cap, *flags = u + 5 * cap,
             *count = flags + 1;
    TGS_CUDA_OK(ctx->stg[2].ensure(sort_scratch_elems(cap) * 4));
    TGS_CUDA_OK(ctx->stg[3].ensure(scan_tmp_elems(sort_scratch_elems(cap)) * 4));
    TGS_CUDA_OK(cudaMemsetAsync(flags, 0, 8, ctx->stream));
    launch_keyed_split(de, m, n_groups, ka, gid, flags, count, ctx->stream);
    // pass A: stable by depth bits (values = entry positions); pass B: stable by group id
    SortBuffers sb;
    sb.keys[0] = ka;
    sb.keys[1] = kb;
    sb.vals[0] = va;
    sb.vals[1] = vb;
    sb.ghist = ctx->stg[2].as<uint32_t>();
    sb.scan_tmp = ctx->stg[3].as<uint32_t>();
    int r = radix_sort(sb, count, count, 32, false, false, cap, ctx->stream, nullptr, true);
    uint32_t* perm = sb.vals[r];
    uint32_t* k2 = sb.keys[r];  // free after pass A (keys not written in its last pass)
    launch_gather_u32(gid, perm, m, k2, ctx->stream);
    SortBuffers sb2 = sb;
    sb2.keys[0] = k2;
    sb2.keys[1] = sb.keys[r ^ 1];
    sb2.vals[0] = perm;
    sb2.vals[1] = sb.vals[r ^ 1];
    const int gbits = std::max(1, ceil_log2((int)n_groups));
    r = radix_sort(sb2, count, count, gbits, false, true, cap, ctx->stream, nullptr, false);
    TGS_CUDA_OK(ctx->stg[4].ensure(cap * sizeof(tgs_group_entry)));
    TGS_CUDA_OK(ctx->stg[5].ensure(cap * 4 + (size_t)(n_groups + 1) * 4));
    uint32_t* gsorted = ctx->stg[5].as<uint32_t>();
    uint32_t* doff = gsorted + cap;
    launch_gather_entries(de, sb2.vals[r], m, ctx->stg[4].as<tgs_group_entry>(), gsorted, ctx->stream);
    launch_offsets_from_sorted(gsorted, m, n_groups, doff, ctx->stream);
    TGS_CUDA_OK(cudaGetLastError());
    uint32_t hflags = 0;
    TGS_CUDA_OK(cudaMemcpyAsync(&hflags, flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    if (hflags & 1u) return set_err(TGS_ERR_VALIDATION, "sort_entries: an entry has non-finite or negative depth");
    if (hflags & 2u) return set_err(TGS_ERR_VALIDATION, "sort_entries: group id outside the GroupConfig");
    if (m) TGS_CUDA_OK(cudaMemcpy(out, ctx->stg[4].p, (size_t)m * sizeof(tgs_group_entry), cudaMemcpyDeviceToHost));
    TGS_CUDA_OK(cudaMemcpy(offsets, doff, (size_t)(n_groups + 1) * 4, cudaMemcpyDeviceToHost));
    return TGS_OK;
}

tgs_status tgs_rasterize_lists(tgs_ctx* ctx, const tgs_group_entry* entries, int64_t n_entries, const uint32_t* offsets,
                               int64_t offsets_count, const tgs_projected* proj, int64_t n, int width, int height,
                               const tgs_options* opt, float* out_rgb) {
    if (!ctx || !opt || !offsets || !out_rgb || n < 0 || n_entries < 0 || (n_entries > 0 && !entries) ||
        (n > 0 && !proj))
        return set_err(TGS_ERR_VALIDATION, "rasterize: bad arguments");
    tgs_camera cam{};
    cam.width = width;
    cam.height = height;
    tgs_status st = validate_options(&cam, opt);
    if (st != TGS_OK) return st;
    const GroupGeom gg = make_geom(opt->group_size, width, height, 0, (height + opt->group_size * kTile - 1) /
                                                                           (opt->group_size * kTile));
    if (gg.groups_x > 512 || gg.band_gy1 > 512 || gg.n_groups_band > 49152)
        return set_err(TGS_ERR_VALIDATION, "rasterize: more than 512 group rows/columns; use a larger group size");
    const int ng = gg.n_groups_band;
    if (offsets_count != (int64_t)ng + 1 || offsets[0] != 0 || (int64_t)offsets[ng] != n_entries)
        return set_err(TGS_ERR_VALIDATION, "rasterize: offsets must hold group_count + 1 prefix offsets of the entries");
    cudaSetDevice(ctx->device);
    const int64_t na = std::max<int64_t>(n, 1);
    if (ctx->proj_cap < na) {
        TGS_CUDA_OK(ctx->proj.ensure((size_t)na * 3 * sizeof(float4)));
        ctx->proj_cap = na;
    }
    tgs_projected* dp = nullptr;
    tgs_group_entry* de = nullptr;
    uint32_t* doff = nullptr;
    if ((st = upload(ctx, 0, proj, (size_t)n, &dp)) != TGS_OK) return st;
    if ((st = upload(ctx, 1, entries, (size_t)n_entries, &de)) != TGS_OK) return st;
    if ((st = upload(ctx, 2, offsets, (size_t)ng + 1, &doff)) != TGS_OK) return st;
    TGS_CUDA_OK(ctx->list.ensure((size_t)std::max<int64_t>(n_entries, 1) * 4));
    const int per = opt->backend == TGS_BACKEND_TENSOR ? raster_units_per_group(gg.g) : 1;
    TGS_CUDA_OK(ctx->order.ensure((size_t)std::max(1, ng * per) * 4));
    TGS_CUDA_OK(ctx->image.ensure((size_t)width * height * 3 * sizeof(float)));
    TGS_CUDA_OK(ctx->stg[3].ensure(4));
    uint32_t* flags = ctx->stg[3].as<uint32_t>();
    FrameCounters* fc = ctx->fc.as<FrameCounters>();
    TGS_CUDA_OK(cudaMemsetAsync(fc, 0, offsetof(FrameCounters, sticky_overflow), ctx->stream));
    TGS_CUDA_OK(cudaMemsetAsync(flags, 0, 4, ctx->stream));
    const DevProjected planes = dev_proj(ctx);
    launch_projected_to_planes(dp, n, opt->alpha_skip, planes, ctx->stream);
    launch_lists_check(de, doff, ng, dp, n, gg, ctx->list.as<uint32_t>(), flags, ctx->stream);
    uint32_t hflags = 0;
    TGS_CUDA_OK(cudaMemcpyAsync(&hflags, flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    if (hflags & 1u) return set_err(TGS_ERR_VALIDATION, "rasterize: an entry's gaussian_index is out of range");
    if (hflags & 4u) return set_err(TGS_ERR_VALIDATION, "rasterize: offsets are not monotone");
    if (hflags & 2u)
        return set_err(TGS_ERR_VALIDATION, "rasterize: an entry's mask is not the one build_group_entries gives its "
                                           "splat in that group");
    launch_unit_order(doff, nullptr, ng * per, per, ctx->order.as<int>(), fc, ctx->stream);
    RasterArgs ra;
    ra.proj = planes;
    ra.list = ctx->list.as<uint32_t>();
    ra.offsets = doff;
    ra.order = ctx->order.as<int>();
    ra.gg = gg;
    ra.image = ctx->image.as<float>();
    ra.image_row0 = 0;
    ra.alpha_skip = opt->alpha_skip;
    ra.alpha_clamp = opt->alpha_clamp;
    ra.t_terminate = opt->t_terminate;
    ra.fc = fc;
    ra.tile_trip = nullptr;
    ra.unit_cost = nullptr;
    ra.tile_cull = ctx->tile_cull;
    if (opt->backend == TGS_BACKEND_SCALAR)
        launch_raster_scalar(ra, ctx->stream);
    else
        launch_raster_tensor(ra, ctx->num_sms, ctx->stream);
    TGS_CUDA_OK(cudaGetLastError());
    TGS_CUDA_OK(cudaMemcpyAsync(out_rgb, ctx->image.p, (size_t)width * height * 3 * sizeof(float),
                                cudaMemcpyDeviceToHost, ctx->stream));
    TGS_CUDA_OK(cudaStreamSynchronize(ctx->stream));
    // the context's frame state no longer describes a pipeline frame
    ctx->ucost_key = 0;
    return TGS_OK;
}

}  // extern "C"
