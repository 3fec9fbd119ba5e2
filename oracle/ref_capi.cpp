// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// A flat C wrapper over the *reference's own* C++ API, compiled together with the unmodified
// reference sources under /root/reference/proj/src (see oracle/Makefile) into
// oracle/_ref/libgsr_ref.so.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
// `--impl reference` legs load it, always as the checker or the timed reference arm — never as
// the product path.
//
// Data layouts are the ones declared in include/tgs.h (scene records = the .gsb record layout of
// scene_io.cpp:45-100; projected = ProjectedGaussian field order; entries = GroupEntry).

#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "gsr/metrics.hpp"
#include "gsr/render.hpp"
#include "oracles.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return -code;
}

struct CCamera {
    float view[16];  // row-major
    float focal_x, focal_y;
    std::int32_t width, height;
    float near_, far_;
};

struct COptions {
    std::int32_t backend, mode, group_size, workers, chunk_len;
    float alpha_skip, alpha_clamp, t_terminate;
};

struct CProjected {
    float mean2d[2];
    float conic[3];
    float color[3];
    float opacity;
    float depth;
    std::int32_t radius;
};
static_assert(sizeof(CProjected) == 44);

gsr::Camera to_cam(const CCamera* c) {
    gsr::Camera cam;
    for (int r = 0; r < 4; ++r)
        for (int k = 0; k < 4; ++k) cam.view(r, k) = c->view[r * 4 + k];
    cam.focal_x = c->focal_x;
    cam.focal_y = c->focal_y;
    cam.width = c->width;
    cam.height = c->height;
    cam.near = c->near_;
    cam.far = c->far_;
    return cam;
}

std::vector<gsr::Gaussian3D> to_scene(const float* rec, std::int64_t n, int deg) {
    const int rf = deg == 3 ? 59 : 14;
    std::vector<gsr::Gaussian3D> s(static_cast<size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) {
        const float* p = rec + i * rf;
        gsr::Gaussian3D& g = s[static_cast<size_t>(i)];
        g.mean = {p[0], p[1], p[2]};
        g.scale = {p[3], p[4], p[5]};
        g.rotation = Eigen::Quaternionf(p[6], p[7], p[8], p[9]);
        g.opacity = p[10];
        g.sh_dc = {p[11], p[12], p[13]};
        if (deg == 3) {
            std::array<float, gsr::kShRestCoeffs> r;
            for (int k = 0; k < gsr::kShRestCoeffs; ++k) r[k] = p[14 + k];
            g.sh_rest = r;
        }
    }
    return s;
}

void from_proj(const gsr::ProjectedGaussian& p, CProjected& o) {
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
}

gsr::ProjectedGaussian to_proj(const CProjected& o) {
    gsr::ProjectedGaussian p;
    p.mean2d = {o.mean2d[0], o.mean2d[1]};
    p.conic_a = o.conic[0];
    p.conic_b = o.conic[1];
    p.conic_c = o.conic[2];
    p.color = {o.color[0], o.color[1], o.color[2]};
    p.opacity = o.opacity;
    p.depth = o.depth;
    p.radius = o.radius;
    return p;
}

gsr::RenderOptions to_opt(const COptions* o) {
    gsr::RenderOptions opt;
    opt.backend = o->backend == 0 ? gsr::Backend::scalar : gsr::Backend::tensor;
    opt.mode = o->mode == 0 ? gsr::PrecisionMode::fp32 : gsr::PrecisionMode::fp16;
    opt.group_size = o->group_size;
    opt.workers = o->workers;
    opt.chunk_len = o->chunk_len;
    opt.constants.alpha_skip = o->alpha_skip;
    opt.constants.alpha_clamp = o->alpha_clamp;
    opt.constants.t_terminate = o->t_terminate;
    return opt;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* gref_last_error() { return g_err.c_str(); }

int gref_hardware_concurrency() { return static_cast<int>(std::thread::hardware_concurrency()); }

// gen_synthetic_scene (scene_io.cpp:218-251) into .gsb-layout records; sh_seed != 0 adds 45
// sh_rest coefficients per Gaussian drawn from SplitMix64(sh_seed).uniform(-1, 1)
// (test_scene_io.cpp:63-77 pattern).  out must hold count * (sh_seed ? 59 : 14) floats.
int gref_gen_scene(std::uint64_t seed, int count, float extent, float smin, float smax,
                   std::uint64_t sh_seed, float* out) {
    try {
        auto s = gsr::gen_synthetic_scene(seed, count, extent, {smin, smax});
        gsr::SplitMix64 rng(sh_seed);
        const int rf = sh_seed ? 59 : 14;
        for (int i = 0; i < count; ++i) {
            float* p = out + static_cast<size_t>(i) * rf;
            const auto& g = s[static_cast<size_t>(i)];
            p[0] = g.mean.x(); p[1] = g.mean.y(); p[2] = g.mean.z();
            p[3] = g.scale.x(); p[4] = g.scale.y(); p[5] = g.scale.z();
            p[6] = g.rotation.w(); p[7] = g.rotation.x(); p[8] = g.rotation.y(); p[9] = g.rotation.z();
            p[10] = g.opacity;
            p[11] = g.sh_dc.x(); p[12] = g.sh_dc.y(); p[13] = g.sh_dc.z();
            if (sh_seed)
                for (int k = 0; k < 45; ++k) p[14 + k] = rng.uniform(-1.0f, 1.0f);
        }
        return 0;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// project_scene (projection.cpp:116-142). Returns the number of projected records (>= 0).
std::int64_t gref_project(const float* rec, std::int64_t n, int deg, const CCamera* cam,
                          int workers, CProjected* out, std::uint64_t* stats3) {
    try {
        const auto scene = to_scene(rec, n, deg);
        gsr::ProjectionStats st;
        const auto pr = gsr::project_scene(scene, to_cam(cam), workers, &st);
        for (size_t i = 0; i < pr.size(); ++i) from_proj(pr[i], out[i]);
        if (stats3) {
            stats3[0] = st.input;
            stats3[1] = st.culled;
            stats3[2] = st.dropped_degenerate;
        }
        return static_cast<std::int64_t>(pr.size());
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// build_group_entries + sort_entries (binning.cpp:46-100) over a projected list.
// Writes up to `cap` entries (index, depth, mask as GroupEntry) plus group_count+1 offsets; the
// return value is the total entry count (call again with a larger cap if it exceeds cap).
// tile_appearances (popcount sum, render.cpp:19-20) goes to *appearances if non-null.
std::int64_t gref_bin_sort(const CProjected* proj, std::int64_t n, int width, int height, int g,
                           gsr::GroupEntry* out, std::int64_t cap, std::uint32_t* offsets,
                           std::uint64_t* appearances) {
    try {
        std::vector<gsr::ProjectedGaussian> pr(static_cast<size_t>(n));
        for (std::int64_t i = 0; i < n; ++i) pr[static_cast<size_t>(i)] = to_proj(proj[i]);
        const auto cfg = gsr::GroupConfig::square(g, width, height);
        auto entries = gsr::build_group_entries(pr, cfg);
        if (appearances) {
            std::uint64_t a = 0;
            for (const auto& e : entries) a += static_cast<std::uint64_t>(std::popcount(e.entry.mask));
            *appearances = a;
        }
        const std::int64_t total = static_cast<std::int64_t>(entries.size());
        if (total > cap) return total;
        const auto lists = gsr::sort_entries(std::move(entries), cfg);
        std::memcpy(out, lists.entries.data(), lists.entries.size() * sizeof(gsr::GroupEntry));
        std::memcpy(offsets, lists.offsets.data(), lists.offsets.size() * sizeof(std::uint32_t));
        return total;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// gsr::render (render.cpp:7-35). out_rgb: width*height*3 floats. stats: see tgs_stats layout
// prefix {input, culled, dropped, entries, tile_appearances, fragment_ops, chunk_loads,
// skipped_pairs, used_lanes, total_lanes} as uint64.
int gref_render(const float* rec, std::int64_t n, int deg, const CCamera* cam, const COptions* opt,
                float* out_rgb, std::uint64_t* stats10) {
    try {
        const auto scene = to_scene(rec, n, deg);
        const auto res = gsr::render(scene, to_cam(cam), to_opt(opt));
        std::memcpy(out_rgb, res.image.rgb.data(), res.image.rgb.size() * sizeof(float));
        if (stats10) {
            const std::uint64_t v[10] = {res.projection.input, res.projection.culled,
                                         res.projection.dropped_degenerate, res.entries,
                                         res.tile_appearances, res.ops.fragment_ops,
                                         res.ops.chunk_loads, res.ops.skipped_pairs,
                                         res.ops.used_lanes, res.ops.total_lanes};
            std::memcpy(stats10, v, sizeof(v));
        }
        return 0;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const gsr::FormatError& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// Rasterize an explicit projected list (projection bypassed) with the reference's own binning,
// sort and rasterizer; used to check GPU rasterizers on hand-built splats.
int gref_raster_projected(const CProjected* proj, std::int64_t n, int width, int height,
                          const COptions* opt, float* out_rgb) {
    try {
        std::vector<gsr::ProjectedGaussian> pr(static_cast<size_t>(n));
        for (std::int64_t i = 0; i < n; ++i) pr[static_cast<size_t>(i)] = to_proj(proj[i]);
        const gsr::RenderOptions o = to_opt(opt);
        const auto cfg = gsr::GroupConfig::square(o.group_size, width, height);
        const auto lists = gsr::sort_entries(gsr::build_group_entries(pr, cfg), cfg);
        gsr::ImageBuffer img;
        if (o.backend == gsr::Backend::scalar) {
            img = gsr::rasterize_tiles_scalar(lists, pr, cfg, o.constants, o.mode, o.workers);
        } else {
            gsr::TensorRasterOptions t;
            t.constants = o.constants;
            t.mode = o.mode;
            t.chunk_len = o.chunk_len;
            t.workers = o.workers;
            img = gsr::rasterize_groups_tensor(lists, pr, cfg, t);
        }
        std::memcpy(out_rgb, img.rgb.data(), img.rgb.size() * sizeof(float));
        return 0;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// tests/oracles.hpp:112-152 tiling-free renderer.
int gref_reference_render(const CProjected* proj, std::int64_t n, int width, int height,
                          float* out_rgb) {
    try {
        std::vector<gsr::ProjectedGaussian> pr(static_cast<size_t>(n));
        for (std::int64_t i = 0; i < n; ++i) pr[static_cast<size_t>(i)] = to_proj(proj[i]);
        const auto img = oracle::reference_render(pr, width, height, gsr::RasterConstants{});
        std::memcpy(out_rgb, img.rgb.data(), img.rgb.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// Per-stage timing of the reference's own public stage API (render.cpp:7-35 decomposed), used as
// the CPU baseline.  band_y0/band_h select a horizontal band of whole group rows (band_h <= 0:
// the full frame): the projected list is shifted by -band_y0 (an exact float subtraction for
// every splat that can reach the band) and binned/sorted/rasterised into a band_h-row image with
// the reference's unmodified functions.  ms4 = {project, bin, sort, raster}; returns entries.
std::int64_t gref_time_stages(const float* rec, std::int64_t n, int deg, const CCamera* cam,
                              const COptions* opt, int band_y0, int band_h, double* ms4) {
    try {
        const auto scene = to_scene(rec, n, deg);
        const gsr::RenderOptions o = to_opt(opt);
        const gsr::Camera c = to_cam(cam);
        auto t0 = std::chrono::steady_clock::now();
        auto pr = gsr::project_scene(scene, c, o.workers);
        ms4[0] = ms_since(t0);
        int h = c.height;
        if (band_h > 0) {
            h = band_h;
            for (auto& p : pr) p.mean2d.y() -= static_cast<float>(band_y0);
        }
        const auto cfg = gsr::GroupConfig::square(o.group_size, c.width, h);
        t0 = std::chrono::steady_clock::now();
        auto entries = gsr::build_group_entries(pr, cfg);
        ms4[1] = ms_since(t0);
        const std::int64_t total = static_cast<std::int64_t>(entries.size());
        t0 = std::chrono::steady_clock::now();
        const auto lists = gsr::sort_entries(std::move(entries), cfg);
        ms4[2] = ms_since(t0);
        t0 = std::chrono::steady_clock::now();
        if (o.backend == gsr::Backend::scalar) {
            auto img = gsr::rasterize_tiles_scalar(lists, pr, cfg, o.constants, o.mode, o.workers);
        } else {
            gsr::TensorRasterOptions t;
            t.constants = o.constants;
            t.mode = o.mode;
            t.chunk_len = o.chunk_len;
            t.workers = o.workers;
            auto img = gsr::rasterize_groups_tensor(lists, pr, cfg, t);
        }
        ms4[3] = ms_since(t0);
        return total;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// The same stage API with project_scene run ONCE per frame and the remaining stages run per
// horizontal band: band k of n_bands covers group rows [round(k*gy/n), round((k+1)*gy/n)).
// Bands [band_first, band_first + band_count) are timed; ms = {project, then per timed band
// bin, sort, raster}.  Returns the sum of the timed bands' image rows.  Each band copies and
// shifts the projected list (untimed), exactly like gref_time_stages.
std::int64_t gref_time_bands(const float* rec, std::int64_t n, int deg, const CCamera* cam, const COptions* opt,
                             int n_bands, int band_first, int band_count, double* ms, float* img) {
    try {
        const auto scene = to_scene(rec, n, deg);
        const gsr::RenderOptions o = to_opt(opt);
        const gsr::Camera c = to_cam(cam);
        auto t0 = std::chrono::steady_clock::now();
        const auto pr_full = gsr::project_scene(scene, c, o.workers);
        ms[0] = ms_since(t0);
        const int g16 = o.group_size * 16;
        const int gy = (c.height + g16 - 1) / g16;
        std::int64_t rows = 0;
        for (int b = 0; b < band_count; ++b) {
            const int k = (band_first + b) % n_bands;
            const int r0 = static_cast<int>(std::lround(static_cast<double>(k) * gy / n_bands));
            const int r1 = static_cast<int>(std::lround(static_cast<double>(k + 1) * gy / n_bands));
            const int y0 = r0 * g16, y1 = std::min(c.height, r1 * g16);
            double* m = ms + 1 + 3 * b;
            m[0] = m[1] = m[2] = 0.0;
            if (y1 <= y0) continue;
            rows += y1 - y0;
            auto pr = pr_full;
            for (auto& p : pr) p.mean2d.y() -= static_cast<float>(y0);
            const auto cfg = gsr::GroupConfig::square(o.group_size, c.width, y1 - y0);
            t0 = std::chrono::steady_clock::now();
            auto entries = gsr::build_group_entries(pr, cfg);
            m[0] = ms_since(t0);
            t0 = std::chrono::steady_clock::now();
            const auto lists = gsr::sort_entries(std::move(entries), cfg);
            m[1] = ms_since(t0);
            t0 = std::chrono::steady_clock::now();
            gsr::ImageBuffer band;
            if (o.backend == gsr::Backend::scalar) {
                band = gsr::rasterize_tiles_scalar(lists, pr, cfg, o.constants, o.mode, o.workers);
            } else {
                gsr::TensorRasterOptions t;
                t.constants = o.constants;
                t.mode = o.mode;
                t.chunk_len = o.chunk_len;
                t.workers = o.workers;
                band = gsr::rasterize_groups_tensor(lists, pr, cfg, t);
            }
            m[2] = ms_since(t0);
            // optional (untimed): the band's rows of the frame image, for a parity check by the caller
            if (img) std::copy(band.rgb.begin(), band.rgb.end(), img + static_cast<size_t>(y0) * c.width * 3);
        }
        return rows;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// load_reduction (metrics.cpp:45-57) over a projected list: out = {n_total, n_group, hist[17]}.
int gref_load_reduction(const CProjected* proj, std::int64_t n, int width, int height, int g,
                        std::uint64_t* out19, double* reduction) {
    try {
        std::vector<gsr::ProjectedGaussian> pr(static_cast<size_t>(n));
        for (std::int64_t i = 0; i < n; ++i) pr[static_cast<size_t>(i)] = to_proj(proj[i]);
        const auto cfg = gsr::GroupConfig::square(g, width, height);
        const auto r = gsr::load_reduction(gsr::build_group_entries(pr, cfg));
        out19[0] = r.n_total;
        out19[1] = r.n_group;
        for (int k = 0; k < 17; ++k) out19[2 + k] = r.mask_popcount_hist[k];
        *reduction = r.load_reduction;
        return 0;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// save_scene / load_scene (scene_io.cpp:43-136) through the reference, for the .gsb I/O parity
// tests: records in .gsb order (14 or 59 floats per Gaussian).
int gref_save_scene(const float* rec, std::int64_t n, int deg, const char* path) {
    try {
        gsr::save_scene(to_scene(rec, n, deg), path);
        return 0;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const gsr::FormatError& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// *count / *deg of the file; out (cap floats) receives the records when large enough.
int gref_load_scene(const char* path, float* out, std::int64_t cap, std::int64_t* count, int* deg) {
    try {
        const auto s = gsr::load_scene(path);
        const int d = (!s.empty() && s[0].sh_rest) ? 3 : 0;
        const int rf = d == 3 ? 59 : 14;
        *count = static_cast<std::int64_t>(s.size());
        *deg = d;
        if (cap < *count * rf) return 0;
        for (size_t i = 0; i < s.size(); ++i) {
            float* p = out + i * rf;
            const auto& g = s[i];
            p[0] = g.mean.x(); p[1] = g.mean.y(); p[2] = g.mean.z();
            p[3] = g.scale.x(); p[4] = g.scale.y(); p[5] = g.scale.z();
            p[6] = g.rotation.w(); p[7] = g.rotation.x(); p[8] = g.rotation.y(); p[9] = g.rotation.z();
            p[10] = g.opacity;
            p[11] = g.sh_dc.x(); p[12] = g.sh_dc.y(); p[13] = g.sh_dc.z();
            if (d == 3)
                for (int k = 0; k < 45; ++k) p[14 + k] = (*g.sh_rest)[static_cast<size_t>(k)];
        }
        return 0;
    } catch (const gsr::ValidationError& e) {
        return fail(e, 1);
    } catch (const gsr::FormatError& e) {
        return fail(e, 2);
    } catch (const std::exception& e) {
        return fail(e, 9);
    }
}

// encode_ppm (scene_io.cpp:253-263) payload bytes (header stripped) for parity of the u8 path.
int gref_encode_ppm(const float* rgb, int width, int height, std::uint8_t* out) {
    gsr::ImageBuffer img(width, height);
    std::memcpy(img.rgb.data(), rgb, img.rgb.size() * sizeof(float));
    const auto bytes = gsr::encode_ppm(img);
    const size_t payload = img.rgb.size();
    std::memcpy(out, bytes.data() + (bytes.size() - payload), payload);
    return 0;
}

}  // extern "C"
