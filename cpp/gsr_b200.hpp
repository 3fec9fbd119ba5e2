// gsr_b200.hpp — C++ drop-in for the reference's render entry point on B200 (libtgs.so).
//
// Source-compatible re-declaration of the types a caller of the reference uses
//   gsr::render(const std::vector<Gaussian3D>&, const Camera&, const RenderOptions&)
//     (reference: proj/include/gsr/render.hpp:8-31, src/render.cpp:7-35)
// with Gaussian3D / Camera / ImageBuffer / FormatError / ValidationError (types.hpp:14-69),
// ProjectionStats (projection.hpp:40-44), OpReport (metrics.hpp:49-69), RasterConstants
// (raster_scalar.hpp:14-18), PrecisionMode (operands.hpp:13).  A program written against the
// reference's render.hpp compiles against this header unchanged and links libtgs.so instead of
// the reference's libgsr; the pipeline runs on the GPU behind the C ABI in include/tgs.h.
//
// Like the reference, the types hold Eigen values, so the caller's Eigen (>= 3.3, the reference's
// own dependency, CMakeLists.txt:14) must be on the include path.
//
// Differences a caller can observe: images are within the stated FP16
// tolerance of the reference's fp32 image instead of byte-identical; RenderResult::ops counts the
// GPU rasteriser's work in the reference's units (include/tgs.h tgs_stats: one tcgen05.mma
// M=128 N=32 K=16 = 16 m16n16k16 fragments, chunks of 32 rows); `workers` and `chunk_len` are
// validated like the reference and otherwise ignored.
#pragma once

#include <Eigen/Core>
#include <Eigen/Geometry>

#include <array>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace gsr {

struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
/// CUDA failure / out of device memory (no counterpart in the CPU reference).
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline constexpr int kShRestCoeffs = 45;
inline constexpr int kFragmentDim = 16;

struct Gaussian3D {
    Eigen::Vector3f mean = Eigen::Vector3f::Zero();
    Eigen::Vector3f scale = Eigen::Vector3f::Ones();
    Eigen::Quaternionf rotation = Eigen::Quaternionf::Identity();
    float opacity = 1.0f;
    Eigen::Vector3f sh_dc = Eigen::Vector3f::Zero();
    std::optional<std::array<float, kShRestCoeffs>> sh_rest;
};

struct Camera {
    Eigen::Matrix4f view = Eigen::Matrix4f::Identity();
    float focal_x = 0.0f;
    float focal_y = 0.0f;
    int width = 0;
    int height = 0;
    float near = 0.0f;
    float far = 0.0f;

    Eigen::Matrix3f rotation() const { return view.topLeftCorner<3, 3>(); }
    Eigen::Vector3f translation() const { return view.topRightCorner<3, 1>(); }
    Eigen::Vector3f position() const { return -(rotation().transpose() * translation()); }
};

struct ImageBuffer {
    int width = 0;
    int height = 0;
    std::vector<float> rgb;

    ImageBuffer() = default;
    ImageBuffer(int w, int h) : width(w), height(h), rgb(static_cast<size_t>(w) * h * 3, 0.0f) {}
    float* pixel(int x, int y) { return &rgb[(static_cast<size_t>(y) * width + x) * 3]; }
    const float* pixel(int x, int y) const { return &rgb[(static_cast<size_t>(y) * width + x) * 3]; }
    void finalize() {
        for (float& v : rgb) v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
    }
};

enum class PrecisionMode { fp32, fp16 };

struct RasterConstants {
    float alpha_skip = 1.0f / 255.0f;
    float alpha_clamp = 0.99f;
    float t_terminate = 1e-4f;
};

struct ProjectionStats {
    std::size_t input = 0;
    std::size_t culled = 0;
    std::size_t dropped_degenerate = 0;
};

struct OpReport {
    std::uint64_t fragment_ops = 0;
    std::uint64_t chunk_loads = 0;
    std::uint64_t skipped_pairs = 0;
    std::uint64_t used_lanes = 0;
    std::uint64_t total_lanes = 0;
    double padding_waste() const {
        return total_lanes ? 1.0 - static_cast<double>(used_lanes) / static_cast<double>(total_lanes) : 0.0;
    }
};

enum class Backend { scalar, tensor };

struct RenderOptions {
    Backend backend = Backend::tensor;
    PrecisionMode mode = PrecisionMode::fp32;
    int group_size = 2;
    int workers = 1;
    int chunk_len = kFragmentDim;
    RasterConstants constants{};
};

struct RenderResult {
    ImageBuffer image;
    ProjectionStats projection;
    OpReport ops;
    std::uint64_t entries = 0;
    std::uint64_t tile_appearances = 0;
};

// ---- stage API (projection.hpp, binning.hpp, raster_scalar.hpp, raster_tensor.hpp) ----------
// Same declarations as the reference's public stage API; every stage runs on the GPU through the
// C ABI on the caller's data (tgs_project_scene, tgs_build_group_entries, tgs_sort_entries,
// tgs_rasterize_lists).  Lists and projected records are bit-exact with the reference; images are
// within the FP16 tolerance.  `workers`/`chunk_len` are validated and otherwise ignored.

/// Screen-space splat (projection.hpp:14-23).
struct ProjectedGaussian {
    Eigen::Vector2f mean2d = Eigen::Vector2f::Zero();
    float conic_a = 0.0f;
    float conic_b = 0.0f;
    float conic_c = 0.0f;
    Eigen::Vector3f color = Eigen::Vector3f::Zero();
    float opacity = 0.0f;
    float depth = 0.0f;
    int radius = 0;
};

/// project_scene (projection.hpp:48-50).
std::vector<ProjectedGaussian> project_scene(const std::vector<Gaussian3D>& scene, const Camera& cam, int workers,
                                             ProjectionStats* stats = nullptr);

inline constexpr int kTileSize = 16;

/// GroupConfig (binning.hpp:15-31).
struct GroupConfig {
    int group_h = 2;
    int group_w = 2;
    int image_width = 0;
    int image_height = 0;
    static GroupConfig square(int g, int image_width, int image_height);
    int tiles_x() const { return (image_width + kTileSize - 1) / kTileSize; }
    int tiles_y() const { return (image_height + kTileSize - 1) / kTileSize; }
    int groups_x() const { return (tiles_x() + group_w - 1) / group_w; }
    int groups_y() const { return (tiles_y() + group_h - 1) / group_h; }
    int group_count() const { return groups_x() * groups_y(); }
    int tiles_per_group() const { return group_h * group_w; }
    void validate() const;
};

/// TileRect (binning.hpp:34-37).
struct TileRect {
    int min_x = 0, min_y = 0, max_x = -1, max_y = -1;
    bool empty() const { return max_x < min_x || max_y < min_y; }
};

/// GroupEntry / KeyedEntry / SortedGroupLists (binning.hpp:41-59).
struct GroupEntry {
    std::uint32_t gaussian_index = 0;
    float depth = 0.0f;
    std::uint32_t mask = 0;
};
struct KeyedEntry {
    std::uint32_t group_id = 0;
    GroupEntry entry;
};
struct SortedGroupLists {
    std::vector<GroupEntry> entries;
    std::vector<std::uint32_t> offsets;  // group_count + 1 prefix offsets
    std::uint32_t group_begin(int group) const { return offsets[group]; }
    std::uint32_t group_end(int group) const { return offsets[group + 1]; }
};

/// tiles_overlapped (binning.hpp:63-64): the splat's AABB clipped to the tile grid (host helper).
TileRect tiles_overlapped(const ProjectedGaussian& p, const GroupConfig& cfg);
/// build_group_entries (binning.hpp:68-69) — on the GPU.
std::vector<KeyedEntry> build_group_entries(const std::vector<ProjectedGaussian>& projected, const GroupConfig& cfg);
/// sort_entries (binning.hpp:72-73) — hand-written radix sort on the GPU.
SortedGroupLists sort_entries(std::vector<KeyedEntry> entries, const GroupConfig& cfg);

/// rasterize_tiles_scalar (raster_scalar.hpp:59-62) — the CUDA-core baseline kernel.
ImageBuffer rasterize_tiles_scalar(const SortedGroupLists& lists, const std::vector<ProjectedGaussian>& projected,
                                   const GroupConfig& cfg, const RasterConstants& k,
                                   PrecisionMode mode = PrecisionMode::fp32, int workers = 1);

/// TensorRasterOptions (raster_tensor.hpp:45-50).
struct TensorRasterOptions {
    RasterConstants constants{};
    PrecisionMode mode = PrecisionMode::fp32;
    int chunk_len = kFragmentDim;
    int workers = 1;
};
/// rasterize_groups_tensor (raster_tensor.hpp:62-65) — the tcgen05 grouped kernel.  `ops` is
/// left untouched (the CPU fragment-emulation counters have no GPU meaning).
ImageBuffer rasterize_groups_tensor(const SortedGroupLists& lists, const std::vector<ProjectedGaussian>& projected,
                                    const GroupConfig& cfg, const TensorRasterOptions& opt, OpReport* ops = nullptr);

/// Drop-in for the reference's gsr::render: uploads the scene, renders on the current B200
/// (device 0 unless gsr::b200::set_device was called), downloads the image.
RenderResult render(const std::vector<Gaussian3D>& scene, const Camera& cam, const RenderOptions& opt);

// .gsb scene files (scene_io.hpp:42-43): same byte layout, checks, messages and quaternion
// renormalisation as the reference (FormatError / ValidationError).
std::vector<Gaussian3D> load_scene(const std::string& path);
void save_scene(const std::vector<Gaussian3D>& gaussians, const std::string& path);

namespace b200 {

/// Device used by gsr::render on this thread (default 0).
void set_device(int device);

/// Per-stage device times of the last render on this thread (CUDA events, milliseconds).
struct StageTimes {
    float preprocess = 0, binning = 0, sort = 0, raster = 0, total = 0;
};
StageTimes last_stage_times();

/// Persistent device-resident scene: marshal + upload once, render many cameras.
class DeviceScene {
public:
    explicit DeviceScene(const std::vector<Gaussian3D>& scene, int device = 0);
    ~DeviceScene();
    DeviceScene(const DeviceScene&) = delete;
    DeviceScene& operator=(const DeviceScene&) = delete;
    RenderResult render(const Camera& cam, const RenderOptions& opt);

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace b200
}  // namespace gsr
