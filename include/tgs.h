/* include/tgs.h — C ABI of the B200-native TensorGS forward render path (libtgs.so).
 *
 * This is the drop-in boundary for the reference's render entry point
 *   gsr::render(const std::vector<Gaussian3D>&, const Camera&, const RenderOptions&)
 *     (reference: proj/include/gsr/render.hpp:30-31, proj/src/render.cpp:7-35)
 * and its stage API (project_scene projection.hpp:48-50, build_group_entries/sort_entries
 * binning.hpp:68-73, rasterize_tiles_scalar raster_scalar.hpp:59-62, rasterize_groups_tensor
 * raster_tensor.hpp:62-65).  Plain pointers and sizes only: no C++ or torch types cross it.
 * The C++ drop-in (cpp/gsr_b200.hpp, cpp/gsr_b200.cpp) and the Python mirror (paper_2605_17855_b200/gsr.py)
 * both sit on top of these entry points; INTEGRATION.md shows the bindings.
 *
 * Every entry point returns a tgs_status; on failure tgs_last_error() describes it.  Status
 * codes map onto the reference's exception types: VALIDATION -> gsr::ValidationError,
 * FORMAT -> gsr::FormatError (types.hpp:14-21); CUDA / OOM have no reference counterpart.
 *
 * Threading: a tgs_ctx owns one CUDA device and one stream; use a context from one host thread
 * at a time.  Contexts on different devices run concurrently (multi-GPU camera batches and
 * screen bands).  There is no CPU fallback: without a usable sm_100
 * device tgs_ctx_create fails with TGS_ERR_CUDA.
 */
#ifndef TGS_H
#define TGS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TGS_ABI_VERSION 2

typedef enum {
    TGS_OK = 0,
    TGS_ERR_VALIDATION = 1, /* gsr::ValidationError */
    TGS_ERR_FORMAT = 2,     /* gsr::FormatError */
    TGS_ERR_CUDA = 3,
    TGS_ERR_OOM = 4
} tgs_status;

/* gsr::Backend (render.hpp:8) */
enum { TGS_BACKEND_SCALAR = 0, TGS_BACKEND_TENSOR = 1 };
/* gsr::PrecisionMode (operands.hpp:13) */
enum { TGS_MODE_FP32 = 0, TGS_MODE_FP16 = 1 };

/* gsr::Camera (types.hpp:36-49): view is the row-major 4x4 world->camera transform,
 * view[r*4 + c] == Camera::view(r, c). */
typedef struct {
    float view[16];
    float focal_x, focal_y;
    int32_t width, height;
    float near_, far_;
} tgs_camera;

/* gsr::RenderOptions (render.hpp:10-17) + RasterConstants (raster_scalar.hpp:14-18).
 * backend: TGS_BACKEND_SCALAR runs the CUDA-core baseline rasterizer (requires group_size 1,
 * like raster_scalar.cpp:56-57); TGS_BACKEND_TENSOR runs the tcgen05 grouped rasterizer.
 * mode: TGS_MODE_FP32 runs the fast rasterisers (tensor: FP16 hi/lo monomial contraction on the
 * tensor cores, images within the tolerance of DESIGN.md §Precision); TGS_MODE_FP16 runs the
 * exact-emulation rasteriser, which reproduces the reference's fp16 lanes (operands.hpp:27-72)
 * bit for bit for either backend and any G.  workers and chunk_len are
 * accepted for source compatibility; the image does not depend on either (the reference pins
 * both invariances: acceptance.cpp:227-238, :359-382). */
typedef struct {
    int32_t backend;
    int32_t mode;
    int32_t group_size; /* 1, 2 or 4 */
    int32_t workers;    /* >= 1, ignored */
    int32_t chunk_len;  /* accepted, ignored */
    float alpha_skip;   /* 1/255 */
    float alpha_clamp;  /* 0.99 */
    float t_terminate;  /* 1e-4 */
} tgs_options;

/* RenderResult counters (render.hpp:19-25) + per-stage device times. */
typedef struct {
    uint64_t input, culled, dropped_degenerate; /* ProjectionStats (projection.hpp:40-44) */
    uint64_t entries;          /* group-level entries N_group */
    uint64_t tile_appearances; /* sum of mask popcounts N_total */
    uint64_t visible;          /* projected splats (input - culled - dropped) */
    float ms_preprocess, ms_binning, ms_sort, ms_raster, ms_total; /* CUDA-event times */
    /* OpReport (metrics.hpp:49-69) of the tensor rasteriser (zero for the scalar backend), in the
     * reference's units: chunk_loads = staged chunks (32 splat rows here, <= 16 there);
     * fragment_ops = m16n16k16-equivalent MMA blocks (one tcgen05.mma M=128 N=32 K=16 = 16);
     * skipped_pairs = (member tile, staged row) pairs whose mask excludes a live tile;
     * used_lanes = rows x pixels x 12 productive K lanes (the hi/lo 6-term contraction), summed
     * over MMAs; total_lanes = 16^3 per fragment. */
    uint64_t fragment_ops, chunk_loads, skipped_pairs, used_lanes, total_lanes;
} tgs_stats;

/* gsr::ProjectedGaussian (projection.hpp:14-23), 44 bytes. */
typedef struct {
    float mean2d[2];
    float conic[3]; /* a, b, c */
    float color[3];
    float opacity;
    float depth;
    int32_t radius;
} tgs_projected;

/* gsr::GroupEntry (binning.hpp:41-45), 12 bytes. */
typedef struct {
    uint32_t gaussian_index; /* index into the projected (compacted) list */
    float depth;
    uint32_t mask; /* bit r*G+c per overlapped member tile */
} tgs_group_entry;

/* gsr::KeyedEntry (binning.hpp:47-50), 16 bytes: build_group_entries output, sort_entries input. */
typedef struct {
    uint32_t group_id;
    tgs_group_entry entry;
} tgs_keyed_entry;

typedef struct tgs_ctx tgs_ctx;
typedef struct tgs_scene tgs_scene;

/* Scene records use the .gsb record layout (scene_io.hpp:38-42): per Gaussian
 *   mean f32x3, scale f32x3, quat f32x4 (w,x,y,z), opacity f32, sh_dc f32x3,
 *   [sh_rest f32x45 iff sh_degree == 3]
 * i.e. 14 or 59 floats, contiguous. */

const char* tgs_last_error(void); /* thread-local message of the last failure */
int tgs_abi_version(void);

tgs_status tgs_ctx_create(int device, tgs_ctx** out);
void tgs_ctx_destroy(tgs_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) for callers that time with their own events. */
void* tgs_ctx_stream(tgs_ctx* ctx);

/* Rasteriser tile cull (default on, both backends): a splat is skipped for a tile (tensor: for a
 * member tile of the unit) when the box of its alpha >= alpha_skip ellipse, padded half a pixel,
 * misses the tile's pixel centres.  Images are identical either way (such a splat has
 * alpha < alpha_skip on every pixel of the tile); off reproduces the reference's 3-sigma-square
 * work (binning.cpp:32-44) for A/B measurement. */
tgs_status tgs_set_tile_cull(tgs_ctx* ctx, int on);

/* Exact emulation (default off): fp32-mode frames also go through the exact-emulation rasteriser,
 * whose images equal the reference CPU build's bit for bit (CUDA cores; a validation mode). */
tgs_status tgs_set_exact_emulation(tgs_ctx* ctx, int on);

/* CUDA-graph frames (default on): the second frame of an unchanged configuration (scene, image
 * size, options, band, buffer capacities) captures the per-frame launch sequence (preprocess,
 * presort, binning, unit order, raster, ~20 launches / memsets / event records) into a graph;
 * later frames replay it with only the camera argument updated.  Images are identical either way. */
tgs_status tgs_set_graphs(tgs_ctx* ctx, int on);

/* Persistent device-resident scene (SoA, float4 planes); amortises marshalling across frames. */
tgs_status tgs_scene_upload(tgs_ctx* ctx, const float* records, int64_t count, int sh_degree,
                            tgs_scene** out);
void tgs_scene_free(tgs_scene* scene);

/* gsr::render equivalent on an uploaded scene: image to a host buffer of width*height*3 floats
 * (row-major RGB, clamped to [0,1] like ImageBuffer::finalize).  Synchronous. */
tgs_status tgs_render(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam,
                      const tgs_options* opt, float* out_rgb, tgs_stats* stats);

/* gsr::render with the reference's call shape: host records in, host image out (uploads the
 * scene, renders, downloads).  This is what the C++ drop-in calls. */
tgs_status tgs_render_records(tgs_ctx* ctx, const float* records, int64_t count, int sh_degree,
                              const tgs_camera* cam, const tgs_options* opt, float* out_rgb,
                              tgs_stats* stats);

/* Asynchronous frame on the context stream; the image stays in a device buffer
 * (tgs_image_device) until the next enqueue.  No host synchronisation. */
tgs_status tgs_render_enqueue(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam,
                              const tgs_options* opt);
/* Waits for the stream, checks capacity / validation flags, fills stats. If a buffer turned out
 * too small the frame is re-rendered synchronously with grown buffers. */
tgs_status tgs_sync(tgs_ctx* ctx, tgs_stats* stats);
const float* tgs_image_device(tgs_ctx* ctx); /* device pointer, width*height*3 floats */

/* Screen band: group rows [group_row0, group_row1) of the frame, rendered with lists restricted
 * to those groups (identical to the same rows of the full frame).  out_rgb receives the band's
 * rows only: (min(H, group_row1*16*G) - group_row0*16*G) * width * 3 floats. */
tgs_status tgs_render_band(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam,
                           const tgs_options* opt, int group_row0, int group_row1, float* out_rgb,
                           tgs_stats* stats);

/* Screen-band work estimate: entries per group row of the frame (rows = ceil(H / (16 G))), i.e.
 * the per-row totals of build_group_entries (binning.cpp:46-74), from one preprocess pass and a
 * row histogram (no lists are built).  Every rank of a band-split frame computes the same counts
 * and cuts its band with them (paper_2605_17855_b200/multigpu.py band_split). */
tgs_status tgs_group_row_entries(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cam,
                                 const tgs_options* opt, uint64_t* counts, int64_t cap, int64_t* n_rows);

/* Camera batch (BASELINE config 5; reference analogue: one gsr::render call per camera,
 * render.hpp:30-31 / tools/gsrender.cpp:112-152): n frames, out_rgb = n * width * height * 3 floats
 * (all cameras share W,H; NULL: no image copies).  Frames are pipelined over up to 3 internal lanes
 * (extra streams + buffers on the same device, created on first use and owned by ctx), so one
 * frame's image copy and latency-bound raster overlap the next frames' preprocess/sort/binning.
 * Images are identical to n single renders. */
tgs_status tgs_render_batch(tgs_ctx* ctx, const tgs_scene* scene, const tgs_camera* cams, int n,
                            const tgs_options* opt, float* out_rgb, tgs_stats* stats);

/* Readback of the last rendered frame's intermediate products, for parity tests and tooling.
 * project: ProjectedGaussian list in input order (project_scene). lists: the (group, depth)
 * sorted GroupEntry array and group_count+1 offsets (sort_entries).  *n receives the count;
 * nothing is written when cap is too small. */
tgs_status tgs_read_projected(tgs_ctx* ctx, tgs_projected* out, int64_t cap, int64_t* n);
tgs_status tgs_read_lists(tgs_ctx* ctx, tgs_group_entry* out, int64_t cap, uint32_t* offsets,
                          int64_t offsets_cap, int64_t* n);

/* ---- The reference's public stage API on caller-provided data (one GPU call per stage). ------
 * Each call is synchronous, uses the context's stream and scratch buffers, and validates like the
 * reference (GroupConfig::validate binning.cpp:22-30 -> VALIDATION).  Variable-size outputs use
 * the two-call pattern: *n receives the size, nothing is written when cap is too small. */

/* project_scene(scene, cam, workers, &stats) (projection.hpp:48-50): compacted projected list in
 * input order; stats receives input / culled / dropped_degenerate.  Non-positive scales of
 * visible Gaussians -> VALIDATION (projection.cpp:37). */
tgs_status tgs_project_scene(tgs_ctx* ctx, const float* records, int64_t count, int sh_degree,
                             const tgs_camera* cam, tgs_projected* out, int64_t cap, int64_t* n,
                             tgs_stats* stats);
/* build_group_entries(projected, GroupConfig::square(G, width, height)) (binning.hpp:68-69): one
 * KeyedEntry per (splat, overlapped group), splat order then group id (gy outer, gx inner). */
tgs_status tgs_build_group_entries(tgs_ctx* ctx, const tgs_projected* proj, int64_t n, int width, int height,
                                   int group_size, tgs_keyed_entry* out, int64_t cap, int64_t* n_out);
/* sort_entries(entries, cfg) (binning.hpp:72-73): entries stably sorted by
 * (group_id << 32) | f32_bits(depth), offsets = group_count + 1 prefix offsets.  A non-finite
 * or negative depth -> VALIDATION (binning.cpp:78-83); a group id >= group_count -> VALIDATION. */
tgs_status tgs_sort_entries(tgs_ctx* ctx, const tgs_keyed_entry* entries, int64_t n, int width, int height,
                            int group_size, tgs_group_entry* out, uint32_t* offsets, int64_t offsets_cap);
/* rasterize_tiles_scalar (opt->backend SCALAR, G must be 1: raster_scalar.cpp:56-57) /
 * rasterize_groups_tensor (TENSOR) (raster_scalar.hpp:59-62, raster_tensor.hpp:62-65) on caller
 * lists: entries/offsets as sort_entries returns them for GroupConfig::square(opt->group_size,
 * width, height).  Every entry's mask must be the one build_group_entries derives from its
 * splat (the GPU rasterisers recompute masks), its index must address proj -> VALIDATION
 * otherwise.  out_rgb: width * height * 3 floats, clamped like ImageBuffer::finalize. */
tgs_status tgs_rasterize_lists(tgs_ctx* ctx, const tgs_group_entry* entries, int64_t n_entries,
                               const uint32_t* offsets, int64_t offsets_count, const tgs_projected* proj,
                               int64_t n, int width, int height, const tgs_options* opt, float* out_rgb);

/* Walked / alpha-contributing pair counts of the last frame (the raster roofline numerator,
 * DESIGN.md §Roofline); computed by an instrumented pass, not by the timed kernels. */
tgs_status tgs_count_pairs(tgs_ctx* ctx, uint64_t* walked, uint64_t* blended);

/* ReuseReport of the last frame's group lists (reference: load_reduction, metrics.cpp:45-57):
 * n_group = group entries, n_total = sum of their mask popcounts (tile appearances),
 * load_reduction = 1 - n_group / n_total, hist[p] = entries whose mask has popcount p (1..16;
 * hist[0] = 0).  Computed on the device from the splats' tile rectangles.  VALIDATION when the
 * frame has no entries (the reference throws on an empty list). */
tgs_status tgs_reuse_report(tgs_ctx* ctx, uint64_t* n_group, uint64_t* n_total, double* load_reduction,
                            uint64_t hist[17]);

/* Per tile of the last frame (band-local, row-major): how many entries of the tile's
 * mask-filtered list the slowest pixel walked before terminating (the tile's trip).  Tooling for
 * load-balance analysis; *n receives the tile count. */
tgs_status tgs_tile_trips(tgs_ctx* ctx, uint32_t* trips, int64_t cap, int64_t* n);

/* Host-side data formats either side of the path (scene_io.cpp). */
tgs_status tgs_gen_synthetic_scene(uint64_t seed, int count, float extent, float scale_min,
                                   float scale_max, uint64_t sh_seed, float* out_records);
/* encode_ppm payload (scene_io.cpp:253-263) of a host RGB float image on the device. */
tgs_status tgs_encode_u8(tgs_ctx* ctx, const float* rgb_device, int64_t n, uint8_t* out_host);

#ifdef __cplusplus
}
#endif
#endif /* TGS_H */
