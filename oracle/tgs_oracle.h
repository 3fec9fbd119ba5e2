/* oracle/tgs_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement ("port") of the reference's forward render path in plain C11, each function
 * citing the reference file:line it follows (paths relative to /root/reference/proj).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and only as the
 * checker.  It is pinned against the reference compiled from its own sources
 * (oracle/_ref/libgsr_ref.so, see oracle/Makefile) and against the golden fixtures in
 * tests/golden/ generated from that build (tests/golden/make_golden.py).
 *
 * Layouts are those of include/tgs.h: scene records = .gsb record layout (14 or 59 floats),
 * tor_projected = ProjectedGaussian field order (44 B), tor_entry = GroupEntry (12 B).
 */
#ifndef TGS_ORACLE_H
#define TGS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    float view[16]; /* row-major world->camera */
    float focal_x, focal_y;
    int32_t width, height;
    float near_, far_;
} tor_camera;

typedef struct {
    int32_t backend, mode, group_size, workers, chunk_len;
    float alpha_skip, alpha_clamp, t_terminate;
} tor_options;

typedef struct {
    float mean2d[2];
    float conic[3];
    float color[3];
    float opacity;
    float depth;
    int32_t radius;
} tor_projected;

typedef struct {
    uint32_t gaussian_index;
    float depth;
    uint32_t mask;
} tor_entry;

typedef struct {
    uint64_t fragment_ops, chunk_loads, skipped_pairs, used_lanes, total_lanes;
    uint64_t walked_pairs;      /* entries visited per pixel until done (src/raster_scalar.cpp:36-41) */
    uint64_t blended_pairs;     /* walked pairs with alpha >= alpha_skip */
} tor_counters;

/* scene_io.cpp:218-251 (+ SplitMix64 sh_rest fill, test_scene_io.cpp:63-77). 0 or -1. */
int tor_gen_scene(uint64_t seed, int count, float extent, float smin, float smax,
                  uint64_t sh_seed, float* out);

/* projection.cpp:116-142. Returns number of projected records; stats3 = input/culled/dropped. */
int64_t tor_project(const float* rec, int64_t n, int deg, const tor_camera* cam,
                    tor_projected* out, uint64_t* stats3);

/* binning.cpp:46-100. Returns total entries; writes when total <= cap. */
int64_t tor_bin_sort(const tor_projected* p, int64_t n, int width, int height, int g,
                     tor_entry* out, int64_t cap, uint32_t* offsets, uint64_t* appearances);
/* Same result as tor_bin_sort in O(entries): (depth, index) order + stable distribution by group.
 * One call: returns total; writes entries/offsets when out != NULL and total <= cap. */
int64_t tor_bin_sort_fast(const tor_projected* p, int64_t n, int width, int height, int g,
                          tor_entry* out, int64_t cap, uint32_t* offsets, uint64_t* appearances);

/* raster_scalar.cpp:52-71 (backend 0, G must be 1) or raster_tensor.cpp:173-191 (backend 1).
 * Works on already-sorted lists; counters may be NULL. Returns 0 or -1 (validation). */
int tor_rasterize(const tor_entry* entries, const uint32_t* offsets, const tor_projected* p,
                  int width, int height, const tor_options* opt, float* out_rgb,
                  tor_counters* counters);

/* render.cpp:7-35 end to end. stats10 = {input, culled, dropped, entries, tile_appearances,
 * fragment_ops, chunk_loads, skipped_pairs, used_lanes, total_lanes}. */
int tor_render(const float* rec, int64_t n, int deg, const tor_camera* cam, const tor_options* opt,
               float* out_rgb, uint64_t* stats10, tor_counters* counters);

/* tests/oracles.hpp:112-152 tiling-free renderer. */
int tor_reference_render(const tor_projected* p, int64_t n, int width, int height, float* out_rgb);

/* half.hpp:37-84 */
uint16_t tor_f32_to_f16(float x);
float tor_f16_to_f32(uint16_t h);

/* scene_io.cpp:253-263 payload bytes. */
void tor_encode_ppm(const float* rgb, int64_t n_floats, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
