// Kernel argument structs and launchers shared between the .cu files of libtgs.
#pragma once

#include "tgs_common.cuh"

namespace tgs {

struct PreprocessArgs {
    DevScene scene;
    DevCamera cam;
    DevProjected out;
    uint32_t* depth_keys;          // [n] depth bits (presort keys; kCulledKey when not projected)
    uint2* rect;                   // [n] tile rect: x0 | x1 << 16, y0 | y1 << 16 (x0 > x1: none;
                                   //     kCulledRect twice: not projected)
    GroupGeom gg;
    FrameCounters* fc;
    float alpha_skip;              // for the tile-cull extents stored in col.w (tight_extents)
};
void launch_preprocess(const PreprocessArgs& a, cudaStream_t st);
// the preprocess kernel's entry (CUDA-graph frames update its camera argument per launch)
const void* preprocess_kernel_fn();

// ---- radix sort (LSD, stable, u32 keys + u32 values, device-side item count) --------------
struct SortBuffers {
    uint32_t* keys[2];
    uint32_t* vals[2];
    uint32_t* ghist;      // sort_scratch_elems(max_items): [digit][tile] counts, scanned in place
    uint32_t* scan_tmp;   // scan_tmp_elems(sort_scratch_elems(max_items))
    // Optional device word: when set, a last pass whose digit is constant (the identity) is skipped
    // instead of copied, and the index of the buffer holding the result is written here.
    uint32_t* result_sel = nullptr;
};
constexpr int kSortBlocks = 592;  // 4 x 148 SMs (grid of the binning/scan helpers)
size_t sort_scratch_elems(size_t max_items);
size_t sort_result_sel_offset();  // a free word of the sort scratch (ghist) for SortBuffers::result_sel
// Sorts keys[0]/vals[0] by bits [0, nbits) in 8-bit passes; the first pass covers
// *count_first items and, with drop_first, drops keys equal to kCulledKey; later passes cover
// *count_rest items (device-side counts, <= max_items).  Result in keys[r]/vals[r], r returned.
// want_keys_last == false skips writing keys in the last pass (only values are needed downstream).
// key_min_inv (device, may be null) holds ~min over the sorted keys: digits are taken from
// (key - min), which keeps the order and leaves the passes above the key range trivial (copies).
// index_vals: the first pass takes item i's value to be i (vals[0] is not read).
// With b.result_sel the result is in vals[*result_sel] (device word; r or r ^ 1).
int radix_sort(SortBuffers& b, const uint32_t* count_first, const uint32_t* count_rest, int nbits,
               bool drop_first, bool want_keys_last, size_t max_items, cudaStream_t st,
               const uint32_t* key_min_inv = nullptr, bool index_vals = false);

// ---- binning: stable counting sort of (group, rank) entries ---------------------------------
// The splats are presorted by (depth, index) (rank order); every warp of the count/scatter grids
// owns a contiguous rank range ("chunk").  count: per-chunk group histograms via 2D difference
// arrays; scan: exclusive scan of the [group][chunk] matrix; scatter: each chunk writes its entries
// at its cursors in rank order.  The result equals std::stable_sort on (group << 32 | depth bits)
// of the reference (binning.cpp:86-91) entry for entry.
struct BinArgs {
    const uint32_t* visible;     // &fc->visible (device-side count)
    const uint32_t* sval[2];     // rank -> splat index: the presort's two value buffers,
    const uint32_t* sval_sel;    // of which buffer *sval_sel holds the result (device word)
    const uint2* rect;           // splat index -> tile rect
    uint2* rrect;                // rank -> tile rect
    GroupGeom gg;
    int row_chunks;              // level-1 chunks (bin_row_chunks)
    uint32_t* hist1;             // [rows * row_chunks] level-1 counts, scanned in place
    uint32_t* hist2;             // [bin_hist2_elems] level-2 counts, scanned in place
    uint32_t* meta;              // [bin_meta_elems] row starts / segment layout
    uint32_t* bsum;              // scan block sums (+1)
    uint32_t* rowidx;            // [capacity] group-row entries: splat index
    uint32_t* rowxp;             // [capacity]                    column range gx0 | gx1 << 16
    uint32_t* offsets;           // [n_groups_band + 1]
    uint32_t* list;              // [capacity] output entries (splat indices)
    uint32_t* segmap;            // [bin_segmap_elems] level-2 segment -> group row (cols_count -> cols_place)
    uint32_t* slicecum;          // [bin_slicecum_elems] per segment and column: entries of slices 0..w
                                 // (w < kBinWarps - 1) — each placement warp's start in the column run
    FrameCounters* fc;
    uint32_t capacity;
};
// level-1 chunks for a frame whose previous frame of the same geometry had `row_entries` group-row
// entries (0: unknown): enough that a block's share fits its output stage
int bin_row_chunks(const GroupGeom& gg, uint64_t row_entries);
size_t bin_hist1_elems(const GroupGeom& gg, int row_chunks);
size_t bin_hist2_elems(const GroupGeom& gg, uint32_t capacity);
size_t bin_segmap_elems(const GroupGeom& gg, uint32_t capacity);
size_t bin_slicecum_elems(const GroupGeom& gg, uint32_t capacity);
size_t bin_meta_elems(const GroupGeom& gg);
void launch_binning(const BinArgs& a, int max_visible, cudaStream_t st);
// In-place exclusive scan of n u32 (one pass, decoupled look-back); tmp holds scan_tmp_elems(n)
// u32; returns the device address of the total.
size_t scan_tmp_elems(size_t n);
// n_dev (optional): device-side length <= n; elements past it are left untouched.
const uint32_t* launch_exclusive_scan(uint32_t* x, size_t n, uint32_t* tmp, cudaStream_t st,
                                      const uint32_t* n_dev = nullptr);

// Sorted lists -> GroupEntry array (for readback).
void launch_lists_readback(const uint32_t* sorted_idx, const uint32_t* offsets, int n_groups,
                           DevProjected proj, GroupGeom gg, tgs_group_entry* out, cudaStream_t st);

// ---- rasterisers ---------------------------------------------------------------------------
struct RasterArgs {
    DevProjected proj;
    const uint32_t* list;     // sorted compacted indices
    const uint32_t* offsets;  // [n_groups + 1]
    const int* order;         // group processing order (longest lists first) or null
    GroupGeom gg;
    float* image;             // H x W x 3 (band rows only when banded)
    int image_row0;           // first image row stored in `image`
    float alpha_skip, alpha_clamp, t_terminate;
    FrameCounters* fc;
    uint32_t* tile_trip;      // optional (count_pairs): per tile, entries of its list walked until done
    uint32_t* unit_cost;      // optional: per unit, list entries walked (next frame's schedule)
    int tile_cull;            // drop splats whose alpha_skip ellipse box misses the tile (tight_cover)
};
void launch_raster_scalar(const RasterArgs& a, cudaStream_t st);
// LPT schedule for the rasterisers: work units (tile / group / quarter group, per_group units per
// group list) bucketed by floor(log2(list length)), longest first.
// With `feedback` (per unit, entries walked by the previous frame of the same geometry) the cost
// is the measured walk, else the list length.
// Also folds the frame's overflow / validation flags into fc's sticky counters.
void launch_unit_order(const uint32_t* offsets, const uint32_t* feedback, int n_units, int per_group, int* order,
                       FrameCounters* fc, cudaStream_t st);
void launch_raster_tensor(const RasterArgs& a, int num_sms, cudaStream_t st);
// Exact emulation of the reference's per-pixel arithmetic (fp32 or fp16 lanes), any G.
void launch_raster_exact(const RasterArgs& a, bool fp16, cudaStream_t st);
// raster work units per group list of the tensor path (schedule / feedback indexing)
int raster_units_per_group(int g);
// Instrumented walk: counts walked / alpha-contributing pairs (reference semantics, G=1 lists).
void launch_count_pairs(const RasterArgs& a, cudaStream_t st);
// mask-popcount histogram (17 bins, index = popcount) of the frame's group entries
void launch_reuse_hist(const FrameCounters* fc, const uint2* rect, const GroupGeom& gg, int max_input,
                       unsigned long long* hist, cudaStream_t st);
void launch_encode_u8(const float* rgb, int64_t n, uint8_t* out, cudaStream_t st);

// ---- stage API on caller-provided data (tgs_stage.cu) -------------------------------------
void launch_entries_count(const tgs_projected* proj, int64_t n, const GroupGeom& gg, uint32_t* counts,
                          cudaStream_t st);
void launch_entries_emit(const tgs_projected* proj, int64_t n, const GroupGeom& gg, const uint32_t* start,
                         tgs_keyed_entry* out, cudaStream_t st);
void launch_keyed_split(const tgs_keyed_entry* e, uint32_t n, uint32_t n_groups, uint32_t* keys, uint32_t* gid,
                        uint32_t* flags, uint32_t* count, cudaStream_t st);
void launch_gather_u32(const uint32_t* src, const uint32_t* perm, uint32_t n, uint32_t* dst, cudaStream_t st);
void launch_gather_entries(const tgs_keyed_entry* e, const uint32_t* perm, uint32_t n, tgs_group_entry* out,
                           uint32_t* gid_sorted, cudaStream_t st);
void launch_offsets_from_sorted(const uint32_t* gid, uint32_t n, uint32_t n_groups, uint32_t* offsets,
                                cudaStream_t st);
void launch_projected_to_planes(const tgs_projected* p, int64_t n, float alpha_skip, DevProjected out,
                                cudaStream_t st);
// entries per group row of the frame whose splat rects are in `rect` (n = &fc->n_input)
void launch_row_entries(const uint2* rect, const uint32_t* n, const GroupGeom& gg, unsigned long long* rows,
                        cudaStream_t st);
void launch_lists_check(const tgs_group_entry* e, const uint32_t* offsets, int n_groups, const tgs_projected* proj,
                        int64_t n_proj, const GroupGeom& gg, uint32_t* list, uint32_t* flags, cudaStream_t st);

}  // namespace tgs
