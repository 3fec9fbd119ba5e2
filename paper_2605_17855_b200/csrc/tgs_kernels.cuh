// Kernel argument structs and launchers shared between the .cu files of libtgs.
#pragma once

#include "tgs_common.cuh"

namespace tgs {

struct PreprocessArgs {
    DevScene scene;
    DevCamera cam;
    DevProjected out;
    uint32_t* depth_keys;          // [visible] depth bits (presort keys)
    uint32_t* idx_vals;            // [visible] compacted index (presort values)
    uint32_t* ngroups;             // [visible] group entries emitted per splat
    GroupGeom gg;
    unsigned long long* tile_status;  // decoupled look-back status words (zeroed per frame)
    FrameCounters* fc;
};
void launch_preprocess(const PreprocessArgs& a, cudaStream_t st);

// ---- radix sort (LSD, stable, u32 keys + u32 values, device-side item count) --------------
struct SortBuffers {
    uint32_t* keys[2];
    uint32_t* vals[2];
    uint32_t* ghist;      // [256 * kSortBlocks]
    uint32_t* gid_count;  // [n_groups] (gid sort only)
};
constexpr int kSortBlocks = 592;  // 4 x 148 SMs
// Sorts count (device) items of keys[0]/vals[0] by bits [0, nbits); result in keys[r]/vals[r]
// where r is returned (ping-pong parity).  If gid_count != null the first pass also builds the
// per-key histogram (keys < n_groups).  keys_out_last == false skips writing keys in the last
// pass (only values are needed downstream).
int radix_sort(SortBuffers& b, const uint32_t* count, int nbits, int n_groups, bool want_keys_last,
               cudaStream_t st);

// ---- binning -------------------------------------------------------------------------------
struct BinArgs {
    const uint32_t* visible;     // &fc->visible
    const uint32_t* sval;        // presorted compacted indices (rank order)
    const uint32_t* ngroups;     // per compacted index
    uint32_t* eoff;              // [visible] exclusive entry offsets (rank order)
    unsigned long long* tile_status;
    FrameCounters* fc;
    uint32_t capacity;           // entry buffer capacity
    DevProjected proj;
    GroupGeom gg;
    uint32_t* keys;              // out: gid
    uint32_t* vals;              // out: compacted idx
};
void launch_entry_scan(const BinArgs& a, int max_items, cudaStream_t st);
void launch_emit(const BinArgs& a, int max_items, cudaStream_t st);
// offsets[0..n] = exclusive scan of counts[0..n-1]; offsets[n] = total.
void launch_offsets_scan(const uint32_t* counts, uint32_t* offsets, int n, cudaStream_t st);

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
};
void launch_raster_scalar(const RasterArgs& a, cudaStream_t st);
// LPT schedule for the rasterisers: work units (tile / group / quarter group, per_group units per
// group list) bucketed by floor(log2(list length)), longest first.
void launch_unit_order(const uint32_t* offsets, int n_units, int per_group, int* order, cudaStream_t st);
void launch_raster_tensor(const RasterArgs& a, int num_sms, cudaStream_t st);
// Instrumented walk: counts walked / alpha-contributing pairs (reference semantics, G=1 lists).
void launch_count_pairs(const RasterArgs& a, cudaStream_t st);
void launch_encode_u8(const float* rgb, int64_t n, uint8_t* out, cudaStream_t st);

}  // namespace tgs
