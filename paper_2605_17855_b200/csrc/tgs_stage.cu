// Kernels behind the reference's public STAGE API on caller-provided data (include/tgs.h:
// tgs_build_group_entries, tgs_sort_entries, tgs_rasterize_lists).  The render path never uses
// these: it fuses the stages (tgs_binning.cu) and keeps splats and lists in its own layout.
//
//   build_group_entries (proj/src/binning.cpp:46-74): per projected splat, one KeyedEntry per
//     overlapped group, gy outer / gx inner, in splat order — count -> exclusive scan -> emit;
//   sort_entries (binning.cpp:76-100): depth validation, then std::stable_sort on
//     (group_id << 32) | f32_bits(depth) as two stable LSD radix sorts (depth bits, then group
//     id) with the hand-written one-sweep sort of tgs_sort.cu, a gather and per-group offsets;
//   rasterize_* on caller lists: the projected records are converted to the rasterisers' SoA
//     planes, and every entry's mask is checked against the one build_group_entries derives from
//     the splat's tile rectangle (the rasterisers recompute masks instead of storing them).
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

namespace tgs {

namespace {

// Tile rectangle of a caller-provided projected record (tiles_overlapped, binning.cpp:32-44).
__device__ __forceinline__ bool rect_of(const tgs_projected& p, const GroupGeom& gg, int& x0, int& y0, int& x1,
                                        int& y1) {
    tile_rect(p.mean2d[0], p.mean2d[1], p.radius, gg.tiles_x, gg.tiles_y, x0, y0, x1, y1);
    return x1 >= x0 && y1 >= y0;
}

__global__ void entries_count_kernel(const tgs_projected* __restrict__ proj, int64_t n, GroupGeom gg,
                                     uint32_t* __restrict__ counts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int x0, y0, x1, y1;
        uint32_t c = 0;
        if (rect_of(proj[i], gg, x0, y0, x1, y1))
            c = (uint32_t)((x1 / gg.g - x0 / gg.g + 1) * (y1 / gg.g - y0 / gg.g + 1));
        counts[i] = c;
    }
}

__global__ void entries_emit_kernel(const tgs_projected* __restrict__ proj, int64_t n, GroupGeom gg,
                                    const uint32_t* __restrict__ start, tgs_keyed_entry* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int x0, y0, x1, y1;
        if (!rect_of(proj[i], gg, x0, y0, x1, y1)) continue;
        uint32_t o = start[i];
        const float depth = proj[i].depth;
        for (int gy = y0 / gg.g; gy <= y1 / gg.g; ++gy)
            for (int gx = x0 / gg.g; gx <= x1 / gg.g; ++gx) {
                tgs_keyed_entry e;
                e.group_id = (uint32_t)(gy * gg.groups_x + gx);
                e.entry.gaussian_index = (uint32_t)i;
                e.entry.depth = depth;
                e.entry.mask = group_mask(gx, gy, gg.g, x0, y0, x1, y1);
                out[o++] = e;
            }
    }
}

// keys = depth bits, gids kept aside; flags: bit 0 bad depth (binning.cpp:78-83), bit 1 group id
// out of range.  count[0] = n for the radix sort's device-side item count.
__global__ void keyed_split_kernel(const tgs_keyed_entry* __restrict__ e, uint32_t n, uint32_t n_groups,
                                   uint32_t* __restrict__ keys, uint32_t* __restrict__ gid,
                                   uint32_t* __restrict__ flags, uint32_t* __restrict__ count) {
    if (blockIdx.x == 0 && threadIdx.x == 0) count[0] = n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float d = e[i].entry.depth;
        if (!isfinite(d) || d < 0.0f) atomicOr(flags, 1u);
        if (e[i].group_id >= n_groups) atomicOr(flags, 2u);
        keys[i] = __float_as_uint(d);
        gid[i] = e[i].group_id;
    }
}

__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm, uint32_t n,
                                  uint32_t* __restrict__ dst) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[perm[i]];
}

__global__ void gather_entries_kernel(const tgs_keyed_entry* __restrict__ e, const uint32_t* __restrict__ perm,
                                      uint32_t n, tgs_group_entry* __restrict__ out, uint32_t* __restrict__ gid_sorted) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const tgs_keyed_entry k = e[perm[i]];
        out[i] = k.entry;
        gid_sorted[i] = k.group_id;
    }
}

// offsets[g] = first position of group >= g in the sorted group ids (offsets[n_groups] = n)
__global__ void offsets_from_sorted_kernel(const uint32_t* __restrict__ gid, uint32_t n, uint32_t n_groups,
                                           uint32_t* __restrict__ offsets) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        const uint32_t lo = i == 0 ? 0u : gid[i - 1] + 1u;
        const uint32_t hi = i == n ? n_groups : gid[i];
        for (uint32_t g = lo; g <= hi; ++g) offsets[g] = i;
    }
}

// Caller-provided ProjectedGaussian records -> the rasterisers' SoA planes (mc, co, col; col.w =
// the tile-cull extents, as preprocess_kernel stores them).
__global__ void projected_to_planes_kernel(const tgs_projected* __restrict__ p, int64_t n, float alpha_skip,
                                           DevProjected out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const tgs_projected r = p[i];
        const float ext = tight_extents(r.conic[0], r.conic[1], r.conic[2], r.opacity, alpha_skip);
        out.mc[i] = make_float4(r.mean2d[0], r.mean2d[1], r.conic[0], r.conic[1]);
        out.co[i] = make_float4(r.conic[2], r.opacity, r.depth, __int_as_float(r.radius));
        out.col[i] = make_float4(r.color[0], r.color[1], r.color[2], ext);
    }
}

// Caller lists -> splat-index lists; flags: bit 0 index out of range, bit 1 mask differs from
// the one build_group_entries gives the splat in that group, bit 2 offsets not monotone.
__global__ void lists_check_kernel(const tgs_group_entry* __restrict__ e, const uint32_t* __restrict__ offsets,
                                   int n_groups, const tgs_projected* __restrict__ proj, int64_t n_proj, GroupGeom gg,
                                   uint32_t* __restrict__ list, uint32_t* __restrict__ flags) {
    for (int g = blockIdx.x; g < n_groups; g += gridDim.x) {
        const uint32_t b = offsets[g], en = offsets[g + 1];
        if (en < b) {
            if (threadIdx.x == 0) atomicOr(flags, 4u);
            continue;
        }
        const int gx = g % gg.groups_x, gy = g / gg.groups_x;
        for (uint32_t k = b + threadIdx.x; k < en; k += blockDim.x) {
            const tgs_group_entry x = e[k];
            list[k] = x.gaussian_index;
            if ((int64_t)x.gaussian_index >= n_proj) {
                atomicOr(flags, 1u);
                continue;
            }
            int x0, y0, x1, y1;
            const bool any = rect_of(proj[x.gaussian_index], gg, x0, y0, x1, y1);
            const uint32_t m = any ? group_mask(gx, gy, gg.g, x0, y0, x1, y1) : 0u;
            if (m != x.mask || m == 0u) atomicOr(flags, 2u);
        }
    }
}

// Entries per group row of a frame (screen-band work estimate): a splat with tile
// rect [x0..x1] x [y0..y1] adds (x1/G - x0/G + 1) entries to every group row y0/G .. y1/G — the
// row totals of build_group_entries (binning.cpp:46-74) without building a list.
__global__ void __launch_bounds__(256) row_entries_kernel(const uint2* __restrict__ rect, const uint32_t* __restrict__ n,
                                                          GroupGeom gg, unsigned long long* __restrict__ rows) {
    extern __shared__ unsigned int srow[];  // one counter per group row
    for (int k = threadIdx.x; k < gg.groups_y; k += blockDim.x) srow[k] = 0;
    __syncthreads();
    const uint32_t cnt = *n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const uint2 r = rect[i];
        if (r.x == kCulledRect && r.y == kCulledRect) continue;
        const int x0 = (int)(r.x & 0xffffu), x1 = (int)(r.x >> 16), y0 = (int)(r.y & 0xffffu), y1 = (int)(r.y >> 16);
        if (x1 < x0 || y1 < y0) continue;
        const unsigned int span = (unsigned int)(x1 / gg.g - x0 / gg.g + 1);
        for (int gy = y0 / gg.g; gy <= y1 / gg.g; ++gy) atomicAdd(&srow[gy], span);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < gg.groups_y; k += blockDim.x)
        if (srow[k]) atomicAdd(&rows[k], (unsigned long long)srow[k]);
}

constexpr int kBlocks = 148 * 4;

}  // namespace

void launch_row_entries(const uint2* rect, const uint32_t* n, const GroupGeom& gg, unsigned long long* rows,
                        cudaStream_t st) {
    cudaMemsetAsync(rows, 0, (size_t)gg.groups_y * sizeof(unsigned long long), st);
    row_entries_kernel<<<kBlocks, 256, (size_t)gg.groups_y * sizeof(unsigned int), st>>>(rect, n, gg, rows);
}

void launch_entries_count(const tgs_projected* proj, int64_t n, const GroupGeom& gg, uint32_t* counts,
                          cudaStream_t st) {
    if (n > 0) entries_count_kernel<<<kBlocks, 256, 0, st>>>(proj, n, gg, counts);
}
void launch_entries_emit(const tgs_projected* proj, int64_t n, const GroupGeom& gg, const uint32_t* start,
                         tgs_keyed_entry* out, cudaStream_t st) {
    if (n > 0) entries_emit_kernel<<<kBlocks, 256, 0, st>>>(proj, n, gg, start, out);
}
void launch_keyed_split(const tgs_keyed_entry* e, uint32_t n, uint32_t n_groups, uint32_t* keys, uint32_t* gid,
                        uint32_t* flags, uint32_t* count, cudaStream_t st) {
    keyed_split_kernel<<<kBlocks, 256, 0, st>>>(e, n, n_groups, keys, gid, flags, count);
}
void launch_gather_u32(const uint32_t* src, const uint32_t* perm, uint32_t n, uint32_t* dst, cudaStream_t st) {
    if (n > 0) gather_u32_kernel<<<kBlocks, 256, 0, st>>>(src, perm, n, dst);
}
void launch_gather_entries(const tgs_keyed_entry* e, const uint32_t* perm, uint32_t n, tgs_group_entry* out,
                           uint32_t* gid_sorted, cudaStream_t st) {
    if (n > 0) gather_entries_kernel<<<kBlocks, 256, 0, st>>>(e, perm, n, out, gid_sorted);
}
void launch_offsets_from_sorted(const uint32_t* gid, uint32_t n, uint32_t n_groups, uint32_t* offsets,
                                cudaStream_t st) {
    offsets_from_sorted_kernel<<<kBlocks, 256, 0, st>>>(gid, n, n_groups, offsets);
}
void launch_projected_to_planes(const tgs_projected* p, int64_t n, float alpha_skip, DevProjected out,
                                cudaStream_t st) {
    if (n > 0) projected_to_planes_kernel<<<kBlocks, 256, 0, st>>>(p, n, alpha_skip, out);
}
void launch_lists_check(const tgs_group_entry* e, const uint32_t* offsets, int n_groups, const tgs_projected* proj,
                        int64_t n_proj, const GroupGeom& gg, uint32_t* list, uint32_t* flags, cudaStream_t st) {
    if (n_groups > 0) lists_check_kernel<<<kBlocks, 256, 0, st>>>(e, offsets, n_groups, proj, n_proj, gg, list, flags);
}

}  // namespace tgs
