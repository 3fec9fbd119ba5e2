// Tile/group binning (north_star 2): per-splat entry counts -> exclusive scan in depth order ->
// warp-cooperative emission of (group id, index) entries -> (tgs_sort.cu) stable group sort ->
// per-group ranges.  Reference: proj/src/binning.cpp:32-100, render.cpp:17-21.
//
// Entries carry only the splat index; the member-tile mask (binning.cpp:56-65) is a pure
// function of the splat's tile rect and the group, so consumers recompute it instead of moving
// it through the sort (4 bytes per entry per pass saved).
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

namespace tgs {

namespace {

constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

__device__ __forceinline__ uint32_t lookback(unsigned long long* status, int tile, uint32_t agg) {
    constexpr unsigned long long kAgg = 1ull << 62, kPre = 2ull << 62;
    if (tile == 0) {
        atomicExch(&status[0], kPre | agg);
        return 0;
    }
    atomicExch(&status[tile], kAgg | agg);
    uint32_t excl = 0;
    int t = tile - 1;
    while (true) {
        unsigned long long s;
        do {
            s = atomicAdd(&status[t], 0ull);
        } while ((s >> 62) == 0);
        excl += (uint32_t)(s & 0xffffffffu);
        if ((s >> 62) == 2) break;
        --t;
    }
    atomicExch(&status[tile], kPre | (unsigned long long)(excl + agg));
    return excl;
}

// eoff[r] = sum_{r' < r} ngroups[sval[r']] over the depth-sorted ranks; total -> fc->n_entries.
__global__ void __launch_bounds__(kScanBlock) entry_scan_kernel(BinArgs a) {
    __shared__ uint32_t s_tile, s_base;
    __shared__ uint32_t s_warp[kScanBlock / 32];
    if (threadIdx.x == 0) s_tile = atomicAdd(&a.fc->scan_tile_counter, 1u);
    __syncthreads();
    const int tile = (int)s_tile;
    const uint32_t n = *a.visible;
    const uint32_t ntiles = (n + kScanTile - 1) / kScanTile;
    if ((uint32_t)tile >= ntiles) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = (uint32_t)tile * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems], sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t r = base + k;
        v[k] = r < n ? a.ngroups[a.sval[r]] : 0u;
        sum += v[k];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int w = 0; w < kScanBlock / 32; ++w) {
            const uint32_t c = s_warp[w];
            s_warp[w] = run;
            run += c;
        }
        s_base = lookback(a.tile_status, tile, run);
        if ((uint32_t)tile == ntiles - 1) {
            const uint32_t total = s_base + run;
            a.fc->n_entries = total;
            if (total > a.capacity)
                a.fc->overflow = 1u;
            else
                a.fc->n_sort = total;
        }
    }
    __syncthreads();
    uint32_t run = s_base + s_warp[warp] + incl - sum;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint32_t r = base + k;
        if (r < n) a.eoff[r] = run;
        run += v[k];
    }
}

// Warp-cooperative load-balanced expansion: a warp takes 32 consecutive ranks, scans their entry
// counts, then emits the warp's entries 32 at a time (each lane finds its owning splat by a
// 5-step shuffle search), so writes are fully coalesced regardless of per-splat fan-out.
__global__ void __launch_bounds__(256) emit_kernel(BinArgs a) {
    const uint32_t n = *a.visible;
    if (a.fc->overflow) return;
    const int lane = threadIdx.x & 31;
    const uint32_t warps_total = gridDim.x * (blockDim.x / 32);
    for (uint32_t w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); w * 32 < n; w += warps_total) {
        const uint32_t r = w * 32 + lane;
        int cnt = 0, gx0 = 0, gy0 = 0, gw = 1;
        uint32_t idx = 0, base = 0;
        if (r < n) {
            idx = a.sval[r];
            base = a.eoff[r];
            const float4 mc = a.proj.mc[idx];
            const float4 co = a.proj.co[idx];
            int tx0, ty0, tx1, ty1, gx1, gy1;
            cnt = group_rect(mc.x, mc.y, __float_as_int(co.w), a.gg, tx0, ty0, tx1, ty1, gx0, gy0, gx1, gy1);
            gw = gx1 - gx0 + 1;
        }
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int excl = incl - cnt;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int e0 = 0; e0 < total; e0 += 32) {
            const int e = e0 + lane;
            int pos = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int t = __shfl_sync(0xffffffffu, excl, (pos + step) & 31);
                if (pos + step < 32 && t <= e) pos += step;
            }
            const int o_excl = __shfl_sync(0xffffffffu, excl, pos);
            const int o_gx0 = __shfl_sync(0xffffffffu, gx0, pos);
            const int o_gy0 = __shfl_sync(0xffffffffu, gy0, pos);
            const int o_gw = __shfl_sync(0xffffffffu, gw, pos);
            const uint32_t o_idx = __shfl_sync(0xffffffffu, idx, pos);
            const uint32_t o_base = __shfl_sync(0xffffffffu, base, pos);
            if (e < total) {
                const int k = e - o_excl;
                const int gy = o_gy0 + k / o_gw;
                const int gx = o_gx0 + k % o_gw;
                const uint32_t slot = o_base + (uint32_t)k;
                a.keys[slot] = (uint32_t)((gy - a.gg.band_gy0) * a.gg.groups_x + gx);
                a.vals[slot] = o_idx;
            }
        }
    }
}

__global__ void lists_readback_kernel(const uint32_t* __restrict__ sorted_idx,
                                      const uint32_t* __restrict__ offsets, int n_groups,
                                      DevProjected proj, GroupGeom gg, tgs_group_entry* out) {
    const int gid = blockIdx.x;
    if (gid >= n_groups) return;
    const int gx = gid % gg.groups_x, gy = gid / gg.groups_x + gg.band_gy0;
    for (uint32_t e = offsets[gid] + threadIdx.x; e < offsets[gid + 1]; e += blockDim.x) {
        const uint32_t idx = sorted_idx[e];
        const float4 mc = proj.mc[idx];
        const float4 co = proj.co[idx];
        int tx0, ty0, tx1, ty1;
        tile_rect(mc.x, mc.y, __float_as_int(co.w), gg.tiles_x, gg.tiles_y, tx0, ty0, tx1, ty1);
        tgs_group_entry ge;
        ge.gaussian_index = idx;
        ge.depth = co.z;
        ge.mask = group_mask(gx, gy, gg.g, tx0, ty0, tx1, ty1);
        out[e] = ge;
    }
}

__global__ void encode_u8_kernel(const float* __restrict__ rgb, int64_t n, uint8_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = rgb[i];
        v = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
        out[i] = (uint8_t)__float2int_rn(__fmul_rn(v, 255.0f));  // lrintf: round half to even
    }
}

// Longest-processing-time-first schedule (bucketed): the rasterisers take work units (G=1:
// tiles; G=2: groups; G=4: quarter groups) in this order, so units with the longest lists start
// first and the tail of the persistent grid is short.  Work estimate = the unit's list length.
__global__ void __launch_bounds__(1024) unit_order_kernel(const uint32_t* __restrict__ offsets, int n_units,
                                                          int per_group, int* __restrict__ order) {
    __shared__ uint32_t cnt[33];
    if (threadIdx.x < 33) cnt[threadIdx.x] = 0;
    __syncthreads();
    auto key = [&](int u) {
        const int gid = u / per_group;
        return __clz(offsets[gid + 1] - offsets[gid] + 1u);  // 0 = longest bucket
    };
    for (int t = threadIdx.x; t < n_units; t += blockDim.x) atomicAdd(&cnt[key(t)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int k = 0; k < 33; ++k) {
            const uint32_t c = cnt[k];
            cnt[k] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_units; t += blockDim.x) order[atomicAdd(&cnt[key(t)], 1u)] = t;
}

}  // namespace

void launch_unit_order(const uint32_t* offsets, int n_units, int per_group, int* order, cudaStream_t st) {
    if (n_units > 0) unit_order_kernel<<<1, 1024, 0, st>>>(offsets, n_units, per_group, order);
}

void launch_entry_scan(const BinArgs& a, int max_items, cudaStream_t st) {
    const int blocks = (max_items + kScanTile - 1) / kScanTile;
    if (blocks > 0) entry_scan_kernel<<<blocks, kScanBlock, 0, st>>>(a);
}

void launch_emit(const BinArgs& a, int max_items, cudaStream_t st) {
    int blocks = (max_items + 255) / 256;
    blocks = blocks < 1 ? 1 : (blocks > 148 * 16 ? 148 * 16 : blocks);
    emit_kernel<<<blocks, 256, 0, st>>>(a);
}

void launch_lists_readback(const uint32_t* sorted_idx, const uint32_t* offsets, int n_groups,
                           DevProjected proj, GroupGeom gg, tgs_group_entry* out, cudaStream_t st) {
    if (n_groups > 0) lists_readback_kernel<<<n_groups, 256, 0, st>>>(sorted_idx, offsets, n_groups, proj, gg, out);
}

void launch_encode_u8(const float* rgb, int64_t n, uint8_t* out, cudaStream_t st) {
    encode_u8_kernel<<<148 * 8, 256, 0, st>>>(rgb, n, out);
}

}  // namespace tgs
