// Tile/group binning + sort (north_star 2): a stable counting sort of (group, rank) entries.
// Reference: proj/src/binning.cpp:32-100 (tiles_overlapped, build_group_entries, sort_entries),
// render.cpp:17-21.
//
// The reference emits one 16-byte entry per (splat, overlapped group) and std::stable_sorts them
// on (group_id << 32) | f32_bits(depth) (ties: emission order = splat index).  Here the splats are
// first radix-sorted by depth bits (tgs_sort.cu, values = compacted index, so ties keep index
// order) — their "rank" order.  Every group's list is then the rank-ordered subsequence of splats
// overlapping it, which a counting sort produces directly, writing each 4-byte entry once:
//   gather  : rank-ordered tile rectangles (8 B per splat);
//   count   : every warp owns a contiguous rank range (a "chunk") and builds its per-group entry
//             counts with a 2D difference array in shared memory (4 atomics per splat, then row and
//             column prefix sums) -> hist[group][chunk];
//   scan    : exclusive scan of hist in group-major order -> the start of every (group, chunk) run;
//   scatter : each warp replays its splats in rank order and writes entry slots from per-warp
//             shared-memory cursors (a splat has at most one entry per group, so the lanes writing
//             one splat's entries never collide).
// Entries carry only the splat index; the member-tile mask (binning.cpp:56-65) is a pure function of
// the splat's tile rectangle and the group, so consumers recompute it.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

#include <algorithm>

namespace tgs {

namespace {

constexpr int kMaxBinWarps = 8;       // warps per count/scatter block (fewer for huge grids)
constexpr int kScanItems = 16;        // per thread in the hist scan
constexpr int kScanBlock = 256;
constexpr int kScanTile = kScanItems * kScanBlock;

__device__ __forceinline__ bool decode_rect(uint2 r, int& x0, int& x1, int& y0, int& y1) {
    x0 = (int)(r.x & 0xffffu);
    x1 = (int)(r.x >> 16);
    y0 = (int)(r.y & 0xffffu);
    y1 = (int)(r.y >> 16);
    return x1 >= x0 && y1 >= y0;
}

// Band-local group rectangle of a tile rectangle; false if no group of the band is overlapped.
__device__ __forceinline__ bool band_groups(const GroupGeom& gg, uint2 r, int& gx0, int& gx1, int& gy0, int& gy1) {
    int x0, x1, y0, y1;
    if (!decode_rect(r, x0, x1, y0, y1)) return false;
    const int sh = gg.g >> 1;  // G in {1, 2, 4}: tile -> group is a shift by 0, 1, 2
    gx0 = x0 >> sh;
    gx1 = x1 >> sh;
    gy0 = max(y0 >> sh, gg.band_gy0) - gg.band_gy0;
    gy1 = min(y1 >> sh, gg.band_gy1 - 1) - gg.band_gy0;
    return gy1 >= gy0;
}

__device__ __forceinline__ void chunk_range(uint32_t n, int n_chunks, int w, uint32_t& r0, uint32_t& r1) {
    const uint32_t per = (n + (uint32_t)n_chunks - 1u) / (uint32_t)n_chunks;
    r0 = min(n, per * (uint32_t)w);
    r1 = min(n, r0 + per);
}

__global__ void __launch_bounds__(256) rank_gather_kernel(BinArgs a) {
    const uint32_t n = *a.visible;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        a.rrect[r] = __ldg(&a.rect[__ldg(&a.sval[r])]);
}

// Per-warp group counts of the rank range [r0, r1): 2D difference array in shared memory (4
// atomics per splat), then prefix sums along x and y.  Afterwards D[gy * pitch + gx] = entries of
// the range in band-local group (gx, gy).
__device__ __forceinline__ void warp_group_counts(const BinArgs& a, int* D, uint32_t r0, uint32_t r1, int lane) {
    const GroupGeom& gg = a.gg;
    const int gx = gg.groups_x, gyb = gg.band_gy1 - gg.band_gy0;
    const int pitch = gx + 1, area = (gyb + 1) * pitch;
    for (int i = lane; i < area; i += 32) D[i] = 0;
    __syncwarp();
    for (uint32_t r = r0 + lane; r < r1; r += 32) {
        int gx0, gx1, gy0, gy1;
        if (!band_groups(gg, __ldg(&a.rrect[r]), gx0, gx1, gy0, gy1)) continue;
        atomicAdd(&D[gy0 * pitch + gx0], 1);
        atomicAdd(&D[gy0 * pitch + gx1 + 1], -1);
        atomicAdd(&D[(gy1 + 1) * pitch + gx0], -1);
        atomicAdd(&D[(gy1 + 1) * pitch + gx1 + 1], 1);
    }
    __syncwarp();
    for (int y = lane; y < gyb; y += 32) {  // prefix along x (one row per lane)
        int run = 0;
        for (int x = 0; x < gx; ++x) {
            run += D[y * pitch + x];
            D[y * pitch + x] = run;
        }
    }
    __syncwarp();
    for (int x = lane; x < gx; x += 32) {  // prefix along y (one column per lane)
        int run = 0;
        for (int y = 0; y < gyb; ++y) {
            run += D[y * pitch + x];
            D[y * pitch + x] = run;
        }
    }
    __syncwarp();
}

// Chunk = one block: the block's rank range, split evenly over its warps.
__device__ __forceinline__ void block_warp_range(const BinArgs& a, int wib, int wpb, uint32_t& r0, uint32_t& r1) {
    uint32_t b0, b1;
    chunk_range(*a.visible, a.n_chunks, blockIdx.x, b0, b1);
    uint32_t w0, w1;
    chunk_range(b1 - b0, wpb, wib, w0, w1);
    r0 = b0 + w0;
    r1 = b0 + w1;
}

// hist[g * n_chunks + chunk] = entries the chunk (one block) contributes to group g.
__global__ void __launch_bounds__(kMaxBinWarps * 32) group_count_kernel(BinArgs a) {
    extern __shared__ int sdiff[];
    const GroupGeom& gg = a.gg;
    const int gx = gg.groups_x, gyb = gg.band_gy1 - gg.band_gy0;
    const int pitch = gx + 1, area = (gyb + 1) * pitch, ng = gx * gyb;
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    uint32_t r0, r1;
    block_warp_range(a, wib, wpb, r0, r1);
    warp_group_counts(a, sdiff + wib * area, r0, r1, lane);
    __syncthreads();
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
        const int y = g / gx, di = y * pitch + (g - y * gx);
        uint32_t t = 0;
        for (int w = 0; w < wpb; ++w) t += (uint32_t)sdiff[w * area + di];
        a.hist[(size_t)g * a.n_chunks + blockIdx.x] = t;
    }
}

// ---- exclusive scan of hist (block sums -> single-block scan of the sums -> apply) ----------
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t& total) {
    __shared__ uint32_t wsum[kScanBlock / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t s = lane < kScanBlock / 32 ? wsum[lane] : 0u;
        uint32_t si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += t;
        }
        if (lane < kScanBlock / 32) wsum[lane] = si - s;
        total = __shfl_sync(0xffffffffu, si, kScanBlock / 32 - 1);
    }
    __syncthreads();
    const uint32_t excl = wsum[warp] + incl - v;
    __shared__ uint32_t stotal;
    if (threadIdx.x == 0) stotal = total;
    __syncthreads();
    total = stotal;
    return excl;
}

__global__ void __launch_bounds__(kScanBlock) scan_reduce_kernel(const uint32_t* __restrict__ x, size_t n,
                                                                 uint32_t* __restrict__ bsum) {
    const size_t base = (size_t)blockIdx.x * kScanTile + (size_t)threadIdx.x * kScanItems;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const size_t i = base + k;
        if (i < n) s += x[i];
    }
    uint32_t total = 0;
    block_exclusive_scan(s, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

// in-place exclusive scan of n values by one block (n = blocks + 1, the last slot is the total)
__global__ void __launch_bounds__(1024) scan_small_kernel(uint32_t* data, int n) {
    __shared__ uint32_t warp_tot[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base < n; base += 1024 * 4) {
        uint32_t v[4], s = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = base + threadIdx.x * 4 + k;
            v[k] = i < n ? data[i] : 0u;
            s += v[k];
        }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = warp_tot[lane];
            uint32_t wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += t;
            }
            warp_tot[lane] = wi - w;
        }
        __syncthreads();
        uint32_t run = carry + warp_tot[warp] + incl - s;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = base + threadIdx.x * 4 + k;
            if (i < n) data[i] = run;
            run += v[k];
        }
        __syncthreads();
        if (threadIdx.x == 1023) carry = run;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kScanBlock) scan_apply_kernel(uint32_t* __restrict__ x, size_t n,
                                                                const uint32_t* __restrict__ bsum) {
    const size_t base = (size_t)blockIdx.x * kScanTile + (size_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems], s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const size_t i = base + k;
        v[k] = i < n ? x[i] : 0u;
        s += v[k];
    }
    uint32_t total = 0;
    uint32_t run = block_exclusive_scan(s, total) + bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const size_t i = base + k;
        if (i < n) x[i] = run;
        run += v[k];
    }
}

// offsets[g] = start of group g's list; offsets[ng] = total; capacity check -> fc flags.
__global__ void offsets_kernel(BinArgs a, int n_scan_blocks) {
    const int ng = a.gg.n_groups_band;
    const uint32_t total = a.bsum[n_scan_blocks];
    const bool over = total > a.capacity;  // lists do not fit: every list empty, host grows + re-renders
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g <= ng; g += gridDim.x * blockDim.x)
        a.offsets[g] = over ? 0u : (g < ng ? a.hist[(size_t)g * a.n_chunks] : total);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.fc->n_entries = total;
        if (total > a.capacity)
            a.fc->overflow = 1u;
        else
            a.fc->n_sort = total;
    }
}

// The block's chunk, sorted locally: per-warp group counts -> per-(warp, group) start inside the
// chunk -> entries placed in shared memory in (group, rank) order -> flushed so that every
// (group, chunk) run lands as one contiguous burst.  Chunks too large for the shared buffer write
// each entry straight to its global slot instead (same slots, scattered writes).
//
// Placement expands the warp's splats 32 entries per step (rank-major, entries of a splat in
// row-major group order, like build_group_entries binning.cpp:50-72); entries of one step that
// hit the same group come from different splats and are ranked by lane (= rank order) with
// match_any, the highest such lane advancing the group's cursor.
__global__ void __launch_bounds__(kMaxBinWarps * 32) group_scatter_kernel(BinArgs a, int buf_cap) {
    extern __shared__ int smem[];
    const GroupGeom& gg = a.gg;
    const int gx = gg.groups_x, gyb = gg.band_gy1 - gg.band_gy0;
    const int pitch = gx + 1, area = (gyb + 1) * pitch, ng = gx * gyb;
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    int* D = smem;                                                 // wpb x area: counts, then cursors
    uint32_t* T = reinterpret_cast<uint32_t*>(smem + wpb * area);  // [ng + 1] local run starts
    uint32_t* G0 = T + ng + 1;                                     // [ng] global run starts
    uint32_t* buf = G0 + ng;                                       // [buf_cap] sorted entries
    uint16_t* gbuf = reinterpret_cast<uint16_t*>(buf + buf_cap);   // [buf_cap] their groups
    __shared__ uint32_t s_total;
    if (a.fc->overflow) return;
    uint32_t r0, r1;
    block_warp_range(a, wib, wpb, r0, r1);
    int* Dw = D + wib * area;
    warp_group_counts(a, Dw, r0, r1, lane);
    __syncthreads();
    // per-(warp, group) exclusive prefix over the warps; T = block totals; G0 = global run starts
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
        const int y = g / gx, di = y * pitch + (g - y * gx);
        uint32_t run = 0;
        for (int w = 0; w < wpb; ++w) {
            const uint32_t c = (uint32_t)D[w * area + di];
            D[w * area + di] = (int)run;
            run += c;
        }
        T[g] = run;
        G0[g] = a.hist[(size_t)g * a.n_chunks + blockIdx.x];
    }
    __syncthreads();
    // exclusive scan of T over the groups (one warp; ng is a few thousand at most)
    if (wib == 0) {
        uint32_t carry = 0;
        for (int base = 0; base < ng; base += 32) {
            const int g = base + lane;
            const uint32_t v = g < ng ? T[g] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (g < ng) T[g] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            T[ng] = carry;
            s_total = carry;
        }
    }
    __syncthreads();
    const bool local = s_total <= (uint32_t)buf_cap;
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t rb = r0; rb < r1; rb += 32) {  // this warp's splats in rank order, 32 at a time
        const uint32_t r = rb + lane;
        int gx0 = 0, gy0 = 0, gw = 1, cnt = 0;
        uint32_t idx = 0;
        if (r < r1) {
            int gx1, gy1;
            if (band_groups(gg, __ldg(&a.rrect[r]), gx0, gx1, gy0, gy1)) {
                gw = gx1 - gx0 + 1;
                cnt = gw * (gy1 - gy0 + 1);
            }
            idx = __ldg(&a.sval[r]);
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
            // owning splat of entry e: the last lane whose exclusive offset is <= e
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
            const bool valid = e < total;
            const int k = e - o_excl;
            const int dy = __float2int_rz(((float)k + 0.5f) * __frcp_rn((float)o_gw)), dx = k - dy * o_gw;
            const int yy = o_gy0 + dy, xx = o_gx0 + dx;
            const int g = valid ? yy * gx + xx : -1 - lane;  // invalid lanes match nobody
            const uint32_t peers = __match_any_sync(0xffffffffu, g);
            if (valid) {
                const int di = yy * pitch + xx;
                const uint32_t before = (uint32_t)Dw[di];
                const uint32_t kk = before + (uint32_t)__popc(peers & lt);
                if ((31 - __clz(peers)) == lane) Dw[di] = (int)(before + (uint32_t)__popc(peers));
                if (local) {
                    const uint32_t p = T[g] + kk;
                    buf[p] = o_idx;
                    gbuf[p] = (uint16_t)g;
                } else {
                    a.list[G0[g] + kk] = o_idx;
                }
            }
            __syncwarp();  // cursor updates visible to the next step
        }
    }
    if (!local) return;
    __syncthreads();
    // flush: entry i of the sorted buffer belongs to group gbuf[i]; runs land contiguously
    const uint32_t tot = s_total;
    for (uint32_t i = threadIdx.x; i < tot; i += blockDim.x) {
        const uint32_t g = gbuf[i];
        a.list[G0[g] + (i - T[g])] = buf[i];
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
// Longest-processing-time-first order of the rasteriser's work units.  A unit's cost is how much
// of its list it walks before its pixels terminate, which the list length alone predicts poorly
// (deep central lists terminate after a few hundred splats, silhouette lists are walked to the
// end); with `feedback` the cost is the walk measured on the previous frame of the same geometry
// (temporal coherence of a camera path), else the list length.  Counting sort on a log2 key with
// 8 buckets per octave; equal keys keep unit order.
__global__ void __launch_bounds__(1024) unit_order_kernel(const uint32_t* __restrict__ offsets,
                                                          const uint32_t* __restrict__ feedback, int n_units,
                                                          int per_group, int* __restrict__ order) {
    constexpr int kBuckets = 264;
    __shared__ uint32_t cnt[kBuckets];
    for (int k = threadIdx.x; k < kBuckets; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    auto key = [&](int u) {
        const int gid = u / per_group;
        const uint32_t cost = feedback ? feedback[u] : offsets[gid + 1] - offsets[gid];
        const int b = (int)(log2f((float)cost + 1.0f) * 8.0f);
        return kBuckets - 1 - min(kBuckets - 1, b);  // 0 = most expensive
    };
    for (int t = threadIdx.x; t < n_units; t += blockDim.x) atomicAdd(&cnt[key(t)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int k = 0; k < kBuckets; ++k) {
            const uint32_t c = cnt[k];
            cnt[k] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_units; t += blockDim.x) order[atomicAdd(&cnt[key(t)], 1u)] = t;
}

}  // namespace

void launch_unit_order(const uint32_t* offsets, const uint32_t* feedback, int n_units, int per_group, int* order,
                       cudaStream_t st) {
    if (n_units > 0) unit_order_kernel<<<1, 1024, 0, st>>>(offsets, feedback, n_units, per_group, order);
}

// Warps per count/scatter block: one difference array ((rows+1) x (cols+1) ints) per warp in
// shared memory, plus (scatter) three per-group arrays and the local entry buffer.
static int bin_warps_per_block(const GroupGeom& gg) {
    const size_t per_warp = (size_t)(gg.band_gy1 - gg.band_gy0 + 1) * (gg.groups_x + 1) * 4;
    int w = kMaxBinWarps;
    while (w > 1 && per_warp * w > 96u * 1024u) w >>= 1;
    return w;
}

int bin_chunks(int n_groups) {
    // chunks (= blocks) so that a chunk's entries usually fit the scatter's shared buffer, with
    // the [group][chunk] matrix kept within ~16M entries
    long c = 148L * 24;
    while (c > 148 && (long)n_groups * c > (16L << 20)) c /= 2;
    return (int)c;
}
size_t bin_hist_elems(int n_groups) { return (size_t)std::max(1, n_groups) * bin_chunks(n_groups); }
size_t bin_bsum_elems(int n_groups) { return (bin_hist_elems(n_groups) + kScanTile - 1) / kScanTile + 1; }

size_t scan_tmp_elems(size_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

void launch_exclusive_scan(uint32_t* x, size_t n, uint32_t* tmp, cudaStream_t st) {
    const int blocks = (int)((n + kScanTile - 1) / kScanTile);
    if (blocks == 0) return;
    scan_reduce_kernel<<<blocks, kScanBlock, 0, st>>>(x, n, tmp);
    cudaMemsetAsync(tmp + blocks, 0, sizeof(uint32_t), st);
    scan_small_kernel<<<1, 1024, 0, st>>>(tmp, blocks + 1);
    scan_apply_kernel<<<blocks, kScanBlock, 0, st>>>(x, n, tmp);
}

void launch_binning(const BinArgs& a, int max_visible, cudaStream_t st) {
    const GroupGeom& gg = a.gg;
    const int wpb = bin_warps_per_block(gg);
    const int ng = gg.n_groups_band;
    const size_t diff_smem = (size_t)wpb * (gg.band_gy1 - gg.band_gy0 + 1) * (gg.groups_x + 1) * sizeof(int);
    const size_t arrays = (size_t)(3 * ng + 1) * sizeof(uint32_t);
    const size_t max_smem = 220u * 1024u;
    // local buffer: u32 entry + u16 group per slot
    const int buf_cap = (int)std::max<long>(0, ((long)max_smem - (long)(diff_smem + arrays)) / 6) & ~1;
    const size_t scatter_smem = diff_smem + arrays + (size_t)buf_cap * 6;
    const size_t n = (size_t)ng * a.n_chunks;
    const int scan_blocks = (int)((n + kScanTile - 1) / kScanTile);
    const int gblocks = std::max(1, std::min(148 * 8, (max_visible + 255) / 256));
    rank_gather_kernel<<<gblocks, 256, 0, st>>>(a);
    cudaFuncSetAttribute(group_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)diff_smem);
    group_count_kernel<<<a.n_chunks, wpb * 32, diff_smem, st>>>(a);
    launch_exclusive_scan(a.hist, n, a.bsum, st);
    offsets_kernel<<<(ng + 256) / 256, 256, 0, st>>>(a, scan_blocks);
    cudaFuncSetAttribute(group_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scatter_smem);
    group_scatter_kernel<<<a.n_chunks, wpb * 32, scatter_smem, st>>>(a, buf_cap);
}

void launch_lists_readback(const uint32_t* sorted_idx, const uint32_t* offsets, int n_groups,
                           DevProjected proj, GroupGeom gg, tgs_group_entry* out, cudaStream_t st) {
    if (n_groups > 0) lists_readback_kernel<<<n_groups, 256, 0, st>>>(sorted_idx, offsets, n_groups, proj, gg, out);
}

void launch_encode_u8(const float* rgb, int64_t n, uint8_t* out, cudaStream_t st) {
    encode_u8_kernel<<<148 * 8, 256, 0, st>>>(rgb, n, out);
}

}  // namespace tgs
