// Tile/group binning + sort (north_star 2): a stable partition of (group, rank) entries.
// Reference: proj/src/binning.cpp:32-100 (tiles_overlapped, build_group_entries, sort_entries),
// render.cpp:17-21.
//
// The reference emits one 16-byte entry per (splat, overlapped group) and std::stable_sorts them
// on (group_id << 32) | f32_bits(depth) (ties: emission order = splat index).  Here the splats are
// first radix-sorted by depth bits (tgs_sort.cu, values = splat index, so ties keep index order) —
// their "rank" order.  Every group's list is then the rank-ordered subsequence of splats
// overlapping it, built by two stable partitions that write each entry once (the level-1 count
// also gathers the rank-ordered tile rectangles, 8 B per splat, for the placement pass):
//   level 1: splats -> group-row lists.  Each warp owns a contiguous rank range (chunk); per-row
//            counts (1D difference array) -> scan over (row, chunk) -> the chunk's splats are
//            appended to their rows in rank order (row entries: splat index, column range, in two
//            4-byte planes);
//   level 2: group-row lists -> group lists.  Each warp owns a segment of one row list; per-column
//            counts -> scan over (row, column, segment) = group-major -> the segment's entries are
//            appended to their columns in order.
// Placement is lane per item, 32 items at a time: an item's slot in row / column c is c's running
// position plus the number of earlier lanes (earlier items) that also cover c, read from a per-warp
// bitmask of c — so order is stable by construction, with no global atomics, and every
// (row, chunk) / (group, segment) run is a contiguous burst.  Entries carry only the splat index; the member-tile mask
// (binning.cpp:56-65) is a pure function of the splat's tile rectangle and the group, so
// consumers recompute it.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

#include <cstdio>

#include <algorithm>

namespace tgs {

namespace {

constexpr int kBinWarps = 8;          // warps per binning block (one chunk / segment per warp)
// level-1 chunks (contiguous rank ranges, one warp each): 148 x 128 (measured best at C3, where a
// block's row entries just fit its stage), doubled while a block's expected share (previous frame)
// exceeds its stage — large frames (C4: 6M splats at 4K) would otherwise write unstaged
constexpr int kRowChunksMin = 148 * 128, kRowChunksMax = 148 * 128 * 16;
// level-1 per-block output staging (row entries), smaller for few rows (more resident blocks)
#ifndef TGS_STAGE1
#define TGS_STAGE1 6144
#endif
#ifndef TGS_STAGE1_WIDE
#define TGS_STAGE1_WIDE 8192
#endif
constexpr int stage1_entries(int kr) { return kr <= 2 ? TGS_STAGE1 : TGS_STAGE1_WIDE; }
// Level 2 cuts every group-row list into segments of kBinWarps slices (one placement block, one
// count warp); a slice is the row entries one warp places.  A segment's output (~entries x the mean
// column span) is staged in shared memory: a 12K-entry stage, 256-entry slices for up to 64 group
// columns (bench G=2), 128 beyond (G=1 at 1080p and C4: 120 columns) — measured per config.
__host__ __device__ constexpr uint32_t slice_len(int kc) { return kc <= 2 ? 256u : 128u; }
__host__ __device__ constexpr uint32_t seg_len_kc(int kc) { return slice_len(kc) * kBinWarps; }
__host__ __device__ inline uint32_t seg_len_gx(int gx) { return seg_len_kc((gx + 31) / 32); }
constexpr int stage2_entries(int) { return 12288; }
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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// ---- level 1: splats -> group-row lists -----------------------------------------------------
// A "chunk" is one warp's contiguous rank range.  Row entries are (splat index, gx0 | gx1 << 16)
// and row y's list is the concatenation over chunks of the chunk's splats overlapping row y.

// hist1[y * row_chunks + chunk] = splats of the chunk overlapping group row y; fc->n_entries +=
// the chunk's (splat, group) entries (the capacity check needs the total before any placement).
__global__ void __launch_bounds__(kBinWarps * 32) rows_count_kernel(BinArgs a) {
    const uint32_t* __restrict__ sval = *a.sval_sel ? a.sval[1] : a.sval[0];
    extern __shared__ int sdiff[];
    const int rows = a.gg.band_gy1 - a.gg.band_gy0;
    const int lane = threadIdx.x & 31, chunk = blockIdx.x * kBinWarps + (threadIdx.x >> 5);
    int* D = sdiff + (threadIdx.x >> 5) * (rows + 1);
    for (int i = lane; i <= rows; i += 32) D[i] = 0;
    __syncwarp();
    uint32_t r0, r1;
    chunk_range(*a.visible, a.row_chunks, chunk, r0, r1);
    uint32_t ent = 0;
    for (uint32_t rb = r0 + lane; rb < r1; rb += 32 * 8) {  // 8 gathers in flight per lane
        uint2 rr[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t r = rb + 32u * u;
            // gather the rank-ordered rectangle once here (rows_place reads it back coalesced)
            rr[u] = r < r1 ? __ldg(&a.rect[__ldg(&sval[r])]) : make_uint2(0xffffu, 0u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t r = rb + 32u * u;
            if (r >= r1) continue;
            a.rrect[r] = rr[u];
            int gx0, gx1, gy0, gy1;
            if (!band_groups(a.gg, rr[u], gx0, gx1, gy0, gy1)) continue;
            atomicAdd(&D[gy0], 1);
            atomicAdd(&D[gy1 + 1], -1);
            ent += (uint32_t)((gx1 - gx0 + 1) * (gy1 - gy0 + 1));
        }
    }
    __syncwarp();
    int carry = 0;
    for (int base = 0; base < rows; base += 32) {
        const int y = base + lane;
        int incl = y < rows ? D[y] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (y < rows) a.hist1[(size_t)y * a.row_chunks + chunk] = (uint32_t)(carry + incl);
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ent += __shfl_xor_sync(0xffffffffu, ent, o);
    // one global atomic per block (same-address atomics serialise in L2)
    __shared__ uint32_t s_ent;
    if (threadIdx.x == 0) s_ent = 0u;
    __syncthreads();
    if (lane == 0 && ent) atomicAdd(&s_ent, ent);
    __syncthreads();
    if (threadIdx.x == 0 && s_ent) atomicAdd(&a.fc->n_entries, s_ent);
}

// One warp: capacity check, row starts, per-row segment counts and the level-2 histogram layout.
//   meta[0 .. rows]            row list starts (meta[rows] = row entries)
//   meta[M1 .. M1 + rows]      prefix of segments per row (M1 = rows + 1; last = segments)
//   meta[M2 .. M2 + rows]      prefix of gx * segments per row: hist2 block of row y (M2 = 2 rows + 2)
__global__ void rows_meta_kernel(BinArgs a, const uint32_t* __restrict__ scan1_total) {
    const int rows = a.gg.band_gy1 - a.gg.band_gy0, gx = a.gg.groups_x, lane = threadIdx.x;
    uint32_t* rowstart = a.meta;
    uint32_t* nsegp = a.meta + rows + 1;
    uint32_t* rowbase2 = a.meta + 2 * rows + 2;
    const uint32_t total = a.fc->n_entries;
    const bool over = total > a.capacity;  // lists do not fit: nothing is placed, host grows + re-renders
    if (lane == 0) {
        if (over)
            a.fc->overflow = 1u;
        else
            a.fc->n_sort = total;
        a.fc->row_entries = *scan1_total;
    }
    uint32_t cs = 0;
    for (int base = 0; base <= rows; base += 32) {
        const int y = base + lane;
        uint32_t start = 0, nseg = 0;
        if (y < rows) {
            start = a.hist1[(size_t)y * a.row_chunks];
            const uint32_t next = y + 1 < rows ? a.hist1[(size_t)(y + 1) * a.row_chunks] : *scan1_total;
            nseg = over ? 0u : (next - start + seg_len_gx(gx) - 1u) / seg_len_gx(gx);
        } else if (y == rows) {
            start = *scan1_total;
        }
        uint32_t inc_s = nseg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc_s, o);
            if (lane >= o) inc_s += t;
        }
        if (y <= rows) {
            rowstart[y] = start;
            nsegp[y] = cs + inc_s - nseg;
            rowbase2[y] = (cs + inc_s - nseg) * (uint32_t)gx;
        }
        cs += __shfl_sync(0xffffffffu, inc_s, 31);
    }
}

// Predicated shared-memory reduction / stores (branch-free per-row / per-column loops).
__device__ __forceinline__ void red_or_if(uint32_t addr, uint32_t v, bool on) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.shared.or.b32 [%0], %1;\n\t}" ::"r"(addr),
                 "r"(v), "r"((uint32_t)on)
                 : "memory");
}
__device__ __forceinline__ void st_shared_if(uint32_t addr, uint32_t v, bool on) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t}" ::"r"(addr),
                 "r"(v), "r"((uint32_t)on)
                 : "memory");
}
__device__ __forceinline__ void st_shared_v2_if(uint32_t addr, uint32_t x, uint32_t y, bool on) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t@p st.shared.v2.u32 [%0], {%1, %2};\n\t}" ::"r"(addr),
                 "r"(x), "r"(y), "r"((uint32_t)on)
                 : "memory");
}
__device__ __forceinline__ uint2 ld_shared_v2(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
    return v;
}

// Row placement.  A block takes kBinWarps consecutive chunks (one per warp); in the [row][chunk]
// layout the block's runs of row y are consecutive, i.e. one contiguous global range inside which
// warp w's part starts after the parts of warps < w.  Lane per splat: the warp walks its chunk 32
// splats at a time; each lane marks the group rows of its splat in a per-warp row bitmask, and the
// splat's slot in row y is the row's running position plus the number of earlier lanes (= earlier
// ranks) that also cover y; after each batch every row advances by its mask's population.  Slots
// are in the block's shared output buffer, every row run is then flushed with coalesced stores.  A
// block whose output exceeds the buffer writes to global slots directly.
template <int KR>
__global__ void __launch_bounds__(kBinWarps * 32) rows_place_kernel(BinArgs a) {
    constexpr int kStage1 = stage1_entries(KR);
    // [kStage1] output (uint2) | [kBinWarps][rows + 1] row positions | [kBinWarps][rows + 1] row masks
    extern __shared__ uint2 sout1[];
    if (a.fc->overflow) return;
    const uint32_t* __restrict__ sval = *a.sval_sel ? a.sval[1] : a.sval[0];
    const int rows = a.gg.band_gy1 - a.gg.band_gy0;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int c0 = blockIdx.x * kBinWarps, chunk = c0 + wib;
    const uint32_t lanebit = 1u << lane, lt = lanebit - 1u;
    const uint32_t total = a.meta[rows];  // row entries
    // per-warp row records (running position, mask of this batch's lanes)
    uint2* rm = sout1 + kStage1 + wib * (rows + 1);
    const uint32_t out0 = smem_u32(sout1), rm0 = smem_u32(rm);
    auto h1at = [&](int y, int c) {       // scanned hist1 at (row y, chunk c); c may be row_chunks
        const size_t i = (size_t)y * a.row_chunks + c;
        return i < (size_t)rows * a.row_chunks ? a.hist1[i] : total;
    };
    uint32_t r0, r1;
    chunk_range(*a.visible, a.row_chunks, chunk, r0, r1);
    uint32_t snext = 0u;  // the chunk's first batch is in flight during the row setup
    uint2 rnext = make_uint2(0u, 0u);
    if (r0 + lane < r1) {
        snext = __ldg(&sval[r0 + lane]);
        rnext = __ldg(&a.rrect[r0 + lane]);
    }
    uint32_t base[KR], len[KR], P[KR], carry = 0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
        const int y = lane + 32 * k;
        base[k] = y < rows ? h1at(y, c0) : 0u;
        len[k] = y < rows ? h1at(y, c0 + kBinWarps) - base[k] : 0u;
        uint32_t incl = len[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        P[k] = carry + incl - len[k];
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    const bool staged = carry <= (uint32_t)kStage1;  // block-uniform
#pragma unroll
    for (int k = 0; k < KR; ++k) {
        const int y = lane + 32 * k;
        if (y < rows) {
            const uint32_t pos = h1at(y, chunk);  // this chunk's first slot of row y
            rm[y] = make_uint2(staged ? P[k] + (pos - base[k]) : pos, 0u);
        }
    }
    __syncwarp();
    for (uint32_t rb = r0; rb < r1; rb += 32) {
        const uint32_t r = rb + lane;
        const uint32_t sv = snext;  // next batch in flight while this one is placed
        const uint2 rr = rnext;
        if (r + 32 < r1) {
            snext = __ldg(&sval[r + 32]);
            rnext = __ldg(&a.rrect[r + 32]);
        }
        // band rows [y0, y0 + span) of this lane's splat (span 0: none; reads row 0) and its
        // column range
        uint32_t y0 = 0u, y1 = 0u, xp = 0u;
        int span = 0;
        if (r < r1) {
            int gx0, gx1, gy0, gy1;
            if (band_groups(a.gg, rr, gx0, gx1, gy0, gy1)) {
                y0 = (uint32_t)gy0;
                y1 = (uint32_t)gy1;
                span = gy1 - gy0 + 1;
                xp = (uint32_t)gx0 | ((uint32_t)gx1 << 16);
            }
        }
        const int ms = (int)__reduce_max_sync(0xffffffffu, (uint32_t)span);
        // record address of step t, clamped to the last row (inactive steps store nothing)
        const uint32_t ra = rm0 + 8u * y0, rz = rm0 + 8u * y1;
        for (int t = 0; t < ms; ++t) red_or_if(min(ra + 8u * (uint32_t)t, rz) + 4u, lanebit, t < span);
        __syncwarp();
        if (staged) {
            for (int t = 0; t < ms; ++t) {
                const uint2 q = ld_shared_v2(min(ra + 8u * (uint32_t)t, rz));
                st_shared_v2_if(out0 + 8u * (q.x + __popc(q.y & lt)), sv, xp, t < span);
            }
        } else {
            for (int t = 0; t < span; ++t) {
                const uint2 q = rm[y0 + t];
                const uint32_t p = q.x + __popc(q.y & lt);
                a.rowidx[p] = sv;
                a.rowxp[p] = xp;
            }
        }
        __syncwarp();
        // advance every row by its entries in this batch (lane-owned rows, race-free)
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int y = lane + 32 * k;
            if (y < rows) {
                const uint2 q = rm[y];
                rm[y] = make_uint2(q.x + __popc(q.y), 0u);
            }
        }
        __syncwarp();
    }
    if (staged) {
        __syncthreads();
        // flush: warp w copies the block runs of rows w, w + 8, ... (coalesced)
#pragma unroll
        for (int k = 0; k < KR; ++k)
            for (int l = wib; l < 32; l += kBinWarps) {
                const uint32_t c = __shfl_sync(0xffffffffu, len[k], l);
                const uint32_t src = __shfl_sync(0xffffffffu, P[k], l);
                const uint32_t dst = __shfl_sync(0xffffffffu, base[k], l);
                for (uint32_t i = lane; i < c; i += 32) {
                    const uint2 e = sout1[src + i];
                    a.rowidx[dst + i] = e.x;
                    a.rowxp[dst + i] = e.y;
                }
            }
    }
}

// ---- level 2: group-row lists -> group lists ----------------------------------------------------
// Row y's list is cut into segments of seg_len_gx entries (one count warp each).  hist2 holds, per row, a
// [column][segment] block, so the exclusive scan of hist2 (rows in order) is directly the global
// start of every (group, segment) run and group g = (y, x) starts at its segment-0 slot.

// Row y and segment s of global segment q (warp-collective): y = last row with nsegp[y] <= q, found
// with independent loads + ballots instead of a dependent binary search (nsegp is non-decreasing,
// nsegp[0] = 0).
__device__ __forceinline__ void seg_locate(const uint32_t* nsegp, int rows, uint32_t q, int& y, uint32_t& s) {
    const int lane = threadIdx.x & 31;
    int cnt = 0;
#pragma unroll 4
    for (int b = 0; b < rows; b += 32) {
        const int i = b + lane;
        cnt += __popc(__ballot_sync(0xffffffffu, i < rows && __ldg(&nsegp[i]) <= q));
    }
    y = cnt - 1;
    s = q - __ldg(&nsegp[y]);
}

__global__ void __launch_bounds__(kBinWarps * 32) cols_count_kernel(BinArgs a) {
    extern __shared__ int sdiff[];
    if (a.fc->overflow) return;
    const int rows = a.gg.band_gy1 - a.gg.band_gy0, gx = a.gg.groups_x;
    const int lane = threadIdx.x & 31;
    const uint32_t* rowstart = a.meta;
    const uint32_t* nsegp = a.meta + rows + 1;
    const uint32_t* rowbase2 = a.meta + 2 * rows + 2;
    const uint32_t nq = nsegp[rows];
    int* D = sdiff + (threadIdx.x >> 5) * (gx + 1);
    for (uint32_t q = blockIdx.x * kBinWarps + (threadIdx.x >> 5); q < nq; q += gridDim.x * kBinWarps) {
        int y;
        uint32_t s;
        seg_locate(nsegp, rows, q, y, s);
        if (lane == 0) a.segmap[q] = (uint32_t)y;  // cols_place reads the row back (one load)
        const uint32_t nseg = nsegp[y + 1] - nsegp[y];
        const uint32_t seg = seg_len_gx(gx);
        const uint32_t e0 = rowstart[y] + s * seg, e1 = min(rowstart[y + 1], e0 + seg);
        for (int i = lane; i <= gx; i += 32) D[i] = 0;
        __syncwarp();
        // slice by slice (the placement warps' shares): after slice w < kBinWarps - 1 the running
        // per-column counts are the start of warp w + 1's part of every column run
        const uint32_t sl = slice_len((gx + 31) / 32);
        for (int w = 0; w < kBinWarps; ++w) {
            const uint32_t s0 = min(e1, e0 + (uint32_t)w * sl), s1 = min(e1, s0 + sl);
            for (uint32_t eb = s0 + lane; eb < s1; eb += 32 * 8) {  // 8 loads in flight per lane
                uint32_t xp[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) xp[u] = eb + 32u * u < s1 ? __ldg(&a.rowxp[eb + 32u * u]) : 0xffffffffu;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (xp[u] != 0xffffffffu) {
                        atomicAdd(&D[xp[u] & 0xffffu], 1);
                        atomicAdd(&D[(xp[u] >> 16) + 1], -1);
                    }
            }
            __syncwarp();
            if (w + 1 < kBinWarps) {
                uint32_t* cum = a.slicecum + ((size_t)q * (kBinWarps - 1) + (size_t)w) * (size_t)gx;
                int run = 0;
                for (int base = 0; base < gx; base += 32) {
                    const int x = base + lane;
                    int incl = x < gx ? D[x] : 0;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += t;
                    }
                    if (x < gx) cum[x] = (uint32_t)(run + incl);
                    run += __shfl_sync(0xffffffffu, incl, 31);
                }
            }
        }
        __syncwarp();
        int carry = 0;
        for (int base = 0; base < gx; base += 32) {
            const int x = base + lane;
            int incl = x < gx ? D[x] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            if (x < gx) a.hist2[rowbase2[y] + (uint32_t)x * nseg + s] = (uint32_t)(carry + incl);
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
    }
}

// offsets[g] = global start of group g = its segment-0 slot of the scanned hist2 (an empty row has
// a zero-size block: the slot holds the running total, which is its groups' start); offsets[ng] =
// total.  Overflow: every list empty.
__global__ void offsets_kernel(BinArgs a) {
    const int rows = a.gg.band_gy1 - a.gg.band_gy0, gx = a.gg.groups_x, ng = a.gg.n_groups_band;
    const uint32_t* nsegp = a.meta + rows + 1;
    const uint32_t* rowbase2 = a.meta + 2 * rows + 2;
    const bool over = a.fc->overflow != 0u;
    const uint32_t total = a.fc->n_entries;
    const size_t hist2_len = rowbase2[rows];
    for (int g = blockIdx.x * blockDim.x + threadIdx.x; g <= ng; g += gridDim.x * blockDim.x) {
        uint32_t v = 0;
        if (!over) {
            if (g == ng) {
                v = total;
            } else {
                const int y = g / gx, x = g - y * gx;
                const size_t i = (size_t)rowbase2[y] + (size_t)x * (nsegp[y + 1] - nsegp[y]);
                v = i < hist2_len ? a.hist2[i] : total;
            }
        }
        a.offsets[g] = v;
    }
}

// Group placement.  A block takes one segment (kBinWarps slices of slice_len row entries, one per
// warp); the segment's run of column x is one contiguous global range [base_x, base_x + len_x),
// inside which warp w's part starts after the parts of warps < w (per-slice column counts, made
// here in shared memory).  Lane per entry: each lane marks the columns of its entry in a per-warp
// column bitmask; the entry's slot in column c is the column's running position plus the number of
// earlier lanes (= earlier entries) that also cover c; after each 32-entry chunk every column
// advances by its mask's population.  The per-column loops are branch-free (predicated shared
// reductions / stores), slots are in the block's shared output buffer in column-major order, and
// every column run is flushed as one coalesced burst; a block whose output exceeds the buffer
// writes global slots.
template <int KC>
__global__ void __launch_bounds__(kBinWarps * 32, KC <= 4 ? 5 : 1) cols_place_kernel(BinArgs a) {
    constexpr uint32_t kSliceLen = slice_len(KC), kSegLen = seg_len_kc(KC);
    constexpr int kPer = kSliceLen / 32;  // row entries per lane
    constexpr int kStage2 = stage2_entries(KC);
    // [kStage2] output | [kBinWarps][gx + 1] column records (running position, mask of this
    // batch's lanes) — one 8-byte load serves the slot formula
    extern __shared__ uint32_t sout[];
    if (a.fc->overflow) return;
    const int rows = a.gg.band_gy1 - a.gg.band_gy0, gx = a.gg.groups_x;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t lanebit = 1u << lane, lt = lanebit - 1u;
    const uint32_t* rowstart = a.meta;
    const uint32_t* nsegp = a.meta + rows + 1;
    const uint32_t* rowbase2 = a.meta + 2 * rows + 2;
    const uint32_t nq = nsegp[rows], h2 = rowbase2[rows], total = a.fc->n_entries;
    uint2* cm = reinterpret_cast<uint2*>(sout + kStage2) + wib * (gx + 1);
    const uint32_t out0 = smem_u32(sout), cm0 = smem_u32(cm);
    auto h2at = [&](uint32_t i) { return i < h2 ? a.hist2[i] : total; };
    // the segment's group row comes from cols_count's map, loaded one segment ahead
    uint32_t ynext = blockIdx.x < nq ? __ldg(&a.segmap[blockIdx.x]) : 0u;
    for (uint32_t q = blockIdx.x; q < nq; q += gridDim.x) {
        const int y = (int)ynext;
        if (q + gridDim.x < nq) ynext = __ldg(&a.segmap[q + gridDim.x]);
        const uint32_t s = q - nsegp[y];
        const uint32_t nseg = nsegp[y + 1] - nsegp[y];
        const uint32_t se0 = rowstart[y] + s * kSegLen, se1 = min(rowstart[y + 1], se0 + kSegLen);
        const uint32_t e0 = min(se1, se0 + (uint32_t)wib * kSliceLen), e1 = min(se1, e0 + kSliceLen);
        // column runs of the segment, [base, base + len) globally (loads in flight during the counts)
        uint32_t base[KC], len[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const int x = lane + 32 * k;
            const uint32_t i0 = rowbase2[y] + (uint32_t)x * nseg + s;
            base[k] = x < gx ? h2at(i0) : 0u;
            len[k] = x < gx ? h2at(i0 + 1) : 0u;
        }
        // this warp's slice, loaded once; its start in every column run is cols_count's running
        // count after the earlier slices (no per-block counting, no barrier)
        uint2 ent[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const uint32_t e = e0 + lane + 32u * i;
            ent[i] = e < e1 ? make_uint2(__ldg(&a.rowidx[e]), __ldg(&a.rowxp[e])) : make_uint2(0u, 0u);
        }
        const uint32_t* cum = a.slicecum + ((size_t)q * (kBinWarps - 1) + (size_t)(wib - 1)) * (size_t)gx;
        // local start P of every column run; this warp's part starts off after earlier warps'
        uint32_t P[KC], off[KC], carry = 0;
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const int x = lane + 32 * k;
            len[k] -= base[k];
            off[k] = (wib > 0 && x < gx) ? __ldg(&cum[x]) : 0u;
            uint32_t incl = len[k];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            P[k] = carry + incl - len[k];
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        const bool staged = carry <= (uint32_t)kStage2;  // block-uniform
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            const int x = lane + 32 * k;
            if (x < gx) cm[x] = make_uint2(staged ? P[k] + off[k] : base[k] + off[k], 0u);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            if (e0 + 32u * i >= e1) break;  // warp-uniform
            const uint2 v = ent[i];
            // columns [x0, x0 + span); a lane without an entry has span 0 (and reads column 0)
            const bool valid = e0 + lane + 32u * i < e1;
            const uint32_t x0 = valid ? (v.y & 0xffffu) : 0u, x1 = valid ? (v.y >> 16) : 0u;
            const int span = valid ? (int)(x1 - x0) + 1 : 0;
            const int ms = (int)__reduce_max_sync(0xffffffffu, (uint32_t)span);
            // record address of step t, clamped to the last column (inactive steps store nothing)
            const uint32_t ra = cm0 + 8u * x0, rz = cm0 + 8u * x1;
#pragma unroll 2
            for (int t = 0; t < ms; ++t) red_or_if(min(ra + 8u * (uint32_t)t, rz) + 4u, lanebit, t < span);
            __syncwarp();
            if (staged) {
#pragma unroll 2
                for (int t = 0; t < ms; ++t) {
                    const uint2 r = ld_shared_v2(min(ra + 8u * (uint32_t)t, rz));
                    st_shared_if(out0 + 4u * (r.x + __popc(r.y & lt)), v.x, t < span);
                }
            } else {
                for (int t = 0; t < span; ++t) {
                    const uint2 r = cm[x0 + t];
                    a.list[r.x + __popc(r.y & lt)] = v.x;
                }
            }
            __syncwarp();
            // advance every column by its entries in this chunk (lane-owned columns, race-free)
#pragma unroll
            for (int k = 0; k < KC; ++k) {
                const int x = lane + 32 * k;
                if (x < gx) {
                    const uint2 r = cm[x];
                    cm[x] = make_uint2(r.x + __popc(r.y), 0u);
                }
            }
            __syncwarp();
        }
        __syncthreads();
        if (staged) {
            // flush: warp w copies the runs of columns w, w + 8, ... (one coalesced burst each)
#pragma unroll
            for (int k = 0; k < KC; ++k)
                for (int l = wib; l < 32; l += kBinWarps) {
                    const uint32_t c = __shfl_sync(0xffffffffu, len[k], l);
                    const uint32_t src = __shfl_sync(0xffffffffu, P[k], l);
                    const uint32_t dst = __shfl_sync(0xffffffffu, base[k], l);
                    uint32_t* __restrict__ d = a.list + dst;
                    const uint32_t* sp = sout + src;
                    uint32_t j = lane;
                    for (; j + 32u < c; j += 64u) {  // two independent copies per step
                        const uint32_t v0 = sp[j], v1 = sp[j + 32u];
                        d[j] = v0;
                        d[j + 32u] = v1;
                    }
                    if (j < c) d[j] = sp[j];
                }
            __syncthreads();
        } else {
            __syncthreads();  // the next segment rewrites the slice counts other warps read above
        }
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

// Single-pass exclusive scan (in place): tiles of kScanTile values are claimed in order from a
// ticket; each tile publishes its aggregate, resolves its prefix by decoupled look-back over the
// 32 preceding tiles per round (warp 0, one status word per lane), publishes its inclusive prefix
// and writes its values.  tmp: [0] ticket, [2] total, status words (u64: flag << 32 | value) from
// tmp + 4; zeroed by the launcher.  n_dev (device length, may be null) caps n.
__global__ void __launch_bounds__(kScanBlock) scan_onepass_kernel(uint32_t* __restrict__ x, size_t n,
                                                                  const uint32_t* __restrict__ n_dev,
                                                                  uint32_t* __restrict__ tmp) {
    if (n_dev) n = min(n, (size_t)*n_dev);
    const uint32_t tiles = (uint32_t)((n + kScanTile - 1) / kScanTile);
    unsigned long long* status = reinterpret_cast<unsigned long long*>(tmp + 4);
    constexpr unsigned long long kAgg = 1ull << 32, kPre = 2ull << 32;
    __shared__ uint32_t s_tile, s_prefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(&tmp[0], 1u);
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= tiles) break;  // block-uniform
        const size_t base = (size_t)tile * kScanTile + (size_t)threadIdx.x * kScanItems;
        uint32_t v[kScanItems], sum = 0;
        const bool full = base + kScanItems <= n;  // 16-byte vector loads/stores (x is 16-aligned)
        if (full) {
#pragma unroll
            for (int k = 0; k < kScanItems; k += 4) {
                const uint4 q = *reinterpret_cast<const uint4*>(x + base + k);
                v[k] = q.x;
                v[k + 1] = q.y;
                v[k + 2] = q.z;
                v[k + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kScanItems; ++k) v[k] = base + k < n ? x[base + k] : 0u;
        }
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) sum += v[k];
        uint32_t total = 0;
        const uint32_t excl = block_exclusive_scan(sum, total);
        if (warp == 0) {
            uint32_t prefix = 0;
            if (tile == 0) {
                if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&status[0]) = kPre | total;
            } else {
                if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&status[tile]) = kAgg | total;
                int j = (int)tile - 1;
                const long long t0 = clock64();
                for (;;) {
                    const int idx = j - lane;
                    const unsigned long long w =
                        idx >= 0 ? *reinterpret_cast<volatile unsigned long long*>(&status[idx]) : kPre;
                    const uint32_t flag = (uint32_t)(w >> 32);
                    const uint32_t pm = __ballot_sync(0xffffffffu, flag == 2u);
                    const uint32_t nm = __ballot_sync(0xffffffffu, flag == 0u);
                    const uint32_t upto = pm ? (pm & (0u - pm)) * 2u - 1u : 0xffffffffu;  // lanes <= first P
                    if (nm & upto) {  // a needed predecessor has not published yet
                        __nanosleep(32);
                        if (clock64() - t0 > 4000000000ll) {
                            if (lane == 0) printf("scan look-back stuck: tile %u\n", tile);
                            __trap();
                        }
                        continue;
                    }
                    const uint32_t mine = (upto >> lane) & 1u ? (uint32_t)w : 0u;
                    prefix += __reduce_add_sync(0xffffffffu, mine);
                    if (pm) break;
                    j -= 32;
                }
                if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&status[tile]) = kPre | (prefix + total);
            }
            if (lane == 0) {
                s_prefix = prefix;
                if (tile == tiles - 1) tmp[2] = prefix + total;
            }
        }
        __syncthreads();
        uint32_t run = s_prefix + excl;
        if (full) {
#pragma unroll
            for (int k = 0; k < kScanItems; k += 4) {
                uint4 q;
                q.x = run;
                q.y = run += v[k];
                q.z = run += v[k + 1];
                q.w = run += v[k + 2];
                run += v[k + 3];
                *reinterpret_cast<uint4*>(x + base + k) = q;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kScanItems; ++k) {
                if (base + k < n) x[base + k] = run;
                run += v[k];
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
// Longest-processing-time-first order of the rasteriser's work units.  A unit's cost is how much
// of its list it walks before its pixels terminate, which the list length alone predicts poorly
// (deep central lists terminate after a few hundred splats, silhouette lists are walked to the
// end); with `feedback` the cost is the walk measured on the previous frame of the same geometry
// (temporal coherence of a camera path), else the list length.  Counting sort on a log2 key with
// 8 buckets per octave; equal keys keep unit order.
__global__ void __launch_bounds__(1024) unit_order_kernel(const uint32_t* __restrict__ offsets,
                                                          const uint32_t* __restrict__ feedback, int n_units,
                                                          int per_group, int* __restrict__ order,
                                                          FrameCounters* __restrict__ fc) {
    if (threadIdx.x == 0) {
        if (fc->overflow) atomicAdd(&fc->sticky_overflow, 1u);
        if (fc->err_validation) atomicAdd(&fc->sticky_invalid, 1u);
    }
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
                       FrameCounters* fc, cudaStream_t st) {
    unit_order_kernel<<<1, 1024, 0, st>>>(offsets, feedback, n_units, per_group, order, fc);
}

int bin_row_chunks(const GroupGeom& gg, uint64_t row_entries) {
    const int kr = (gg.band_gy1 - gg.band_gy0 + 31) / 32;
    int c = kRowChunksMin;
    while (c < kRowChunksMax && row_entries * kBinWarps > (uint64_t)c * (uint64_t)stage1_entries(kr)) c *= 2;
    return c;
}
size_t bin_hist1_elems(const GroupGeom& gg, int row_chunks) {
    return (size_t)std::max(1, gg.band_gy1 - gg.band_gy0) * (size_t)row_chunks;
}
size_t bin_hist2_elems(const GroupGeom& gg, uint32_t capacity) {
    const size_t rows = (size_t)std::max(1, gg.band_gy1 - gg.band_gy0);
    return (size_t)gg.groups_x * (rows + capacity / seg_len_gx(gg.groups_x) + 1);
}
size_t bin_meta_elems(const GroupGeom& gg) { return 4 * (size_t)(gg.band_gy1 - gg.band_gy0 + 1) + 1; }
size_t bin_slicecum_elems(const GroupGeom& gg, uint32_t capacity) {
    return bin_segmap_elems(gg, capacity) * (size_t)(kBinWarps - 1) * (size_t)gg.groups_x;
}
size_t bin_segmap_elems(const GroupGeom& gg, uint32_t capacity) {
    return (size_t)std::max(1, gg.band_gy1 - gg.band_gy0) + capacity / seg_len_gx(gg.groups_x) + 1;
}

size_t scan_tmp_elems(size_t n) { return 4 + 2 * ((n + kScanTile - 1) / kScanTile); }

const uint32_t* launch_exclusive_scan(uint32_t* x, size_t n, uint32_t* tmp, cudaStream_t st, const uint32_t* n_dev) {
    const size_t tiles = (n + kScanTile - 1) / kScanTile;
    cudaMemsetAsync(tmp, 0, scan_tmp_elems(n) * sizeof(uint32_t), st);
    const int grid = (int)std::min<size_t>(tiles, 148 * 8);
    if (grid > 0) scan_onepass_kernel<<<grid, kScanBlock, 0, st>>>(x, n, n_dev, tmp);
    return tmp + 2;
}

void launch_binning(const BinArgs& a, int max_visible, cudaStream_t st) {
    const GroupGeom& gg = a.gg;
    const int rows = gg.band_gy1 - gg.band_gy0, gx = gg.groups_x;
    (void)max_visible;
    // level 1
    const size_t n1 = bin_hist1_elems(gg, a.row_chunks);
    rows_count_kernel<<<a.row_chunks / kBinWarps, kBinWarps * 32, kBinWarps * (rows + 1) * sizeof(int), st>>>(a);
    uint32_t* tmp = a.bsum;
    const uint32_t* scan1_total = launch_exclusive_scan(a.hist1, n1, tmp, st, nullptr);
    rows_meta_kernel<<<1, 32, 0, st>>>(a, scan1_total);
    const int kr = (rows + 31) / 32, b1 = a.row_chunks / kBinWarps, t1 = kBinWarps * 32;
    // output stage, per-warp row records
    const size_t so1 = (size_t)stage1_entries(kr) * sizeof(uint2) + (size_t)kBinWarps * (rows + 1) * sizeof(uint2);
    auto launch1 = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)so1);
        kern<<<b1, t1, so1, st>>>(a);
    };
    if (kr <= 1)
        launch1(rows_place_kernel<1>);
    else if (kr <= 2)
        launch1(rows_place_kernel<2>);
    else if (kr <= 4)
        launch1(rows_place_kernel<4>);
    else if (kr <= 8)
        launch1(rows_place_kernel<8>);
    else
        launch1(rows_place_kernel<16>);
    // level 2
    const size_t n2 = bin_hist2_elems(gg, a.capacity);
    const uint32_t* h2_len = a.meta + 3 * rows + 2;  // rowbase2[rows]: device-side hist2 length
    const size_t max_seg = (size_t)rows + a.capacity / seg_len_gx(gx) + 1;
    const int qblocks = (int)std::max<size_t>(1, std::min<size_t>(148 * 8, (max_seg + kBinWarps - 1) / kBinWarps));
    cols_count_kernel<<<qblocks, kBinWarps * 32, kBinWarps * (gx + 1) * sizeof(int), st>>>(a);
    launch_exclusive_scan(a.hist2, n2, tmp, st, h2_len);
    offsets_kernel<<<(gg.n_groups_band + 256) / 256, 256, 0, st>>>(a);
    const int kc = (gx + 31) / 32, t2 = kBinWarps * 32;
    // output stage + column ids, column bias, per-warp slice counts / column positions / masks
    // output stage, per-warp column records
    const size_t so = (size_t)stage2_entries(kc) * sizeof(uint32_t) + (size_t)kBinWarps * (gx + 1) * sizeof(uint2);
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)so);
        kern<<<qblocks, t2, so, st>>>(a);
    };
    if (kc <= 1)
        launch(cols_place_kernel<1>);
    else if (kc <= 2)
        launch(cols_place_kernel<2>);
    else if (kc <= 4)
        launch(cols_place_kernel<4>);
    else if (kc <= 8)
        launch(cols_place_kernel<8>);
    else
        launch(cols_place_kernel<16>);
}

// ReuseReport of the last frame's group lists (metrics.cpp:45-57) without materialising masks: a
// splat's entry in group (gx, gy) has popcount wx(gx) * wy(gy), the numbers of its tile columns /
// rows inside that group, so per splat the histogram is the product of two width histograms.
__global__ void __launch_bounds__(256) reuse_hist_kernel(const FrameCounters* __restrict__ fc,
                                                         const uint2* __restrict__ rect, GroupGeom gg,
                                                         unsigned long long* __restrict__ hist) {
    __shared__ unsigned long long h[17];
    if (threadIdx.x < 17) h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t n = fc->n_input;
    const int G = gg.g;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        int x0, x1, y0, y1;
        const uint2 r = __ldg(&rect[i]);
        if (r.x == kCulledRect && r.y == kCulledRect) continue;  // not projected
        if (!decode_rect(r, x0, x1, y0, y1)) continue;
        // band: keep tile rows of the band's group rows
        y0 = max(y0, gg.band_gy0 * G);
        y1 = min(y1, gg.band_gy1 * G - 1);
        if (y1 < y0) continue;
        uint32_t nx[5] = {0, 0, 0, 0, 0}, ny[5] = {0, 0, 0, 0, 0};
        for (int g = x0 / G; g <= x1 / G; ++g) ++nx[min(x1, g * G + G - 1) - max(x0, g * G) + 1];
        for (int g = y0 / G; g <= y1 / G; ++g) ++ny[min(y1, g * G + G - 1) - max(y0, g * G) + 1];
        for (int wx = 1; wx <= G; ++wx)
            for (int wy = 1; wy <= G; ++wy)
                if (nx[wx] && ny[wy]) atomicAdd(&h[wx * wy], (unsigned long long)nx[wx] * ny[wy]);
    }
    __syncthreads();
    if (threadIdx.x < 17 && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

void launch_reuse_hist(const FrameCounters* fc, const uint2* rect, const GroupGeom& gg, int max_input,
                       unsigned long long* hist, cudaStream_t st) {
    cudaMemsetAsync(hist, 0, 17 * sizeof(unsigned long long), st);
    const int blocks = std::max(1, std::min(148 * 4, (max_input + 255) / 256));
    reuse_hist_kernel<<<blocks, 256, 0, st>>>(fc, rect, gg, hist);
}

void launch_lists_readback(const uint32_t* sorted_idx, const uint32_t* offsets, int n_groups,
                           DevProjected proj, GroupGeom gg, tgs_group_entry* out, cudaStream_t st) {
    if (n_groups > 0) lists_readback_kernel<<<n_groups, 256, 0, st>>>(sorted_idx, offsets, n_groups, proj, gg, out);
}

void launch_encode_u8(const float* rgb, int64_t n, uint8_t* out, cudaStream_t st) {
    encode_u8_kernel<<<148 * 8, 256, 0, st>>>(rgb, n, out);
}

}  // namespace tgs
