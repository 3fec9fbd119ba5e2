// Shared device-side definitions of libtgs (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/tgs.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libtgs is written for sm_100a (B200) only"
#endif

namespace tgs {

constexpr int kTile = 16;  // binning.hpp:11 kTileSize
constexpr uint32_t kCulledKey = 0xffffffffu;   // presort key of a culled/dropped splat (dropped by pass 1)
constexpr uint32_t kCulledRect = 0xffffffffu;  // rect word of a culled/dropped splat

// Camera parameters as the preprocess kernel consumes them (row-major R, t).
struct DevCamera {
    float r[3][3];
    float t[3];
    float fx, fy;
    int width, height;
    float near_, far_;
};

// Device scene: SoA float4 planes, coalesced 16/8-byte loads per Gaussian.
struct DevScene {
    const float4* pos_op;     // mean.xyz, opacity
    const float4* quat;       // w, x, y, z
    const float4* scale_dcr;  // scale.xyz, sh_dc.r
    const float2* dc_gb;      // sh_dc.g, sh_dc.b
    const float4* sh_rest;    // 12 planes of n float4 (coefficients 4p..4p+3), or null
    int n;
    int sh_degree;
};

// Projected splats, indexed by the compacted (project_scene output) index.
struct DevProjected {
    float4* mc;   // mean2d.x, mean2d.y, conic_a, conic_b
    float4* co;   // conic_c, opacity, depth, radius (int bits)
    float4* col;  // color r, g, b, tile-cull extents (half2, tight_extents)
};

// Device counters / flags of one frame (zeroed per frame).
struct FrameCounters {
    unsigned long long culled;
    unsigned long long dropped;
    unsigned long long appearances;
    unsigned int visible;           // projected (kept) splats
    unsigned int n_entries;         // emitted entries (may exceed capacity -> overflow)
    unsigned int n_sort;            // entries handed to the group sort (0 on overflow)
    unsigned int err_validation;    // non-positive scale (projection.cpp:37) / bad depth (binning.cpp:78-83)
    unsigned int overflow;          // entry capacity exceeded
    unsigned int n_input;           // scene size (first presort pass item count)
    unsigned int group_counter;     // persistent raster scheduler ticket
    unsigned long long walked;      // instrumented pair counters (tgs_count_pairs)
    unsigned long long blended;
    unsigned int key_min_inv;       // ~min and max of the visible depth keys: the presort ranks
    unsigned int key_max;           // (key - min), so passes above the key range are plain copies
    // OpReport (metrics.hpp:49-69) of the tensor rasteriser: chunks staged, tcgen05.mma issued,
    // splat rows those MMAs carried, (member tile, staged row) pairs the mask filtered out
    unsigned long long op_chunks, op_mmas, op_mma_rows, op_skipped;
    unsigned int row_entries;       // group-row entries of the frame (sizes the next frame's chunks)
    // not zeroed per frame: frames of this context that overflowed / failed validation so far
    // (counted by unit_order_kernel, checked by tgs_sync so no un-synced frame fails silently)
    unsigned int sticky_overflow;
    unsigned int sticky_invalid;
};

// Group geometry (GroupConfig, binning.hpp:15-31) with an optional band of group rows.
struct GroupGeom {
    int g;          // tiles per group side
    int width, height;
    int tiles_x, tiles_y;
    int groups_x, groups_y;
    int band_gy0, band_gy1;  // group rows [gy0, gy1) are binned; others dropped
    int n_groups_band;       // groups_x * (gy1 - gy0)
};

// Exact IEEE single operations (no FMA contraction) for the bit-exact stages.
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float fsqrt(float a) { return __fsqrt_rn(a); }
// Eigen fixed-size 3-term reduction order: e0 + (e1 + e2).
__device__ __forceinline__ float sum3(float e0, float e1, float e2) { return fadd(e0, fadd(e1, e2)); }

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// binning.cpp:32-44 tiles_overlapped, clipped to the tile grid. Same float ops as the reference:
// floor((mean - r) / 16), division by 16 is exact.
__device__ __forceinline__ void tile_rect(float mx, float my, int radius, int tiles_x, int tiles_y,
                                          int& x0, int& y0, int& x1, int& y1) {
    const float r = (float)radius;
    // x / 16 (binning.cpp:32-44) == x * 2^-4 exactly (same real value, same rounding), so the
    // multiply is bit-identical to the reference's division and avoids the IEEE divide sequence
    x0 = (int)floorf(__fmul_rn(__fsub_rn(mx, r), 0.0625f));
    x1 = (int)floorf(__fmul_rn(__fadd_rn(mx, r), 0.0625f));
    y0 = (int)floorf(__fmul_rn(__fsub_rn(my, r), 0.0625f));
    y1 = (int)floorf(__fmul_rn(__fadd_rn(my, r), 0.0625f));
    x0 = max(x0, 0);
    y0 = max(y0, 0);
    x1 = min(x1, tiles_x - 1);
    y1 = min(y1, tiles_y - 1);
}

// Group-rect of a splat (restricted to the band), returns number of groups (0 = no entries).
__device__ __forceinline__ int group_rect(float mx, float my, int radius, const GroupGeom& gg,
                                          int& tx0, int& ty0, int& tx1, int& ty1, int& gx0,
                                          int& gy0, int& gx1, int& gy1) {
    tile_rect(mx, my, radius, gg.tiles_x, gg.tiles_y, tx0, ty0, tx1, ty1);
    if (tx1 < tx0 || ty1 < ty0) return 0;
    const int sh = gg.g >> 1;  // G in {1, 2, 4}
    gx0 = tx0 >> sh;
    gx1 = tx1 >> sh;
    gy0 = max(ty0 >> sh, gg.band_gy0);
    gy1 = min(ty1 >> sh, gg.band_gy1 - 1);
    if (gy1 < gy0) return 0;
    return (gx1 - gx0 + 1) * (gy1 - gy0 + 1);
}

// Member-tile mask of group (gx, gy) for tile rect [tx0..tx1]x[ty0..ty1] (binning.cpp:56-65).
__device__ __forceinline__ uint32_t group_mask(int gx, int gy, int g, int tx0, int ty0, int tx1,
                                               int ty1) {
    const int a0 = max(tx0, gx * g), a1 = min(tx1, gx * g + g - 1);
    const int b0 = max(ty0, gy * g), b1 = min(ty1, gy * g + g - 1);
    uint32_t m = 0;
    for (int ty = b0; ty <= b1; ++ty)
        for (int tx = a0; tx <= a1; ++tx) m |= 1u << ((ty - gy * g) * g + (tx - gx * g));
    return m;
}

// Tile cull (rasterisers, tgs_set_tile_cull): the axis-aligned box of the ellipse
// power >= ln(alpha_skip / o)  (conic (a, b, c); half-extents sqrt(2 lnt Sigma_xx), sqrt(2 lnt
// Sigma_yy) with Sigma the 2D covariance) padded by half a pixel — far more than the FP16 hi/lo error
// of the tensor path's D — contains every pixel centre where the splat can reach alpha_skip.  The
// preprocess stores the padded half-extents as a half2 rounded up (a superset) in col.w; +inf
// halves mean "no bound" (opacity at or below alpha_skip, degenerate conic).  Tighter than the
// reference's 3-sigma square (binning.cpp:32-44), which stays the list criterion.
// The box only has to be a superset, so it is computed with the MUFU approximations (log2, rcp,
// rsqrt; relative errors ~2^-21) and widened by 2^-12 relative before the half-pixel pad.
__device__ __forceinline__ float tight_extents(float ca, float cb, float cc, float o, float skip) {
    const float det = ca * cc - cb * cb;
    const float lnt = __logf(__fdividef(o, skip));
    __half2 e = __halves2half2(__ushort_as_half((unsigned short)0x7c00u), __ushort_as_half((unsigned short)0x7c00u));
    if (det > 0.0f && lnt > 0.0f) {
        const float s2 = 2.0f * lnt * __frcp_rn(det) * (1.0f + 0x1p-12f);
        const float vx = s2 * cc, vy = s2 * ca;  // >= 0: a positive-definite conic
        // sqrt as v * rsqrt(v); an overflowed v stays +inf ("no bound"), 0 stays 0 (never inf * 0)
        auto root = [](float v) { return v > 0.0f && v < 0x1p126f ? v * rsqrtf(v) : v; };
        const float ex = root(vx), ey = root(vy);
        e = __halves2half2(__float2half_ru(ex + 0.5f), __float2half_ru(ey + 0.5f));
    }
    return __uint_as_float(*reinterpret_cast<const uint32_t*>(&e));
}

// Member tiles (bit k: tile (tx0 + (k & 1), ty0 + (k >> 1))) whose pixel centres meet the box.
__device__ __forceinline__ uint32_t tight_cover(float mx, float my, float ext, int tx0, int ty0, int slots) {
    const uint32_t eb = __float_as_uint(ext);
    const float2 e = __half22float2(*reinterpret_cast<const __half2*>(&eb));
    uint32_t m = 0;
    for (int k = 0; k < slots; ++k) {
        const float px0 = (float)((tx0 + (k & 1)) * kTile) + 0.5f, py0 = (float)((ty0 + (k >> 1)) * kTile) + 0.5f;
        if (mx - e.x <= px0 + (kTile - 1) && mx + e.x >= px0 && my - e.y <= py0 + (kTile - 1) && my + e.y >= py0)
            m |= 1u << k;
    }
    return m;
}

// Tile span [lo, hi] along one axis whose pixel centres meet the padded alpha_skip box
// [m - e, m + e] — exactly the tiles tight_cover accepts (same float comparisons) — intersected
// with the 3-sigma span [lo3, hi3] of binning.cpp:32-44.  lo > hi: none.
__device__ __forceinline__ void tight_span(float m, float e, int lo3, int hi3, int& lo, int& hi) {
    // floor() of the real bounds is off by at most one tile after rounding; the exact per-tile
    // tests settle it (cvt saturates for an unbounded +-inf extent)
    lo = max(lo3, (int)floorf((m - e - 15.5f) * 0.0625f));
    while (lo <= hi3 && !(m - e <= (float)(lo * kTile) + 0.5f + (kTile - 1))) ++lo;
    hi = min(hi3, (int)floorf((m + e - 0.5f) * 0.0625f));
    if (hi < hi3 && m + e >= (float)((hi + 1) * kTile) + 0.5f) ++hi;
    while (hi >= lo && !(m + e >= (float)(hi * kTile) + 0.5f)) --hi;
}

}  // namespace tgs

#define TGS_CUDA_OK(expr)                                                   \
    do {                                                                    \
        cudaError_t _e = (expr);                                            \
        if (_e != cudaSuccess) return tgs::cuda_fail(_e, #expr, __FILE__, __LINE__); \
    } while (0)
