// Exact-emulation rasteriser: the reference's per-pixel arithmetic
// reproduced bit for bit on CUDA cores, for either precision mode and any group size.
//
// Reference semantics followed operation by operation (all binary32, no contraction — the
// reference builds with -ffp-contract=off, CMakeLists.txt:10-12):
//   stage_operands  (operands.hpp:27-37):  q1 = Q(-0.5f * a), q2 = Q(-b), q3 = Q(-0.5f * c),
//                                          mean = Q(mean2d), opacity = Q(opacity);
//   pixel_basis     (operands.hpp:49-58):  dx = Q(px - mean_x), dy = Q(py - mean_y),
//                                          f1 = Q(dx * dx), f2 = Q(dx * dy), f3 = Q(dy * dy);
//   splat_power     (operands.hpp:65-72):  ((0 + q1 f1) + q2 f2) + q3 f3;
//   alpha_of        (raster_scalar.hpp:40-45): power > 0 -> 0, min(clamp, o * expf(power)), skip;
//   blend           (raster_scalar.hpp:49-55): w = T a, accum += w c, T *= (1 - a), done at T < t;
// with Q = lane_quantize: identity in fp32 mode, binary16 round-to-nearest-even in fp16 mode
// (half.hpp:12-84; __float2half_rn is the same rounding).  expf is the reference toolchain's
// libm expf (glibc 2.39, the ARM optimized-routines algorithm: 32-entry 2^(i/32) table, cubic in
// double precision) restated in double precision; it equals the host expf on every negative float
// above -88 but one (x = -0x1.f8cbb2p+5, far below any alpha_skip threshold; checked exhaustively
// by tests/test_oracle.py).  Every tile walks its group's list and keeps the entries whose 3-sigma
// tile rectangle contains it (the mask bit, binning.cpp:56-65), which is exactly the per-tile entry
// sequence of both rasterize_tiles_scalar and rasterize_groups_tensor — the reference's own
// acceptance criteria make those images identical (acceptance.cpp:177-238).
//
// This is a validation mode (PrecisionMode::fp16, or tgs_set_exact_emulation), not the fast path.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"
#include "tgs_expf.cuh"

namespace tgs {

namespace {

template <bool kHalf>
__device__ __forceinline__ float lane_q(float v) {
    return kHalf ? __half2float(__float2half_rn(v)) : v;
}

constexpr int kBatch = 256;

template <bool kHalf>
__global__ void __launch_bounds__(256) raster_exact_kernel(RasterArgs a) {
    __shared__ float4 s_q[kBatch];   // q1, q2, q3, opacity (lane precision, widened)
    __shared__ float4 s_m[kBatch];   // mean x, mean y (lane precision), color r, g
    __shared__ float s_b[kBatch];    // color b
    __shared__ int s_wcnt[8];
    const GroupGeom& gg = a.gg;
    // one CTA per tile of the band; the tile walks its group's list
    const int tiles_band = gg.tiles_x * (gg.band_gy1 - gg.band_gy0) * gg.g;
    if ((int)blockIdx.x >= tiles_band) return;
    const int tx = blockIdx.x % gg.tiles_x, ty = blockIdx.x / gg.tiles_x + gg.band_gy0 * gg.g;
    const bool tile_in = ty < gg.tiles_y;
    const int gid = (ty / gg.g - gg.band_gy0) * gg.groups_x + tx / gg.g;
    const int px = tx * kTile + (threadIdx.x & 15), py = ty * kTile + (threadIdx.x >> 4);
    const bool inside = tile_in && px < gg.width && py < gg.height;
    const float fx = (float)px + 0.5f, fy = (float)py + 0.5f;  // pixel_center (operands.hpp:16)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    bool done = !inside;
    const uint32_t begin = tile_in ? a.offsets[gid] : 0u, end = tile_in ? a.offsets[gid + 1] : 0u;
    for (uint32_t base = begin; base < end; base += kBatch) {
        if (__syncthreads_count(done) == (int)blockDim.x) break;
        const uint32_t e = base + threadIdx.x;
        bool ok = false;
        float4 q = make_float4(0, 0, 0, 0), m = q;
        float bcol = 0.0f;
        if (e < end) {
            const uint32_t idx = a.list[e];
            const float4 mc = a.proj.mc[idx], co = a.proj.co[idx], col = a.proj.col[idx];
            int x0, y0, x1, y1;
            tile_rect(mc.x, mc.y, __float_as_int(co.w), gg.tiles_x, gg.tiles_y, x0, y0, x1, y1);
            ok = tx >= x0 && tx <= x1 && ty >= y0 && ty <= y1;  // the entry's mask has this tile
            q = make_float4(lane_q<kHalf>(__fmul_rn(-0.5f, mc.z)), lane_q<kHalf>(-mc.w),
                            lane_q<kHalf>(__fmul_rn(-0.5f, co.x)), lane_q<kHalf>(co.y));
            m = make_float4(lane_q<kHalf>(mc.x), lane_q<kHalf>(mc.y), col.x, col.y);
            bcol = col.z;
        }
        // in-order compaction of the batch's entries that belong to this tile
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) s_wcnt[warp] = __popc(bal);
        __syncthreads();
        int pos = __popc(bal & ((1u << lane) - 1u)), n = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const int c = s_wcnt[w];
            if (w < warp) pos += c;
            n += c;
        }
        if (ok) {
            s_q[pos] = q;
            s_m[pos] = m;
            s_b[pos] = bcol;
        }
        __syncthreads();
        if (!done) {
            for (int j = 0; j < n; ++j) {
                const float4 qq = s_q[j], mm = s_m[j];
                const float dx = lane_q<kHalf>(__fsub_rn(fx, mm.x)), dy = lane_q<kHalf>(__fsub_rn(fy, mm.y));
                const float f1 = lane_q<kHalf>(__fmul_rn(dx, dx)), f2 = lane_q<kHalf>(__fmul_rn(dx, dy)),
                            f3 = lane_q<kHalf>(__fmul_rn(dy, dy));
                float power = __fadd_rn(0.0f, __fmul_rn(qq.x, f1));
                power = __fadd_rn(power, __fmul_rn(qq.y, f2));
                power = __fadd_rn(power, __fmul_rn(qq.z, f3));
                if (power > 0.0f) power = 0.0f;
                const float ev = __fmul_rn(qq.w, expf_glibc(power));
                const float alpha = ev < a.alpha_clamp ? ev : a.alpha_clamp;  // std::min(clamp, .)
                if (alpha < a.alpha_skip) continue;
                const float w = __fmul_rn(T, alpha);
                cr = __fadd_rn(cr, __fmul_rn(w, mm.z));
                cg = __fadd_rn(cg, __fmul_rn(w, mm.w));
                cb = __fadd_rn(cb, __fmul_rn(w, s_b[j]));
                T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
                if (T < a.t_terminate) {
                    done = true;
                    break;
                }
            }
        }
    }
    if (inside) {
        float* o = a.image + ((size_t)(py - a.image_row0) * gg.width + px) * 3;
        o[0] = fminf(fmaxf(cr, 0.0f), 1.0f);
        o[1] = fminf(fmaxf(cg, 0.0f), 1.0f);
        o[2] = fminf(fmaxf(cb, 0.0f), 1.0f);
    }
}

}  // namespace

void launch_raster_exact(const RasterArgs& a, bool fp16, cudaStream_t st) {
    const int tiles = a.gg.tiles_x * (a.gg.band_gy1 - a.gg.band_gy0) * a.gg.g;
    if (tiles <= 0) return;
    if (fp16)
        raster_exact_kernel<true><<<tiles, 256, 0, st>>>(a);
    else
        raster_exact_kernel<false><<<tiles, 256, 0, st>>>(a);
}

}  // namespace tgs
