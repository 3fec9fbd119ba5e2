// CUDA-core baseline rasterizer (the denominator of the >= 1.65x raster target).
//
// Reference semantics: proj/src/raster_scalar.cpp:9-71 with raster_scalar.hpp:29-55 — per tile
// (G = 1 lists), every pixel walks its tile's depth-sorted list; power clamped to <= 0,
// alpha = min(alpha_clamp, opacity * exp(power)), skip alpha < alpha_skip, blend, and the splat
// that drives T below t_terminate is blended before the pixel stops.  No background colour;
// output clamped to [0,1] (ImageBuffer::finalize, types.hpp:66-68).
//
// Structure: the classic 3DGS forward kernel, written for sm_100a — one 256-thread CTA per
// 16x16 tile, one thread per pixel, the list consumed in smem-staged batches of 256 splats
// (coalesced index loads, 3 float4 gathers per splat), CTA-wide early exit with
// __syncthreads_count.  It is deliberately a *good* CUDA-core kernel: exp runs on MUFU (ex2 of
// power*log2e), the power uses FMA, per-splat operands are broadcast from smem.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

namespace tgs {

namespace {

constexpr int kBatch = 256;
constexpr float kLog2e = 1.4426950408889634f;

__global__ void __launch_bounds__(256) raster_scalar_kernel(RasterArgs a) {
    __shared__ float4 s_geo[kBatch];  // mx, my, q1=-a/2*log2e, q2=-b*log2e
    __shared__ float4 s_gc[kBatch];   // q3=-c/2*log2e, opacity, r, g
    __shared__ float s_b[kBatch];     // b
    __shared__ int s_wcnt[8];         // kept splats per warp of the staged batch
    const GroupGeom& gg = a.gg;
    const int tile = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;  // LPT order, as the tensor path
    const int tx = tile % gg.tiles_x, ty = tile / gg.tiles_x + gg.band_gy0;  // G == 1: group == tile
    const int px = tx * kTile + (threadIdx.x & 15);
    const int py = ty * kTile + (threadIdx.x >> 4);
    const bool inside = px < gg.width && py < gg.height;
    const float fx = (float)px + 0.5f, fy = (float)py + 0.5f;  // pixel_center (operands.hpp:16)

    const uint32_t begin = a.offsets[tile], end = a.offsets[tile + 1];
    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    bool done = !inside;
    uint32_t base = begin;
    for (; base < end; base += kBatch) {
        if (__syncthreads_count(done) == kBatch) break;
        const uint32_t e = base + threadIdx.x;
        // stage the batch, keeping (in list order) only splats that can reach alpha_skip on this
        // tile: min(clamp, o) >= skip and the padded alpha_skip ellipse box meets the tile (the
        // same test the tensor producer applies, tight_cover)
        bool ok = false;
        float4 G, H;
        float B = 0.0f;
        if (e < end) {
            const uint32_t idx = a.list[e];
            const float4 mc = a.proj.mc[idx];
            const float4 co = a.proj.co[idx];
            const float4 col = a.proj.col[idx];
            ok = !(fminf(a.alpha_clamp, co.y) < a.alpha_skip) &&
                 (!a.tile_cull || tight_cover(mc.x, mc.y, col.w, tx, ty, 1) != 0u);
            G = make_float4(mc.x, mc.y, -0.5f * mc.z * kLog2e, -mc.w * kLog2e);
            H = make_float4(-0.5f * co.x * kLog2e, co.y, col.x, col.y);
            B = col.z;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) s_wcnt[warp] = __popc(bal);
        __syncthreads();
        int pos = __popc(bal & ((1u << lane) - 1u)), n = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const int cw = s_wcnt[w];
            if (w < warp) pos += cw;
            n += cw;
        }
        if (ok) {
            s_geo[pos] = G;
            s_gc[pos] = H;
            s_b[pos] = B;
        }
        __syncthreads();
        if (!done) {
            for (int j = 0; j < n; ++j) {
                const float4 g = s_geo[j];
                const float4 h = s_gc[j];
                const float dx = fx - g.x, dy = fy - g.y;
                // power * log2e, clamped at 0 (raster_scalar.hpp:41)
                const float p2 = fminf(g.z * dx * dx + g.w * dx * dy + h.x * dy * dy, 0.0f);
                const float alpha = fminf(a.alpha_clamp, h.y * ex2_approx(p2));
                if (alpha < a.alpha_skip) continue;
                const float w = T * alpha;
                cr += w * h.z;
                cg += w * h.w;
                cb += w * s_b[j];
                T *= (1.0f - alpha);
                if (T < a.t_terminate) {
                    done = true;
                    break;
                }
            }
        }
    }
    // schedule feedback: list entries this tile walked
    if (a.unit_cost && threadIdx.x == 0) a.unit_cost[tile] = min(base, end) - begin;
    if (inside) {
        float* o = a.image + ((size_t)(py - a.image_row0) * gg.width + px) * 3;
        o[0] = fminf(fmaxf(cr, 0.0f), 1.0f);
        o[1] = fminf(fmaxf(cg, 0.0f), 1.0f);
        o[2] = fminf(fmaxf(cb, 0.0f), 1.0f);
    }
}

// Instrumented reference walk (no timing role): counts walked pairs (entries of the tile's list
// visited before the pixel is done, raster_scalar.cpp:36-41 / raster_tensor.cpp:130-143) and
// alpha-contributing pairs, with the reference's exact fp32 power (operands.hpp:65-72) and expf.
// Works on any G: a tile walks its group's list and skips entries whose mask lacks the tile.
__global__ void __launch_bounds__(256) count_pairs_kernel(RasterArgs a) {
    const GroupGeom& gg = a.gg;
    const int tx = blockIdx.x % gg.tiles_x, ty = blockIdx.x / gg.tiles_x + gg.band_gy0 * gg.g;
    const int px = tx * kTile + (threadIdx.x & 15);
    const int py = ty * kTile + (threadIdx.x >> 4);
    const int gid = (ty / gg.g - gg.band_gy0) * gg.groups_x + tx / gg.g;
    unsigned long long walked = 0, blended = 0;
    uint32_t trip = 0;  // position in the tile's (mask-filtered) list where this pixel stopped
    if (px < gg.width && py < gg.height && ty < gg.tiles_y) {
        const float fx = (float)px + 0.5f, fy = (float)py + 0.5f;
        float T = 1.0f;
        for (uint32_t e = a.offsets[gid]; e < a.offsets[gid + 1]; ++e) {
            const uint32_t idx = a.list[e];
            const float4 mc = a.proj.mc[idx];
            const float4 co = a.proj.co[idx];
            int x0, y0, x1, y1;
            tile_rect(mc.x, mc.y, __float_as_int(co.w), gg.tiles_x, gg.tiles_y, x0, y0, x1, y1);
            if (tx < x0 || tx > x1 || ty < y0 || ty > y1) continue;
            ++trip;
            const float dx = __fsub_rn(fx, mc.x), dy = __fsub_rn(fy, mc.y);
            float acc = 0.0f;
            acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(-0.5f, mc.z), __fmul_rn(dx, dx)));
            acc = __fadd_rn(acc, __fmul_rn(-mc.w, __fmul_rn(dx, dy)));
            acc = __fadd_rn(acc, __fmul_rn(__fmul_rn(-0.5f, co.x), __fmul_rn(dy, dy)));
            if (acc > 0.0f) acc = 0.0f;
            const float ev = __fmul_rn(co.y, expf(acc));
            const float alpha = ev < a.alpha_clamp ? ev : a.alpha_clamp;
            ++walked;
            if (alpha < a.alpha_skip) continue;
            ++blended;
            T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
            if (T < a.t_terminate) break;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        walked += __shfl_xor_sync(0xffffffffu, walked, o);
        blended += __shfl_xor_sync(0xffffffffu, blended, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&a.fc->walked, walked);
        atomicAdd(&a.fc->blended, blended);
    }
    if (a.tile_trip) {
        __shared__ uint32_t s_trip;
        if (threadIdx.x == 0) s_trip = 0;
        __syncthreads();
        atomicMax(&s_trip, trip);
        __syncthreads();
        if (threadIdx.x == 0) a.tile_trip[blockIdx.x] = s_trip;
    }
}

}  // namespace

void launch_raster_scalar(const RasterArgs& a, cudaStream_t st) {
    const int tiles = a.gg.tiles_x * (a.gg.band_gy1 - a.gg.band_gy0);
    if (tiles > 0) raster_scalar_kernel<<<tiles, 256, 0, st>>>(a);
}

void launch_count_pairs(const RasterArgs& a, cudaStream_t st) {
    const int tiles = a.gg.tiles_x * (a.gg.band_gy1 - a.gg.band_gy0) * a.gg.g;
    if (tiles > 0) count_pairs_kernel<<<tiles, 256, 0, st>>>(a);
}

}  // namespace tgs
