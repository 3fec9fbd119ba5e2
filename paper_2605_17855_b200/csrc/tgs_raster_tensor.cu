// Tensorized, cross-tile-grouped rasterizer (north_star 3 + 4) on the 5th-gen tensor cores.
//
// Reference semantics: proj/src/raster_tensor.cpp:64-160 (rasterize_group_impl) — a group of
// G x G tiles walks its depth-sorted list chunk by chunk; every live member tile consumes the
// chunk's entries whose mask has its bit, in list order; per pixel the power feeds
// alpha_of/blend (raster_scalar.hpp:40-55) until T < t_terminate; tiles/groups retire early.
//
// B200 formulation.  The reference builds a pixel operand per Gaussian row
// (raster_tensor.cpp:118-123), which no hardware MMA can do.  Here the power is expanded around
// each tile's centre o:  u = pixel - o, m = mean - o,
//     log2(e) * power + log2(opacity) = w . phi(u),
//     phi(u) = [ux^2, ux*uy, uy^2, ux, uy, 1]                      (pixel side, exact in FP16)
//     w      = log2e * [-a/2, -b, -c/2, a mx + b my, b mx + c my,
//                       -(a mx^2/2 + b mx my + c my^2/2)] + [0,0,0,0,0, log2 o]  (splat side)
// and w is carried as an FP16 hi/lo pair, so K = 6 (hi) + 6 (lo) + 4 zero lanes = 16:
//     D[pixel][splat] = A[pixel][0:16] . B[splat][0:16]      (one tcgen05.mma, M=128, K=16)
// gives the ex2 argument directly: alpha = min(min(alpha_clamp, o), ex2(D)), skip D < log2(skip).
// Splats outside a tile's mask (binning.cpp:56-65), rows past the list end and splats whose
// min(clamp, o) < alpha_skip get the row "D = -30000", so the alpha-skip test also realises the
// mask filter — the epilogue has no per-tile branch.  Any row with |w| > 16384 cannot contribute
// to its tile (the +0.3 dilation bounds the conic) and gets the same row.
//
// CTA = one group at a time (persistent over groups):
//   warps [0, EPI)  epilogue: each thread owns PPT pixels (TMEM lane = pixel), tcgen05.ld's its
//                   D rows and runs the ordered blend on CUDA cores + MUFU ex2;
//   warp EPI        producer: gathers the chunk's splats (one per lane), derives the per-tile
//                   coefficient rows (hi/lo FP16) into smem — the chunk is staged once and
//                   shared by all G*G tiles (north_star 4);
//   warp EPI+1      TMEM owner + MMA issuer: one tcgen05.mma per 128-pixel M-tile per chunk,
//                   tcgen05.commit -> epilogue.
// A (pixel monomials) is identical for every tile, built once per CTA (256 rows x 32 B).
// Chunks flow through STAGES smem/TMEM stages guarded by mbarriers; the chunk header carries
// the group id, so group boundaries need no extra synchronisation.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"
#include "tgs_ptx.cuh"

namespace tgs {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kNeverRow = -30000.0f;
constexpr float kInf = __builtin_huge_valf();

template <int G>
struct Cfg {
    static constexpr int TILES = G * G;
    static constexpr int MT = 2 * TILES;                      // 128-pixel M-tiles
    static constexpr int N = (G == 4) ? 16 : 32;              // splats per chunk (MMA N)
    static constexpr int STAGES = (G == 4) ? 1 : 2;
    static constexpr int COLS_USED = STAGES * MT * N;
    static constexpr int TMEM_COLS = COLS_USED <= 32 ? 32 : COLS_USED <= 64 ? 64 : COLS_USED <= 128 ? 128
                                     : COLS_USED <= 256 ? 256 : 512;
    static constexpr int EPI = (G == 1) ? 8 : 16;             // epilogue warps
    static constexpr int PPT = MT * 4 / EPI;                  // pixels per epilogue thread
    static constexpr int THREADS = (EPI + 2) * 32;
    static constexpr int CTAS_PER_SM = 512 / TMEM_COLS;
    static constexpr int B_BYTES = N * 32;                    // one tile's B operand
};

struct ChunkHeader {
    int gid;      // band-local group id, -1 = end of stream
    int n_valid;  // splats in the chunk (0: empty group)
};

template <int G>
struct Smem {
    alignas(128) uint8_t a[256 * 32];                                        // pixel monomials
    alignas(128) uint8_t b[Cfg<G>::STAGES][Cfg<G>::TILES][Cfg<G>::B_BYTES];  // splat rows
    float4 epi[Cfg<G>::STAGES][Cfg<G>::N];                                   // r, g, b, min(clamp, o)
    ChunkHeader hdr[Cfg<G>::STAGES];
    int alive[Cfg<G>::STAGES];
    uint64_t full[Cfg<G>::STAGES];      // producer -> MMA
    uint64_t tfull[Cfg<G>::STAGES];     // MMA -> epilogue (tcgen05.commit)
    uint64_t done[Cfg<G>::STAGES];      // epilogue -> producer (stage reusable)
    uint32_t tmem_base;
};

// byte offset of (row, k-half) in a K-major no-swizzle operand: 8x16B core matrices
__device__ __forceinline__ uint32_t core_off(int row, int khalf) {
    return (uint32_t)((row >> 3) * 256 + khalf * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

template <int G>
__global__ void __launch_bounds__(Cfg<G>::THREADS, 1) raster_tensor_kernel(RasterArgs a) {
    using C = Cfg<G>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem<G>& sm = *reinterpret_cast<Smem<G>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const GroupGeom& gg = a.gg;
    const int n_groups = gg.n_groups_band;

    // ---- setup: A operand, barriers, TMEM ----------------------------------------------------
    if (threadIdx.x < 256) {
        const int p = threadIdx.x;
        const float ux = (float)(p & 15) - 7.5f, uy = (float)(p >> 4) - 7.5f;
        const float phi[6] = {ux * ux, ux * uy, uy * uy, ux, uy, 1.0f};
        uint4 lo, hi;
        lo.x = pack_half2(phi[0], phi[1]);
        lo.y = pack_half2(phi[2], phi[3]);
        lo.z = pack_half2(phi[4], phi[5]);
        lo.w = pack_half2(phi[0], phi[1]);
        hi.x = pack_half2(phi[2], phi[3]);
        hi.y = pack_half2(phi[4], phi[5]);
        hi.z = 0u;
        hi.w = 0u;
        *reinterpret_cast<uint4*>(sm.a + core_off(p, 0)) = lo;
        *reinterpret_cast<uint4*>(sm.a + core_off(p, 1)) = hi;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            ptx::mbar_init(&sm.full[s], 1);
            ptx::mbar_init(&sm.tfull[s], 1);
            ptx::mbar_init(&sm.done[s], C::EPI);
            sm.alive[s] = 0;
        }
        ptx::mbar_fence_init();
    }
    if (warp == C::EPI + 1) ptx::tmem_alloc<C::TMEM_COLS>(&sm.tmem_base);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == C::EPI) {
        // ================================ producer ===========================================
        const float L = a.alpha_skip;
        uint32_t c = 0;
        for (;;) {
            int g = 0;
            if (lane == 0) g = (int)atomicAdd(&a.fc->group_counter, 1u);
            g = __shfl_sync(0xffffffffu, g, 0);
            if (g >= n_groups) break;
            const int gx = g % gg.groups_x, gy = g / gg.groups_x + gg.band_gy0;
            const uint32_t begin = a.offsets[g], end = a.offsets[g + 1];
            const uint32_t nchunks = end > begin ? (end - begin + C::N - 1) / C::N : 1u;
            for (uint32_t ch = 0; ch < nchunks; ++ch, ++c) {
                const int s = (int)(c % C::STAGES);
                // prefetch this lane's splat before waiting for the stage
                const uint32_t e = begin + ch * C::N + (uint32_t)lane;
                const bool valid = lane < C::N && e < end;
                float4 mc = make_float4(0, 0, 0, 0), co = mc, col = mc;
                if (valid) {
                    const uint32_t idx = a.list[e];
                    mc = a.proj.mc[idx];
                    co = a.proj.co[idx];
                    col = a.proj.col[idx];
                }
                if (c >= (uint32_t)C::STAGES) {
                    ptx::mbar_wait(&sm.done[s], ((c / C::STAGES) - 1) & 1);
                    const int alive = sm.alive[s];
                    __syncwarp();
                    if (lane == 0) sm.alive[s] = 0;
                    // chunk c-STAGES belonged to this group and left nothing alive: retire
                    if (ch >= (uint32_t)C::STAGES && !alive) break;
                }
                // per-tile coefficient rows of this lane's splat
                int tx0 = 0, ty0 = 0, tx1 = -1, ty1 = -1;
                float c_o = 0.0f;
                if (valid) {
                    tile_rect(mc.x, mc.y, __float_as_int(co.w), gg.tiles_x, gg.tiles_y, tx0, ty0, tx1, ty1);
                    c_o = fminf(a.alpha_clamp, co.y);
                }
                const bool can = valid && !(c_o < L);
                const double qa = mc.z, qb = mc.w, qc = co.x;
                const double lo2 = can ? (double)lg2_approx(co.y) : 0.0;
#pragma unroll
                for (int t = 0; t < C::TILES; ++t) {
                    const int tcx = gx * G + (t % G), tcy = gy * G + (t / G);
                    float w[6];
                    bool row_ok = can && tcx >= tx0 && tcx <= tx1 && tcy >= ty0 && tcy <= ty1;
                    if (row_ok) {
                        const double mx = (double)mc.x - (double)(tcx * kTile + 8);
                        const double my = (double)mc.y - (double)(tcy * kTile + 8);
                        const double L2E = 1.4426950408889634;
                        w[0] = (float)(-0.5 * qa * L2E);
                        w[1] = (float)(-qb * L2E);
                        w[2] = (float)(-0.5 * qc * L2E);
                        w[3] = (float)((qa * mx + qb * my) * L2E);
                        w[4] = (float)((qb * mx + qc * my) * L2E);
                        w[5] = (float)(-(0.5 * qa * mx * mx + qb * mx * my + 0.5 * qc * my * my) * L2E + lo2);
#pragma unroll
                        for (int k = 0; k < 6; ++k) row_ok = row_ok && fabsf(w[k]) <= 16384.0f;
                    }
                    uint4 r0, r1;
                    if (row_ok) {
                        float h[6], l[6];
#pragma unroll
                        for (int k = 0; k < 6; ++k) {
                            h[k] = __half2float(__float2half_rn(w[k]));
                            l[k] = w[k] - h[k];
                        }
                        r0.x = pack_half2(h[0], h[1]);
                        r0.y = pack_half2(h[2], h[3]);
                        r0.z = pack_half2(h[4], h[5]);
                        r0.w = pack_half2(l[0], l[1]);
                        r1.x = pack_half2(l[2], l[3]);
                        r1.y = pack_half2(l[4], l[5]);
                    } else {
                        r0.x = 0u;
                        r0.y = 0u;
                        r0.z = pack_half2(0.0f, kNeverRow);
                        r0.w = 0u;
                        r1.x = 0u;
                        r1.y = 0u;
                    }
                    r1.z = 0u;
                    r1.w = 0u;
                    if (lane < C::N) {
                        *reinterpret_cast<uint4*>(&sm.b[s][t][core_off(lane, 0)]) = r0;
                        *reinterpret_cast<uint4*>(&sm.b[s][t][core_off(lane, 1)]) = r1;
                    }
                }
                if (lane < C::N) sm.epi[s][lane] = make_float4(col.x, col.y, col.z, c_o);
                if (lane == 0) {
                    sm.hdr[s].gid = g;
                    sm.hdr[s].n_valid = (int)min((uint32_t)C::N, end > begin + ch * C::N ? end - begin - ch * C::N : 0u);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&sm.full[s]);
            }
        }
        // end of stream
        const int s = (int)(c % C::STAGES);
        if (c >= (uint32_t)C::STAGES) ptx::mbar_wait(&sm.done[s], ((c / C::STAGES) - 1) & 1);
        if (lane == 0) {
            sm.hdr[s].gid = -1;
            sm.hdr[s].n_valid = 0;
            ptx::mbar_arrive(&sm.full[s]);
        }
        __syncwarp();
    } else if (warp == C::EPI + 1) {
        // ================================ MMA issuer ==========================================
        constexpr uint32_t idesc = ptx::idesc_f16(128, C::N);
        const uint32_t a_base = ptx::smem_u32(sm.a);
        for (uint32_t c = 0;; ++c) {
            const int s = (int)(c % C::STAGES);
            ptx::mbar_wait(&sm.full[s], (c / C::STAGES) & 1);
            ptx::tc_fence_after();
            const ChunkHeader h = sm.hdr[s];
            if (lane == 0) {
                if (h.gid >= 0 && h.n_valid > 0) {
#pragma unroll
                    for (int m = 0; m < C::MT; ++m) {
                        const uint64_t ad = ptx::smem_desc(a_base + (uint32_t)(m & 1) * 4096u, 128, 256);
                        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(&sm.b[s][m >> 1][0]), 128, 256);
                        ptx::mma_f16_ss(tmem + (uint32_t)(s * C::MT * C::N + m * C::N), ad, bd, idesc, 0u);
                    }
                    ptx::mma_commit(&sm.tfull[s]);
                } else {
                    ptx::mbar_arrive(&sm.tfull[s]);
                }
            }
            __syncwarp();
            if (h.gid < 0) break;
        }
    } else {
        // ================================ epilogue ============================================
        const int q = warp & 3;  // TMEM lane quadrant of this warp
        int mtile[C::PPT];
        int prow[C::PPT], pcol[C::PPT];
#pragma unroll
        for (int k = 0; k < C::PPT; ++k) {
            mtile[k] = (warp >> 2) + k * (C::EPI / 4);
            const int p = (mtile[k] & 1) * 128 + q * 32 + lane;  // pixel within its tile
            prow[k] = p >> 4;
            pcol[k] = p & 15;
        }
        float T[C::PPT], cr[C::PPT], cg[C::PPT], cb[C::PPT], thr[C::PPT];
        int px[C::PPT], py[C::PPT];
        bool inside[C::PPT];
        const float L = log2f(a.alpha_skip);
        int cur = -1;
        for (uint32_t c = 0;; ++c) {
            const int s = (int)(c % C::STAGES);
            ptx::mbar_wait(&sm.tfull[s], (c / C::STAGES) & 1);
            ptx::tc_fence_after();
            const ChunkHeader h = sm.hdr[s];
            if (h.gid != cur) {
                if (cur >= 0) {
#pragma unroll
                    for (int k = 0; k < C::PPT; ++k)
                        if (inside[k]) {
                            float* o = a.image + ((size_t)(py[k] - a.image_row0) * gg.width + px[k]) * 3;
                            o[0] = fminf(fmaxf(cr[k], 0.0f), 1.0f);
                            o[1] = fminf(fmaxf(cg[k], 0.0f), 1.0f);
                            o[2] = fminf(fmaxf(cb[k], 0.0f), 1.0f);
                        }
                }
                if (h.gid < 0) break;
                cur = h.gid;
                const int gx = cur % gg.groups_x, gy = cur / gg.groups_x + gg.band_gy0;
#pragma unroll
                for (int k = 0; k < C::PPT; ++k) {
                    const int t = mtile[k] >> 1;
                    const int tx = gx * G + (t % G), ty = gy * G + (t / G);
                    px[k] = tx * kTile + pcol[k];
                    py[k] = ty * kTile + prow[k];
                    inside[k] = tx < gg.tiles_x && ty < gg.tiles_y && px[k] < gg.width && py[k] < gg.height;
                    T[k] = 1.0f;
                    cr[k] = cg[k] = cb[k] = 0.0f;
                    thr[k] = inside[k] ? L : kInf;
                }
            }
            bool any = false;
#pragma unroll
            for (int k = 0; k < C::PPT; ++k) any = any || thr[k] != kInf;
            const bool warp_alive = __any_sync(0xffffffffu, any);
            if (h.n_valid > 0 && warp_alive) {
                constexpr int PP = C::PPT >= 2 ? 2 : 1;  // pixels blended together (ILP)
#pragma unroll
                for (int k0 = 0; k0 < C::PPT; k0 += PP) {
                    uint32_t d[PP][C::N];
#pragma unroll
                    for (int kk = 0; kk < PP; ++kk) {
                        const uint32_t col0 = (uint32_t)(s * C::MT * C::N + mtile[k0 + kk] * C::N);
#pragma unroll
                        for (int j0 = 0; j0 < C::N; j0 += 16)
                            ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + col0 + j0, &d[kk][j0]);
                    }
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int kk = 0; kk < PP; ++kk)
#pragma unroll
                        for (int j0 = 0; j0 < C::N; j0 += 16) ptx::reg_fence16(&d[kk][j0]);
#pragma unroll
                    for (int j = 0; j < C::N; ++j) {
                        const float4 ej = sm.epi[s][j];
#pragma unroll
                        for (int kk = 0; kk < PP; ++kk) {
                            const int k = k0 + kk;
                            const float dv = __uint_as_float(d[kk][j]);
                            if (dv >= thr[k]) {
                                const float al = fminf(ej.w, ex2_approx(dv));
                                const float wt = T[k] * al;
                                cr[k] = fmaf(wt, ej.x, cr[k]);
                                cg[k] = fmaf(wt, ej.y, cg[k]);
                                cb[k] = fmaf(wt, ej.z, cb[k]);
                                T[k] = T[k] - wt;
                                if (T[k] < a.t_terminate) thr[k] = kInf;
                            }
                        }
                    }
                }
            }
            any = false;
#pragma unroll
            for (int k = 0; k < C::PPT; ++k) any = any || thr[k] != kInf;
            const bool still = __any_sync(0xffffffffu, any);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (still) sm.alive[s] = 1;
                ptx::mbar_arrive(&sm.done[s]);
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == C::EPI + 1) ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
}

template <int G>
void launch_g(const RasterArgs& a, int num_sms, cudaStream_t st) {
    using C = Cfg<G>;
    // Dynamic smem is padded so that exactly CTAS_PER_SM CTAs fit on an SM: TMEM columns are the
    // binding resource and a CTA that cannot allocate would otherwise spin.
    size_t smem = sizeof(Smem<G>) + 1024;
    const size_t min_smem = (size_t)(228 * 1024) / (C::CTAS_PER_SM + 1) + 1024;
    if (smem < min_smem) smem = min_smem;
    cudaFuncSetAttribute(raster_tensor_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int n = a.gg.n_groups_band;
    int grid = num_sms * C::CTAS_PER_SM;
    if (grid > n) grid = n;
    if (grid > 0) raster_tensor_kernel<G><<<grid, C::THREADS, smem, st>>>(a);
}

}  // namespace

void launch_raster_tensor(const RasterArgs& a, int num_sms, cudaStream_t st) {
    if (a.gg.g == 1)
        launch_g<1>(a, num_sms, st);
    else if (a.gg.g == 2)
        launch_g<2>(a, num_sms, st);
    else
        launch_g<4>(a, num_sms, st);
}

}  // namespace tgs

// ---- self-test hook: one M=128 x N=32 x K=16 tcgen05.mma through the same descriptors --------
namespace tgs {
namespace {
__global__ void __launch_bounds__(128, 1) debug_mma_kernel(const uint16_t* __restrict__ a,
                                                            const uint16_t* __restrict__ b,
                                                            float* __restrict__ d) {
    __shared__ __align__(1024) uint8_t sa[128 * 32];
    __shared__ __align__(1024) uint8_t sb[32 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    // row t of A (16 halves) -> core-matrix layout
    for (int kh = 0; kh < 2; ++kh) {
        uint4 v = *reinterpret_cast<const uint4*>(a + t * 16 + kh * 8);
        *reinterpret_cast<uint4*>(sa + core_off(t, kh)) = v;
        if (t < 32) {
            uint4 w = *reinterpret_cast<const uint4*>(b + t * 16 + kh * 8);
            *reinterpret_cast<uint4*>(sb + core_off(t, kh)) = w;
        }
    }
    if (t == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_fence_init();
    }
    if (warp == 0) ptx::tmem_alloc<32>(&tbase);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    if (t == 0) {
        ptx::mma_f16_ss(tm, ptx::smem_desc(ptx::smem_u32(sa), 128, 256), ptx::smem_desc(ptx::smem_u32(sb), 128, 256),
                        ptx::idesc_f16(128, 32), 0u);
        ptx::mma_commit(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    uint32_t r[32];
    ptx::tmem_ld16(tm + ((uint32_t)(warp * 32) << 16), r);
    ptx::tmem_ld16(tm + ((uint32_t)(warp * 32) << 16) + 16, r + 16);
    ptx::tmem_wait_ld();
    ptx::reg_fence16(r);
    ptx::reg_fence16(r + 16);
    for (int j = 0; j < 32; ++j) d[t * 32 + j] = __uint_as_float(r[j]);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc<32>(tm);
    (void)lane;
}
}  // namespace

void launch_debug_mma(const uint16_t* a, const uint16_t* b, float* d, cudaStream_t st) {
    debug_mma_kernel<<<1, 128, 0, st>>>(a, b, d);
}
}  // namespace tgs
