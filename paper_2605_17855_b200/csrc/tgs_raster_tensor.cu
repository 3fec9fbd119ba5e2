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
    static constexpr int TS = (G == 4) ? 1 : 2;               // TMEM accumulator stages
    static constexpr int SS = 3;                              // smem (operand + epilogue data) stages
    static constexpr int COLS_USED = TS * MT * N;
    static constexpr int TMEM_COLS = COLS_USED <= 32 ? 32 : COLS_USED <= 64 ? 64 : COLS_USED <= 128 ? 128
                                     : COLS_USED <= 256 ? 256 : 512;
    static constexpr int EPI = (G == 1) ? 4 : (G == 2) ? 8 : 16;  // epilogue warps
    static constexpr int PPT = MT * 4 / EPI;                  // pixels per epilogue thread (2, 4, 8)
    static constexpr int PB = PPT < 4 ? PPT : 4;              // pixels blended together (ILP)
    static constexpr int JB = 32 / PB;                        // splat columns per TMEM load block
    static constexpr int PROD = (G == 1) ? 1 : 4;             // producer warps
    static constexpr int TPP = TILES / PROD;                  // tiles per producer warp
    static constexpr int THREADS = (EPI + PROD + 1) * 32;
    static constexpr int CTAS_PER_SM = 512 / TMEM_COLS;
    static constexpr int B_BYTES = N * 32;                    // one tile's B operand
};

struct ChunkHeader {
    int gid;      // band-local group id, -1 = end of stream
    int n_valid;  // splats in the chunk (0: empty group)
};

template <int G>
struct Smem {
    alignas(128) uint8_t a[256 * 32];                                     // pixel monomials
    alignas(128) uint8_t b[Cfg<G>::SS][Cfg<G>::TILES][Cfg<G>::B_BYTES];   // splat rows
    float4 epi[Cfg<G>::SS][Cfg<G>::N];                                    // r, g, b, min(clamp, o)
    ChunkHeader hdr[Cfg<G>::SS];
    int alive_tag[Cfg<G>::SS];        // max over epilogue warps of (chunk << 1 | any pixel alive)
    int gq[2];                        // group ticket broadcast to producer warps
    uint64_t full[Cfg<G>::SS];        // producers -> MMA          (count PROD)
    uint64_t done[Cfg<G>::SS];        // epilogue -> producers     (count EPI): smem stage reusable
    uint64_t tfull[Cfg<G>::TS];       // MMA -> epilogue           (tcgen05.commit)
    uint64_t tempty[Cfg<G>::TS];      // epilogue -> MMA           (count EPI): TMEM stage drained
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

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Coefficient row of one splat for one tile (centre (ox, oy)) as FP16 hi/lo halves.
__device__ __forceinline__ void make_row(bool ok, float mx, float my, float qa, float qb, float qc, float lo2,
                                         float ox, float oy, uint4& r0, uint4& r1) {
    float w[6];
    if (ok) {
        const float dx = mx - ox, dy = my - oy;
        const float ha = 0.5f * qa, hc = 0.5f * qc;
        w[0] = -ha * kLog2e;
        w[1] = -qb * kLog2e;
        w[2] = -hc * kLog2e;
        w[3] = fmaf(qa, dx, qb * dy) * kLog2e;
        w[4] = fmaf(qb, dx, qc * dy) * kLog2e;
        const float quad = fmaf(ha * dx, dx, fmaf(qb * dx, dy, hc * dy * dy));
        w[5] = fmaf(-quad, kLog2e, lo2);
#pragma unroll
        for (int k = 0; k < 6; ++k) ok = ok && fabsf(w[k]) <= 16384.0f;
    }
    if (ok) {
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
        r0 = make_uint4(0u, 0u, pack_half2(0.0f, kNeverRow), 0u);
        r1.x = 0u;
        r1.y = 0u;
    }
    r1.z = 0u;
    r1.w = 0u;
}

template <int G>
__global__ void __launch_bounds__(Cfg<G>::THREADS, 1) raster_tensor_kernel(RasterArgs a) {
    using C = Cfg<G>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem<G>& sm = *reinterpret_cast<Smem<G>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const GroupGeom& gg = a.gg;
    const int n_groups = gg.n_groups_band;
    constexpr int kProd0 = C::EPI, kMma = C::EPI + C::PROD;

    // ---- setup: A operand, barriers, TMEM ----------------------------------------------------
    for (int p = threadIdx.x; p < 256; p += blockDim.x) {
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
        for (int s = 0; s < C::SS; ++s) {
            ptx::mbar_init(&sm.full[s], C::PROD);
            ptx::mbar_init(&sm.done[s], C::EPI);
            sm.alive_tag[s] = -1;
        }
        for (int s = 0; s < C::TS; ++s) {
            ptx::mbar_init(&sm.tfull[s], 1);
            ptx::mbar_init(&sm.tempty[s], C::EPI);
        }
        ptx::mbar_fence_init();
    }
    if (warp == kMma) ptx::tmem_alloc<C::TMEM_COLS>(&sm.tmem_base);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp >= kProd0 && warp < kMma) {
        // ================================ producers ==========================================
        // Producer warp p builds the coefficient rows of tiles [p*TPP, (p+1)*TPP) for all N splats
        // of the chunk (lane = splat); warp 0 also writes the epilogue data and the header.
        const int p = warp - kProd0;
        const float skip = a.alpha_skip;
        uint32_t c = 0;
        int slot = 0;
        for (;;) {
            if (p == 0 && lane == 0) {
                const int t = (int)atomicAdd(&a.fc->group_counter, 1u);
                sm.gq[slot] = t < n_groups ? (a.order ? a.order[t] : t) : -1;
            }
            if (C::PROD > 1) named_bar_sync(1, C::PROD * 32); else __syncwarp();
            const int g = sm.gq[slot];
            slot ^= 1;
            if (g < 0) break;
            const int gx = g % gg.groups_x, gy = g / gg.groups_x + gg.band_gy0;
            const uint32_t begin = a.offsets[g], end = a.offsets[g + 1];
            const uint32_t nchunks = end > begin ? (end - begin + C::N - 1) / C::N : 1u;
            for (uint32_t ch = 0; ch < nchunks; ++ch, ++c) {
                const int s = (int)(c % C::SS);
                const uint32_t e = begin + ch * C::N + (uint32_t)lane;
                const bool valid = lane < C::N && e < end;
                float4 mc = make_float4(0, 0, 0, 0), co = mc, col = mc;
                if (valid) {
                    const uint32_t idx = a.list[e];
                    mc = a.proj.mc[idx];
                    co = a.proj.co[idx];
                    if (p == 0) col = a.proj.col[idx];
                }
                if (c >= (uint32_t)C::SS) {
                    ptx::mbar_wait(&sm.done[s], ((c / C::SS) - 1) & 1);
                    const int tag = sm.alive_tag[s];
                    // the last chunk of this group in this stage left no pixel alive: retire
                    if (ch >= (uint32_t)C::SS && tag == (int)((c - C::SS) << 1)) break;
                }
                int tx0 = 0, ty0 = 0, tx1 = -1, ty1 = -1;
                float c_o = 0.0f, lo2 = 0.0f;
                if (valid) {
                    tile_rect(mc.x, mc.y, __float_as_int(co.w), gg.tiles_x, gg.tiles_y, tx0, ty0, tx1, ty1);
                    c_o = fminf(a.alpha_clamp, co.y);
                    lo2 = lg2_approx(co.y);
                }
                const bool can = valid && !(c_o < skip);
#pragma unroll
                for (int tt = 0; tt < C::TPP; ++tt) {
                    const int t = p * C::TPP + tt;
                    const int tcx = gx * G + (t % G), tcy = gy * G + (t / G);
                    const bool row_ok = can && tcx >= tx0 && tcx <= tx1 && tcy >= ty0 && tcy <= ty1;
                    uint4 r0, r1;
                    make_row(row_ok, mc.x, mc.y, mc.z, mc.w, co.x, lo2, (float)(tcx * kTile + 8),
                             (float)(tcy * kTile + 8), r0, r1);
                    if (lane < C::N) {
                        *reinterpret_cast<uint4*>(&sm.b[s][t][core_off(lane, 0)]) = r0;
                        *reinterpret_cast<uint4*>(&sm.b[s][t][core_off(lane, 1)]) = r1;
                    }
                }
                if (p == 0) {
                    if (lane < C::N) sm.epi[s][lane] = make_float4(col.x, col.y, col.z, c_o);
                    if (lane == 0) {
                        sm.hdr[s].gid = g;
                        sm.hdr[s].n_valid =
                            (int)min((uint32_t)C::N, end > begin + ch * C::N ? end - begin - ch * C::N : 0u);
                    }
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&sm.full[s]);
            }
        }
        // end of stream
        const int s = (int)(c % C::SS);
        if (c >= (uint32_t)C::SS) ptx::mbar_wait(&sm.done[s], ((c / C::SS) - 1) & 1);
        if (lane == 0) {
            if (p == 0) {
                sm.hdr[s].gid = -1;
                sm.hdr[s].n_valid = 0;
            }
            ptx::mbar_arrive(&sm.full[s]);
        }
        __syncwarp();
    } else if (warp == kMma) {
        // ================================ MMA issuer ==========================================
        constexpr uint32_t idesc = ptx::idesc_f16(128, C::N);
        const uint32_t a_base = ptx::smem_u32(sm.a);
        for (uint32_t c = 0;; ++c) {
            const int s = (int)(c % C::SS), ts = (int)(c % C::TS);
            ptx::mbar_wait(&sm.full[s], (c / C::SS) & 1);
            if (c >= (uint32_t)C::TS) ptx::mbar_wait(&sm.tempty[ts], ((c / C::TS) - 1) & 1);
            ptx::tc_fence_after();
            const ChunkHeader h = sm.hdr[s];
            if (lane == 0) {
                if (h.gid >= 0 && h.n_valid > 0) {
#pragma unroll
                    for (int m = 0; m < C::MT; ++m) {
                        const uint64_t ad = ptx::smem_desc(a_base + (uint32_t)(m & 1) * 4096u, 128, 256);
                        const uint64_t bd = ptx::smem_desc(ptx::smem_u32(&sm.b[s][m >> 1][0]), 128, 256);
                        ptx::mma_f16_ss(tmem + (uint32_t)(ts * C::MT * C::N + m * C::N), ad, bd, idesc, 0u);
                    }
                    ptx::mma_commit(&sm.tfull[ts]);
                } else {
                    ptx::mbar_arrive(&sm.tfull[ts]);
                }
            }
            __syncwarp();
            if (h.gid < 0) break;
        }
    } else {
        // ================================ epilogue ============================================
        // warp w: TMEM lane quadrant q = w % 4; M-tiles m_k = w/4 + k * EPI/4 (k < PPT), which for
        // G = 2 gives every thread one pixel in each of the 4 member tiles (balanced work per warp,
        // PB = 4 independent blend chains per thread).
        const int q = warp & 3;
        const int mg = warp >> 2;
        int prow[C::PPT], pcol[C::PPT], ptile[C::PPT], pm[C::PPT];
#pragma unroll
        for (int k = 0; k < C::PPT; ++k) {
            const int m = mg + k * (C::EPI / 4);
            const int pix = (m & 1) * 128 + q * 32 + lane;  // pixel within its tile
            pm[k] = m;
            prow[k] = pix >> 4;
            pcol[k] = pix & 15;
            ptile[k] = m >> 1;
        }
        float T[C::PPT], cr[C::PPT], cg[C::PPT], cb[C::PPT], thr[C::PPT];
        int px[C::PPT], py[C::PPT];
        bool inside[C::PPT];
        const float L = log2f(a.alpha_skip);
        const float tterm = a.t_terminate;
        int cur = -1;
        for (uint32_t c = 0;; ++c) {
            const int s = (int)(c % C::SS), ts = (int)(c % C::TS);
            ptx::mbar_wait(&sm.tfull[ts], (c / C::TS) & 1);
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
                    const int t = ptile[k];
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
            const bool work = h.n_valid > 0 && __any_sync(0xffffffffu, any);
            const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ts * C::MT * C::N);
            // D is consumed in blocks of PB pixels x JB splats (32 registers); the TMEM stage is
            // released as soon as the warp's last block is in registers.
            constexpr int NBLK = (C::PPT / C::PB) * (C::N / C::JB);
#pragma unroll
            for (int blk = 0; blk < NBLK; ++blk) {
                const int k0 = (blk / (C::N / C::JB)) * C::PB;
                const int j0 = (blk % (C::N / C::JB)) * C::JB;
                uint32_t d[C::PB][C::JB];
                if (work) {
#pragma unroll
                    for (int kk = 0; kk < C::PB; ++kk) {
                        const uint32_t ad = lane_base + (uint32_t)(pm[k0 + kk] * C::N + j0);
                        if constexpr (C::JB == 16) ptx::tmem_ld16(ad, d[kk]); else ptx::tmem_ld8(ad, d[kk]);
                    }
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int kk = 0; kk < C::PB; ++kk) {
                        if constexpr (C::JB == 16) ptx::reg_fence16(d[kk]); else ptx::reg_fence8(d[kk]);
                    }
                }
                if (blk == NBLK - 1) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&sm.tempty[ts]);
                }
                if (!work) continue;
                // Speculative pass: blend every splat with D >= thr without the per-splat
                // termination test (no loop-carried compare chain); T only decreases, so
                // T_end < t_terminate <=> the pixel terminated inside this block, in which case
                // the block is replayed exactly below (at most once per pixel per group).
                float T0[C::PB], r0[C::PB], g0[C::PB], b0[C::PB];
#pragma unroll
                for (int kk = 0; kk < C::PB; ++kk) {
                    T0[kk] = T[k0 + kk];
                    r0[kk] = cr[k0 + kk];
                    g0[kk] = cg[k0 + kk];
                    b0[kk] = cb[k0 + kk];
                }
#pragma unroll
                for (int jj = 0; jj < C::JB; ++jj) {
                    bool tk[C::PB], anyt = false;
#pragma unroll
                    for (int kk = 0; kk < C::PB; ++kk) {
                        tk[kk] = __uint_as_float(d[kk][jj]) >= thr[k0 + kk];
                        anyt = anyt || tk[kk];
                    }
                    if (anyt) {
                        const float4 ej = sm.epi[s][j0 + jj];
#pragma unroll
                        for (int kk = 0; kk < C::PB; ++kk) {
                            const int k = k0 + kk;
                            const float al = tk[kk] ? fminf(ej.w, ex2_approx(__uint_as_float(d[kk][jj]))) : 0.0f;
                            const float wt = T[k] * al;
                            cr[k] = fmaf(wt, ej.x, cr[k]);
                            cg[k] = fmaf(wt, ej.y, cg[k]);
                            cb[k] = fmaf(wt, ej.z, cb[k]);
                            T[k] -= wt;
                        }
                    }
                }
#pragma unroll
                for (int kk = 0; kk < C::PB; ++kk) {
                    const int k = k0 + kk;
                    if (T[k] < tterm) {  // terminated inside the block: exact replay
                        T[k] = T0[kk];
                        cr[k] = r0[kk];
                        cg[k] = g0[kk];
                        cb[k] = b0[kk];
                        bool stop = false;
#pragma unroll
                        for (int jj = 0; jj < C::JB; ++jj) {
                            const float dv = __uint_as_float(d[kk][jj]);
                            if (!stop && dv >= thr[k]) {
                                const float4 ej = sm.epi[s][j0 + jj];
                                const float wt = T[k] * fminf(ej.w, ex2_approx(dv));
                                cr[k] = fmaf(wt, ej.x, cr[k]);
                                cg[k] = fmaf(wt, ej.y, cg[k]);
                                cb[k] = fmaf(wt, ej.z, cb[k]);
                                T[k] -= wt;
                                stop = T[k] < tterm;
                            }
                        }
                        thr[k] = kInf;
                    }
                }
            }
            any = false;
#pragma unroll
            for (int k = 0; k < C::PPT; ++k) any = any || thr[k] != kInf;
            const bool still = __any_sync(0xffffffffu, any);
            __syncwarp();
            if (lane == 0) {
                atomicMax(&sm.alive_tag[s], (int)((c << 1) | (still ? 1u : 0u)));
                ptx::mbar_arrive(&sm.done[s]);
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == kMma) ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
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
