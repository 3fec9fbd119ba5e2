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
// CTA = one 16x16 tile at a time, persistent over tiles (longest group lists first), several CTAs
// per SM so the hardware balances tiles of unequal depth:
//   warps 0-3  epilogue: TMEM lane quadrant q = warp; each thread owns two pixels of the tile
//              (rows 2q + lane/16 and 8 + 2q + lane/16), tcgen05.ld's its D rows and runs the
//              ordered blend on CUDA cores + MUFU ex2;
//   warp 4     producer: streams the tile's G x G group list (north_star 4: group lists are
//              G^2-fold shorter to bin and sort, reference binning.cpp:46-74), gathers 32 splats
//              per step, keeps those whose mask has this tile (warp ballot compaction, so no MMA
//              column or blend slot is spent on another tile's splats), derives the
//              tile-centred coefficient rows (FP16 hi/lo) into smem;
//   warp 5     TMEM owner + MMA issuer: two tcgen05.mma (M=128 pixels, N=32 splats, K=16) per
//              chunk, tcgen05.commit -> epilogue.
// A (pixel monomials) is identical for every tile, built once per CTA (256 rows x 32 B).
// Chunks flow through SS smem stages and one TMEM stage (drained into registers before the
// blend, so the next MMA overlaps it), guarded by mbarriers; chunk headers carry the tile, so
// tile boundaries need no extra synchronisation.  A tile retires as soon as its 4 epilogue warps
// report all pixels terminated.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"
#include "tgs_ptx.cuh"

#include <algorithm>

namespace tgs {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kNeverRow = -30000.0f;
constexpr float kInf = __builtin_huge_valf();

constexpr int kN = 32;          // splats per chunk (MMA N)
constexpr int kSS = 4;          // smem stages
constexpr int kEpi = 4;         // epilogue warps
constexpr int kThreads = (kEpi + 2) * 32;
constexpr int kTS = 2;          // TMEM accumulator stages
constexpr int kTmemCols = 128;  // kTS x 2 M-tiles x 32 columns
constexpr int kCtasPerSm = 4;

struct ChunkHeader {
    int seq;      // per-CTA tile sequence number, -1 = end of stream
    int tile;     // band-local tile index
    int n_valid;  // splats in the chunk (0: tile without contributing splats)
};

struct Smem {
    alignas(128) uint8_t a[256 * 32];      // pixel monomials (both M-tiles)
    alignas(128) uint8_t b[kSS][kN * 32];  // splat coefficient rows
    float4 epi[kSS][kN];                   // r, g, b, min(alpha_clamp, opacity)
    ChunkHeader hdr[kSS];
    int dead_seq[kEpi];                    // last tile seq whose pixels (per warp) all terminated
    uint64_t full[kSS];                    // producer -> MMA
    uint64_t done[kSS];                    // epilogue -> producer (count kEpi)
    uint64_t tfull[kTS];                   // MMA -> epilogue (tcgen05.commit)
    uint64_t tempty[kTS];                  // epilogue -> MMA (count kEpi)
    uint32_t tmem_base;
};

// Pixel owned by TMEM lane l (0..127) of M-tile m (0/1): epilogue warp q = l/32 owns the 8x8
// quadrant (q%2, q/2) of the tile, lane j = l%32 the column j%8 of rows 4m + j/8 inside it, so a
// thread's two pixels are 4 rows apart and a splat footprint touches as few warps as possible.
__device__ __forceinline__ int lane_pixel(int m, int l) {
    const int q = l >> 5, j = l & 31;
    const int x = (q & 1) * 8 + (j & 7);
    const int y = (q >> 1) * 8 + m * 4 + (j >> 3);
    return y * 16 + x;
}

// byte offset of (row, k-half) in a K-major no-swizzle operand: 8x16B core matrices
__device__ __forceinline__ uint32_t core_off(int row, int khalf) {
    return (uint32_t)((row >> 3) * 256 + khalf * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// Coefficient row of one splat for the tile centred at (ox, oy), as FP16 hi/lo halves.
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

__device__ __forceinline__ void write_row(Smem& sm, int s, int slot, const uint4& r0, const uint4& r1) {
    *reinterpret_cast<uint4*>(&sm.b[s][core_off(slot, 0)]) = r0;
    *reinterpret_cast<uint4*>(&sm.b[s][core_off(slot, 1)]) = r1;
}

__global__ void __launch_bounds__(kThreads, kCtasPerSm) raster_tensor_kernel(RasterArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const GroupGeom& gg = a.gg;
    const int G = gg.g;
    const int trow0 = gg.band_gy0 * G;                                  // first tile row of the band
    const int trows = min(gg.tiles_y, gg.band_gy1 * G) - trow0;
    const int n_tiles = gg.tiles_x * trows;
    constexpr int kProd = kEpi, kMma = kEpi + 1;

    // ---- setup: A operand, barriers, TMEM ----------------------------------------------------
    for (int p = threadIdx.x; p < 256; p += blockDim.x) {
        const int pix = lane_pixel(p >> 7, p & 127);  // A row p feeds TMEM lane p%128 of M-tile p/128
        const float ux = (float)(pix & 15) - 7.5f, uy = (float)(pix >> 4) - 7.5f;
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
        for (int s = 0; s < kSS; ++s) {
            ptx::mbar_init(&sm.full[s], 1);
            ptx::mbar_init(&sm.done[s], kEpi);
        }
        for (int s = 0; s < kTS; ++s) {
            ptx::mbar_init(&sm.tfull[s], 1);
            ptx::mbar_init(&sm.tempty[s], kEpi);
        }
        for (int w = 0; w < kEpi; ++w) sm.dead_seq[w] = -1;
        ptx::mbar_fence_init();
    }
    if (warp == kMma) ptx::tmem_alloc<kTmemCols>(&sm.tmem_base);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == kProd) {
        // ================================ producer ===========================================
        const float skip = a.alpha_skip;
        uint32_t c = 0;     // chunks emitted so far
        int seq = 0;        // tiles started by this CTA
        const uint32_t lt = (1u << lane) - 1u;
        for (;; ++seq) {
            int t = 0;
            if (lane == 0) t = (int)atomicAdd(&a.fc->group_counter, 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n_tiles) break;
            const int tile = a.order ? a.order[t] : t;
            const int tx = tile % gg.tiles_x, ty = tile / gg.tiles_x + trow0;
            const int gid = (ty / G - gg.band_gy0) * gg.groups_x + tx / G;
            const uint32_t begin = a.offsets[gid], end = a.offsets[gid + 1];
            const float ox = (float)(tx * kTile + 8), oy = (float)(ty * kTile + 8);
            int fill = 0;                 // rows placed in the open chunk
            bool open = false;            // a stage is open for this tile
            bool emitted = false;         // at least one chunk of this tile emitted
            int s = 0;
            // Software-pipelined gather: list indices two batches ahead, splat records one
            // batch ahead, so the dependent idx -> record loads overlap the row building.
            const uint32_t nb = (end - begin + 31u) / 32u;
            auto ld_idx = [&](uint32_t b) -> uint32_t {
                const uint32_t e = begin + b * 32u + (uint32_t)lane;
                return (b < nb && e < end) ? __ldg(&a.list[e]) : 0xffffffffu;
            };
            struct Rec { float4 mc, co, col; uint32_t idx; };
            auto ld_rec = [&](uint32_t idx) -> Rec {
                Rec r;
                r.idx = idx;
                if (idx != 0xffffffffu) {
                    r.mc = __ldg(&a.proj.mc[idx]);
                    r.co = __ldg(&a.proj.co[idx]);
                    r.col = __ldg(&a.proj.col[idx]);
                } else {
                    r.mc = r.co = r.col = make_float4(0, 0, 0, 0);
                }
                return r;
            };
            uint32_t idx_next2 = ld_idx(1);
            Rec nxt = ld_rec(ld_idx(0));
            for (uint32_t bi = 0; bi < nb; ++bi) {
                const Rec cur = nxt;
                nxt = ld_rec(idx_next2);
                idx_next2 = ld_idx(bi + 2);
                // retire as soon as every epilogue warp reported the tile terminated
                if (emitted) {
                    int dmin = ((volatile int*)sm.dead_seq)[0];
#pragma unroll
                    for (int w = 1; w < kEpi; ++w) dmin = min(dmin, ((volatile int*)sm.dead_seq)[w]);
                    if (dmin >= seq) break;
                }
                bool keep = false;
                if (cur.idx != 0xffffffffu) {
                    int x0, y0, x1, y1;
                    tile_rect(cur.mc.x, cur.mc.y, __float_as_int(cur.co.w), gg.tiles_x, gg.tiles_y, x0, y0, x1, y1);
                    keep = tx >= x0 && tx <= x1 && ty >= y0 && ty <= y1 && !(fminf(a.alpha_clamp, cur.co.y) < skip);
                }
                const uint32_t km = __ballot_sync(0xffffffffu, keep);
                if (km == 0u) continue;
                const int nk = __popc(km);
                const int rank = __popc(km & lt);
                uint4 r0, r1;
                float4 epi_v = make_float4(0, 0, 0, 0);
                if (keep) {
                    make_row(true, cur.mc.x, cur.mc.y, cur.mc.z, cur.mc.w, cur.co.x, lg2_approx(cur.co.y), ox, oy,
                             r0, r1);
                    epi_v = make_float4(cur.col.x, cur.col.y, cur.col.z, fminf(a.alpha_clamp, cur.co.y));
                }
                if (!open) {
                    s = (int)(c % kSS);
                    if (c >= (uint32_t)kSS) ptx::mbar_wait(&sm.done[s], ((c / kSS) - 1) & 1);
                    open = true;
                    fill = 0;
                }
                const int room = kN - fill;
                if (keep && rank < room) {
                    write_row(sm, s, fill + rank, r0, r1);
                    sm.epi[s][fill + rank] = epi_v;
                }
                if (nk >= room) {
                    // chunk full: publish it and open the next one for the remaining ranks
                    if (lane == 0) {
                        sm.hdr[s].seq = seq;
                        sm.hdr[s].tile = tile;
                        sm.hdr[s].n_valid = kN;
                    }
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&sm.full[s]);
                    ++c;
                    emitted = true;
                    s = (int)(c % kSS);
                    if (c >= (uint32_t)kSS) ptx::mbar_wait(&sm.done[s], ((c / kSS) - 1) & 1);
                    if (keep && rank >= room) {
                        write_row(sm, s, rank - room, r0, r1);
                        sm.epi[s][rank - room] = epi_v;
                    }
                    fill = nk - room;
                } else {
                    fill += nk;
                }
            }
            // close the tile: pad and publish the partial chunk (or an empty one so the
            // epilogue still writes the tile)
            if (open && (fill > 0 || !emitted)) {
                if (lane >= fill) {
                    uint4 r0, r1;
                    make_row(false, 0, 0, 0, 0, 0, 0, 0, 0, r0, r1);
                    write_row(sm, s, lane, r0, r1);
                }
                if (lane == 0) {
                    sm.hdr[s].seq = seq;
                    sm.hdr[s].tile = tile;
                    sm.hdr[s].n_valid = fill;
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&sm.full[s]);
                ++c;
            } else if (!open) {
                s = (int)(c % kSS);
                if (c >= (uint32_t)kSS) ptx::mbar_wait(&sm.done[s], ((c / kSS) - 1) & 1);
                if (lane == 0) {
                    sm.hdr[s].seq = seq;
                    sm.hdr[s].tile = tile;
                    sm.hdr[s].n_valid = 0;
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&sm.full[s]);
                ++c;
            }
        }
        // end of stream
        const int s = (int)(c % kSS);
        if (c >= (uint32_t)kSS) ptx::mbar_wait(&sm.done[s], ((c / kSS) - 1) & 1);
        if (lane == 0) {
            sm.hdr[s].seq = -1;
            sm.hdr[s].tile = -1;
            sm.hdr[s].n_valid = 0;
            ptx::mbar_arrive(&sm.full[s]);
        }
        __syncwarp();
    } else if (warp == kMma) {
        // ================================ MMA issuer ==========================================
        constexpr uint32_t idesc = ptx::idesc_f16(128, kN);
        const uint32_t a_base = ptx::smem_u32(sm.a);
        for (uint32_t c = 0;; ++c) {
            const int s = (int)(c % kSS), ts = (int)(c % kTS);
            ptx::mbar_wait(&sm.full[s], (c / kSS) & 1);
            if (c >= (uint32_t)kTS) ptx::mbar_wait(&sm.tempty[ts], ((c / kTS) - 1) & 1);
            ptx::tc_fence_after();
            const ChunkHeader h = sm.hdr[s];
            if (lane == 0) {
                if (h.seq >= 0 && h.n_valid > 0) {
                    const uint32_t dcol = tmem + (uint32_t)(ts * 2 * kN);
                    const uint64_t bd = ptx::smem_desc(ptx::smem_u32(&sm.b[s][0]), 128, 256);
                    ptx::mma_f16_ss(dcol, ptx::smem_desc(a_base, 128, 256), bd, idesc, 0u);
                    ptx::mma_f16_ss(dcol + (uint32_t)kN, ptx::smem_desc(a_base + 4096u, 128, 256), bd, idesc, 0u);
                    ptx::mma_commit(&sm.tfull[ts]);
                } else {
                    ptx::mbar_arrive(&sm.tfull[ts]);
                }
            }
            __syncwarp();
            if (h.seq < 0) break;
        }
    } else {
        // ================================ epilogue ============================================
        const int q = warp;
        const int p0 = lane_pixel(0, q * 32 + lane), p1 = lane_pixel(1, q * 32 + lane);
        const int prow[2] = {p0 >> 4, p1 >> 4};
        const int pcol = p0 & 15;
        float T[2], cr[2], cg[2], cb[2], thr[2];
        int px = 0, py[2] = {0, 0};
        bool inside[2] = {false, false};
        const float L = log2f(a.alpha_skip);
        const float tterm = a.t_terminate;
        int cur = -1;
        bool reported = false;
        for (uint32_t c = 0;; ++c) {
            const int s = (int)(c % kSS), ts = (int)(c % kTS);
            ptx::mbar_wait(&sm.tfull[ts], (c / kTS) & 1);
            ptx::tc_fence_after();
            const ChunkHeader h = sm.hdr[s];
            if (h.seq != cur) {
                if (cur >= 0) {
#pragma unroll
                    for (int k = 0; k < 2; ++k)
                        if (inside[k]) {
                            float* o = a.image + ((size_t)(py[k] - a.image_row0) * gg.width + px) * 3;
                            o[0] = fminf(fmaxf(cr[k], 0.0f), 1.0f);
                            o[1] = fminf(fmaxf(cg[k], 0.0f), 1.0f);
                            o[2] = fminf(fmaxf(cb[k], 0.0f), 1.0f);
                        }
                }
                if (h.seq < 0) break;
                cur = h.seq;
                reported = false;
                const int tx = h.tile % gg.tiles_x, ty = h.tile / gg.tiles_x + trow0;
                px = tx * kTile + pcol;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    py[k] = ty * kTile + prow[k];
                    inside[k] = px < gg.width && py[k] < gg.height;
                    T[k] = 1.0f;
                    cr[k] = cg[k] = cb[k] = 0.0f;
                    thr[k] = inside[k] ? L : kInf;
                }
            }
            const bool work = h.n_valid > 0 && __any_sync(0xffffffffu, thr[0] != kInf || thr[1] != kInf);
            const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ts * 2 * kN);
#pragma unroll
            for (int blk = 0; blk < 2; ++blk) {
                const int j0 = blk * 16;
                uint32_t d[2][16];
                if (work) {
                    ptx::tmem_ld16(lane_base + (uint32_t)j0, d[0]);
                    ptx::tmem_ld16(lane_base + (uint32_t)(kN + j0), d[1]);
                    ptx::tmem_wait_ld();
                    ptx::reg_fence16(d[0]);
                    ptx::reg_fence16(d[1]);
                }
                if (blk == 1) {  // TMEM drained into registers: the next MMA may overwrite it
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&sm.tempty[ts]);
                }
                if (!work) continue;
                // Speculative pass: blend every splat with D >= thr without the per-splat
                // termination test (no loop-carried compare chain); T only decreases, so
                // T_end < t_terminate <=> the pixel terminated inside this block, which is then
                // replayed exactly (at most once per pixel per tile).
                float T0[2], r0[2], g0[2], b0[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    T0[k] = T[k];
                    r0[k] = cr[k];
                    g0[k] = cg[k];
                    b0[k] = cb[k];
                }
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    const float dA = __uint_as_float(d[0][jj]), dB = __uint_as_float(d[1][jj]);
                    const bool ta = dA >= thr[0], tb = dB >= thr[1];
                    if (ta || tb) {
                        const float4 ej = sm.epi[s][j0 + jj];
                        const float aA = ta ? fminf(ej.w, ex2_approx(dA)) : 0.0f;
                        const float aB = tb ? fminf(ej.w, ex2_approx(dB)) : 0.0f;
                        const float wA = T[0] * aA, wB = T[1] * aB;
                        cr[0] = fmaf(wA, ej.x, cr[0]);
                        cg[0] = fmaf(wA, ej.y, cg[0]);
                        cb[0] = fmaf(wA, ej.z, cb[0]);
                        cr[1] = fmaf(wB, ej.x, cr[1]);
                        cg[1] = fmaf(wB, ej.y, cg[1]);
                        cb[1] = fmaf(wB, ej.z, cb[1]);
                        T[0] -= wA;
                        T[1] -= wB;
                    }
                }
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (T[k] < tterm) {  // terminated inside the block: exact replay
                        T[k] = T0[k];
                        cr[k] = r0[k];
                        cg[k] = g0[k];
                        cb[k] = b0[k];
                        bool stop = false;
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            const float dv = __uint_as_float(d[k][jj]);
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
            // report this warp's pixels terminated (once per tile) so the producer can retire
            const bool dead = !__any_sync(0xffffffffu, thr[0] != kInf || thr[1] != kInf);
            __syncwarp();
            if (lane == 0) {
                if (dead && !reported) ((volatile int*)sm.dead_seq)[q] = cur;
                ptx::mbar_arrive(&sm.done[s]);
            }
            reported = reported || dead;
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == kMma) ptx::tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

void launch_raster_tensor(const RasterArgs& a, int num_sms, cudaStream_t st) {
    const size_t smem = sizeof(Smem) + 1024;
    cudaFuncSetAttribute(raster_tensor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int trows = std::min(a.gg.tiles_y, a.gg.band_gy1 * a.gg.g) - a.gg.band_gy0 * a.gg.g;
    const int n_tiles = a.gg.tiles_x * trows;
    int grid = num_sms * kCtasPerSm;
    if (grid > n_tiles) grid = n_tiles;
    if (grid > 0) raster_tensor_kernel<<<grid, kThreads, smem, st>>>(a);
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
