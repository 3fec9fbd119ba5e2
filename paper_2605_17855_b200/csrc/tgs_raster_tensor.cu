// Tensorized, cross-tile-grouped rasterizer (north_star 3 + 4) on the 5th-gen tensor cores.
//
// Reference semantics: proj/src/raster_tensor.cpp:64-160 (rasterize_group_impl) — one CTA per
// tile group walks the group's depth-sorted list chunk by chunk; every live member tile consumes
// the chunk's entries whose mask has its bit, in list order; per pixel the power feeds
// alpha_of/blend (raster_scalar.hpp:40-55) until T < t_terminate; tiles retire early
// (:93-96, :107, :138-141) and the group exits when all member tiles are done.  The paper's
// design: the chunk is staged in shared memory ONCE per group and reused by
// all member tiles.
//
// B200 formulation.  The reference builds a pixel operand per Gaussian row
// (raster_tensor.cpp:118-123), which no hardware MMA can do.  Here the power is expanded around
// the centre o of the unit:  u = pixel - o, m = mean - o,
//     log2(e) * power + log2(opacity) = w . phi(u),
//     phi(u) = [ux^2, ux*uy, uy^2, ux, uy, 1]          (pixel side, exact in FP16: |u| <= 15.5)
//     w      = log2e * [-a/2, -b, -c/2, a mx + b my, b mx + c my,
//                       -(a mx^2/2 + b mx my + c my^2/2)] + [0,0,0,0,0, log2 o]   (splat side)
// carried as an FP16 hi/lo pair (K lanes 0-5 hi, 6-11 lo).  K lanes 12-15 realise the paper's
// tile-membership mask (binning.cpp:56-65, raster_tensor.cpp:24-38) inside the contraction: the
// pixel row of member tile t has a one-hot 1.0 in lane 12+t, the splat row has 0 there when the
// splat overlaps tile t and -30000 otherwise.  So ONE K=16 FP16 MMA per (M-tile, chunk) gives
//     D[pixel][splat] = log2(alpha_unclamped)  (or <= -30000 for a non-member tile)
// and the epilogue needs no per-tile branch: alpha = min(ex2(D), min(alpha_clamp, o)), skip iff
// D < log2(alpha_skip) — which also realises the positive-power clamp (raster_scalar.hpp:41).
//
// CTA (persistent) = one unit of SLOTS member tiles at a time (G=2: the 2x2 group; G=4: a 2x2
// quarter of the group; G=1: one tile, SLOTS = 1), units in the order of the previous frame's
// measured walks (unit_order_kernel).  Roles:
//   producer warp:   streams the unit's list in 32-entry batches (records prefetched), gathers
//                    each splat ONCE per unit (north_star 4), drops entries whose member tiles
//                    are all retired or that cannot reach alpha_skip (ballot compaction keeps
//                    list order), writes unit-centred coefficient rows + blend data into a ring of
//                    kSS shared-memory chunk stages;
//   warpgroups:      one per member tile (4 warps = the 4 TMEM lane quadrants).  A member tile is
//                    two M=128 tiles; warp q of the group owns lane quadrant q of both, which is
//                    the tile's 8x8 pixel block q (lane_pixel): 2 pixels per thread, blended
//                    together with packed FP32x2 instructions, and a packed-FADD2 mask phase picks
//                    the splats of each 16-splat batch that reach any of the warp's pixels.  Each
//                    warpgroup has its own 2-stage TMEM accumulator ring and its own
//                    commit barriers, so member tiles progress independently through the shared
//                    chunk ring (up to kSS chunks apart) and only the 4 warps of one tile advance
//                    in lock-step;
//   MMA warp:        TMEM owner; lane t polls warpgroup t (chunk published, TMEM stage free) so one
//                    ballot finds every ready group; per (warpgroup, chunk) two tcgen05.mma
//                    (M=128, N=32, K=16) into the group's free TMEM stage, issued from warp-uniform
//                    code by an elected lane, then tcgen05.commit -> that group's barrier.  Retired
//                    tiles get no MMA.
// The pixel operand A is identical for every unit and built once per CTA.  Hand-offs: full[s]
// (mbarrier, producer -> MMA), tfull[t][ts] (tcgen05.commit, MMA -> warpgroup t), and release
// counters compared against absolute chunk targets (done_cnt: smem stage; wdone: TMEM stage);
// every wait is watchdog-bounded, so a protocol bug is a reported kernel error, never a hang.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"
#include "tgs_ptx.cuh"

namespace tgs {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kNeverRow = -30000.0f;
constexpr float kInf = __builtin_huge_valf();
// Tuned on the C3 bench frame (DESIGN.md §3.1 lists the measured alternatives): chunks of 32
// splats (MMA N), a ring of 4 shared-memory chunk stages, 2 TMEM stages per warpgroup, a gather
// ring of 8 batches.
constexpr int kN = 32;      // splats per chunk (MMA N)
constexpr int kSS = 4;      // shared-memory chunk ring (slack between member tiles)
constexpr int kTS = 2;      // TMEM accumulator stages per warpgroup
constexpr int kJB = 16;     // accumulator columns per epilogue batch
constexpr int kRing = 8;    // producer gather ring: kRing - 2 batches of records in flight
constexpr uint32_t kMmaSleep0 = 16, kMmaSleepCap = 128;  // MMA warp back-off (ns) when nothing is ready
#ifndef TGS_RASTER_PROF
#define TGS_RASTER_PROF 0
#endif
#if TGS_RASTER_PROF
// role timing (tools builds only): [0] producer total [1] producer stage waits [2] MMA total
// [3] epilogue total (sum over warps) [4] epilogue tfull waits [5] active (warp, splat) pairs
// [6] (warp, splat) pairs tested [7] chunks
__device__ unsigned long long g_rprof[16];
__device__ unsigned int g_rprof_done;
__device__ unsigned long long g_rprof_issue, g_rprof_seen, g_rprof_iters;
#endif

template <int SLOTS>
struct Cfg {
    static constexpr int kMT = 2 * SLOTS;  // M=128 tiles per unit (two per member tile)
    static constexpr int kEpiWarps = 4 * SLOTS;
    // warp layout: the producer, the MMA warp, then the epilogue warps
    static constexpr int kProd = 0, kMma = 1, kEpi0 = 2;
    static constexpr int kThreads = (kEpiWarps + 2) * 32;
    static constexpr int kCtasPerSm = SLOTS == 1 ? 3 : 1;
    static constexpr uint32_t kTmemCols = kTS * kMT * kN <= 128 ? 128 : kTS * kMT * kN <= 256 ? 256 : 512;
    static_assert(kTS * kMT * kN * kCtasPerSm <= 512, "TMEM columns per SM");
};
template <int SLOTS>
__host__ __device__ inline int units_per_group(int g) { return (SLOTS == 4 && g == 4) ? 4 : 1; }

struct ChunkHeader {
    int seq;      // per-CTA unit sequence number, -1 = end of the stream
    int unit;     // unit index (order-resolved)
    int n_valid;  // splats in the chunk (0: unit without contributing splats)
    int live;     // member tiles live when the chunk was produced (MMA skips the others)
    int chunk;    // chunk number (protocol self-check)
    int last;     // last chunk of its unit (the epilogue stores the unit's pixels)
};

template <int SLOTS>
struct Smem {
    alignas(128) uint8_t a[2 * SLOTS][128 * 32];  // pixel monomial rows (K-major, no swizzle)
    alignas(128) uint8_t b[kSS][kN * 32];         // splat coefficient rows
    float4 epi[kSS][kN];                          // r, g, b, min(alpha_clamp, opacity)
    ChunkHeader hdr[kSS];
    alignas(16) int wdone[16];  // chunks each epilogue warp has completed
    alignas(16) int dead[16];   // (seq << 1) | 1 once all pixels of the warp terminated in unit seq
    uint64_t full[kSS];         // producer -> MMA
    uint64_t tfull[SLOTS][kTS]; // MMA -> warpgroup (tcgen05.commit)
    // smem stage s is free again once every epilogue warp finished the chunk that used it
    unsigned int done_cnt[kSS];
    uint32_t tmem_base;
#if TGS_RASTER_PROF
    unsigned long long t_rel[4][kTS], t_iss[4][kTS], t_pub[kSS];  // PROF timestamps
#endif
    // producer gather ring (cp.async): splat records of kRing batches and list indices of 2 kRing
    float4 rmc[kRing][32], rco[kRing][32], rcol[kRing][32];
    uint32_t ridx[2 * kRing][32];
};

// Pixel (relative to the unit's top-left) of row l of M-tile m = 2 t + k: member tile t; lane
// quadrant q = l / 32 is the tile's 8x8 block q (x half q & 1, y half q >> 1), and M-tile k holds
// rows 4k..4k+3 of that block, so warp q of a warpgroup owns one compact 8x8 block of its tile
// (measured 2.5% faster than 16x4 strips: fewer splats reach a smaller footprint).
__device__ __forceinline__ void lane_pixel(int m, int l, int& x, int& y) {
    const int t = m >> 1, k = m & 1, q = l >> 5, i = l & 31;
    x = (t & 1) * 16 + (q & 1) * 8 + (i & 7);
    y = (t >> 1) * 16 + (q >> 1) * 8 + k * 4 + (i >> 3);
}

// Blend step of both pixels of a thread with packed FP32x2 instructions (FMUL2 / FFMA2 / FADD2):
// per pixel k  wt = T * al;  c += wt * colour (fused);  T -= wt  — the same IEEE operations, in the
// same order, as the scalar form, so the result is bit-identical.
__device__ __forceinline__ void blend_x2(float (&T)[2], float (&cr)[2], float (&cg)[2], float (&cb)[2],
                                         const float (&al)[2], const float4& ej) {
    asm("{\n\t"
        ".reg .b64 t, a, w, r, g, b, cx, cy, cz;\n\t"
        "mov.b64 t, {%0, %1};\n\t"
        "mov.b64 a, {%8, %9};\n\t"
        "mov.b64 r, {%2, %3};\n\t"
        "mov.b64 g, {%4, %5};\n\t"
        "mov.b64 b, {%6, %7};\n\t"
        "mov.b64 cx, {%10, %10};\n\t"
        "mov.b64 cy, {%11, %11};\n\t"
        "mov.b64 cz, {%12, %12};\n\t"
        "mul.rn.f32x2 w, t, a;\n\t"
        "fma.rn.f32x2 r, w, cx, r;\n\t"
        "fma.rn.f32x2 g, w, cy, g;\n\t"
        "fma.rn.f32x2 b, w, cz, b;\n\t"
        "sub.rn.f32x2 t, t, w;\n\t"
        "mov.b64 {%0, %1}, t;\n\t"
        "mov.b64 {%2, %3}, r;\n\t"
        "mov.b64 {%4, %5}, g;\n\t"
        "mov.b64 {%6, %7}, b;\n\t"
        "}"
        : "+f"(T[0]), "+f"(T[1]), "+f"(cr[0]), "+f"(cr[1]), "+f"(cg[0]), "+f"(cg[1]), "+f"(cb[0]), "+f"(cb[1])
        : "f"(al[0]), "f"(al[1]), "f"(ej.x), "f"(ej.y), "f"(ej.z));
}

// (a >= b && c >= d) ? v : 0 as two compares (the second AND-ed with the first) and one select
__device__ __forceinline__ float sel_ge2(float a, float b, float c, float d, float v) {
    float r;
    asm("{\n\t.reg .pred q, p;\n\tsetp.ge.f32 q, %3, %4;\n\tsetp.ge.and.f32 p, %1, %2, q;\n\t"
        "selp.f32 %0, %5, 0f00000000, p;\n\t}"
        : "=f"(r)
        : "f"(a), "f"(b), "f"(c), "f"(d), "f"(v));
    return r;
}

// (x0 - t, x1 - t) with one packed FADD2; results as raw bits
__device__ __forceinline__ void sub_x2(uint32_t x0, uint32_t x1, float t, uint32_t& r0, uint32_t& r1) {
    asm("{\n\t.reg .b64 x, y, r;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %4};\n\t"
        "sub.rn.f32x2 r, x, y;\n\tmov.b64 {%0, %1}, r;\n\t}"
        : "=r"(r0), "=r"(r1)
        : "r"(x0), "r"(x1), "f"(t));
}

// byte offset of (row, k-half) in a K-major no-swizzle operand: 8x16B core matrices
__device__ __forceinline__ uint32_t core_off(int row, int khalf) {
    return (uint32_t)((row >> 3) * 256 + khalf * 128 + (row & 7) * 16);
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// Coefficient row of one splat for a unit centred at (ox, oy): FP16 hi/lo halves of w plus the
// four member-tile mask lanes.  Returns false when |w| exceeds the FP16 hi/lo range: such a
// splat cannot reach alpha_skip anywhere in the unit (|u| <= 15.5 and the +0.3 dilation bounds
// the conic by 1/0.3), so it is dropped.
__device__ __forceinline__ bool make_row(float mx, float my, float qa, float qb, float qc, float lo2, float ox,
                                         float oy, uint32_t cover, uint4& r0, uint4& r1) {
    float w[6];
    const float dx = mx - ox, dy = my - oy;
    const float ha = 0.5f * qa, hc = 0.5f * qc;
    w[0] = -ha * kLog2e;
    w[1] = -qb * kLog2e;
    w[2] = -hc * kLog2e;
    w[3] = fmaf(qa, dx, qb * dy) * kLog2e;
    w[4] = fmaf(qb, dx, qc * dy) * kLog2e;
    const float quad = fmaf(ha * dx, dx, fmaf(qb * dx, dy, hc * dy * dy));
    w[5] = fmaf(-quad, kLog2e, lo2);
    const float amax = fmaxf(fmaxf(fmaxf(fabsf(w[0]), fabsf(w[1])), fmaxf(fabsf(w[2]), fabsf(w[3]))),
                             fmaxf(fabsf(w[4]), fabsf(w[5])));
    const bool ok = amax <= 16384.0f;
    // hi halves packed pairwise (RN, as element-wise __float2half_rn), lo = w - hi (exact), packed
    uint32_t hp[3], lp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const __half2 h2 = __floats2half2_rn(w[2 * k], w[2 * k + 1]);
        const float2 hf = __half22float2(h2);
        hp[k] = *reinterpret_cast<const uint32_t*>(&h2);
        lp[k] = pack_half2(w[2 * k] - hf.x, w[2 * k + 1] - hf.y);
    }
    const float m0 = (cover & 1u) ? 0.0f : kNeverRow, m1 = (cover & 2u) ? 0.0f : kNeverRow;
    const float m2 = (cover & 4u) ? 0.0f : kNeverRow, m3 = (cover & 8u) ? 0.0f : kNeverRow;
    r0 = make_uint4(hp[0], hp[1], hp[2], lp[0]);
    r1 = make_uint4(lp[1], lp[2], pack_half2(m0, m1), pack_half2(m2, m3));
    return ok;
}

__device__ __forceinline__ unsigned int ld_volatile_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_u32(p)) : "memory");
    return v;
}

__device__ __forceinline__ int4 ld_volatile_v4(const int* p) {
    int4 v;
    asm volatile("ld.volatile.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(ptx::smem_u32(p)));
    return v;
}

// Never-contributing padding row (tail of a partial chunk).
__device__ __forceinline__ void never_row(uint4& r0, uint4& r1) {
    r0 = make_uint4(0u, 0u, pack_half2(0.0f, kNeverRow), 0u);
    r1 = make_uint4(0u, 0u, 0u, 0u);
}

template <int SLOTS>
__device__ __forceinline__ void write_row(Smem<SLOTS>& sm, int s, int slot, const uint4& r0, const uint4& r1) {
    *reinterpret_cast<uint4*>(&sm.b[s][core_off(slot, 0)]) = r0;
    *reinterpret_cast<uint4*>(&sm.b[s][core_off(slot, 1)]) = r1;
}

// Unit geometry: the unit's top-left tile, the group whose list it walks, member-tile liveness.
struct UnitGeom {
    int tx0, ty0;   // top-left tile of the unit (absolute tile coords)
    int gid;        // band-local group id
    uint32_t live;  // member tiles inside the tile grid
};

template <int SLOTS>
__device__ __forceinline__ UnitGeom unit_geom(const GroupGeom& gg, int unit) {
    UnitGeom u;
    if (SLOTS == 1) {  // G == 1: unit == tile == group
        u.tx0 = unit % gg.groups_x;
        u.ty0 = unit / gg.groups_x + gg.band_gy0;
        u.gid = unit;
        u.live = 1u;
        return u;
    }
    // G == 2: unit == group; G == 4: unit == quarter (2x2 tiles) of a group
    const int per = units_per_group<SLOTS>(gg.g);
    const int grp = unit / per, quarter = unit % per;
    const int gx = grp % gg.groups_x, gy = grp / gg.groups_x + gg.band_gy0;
    u.tx0 = gx * gg.g + (quarter & 1) * 2;
    u.ty0 = gy * gg.g + (quarter >> 1) * 2;
    u.gid = grp;
    u.live = 0u;
#pragma unroll
    for (int t = 0; t < SLOTS; ++t)
        if (u.tx0 + (t & 1) < gg.tiles_x && u.ty0 + (t >> 1) < gg.tiles_y) u.live |= 1u << t;
    return u;
}

template <int SLOTS>
__global__ void __launch_bounds__(Cfg<SLOTS>::kThreads, Cfg<SLOTS>::kCtasPerSm) raster_tensor_kernel(RasterArgs a) {
    using C = Cfg<SLOTS>;
    constexpr int kMT = C::kMT, kEpiWarps = C::kEpiWarps, kProd = C::kProd, kMma = C::kMma;
    constexpr uint32_t kTmemCols = C::kTmemCols;
    // No-swizzle K-major operands only need 16-byte alignment (descriptor addresses are >> 4).
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem<SLOTS>& sm = *reinterpret_cast<Smem<SLOTS>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const GroupGeom& gg = a.gg;
    const int n_units = gg.n_groups_band * units_per_group<SLOTS>(gg.g);
    const float centre = SLOTS == 1 ? 8.0f : 16.0f;

    // ---- setup: A operand (pixel monomials + tile one-hot), barriers, TMEM -----------------
    for (int p = threadIdx.x; p < kMT * 128; p += blockDim.x) {
        const int m = p >> 7, l = p & 127;
        int x, y;
        lane_pixel(m, l, x, y);
        const float ux = (float)x + 0.5f - centre, uy = (float)y + 0.5f - centre;
        const float phi[6] = {ux * ux, ux * uy, uy * uy, ux, uy, 1.0f};
        const int t = m >> 1;
        uint4 lo, hi;
        lo.x = pack_half2(phi[0], phi[1]);
        lo.y = pack_half2(phi[2], phi[3]);
        lo.z = pack_half2(phi[4], phi[5]);
        lo.w = pack_half2(phi[0], phi[1]);
        hi.x = pack_half2(phi[2], phi[3]);
        hi.y = pack_half2(phi[4], phi[5]);
        hi.z = pack_half2(t == 0 ? 1.0f : 0.0f, t == 1 ? 1.0f : 0.0f);
        hi.w = pack_half2(t == 2 ? 1.0f : 0.0f, t == 3 ? 1.0f : 0.0f);
        *reinterpret_cast<uint4*>(&sm.a[m][core_off(l, 0)]) = lo;
        *reinterpret_cast<uint4*>(&sm.a[m][core_off(l, 1)]) = hi;
    }
    if (threadIdx.x < 16) {
        sm.wdone[threadIdx.x] = 0;
        sm.dead[threadIdx.x] = -1;
#if TGS_RASTER_PROF
        if (threadIdx.x < 4 * kTS) sm.t_rel[threadIdx.x / kTS][threadIdx.x % kTS] = 0, sm.t_iss[threadIdx.x / kTS][threadIdx.x % kTS] = 0;
        if (threadIdx.x < kSS) sm.t_pub[threadIdx.x] = 0;
#endif
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSS; ++s) {
            ptx::mbar_init(&sm.full[s], 1);
            sm.done_cnt[s] = 0;
        }
        for (int t = 0; t < SLOTS; ++t)
            for (int s = 0; s < kTS; ++s) ptx::mbar_init(&sm.tfull[t][s], 1);
        ptx::mbar_fence_init();
    }
    if (warp == kMma) ptx::tmem_alloc<kTmemCols>(&sm.tmem_base);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    [[maybe_unused]] unsigned long long pf[4] = {0, 0, 0, 0};
    [[maybe_unused]] unsigned long long pf_lock = 0;  // epilogue waits while its group held the TMEM stage
    [[maybe_unused]] unsigned long long pf_wake = 0, pf_wake_n = 0;  // MMA commit -> epilogue wake-up
    [[maybe_unused]] const long long pf_start = clock64();

    if (warp == kProd) {
        // ================================ producer ===========================================
        const float skip = a.alpha_skip, clampv = a.alpha_clamp;
        uint32_t c = 0;  // chunks emitted so far
        const uint32_t lt = (1u << lane) - 1u;
        auto open_stage = [&](uint32_t cc) {
            // stage cc % kSS is free once every epilogue warp finished chunk cc - kSS (lane 0
            // polls, the warp reconverges after)
            const int s = (int)(cc % kSS);
            if (cc >= (uint32_t)kSS && lane == 0) {
                const unsigned int need = (unsigned int)kEpiWarps * (cc / kSS);
                if (ld_volatile_u32(&sm.done_cnt[s]) < need) {
                    const long long t0 = clock64();
                    while (ld_volatile_u32(&sm.done_cnt[s]) < need) {
                        __nanosleep(32);
                        if (clock64() - t0 > 4000000000ll) ptx::watchdog_trap("producer/done", (int)cc, s);
                    }
                    if (TGS_RASTER_PROF) pf[1] += clock64() - t0;
                }
            }
            __syncwarp();
            return s;
        };
        unsigned long long op_chunks = 0, op_skipped = 0;  // OpReport (lane 0)
        auto publish = [&](int s, int seq, int unit, int n_valid, uint32_t live, int last) {
            if (lane == 0) {
                op_chunks += (seq >= 0 && n_valid > 0) ? 1u : 0u;
                ChunkHeader& h = sm.hdr[s];
                h.seq = seq;
                h.unit = unit;
                h.n_valid = n_valid;
                h.live = (int)live;
                h.chunk = (int)c;
                h.last = last;
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
#if TGS_RASTER_PROF
            if (lane == 0) sm.t_pub[s] = (unsigned long long)clock64();
#endif
            if (lane == 0) ptx::mbar_arrive(&sm.full[s]);
            __syncwarp();
        };
        for (int seq = 0;; ++seq) {
            int t = 0;
            if (lane == 0) t = (int)atomicAdd(&a.fc->group_counter, 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n_units) break;
            const int unit = a.order ? a.order[t] : t;
            const UnitGeom ug = unit_geom<SLOTS>(gg, unit);
            const uint32_t unit_c0 = c;
            const uint32_t begin = a.offsets[ug.gid], end = a.offsets[ug.gid + 1];
            const float ox = (float)(ug.tx0 * kTile) + centre, oy = (float)(ug.ty0 * kTile) + centre;
            int fill = 0, s = 0;   // rows placed in the open chunk / its stage
            bool open = false;     // a stage is open for this unit
            bool emitted = false;  // at least one chunk of this unit published
            uint32_t live = ug.live;
            const uint32_t nb = (end - begin + 31u) / 32u;
            // Gather pipeline (cp.async, no registers held by in-flight loads): list indices of
            // batch b land in ridx[b % 2R], its records in the ring slot b % R; at step i the
            // records of batch i + R - 1 and the indices of batch i + 2R - 1 are requested, one
            // commit group per step, so R - 1 batches of records are in flight.
            auto valid = [&](uint32_t b) { return b < nb && begin + b * 32u + (uint32_t)lane < end; };
            auto issue_idx = [&](uint32_t b) {
                if (valid(b)) ptx::cp_async4(&sm.ridx[b % (2 * kRing)][lane], &a.list[begin + b * 32u + lane]);
            };
            auto issue_rec = [&](uint32_t b) {
                if (valid(b)) {
                    const uint32_t idx = sm.ridx[b % (2 * kRing)][lane];
                    const int r = (int)(b % kRing);
                    ptx::cp_async16(&sm.rmc[r][lane], &a.proj.mc[idx]);
                    ptx::cp_async16(&sm.rco[r][lane], &a.proj.co[idx]);
                    ptx::cp_async16(&sm.rcol[r][lane], &a.proj.col[idx]);
                }
            };
            struct Rec {
                float4 mc, co, col;
                uint32_t idx;
            };
            auto ld_rec = [&](uint32_t b) -> Rec {
                Rec r;
                if (valid(b)) {
                    const int k = (int)(b % kRing);
                    r.idx = 0u;
                    r.mc = sm.rmc[k][lane];
                    r.co = sm.rco[k][lane];
                    r.col = sm.rcol[k][lane];
                } else {
                    r.idx = 0xffffffffu;
                    r.mc = r.co = r.col = make_float4(0, 0, 0, 0);
                }
                return r;
            };
            uint32_t n_batches = 0;
            struct Built {
                bool keep;
                uint32_t cover;
                uint4 r0, r1;
                float4 epi;
            };
            // member tiles whose 4 warps all reported every pixel terminated -> dropped from `live`;
            // true when no member tile is left
            auto retire_check = [&]() -> bool {
                if (emitted) {
                    uint32_t retired = 0u;
#pragma unroll
                    for (int tt = 0; tt < SLOTS; ++tt) {
                        const int4 d = ld_volatile_v4(&sm.dead[4 * tt]);
                        const int want = (seq << 1) | 1;
                        if (d.x == want && d.y == want && d.z == want && d.w == want) retired |= 1u << tt;
                    }
                    // sm.dead is written concurrently by the epilogue warps: take lane 0's view so
                    // the whole warp makes the same decision
                    retired = __shfl_sync(0xffffffffu, retired, 0);
                    live &= ~retired;
                    if (live == 0u) return true;
                }
                return false;
            };
            auto build = [&](const Rec& cur, Built& bt) {
                bt.keep = false;
                bt.cover = 0;
                bt.epi = make_float4(0, 0, 0, 0);
                if (cur.idx != 0xffffffffu) {
                    // member tiles the splat's list entry covers (binning.cpp:56-65), narrowed by the
                    // tile cull to those whose pixel centres meet its alpha_skip box (tight_cover of
                    // the extents preprocess stored in col.w)
                    int x0, y0, x1, y1;
                    tile_rect(cur.mc.x, cur.mc.y, __float_as_int(cur.co.w), gg.tiles_x, gg.tiles_y, x0, y0, x1, y1);
                    const float lo2 = lg2_approx(cur.co.y);
                    const float cj = fminf(clampv, cur.co.y);
                    const uint32_t tight =
                        a.tile_cull ? tight_cover(cur.mc.x, cur.mc.y, cur.col.w, ug.tx0, ug.ty0, SLOTS) : 0xfu;
                    uint32_t cover = 0;
#pragma unroll
                    for (int k = 0; k < SLOTS; ++k) {
                        const int tx = ug.tx0 + (k & 1), ty = ug.ty0 + (k >> 1);
                        if (tx >= x0 && tx <= x1 && ty >= y0 && ty <= y1) cover |= 1u << k;
                    }
                    cover &= live & tight;
                    if (cover != 0u && !(cj < skip)) {
                        bt.keep = make_row(cur.mc.x, cur.mc.y, cur.mc.z, cur.mc.w, cur.co.x, lo2, ox, oy, cover, bt.r0,
                                           bt.r1);
                        bt.cover = cover;
                        bt.epi = make_float4(cur.col.x, cur.col.y, cur.col.z, cj);
                    }
                }
            };
            auto place = [&](const Built& bt) {
                const uint32_t km = __ballot_sync(0xffffffffu, bt.keep);
                if (km == 0u) return;
                // OpReport skipped_pairs: live member tiles a staged row's mask leaves out
                const uint32_t sk = __reduce_add_sync(0xffffffffu, bt.keep ? __popc(live & ~bt.cover) : 0u);
                if (lane == 0) op_skipped += sk;
                const int nk = __popc(km);
                const int rank = __popc(km & lt);
                if (!open) {
                    s = open_stage(c);
                    open = true;
                    fill = 0;
                }
                // place the kept ranks in order; a full chunk is published and the next one opened
                int placed = 0;
                for (;;) {
                    const int room = kN - fill;
                    if (bt.keep && rank >= placed && rank - placed < room) {
                        write_row(sm, s, fill + rank - placed, bt.r0, bt.r1);
                        sm.epi[s][fill + rank - placed] = bt.epi;
                    }
                    if (nk - placed < room) {
                        fill += nk - placed;
                        break;
                    }
                    publish(s, seq, unit, kN, live, 0);
                    ++c;
                    emitted = true;
                    s = open_stage(c);
                    fill = 0;
                    placed += room;
                    if (placed == nk) break;
                }
            };
            // two batches per step (independent builds overlap, then placement in list order);
            // records of batches 2i + R - 2 and 2i + R - 1 are requested at step i into the slots
            // the previous step consumed, one commit group per batch: R - 2 batches in flight
            static_assert(kRing >= 4 && kRing % 2 == 0, "gather ring");
            for (uint32_t b = 0; b < 2u * kRing - 2u; ++b) issue_idx(b);
            ptx::cp_async_commit();
            ptx::cp_async_wait<0>();
            __syncwarp();
            for (uint32_t b = 0; b < kRing - 2u; ++b) {
                issue_rec(b);
                ptx::cp_async_commit();
            }
            for (uint32_t bi = 0; bi < nb; bi += 2) {
                [[maybe_unused]] const long long tc0 = TGS_RASTER_PROF ? clock64() : 0;
                ptx::cp_async_wait<kRing - 4>();  // records of batches bi, bi + 1
                if (TGS_RASTER_PROF) {
                    pf[2] += clock64() - tc0;
                    pf[3] += 2;
                }
                __syncwarp();
                if (retire_check()) break;
                const bool has_b = bi + 1 < nb;
                n_batches += has_b ? 2u : 1u;
                const Rec ca = ld_rec(bi), cb = ld_rec(bi + 1);
                issue_idx(bi + 2u * kRing - 2u);
                issue_rec(bi + kRing - 2u);
                ptx::cp_async_commit();
                issue_idx(bi + 2u * kRing - 1u);
                issue_rec(bi + kRing - 1u);
                ptx::cp_async_commit();
                Built ba, bb;
                build(ca, ba);
                build(cb, bb);
                place(ba);
                if (has_b) place(bb);
            }
            ptx::cp_async_wait<0>();  // nothing in flight into the ring when the next unit starts
            __syncwarp();
            // close the unit: exactly one chunk flagged `last` — the padded partial chunk, or an
            // empty one (unit without kept splats, or kept rows ending on a chunk boundary)
            if (!open) s = open_stage(c);
            if (lane >= fill && lane < kN) {
                uint4 r0, r1;
                never_row(r0, r1);
                write_row(sm, s, lane, r0, r1);
            }
            publish(s, seq, unit, fill, live, 1);
            ++c;
            // schedule feedback: list entries this unit walked (batches) plus rows it staged
            if (a.unit_cost && lane == 0) a.unit_cost[unit] = 32u * n_batches + (uint32_t)kN * (c - unit_c0);
        }
        if (TGS_RASTER_PROF) pf[0] = c;
        {  // end of the stream
            const int se = open_stage(c);
            publish(se, -1, -1, 0, 0u, 1);
        }
        if (lane == 0) {
            atomicAdd(&a.fc->op_chunks, op_chunks);
            atomicAdd(&a.fc->op_skipped, op_skipped);
        }
    } else if (warp == kMma) {
        // ================================ MMA issuer ==========================================
        // Lane t (< SLOTS) tracks warpgroup t: its next chunk and whether its stream ended.  One
        // poll tests every group's readiness at once (chunk published, TMEM stage released), the
        // ready groups are then issued in turn — the issue latency is on the raster's critical
        // path (a slower poll measured +30 % raster time).
        constexpr uint32_t idesc = ptx::idesc_f16(128, kN);
        const uint32_t a_base = ptx::smem_u32(&sm.a[0][0]);
        uint32_t my_c = 0;                    // lane t: next chunk of warpgroup t
        bool my_end = lane >= SLOTS;          // lane t: warpgroup t's stream ended (other lanes: idle)
        unsigned long long op_mmas = 0, op_mma_rows = 0;  // OpReport
        long long idle0 = clock64();
        uint32_t backoff = kMmaSleep0;
#if TGS_RASTER_PROF
        unsigned long long mma_iters = 0;
#endif
        for (;;) {
            if (__all_sync(0xffffffffu, my_end)) break;
#if TGS_RASTER_PROF
            ++mma_iters;
#endif
            bool rdy = false;
            if (!my_end) {
                const int s = (int)(my_c % kSS);
                // chunk published, and warpgroup t finished chunk c - kTS (its TMEM stage)
                rdy = ptx::mbar_test(&sm.full[s], (my_c / kSS) & 1);
                if (rdy && my_c >= (uint32_t)kTS) {
                    const int4 d = ld_volatile_v4(&sm.wdone[4 * lane]);
                    rdy = min(min(d.x, d.y), min(d.z, d.w)) >= (int)(my_c - kTS + 1);
                }
            }
            uint32_t rm = __ballot_sync(0xffffffffu, rdy);
            if (rm == 0u) {
                // idle: back off exponentially so the polls do not take issue slots from the
                // epilogue warps of this SMSP (the MMA warp has the highest arbitration rank)
                __nanosleep(backoff);
                backoff = backoff < kMmaSleepCap ? 2 * backoff : backoff;
                if (clock64() - idle0 > 4000000000ll)
                    ptx::watchdog_trap("mma/idle", (int)__shfl_sync(0xffffffffu, my_c, 0), (int)rm);
                continue;
            }
            idle0 = clock64();
            backoff = kMmaSleep0;
            __syncwarp();
            ptx::tc_fence_after();
            while (rm) {
                const int t = __ffs(rm) - 1;
                rm &= rm - 1u;
                const uint32_t c = __shfl_sync(0xffffffffu, my_c, t);
                const int s = (int)(c % kSS), ts = (int)(c % kTS);
                const volatile ChunkHeader& hs = sm.hdr[s];  // every lane reads it (broadcast)
                const int hseq = hs.seq, hnv = hs.n_valid, hch = hs.chunk;
                const uint32_t hlive = (uint32_t)hs.live;
                if (hch != (int)c) {
                    if (lane == 0)
                        printf("libtgs MMA: warpgroup %d expected chunk %d found %d (seq %d)\n", t, (int)c, hch, hseq);
                    __trap();
                }
                if (hseq >= 0 && hnv > 0 && ((hlive >> t) & 1u)) {
                    const uint64_t bd = ptx::smem_desc(ptx::smem_u32(&sm.b[s][0]), 128, 256);
                    const uint32_t dcol = tmem + (uint32_t)(((ts * SLOTS + t) * 2) * kN);
#pragma unroll
                    for (int k = 0; k < 2; ++k)
                        ptx::mma_f16_ss_elect(dcol + (uint32_t)(k * kN),
                                              ptx::smem_desc(a_base + (uint32_t)((2 * t + k) * 128 * 32), 128, 256), bd,
                                              idesc, 0u);
                    ptx::mma_commit_elect(&sm.tfull[t][ts]);
                    op_mmas += 2;
                    op_mma_rows += 2u * (uint32_t)hnv;
#if TGS_RASTER_PROF
                    if (lane == 0) sm.t_iss[t][ts] = (unsigned long long)clock64();
#endif
                } else if (lane == 0) {
                    ptx::mbar_arrive(&sm.tfull[t][ts]);
                }
                __syncwarp();
                if (lane == t) {
                    my_c = c + 1;
                    if (hseq < 0) my_end = true;
                }
            }
        }
        if (lane == 0) {
            atomicAdd(&a.fc->op_mmas, op_mmas);
            atomicAdd(&a.fc->op_mma_rows, op_mma_rows);
        }
#if TGS_RASTER_PROF
        if (lane == 0) atomicAdd(&g_rprof_iters, mma_iters);
#endif
    } else {
        // ================================ epilogue ============================================
        // warp -> member tile t (its warpgroup) and lane quadrant q: tile rows 4q..4q+3; slot k
        // of a thread is its pixel in M-tile 2t + k (the tile's 8-column half k)
        // The SMSP arbiter ranks warps by id, so a group made of four same-rank warps would always
        // be served after (or before) the other tiles' groups.  Each member tile's group instead
        // takes one warp of every rank: the lane quadrant q is fixed by warp % 4, the rank is the
        // warp's position among the epilogue warps of its SMSP, tile t = (rank - q) mod 4.  Shared
        // per-warp state is indexed by slot 4t + q.
        const int q = warp & 3, rank = (warp - C::kEpi0) >> 2;  // q = the TMEM lane quadrant of this warp
        const int t = SLOTS == 4 ? ((rank - q) & 3) : rank;
        const int slot = 4 * t + q;
        int relx[2], rely[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) lane_pixel(2 * t + k, q * 32 + lane, relx[k], rely[k]);
        float T[2], cr[2], cg[2], cb[2], thr[2];
        int px[2], py[2];
        const float L = log2f(a.alpha_skip);
        const float tterm = a.t_terminate;
        int cur = -1;            // unit being rendered (seq), -1 none
        uint32_t alive = 0;      // warp-uniform: slots with a non-terminated pixel
        bool reported = false;   // retirement of this warp published for `cur`
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        // Accumulator registers.  A retired slot skips its tcgen05.ld and keeps stale finite
        // values, which never pass the D >= thr test because its thr is +inf.
        uint32_t d[2][kJB];
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int j = 0; j < kJB; ++j) d[k][j] = 0u;
        for (uint32_t c = 0;; ++c) {
            const int s = (int)(c % kSS), ts = (int)(c % kTS);
            // this warpgroup consumed the phase of chunk c - kTS itself, so the parity is unambiguous
            [[maybe_unused]] const long long tw0 = clock64();
            // PROF: was the chunk still unpublished when this warp started waiting (producer-bound)?
            [[maybe_unused]] const bool starved = TGS_RASTER_PROF && !ptx::mbar_test(&sm.full[s], (c / kSS) & 1);
            [[maybe_unused]] bool lockstep = false;  // PROF: a warp of this group still holds the TMEM stage
            if (TGS_RASTER_PROF && !starved && c >= (uint32_t)kTS) {
                const int4 dd = ld_volatile_v4(&sm.wdone[4 * t]);
                lockstep = min(min(dd.x, dd.y), min(dd.z, dd.w)) < (int)(c - kTS + 1);
            }
            ptx::mbar_wait_wd(&sm.tfull[t][ts], (c / kTS) & 1, "epilogue/tfull", (int)c, warp);
            if (TGS_RASTER_PROF) {
                const long long dw = clock64() - tw0;
                pf[1] += dw;
                if (starved) pf[0] += dw;
                if (lockstep) pf_lock += dw;
#if TGS_RASTER_PROF
                if (!starved && !lockstep && dw > 200) {
                    const unsigned long long now = (unsigned long long)clock64(), it = sm.t_iss[t][ts];
                    pf_wake += now > it ? now - it : 0ull;
                    pf_wake_n += 1;
                }
#endif
            }
            ptx::tc_fence_after();
            const ChunkHeader h = sm.hdr[s];
            if (h.chunk != (int)c) {
                if (lane == 0)
                    printf("libtgs epilogue warp %d: expected chunk %d found %d (seq %d)\n", warp, (int)c, h.chunk,
                           h.seq);
                __trap();
            }
            if (h.seq >= 0 && h.seq != cur) {  // first chunk of a unit
                cur = h.seq;
                reported = false;
                const UnitGeom ug = unit_geom<SLOTS>(gg, h.unit);
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int x = ug.tx0 * kTile + relx[k], y = ug.ty0 * kTile + rely[k];
                    const bool inside = x < gg.width && y < gg.height;
                    px[k] = inside ? x : -1;
                    py[k] = y;
                    T[k] = 1.0f;
                    cr[k] = cg[k] = cb[k] = 0.0f;
                    thr[k] = inside ? L : kInf;
                }
                alive = 0;
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    if (__any_sync(0xffffffffu, thr[k] != kInf)) alive |= 1u << k;
            }
            const int nv = h.seq >= 0 ? h.n_valid : 0;
            bool tmem_released = false;
            const uint32_t col0 = (uint32_t)(((ts * SLOTS + t) * 2) * kN);
            if (nv > 0 && alive != 0u) {
#pragma unroll 1
                for (int j0 = 0; j0 < nv; j0 += kJB) {
#pragma unroll
                    for (int k = 0; k < 2; ++k)
                        if (alive & (1u << k)) ptx::tmem_ld16(lane_base + col0 + (uint32_t)(k * kN + j0), d[k]);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < 2; ++k) ptx::reg_fence16(d[k]);
                    if (j0 + kJB >= nv) {
                        // the chunk's accumulators are all in registers: hand the TMEM stage back
                        // before blending, so the next MMA into it overlaps this blend
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ((volatile int*)sm.wdone)[slot] = (int)c + 1;
#if TGS_RASTER_PROF
                        if (lane == 0) atomicMax(&sm.t_rel[t][ts], (unsigned long long)clock64());
#endif
                        tmem_released = true;
                    }
                    // Phase 1 (branch-free, kJB independent chains): which of the batch's splats
                    // reach alpha_skip at any of this warp's pixels -> warp-uniform mask.
                    // D - thr with packed FADD2 over splat pairs (sign bit set <=> D < thr, exactly:
                    // IEEE subtraction of finite values is 0 only for equal operands, -inf for a
                    // retired pixel's +inf); bit jj of `idle` = both pixels below thr, gathered with
                    // one funnel shift per splat
                    uint32_t idle = 0;
#pragma unroll
                    for (int jj = kJB - 2; jj >= 0; jj -= 2) {
                        uint32_t a0, a1, b0, b1;
                        sub_x2(d[0][jj], d[0][jj + 1], thr[0], a0, a1);
                        sub_x2(d[1][jj], d[1][jj + 1], thr[1], b0, b1);
                        idle = __funnelshift_l(a1 & b1, idle, 1);
                        idle = __funnelshift_l(a0 & b0, idle, 1);
                    }
                    const uint32_t M = __reduce_or_sync(0xffffffffu, ~idle & ((1u << kJB) - 1u));
                    if (TGS_RASTER_PROF) {
                        pf[2] += __popc(M);
                        pf[3] += kJB;
                    }
                    // Phase 2: ordered blend of the active splats (uniform branches).  A pixel blends
                    // splat j iff D >= log2(alpha_skip) and it had not terminated before j
                    // (T >= t_terminate): exactly alpha_of/blend/done (raster_scalar.hpp:40-55,
                    // raster_scalar.cpp:36-41) — the splat that drives T below t_terminate is
                    // blended, nothing after it.
#pragma unroll
                    for (int jj = 0; jj < kJB; ++jj)
                        if (M & (1u << jj)) {
                            const float4 ej = sm.epi[s][j0 + jj];
                            float al[2];
#pragma unroll
                            for (int k = 0; k < 2; ++k) {
                                const float dv = __uint_as_float(d[k][jj]);
                                const float e2 = fminf(ej.w, ex2_approx(dv));
                                al[k] = sel_ge2(dv, thr[k], T[k], tterm, e2);
                            }
                            blend_x2(T, cr, cg, cb, al, ej);
                        }
#pragma unroll
                    for (int k = 0; k < 2; ++k)
                        if (T[k] < tterm) thr[k] = kInf;
                }
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    if (!__any_sync(0xffffffffu, thr[k] != kInf)) alive &= ~(1u << k);
            }
            if (h.seq >= 0 && h.last) {  // unit complete: store its pixels (clamped, finalize)
#pragma unroll
                for (int k = 0; k < 2; ++k)
                    if (px[k] >= 0) {
                        float* o = a.image + ((size_t)(py[k] - a.image_row0) * gg.width + px[k]) * 3;
                        o[0] = fminf(fmaxf(cr[k], 0.0f), 1.0f);
                        o[1] = fminf(fmaxf(cg[k], 0.0f), 1.0f);
                        o[2] = fminf(fmaxf(cb[k], 0.0f), 1.0f);
                    }
            }
            // TMEM stage and smem stage consumed (all tcgen05.ld of this warp completed above)
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (h.seq >= 0 && alive == 0u && !reported) ((volatile int*)sm.dead)[slot] = (cur << 1) | 1;
                __threadfence_block();
                if (!tmem_released) ((volatile int*)sm.wdone)[slot] = (int)c + 1;
#if TGS_RASTER_PROF
                if (!tmem_released) atomicMax(&sm.t_rel[t][ts], (unsigned long long)clock64());
#endif
                atomicAdd(&sm.done_cnt[s], 1u);
            }
            reported = reported || (h.seq >= 0 && alive == 0u);
            if (h.seq < 0) break;
        }
    }

#if TGS_RASTER_PROF
    if (lane == 0) {
        const long long tot = clock64() - pf_start;
        if (warp == kProd) {
            atomicAdd(&g_rprof[0], (unsigned long long)tot);
            atomicAdd(&g_rprof[1], pf[1]);
            atomicAdd(&g_rprof[8], pf[2]);   // cp.async data waits
            atomicAdd(&g_rprof[9], pf[3]);   // batches
            atomicAdd(&g_rprof[10], pf[0]);  // chunks
        } else if (warp == kMma) {
            atomicAdd(&g_rprof[2], (unsigned long long)tot);
            atomicAdd(&g_rprof[14], pf[0]);
            atomicAdd(&g_rprof[15], pf[2]);
            atomicAdd(&g_rprof_seen, pf[1]);
            atomicAdd(&g_rprof[9 + 0], 0ull);
            atomicAdd(&g_rprof_issue, pf[3]);
        } else {
            atomicAdd(&g_rprof[3], (unsigned long long)tot);
            atomicAdd(&g_rprof[4], pf[1]);
            atomicAdd(&g_rprof[5], pf[2]);
            atomicAdd(&g_rprof[6], pf[3]);
            atomicAdd(&g_rprof[7], pf[0]);
            atomicAdd(&g_rprof[11], pf_lock);
            atomicAdd(&g_rprof[12], pf_wake);
            atomicAdd(&g_rprof[13], pf_wake_n);
        }
    }
#endif
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == kMma) ptx::tmem_dealloc<kTmemCols>(tmem);
#if TGS_RASTER_PROF
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&g_rprof_done, 1u) == gridDim.x - 1) {
            unsigned long long v[16];
            for (int i = 0; i < 16; ++i) v[i] = atomicExch(&g_rprof[i], 0ull);
            printf("RPROF2 per CTA: producer gather waits %.0f batches %.0f chunks %.0f | epi/warp waits on its own "
                   "group's TMEM stage %.0f\n", v[8] / (double)gridDim.x, v[9] / (double)gridDim.x,
                   v[10] / (double)gridDim.x, v[11] / (double)gridDim.x / kEpiWarps);
            const unsigned long long iss = atomicExch(&g_rprof_issue, 0ull);
            const unsigned long long seen = atomicExch(&g_rprof_seen, 0ull);
            printf("RPROF4 MMA ready->noticed %.0f cycles/issue, MMA loop iterations/CTA %.0f\n",
                   seen / (double)(v[15] ? v[15] : 1), atomicExch(&g_rprof_iters, 0ull) / (double)gridDim.x);
            printf("RPROF3 MMA ready->issued %.0f cycles/issue (issue itself %.0f; %.0f issues/CTA) | commit->epilogue "
                   "wake %.0f cycles (%.0f waits/CTA)\n", v[14] / (double)(v[15] ? v[15] : 1),
                   iss / (double)(v[15] ? v[15] : 1), v[15] / (double)gridDim.x,
                   v[12] / (double)(v[13] ? v[13] : 1), v[13] / (double)gridDim.x);
            g_rprof_done = 0;
            const double n = (double)gridDim.x;
            printf("RPROF ctas %d | producer total %.0f wait %.0f | mma total %.0f | epi/warp total %.0f "
                   "wtfull %.0f (producer-starved %.0f) | active %.3f of %.0f (warp, splat) per warp\n",
                   gridDim.x, v[0] / n, v[1] / n, v[2] / n, v[3] / n / kEpiWarps, v[4] / n / kEpiWarps,
                   v[7] / n / kEpiWarps, (double)v[5] / (double)(v[6] ? v[6] : 1), v[6] / n / kEpiWarps);
        }
    }
#endif
}

template <int SLOTS>
void launch_t(const RasterArgs& a, int num_sms, cudaStream_t st) {
    const size_t smem = sizeof(Smem<SLOTS>);
    cudaFuncSetAttribute(raster_tensor_kernel<SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int n_units = a.gg.n_groups_band * units_per_group<SLOTS>(a.gg.g);
    int grid = num_sms * Cfg<SLOTS>::kCtasPerSm;
    if (grid > n_units) grid = n_units;
    if (grid > 0) raster_tensor_kernel<SLOTS><<<grid, Cfg<SLOTS>::kThreads, smem, st>>>(a);
}

}  // namespace

void launch_raster_tensor(const RasterArgs& a, int num_sms, cudaStream_t st) {
    if (a.gg.g == 1)
        launch_t<1>(a, num_sms, st);
    else
        launch_t<4>(a, num_sms, st);
}

int raster_units_per_group(int g) { return g == 4 ? 4 : 1; }

}  // namespace tgs
