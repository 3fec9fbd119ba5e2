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
// the centre o of the 2x2-tile unit:  u = pixel - o, m = mean - o,
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
// CTA (persistent, one per SM) = one unit of 2x2 tiles at a time (G=2: the group; G=4: a
// quarter group; G=1: a single tile with SLOTS = 1), units in the order of the previous frame's
// measured walks (unit_order_kernel):
//   epilogue warps (8): compact mapping — warp w owns the 16x8 half-tile w and reads TMEM lane
//              quadrant w%4 of M-tiles 4*(w/4)+k, k<4 (its four 8x4 pixel blocks), so each thread
//              owns four pixels of one half-tile; the ordered blend runs on CUDA cores + MUFU ex2;
//              a half-tile whose pixels all terminated drops out at once;
//   producer warp: streams the unit's list in 32-entry batches (records two batches ahead), gathers
//              each splat once per group, drops entries whose member tiles are all retired or
//              that can never reach alpha_skip (ballot compaction keeps list order), and writes the
//              unit-centred coefficient rows (+ mask lanes) and blend data into an smem stage;
//   MMA warp:  TMEM owner; per chunk one tcgen05.mma (M=128, N=32, K=16) per live M-tile into a
//              TMEM stage (2 stages x 2*SLOTS M-tiles x 32 columns), issued from warp-uniform code
//              by an elected lane, then tcgen05.commit -> epilogue.
// The pixel operand A (2*SLOTS M-tiles x 128 rows x 32 B) is identical for every unit and is
// built once per CTA.  Hand-offs: full[s] (mbarrier), tfull[ts] (tcgen05.commit), and release
// counters compared against absolute chunk targets; every wait is watchdog-bounded.
#include <cstdlib>
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"
#include "tgs_ptx.cuh"

#include <algorithm>

namespace tgs {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kNeverRow = -30000.0f;
constexpr float kInf = __builtin_huge_valf();

#ifndef TGS_RASTER_N
#define TGS_RASTER_N 32
#endif
constexpr int kN = TGS_RASTER_N;  // splats per chunk (MMA N): 16 or 32
#ifndef TGS_RASTER_SS
#define TGS_RASTER_SS 3
#endif
constexpr int kSS = TGS_RASTER_SS;  // smem stages
#ifndef TGS_RASTER_TS
#define TGS_RASTER_TS 2
#endif
constexpr int kTS = TGS_RASTER_TS;  // TMEM accumulator stages
#ifndef TGS_RASTER_SPW
#define TGS_RASTER_SPW 4
#endif
#ifndef TGS_RASTER_CTAS
#define TGS_RASTER_CTAS 1
#endif
constexpr int kCtasPerSm = TGS_RASTER_CTAS;  // resident CTAs per SM (TMEM columns must fit)
#ifndef TGS_RASTER_CTAS_G1
#define TGS_RASTER_CTAS_G1 1
#endif
#ifndef TGS_RASTER_SPW2
#define TGS_RASTER_SPW2 4
#endif
#ifndef TGS_RASTER_HALF
#define TGS_RASTER_HALF 0
#endif
// units per group and resident CTAs per SM of the SLOTS instance: SLOTS = 2 rasterises a G=2 group
// as two half units (its top and bottom tile rows), two CTAs per SM (256 TMEM columns each)
template <int SLOTS>
constexpr int ctas_per_sm() { return SLOTS == 1 ? TGS_RASTER_CTAS_G1 : SLOTS == 2 ? 2 : kCtasPerSm; }
template <int SLOTS>
__host__ __device__ inline int units_per_group(int g) { return SLOTS == 2 ? 2 : (SLOTS == 4 && g == 4) ? 4 : 1; }
#ifndef TGS_RASTER_JB
#define TGS_RASTER_JB 16
#endif
constexpr int kJB = TGS_RASTER_JB;  // accumulator columns (splats) per epilogue batch: 16 or 8
#ifndef TGS_RASTER_ATMEM
#define TGS_RASTER_ATMEM 0
#endif
constexpr bool kATmem = TGS_RASTER_ATMEM;  // pixel operand A held in TMEM (8 columns per M-tile)
#ifndef TGS_RASTER_PROF
#define TGS_RASTER_PROF 0
#endif
#if TGS_RASTER_PROF
// role timing (debug builds only): [0] producer total [1] producer stage waits [2] producer
// batches [3] chunks; [4] MMA total [5] MMA full waits [6] MMA TMEM-release waits; [8] epilogue
// total (sum over warps) [9] epilogue tfull waits [10] active splat blocks [11] splat blocks
__device__ unsigned long long g_rprof[16];
__device__ unsigned int g_rprof_done;
__device__ unsigned int g_ucyc[65536];  // per-unit cycles (unit index) and start order
__device__ unsigned int g_uch[65536];
__device__ unsigned int g_uent[65536];
__device__ unsigned int g_uwait[65536];  // producer stage-wait cycles within the unit
__device__ unsigned int g_usec[65536][3];  // producer cycles: retire check, row build, placement
#endif
#ifndef TGS_RASTER_COMPACT
#define TGS_RASTER_COMPACT 1
#endif
#ifndef TGS_RASTER_PAIR  // producer batches built together before placement: 1, 2 or 4
#define TGS_RASTER_PAIR 2
#endif
#ifndef TGS_RASTER_TIGHT
#define TGS_RASTER_TIGHT 1
#endif
constexpr bool kTightCover = TGS_RASTER_TIGHT;  // producer drops splats by the alpha_skip ellipse box
#ifndef TGS_RASTER_PREFETCH4
#define TGS_RASTER_PREFETCH4 0
#endif
#ifndef TGS_RASTER_STREAMS
#define TGS_RASTER_STREAMS 1
#endif

struct ChunkHeader {
    int seq;      // per-CTA unit sequence number, -1 = end of stream
    int unit;     // unit index (order-resolved)
    int n_valid;  // splats in the chunk (0: unit without contributing splats)
    int live;     // member tiles live when the chunk was produced (MMA skips the others)
    int chunk;    // chunk number (protocol self-check)
};

// Roles: SLOTS member tiles per unit -> 2*SLOTS M=128 tiles.  Each epilogue warp owns SPW
// (slot) pixel blocks: lane quadrant q = warp % 4 (the TMEM lanes it may read) of M-tiles
// 2*(k0+i) + half, i < SPW; so each thread owns one pixel in SPW member tiles.
template <int SLOTS>
struct Roles {
    static constexpr int kMT = 2 * SLOTS;
    static constexpr int kSPW = SLOTS == 1 ? 1 : SLOTS == 2 ? TGS_RASTER_SPW2 : TGS_RASTER_SPW;  // slots per warp
    static constexpr int kEpiWarps = 8 * SLOTS / kSPW;         // 16 (G>=2) or 8 (G=1)
    static constexpr int kThreads = (kEpiWarps + 2) * 32;
    static constexpr int kProd = kEpiWarps, kMma = kEpiWarps + 1;
    static constexpr bool kCompact = SLOTS >= 2 && kSPW == 4 && TGS_RASTER_COMPACT;
    // chunk streams: with 2, the unit's top tile row (tiles 0,1: warps 0-3, M-tiles 0-3) and bottom
    // row (tiles 2,3: warps 4-7, M-tiles 4-7) get their own chunk streams carrying only the splats
    // that overlap them, and progress independently
    static constexpr int kNS = (kCompact && TGS_RASTER_STREAMS == 2) ? 2 : 1;
};

template <int SLOTS>
struct Smem {
    static constexpr int kMT = 2 * SLOTS;
    static constexpr int kNS = Roles<SLOTS>::kNS;
    alignas(128) uint8_t a[kMT][128 * 32];   // pixel monomial rows (K-major, no swizzle)
    alignas(128) uint8_t b[kNS][kSS][kN * 32];  // splat coefficient rows, per stream
    float4 epi[kNS][kSS][kN];                // r, g, b, min(alpha_clamp, opacity)
    ChunkHeader hdr[kNS][kSS];
    alignas(16) int wdone[16];               // chunks (of its stream) each epilogue warp has completed
    alignas(16) int dead[16];                // (seq << 4) | retired member tiles, per warp
    uint64_t full[kNS][kSS];                 // producer -> MMA
    uint64_t tfull[kNS][kTS];                // MMA -> epilogue (tcgen05.commit)
    // Releases are monotonic counters compared with absolute targets (no mbarrier phase
    // aliasing): done_cnt[s] = warps that finished a chunk on smem stage s; a TMEM stage is free
    // once every epilogue warp's wdone passed the chunk that used it.
    unsigned int done_cnt[kNS][kSS];
    uint32_t tmem_base;
};

template <int SLOTS>
constexpr uint32_t tmem_cols() {
    constexpr int c = kTS * 2 * SLOTS * kN + (kATmem ? 8 * 2 * SLOTS : 0);
    return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

// Pixel (relative to the unit's top-left) of TMEM lane l of M-tile m = 2*slot + half: the lane
// quadrant q = l/32 is an 8x4 block of the half tile, so an epilogue warp's 32 pixels are
// spatially compact and a splat footprint touches few warps.
__device__ __forceinline__ void lane_pixel(int m, int l, int& x, int& y) {
    const int slot = m >> 1, half = m & 1;
    const int q = l >> 5, i = l & 31;
    x = (slot & 1) * 16 + (q & 1) * 8 + (i & 7);
    y = (slot >> 1) * 16 + half * 8 + (q >> 1) * 4 + (i >> 3);
}

// Compact mapping (G >= 2 with 4 slots per warp): epilogue warp w owns half-tile w of the unit
// (tile w >> 1, rows (w & 1) * 8 ..), its slot k is the 8x4 block k of that half-tile.  Warp w may
// only read TMEM lane quadrant w % 4, so its slots live in M-tiles 4 * (w >> 2) + k at quadrant
// w % 4.  A splat footprint then activates the few warps whose half-tiles it overlaps, and all four
// slots of an active warp are spatially adjacent.
__device__ __forceinline__ void lane_pixel_compact(int m, int l, int& x, int& y) {
    const int w = 4 * (m >> 2) + (l >> 5), k = m & 3, i = l & 31;
    const int t = w >> 1;
    x = (t & 1) * 16 + (k & 1) * 8 + (i & 7);
    y = (t >> 1) * 16 + (w & 1) * 8 + (k >> 1) * 4 + (i >> 3);
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

// 0xffffffff if a >= b else 0 (opaque to CSE, so the blend's own compare stays a predicate)
__device__ __forceinline__ uint32_t fset_ge(float a, float b) {
    uint32_t r;
    asm volatile("set.ge.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
    return r;
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
__device__ __forceinline__ void write_row(Smem<SLOTS>& sm, int h, int s, int slot, const uint4& r0, const uint4& r1) {
    *reinterpret_cast<uint4*>(&sm.b[h][s][core_off(slot, 0)]) = r0;
    *reinterpret_cast<uint4*>(&sm.b[h][s][core_off(slot, 1)]) = r1;
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
        const int gx = unit % gg.groups_x, gy = unit / gg.groups_x + gg.band_gy0;
        u.tx0 = gx;
        u.ty0 = gy;
        u.gid = unit;
        u.live = 1u;
        return u;
    }
    // G == 2: unit == group (SLOTS 4) or tile row of a group (SLOTS 2); G == 4: unit == quarter
    // (2x2 tiles) of a group
    const int per = units_per_group<SLOTS>(gg.g);
    const int grp = unit / per, quarter = unit % per;
    const int gx = grp % gg.groups_x, gy = grp / gg.groups_x + gg.band_gy0;
    if (SLOTS == 2) {
        u.tx0 = gx * gg.g;
        u.ty0 = gy * gg.g + quarter;
    } else {
        u.tx0 = gx * gg.g + (quarter & 1) * 2;
        u.ty0 = gy * gg.g + (quarter >> 1) * 2;
    }
    u.gid = grp;
    u.live = 0u;
#pragma unroll
    for (int t = 0; t < SLOTS; ++t)
        if (u.tx0 + (t & 1) < gg.tiles_x && u.ty0 + (t >> 1) < gg.tiles_y) u.live |= 1u << t;
    return u;
}

template <int SLOTS, int P2>
__global__ void __launch_bounds__(Roles<SLOTS>::kThreads, ctas_per_sm<SLOTS>()) raster_tensor_kernel(RasterArgs a) {
    using R = Roles<SLOTS>;
    constexpr int kMT = R::kMT, SPW = R::kSPW, kEpiWarps = R::kEpiWarps;
    constexpr int kProd = R::kProd, kMma = R::kMma;
    constexpr bool kCompact = R::kCompact;
    constexpr int kNS = R::kNS, kWPS = kEpiWarps / kNS, kMPS = kMT / kNS;  // warps, M-tiles per stream
    constexpr int kColsPerStage = kMT * kN;
    constexpr uint32_t kTmemCols = tmem_cols<SLOTS>();
    // No-swizzle K-major operands only need 16-byte alignment (descriptor addresses are >> 4).
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem<SLOTS>& sm = *reinterpret_cast<Smem<SLOTS>*>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const GroupGeom& gg = a.gg;
    const int n_units = SLOTS == 1 ? gg.n_groups_band : gg.n_groups_band * units_per_group<SLOTS>(gg.g);
    const float centre = SLOTS == 1 ? 8.0f : 16.0f;

    // ---- setup: A operand (pixel monomials + tile one-hot), barriers, TMEM -----------------
    for (int p = threadIdx.x; p < kMT * 128; p += blockDim.x) {
        const int m = p >> 7, l = p & 127;
        int x, y;
        if (kCompact)
            lane_pixel_compact(m, l, x, y);
        else
            lane_pixel(m, l, x, y);
        const float ux = (float)x + 0.5f - centre, uy = (float)y + 0.5f - centre;
        const float phi[6] = {ux * ux, ux * uy, uy * uy, ux, uy, 1.0f};
        const int t = kCompact ? 2 * (m >> 2) + (l >> 6) : m >> 1;
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
        sm.wdone[threadIdx.x] = threadIdx.x < kEpiWarps ? 0 : 0x7fffffff;
        sm.dead[threadIdx.x] = -1;
    }
    if (threadIdx.x == 0) {
        for (int h = 0; h < kNS; ++h) {
            for (int s = 0; s < kSS; ++s) {
                ptx::mbar_init(&sm.full[h][s], 1);
                sm.done_cnt[h][s] = 0;
            }
            for (int s = 0; s < kTS; ++s) ptx::mbar_init(&sm.tfull[h][s], 1);
        }
        ptx::mbar_fence_init();
    }
    if (warp == kMma) ptx::tmem_alloc<kTmemCols>(&sm.tmem_base);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    constexpr uint32_t kACol = (uint32_t)(kTS * kColsPerStage);  // A operand columns (kATmem)
    if constexpr (kATmem) {
        // warps 0..3 write the pixel operand rows of their lane quadrant into TMEM (row = lane,
        // K pairs in 8 consecutive 32-bit columns)
        if (warp < 4) {
            for (int m = 0; m < kMT; ++m) {
                const int l = warp * 32 + lane;
                const uint4 lo = *reinterpret_cast<const uint4*>(&sm.a[m][core_off(l, 0)]);
                const uint4 hi = *reinterpret_cast<const uint4*>(&sm.a[m][core_off(l, 1)]);
                const uint32_t r[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
                ptx::tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + kACol + (uint32_t)(8 * m), r);
            }
            ptx::tmem_wait_st();
        }
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
    }
    [[maybe_unused]] unsigned long long pf[4] = {0, 0, 0, 0};
    [[maybe_unused]] const long long pf_start = clock64();

    if (warp == kProd) {
        // ================================ producer ===========================================
        const float skip = a.alpha_skip, clampv = a.alpha_clamp;
        uint32_t c[kNS];  // chunks emitted so far, per stream
#pragma unroll
        for (int h = 0; h < kNS; ++h) c[h] = 0;
        const uint32_t lt = (1u << lane) - 1u;
        auto open_stage = [&](int h, uint32_t cc) {
            // stage cc % kSS of stream h is free once the stream's epilogue warps finished chunk
            // cc - kSS (lane 0 polls, the warp reconverges after)
            const int s = (int)(cc % kSS);
            if (cc >= (uint32_t)kSS && lane == 0) {
                const unsigned int need = (unsigned int)kWPS * (cc / kSS);
                if (ld_volatile_u32(&sm.done_cnt[h][s]) < need) {
                    const long long t0 = clock64();
                    while (ld_volatile_u32(&sm.done_cnt[h][s]) < need) {
                        __nanosleep(32);
                        if (clock64() - t0 > 4000000000ll) ptx::watchdog_trap("producer/done", (int)cc, s);
                    }
                    if (TGS_RASTER_PROF) pf[1] += clock64() - t0;
                }
            }
            __syncwarp();
            return s;
        };
        auto publish = [&](int h, int s, int seq, int unit, int n_valid, uint32_t live) {
            if (lane == 0) {
                sm.hdr[h][s].seq = seq;
                sm.hdr[h][s].unit = unit;
                sm.hdr[h][s].n_valid = n_valid;
                sm.hdr[h][s].live = (int)live;
                sm.hdr[h][s].chunk = (int)c[h];
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&sm.full[h][s]);
            __syncwarp();
        };
        // member tiles of stream h
        auto smask = [&](int h) -> uint32_t { return kNS == 1 ? 0xfu : (h == 0 ? 0x3u : 0xcu); };
        for (int seq = 0;; ++seq) {
            int t = 0;
            if (lane == 0) t = (int)atomicAdd(&a.fc->group_counter, 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n_units) break;
            const int unit = a.order ? a.order[t] : t;
            const UnitGeom ug = unit_geom<SLOTS>(gg, unit);
            [[maybe_unused]] const long long unit_t0 = clock64();
            [[maybe_unused]] uint32_t unit_c0 = 0;
#pragma unroll
            for (int h = 0; h < kNS; ++h) unit_c0 += c[h];
            [[maybe_unused]] const unsigned long long unit_w0 = pf[1];
            [[maybe_unused]] unsigned long long sec[3] = {0, 0, 0};
            const uint32_t begin = a.offsets[ug.gid], end = a.offsets[ug.gid + 1];
            const float ox = (float)(ug.tx0 * kTile) + centre, oy = (float)(ug.ty0 * kTile) + centre;
            int fill[kNS], s[kNS];   // rows placed in the open chunk / its stage, per stream
            bool open[kNS];          // a stage is open for this unit
            bool emitted_h[kNS];     // at least one chunk of this unit emitted
#pragma unroll
            for (int h = 0; h < kNS; ++h) {
                fill[h] = 0;
                s[h] = 0;
                open[h] = false;
                emitted_h[h] = false;
            }
            bool emitted = false;    // any stream
            uint32_t live = ug.live;
            // software-pipelined gather: list indices two batches ahead, records one ahead
            const uint32_t nb = (end - begin + 31u) / 32u;
            auto ld_idx = [&](uint32_t b) -> uint32_t {
                const uint32_t e = begin + b * 32u + (uint32_t)lane;
                return (b < nb && e < end) ? __ldg(&a.list[e]) : 0xffffffffu;
            };
            struct Rec {
                float4 mc, co, col;
                uint32_t idx;
            };
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
            // Software-pipelined gather without register moves of in-flight loads (a move would
            // wait on the load's scoreboard): two record slots consumed in turn, each refilled two
            // batches ahead right after use; list indices four batches ahead.
            uint32_t n_batches = 0;
            // one batch: retire check, row build, ordered placement; true = unit finished
            // producer work on one batch, in three parts: the retire check (drops member tiles
            // whose pixels all terminated), the build (cover tests and coefficient rows per lane)
            // and the ordered placement into the open chunk(s)
            struct Built {
                bool keep;
                uint32_t cover;
                uint4 r0, r1;
                float4 epi;
            };
            auto retire_check = [&]() -> bool {  // true = every member tile retired
                if (emitted) {
                    uint32_t retired = 0xfu;
#pragma unroll
                    for (int w4 = 0; w4 < kEpiWarps; w4 += 4) {
                        const int4 d = ld_volatile_v4(&sm.dead[w4]);
                        const int dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int w = w4 + j;
                            const uint32_t owned =
                                kCompact ? 1u << (w >> 1) : ((1u << SPW) - 1u) << ((w >> 3) * SPW);
                            retired &= ((dd[j] >> 4) == seq ? (uint32_t)(dd[j] & 15) : 0u) | (0xfu & ~owned);
                        }
                    }
                    // sm.dead is written concurrently by the epilogue warps: take lane 0's view so
                    // the whole warp makes the same decision (lanes may read it at different times)
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
                    int x0, y0, x1, y1;
                    tile_rect(cur.mc.x, cur.mc.y, __float_as_int(cur.co.w), gg.tiles_x, gg.tiles_y, x0, y0, x1, y1);
                    uint32_t cover = 0;
#pragma unroll
                    for (int k = 0; k < SLOTS; ++k) {
                        const int tx = ug.tx0 + (k & 1), ty = ug.ty0 + (k >> 1);
                        if (tx >= x0 && tx <= x1 && ty >= y0 && ty <= y1) cover |= 1u << k;
                    }
                    cover &= live;
                    const float cj = fminf(clampv, cur.co.y);
                    if (kTightCover && a.tile_cull && cover != 0u && !(cj < skip))
                        cover &= tight_cover(cur.mc.x, cur.mc.y, cur.col.w, ug.tx0, ug.ty0, SLOTS);
                    if (cover != 0u && !(cj < skip)) {
                        bt.keep = make_row(cur.mc.x, cur.mc.y, cur.mc.z, cur.mc.w, cur.co.x, lg2_approx(cur.co.y), ox,
                                           oy, cover, bt.r0, bt.r1);
                        bt.cover = cover;
                        bt.epi = make_float4(cur.col.x, cur.col.y, cur.col.z, cj);
                    }
                }
            };
            auto place = [&](const Built& bt) {
#pragma unroll
                for (int h = 0; h < kNS; ++h) {
                    const bool keep_h = bt.keep && (bt.cover & smask(h)) != 0u;
                    const uint32_t km = __ballot_sync(0xffffffffu, keep_h);
                    if (km == 0u) continue;
                    const int nk = __popc(km);
                    const int rank = __popc(km & lt);
                    if (!open[h]) {
                        s[h] = open_stage(h, c[h]);
                        open[h] = true;
                        fill[h] = 0;
                    }
                    // place the kept ranks in order; a full chunk is published and the next one
                    // opened (a 32-lane batch spans at most 32 / kN + 1 chunks)
                    int placed = 0;
                    for (;;) {
                        const int room = kN - fill[h];
                        if (keep_h && rank >= placed && rank - placed < room) {
                            write_row(sm, h, s[h], fill[h] + rank - placed, bt.r0, bt.r1);
                            sm.epi[h][s[h]][fill[h] + rank - placed] = bt.epi;
                        }
                        if (nk - placed < room) {
                            fill[h] += nk - placed;
                            break;
                        }
                        publish(h, s[h], seq, unit, kN, live & smask(h));
                        ++c[h];
                        emitted = true;
                        emitted_h[h] = true;
                        s[h] = open_stage(h, c[h]);
                        fill[h] = 0;
                        placed += room;
                        if (placed == nk) break;
                    }
                }
            };
            auto batch = [&](const Rec& cur) -> bool {
                ++n_batches;
                [[maybe_unused]] const long long tb0 = TGS_RASTER_PROF ? clock64() : 0;
                if (retire_check()) return true;
                [[maybe_unused]] const long long tb1 = TGS_RASTER_PROF ? clock64() : 0;
                Built bt;
                build(cur, bt);
                [[maybe_unused]] const long long tb2 = TGS_RASTER_PROF ? clock64() : 0;
                if (TGS_RASTER_PROF) {
                    pf[2] += 1;
                    sec[0] += tb1 - tb0;
                    sec[1] += tb2 - tb1;
                }
                place(bt);
                if (TGS_RASTER_PROF) sec[2] += clock64() - tb2;
                return false;
            };
            // pair mode: two batches built back to back (independent work overlaps), then placed
            // in list order
            [[maybe_unused]] auto batch_pair = [&](const Rec& ca, const Rec& cb, bool has_b) -> bool {
                n_batches += has_b ? 2u : 1u;
                if (retire_check()) return true;
                Built ba, bb;
                build(ca, ba);
                if (has_b) build(cb, bb);
                place(ba);
                if (has_b) place(bb);
                return false;
            };
#if TGS_RASTER_PREFETCH4
            Rec q0 = ld_rec(ld_idx(0)), q1 = ld_rec(ld_idx(1)), q2 = ld_rec(ld_idx(2)), q3 = ld_rec(ld_idx(3));
            uint32_t i0 = ld_idx(4), i1 = ld_idx(5), i2 = ld_idx(6), i3 = ld_idx(7);
            for (uint32_t bi = 0; bi < nb; bi += 4) {
                if (batch(q0)) break;
                q0 = ld_rec(i0);
                i0 = ld_idx(bi + 8);
                if (bi + 1 >= nb || batch(q1)) break;
                q1 = ld_rec(i1);
                i1 = ld_idx(bi + 9);
                if (bi + 2 >= nb || batch(q2)) break;
                q2 = ld_rec(i2);
                i2 = ld_idx(bi + 10);
                if (bi + 3 >= nb || batch(q3)) break;
                q3 = ld_rec(i3);
                i3 = ld_idx(bi + 11);
            }
#elif TGS_RASTER_PAIR == 4
            Rec q0 = ld_rec(ld_idx(0)), q1 = ld_rec(ld_idx(1)), q2 = ld_rec(ld_idx(2)), q3 = ld_rec(ld_idx(3));
            uint32_t i0 = ld_idx(4), i1 = ld_idx(5), i2 = ld_idx(6), i3 = ld_idx(7);
            for (uint32_t bi = 0; bi < nb; bi += 4) {
                n_batches += min(4u, nb - bi);
                if (retire_check()) break;
                Built b0, b1, b2, b3;
                build(q0, b0);
                build(q1, b1);
                build(q2, b2);
                build(q3, b3);
                place(b0);
                place(b1);
                place(b2);
                place(b3);
                q0 = ld_rec(i0);
                q1 = ld_rec(i1);
                q2 = ld_rec(i2);
                q3 = ld_rec(i3);
                i0 = ld_idx(bi + 8);
                i1 = ld_idx(bi + 9);
                i2 = ld_idx(bi + 10);
                i3 = ld_idx(bi + 11);
            }
#elif TGS_RASTER_PAIR == 2
            Rec qa = ld_rec(ld_idx(0)), qb = ld_rec(ld_idx(1));
            uint32_t ia = ld_idx(2), ib = ld_idx(3);
            for (uint32_t bi = 0; bi < nb; bi += 2) {
                if (batch_pair(qa, qb, bi + 1 < nb)) break;
                qa = ld_rec(ia);
                qb = ld_rec(ib);
                ia = ld_idx(bi + 4);
                ib = ld_idx(bi + 5);
            }
#else
            Rec qa = ld_rec(ld_idx(0)), qb = ld_rec(ld_idx(1));
            uint32_t ia = ld_idx(2), ib = ld_idx(3);
            for (uint32_t bi = 0; bi < nb; bi += 2) {
                if (batch(qa)) break;
                qa = ld_rec(ia);
                ia = ld_idx(bi + 4);
                if (bi + 1 >= nb) break;
                if (batch(qb)) break;
                qb = ld_rec(ib);
                ib = ld_idx(bi + 5);
            }
#endif
            // close the unit: pad and publish the partial chunk (or an empty one so the
            // epilogue still writes the unit's pixels)
#pragma unroll
            for (int h = 0; h < kNS; ++h) {
                if (open[h] && (fill[h] > 0 || !emitted_h[h])) {
                    if (lane >= fill[h] && lane < kN) {
                        uint4 r0, r1;
                        never_row(r0, r1);
                        write_row(sm, h, s[h], lane, r0, r1);
                    }
                    publish(h, s[h], seq, unit, fill[h], live & smask(h));
                    ++c[h];
                } else if (!open[h]) {
                    s[h] = open_stage(h, c[h]);
                    publish(h, s[h], seq, unit, 0, live & smask(h));
                    ++c[h];
                }
            }
            uint32_t c_now = 0;
#pragma unroll
            for (int h = 0; h < kNS; ++h) c_now += c[h];
            // schedule feedback: list entries this unit walked (batches) plus rows it staged
            if (a.unit_cost && lane == 0) a.unit_cost[unit] = 32u * n_batches + (uint32_t)kN * (c_now - unit_c0);
#if TGS_RASTER_PROF
            if (lane == 0) {
                atomicMax(&g_rprof[13], (unsigned long long)(clock64() - unit_t0));
                atomicMax(&g_rprof[14], (unsigned long long)(c_now - unit_c0));
                if (unit < 65536) {
                    g_ucyc[unit] = (unsigned int)(clock64() - unit_t0);
                    g_uch[unit] = c_now - unit_c0;
                    g_uent[unit] = (unsigned)t;
                    g_uwait[unit] = (unsigned)(pf[1] - unit_w0);
                    for (int k = 0; k < 3; ++k) g_usec[unit][k] = (unsigned)sec[k];
                }
            }
#endif
        }
#pragma unroll
        for (int h = 0; h < kNS; ++h) {  // end of stream
            const int se = open_stage(h, c[h]);
            publish(h, se, -1, -1, 0, 0u);
        }
    } else if (warp == kMma) {
        // ================================ MMA issuer ==========================================
        constexpr uint32_t idesc = ptx::idesc_f16(128, kN);
        const uint32_t a_base = ptx::smem_u32(&sm.a[0][0]);
        uint32_t cs[kNS];
        bool ended[kNS];
#pragma unroll
        for (int h = 0; h < kNS; ++h) {
            cs[h] = 0;
            ended[h] = false;
        }
        int n_ended = 0;
        long long idle0 = clock64();
        // stream h's TMEM stage for chunk c is free once its warps finished chunk c - kTS
        auto released = [&](int h, int need) {
            int mn = 0x7fffffff;
#pragma unroll
            for (int w4 = 0; w4 < kWPS; w4 += 4) {
                const int4 d = ld_volatile_v4(&sm.wdone[h * kWPS + w4]);
                mn = min(mn, min(min(d.x, d.y), min(d.z, d.w)));
            }
            return mn >= need;
        };
        while (n_ended < kNS) {
            bool did = false;
#pragma unroll
            for (int h = 0; h < kNS; ++h) {
                if (ended[h]) continue;
                const uint32_t c = cs[h];
                const int s = (int)(c % kSS), ts = (int)(c % kTS);
                int ready = 0;
                if (lane == 0)
                    ready = ptx::mbar_test(&sm.full[h][s], (c / kSS) & 1) &&
                            (c < (uint32_t)kTS || released(h, (int)(c - kTS + 1)));
                ready = __shfl_sync(0xffffffffu, ready, 0);
                if (!ready) continue;
                __syncwarp();
                ptx::tc_fence_after();
                // warp-uniform issue (operands stay uniform; one elected lane issues)
                const int hseq = __shfl_sync(0xffffffffu, sm.hdr[h][s].seq, 0);
                const int hnv = __shfl_sync(0xffffffffu, sm.hdr[h][s].n_valid, 0);
                const uint32_t hlive = __shfl_sync(0xffffffffu, (uint32_t)sm.hdr[h][s].live, 0);
                const int hch = __shfl_sync(0xffffffffu, sm.hdr[h][s].chunk, 0);
                if (hch != (int)c) {
                    if (lane == 0)
                        printf("MMA header mismatch: stream %d expected chunk %d found %d (seq %d)\n", h, (int)c, hch, hseq);
                    __trap();
                }
                [[maybe_unused]] const long long ti0 = TGS_RASTER_PROF ? clock64() : 0;
                if (hseq >= 0 && hnv > 0) {
                    const uint64_t bd = ptx::smem_desc(ptx::smem_u32(&sm.b[h][s][0]), 128, 256);
                    const uint32_t dcol = tmem + (uint32_t)(ts * kColsPerStage);
#pragma unroll
                    for (int mm = 0; mm < kMPS; ++mm) {
                        const int m = h * kMPS + mm;
                        if (kCompact ? ((hlive >> (2 * (m >> 2))) & 3u) : ((hlive >> (m >> 1)) & 1u)) {
                            if constexpr (kATmem)
                                ptx::mma_f16_ts_elect(dcol + (uint32_t)(m * kN), tmem + kACol + (uint32_t)(8 * m), bd,
                                                      idesc, 0u);
                            else
                                ptx::mma_f16_ss_elect(dcol + (uint32_t)(m * kN),
                                                      ptx::smem_desc(a_base + (uint32_t)(m * 128 * 32), 128, 256), bd,
                                                      idesc, 0u);
                        }
                    }
                    ptx::mma_commit_elect(&sm.tfull[h][ts]);
                } else if (lane == 0) {
                    ptx::mbar_arrive(&sm.tfull[h][ts]);
                }
                __syncwarp();
                if (TGS_RASTER_PROF) pf[3] += clock64() - ti0;
                cs[h] = c + 1;
                if (hseq < 0) {
                    ended[h] = true;
                    ++n_ended;
                }
                did = true;
            }
            if (did) {
                idle0 = clock64();
            } else {
                __nanosleep(20);
                if (clock64() - idle0 > 4000000000ll) ptx::watchdog_trap("mma/idle", (int)cs[0], n_ended);
            }
        }
    } else {
        // ================================ epilogue ============================================
        // warp -> (lane quadrant q, tile half, slots k0 .. k0+SPW-1); slot i of a thread is a
        // pixel of member tile k0 + i
        const int q = warp & 3, half = (warp >> 2) & 1, k0 = (warp >> 3) * SPW;
        const int hs = warp / kWPS;  // this warp's chunk stream
        // M-tile holding slot k of this warp
        auto mtile = [&](int k) { return kCompact ? 4 * (warp >> 2) + k : 2 * (k0 + k) + half; };
        int relx[SPW], rely[SPW];
#pragma unroll
        for (int k = 0; k < SPW; ++k) {
            if (kCompact)
                lane_pixel_compact(mtile(k), q * 32 + lane, relx[k], rely[k]);
            else
                lane_pixel(mtile(k), q * 32 + lane, relx[k], rely[k]);
        }
        float T[SPW], cr[SPW], cg[SPW], cb[SPW], thr[SPW];
        int px[SPW], py[SPW];
        const float L = log2f(a.alpha_skip);
        const float tterm = a.t_terminate;
        int cur = -1;
        uint32_t alive = 0;     // warp-uniform: slots with a non-terminated pixel
        uint32_t reported = 0;  // dead slots already published for `cur`
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        // Accumulator registers.  A retired slot skips its tcgen05.ld and keeps stale finite
        // values, which never pass the D >= thr test because its thr is +inf.
        uint32_t d[SPW][kJB];
#pragma unroll
        for (int k = 0; k < SPW; ++k)
#pragma unroll
            for (int j = 0; j < kJB; ++j) d[k][j] = 0u;
        for (uint32_t c = 0;; ++c) {
            const int s = (int)(c % kSS), ts = (int)(c % kTS);
            // this warp consumed the phase of chunk c - kTS itself, so the parity is unambiguous
            [[maybe_unused]] const long long tw0 = clock64();
            ptx::mbar_wait_wd(&sm.tfull[hs][ts], (c / kTS) & 1, "epilogue/tfull", (int)c, warp);
            if (TGS_RASTER_PROF) pf[1] += clock64() - tw0;
            ptx::tc_fence_after();
            const ChunkHeader h = sm.hdr[hs][s];
            if (h.chunk != (int)c) {
                if (lane == 0)
                    printf("EPI w%d header mismatch: expected chunk %d found %d (seq %d)\n", warp, (int)c, h.chunk, h.seq);
                __trap();
            }
            if (h.seq != cur) {
                if (cur >= 0) {
#pragma unroll
                    for (int k = 0; k < SPW; ++k)
                        if (px[k] >= 0) {
                            float* o = a.image + ((size_t)(py[k] - a.image_row0) * gg.width + px[k]) * 3;
                            o[0] = fminf(fmaxf(cr[k], 0.0f), 1.0f);
                            o[1] = fminf(fmaxf(cg[k], 0.0f), 1.0f);
                            o[2] = fminf(fmaxf(cb[k], 0.0f), 1.0f);
                        }
                }
                if (h.seq < 0) break;
                cur = h.seq;
                reported = 0;
                const UnitGeom ug = unit_geom<SLOTS>(gg, h.unit);
#pragma unroll
                for (int k = 0; k < SPW; ++k) {
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
                for (int k = 0; k < SPW; ++k)
                    if (__any_sync(0xffffffffu, thr[k] != kInf)) alive |= 1u << k;
            }
            const int nv = h.n_valid;
            const uint32_t stage_col = (uint32_t)(ts * kColsPerStage);
            if (nv > 0 && alive != 0u) {
#pragma unroll 1
                for (int j0 = 0; j0 < nv; j0 += kJB) {
#pragma unroll
                    for (int k = 0; k < SPW; ++k)
                        if (alive & (1u << k)) {
                            const uint32_t ta = lane_base + stage_col + (uint32_t)(mtile(k) * kN + j0);
                            if constexpr (kJB == 16)
                                ptx::tmem_ld16(ta, d[k]);
                            else
                                ptx::tmem_ld8(ta, d[k]);
                        }
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < SPW; ++k) {
                        if constexpr (kJB == 16)
                            ptx::reg_fence16(d[k]);
                        else
                            ptx::reg_fence8(d[k]);
                    }
                    // Phase 1 (branch-free, kJB independent chains): which of the batch's splats
                    // reach alpha_skip at any of this warp's pixels -> warp-uniform mask.
                    uint32_t mk = 0;
#pragma unroll
                    for (int jj = 0; jj < kJB; ++jj) {
                        uint32_t p = 0;
#pragma unroll
                        for (int k = 0; k < SPW; ++k) p |= fset_ge(__uint_as_float(d[k][jj]), thr[k]);
                        mk |= p & (1u << jj);
                    }
                    const uint32_t M = __reduce_or_sync(0xffffffffu, mk);
                    if (TGS_RASTER_PROF) {
                        pf[2] += __popc(M);
                        pf[3] += kJB;
                    }
                    // Phase 2: ordered blend of the active splats (uniform branches).  A pixel blends
                    // splat j iff D >= log2(alpha_skip) and it had not terminated before j
                    // (T >= t_terminate): exactly alpha_of/blend/done (raster_scalar.hpp:40-55,
                    // raster_scalar.cpp:36-41) — the splat that drives T below t_terminate is
                    // blended, nothing after it.
                    auto blend = [&](int jj, const uint32_t* dk) {
                        const float4 ej = sm.epi[hs][s][j0 + jj];
#pragma unroll
                        for (int k = 0; k < SPW; ++k) {
                            const float dv = __uint_as_float(dk[k]);
                            const float e2 = fminf(ej.w, ex2_approx(dv));
                            const float al = (dv >= thr[k] && T[k] >= tterm) ? e2 : 0.0f;
                            const float wt = T[k] * al;
                            cr[k] = fmaf(wt, ej.x, cr[k]);
                            cg[k] = fmaf(wt, ej.y, cg[k]);
                            cb[k] = fmaf(wt, ej.z, cb[k]);
                            T[k] -= wt;
                        }
                    };
                    if constexpr (P2 == 0) {
#pragma unroll
                        for (int jj = 0; jj < kJB; ++jj)
                            if (M & (1u << jj)) {
                                uint32_t dk[SPW];
#pragma unroll
                                for (int k = 0; k < SPW; ++k) dk[k] = d[k][jj];
                                blend(jj, dk);
                            }
                    } else {
                        // loop over the active splats only, re-reading each one's D column from TMEM
                        // (tcgen05.ld 32x32b.x1 per slot, next splat prefetched while this one blends)
                        uint32_t Mr = M;
                        if (Mr) {
                            int jj = __ffs(Mr) - 1;
                            Mr &= Mr - 1u;
                            const uint32_t cbase = lane_base + stage_col + (uint32_t)j0;
                            uint32_t dc[SPW];
#pragma unroll
                            for (int k = 0; k < SPW; ++k) ptx::tmem_ld1(cbase + (uint32_t)(mtile(k) * kN + jj), dc[k]);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int k = 0; k < SPW; ++k) ptx::reg_fence1(dc[k]);
#pragma unroll 1
                            for (;;) {
                                const bool more = Mr != 0u;
                                int jn = jj;
                                uint32_t dn[SPW];
                                if (more) {
                                    jn = __ffs(Mr) - 1;
                                    Mr &= Mr - 1u;
#pragma unroll
                                    for (int k = 0; k < SPW; ++k)
                                        ptx::tmem_ld1(cbase + (uint32_t)(mtile(k) * kN + jn), dn[k]);
                                }
                                blend(jj, dc);
                                if (!more) break;
                                ptx::tmem_wait_ld();
#pragma unroll
                                for (int k = 0; k < SPW; ++k) {
                                    ptx::reg_fence1(dn[k]);
                                    dc[k] = dn[k];
                                }
                                jj = jn;
                            }
                        }
                    }
#pragma unroll
                    for (int k = 0; k < SPW; ++k)
                        if (T[k] < tterm) thr[k] = kInf;
                }
            }
            // retire slots whose pixels all terminated; report once per unit
            uint32_t dead = 0;
#pragma unroll
            for (int k = 0; k < SPW; ++k)
                if (!__any_sync(0xffffffffu, thr[k] != kInf)) dead |= 1u << k;
            alive &= ~dead;
            // TMEM stage and smem stage consumed (all tcgen05.ld of this warp completed above)
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                // published in member-tile bits (compact: the warp's half of tile warp >> 1)
                const uint32_t dtiles = kCompact ? (dead == (1u << SPW) - 1u ? 1u << (warp >> 1) : 0u) : dead << k0;
                if (dead != reported) ((volatile int*)sm.dead)[warp] = (cur << 4) | (int)dtiles;
__threadfence_block();
                ((volatile int*)sm.wdone)[warp] = (int)c + 1;
                atomicAdd(&sm.done_cnt[hs][s], 1u);
            }
            reported = dead;
        }
    }

#if TGS_RASTER_PROF
    if (lane == 0) {
        const int base = warp == kProd ? 0 : warp == kMma ? 4 : 8;
        atomicAdd(&g_rprof[base], (unsigned long long)(clock64() - pf_start));
        if (warp == kProd) atomicMax(&g_rprof[12], (unsigned long long)(clock64() - pf_start));
        for (int i = 1; i < 4; ++i) atomicAdd(&g_rprof[base + i], pf[i]);
        if (warp == kProd) atomicAdd(&g_rprof[3], (unsigned long long)0);
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
            g_rprof_done = 0;
            // the 12 most expensive units: cycles, chunks, list length, position in the start order
            for (int r = 0; r < 12; ++r) {
                unsigned int best = 0;
                int bu = -1;
                for (int u = 0; u < n_units && u < 65536; ++u)
                    if (g_ucyc[u] > best) { best = g_ucyc[u]; bu = u; }
                if (bu < 0) break;
                const int gid = SLOTS == 1 ? bu : bu / units_per_group<SLOTS>(gg.g);
                printf("RUNIT %d cycles %u chunks %u list %u started #%u | producer wait %u retire %u row %u place %u\n",
                       bu, best, g_uch[bu], a.offsets[gid + 1] - a.offsets[gid], g_uent[bu], g_uwait[bu],
                       g_usec[bu][0], g_usec[bu][1], g_usec[bu][2]);
                g_ucyc[bu] = 0;
            }
            const double n = (double)gridDim.x;
            printf("RPROF ctas %d | producer total %.0f wait %.0f batches %.0f | mma total %.0f wfull %.0f wtmem %.0f | "
                   "mma issue %.0f | epi/warp total %.0f wtfull %.0f | active blocks %.3f of %.0f | cta max %llu unit max %llu "
                   "chunks max %llu\n", gridDim.x, v[0] / n, v[1] / n,
                   v[2] / n, v[4] / n, v[5] / n, v[6] / n, v[7] / n, v[8] / n / kEpiWarps, v[9] / n / kEpiWarps,
                   (double)v[10] / (double)(v[11] ? v[11] : 1), v[11] / n / kEpiWarps, v[12], v[13], v[14]);
        }
    }
#endif
}

template <int SLOTS, int P2>
void launch_t(const RasterArgs& a, int num_sms, cudaStream_t st) {
    const size_t smem = sizeof(Smem<SLOTS>);
    cudaFuncSetAttribute(raster_tensor_kernel<SLOTS, P2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int n_units = SLOTS == 1 ? a.gg.n_groups_band : a.gg.n_groups_band * units_per_group<SLOTS>(a.gg.g);
    int grid = num_sms * ctas_per_sm<SLOTS>();
    if (grid > n_units) grid = n_units;
    if (grid > 0) raster_tensor_kernel<SLOTS, P2><<<grid, Roles<SLOTS>::kThreads, smem, st>>>(a);
}

}  // namespace

void launch_raster_tensor(const RasterArgs& a, int num_sms, cudaStream_t st) {
    static const int variant = [] {
        const char* e = getenv("TGS_RASTER_VARIANT");  // A/B aid for epilogue experiments
        return e ? atoi(e) : 0;
    }();
    if (a.gg.g == 1)
        variant == 4 ? launch_t<1, 4>(a, num_sms, st) : launch_t<1, 0>(a, num_sms, st);
    else if (a.gg.g == 2 && TGS_RASTER_HALF)
        launch_t<2, 0>(a, num_sms, st);
    else
        variant == 4 ? launch_t<4, 4>(a, num_sms, st) : launch_t<4, 0>(a, num_sms, st);
}

int raster_units_per_group(int g) { return g == 1 ? 1 : (g == 2 && TGS_RASTER_HALF) ? 2 : g == 4 ? 4 : 1; }

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
    const int t = threadIdx.x, warp = t >> 5;
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
}
}  // namespace

void launch_debug_mma(const uint16_t* a, const uint16_t* b, float* d, cudaStream_t st) {
    debug_mma_kernel<<<1, 128, 0, st>>>(a, b, d);
}
}  // namespace tgs
