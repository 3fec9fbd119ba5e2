// Hand-written stable LSD radix sort (north_star 2) for u32 keys + u32 values with a
// device-resident item count (no host round trip inside a frame).
//
// Reference semantics it realises: std::stable_sort on (group_id << 32) | f32_bits(depth) with
// ties in emission order (proj/src/binning.cpp:86-91).  The render path sorts once: the presort
// of projected splats by depth bits (values = splat index, so ties keep index order); binning then
// partitions the rank-ordered splats stably by group (tgs_binning.cu), which yields the reference's
// (group, depth, index) lists bit for bit (tests/test_gpu_parity.py checks full list equality).
//
// One-sweep passes (8-bit digits, tiles of 3072 items):
//   digits : one kernel reads the keys once and builds the histograms of every pass;
//   pass   : one kernel per digit.  Tiles are claimed in order from a counter; each tile ranks its
//            items stably (per-warp digit peers from 8 ballots against running digit counters, warps
//            ordered by a per-digit prefix), publishes its per-digit totals, resolves its global
//            per-digit offsets by decoupled look-back over earlier tiles (2 predecessors per
//            round trip), sorts the tile by digit in shared memory and writes every digit run as
//            one contiguous burst.
// (Reduce-then-scan over the same tiles measured slower: 0.27 vs 0.21 ms for the 3M presort.)
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

#include <algorithm>
#include <cstdio>

namespace tgs {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef TGS_SORT_STEPS
#define TGS_SORT_STEPS 12  // 77 registers: 3 resident blocks per SM
#endif
constexpr int kSteps = TGS_SORT_STEPS;            // 32-item steps per warp per tile
constexpr int kTileItems = kThreads * kSteps;     // 3072
constexpr int kRadix = 256;
#ifndef TGS_SWEEP_BLOCKS
#define TGS_SWEEP_BLOCKS 3
#endif
constexpr int kSweepBlocks = 148 * TGS_SWEEP_BLOCKS;  // persistent one-sweep blocks
constexpr unsigned kLookbackSleepNs = 20;  // look-back back-off when no predecessor has published
constexpr int kLookbackWin = 2;  // predecessors read per look-back round trip (1-32 measured: 2 best)


constexpr uint32_t kFlagAgg = 1u << 30;  // look-back status: tile aggregate published
constexpr uint32_t kFlagPre = 2u << 30;  // look-back status: inclusive prefix published
constexpr uint32_t kValMask = (1u << 30) - 1u;
// scratch layout (u32): [0, 1024) digit histograms of the 4 passes; [1024, 1032) tile counters;
// then the per-(tile, digit) look-back status words
constexpr int kHistOff = 0, kCtrOff = 4 * kRadix, kStatusOff = kCtrOff + 8;

// Lanes of the warp holding the same 8-bit digit (valid lanes only): 8 ballots, one per digit
// bit.  __match_any_sync is several times slower on sm_100 for this use.
__device__ __forceinline__ uint32_t match_digit(uint32_t d, bool valid) {
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

// Digit histograms of every pass in one read of the keys (shared-memory atomics; warp
// aggregation via match/ballots measured slower).
__global__ void __launch_bounds__(kThreads) digits_kernel(const uint32_t* __restrict__ keys,
                                                          const uint32_t* count_ptr, int passes, bool drop,
                                                          const uint32_t* key_min_inv,
                                                          uint32_t* __restrict__ scratch) {
    __shared__ uint32_t h[4][kRadix];
    for (int i = threadIdx.x; i < 4 * kRadix; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t n = *count_ptr;
    const uint32_t kb = key_min_inv ? ~*key_min_inv : 0u;
    const uint32_t stride = gridDim.x * kThreads;
    for (uint32_t base = blockIdx.x * kThreads; base < n; base += 4 * stride) {  // 4 loads in flight
        uint32_t k[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t i = base + u * stride + threadIdx.x;
            k[u] = i < n ? keys[i] : kCulledKey;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t i = base + u * stride + threadIdx.x;
            const bool valid = i < n && !(drop && k[u] == kCulledKey);
            if (valid)
                for (int p = 0; p < passes; ++p) atomicAdd(&h[p][((k[u] - kb) >> (8 * p)) & 0xffu], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += kThreads) {
        const uint32_t c = (&h[0][0])[i];
        if (c) atomicAdd(&scratch[kHistOff + i], c);
    }
}

__global__ void __launch_bounds__(kThreads) onesweep_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, const uint32_t* count_ptr, int pass, bool write_keys, bool drop,
    const uint32_t* key_min_inv, uint32_t* __restrict__ scratch, uint32_t* sel, uint32_t src_idx) {
    __shared__ uint32_t wcnt[kWarps][kRadix];   // per-warp digit counts -> per-warp offsets
    __shared__ uint32_t tot[kRadix];            // tile digit totals
    __shared__ uint32_t lstart[kRadix];         // tile-local start of each digit
    __shared__ uint32_t gbase[kRadix];          // global slot of each digit's first item
    __shared__ uint32_t skey[kTileItems], sval[kTileItems];
    __shared__ uint32_t s_tile, s_n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int shift = 8 * pass;
    uint32_t* status = scratch + kStatusOff;
    const uint32_t n = *count_ptr;
    const uint32_t kb = key_min_inv ? ~*key_min_inv : 0u;
    const uint32_t lt = (1u << lane) - 1u;
    // A pass whose digit is the same for every item (e.g. the top byte of depth keys that share
    // their float exponent's high bits) is the identity permutation: copy instead of ranking.
    if (!drop && vin && __syncthreads_or(scratch[kHistOff + pass * kRadix + threadIdx.x] == n)) {
        if (sel) {  // last pass of a caller that reads the result buffer index: nothing to move
            if (blockIdx.x == 0 && threadIdx.x == 0) *sel = src_idx;
            return;
        }
        const uint32_t tid = blockIdx.x * kThreads + threadIdx.x, nt = gridDim.x * kThreads, n4 = n / 4u;
        auto copy = [&](const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src);  // cudaMalloc'd: 16-byte aligned
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll 4
            for (uint32_t i = tid; i < n4; i += nt) d4[i] = __ldcs(s4 + i);
            for (uint32_t i = 4u * n4 + tid; i < n; i += nt) dst[i] = src[i];
        };
        if (write_keys) copy(kin, kout);
        copy(vin, vout);
        return;
    }
    if (sel && blockIdx.x == 0 && threadIdx.x == 0) *sel = src_idx ^ 1u;
    // persistent blocks claim tiles in order, so only ~gridDim tiles are in flight and look-back
    // walks stay short
    for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&scratch[kCtrOff + pass], 1u);
    for (int d = lane; d < kRadix; d += 32) wcnt[warp][d] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t t0 = tile * (uint32_t)kTileItems;
    if (t0 >= n) return;

    // 1. load + stable per-warp ranking (warp w owns items [w * 32 kSteps, (w + 1) * 32 kSteps) of the tile)
    uint32_t k[kSteps], v[kSteps], rk[kSteps];
#pragma unroll
    for (int s = 0; s < kSteps; ++s) {
        const uint32_t i = t0 + warp * (32 * kSteps) + s * 32 + lane;
        k[s] = i < n ? kin[i] : kCulledKey;
        v[s] = i < n ? (vin ? vin[i] : i) : 0u;  // null vin: values are the item indices
    }
    // rank within the warp: per step, lanes with equal digits (ballot match); the highest such lane
    // adds the group to the warp's running digit counter with one shared atomic (program order per
    // address keeps steps ordered) and the group reads the old value from it — no barriers, so the
    // 16 steps overlap
    uint32_t peers[kSteps], old[kSteps];
#pragma unroll
    for (int s = 0; s < kSteps; ++s) {
        const uint32_t i = t0 + warp * (32 * kSteps) + s * 32 + lane;
        const bool valid = i < n && !(drop && k[s] == kCulledKey);
        const uint32_t d = ((k[s] - kb) >> shift) & 0xffu;
        peers[s] = match_digit(d, valid);
        old[s] = 0;
        if (valid && (31 - __clz(peers[s])) == lane) old[s] = atomicAdd(&wcnt[warp][d], (uint32_t)__popc(peers[s]));
        if (!valid) peers[s] = 0;
    }
#pragma unroll
    for (int s = 0; s < kSteps; ++s) {
        const int leader = peers[s] ? 31 - __clz(peers[s]) : lane;
        const uint32_t before = __shfl_sync(0xffffffffu, old[s], leader);
        rk[s] = peers[s] ? before + __popc(peers[s] & lt) : 0xffffffffu;
    }
    __syncthreads();
    // 2. per digit: warp offsets inside the tile, tile total
    {
        const int d = threadIdx.x;  // kThreads == kRadix
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t c = wcnt[w][d];
            wcnt[w][d] = run;
            run += c;
        }
        tot[d] = run;
        // publish the aggregate early so later tiles can make progress
        __stcg(&status[(size_t)tile * kRadix + d], (tile == 0 ? kFlagPre : kFlagAgg) | run);
    }
    __syncthreads();
    // 3. tile-local digit starts (exclusive scan of tot over digits), global digit offsets of the
    // pass (exclusive scan of the histogram) and decoupled look-back over earlier tiles
    {
        const int d = threadIdx.x;
        uint32_t incl = tot[d];
        const uint32_t hd = scratch[kHistOff + pass * kRadix + d];
        uint32_t hincl = hd;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            const uint32_t u = __shfl_up_sync(0xffffffffu, hincl, o);
            if (lane >= o) {
                incl += t;
                hincl += u;
            }
        }
        __shared__ uint32_t wsum[kWarps], hsum[kWarps];
        if (lane == 31) {
            wsum[warp] = incl;
            hsum[warp] = hincl;
        }
        __syncthreads();
        uint32_t wo = 0, ho = 0;
        for (int w = 0; w < warp; ++w) {
            wo += wsum[w];
            ho += hsum[w];
        }
        lstart[d] = wo + incl - tot[d];
        // look-back: sum earlier tiles' digit-d counts until one with an inclusive prefix, reading
        // kWin predecessors per round trip (independent loads)
        uint32_t prefix = 0;
        if (tile > 0) {
            constexpr int kWin = kLookbackWin;
            int j = (int)tile - 1;
            const long long w0 = clock64();
            for (;;) {
                uint32_t st[kWin];
#pragma unroll
                for (int i = 0; i < kWin; ++i) {
                    st[i] = 2u << 30;  // before tile 0: inclusive prefix 0
                    if (j - i >= 0) st[i] = *reinterpret_cast<volatile uint32_t*>(&status[(size_t)(j - i) * kRadix + d]);
                }
                // consume the ready run from j downwards; stop at the first inclusive prefix
                int used = 0;
                bool done = false;
#pragma unroll
                for (int i = 0; i < kWin; ++i) {
                    if (done || used != i) continue;
                    if ((st[i] & ~kValMask) == 0u) continue;  // not published yet: retry from here
                    prefix += st[i] & kValMask;
                    ++used;
                    if (st[i] & kFlagPre) done = true;
                }
                if (done) break;
                j -= used;
                if (used == 0) {
                    __nanosleep(kLookbackSleepNs);
                    if (clock64() - w0 > 4000000000ll) {  // bounded wait: report, never hang
                        printf("radix look-back stuck: pass %d tile %u waits on %d\n", pass, tile, j);
                        __trap();
                    }
                }
            }
            __stcg(&status[(size_t)tile * kRadix + d], kFlagPre | (prefix + tot[d]));
        }
        gbase[d] = ho + hincl - hd + prefix;
    }
    __syncthreads();
    // 4. digit-sorted tile in shared memory, then contiguous runs to global memory
#pragma unroll
    for (int s = 0; s < kSteps; ++s) {
        if (rk[s] != 0xffffffffu) {
            const uint32_t d = ((k[s] - kb) >> shift) & 0xffu;
            const uint32_t p = lstart[d] + wcnt[warp][d] + rk[s];
            skey[p] = k[s];
            sval[p] = v[s];
        }
    }
    if (threadIdx.x == 0) s_n = lstart[kRadix - 1] + tot[kRadix - 1];
    __syncthreads();
    const uint32_t m = s_n;
    for (uint32_t j = threadIdx.x; j < m; j += kThreads) {
        const uint32_t key = skey[j];
        const uint32_t d = ((key - kb) >> shift) & 0xffu;
        const uint32_t pos = gbase[d] + (j - lstart[d]);
        if (write_keys) kout[pos] = key;
        vout[pos] = sval[j];
    }
    __syncthreads();
    }
}

}  // namespace

size_t sort_result_sel_offset() { return kCtrOff + 7; }  // tile counters use kCtrOff + pass (< 4)

size_t sort_scratch_elems(size_t max_items) {
    return (size_t)kStatusOff + ((max_items + kTileItems - 1) / kTileItems + 1) * kRadix;
}

int radix_sort(SortBuffers& b, const uint32_t* count_first, const uint32_t* count_rest, int nbits,
               bool drop_first, bool want_keys_last, size_t max_items, cudaStream_t st,
               const uint32_t* key_min_inv, bool index_vals) {
    const int passes = std::max(1, std::min(4, (nbits + 7) / 8));
    const int tiles = (int)std::max<size_t>(1, (max_items + kTileItems - 1) / kTileItems);
    cudaMemsetAsync(b.ghist, 0, sort_scratch_elems(max_items) * sizeof(uint32_t), st);
    digits_kernel<<<148 * 4, kThreads, 0, st>>>(b.keys[0], count_first, passes, drop_first, key_min_inv, b.ghist);
    int src = 0;
    for (int p = 0; p < passes; ++p) {
        const bool last = p == passes - 1;
        if (p > 0)  // look-back status of the previous pass
            cudaMemsetAsync(b.ghist + kStatusOff, 0, (size_t)tiles * kRadix * sizeof(uint32_t), st);
        onesweep_kernel<<<std::min(tiles, kSweepBlocks), kThreads, 0, st>>>(b.keys[src], p == 0 && index_vals ? nullptr : b.vals[src], b.keys[src ^ 1], b.vals[src ^ 1],
                                                   p == 0 ? count_first : count_rest, p, !last || want_keys_last,
                                                   p == 0 && drop_first, key_min_inv, b.ghist,
                                                   last ? b.result_sel : nullptr, (uint32_t)src);
        src ^= 1;
    }
    return src;
}

}  // namespace tgs
