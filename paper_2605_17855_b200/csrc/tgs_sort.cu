// Hand-written stable LSD radix sort (north_star 2) for u32 keys + u32 values with a
// device-resident item count (no host round trip inside a frame / CUDA graph).
//
// Reference semantics it realises: std::stable_sort on (group_id << 32) | f32_bits(depth) with
// ties in emission order (proj/src/binning.cpp:86-91).  The path sorts twice:
//   1. presort of visible splats by depth bits (values = project_scene index) — 32-bit keys;
//   2. stable sort of the emitted (group id, index) entries by group id only.
// Emission happens in presorted order, so (2) yields (group, depth, index) order == the
// reference's list, bit for bit (tests/test_gpu_parity.py checks full list equality).
//
// Per pass (reduce-then-scan, fixed grid of kSortBlocks blocks, each owning a contiguous range):
//   hist    : per-block digit histogram (smem atomics); the first gid pass also accumulates the
//             per-group counts that become the list offsets;
//   scan    : one block scans the [digit][block] matrix;
//   scatter : stable block-local ranking — each warp ranks 32 items per step with
//             __match_any_sync against warp-private running digit counters, a block-wide
//             per-digit prefix across warps orders the warps, then every item is written to
//             its global slot.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

namespace tgs {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSteps = 8;                              // 32-item steps per warp per tile
constexpr int kTileItems = kThreads * kSteps;          // 2048

__device__ __forceinline__ void block_range(uint32_t count, uint32_t& begin, uint32_t& end) {
    const uint32_t per = ((count + kSortBlocks - 1) / kSortBlocks + kTileItems - 1) / kTileItems * kTileItems;
    begin = min(count, per * blockIdx.x);
    end = min(count, begin + per);
}

template <int BITS>
__global__ void __launch_bounds__(kThreads) hist_kernel(const uint32_t* __restrict__ keys,
                                                        const uint32_t* count_ptr, int shift,
                                                        uint32_t* __restrict__ ghist, bool drop) {
    constexpr int R = 1 << BITS;
    __shared__ uint32_t dh[R];
    for (int d = threadIdx.x; d < R; d += kThreads) dh[d] = 0;
    __syncthreads();
    uint32_t begin, end;
    block_range(*count_ptr, begin, end);
    for (uint32_t i = begin + threadIdx.x; i < end; i += kThreads) {
        const uint32_t k = keys[i];
        if (!(drop && k == kCulledKey)) atomicAdd(&dh[(k >> shift) & (R - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < R; d += kThreads) ghist[d * kSortBlocks + blockIdx.x] = dh[d];
}

template <int BITS>
__global__ void __launch_bounds__(kThreads) scatter_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, const uint32_t* count_ptr, int shift,
    const uint32_t* __restrict__ ghist, bool write_keys, bool drop) {
    constexpr int R = 1 << BITS;
    __shared__ uint32_t blk_off[R];
    __shared__ uint32_t wcnt[kWarps][R];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < R; d += kThreads) blk_off[d] = ghist[d * kSortBlocks + blockIdx.x];
    uint32_t begin, end;
    block_range(*count_ptr, begin, end);
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t tile = begin; tile < end; tile += kTileItems) {
        for (int d = lane; d < R; d += 32) wcnt[warp][d] = 0;
        __syncwarp();
        uint32_t k[kSteps], v[kSteps], rk[kSteps];
#pragma unroll
        for (int s = 0; s < kSteps; ++s) {
            const uint32_t i = tile + warp * (32 * kSteps) + s * 32 + lane;
            k[s] = i < end ? kin[i] : 0u;
            const bool valid = i < end && !(drop && k[s] == kCulledKey);  // pass 1 drops culled splats
            v[s] = valid ? vin[i] : 0u;
            const uint32_t d = (k[s] >> shift) & (R - 1);
            const uint32_t key = valid ? d : (uint32_t)(R + lane);  // invalid lanes match nobody
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            uint32_t before = 0;
            if (valid) before = wcnt[warp][d];
            __syncwarp();
            if (valid && (31 - __clz(peers)) == lane) wcnt[warp][d] = before + __popc(peers);
            rk[s] = before + __popc(peers & lt);
            if (!valid) rk[s] = 0xffffffffu;
            __syncwarp();
        }
        __syncthreads();
        for (int d = threadIdx.x; d < R; d += kThreads) {
            uint32_t run = blk_off[d];
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t c = wcnt[w][d];
                wcnt[w][d] = run;
                run += c;
            }
            blk_off[d] = run;
        }
        __syncthreads();
#pragma unroll
        for (int s = 0; s < kSteps; ++s) {
            if (rk[s] != 0xffffffffu) {
                const uint32_t d = (k[s] >> shift) & (R - 1);
                const uint32_t pos = wcnt[warp][d] + rk[s];
                if (write_keys) kout[pos] = k[s];
                vout[pos] = v[s];
            }
        }
        __syncthreads();
    }
}

template <int BITS>
void run_pass(SortBuffers& b, int src, const uint32_t* count, int shift, bool write_keys, bool drop,
              cudaStream_t st) {
    const int R = 1 << BITS;
    hist_kernel<BITS><<<kSortBlocks, kThreads, 0, st>>>(b.keys[src], count, shift, b.ghist, drop);
    launch_exclusive_scan(b.ghist, (size_t)R * kSortBlocks, b.scan_tmp, st);
    scatter_kernel<BITS><<<kSortBlocks, kThreads, 0, st>>>(b.keys[src], b.vals[src], b.keys[src ^ 1],
                                                           b.vals[src ^ 1], count, shift, b.ghist,
                                                           write_keys, drop);
}

typedef void (*PassFn)(SortBuffers&, int, const uint32_t*, int, bool, bool, cudaStream_t);
const PassFn kPass[9] = {nullptr,        run_pass<1>, run_pass<2>, run_pass<3>, run_pass<4>,
                         run_pass<5>,    run_pass<6>, run_pass<7>, run_pass<8>};

}  // namespace

int radix_sort(SortBuffers& b, const uint32_t* count_first, const uint32_t* count_rest, int nbits,
               bool drop_first, bool want_keys_last, cudaStream_t st) {
    if (nbits < 1) nbits = 1;
    const int passes = (nbits + 7) / 8;
    const int per = (nbits + passes - 1) / passes;
    int src = 0, shift = 0;
    for (int p = 0; p < passes; ++p) {
        const int bits = (p == passes - 1) ? nbits - shift : per;
        const bool last = p == passes - 1;
        kPass[bits](b, src, p == 0 ? count_first : count_rest, shift, !last || want_keys_last,
                    p == 0 && drop_first, st);
        src ^= 1;
        shift += bits;
    }
    return src;
}


}  // namespace tgs
