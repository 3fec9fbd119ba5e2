// TOOLS ONLY (libtgs_debug.so, built by tools/debug/build.py; not part of libtgs.so or its ABI):
// microbenchmarks of the rasterizer's tcgen05 building blocks —
//   tgs_debug_pipeline: per-chunk latency of the producer -> MMA -> epilogue hand-off (no blending),
//   tgs_debug_mma_rate: tcgen05.mma issue rate / group latency in isolation,
//   tgs_debug_mma:      one M=128 x N=32 x K=16 MMA through the rasterizer's descriptors
//                       (tests/test_gpu_tcgen05.py checks it against float64).
#include "../../paper_2605_17855_b200/csrc/tgs_common.cuh"
#include "../../paper_2605_17855_b200/csrc/tgs_ptx.cuh"
#include "tgs_debug.h"

namespace tgs {
namespace {

constexpr int kDbgSS = 8, kDbgTS = 4, kDbgEpi = 4;

struct DbgSmem {
    alignas(128) uint8_t a[256 * 32];
    alignas(128) uint8_t b[kDbgSS][32 * 32];
    uint64_t full[kDbgSS], done[kDbgSS], tfull[kDbgTS], tempty[kDbgTS];
    uint32_t tmem_base;
};

// mode bit 0: issue the MMAs; bit 1: epilogue tcgen05.ld's the accumulators; bit 2: producer fences
__global__ void __launch_bounds__(192, 1) debug_pipeline_kernel(int chunks, int mode, long long* out) {
    __shared__ DbgSmem sm;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 256 * 32 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm.a)[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < kDbgSS * 32 * 32 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(&sm.b[0][0])[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kDbgSS; ++s) {
            ptx::mbar_init(&sm.full[s], 1);
            ptx::mbar_init(&sm.done[s], kDbgEpi);
        }
        for (int s = 0; s < kDbgTS; ++s) {
            ptx::mbar_init(&sm.tfull[s], 1);
            ptx::mbar_init(&sm.tempty[s], kDbgEpi);
        }
        ptx::mbar_fence_init();
    }
    if (warp == 5) ptx::tmem_alloc<256>(&sm.tmem_base);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const long long t0 = clock64();
    if (warp == 4) {
        for (int c = 0; c < chunks; ++c) {
            const int s = c % kDbgSS;
            if (c >= kDbgSS) ptx::mbar_wait(&sm.done[s], ((c / kDbgSS) - 1) & 1);
            if (mode & 4) ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&sm.full[s]);
        }
    } else if (warp == 5) {
        const uint32_t idesc = ptx::idesc_f16(128, 32);
        const uint32_t a_base = ptx::smem_u32(sm.a);
        for (int c = 0; c < chunks; ++c) {
            const int s = c % kDbgSS, ts = c % kDbgTS;
            ptx::mbar_wait(&sm.full[s], (c / kDbgSS) & 1);
            if (c >= kDbgTS) ptx::mbar_wait(&sm.tempty[ts], ((c / kDbgTS) - 1) & 1);
            ptx::tc_fence_after();
            if (lane == 0) {
                if (mode & 1) {
                    const uint64_t bd = ptx::smem_desc(ptx::smem_u32(&sm.b[s][0]), 128, 256);
                    ptx::mma_f16_ss(tmem + ts * 64, ptx::smem_desc(a_base, 128, 256), bd, idesc, 0u);
                    ptx::mma_f16_ss(tmem + ts * 64 + 32, ptx::smem_desc(a_base + 4096, 128, 256), bd, idesc, 0u);
                    ptx::mma_commit(&sm.tfull[ts]);
                } else {
                    ptx::mbar_arrive(&sm.tfull[ts]);
                }
            }
            __syncwarp();
        }
    } else {
        float acc = 0.0f;
        for (int c = 0; c < chunks; ++c) {
            const int s = c % kDbgSS, ts = c % kDbgTS;
            ptx::mbar_wait(&sm.tfull[ts], (c / kDbgTS) & 1);
            ptx::tc_fence_after();
            if (mode & 2) {
                uint32_t d[2][16];
                const uint32_t base = tmem + ((uint32_t)(warp * 32) << 16) + ts * 64;
                ptx::tmem_ld16(base, d[0]);
                ptx::tmem_ld16(base + 32, d[1]);
                ptx::tmem_wait_ld();
                ptx::reg_fence16(d[0]);
                ptx::reg_fence16(d[1]);
                acc += __uint_as_float(d[0][lane & 15]) + __uint_as_float(d[1][3]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(&sm.tempty[ts]);
                ptx::mbar_arrive(&sm.done[s]);
            }
        }
        if (acc == 12345.0f) out[3] = 1;
    }
    const long long t1 = clock64();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 5) ptx::tmem_dealloc<256>(tmem);
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

// MMA issue-rate probe: one thread issues n tcgen05.mma (M=128, N=ncols, K=16, A and B from
// smem) into rotating TMEM columns, committing to an mbarrier every `per_commit` MMAs and
// waiting for that commit before continuing when `wait_each` is set; reports total cycles.
__global__ void __launch_bounds__(128, 1) debug_mma_rate_kernel(int n, int per_commit, int wait_each, int ncols,
                                                                 long long* out) {
    const int variant = per_commit >> 16;  // 0 SS no-swizzle, 1 A in TMEM, 2 SS 32B-swizzle, 3 M=64
    per_commit &= 0xffff;
    __shared__ __align__(128) uint8_t sa[128 * 32];
    __shared__ __align__(128) uint8_t sb[64 * 32];
    __shared__ uint64_t bar, bar_end;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 128 * 32 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sa)[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < 64 * 32 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sb)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_init(&bar_end, 1);
        ptx::mbar_fence_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tbase);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = tbase;
    long long t0 = clock64(), t1 = t0;
    if (variant == 4) {  // warp-uniform issue: whole warp 0 runs the loop, one elected lane issues
        if (warp == 0) {
            const uint32_t idesc = ncols == 16 ? ptx::idesc_f16(128, 16) : ncols == 64 ? ptx::idesc_f16(128, 64)
                                                                               : ptx::idesc_f16(128, 32);
            const uint64_t ad = ptx::smem_desc(ptx::smem_u32(sa), 128, 256);
            const uint64_t bd = ptx::smem_desc(ptx::smem_u32(sb), 128, 256);
            uint32_t phase = 0;
            int pending = 0;
            for (int i = 0; i < n; ++i) {
                ptx::mma_f16_ss_elect(tm + 8u + (uint32_t)((i * ncols) & 255), ad, bd, idesc, 0u);
                if (++pending == per_commit) {
                    ptx::mma_commit_elect(&bar);
                    pending = 0;
                    if (wait_each) {
                        ptx::mbar_wait(&bar, phase);
                        phase ^= 1;
                    }
                }
            }
            ptx::mma_commit_elect(&bar_end);
            ptx::mbar_wait(&bar_end, 0);
            t1 = clock64();
        }
    } else if (threadIdx.x == 0) {
        const int mm = variant == 3 ? 64 : 128;
        const uint32_t idesc = ncols == 16 ? ptx::idesc_f16(mm, 16) : ncols == 64 ? ptx::idesc_f16(mm, 64)
                                                                           : ptx::idesc_f16(mm, 32);
        uint64_t ad = ptx::smem_desc(ptx::smem_u32(sa), 128, 256);
        uint64_t bd = ptx::smem_desc(ptx::smem_u32(sb), 128, 256);
        if (variant == 2) {  // SWIZZLE_32B (layout type 6): 8 rows x 32 B atoms, SBO 256 B
            ad = ptx::smem_desc(ptx::smem_u32(sa), 16, 256) | (6ull << 61);
            bd = ptx::smem_desc(ptx::smem_u32(sb), 16, 256) | (6ull << 61);
        }
        uint32_t phase = 0;
        int pending = 0;
        for (int i = 0; i < n; ++i) {
            const uint32_t dcol = tm + 8u + (uint32_t)((i * ncols) & 255);
            if (variant == 1)
                ptx::mma_f16_ts(dcol, tm, bd, idesc, 0u);  // A = TMEM columns 0..7
            else
                ptx::mma_f16_ss(dcol, ad, bd, idesc, 0u);
            if (++pending == per_commit) {
                ptx::mma_commit(&bar);
                pending = 0;
                if (wait_each) {
                    ptx::mbar_wait(&bar, phase);
                    phase ^= 1;
                }
            }
        }
        ptx::mma_commit(&bar_end);  // arrives when every MMA above has completed
        ptx::mbar_wait(&bar_end, 0);
        t1 = clock64();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 0) ptx::tmem_dealloc<512>(tm);
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

}  // namespace

cudaError_t debug_mma_rate(int n, int per_commit, int wait_each, int ncols, long long* cycles) {
    long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(long long));
    if (e != cudaSuccess) return e;
    debug_mma_rate_kernel<<<1, 128>>>(n, per_commit, wait_each, ncols, d);
    e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(cycles, d, sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e;
}

cudaError_t debug_pipeline(int chunks, int mode, long long* cycles) {
    long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, 4 * sizeof(long long));
    if (e != cudaSuccess) return e;
    debug_pipeline_kernel<<<1, 192>>>(chunks, mode, d);
    e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(cycles, d, sizeof(long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e;
}

}  // namespace tgs

extern "C" tgs_status tgs_debug_mma_rate(int n, int per_commit, int wait_each, int ncols, long long* cycles) {
    const cudaError_t e = tgs::debug_mma_rate(n, per_commit, wait_each, ncols, cycles);
    return e == cudaSuccess ? TGS_OK : TGS_ERR_CUDA;
}

extern "C" tgs_status tgs_debug_pipeline(int chunks, int mode, long long* cycles) {
    const cudaError_t e = tgs::debug_pipeline(chunks, mode, cycles);
    return e == cudaSuccess ? TGS_OK : TGS_ERR_CUDA;
}

// ---- self-test hook: one M=128 x N=32 x K=16 tcgen05.mma through the rasterizer's descriptors --
namespace tgs {
__device__ __forceinline__ uint32_t dbg_core_off(int row, int khalf) {
    return (uint32_t)((row >> 3) * 256 + khalf * 128 + (row & 7) * 16);
}
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
        *reinterpret_cast<uint4*>(sa + dbg_core_off(t, kh)) = v;
        if (t < 32) {
            uint4 w = *reinterpret_cast<const uint4*>(b + t * 16 + kh * 8);
            *reinterpret_cast<uint4*>(sb + dbg_core_off(t, kh)) = w;
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
}  // namespace tgs

extern "C" tgs_status tgs_debug_mma(const uint16_t* a_host_128x16, const uint16_t* b_host_32x16, float* d_host_128x32) {
    uint16_t *a = nullptr, *b = nullptr;
    float* d = nullptr;
    cudaError_t e = cudaMalloc(&a, 128 * 16 * 2);
    if (e == cudaSuccess) e = cudaMalloc(&b, 32 * 16 * 2);
    if (e == cudaSuccess) e = cudaMalloc(&d, 128 * 32 * 4);
    if (e == cudaSuccess) e = cudaMemcpy(a, a_host_128x16, 128 * 16 * 2, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(b, b_host_32x16, 32 * 16 * 2, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        tgs::debug_mma_kernel<<<1, 128>>>(a, b, d);
        e = cudaDeviceSynchronize();
    }
    if (e == cudaSuccess) e = cudaMemcpy(d_host_128x32, d, 128 * 32 * 4, cudaMemcpyDeviceToHost);
    cudaFree(a);
    cudaFree(b);
    cudaFree(d);
    return e == cudaSuccess ? TGS_OK : TGS_ERR_CUDA;
}
