/* tools/debug/tgs_debug.h — TOOLS ONLY: microbenchmarks of the rasterizer's tcgen05 building
 * blocks (libtgs_debug.so, tools/debug/build.py).  Not part of libtgs.so or include/tgs.h. */
#ifndef TGS_DEBUG_H
#define TGS_DEBUG_H
#include <stdint.h>
#include "../../include/tgs.h"
#ifdef __cplusplus
extern "C" {
#endif
/* One M=128 x N=32 x K=16 FP16 MMA through the rasterizer's shared-memory / instruction
 * descriptors (row-major A[128][16], B[32][16] binary16; D[128][32] = A . B^T in FP32). */
tgs_status tgs_debug_mma(const uint16_t* a_128x16, const uint16_t* b_32x16, float* d_128x32);
/* Device cycles of `chunks` producer -> MMA -> epilogue hand-offs with no blending; mode bits:
 * 1 issue MMAs, 2 tcgen05.ld the accumulators, 4 producer proxy fence. */
tgs_status tgs_debug_pipeline(int chunks, int mode, long long* cycles);
/* n MMAs (M=128, N=ncols in {16,32,64}, K=16), a commit every per_commit, optionally waited. */
tgs_status tgs_debug_mma_rate(int n, int per_commit, int wait_each, int ncols, long long* cycles);
#ifdef __cplusplus
}
#endif
#endif
