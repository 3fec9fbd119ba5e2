// glibc 2.39 expf restated in double precision (see tgs_raster_exact.cu); shared by the exact
// rasteriser and the tools probe that checks it against the host libm (tools/debug).
#pragma once

namespace tgs {

static __constant__ unsigned long long kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

// glibc expf (sysdeps/ieee754/flt-32/e_expf.c) for x <= 0: k = round(x * 32 / ln2) by the
// 0x1.8p52 shift, r = x * 32 / ln2 - k, 2^(k/32) from the table, 2^(r/32) by a cubic.  Inputs
// below -103.97 (glibc's underflow threshold) return 0.
__device__ __forceinline__ float expf_glibc(float x) {
    if (x < -0x1.9fe368p6f) return 0.0f;
    const double kInvLn2N = 0x1.71547652b82fep+0 * 32.0, kShift = 0x1.8p+52;
    const double kC0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0, kC1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0,
                 kC2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    const double z = __dmul_rn(kInvLn2N, (double)x);
    double kd = __dadd_rn(z, kShift);
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = __dsub_rn(kd, kShift);
    const double r = __dsub_rn(z, kd);
    const unsigned long long t = kExp2fTab[ki % 32] + (ki << 47);
    const double s = __longlong_as_double((long long)t);
    const double zz = __dadd_rn(__dmul_rn(kC0, r), kC1);
    const double r2 = __dmul_rn(r, r);
    double y = __dadd_rn(__dmul_rn(kC2, r), 1.0);
    y = __dadd_rn(__dmul_rn(zz, r2), y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}

}  // namespace tgs
