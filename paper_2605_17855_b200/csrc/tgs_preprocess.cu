// Preprocess (north_star 1): frustum cull, 3D->2D covariance, conic, radius, SH colour, and the
// order-preserving compaction of project_scene — one kernel.
//
// Reference: proj/src/projection.cpp:25-142 (+ types.hpp:45-48 for Camera::position).  Every
// value that feeds tile binning (mean2d, depth, radius) must be bit-identical to the reference,
// so this file uses only correctly-rounded single-precision intrinsics (__fmul_rn etc., no FMA
// contraction) in the reference's operation order, with Eigen's fixed-size reduction order
// e0 + (e1 + e2) for every 3-term dot product (oracle/eigen_min/Eigen/Core documents it).
// Colour and conic follow the same discipline, so the whole ProjectedGaussian is bit-exact.
//
// Outputs land at the input index: project_scene's order-preserving compaction
// (projection.cpp:131-139) is realised by the depth presort, which drops culled splats, and by the
// readback path (tgs_read_projected), which compacts on demand.
#include "tgs_common.cuh"
#include "tgs_kernels.cuh"

namespace tgs {

namespace {

constexpr float kShC0 = 0.28209479177f;
constexpr float kShC1 = 0.4886025119029199f;
__device__ __constant__ float kShC2[5] = {1.0925484305920792f, -1.0925484305920792f,
                                          0.31539156525252005f, -1.0925484305920792f,
                                          0.5462742152960396f};
__device__ __constant__ float kShC3[7] = {-0.5900435899266435f, 2.890611442640554f,
                                          -0.4570457994644658f, 0.3731763325901154f,
                                          -0.4570457994644658f, 1.445305721320277f,
                                          -0.5900435899266435f};

struct Proj {
    float mx, my, a, b, c, depth, r, g, bl;
    int radius;
};

// projection.cpp:25-27  R * mean + t
__device__ __forceinline__ void camera_space(const DevCamera& cam, float x, float y, float z,
                                             float p[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        p[i] = fadd(sum3(fmul(cam.r[i][0], x), fmul(cam.r[i][1], y), fmul(cam.r[i][2], z)), cam.t[i]);
}

// projection.cpp:55-77 eval_sh_color, coefficient-wise as written, then cwiseMax(0).
__device__ __forceinline__ void sh_color(const DevScene& s, int i, float dcr, float dcg, float dcb,
                                         const float d[3], float out[3]) {
    out[0] = fadd(0.5f, fmul(kShC0, dcr));
    out[1] = fadd(0.5f, fmul(kShC0, dcg));
    out[2] = fadd(0.5f, fmul(kShC0, dcb));
    if (s.sh_rest) {
        float co[48];
#pragma unroll
        for (int p = 0; p < 12; ++p) {
            const float4 v = s.sh_rest[(size_t)p * s.n + i];
            co[4 * p + 0] = v.x;
            co[4 * p + 1] = v.y;
            co[4 * p + 2] = v.z;
            co[4 * p + 3] = v.w;
        }
        const float x = d[0], y = d[1], z = d[2];
        const float xx = fmul(x, x), yy = fmul(y, y), zz = fmul(z, z);
        const float xy = fmul(x, y), yz = fmul(y, z), xz = fmul(x, z);
        const float nc1 = -kShC1;
        const float s1a = fmul(nc1, y), s1b = fmul(kShC1, z), s1c = fmul(kShC1, x);
        const float s2a = fmul(kShC2[0], xy), s2b = fmul(kShC2[1], yz);
        const float s2c = fmul(kShC2[2], fsub(fsub(fmul(2.0f, zz), xx), yy));
        const float s2d = fmul(kShC2[3], xz), s2e = fmul(kShC2[4], fsub(xx, yy));
        const float s3a = fmul(fmul(kShC3[0], y), fsub(fmul(3.0f, xx), yy));
        const float s3b = fmul(fmul(kShC3[1], xy), z);
        const float s3c = fmul(fmul(kShC3[2], y), fsub(fsub(fmul(4.0f, zz), xx), yy));
        const float s3d = fmul(fmul(kShC3[3], z), fsub(fsub(fmul(2.0f, zz), fmul(3.0f, xx)), fmul(3.0f, yy)));
        const float s3e = fmul(fmul(kShC3[4], x), fsub(fsub(fmul(4.0f, zz), xx), yy));
        const float s3f = fmul(fmul(kShC3[5], z), fsub(xx, yy));
        const float s3g = fmul(fmul(kShC3[6], x), fsub(fsub(xx, yy), fmul(3.0f, zz)));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
#define CO(k) co[3 * (k) + c]
            const float t1 = fsub(fadd(fmul(s1a, CO(0)), fmul(s1b, CO(1))), fmul(s1c, CO(2)));
            out[c] = fadd(out[c], t1);
            const float t2 = fadd(fadd(fadd(fadd(fmul(s2a, CO(3)), fmul(s2b, CO(4))), fmul(s2c, CO(5))),
                                       fmul(s2d, CO(6))),
                                  fmul(s2e, CO(7)));
            out[c] = fadd(out[c], t2);
            const float t3 =
                fadd(fadd(fadd(fadd(fadd(fadd(fmul(s3a, CO(8)), fmul(s3b, CO(9))), fmul(s3c, CO(10))),
                                    fmul(s3d, CO(11))),
                               fmul(s3e, CO(12))),
                          fmul(s3f, CO(13))),
                     fmul(s3g, CO(14)));
            out[c] = fadd(out[c], t3);
#undef CO
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) out[c] = (out[c] < 0.0f) ? 0.0f : out[c];
}

// projection.cpp:79-114 project_gaussian (after frustum_cull passed).
// Returns 1 kept, 0 degenerate (det <= 1e-12 or NaN), -1 non-positive scale.
__device__ __forceinline__ int project_one(const DevScene& s, const DevCamera& cam, int i,
                                           const float p[3], const float4& po, const float4& q, const float4& sd,
                                           const float2& gb, Proj& o) {
    // compute_cov3d (projection.cpp:36-43): Eigen minCoeff, then R * diag(s), M * M^T
    const float m12 = (sd.z < sd.y) ? sd.z : sd.y;
    const float mn = (m12 < sd.x) ? m12 : sd.x;
    if (!(mn > 0.0f)) return -1;
    const float w = q.x, x = q.y, y = q.z, z = q.w;
    const float tx = fmul(2.0f, x), ty = fmul(2.0f, y), tz = fmul(2.0f, z);
    const float twx = fmul(tx, w), twy = fmul(ty, w), twz = fmul(tz, w);
    const float txx = fmul(tx, x), txy = fmul(ty, x), txz = fmul(tz, x);
    const float tyy = fmul(ty, y), tyz = fmul(tz, y), tzz = fmul(tz, z);
    float r[3][3];
    r[0][0] = fsub(1.0f, fadd(tyy, tzz));
    r[0][1] = fsub(txy, twz);
    r[0][2] = fadd(txz, twy);
    r[1][0] = fadd(txy, twz);
    r[1][1] = fsub(1.0f, fadd(txx, tzz));
    r[1][2] = fsub(tyz, twx);
    r[2][0] = fsub(txz, twy);
    r[2][1] = fadd(tyz, twx);
    r[2][2] = fsub(1.0f, fadd(txx, tyy));
    const float sc[3] = {sd.x, sd.y, sd.z};
    float m[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) m[a][b] = fmul(r[a][b], sc[b]);
    float sig[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) {
            sig[a][b] = sum3(fmul(m[a][0], m[b][0]), fmul(m[a][1], m[b][1]), fmul(m[a][2], m[b][2]));
            sig[b][a] = sig[a][b];
        }
    // Jacobian, t = J * W, cov2 = (t * Sigma) * t^T (projection.cpp:87-94)
    const float zz = p[2];
    const float z2 = fmul(zz, zz);
    const float jac[2][3] = {{fdiv(cam.fx, zz), 0.0f, fdiv(fmul(-cam.fx, p[0]), z2)},
                             {0.0f, fdiv(cam.fy, zz), fdiv(fmul(-cam.fy, p[1]), z2)}};
    float t[2][3], ts[2][3], cov[2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            t[a][b] = sum3(fmul(jac[a][0], cam.r[0][b]), fmul(jac[a][1], cam.r[1][b]),
                           fmul(jac[a][2], cam.r[2][b]));
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            ts[a][b] = sum3(fmul(t[a][0], sig[0][b]), fmul(t[a][1], sig[1][b]), fmul(t[a][2], sig[2][b]));
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
            cov[a][b] = sum3(fmul(ts[a][0], t[b][0]), fmul(ts[a][1], t[b][1]), fmul(ts[a][2], t[b][2]));
    cov[0][0] = fadd(cov[0][0], 0.3f);
    cov[1][1] = fadd(cov[1][1], 0.3f);
    const float det = fsub(fmul(cov[0][0], cov[1][1]), fmul(cov[0][1], cov[0][1]));
    if (!(det > 1e-12f)) return 0;
    o.a = fdiv(cov[1][1], det);
    o.b = fdiv(-cov[0][1], det);
    o.c = fdiv(cov[0][0], det);
    const float mid = fmul(0.5f, fadd(cov[0][0], cov[1][1]));
    const float disc = fsub(fmul(mid, mid), det);
    const float lmax = fadd(mid, fsqrt((0.0f < disc) ? disc : 0.0f));
    int rad = (int)ceilf(fmul(3.0f, fsqrt(lmax)));
    o.radius = rad < 1 ? 1 : rad;
    o.depth = zz;
    // colour: dir = (mean - position).normalized(), position = -(R^T t)
    float pos[3], d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        pos[k] = -sum3(fmul(cam.r[0][k], cam.t[0]), fmul(cam.r[1][k], cam.t[1]), fmul(cam.r[2][k], cam.t[2]));
    d[0] = fsub(po.x, pos[0]);
    d[1] = fsub(po.y, pos[1]);
    d[2] = fsub(po.z, pos[2]);
    const float n2 = sum3(fmul(d[0], d[0]), fmul(d[1], d[1]), fmul(d[2], d[2]));
    if (n2 > 0.0f) {
        const float sn = fsqrt(n2);
        d[0] = fdiv(d[0], sn);
        d[1] = fdiv(d[1], sn);
        d[2] = fdiv(d[2], sn);
    }
    float col[3];
    sh_color(s, i, sd.w, gb.x, gb.y, d, col);
    o.r = col[0];
    o.g = col[1];
    o.bl = col[2];
    return 1;
}

#ifndef TGS_PRE_BLOCK
#define TGS_PRE_BLOCK 128
#endif
constexpr int kPreBlock = TGS_PRE_BLOCK;
#ifndef TGS_PRE_PER
#define TGS_PRE_PER 2
#endif
constexpr int kPrePer = TGS_PRE_PER;

// Per-thread frame tallies (summed over the thread's Gaussians, then warp/block aggregated).
struct PreTally {
    uint32_t culled = 0, dropped = 0, kept = 0, kmin_inv = 0, kmax = 0;
    unsigned long long app = 0;
};

// Projection + outputs of Gaussian i (i < n) from its SH0 planes.
__device__ __forceinline__ void preprocess_one(const PreprocessArgs& a, int i, float4 po, float4 q, float4 sd,
                                               float2 gb, PreTally& t) {
    bool keep = false, culled = false, dropped = false;
    Proj pr;
    {
        float p[3];
        camera_space(a.cam, po.x, po.y, po.z, p);
        bool vis = p[2] > a.cam.near_ && p[2] < a.cam.far_;  // frustum_cull (projection.cpp:45-53)
        if (vis) {
            pr.mx = fadd(fmul(0.5f, (float)a.cam.width), fdiv(fmul(a.cam.fx, p[0]), p[2]));
            pr.my = fadd(fmul(0.5f, (float)a.cam.height), fdiv(fmul(a.cam.fy, p[1]), p[2]));
            const float hw = fmul(0.5f, (float)a.cam.width), hh = fmul(0.5f, (float)a.cam.height);
            vis = fabsf(fsub(pr.mx, hw)) <= fmul(1.3f, hw) && fabsf(fsub(pr.my, hh)) <= fmul(1.3f, hh);
        }
        if (!vis) {
            culled = true;
        } else {
            const int rc = project_one(a.scene, a.cam, i, p, po, q, sd, gb, pr);
            if (rc < 0) {
                atomicOr(&a.fc->err_validation, 1u);
                dropped = true;  // the reference throws; the host reports VALIDATION
            } else if (rc == 0) {
                dropped = true;
            } else {
                keep = true;
            }
        }
    }
    {
        if (keep) {
            a.out.mc[i] = make_float4(pr.mx, pr.my, pr.a, pr.b);
            a.out.co[i] = make_float4(pr.c, po.w, pr.depth, __int_as_float(pr.radius));
            const float ext = tight_extents(pr.a, pr.b, pr.c, po.w, a.alpha_skip);
            a.out.col[i] = make_float4(pr.r, pr.g, pr.bl, ext);
            a.depth_keys[i] = __float_as_uint(pr.depth);
            int tx0, ty0, tx1, ty1, gx0, gy0, gx1, gy1;
            const int ng = group_rect(pr.mx, pr.my, pr.radius, a.gg, tx0, ty0, tx1, ty1, gx0, gy0, gx1, gy1);
            // tile rectangle (binning.cpp:32-44) for the group counting sort; empty -> x0 > x1
            a.rect[i] = (tx1 >= tx0 && ty1 >= ty0)
                            ? make_uint2((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16))
                            : make_uint2(0xffffu, 0u);
            // tile appearances of the band's tile rows only (the band's N_total, like its entries)
            const int by0 = max(ty0, a.gg.band_gy0 * a.gg.g), by1 = min(ty1, a.gg.band_gy1 * a.gg.g - 1);
            if (tx1 >= tx0 && by1 >= by0) t.app += (unsigned long long)(tx1 - tx0 + 1) * (by1 - by0 + 1);
            // sort_entries depth validation (binning.cpp:78-83) for splats that emit entries
            if (ng > 0 && !(isfinite(pr.depth) && pr.depth >= 0.0f)) atomicOr(&a.fc->err_validation, 2u);
        } else {
            a.depth_keys[i] = kCulledKey;
            a.rect[i] = make_uint2(kCulledRect, kCulledRect);
        }
    }
    t.culled += culled;
    t.dropped += dropped;
    if (keep) {
        const uint32_t kv = __float_as_uint(pr.depth);
        t.kept += 1u;
        t.kmin_inv = max(t.kmin_inv, ~kv);
        t.kmax = max(t.kmax, kv);
    }
}

// kPrePer Gaussians per thread, block-strided (all their SH0 planes are loaded up front, so the
// second Gaussian's loads are in flight while the first is projected); outputs at the INPUT index
// (no compaction pass: the depth presort drops culled splats, whose key is 0xffffffff, and
// project_scene's compacted order is only materialised on readback).  Counters are
// block-aggregated.
__global__ void __launch_bounds__(kPreBlock) preprocess_kernel(PreprocessArgs a) {
    __shared__ unsigned long long s_cnt[4];
    __shared__ unsigned int s_key[2];
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0;
    if (threadIdx.x < 2) s_key[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.fc->n_input = (unsigned)a.scene.n;
    __syncthreads();
    const int i0 = blockIdx.x * kPreBlock * kPrePer + threadIdx.x;
    const int lane = threadIdx.x & 31;
    float4 po[kPrePer], q[kPrePer], sd[kPrePer];
    float2 gb[kPrePer];
#pragma unroll
    for (int u = 0; u < kPrePer; ++u) {
        const int i = i0 + u * kPreBlock;
        if (i < a.scene.n) {
            po[u] = a.scene.pos_op[i];
            q[u] = a.scene.quat[i];
            sd[u] = a.scene.scale_dcr[i];
            gb[u] = a.scene.dc_gb[i];
        }
    }
    PreTally t;
#pragma unroll
    for (int u = 0; u < kPrePer; ++u) {
        const int i = i0 + u * kPreBlock;
        if (i < a.scene.n) preprocess_one(a, i, po[u], q[u], sd[u], gb[u], t);
    }
    const unsigned long long nc = __reduce_add_sync(0xffffffffu, t.culled);
    const unsigned long long nd = __reduce_add_sync(0xffffffffu, t.dropped);
    const unsigned long long nk = __reduce_add_sync(0xffffffffu, t.kept);
    const uint32_t kmin_inv = __reduce_max_sync(0xffffffffu, t.kmin_inv);
    const uint32_t kmax = __reduce_max_sync(0xffffffffu, t.kmax);
    unsigned long long app = t.app;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) app += __shfl_xor_sync(0xffffffffu, app, o);
    if (lane == 0) {
        if (nc) atomicAdd(&s_cnt[0], nc);
        if (nd) atomicAdd(&s_cnt[1], nd);
        if (app) atomicAdd(&s_cnt[2], app);  // tile appearances (render.cpp:19-20)
        if (nk) {
            atomicAdd(&s_cnt[3], nk);
            atomicMax(&s_key[0], kmin_inv);
            atomicMax(&s_key[1], kmax);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_cnt[0]) atomicAdd(&a.fc->culled, s_cnt[0]);
        if (s_cnt[1]) atomicAdd(&a.fc->dropped, s_cnt[1]);
        if (s_cnt[2]) atomicAdd(&a.fc->appearances, s_cnt[2]);
        if (s_cnt[3]) {
            atomicAdd(&a.fc->visible, (unsigned)s_cnt[3]);
            atomicMax(&a.fc->key_min_inv, s_key[0]);
            atomicMax(&a.fc->key_max, s_key[1]);
        }
    }
}

}  // namespace

const void* preprocess_kernel_fn() { return reinterpret_cast<const void*>(&preprocess_kernel); }

void launch_preprocess(const PreprocessArgs& a, cudaStream_t st) {
    const int blocks = (a.scene.n + kPreBlock * kPrePer - 1) / (kPreBlock * kPrePer);
    if (blocks > 0) preprocess_kernel<<<blocks, kPreBlock, 0, st>>>(a);
}

}  // namespace tgs
