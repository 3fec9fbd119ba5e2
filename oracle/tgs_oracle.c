/* oracle/tgs_oracle.c — TEST INFRASTRUCTURE ONLY (see tgs_oracle.h).
 *
 * Plain-C restatement of the reference forward render path.  Every arithmetic expression keeps
 * the reference's operation order (and, where the reference goes through Eigen, the Eigen 3.x
 * fixed-size evaluation order documented in oracle/eigen_min/Eigen/Core), and the file is built
 * with -ffp-contract=off like the reference (CMakeLists.txt:10-12), so on the same host it is
 * bit-identical to oracle/_ref/libgsr_ref.so (checked by tests/test_oracle.py).
 */
#define _DEFAULT_SOURCE
#include "tgs_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* half.hpp:37-84 — binary16 RNE conversion and exact widening                                */
/* ------------------------------------------------------------------------------------------ */
static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

uint16_t tor_f32_to_f16(float x) {
    const uint32_t u = f2u(x);
    const uint32_t sign = (u >> 16) & 0x8000u;
    const uint32_t mag = u & 0x7FFFFFFFu;
    if (mag > 0x7F800000u) return 0x7E00u;
    if (mag >= 0x477FF000u) return (uint16_t)(sign | 0x7C00u);
    if (mag >= 0x38800000u) {
        uint32_t half = sign | (((mag >> 23) - 112u) << 10) | ((mag & 0x7FFFFFu) >> 13);
        const uint32_t rem = mag & 0x1FFFu;
        if (rem > 0x1000u || (rem == 0x1000u && (half & 1u))) ++half;
        return (uint16_t)half;
    }
    if (mag < 0x33000000u) return (uint16_t)sign;
    {
        const uint32_t mant = (mag & 0x7FFFFFu) | 0x800000u;
        const int shift = 126 - (int)(mag >> 23);
        uint32_t q = mant >> shift;
        const uint32_t rem = mant & ((1u << shift) - 1u);
        const uint32_t halfway = 1u << (shift - 1);
        if (rem > halfway || (rem == halfway && (q & 1u))) ++q;
        return (uint16_t)(sign | q);
    }
}

float tor_f16_to_f32(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t exp5 = (h >> 10) & 0x1Fu;
    const uint32_t man = h & 0x3FFu;
    if (exp5 == 0u) {
        if (man == 0u) return u2f(sign);
        {
            const int top = 31 - __builtin_clz(man);
            const uint32_t exp32 = (uint32_t)(103 + top);
            const uint32_t man32 = (man << (23 - top)) & 0x7FFFFFu;
            return u2f(sign | (exp32 << 23) | man32);
        }
    }
    if (exp5 == 31u) return u2f(sign | 0x7F800000u | (man << 13));
    return u2f(sign | ((exp5 + 112u) << 23) | (man << 13));
}

/* lane_quantize<Half> then lane_widen: the value an fp16 lane holds (half.hpp:88-96). */
static float q16(float x) { return tor_f16_to_f32(tor_f32_to_f16(x)); }

/* ------------------------------------------------------------------------------------------ */
/* scene_io.hpp:14-31 SplitMix64, scene_io.cpp:218-251 gen_synthetic_scene                    */
/* ------------------------------------------------------------------------------------------ */
typedef struct { uint64_t state; } smx;
static uint64_t smx_next(smx* r) {
    uint64_t z = (r->state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static float smx_uniform(smx* r) { return (float)(smx_next(r) >> 40) * 0x1.0p-24f; }
static float smx_uniform_in(smx* r, float lo, float hi) { return lo + (hi - lo) * smx_uniform(r); }

/* Eigen Vector4f::squaredNorm on SSE (predux<Packet4f>): (x^2 + z^2) + (y^2 + w^2). */
static float quat_norm(const float q[4] /* x,y,z,w */) {
    const float a = q[0] * q[0], b = q[1] * q[1], c = q[2] * q[2], d = q[3] * q[3];
    return sqrtf((a + c) + (b + d));
}

int tor_gen_scene(uint64_t seed, int count, float extent, float smin, float smax,
                  uint64_t sh_seed, float* out) {
    if (count < 0 || !(extent > 0.0f) || !(smin > 0.0f) || !(smin <= smax)) return -1;
    smx rng = {seed};
    smx rng_sh = {sh_seed};
    const int rf = sh_seed ? 59 : 14;
    for (int i = 0; i < count; ++i) {
        float* p = out + (size_t)i * rf;
        p[0] = smx_uniform_in(&rng, -extent, extent);
        p[1] = smx_uniform_in(&rng, -extent, extent);
        p[2] = smx_uniform_in(&rng, -extent, extent) + 3.0f * extent;
        p[3] = smx_uniform_in(&rng, smin, smax);
        p[4] = smx_uniform_in(&rng, smin, smax);
        p[5] = smx_uniform_in(&rng, smin, smax);
        {
            const float u1 = smx_uniform(&rng), u2 = smx_uniform(&rng), u3 = smx_uniform(&rng);
            const float s1 = sqrtf(1.0f - u1), s2 = sqrtf(u1);
            const float a = 2.0f * (float)M_PI * u2;
            const float b = 2.0f * (float)M_PI * u3;
            /* Quaternionf(w, x, y, z) = (s2 cos b, s1 sin a, s1 cos a, s2 sin b); coeffs x,y,z,w */
            float q[4] = {s1 * sinf(a), s1 * cosf(a), s2 * sinf(b), s2 * cosf(b)};
            /* renormalize_quat (scene_io.cpp:35-43) */
            const float n = quat_norm(q);
            if (!(n > 0.0f) || !isfinite(n)) return -1;
            if (fabsf(n - 1.0f) > 1e-6f)
                for (int k = 0; k < 4; ++k) q[k] = q[k] / n;
            p[6] = q[3]; p[7] = q[0]; p[8] = q[1]; p[9] = q[2];
        }
        p[10] = smx_uniform_in(&rng, 0.2f, 0.95f);
        for (int c = 0; c < 3; ++c) p[11 + c] = (smx_uniform(&rng) - 0.5f) / 0.28209479177f;
        if (sh_seed)
            for (int k = 0; k < 45; ++k) p[14 + k] = smx_uniform_in(&rng_sh, -1.0f, 1.0f);
    }
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* projection.cpp — Eigen fixed-size order: 3-term products e0 + (e1 + e2)                     */
/* ------------------------------------------------------------------------------------------ */
static float sum3(float e0, float e1, float e2) { return e0 + (e1 + e2); }

#define R_(cam, i, j) ((cam)->view[(i) * 4 + (j)])
#define T_(cam, i) ((cam)->view[(i) * 4 + 3])

/* projection.cpp:25-27 camera_space = R * mean + t */
static void camera_space(const float* m, const tor_camera* cam, float p[3]) {
    for (int i = 0; i < 3; ++i)
        p[i] = sum3(R_(cam, i, 0) * m[0], R_(cam, i, 1) * m[1], R_(cam, i, 2) * m[2]) + T_(cam, i);
}

/* projection.cpp:29-32 to_pixels */
static void to_pixels(const float p[3], const tor_camera* cam, float px[2]) {
    px[0] = 0.5f * (float)cam->width + cam->focal_x * p[0] / p[2];
    px[1] = 0.5f * (float)cam->height + cam->focal_y * p[1] / p[2];
}

/* projection.cpp:45-53 frustum_cull */
static int frustum_cull(const float* m, const tor_camera* cam) {
    float p[3], px[2];
    camera_space(m, cam, p);
    if (!(p[2] > cam->near_ && p[2] < cam->far_)) return 0;
    to_pixels(p, cam, px);
    {
        const float half_w = 0.5f * (float)cam->width;
        const float half_h = 0.5f * (float)cam->height;
        return fabsf(px[0] - half_w) <= 1.3f * half_w && fabsf(px[1] - half_h) <= 1.3f * half_h;
    }
}

/* projection.cpp:36-43 compute_cov3d; quat q = (w, x, y, z). Returns -1 on non-positive scale. */
static int compute_cov3d(const float s[3], const float q[4], float c6[6]) {
    /* Eigen minCoeff (novec redux): mini(e0, mini(e1, e2)), mini(a,b) = (b < a) ? b : a */
    const float m12 = (s[2] < s[1]) ? s[2] : s[1];
    const float mn = (m12 < s[0]) ? m12 : s[0];
    if (!(mn > 0.0f)) return -1;
    {
        const float w = q[0], x = q[1], y = q[2], z = q[3];
        /* Eigen Quaternion::toRotationMatrix */
        const float tx = 2.0f * x, ty = 2.0f * y, tz = 2.0f * z;
        const float twx = tx * w, twy = ty * w, twz = tz * w;
        const float txx = tx * x, txy = ty * x, txz = tz * x;
        const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
        float r[3][3], mm[3][3];
        r[0][0] = 1.0f - (tyy + tzz);
        r[0][1] = txy - twz;
        r[0][2] = txz + twy;
        r[1][0] = txy + twz;
        r[1][1] = 1.0f - (txx + tzz);
        r[1][2] = tyz - twx;
        r[2][0] = txz - twy;
        r[2][1] = tyz + twx;
        r[2][2] = 1.0f - (txx + tyy);
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) mm[i][j] = r[i][j] * s[j];
#define SIG(i, j) sum3(mm[i][0] * mm[j][0], mm[i][1] * mm[j][1], mm[i][2] * mm[j][2])
        c6[0] = SIG(0, 0);
        c6[1] = SIG(0, 1);
        c6[2] = SIG(0, 2);
        c6[3] = SIG(1, 1);
        c6[4] = SIG(1, 2);
        c6[5] = SIG(2, 2);
#undef SIG
    }
    return 0;
}

static const float kShC0 = 0.28209479177f;
static const float kShC1 = 0.4886025119029199f;
static const float kShC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                               -1.0925484305920792f, 0.5462742152960396f};
static const float kShC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                               0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                               -0.5900435899266435f};

/* projection.cpp:55-77 eval_sh_color (coefficient-wise, as written, then cwiseMax(0)) */
static void eval_sh_color(const float* dc, const float* rest, const float d[3], float out[3]) {
    for (int c = 0; c < 3; ++c) out[c] = 0.5f + kShC0 * dc[c];
    if (rest) {
        const float x = d[0], y = d[1], z = d[2];
        const float xx = x * x, yy = y * y, zz = z * z;
        const float xy = x * y, yz = y * z, xz = x * z;
#define CO(i) (rest + 3 * (i))
        for (int c = 0; c < 3; ++c) {
            const float t1 = -kShC1 * y * CO(0)[c] + kShC1 * z * CO(1)[c] - kShC1 * x * CO(2)[c];
            out[c] = out[c] + t1;
        }
        for (int c = 0; c < 3; ++c) {
            const float t2 = kShC2[0] * xy * CO(3)[c] + kShC2[1] * yz * CO(4)[c] +
                             kShC2[2] * (2.0f * zz - xx - yy) * CO(5)[c] + kShC2[3] * xz * CO(6)[c] +
                             kShC2[4] * (xx - yy) * CO(7)[c];
            out[c] = out[c] + t2;
        }
        for (int c = 0; c < 3; ++c) {
            const float t3 = kShC3[0] * y * (3.0f * xx - yy) * CO(8)[c] + kShC3[1] * xy * z * CO(9)[c] +
                             kShC3[2] * y * (4.0f * zz - xx - yy) * CO(10)[c] +
                             kShC3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy) * CO(11)[c] +
                             kShC3[4] * x * (4.0f * zz - xx - yy) * CO(12)[c] +
                             kShC3[5] * z * (xx - yy) * CO(13)[c] +
                             kShC3[6] * x * (xx - yy - 3.0f * zz) * CO(14)[c];
            out[c] = out[c] + t3;
        }
#undef CO
    }
    for (int c = 0; c < 3; ++c) out[c] = (out[c] < 0.0f) ? 0.0f : out[c];
}

/* projection.cpp:79-114 project_gaussian. Returns 1 kept, 0 degenerate, -1 validation error. */
static int project_gaussian(const float* g, int deg, const tor_camera* cam, tor_projected* o) {
    float p[3], c6[6];
    camera_space(g, cam, p);
    {
        const float z = p[2];
        if (compute_cov3d(g + 3, g + 6, c6) != 0) return -1;
        const float sig[3][3] = {{c6[0], c6[1], c6[2]}, {c6[1], c6[3], c6[4]}, {c6[2], c6[4], c6[5]}};
        const float jac[2][3] = {{cam->focal_x / z, 0.0f, -cam->focal_x * p[0] / (z * z)},
                                 {0.0f, cam->focal_y / z, -cam->focal_y * p[1] / (z * z)}};
        float t[2][3], ts[2][3], cov[2][2];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 3; ++j)
                t[i][j] = sum3(jac[i][0] * R_(cam, 0, j), jac[i][1] * R_(cam, 1, j),
                               jac[i][2] * R_(cam, 2, j));
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 3; ++j)
                ts[i][j] = sum3(t[i][0] * sig[0][j], t[i][1] * sig[1][j], t[i][2] * sig[2][j]);
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                cov[i][j] = sum3(ts[i][0] * t[j][0], ts[i][1] * t[j][1], ts[i][2] * t[j][2]);
        cov[0][0] += 0.3f;
        cov[1][1] += 0.3f;
        {
            const float det = cov[0][0] * cov[1][1] - cov[0][1] * cov[0][1];
            if (!(det > 1e-12f)) return 0;
            o->conic[0] = cov[1][1] / det;
            o->conic[1] = -cov[0][1] / det;
            o->conic[2] = cov[0][0] / det;
            {
                const float mid = 0.5f * (cov[0][0] + cov[1][1]);
                const float disc = mid * mid - det;
                const float lambda_max = mid + sqrtf((0.0f < disc) ? disc : 0.0f);
                int radius = (int)ceilf(3.0f * sqrtf(lambda_max));
                if (radius < 1) radius = 1;
                o->radius = radius;
            }
        }
        to_pixels(p, cam, o->mean2d);
        o->depth = z;
        o->opacity = g[10];
        {
            /* position = -(R^T t) (types.hpp:48); dir = (mean - position).normalized() */
            float pos[3], d[3];
            for (int i = 0; i < 3; ++i)
                pos[i] = -sum3(R_(cam, 0, i) * T_(cam, 0), R_(cam, 1, i) * T_(cam, 1),
                               R_(cam, 2, i) * T_(cam, 2));
            for (int i = 0; i < 3; ++i) d[i] = g[i] - pos[i];
            {
                const float n2 = sum3(d[0] * d[0], d[1] * d[1], d[2] * d[2]);
                if (n2 > 0.0f) {
                    const float s = sqrtf(n2);
                    for (int i = 0; i < 3; ++i) d[i] = d[i] / s;
                }
            }
            eval_sh_color(g + 11, deg == 3 ? g + 14 : NULL, d, o->color);
        }
    }
    return 1;
}

int64_t tor_project(const float* rec, int64_t n, int deg, const tor_camera* cam,
                    tor_projected* out, uint64_t* stats3) {
    const int rf = deg == 3 ? 59 : 14;
    int64_t k = 0;
    uint64_t culled = 0, dropped = 0;
    for (int64_t i = 0; i < n; ++i) {
        const float* g = rec + i * rf;
        if (!frustum_cull(g, cam)) { ++culled; continue; }
        {
            const int r = project_gaussian(g, deg, cam, &out[k]);
            if (r < 0) return -1;
            if (r == 0) { ++dropped; continue; }
            ++k;
        }
    }
    if (stats3) { stats3[0] = (uint64_t)n; stats3[1] = culled; stats3[2] = dropped; }
    return k;
}

/* ------------------------------------------------------------------------------------------ */
/* binning.cpp:12-100                                                                          */
/* ------------------------------------------------------------------------------------------ */
typedef struct { int g, w, h, tiles_x, tiles_y, groups_x, groups_y; } gcfg;

static int gcfg_make(int g, int w, int h, gcfg* c) {
    if (w <= 0 || h <= 0) return -1;
    if (!(g == 1 || g == 2 || g == 4)) return -1;
    c->g = g; c->w = w; c->h = h;
    c->tiles_x = (w + 15) / 16;
    c->tiles_y = (h + 15) / 16;
    c->groups_x = (c->tiles_x + g - 1) / g;
    c->groups_y = (c->tiles_y + g - 1) / g;
    return 0;
}

/* binning.cpp:32-44 tiles_overlapped */
static void tile_rect(const tor_projected* p, const gcfg* c, int r[4]) {
    const float rad = (float)p->radius;
    int x0 = (int)floorf((p->mean2d[0] - rad) / 16);
    int x1 = (int)floorf((p->mean2d[0] + rad) / 16);
    int y0 = (int)floorf((p->mean2d[1] - rad) / 16);
    int y1 = (int)floorf((p->mean2d[1] + rad) / 16);
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (x1 > c->tiles_x - 1) x1 = c->tiles_x - 1;
    if (y1 > c->tiles_y - 1) y1 = c->tiles_y - 1;
    r[0] = x0; r[1] = y0; r[2] = x1; r[3] = y1;
}

typedef struct { uint32_t gid; uint32_t idx; float depth; uint32_t mask; uint64_t order; } kentry;

static int kentry_cmp(const void* a, const void* b) {
    const kentry* x = (const kentry*)a;
    const kentry* y = (const kentry*)b;
    const uint64_t kx = ((uint64_t)x->gid << 32) | f2u(x->depth);
    const uint64_t ky = ((uint64_t)y->gid << 32) | f2u(y->depth);
    if (kx != ky) return kx < ky ? -1 : 1;
    return x->order < y->order ? -1 : (x->order > y->order ? 1 : 0);  /* std::stable_sort */
}

/* binning.cpp:46-74 build_group_entries (emission order: Gaussian, then gy, then gx). */
static int64_t build_entries(const tor_projected* p, int64_t n, const gcfg* c, kentry* out,
                             int64_t cap) {
    int64_t k = 0;
    for (int64_t i = 0; i < n; ++i) {
        int r[4];
        tile_rect(&p[i], c, r);
        if (r[2] < r[0] || r[3] < r[1]) continue;
        {
            const int gx0 = r[0] / c->g, gx1 = r[2] / c->g, gy0 = r[1] / c->g, gy1 = r[3] / c->g;
            for (int gy = gy0; gy <= gy1; ++gy)
                for (int gx = gx0; gx <= gx1; ++gx) {
                    if (out && k < cap) {
                        uint32_t mask = 0;
                        const int ty0 = r[1] > gy * c->g ? r[1] : gy * c->g;
                        const int ty1 = r[3] < gy * c->g + c->g - 1 ? r[3] : gy * c->g + c->g - 1;
                        const int tx0 = r[0] > gx * c->g ? r[0] : gx * c->g;
                        const int tx1 = r[2] < gx * c->g + c->g - 1 ? r[2] : gx * c->g + c->g - 1;
                        for (int ty = ty0; ty <= ty1; ++ty)
                            for (int tx = tx0; tx <= tx1; ++tx)
                                mask |= 1u << ((ty - gy * c->g) * c->g + (tx - gx * c->g));
                        out[k].gid = (uint32_t)(gy * c->groups_x + gx);
                        out[k].idx = (uint32_t)i;
                        out[k].depth = p[i].depth;
                        out[k].mask = mask;
                        out[k].order = (uint64_t)k;
                    }
                    ++k;
                }
        }
    }
    return k;
}

int64_t tor_bin_sort(const tor_projected* p, int64_t n, int width, int height, int g,
                     tor_entry* out, int64_t cap, uint32_t* offsets, uint64_t* appearances) {
    gcfg c;
    if (gcfg_make(g, width, height, &c) != 0) return -1;
    {
        const int64_t total = build_entries(p, n, &c, NULL, 0);
        if (total > cap && !appearances) return total;
        {
            kentry* e = (kentry*)malloc((size_t)(total ? total : 1) * sizeof(kentry));
            if (!e) return -2;
            build_entries(p, n, &c, e, total);
            if (appearances) {
                uint64_t a = 0;
                for (int64_t i = 0; i < total; ++i) a += (uint64_t)__builtin_popcount(e[i].mask);
                *appearances = a;
            }
            if (total > cap) { free(e); return total; }
            /* sort_entries: reject non-finite / negative depths (binning.cpp:78-83) */
            for (int64_t i = 0; i < total; ++i)
                if (!isfinite(e[i].depth) || e[i].depth < 0.0f) { free(e); return -1; }
            qsort(e, (size_t)total, sizeof(kentry), kentry_cmp);
            {
                const int ng = c.groups_x * c.groups_y;
                for (int i = 0; i <= ng; ++i) offsets[i] = 0;
                for (int64_t i = 0; i < total; ++i) ++offsets[e[i].gid + 1];
                for (int i = 1; i <= ng; ++i) offsets[i] += offsets[i - 1];
                for (int64_t i = 0; i < total; ++i) {
                    out[i].gaussian_index = e[i].idx;
                    out[i].depth = e[i].depth;
                    out[i].mask = e[i].mask;
                }
            }
            free(e);
            return total;
        }
    }
}

/* Same lists as tor_bin_sort, in O(entries) instead of a comparison sort of every entry, so the
 * oracle can check full-size frames (C3 G=1: 195M entries).  build_group_entries emits a
 * Gaussian's entries in index order and at most one per group; std::stable_sort on
 * (gid << 32 | depth bits) (binning.cpp:86-91) therefore leaves group g's list = the Gaussians
 * overlapping g ordered by (depth bits, index).  So: order the Gaussians by (depth bits, index)
 * once, then distribute them into the groups they overlap (a stable counting sort by gid).
 * Pinned against tor_bin_sort by tests/test_oracle.py. */
typedef struct { uint32_t key; uint32_t idx; } dpair;

static int dpair_cmp(const void* a, const void* b) {
    const dpair* x = (const dpair*)a;
    const dpair* y = (const dpair*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

int64_t tor_bin_sort_fast(const tor_projected* p, int64_t n, int width, int height, int g,
                          tor_entry* out, int64_t cap, uint32_t* offsets, uint64_t* appearances) {
    gcfg c;
    int64_t total = 0, i;
    uint64_t app = 0;
    dpair* ord;
    uint64_t* cur;
    int ng;
    if (gcfg_make(g, width, height, &c) != 0) return -1;
    ng = c.groups_x * c.groups_y;
    for (i = 0; i < n; ++i) {
        int r[4];
        tile_rect(&p[i], &c, r);
        if (r[2] < r[0] || r[3] < r[1]) continue;
        total += (int64_t)(r[2] / g - r[0] / g + 1) * (r[3] / g - r[1] / g + 1);
        app += (uint64_t)(r[2] - r[0] + 1) * (uint64_t)(r[3] - r[1] + 1);
    }
    if (appearances) *appearances = app;
    if (!out || total > cap) return total;
    ord = (dpair*)malloc((size_t)(n ? n : 1) * sizeof(dpair));
    cur = (uint64_t*)calloc((size_t)ng + 1, sizeof(uint64_t));
    if (!ord || !cur) { free(ord); free(cur); return -2; }
    for (i = 0; i < n; ++i) {
        int r[4];
        tile_rect(&p[i], &c, r);
        if (r[2] < r[0] || r[3] < r[1]) { ord[i].key = 0; ord[i].idx = (uint32_t)i; continue; }
        if (!isfinite(p[i].depth) || p[i].depth < 0.0f) { free(ord); free(cur); return -1; }
        ord[i].key = f2u(p[i].depth);
        ord[i].idx = (uint32_t)i;
        {
            const int gx0 = r[0] / g, gx1 = r[2] / g, gy0 = r[1] / g, gy1 = r[3] / g;
            int gy, gx;
            for (gy = gy0; gy <= gy1; ++gy)
                for (gx = gx0; gx <= gx1; ++gx) ++cur[gy * c.groups_x + gx + 1];
        }
    }
    for (i = 1; i <= ng; ++i) cur[i] += cur[i - 1];
    for (i = 0; i <= ng; ++i) offsets[i] = (uint32_t)cur[i];
    qsort(ord, (size_t)n, sizeof(dpair), dpair_cmp);
    for (i = 0; i < n; ++i) {
        const tor_projected* q = &p[ord[i].idx];
        int r[4];
        tile_rect(q, &c, r);
        if (r[2] < r[0] || r[3] < r[1]) continue;
        {
            const int gx0 = r[0] / g, gx1 = r[2] / g, gy0 = r[1] / g, gy1 = r[3] / g;
            int gy, gx;
            for (gy = gy0; gy <= gy1; ++gy)
                for (gx = gx0; gx <= gx1; ++gx) {
                    const int gid = gy * c.groups_x + gx;
                    tor_entry* o = &out[cur[gid]++];
                    uint32_t mask = 0;
                    const int ty0 = r[1] > gy * g ? r[1] : gy * g;
                    const int ty1 = r[3] < gy * g + g - 1 ? r[3] : gy * g + g - 1;
                    const int tx0 = r[0] > gx * g ? r[0] : gx * g;
                    const int tx1 = r[2] < gx * g + g - 1 ? r[2] : gx * g + g - 1;
                    int ty, tx;
                    for (ty = ty0; ty <= ty1; ++ty)
                        for (tx = tx0; tx <= tx1; ++tx) mask |= 1u << ((ty - gy * g) * g + (tx - gx * g));
                    o->gaussian_index = ord[i].idx;
                    o->depth = q->depth;
                    o->mask = mask;
                }
        }
    }
    free(ord);
    free(cur);
    return total;
}

/* ------------------------------------------------------------------------------------------ */
/* operands.hpp:16-72, raster_scalar.hpp:29-55 — staged operands, canonical power, alpha, blend */
/* ------------------------------------------------------------------------------------------ */
typedef struct { float q1, q2, q3, mx, my, op; } sop;  /* widened lane values */

static sop stage(const tor_projected* p, int fp16) {
    sop s;
    s.q1 = -0.5f * p->conic[0];
    s.q2 = -p->conic[1];
    s.q3 = -0.5f * p->conic[2];
    s.mx = p->mean2d[0];
    s.my = p->mean2d[1];
    s.op = p->opacity;
    if (fp16) {
        s.q1 = q16(s.q1); s.q2 = q16(s.q2); s.q3 = q16(s.q3);
        s.mx = q16(s.mx); s.my = q16(s.my); s.op = q16(s.op);
    }
    return s;
}

/* pixel_basis + splat_power (operands.hpp:48-72): zero accumulator, terms in order, no FMA. */
static float power_of(const sop* s, float px, float py, int fp16) {
    float dx = px - s->mx, dy = py - s->my, f1, f2, f3, acc;
    if (fp16) { dx = q16(dx); dy = q16(dy); }
    f1 = dx * dx; f2 = dx * dy; f3 = dy * dy;
    if (fp16) { f1 = q16(f1); f2 = q16(f2); f3 = q16(f3); }
    acc = 0.0f;
    acc += s->q1 * f1;
    acc += s->q2 * f2;
    acc += s->q3 * f3;
    return acc;
}

typedef struct { float t, a[3]; int done; } pstate;

/* alpha_of (raster_scalar.hpp:40-45) + blend (:49-55). Returns 1 if blended. */
static int step(pstate* st, float power, float op, const float* color, const tor_options* k) {
    float alpha, e;
    if (power > 0.0f) power = 0.0f;
    e = op * expf(power);
    alpha = (e < k->alpha_clamp) ? e : k->alpha_clamp; /* std::min(clamp, e) */
    if (alpha < k->alpha_skip) return 0;
    {
        const float w = st->t * alpha;
        for (int c = 0; c < 3; ++c) st->a[c] = st->a[c] + w * color[c];
        st->t *= (1.0f - alpha);
        if (st->t < k->t_terminate) st->done = 1;
    }
    return 1;
}

static float clamp01(float v) { return v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v); }

/* raster_scalar.cpp:9-48 rasterize_tile (per pixel walk of a tile list). */
static void raster_tile(int tx, int ty, const tor_entry* e, const uint32_t* off,
                        const tor_projected* p, const gcfg* c, const tor_options* k, float* img,
                        tor_counters* cnt) {
    const int tid = ty * c->tiles_x + tx;
    const uint32_t b = off[tid], en = off[tid + 1];
    const int fp16 = k->mode != 0;
    const int x0 = tx * 16, y0 = ty * 16;
    const int x1 = x0 + 16 < c->w ? x0 + 16 : c->w;
    const int y1 = y0 + 16 < c->h ? y0 + 16 : c->h;
    if (b == en) return;
    for (int y = y0; y < y1; ++y)
        for (int x = x0; x < x1; ++x) {
            const float px = (float)x + 0.5f, py = (float)y + 0.5f;
            pstate st = {1.0f, {0.0f, 0.0f, 0.0f}, 0};
            for (uint32_t i = b; i < en; ++i) {
                const tor_projected* g = &p[e[i].gaussian_index];
                const sop s = stage(g, fp16);
                const int bl = step(&st, power_of(&s, px, py, fp16), s.op, g->color, k);
                if (cnt) { cnt->walked_pairs++; cnt->blended_pairs += (uint64_t)bl; }
                if (st.done) break;
            }
            {
                float* o = img + ((size_t)y * c->w + x) * 3;
                o[0] = st.a[0]; o[1] = st.a[1]; o[2] = st.a[2];
            }
        }
}

/* raster_tensor.cpp:64-160 rasterize_group_impl: chunk -> live tile -> panel -> pixel walk, with
 * the OpReport counters.  The fragment reduction is bit-identical to splat_power (the reference
 * pins this: tests/acceptance.cpp:82-171), so power_of() stands in for fragment_dot(). */
static void raster_group(int gidx, const tor_entry* e, const uint32_t* off, const tor_projected* p,
                         const gcfg* c, const tor_options* k, float* img, tor_counters* cnt) {
    const int gx = gidx % c->groups_x, gy = gidx / c->groups_x;
    const int nt = c->g * c->g;
    const int fp16 = k->mode != 0;
    const uint32_t b = off[gidx], en = off[gidx + 1];
    int chunk_len = k->chunk_len < 1 ? 1 : (k->chunk_len > 16 ? 16 : k->chunk_len);
    typedef struct { int px0, py0, w, h, live, in_grid; pstate px[256]; } tctx;
    tctx* t = (tctx*)calloc((size_t)nt, sizeof(tctx));
    for (int r = 0; r < c->g; ++r)
        for (int cc = 0; cc < c->g; ++cc) {
            tctx* tc = &t[r * c->g + cc];
            const int tx = gx * c->g + cc, ty = gy * c->g + r;
            tc->in_grid = tx < c->tiles_x && ty < c->tiles_y;
            for (int i = 0; i < 256; ++i) { tc->px[i].t = 1.0f; }
            if (!tc->in_grid) continue;
            tc->px0 = tx * 16;
            tc->py0 = ty * 16;
            tc->w = c->w - tc->px0 < 16 ? c->w - tc->px0 : 16;
            tc->h = c->h - tc->py0 < 16 ? c->h - tc->py0 : 16;
            tc->live = tc->w * tc->h;
        }
    for (uint32_t at = b; at < en;) {
        int live_tiles = 0;
        for (int i = 0; i < nt; ++i)
            if (t[i].in_grid && t[i].live > 0) ++live_tiles;
        if (live_tiles == 0) break;
        {
            const int len = (uint32_t)chunk_len < en - at ? chunk_len : (int)(en - at);
            const tor_entry* ch = e + at;
            at += (uint32_t)len;
            if (cnt) cnt->chunk_loads++;
            for (int local = 0; local < nt; ++local) {
                tctx* tc = &t[local];
                int rows[16], nrows = 0;
                if (!tc->in_grid || tc->live == 0) continue;
                for (int i = 0; i < len; ++i)
                    if (ch[i].mask & (1u << local)) rows[nrows++] = i;
                if (cnt) cnt->skipped_pairs += (uint64_t)(len - nrows);
                if (nrows == 0) continue;
                for (int panel = 0; panel < 16; ++panel) {
                    if (panel >= tc->h) break;
                    if (cnt) {
                        cnt->fragment_ops++;
                        cnt->used_lanes += (uint64_t)nrows * 16 * 3;
                        cnt->total_lanes += 16 * 16 * 16;
                    }
                    for (int x = 0; x < tc->w; ++x) {
                        pstate* st = &tc->px[panel * 16 + x];
                        const float pxc = (float)(tc->px0 + x) + 0.5f;
                        const float pyc = (float)(tc->py0 + panel) + 0.5f;
                        if (st->done) continue;
                        for (int gi = 0; gi < nrows; ++gi) {
                            const tor_projected* g = &p[ch[rows[gi]].gaussian_index];
                            const sop s = stage(g, fp16);
                            const int bl = step(st, power_of(&s, pxc, pyc, fp16), s.op, g->color, k);
                            if (cnt) { cnt->walked_pairs++; cnt->blended_pairs += (uint64_t)bl; }
                            if (st->done) { --tc->live; break; }
                        }
                    }
                }
            }
        }
    }
    for (int i = 0; i < nt; ++i) {
        const tctx* tc = &t[i];
        if (!tc->in_grid) continue;
        for (int y = 0; y < tc->h; ++y)
            for (int x = 0; x < tc->w; ++x) {
                float* o = img + ((size_t)(tc->py0 + y) * c->w + (tc->px0 + x)) * 3;
                const pstate* st = &tc->px[y * 16 + x];
                o[0] = st->a[0]; o[1] = st->a[1]; o[2] = st->a[2];
            }
    }
    free(t);
}

int tor_rasterize(const tor_entry* entries, const uint32_t* offsets, const tor_projected* p,
                  int width, int height, const tor_options* opt, float* out_rgb,
                  tor_counters* counters) {
    gcfg c;
    if (gcfg_make(opt->group_size, width, height, &c) != 0) return -1;
    if (counters) memset(counters, 0, sizeof(*counters));
    memset(out_rgb, 0, (size_t)width * height * 3 * sizeof(float));
    if (opt->backend == 0) {
        if (opt->group_size != 1) return -1; /* raster_scalar.cpp:56-57 */
        for (int ty = 0; ty < c.tiles_y; ++ty)
            for (int tx = 0; tx < c.tiles_x; ++tx)
                raster_tile(tx, ty, entries, offsets, p, &c, opt, out_rgb, counters);
    } else {
        for (int gi = 0; gi < c.groups_x * c.groups_y; ++gi)
            raster_group(gi, entries, offsets, p, &c, opt, out_rgb, counters);
    }
    for (int64_t i = 0; i < (int64_t)width * height * 3; ++i) out_rgb[i] = clamp01(out_rgb[i]);
    return 0;
}

/* render.cpp:7-35 */
int tor_render(const float* rec, int64_t n, int deg, const tor_camera* cam, const tor_options* opt,
               float* out_rgb, uint64_t* stats10, tor_counters* counters) {
    gcfg c;
    uint64_t st3[3], app = 0;
    tor_counters local;
    int rc;
    if (opt->backend == 0 && opt->group_size != 1) return -1;
    if (opt->workers < 1) return -1;
    if (gcfg_make(opt->group_size, cam->width, cam->height, &c) != 0) return -1;
    {
        tor_projected* p = (tor_projected*)malloc((size_t)(n ? n : 1) * sizeof(tor_projected));
        const int64_t np = tor_project(rec, n, deg, cam, p, st3);
        if (np < 0) { free(p); return -1; }
        {
            const int64_t total = tor_bin_sort(p, np, cam->width, cam->height, opt->group_size,
                                               NULL, 0, NULL, &app);
            tor_entry* e = (tor_entry*)malloc((size_t)(total ? total : 1) * sizeof(tor_entry));
            uint32_t* off = (uint32_t*)malloc((size_t)(c.groups_x * c.groups_y + 1) * 4);
            if (tor_bin_sort(p, np, cam->width, cam->height, opt->group_size, e, total, off, NULL) < 0) {
                free(p); free(e); free(off);
                return -1;
            }
            rc = tor_rasterize(e, off, p, cam->width, cam->height, opt, out_rgb, &local);
            if (stats10) {
                stats10[0] = st3[0]; stats10[1] = st3[1]; stats10[2] = st3[2];
                stats10[3] = (uint64_t)total; stats10[4] = app;
                if (opt->backend == 0) {
                    stats10[5] = stats10[6] = stats10[7] = stats10[8] = stats10[9] = 0;
                } else {
                    stats10[5] = local.fragment_ops; stats10[6] = local.chunk_loads;
                    stats10[7] = local.skipped_pairs; stats10[8] = local.used_lanes;
                    stats10[9] = local.total_lanes;
                }
            }
            if (counters) *counters = local;
            free(e); free(off);
        }
        free(p);
    }
    return rc;
}

/* tests/oracles.hpp:112-152 */
typedef struct { float d; uint32_t i; } dkey;
static int dkey_cmp(const void* a, const void* b) {
    const dkey* x = (const dkey*)a;
    const dkey* y = (const dkey*)b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

int tor_reference_render(const tor_projected* p, int64_t n, int width, int height, float* out_rgb) {
    dkey* ord = (dkey*)malloc((size_t)(n ? n : 1) * sizeof(dkey));
    for (int64_t i = 0; i < n; ++i) { ord[i].d = p[i].depth; ord[i].i = (uint32_t)i; }
    qsort(ord, (size_t)n, sizeof(dkey), dkey_cmp);
    for (int y = 0; y < height; ++y)
        for (int x = 0; x < width; ++x) {
            const float px = (float)x + 0.5f, py = (float)y + 0.5f;
            float t = 1.0f, acc[3] = {0.0f, 0.0f, 0.0f};
            for (int64_t j = 0; j < n; ++j) {
                const tor_projected* g = &p[ord[j].i];
                const float dx = px - g->mean2d[0];
                const float dy = py - g->mean2d[1];
                float power = 0.0f, alpha, e;
                power += (-0.5f * g->conic[0]) * (dx * dx);
                power += (-g->conic[1]) * (dx * dy);
                power += (-0.5f * g->conic[2]) * (dy * dy);
                if (power > 0.0f) power = 0.0f;
                e = g->opacity * expf(power);
                alpha = (e < 0.99f) ? e : 0.99f;
                if (alpha < 1.0f / 255.0f) continue;
                {
                    const float w = t * alpha;
                    acc[0] += w * g->color[0];
                    acc[1] += w * g->color[1];
                    acc[2] += w * g->color[2];
                    t *= (1.0f - alpha);
                    if (t < 1e-4f) break;
                }
            }
            {
                float* o = out_rgb + ((size_t)y * width + x) * 3;
                for (int c = 0; c < 3; ++c) o[c] = clamp01(acc[c]);
            }
        }
    free(ord);
    return 0;
}

void tor_encode_ppm(const float* rgb, int64_t n_floats, uint8_t* out) {
    for (int64_t i = 0; i < n_floats; ++i) out[i] = (uint8_t)lrintf(clamp01(rgb[i]) * 255.0f);
}

/* glibc 2.39 expf restated (the algorithm the GPU exact-emulation rasteriser runs in
 * paper_2605_17855_b200/csrc/tgs_expf.cuh): k = round(x 32/ln2) by the 0x1.8p52 shift, a 32-entry
 * 2^(i/32) table, a cubic in double precision.  tests/test_oracle.py compares it with this host's
 * libm expf over a dense sweep of the negative floats. */
static double tor_asdouble(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
static uint64_t tor_asuint64(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
float tor_expf_glibc(float x) {
    static uint64_t tab[32];
    static int init = 0;
    if (!init) {
        for (int i = 0; i < 32; ++i) tab[i] = tor_asuint64(exp2((double)i / 32)) - ((uint64_t)i << 47);
        init = 1;
    }
    if (x < -0x1.9fe368p6f) return 0.0f;
    const double inv = 0x1.71547652b82fep+0 * 32.0, shift = 0x1.8p+52;
    const double c0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0, c1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0,
                 c2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    const double z = inv * (double)x;
    double kd = z + shift;
    const uint64_t ki = tor_asuint64(kd);
    kd -= shift;
    const double r = z - kd;
    const double s = tor_asdouble(tab[ki % 32] + (ki << 47));
    const double zz = c0 * r + c1, r2 = r * r;
    double y = c2 * r + 1.0;
    y = zz * r2 + y;
    return (float)(y * s);
}

/* count of floats x = -(bits of step*k) in [lo_bits, hi_bits] where tor_expf_glibc(x) != expf(x) */
int64_t tor_expf_sweep(uint32_t lo_bits, uint32_t hi_bits, uint32_t step, float* first_bad) {
    int64_t bad = 0;
    for (uint64_t u = lo_bits; u <= hi_bits; u += step) {
        float x;
        const uint32_t b = (uint32_t)u;
        memcpy(&x, &b, 4);
        const float a = tor_expf_glibc(x), e = expf(x);
        if (memcmp(&a, &e, 4) != 0) {
            if (!bad && first_bad) *first_bad = x;
            ++bad;
        }
    }
    return bad;
}
