// Host-side data format either side of the path: the deterministic synthetic scene generator
// (reference: proj/src/scene_io.cpp:218-251, SplitMix64 scene_io.hpp:14-31), producing .gsb
// record layout (scene_io.cpp:102-137) directly.  Compiled with -ffp-contract=off so the
// float arithmetic (and libm sqrtf/sinf/cosf) matches the reference build bit for bit.
#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/tgs.h"

namespace tgs {
tgs_status set_err(tgs_status s, const std::string& msg);
}

namespace {

struct SplitMix64 {
    uint64_t state;
    uint64_t next() {
        uint64_t z = (state += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    float uniform() { return static_cast<float>(next() >> 40) * 0x1.0p-24f; }
    float uniform(float lo, float hi) { return lo + (hi - lo) * uniform(); }
};

}  // namespace

extern "C" tgs_status tgs_gen_synthetic_scene(uint64_t seed, int count, float extent, float scale_min,
                                              float scale_max, uint64_t sh_seed, float* out) {
    if (count < 0) return tgs::set_err(TGS_ERR_VALIDATION, "gen_synthetic_scene: count must be >= 0");
    if (!(extent > 0.0f)) return tgs::set_err(TGS_ERR_VALIDATION, "gen_synthetic_scene: extent must be > 0");
    if (!(scale_min > 0.0f) || !(scale_min <= scale_max))
        return tgs::set_err(TGS_ERR_VALIDATION, "gen_synthetic_scene: require 0 < scale_min <= scale_max");
    if (count > 0 && !out) return tgs::set_err(TGS_ERR_VALIDATION, "gen_synthetic_scene: null output");
    SplitMix64 rng{seed}, rng_sh{sh_seed};
    const int rf = sh_seed ? 59 : 14;
    for (int i = 0; i < count; ++i) {
        float* p = out + static_cast<size_t>(i) * rf;
        p[0] = rng.uniform(-extent, extent);
        p[1] = rng.uniform(-extent, extent);
        p[2] = rng.uniform(-extent, extent) + 3.0f * extent;
        p[3] = rng.uniform(scale_min, scale_max);
        p[4] = rng.uniform(scale_min, scale_max);
        p[5] = rng.uniform(scale_min, scale_max);
        // Shoemake uniform quaternion (w, x, y, z) = (s2 cos b, s1 sin a, s1 cos a, s2 sin b)
        const float u1 = rng.uniform(), u2 = rng.uniform(), u3 = rng.uniform();
        const float s1 = std::sqrt(1.0f - u1), s2 = std::sqrt(u1);
        const float a = 2.0f * static_cast<float>(M_PI) * u2;
        const float b = 2.0f * static_cast<float>(M_PI) * u3;
        float q[4] = {s1 * std::sin(a), s1 * std::cos(a), s2 * std::sin(b), s2 * std::cos(b)};  // x y z w
        // renormalize_quat (scene_io.cpp:35-43); Eigen Vector4f norm = SSE predux order
        const float n = std::sqrt((q[0] * q[0] + q[2] * q[2]) + (q[1] * q[1] + q[3] * q[3]));
        if (!(n > 0.0f) || !std::isfinite(n))
            return tgs::set_err(TGS_ERR_VALIDATION, "scene record " + std::to_string(i) +
                                                        ": quaternion has non-finite or zero norm");
        if (std::fabs(n - 1.0f) > 1e-6f)
            for (float& c : q) c /= n;
        p[6] = q[3];
        p[7] = q[0];
        p[8] = q[1];
        p[9] = q[2];
        p[10] = rng.uniform(0.2f, 0.95f);
        constexpr float kShC0 = 0.28209479177f;
        for (int c = 0; c < 3; ++c) p[11 + c] = (rng.uniform() - 0.5f) / kShC0;
        if (sh_seed)
            for (int k = 0; k < 45; ++k) p[14 + k] = rng_sh.uniform(-1.0f, 1.0f);
    }
    return TGS_OK;
}
