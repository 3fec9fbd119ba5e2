// Test driver for the C++ drop-in (cpp/gsr_b200.hpp): written against the reference's public API
// (gsr::Gaussian3D / Camera / RenderOptions / render), the way a reference user calls it.
//   dropin <records.f32> <n> <sh_degree> <camera.f32 (16 view + fx fy w h near far)> <backend> <G>
//          <out.f32>
// Writes the RGB image followed by the RenderResult counters (input culled dropped entries
// tile_appearances as float64).  Exit codes follow the reference CLI: 0 ok, 2 exception
// (tools/gsrender.cpp:237-240).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "gsr_b200.hpp"

int main(int argc, char** argv) {
    if (argc != 8) {
        std::fprintf(stderr, "usage: dropin records n sh_degree camera backend G out\n");
        return 1;
    }
    try {
        const long n = std::atol(argv[2]);
        const int deg = std::atoi(argv[3]);
        const int rf = deg == 3 ? 59 : 14;
        std::vector<float> rec(static_cast<size_t>(n) * rf);
        std::ifstream fr(argv[1], std::ios::binary);
        fr.read(reinterpret_cast<char*>(rec.data()), static_cast<std::streamsize>(rec.size() * sizeof(float)));
        std::vector<gsr::Gaussian3D> scene(n);
        for (long i = 0; i < n; ++i) {
            const float* r = &rec[i * rf];
            gsr::Gaussian3D& g = scene[i];
            g.mean = Eigen::Vector3f(r[0], r[1], r[2]);
            g.scale = Eigen::Vector3f(r[3], r[4], r[5]);
            g.rotation = Eigen::Quaternionf(r[6], r[7], r[8], r[9]);
            g.opacity = r[10];
            g.sh_dc = Eigen::Vector3f(r[11], r[12], r[13]);
            if (deg == 3) {
                std::array<float, gsr::kShRestCoeffs> sh{};
                for (int k = 0; k < gsr::kShRestCoeffs; ++k) sh[k] = r[14 + k];
                g.sh_rest = sh;
            }
        }
        float cv[22];
        std::ifstream fc(argv[4], std::ios::binary);
        fc.read(reinterpret_cast<char*>(cv), sizeof(cv));
        gsr::Camera cam;
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) cam.view(r, c) = cv[r * 4 + c];
        cam.focal_x = cv[16];
        cam.focal_y = cv[17];
        cam.width = static_cast<int>(cv[18]);
        cam.height = static_cast<int>(cv[19]);
        cam.near = cv[20];
        cam.far = cv[21];
        gsr::RenderOptions opt;
        opt.backend = std::atoi(argv[5]) == 0 ? gsr::Backend::scalar : gsr::Backend::tensor;
        opt.group_size = std::atoi(argv[6]);
        const gsr::RenderResult res = gsr::render(scene, cam, opt);
        // the persistent-scene path must agree with the one-shot call
        gsr::b200::DeviceScene ds(scene);
        const gsr::RenderResult res2 = ds.render(cam, opt);
        if (res2.image.rgb != res.image.rgb) {
            std::fprintf(stderr, "DeviceScene image differs from gsr::render\n");
            return 3;
        }
        std::ofstream fo(argv[7], std::ios::binary);
        fo.write(reinterpret_cast<const char*>(res.image.rgb.data()),
                 static_cast<std::streamsize>(res.image.rgb.size() * sizeof(float)));
        const double counters[5] = {double(res.projection.input), double(res.projection.culled),
                                    double(res.projection.dropped_degenerate), double(res.entries),
                                    double(res.tile_appearances)};
        fo.write(reinterpret_cast<const char*>(counters), sizeof(counters));
        return 0;
    } catch (const gsr::ValidationError& e) {
        std::fprintf(stderr, "validation: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
