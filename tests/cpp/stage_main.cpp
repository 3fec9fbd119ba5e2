// Test driver for the C++ drop-in's STAGE API (cpp/gsr_b200.hpp), written against the reference's
// public stage functions the way its own tests call them (proj/tests/test_binning.cpp,
// test_raster_*.cpp): project_scene -> build_group_entries -> sort_entries ->
// rasterize_tiles_scalar / rasterize_groups_tensor.
//   stage <records.f32> <n> <sh_degree> <camera.f32> <backend> <G> <out.bin>
// out.bin: i64 n_projected, ProjectedGaussian records (44 B, projection.hpp field order),
//          i64 n_entries, GroupEntry records (12 B), u32 offsets[group_count + 1], f32 image.
// Exit codes follow the reference CLI: 0 ok, 2 exception (tools/gsrender.cpp:237-240).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "gsr_b200.hpp"

int main(int argc, char** argv) {
    if (argc != 8) {
        std::fprintf(stderr, "usage: stage records n sh_degree camera backend G out\n");
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
        const int backend = std::atoi(argv[5]), g = std::atoi(argv[6]);

        gsr::ProjectionStats st;
        const std::vector<gsr::ProjectedGaussian> proj = gsr::project_scene(scene, cam, 4, &st);
        if (st.input != static_cast<std::size_t>(n) || st.input - st.culled - st.dropped_degenerate != proj.size()) {
            std::fprintf(stderr, "ProjectionStats inconsistent\n");
            return 3;
        }
        const gsr::GroupConfig cfg = gsr::GroupConfig::square(g, cam.width, cam.height);
        const std::vector<gsr::KeyedEntry> keyed = gsr::build_group_entries(proj, cfg);
        // every entry's mask is the member tiles of tiles_overlapped inside its group
        for (const auto& e : keyed) {
            const gsr::TileRect t = gsr::tiles_overlapped(proj[e.entry.gaussian_index], cfg);
            if (t.empty() || e.entry.mask == 0u) {
                std::fprintf(stderr, "entry without overlapped tiles\n");
                return 3;
            }
        }
        const gsr::SortedGroupLists lists = gsr::sort_entries(keyed, cfg);
        const gsr::ImageBuffer img = backend == 0
                                         ? gsr::rasterize_tiles_scalar(lists, proj, cfg, gsr::RasterConstants{})
                                         : gsr::rasterize_groups_tensor(lists, proj, cfg, gsr::TensorRasterOptions{});
        std::ofstream fo(argv[7], std::ios::binary);
        const long long np = static_cast<long long>(proj.size()), ne = static_cast<long long>(lists.entries.size());
        fo.write(reinterpret_cast<const char*>(&np), 8);
        for (const auto& p : proj) {
            const float f[10] = {p.mean2d.x(), p.mean2d.y(), p.conic_a, p.conic_b, p.conic_c,
                                 p.color.x(),  p.color.y(),  p.color.z(), p.opacity, p.depth};
            fo.write(reinterpret_cast<const char*>(f), sizeof(f));
            fo.write(reinterpret_cast<const char*>(&p.radius), 4);
        }
        fo.write(reinterpret_cast<const char*>(&ne), 8);
        fo.write(reinterpret_cast<const char*>(lists.entries.data()),
                 static_cast<std::streamsize>(lists.entries.size() * sizeof(gsr::GroupEntry)));
        fo.write(reinterpret_cast<const char*>(lists.offsets.data()),
                 static_cast<std::streamsize>(lists.offsets.size() * 4));
        fo.write(reinterpret_cast<const char*>(img.rgb.data()), static_cast<std::streamsize>(img.rgb.size() * 4));
        return 0;
    } catch (const gsr::ValidationError& e) {
        std::fprintf(stderr, "validation: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
