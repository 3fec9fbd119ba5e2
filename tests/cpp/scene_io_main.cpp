// .gsb driver for the C++ drop-in's gsr::load_scene / gsr::save_scene (the reference's scene_io
// API, scene_io.hpp:42-43):
//   scene_io load <in.gsb> <out.f32>   records (14 or 59 floats each) of the loaded scene
//   scene_io copy <in.gsb> <out.gsb>   load then save
// Exit codes like the reference CLI: 0 ok, 2 exception (message on stderr).
#include <cstdio>
#include <cstring>
#include <fstream>
#include <vector>

#include "gsr_b200.hpp"

int main(int argc, char** argv) {
    if (argc != 4) return 1;
    try {
        const auto scene = gsr::load_scene(argv[2]);
        if (std::strcmp(argv[1], "copy") == 0) {
            gsr::save_scene(scene, argv[3]);
            return 0;
        }
        std::ofstream out(argv[3], std::ios::binary);
        for (const auto& g : scene) {
            std::vector<float> r = {g.mean.x(), g.mean.y(), g.mean.z(), g.scale.x(), g.scale.y(), g.scale.z(),
                                    g.rotation.w(), g.rotation.x(), g.rotation.y(), g.rotation.z(), g.opacity,
                                    g.sh_dc.x(), g.sh_dc.y(), g.sh_dc.z()};
            if (g.sh_rest) r.insert(r.end(), g.sh_rest->begin(), g.sh_rest->end());
            out.write(reinterpret_cast<const char*>(r.data()), static_cast<std::streamsize>(r.size() * 4));
        }
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return 2;
    }
}
