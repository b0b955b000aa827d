// shim_demo.cpp -- the drop-in in use: a reference-side program renders the
// same frame with rlcuts::render_frame (CPU reference library) and with
// rlcuts::b200::render_frame (this repo, via the C-ABI) and compares them.
// Prints "MATCH <lookups> <cells>" when image, statistics, per-pass
// split-collapse counts and per-pass mse against a reference image are
// identical.
#include <cstdio>
#include <cstring>
#include <exception>

#include "rlcuts/render.hpp"
#include "rlcuts/scene_gen.hpp"
#include "rlcuts_b200_shim.hpp"

int main(int argc, char** argv) {
  try {
    const int k = argc > 1 ? std::atoi(argv[1]) : 2;
    rlcuts::Scene scene = rlcuts::gen_cornell_grid(k, 1, 128);
    scene.camera.width = 64;
    scene.camera.height = 48;
    rlcuts::RenderConfig cfg;
    cfg.spp = 8;
    cfg.passes = 4;
    cfg.sampler = rlcuts::SamplerKind::rl_lightcuts;
    const rlcuts::RenderContext ctx = rlcuts::build_context(scene, cfg);
    // scored against a reference image after every pass (render.cpp:226-228):
    // a shorter render of the same scene stands in for the ground truth
    rlcuts::RenderConfig ref_cfg = cfg;
    ref_cfg.seed = 9;
    const rlcuts::Image truth = rlcuts::render_frame(ctx, ref_cfg).image;
    const rlcuts::RenderResult cpu = rlcuts::render_frame(ctx, cfg, &truth);
    const rlcuts::RenderResult gpu = rlcuts::b200::render_frame(ctx, cfg, &truth);
    bool same = cpu.image.pixels.size() == gpu.image.pixels.size() &&
                cpu.lookups == gpu.lookups && cpu.occupied_cells == gpu.occupied_cells &&
                cpu.fallback_hits == gpu.fallback_hits && cpu.sc_changes == gpu.sc_changes &&
                cpu.pass_mse == gpu.pass_mse && gpu.pass_mse.size() == cfg.passes;
    for (size_t i = 0; same && i < cpu.image.pixels.size(); ++i)
      same = cpu.image.pixels[i] == gpu.image.pixels[i];
    std::printf("%s %llu %u cpu_ms=%.1f gpu_ms=%.1f\n", same ? "MATCH" : "DIFFER",
                (unsigned long long)gpu.lookups, gpu.occupied_cells, cpu.wall_ms, gpu.wall_ms);
    return same ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("ERROR %s\n", e.what());
    return 2;
  }
}
