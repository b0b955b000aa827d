// shim_demo.cpp -- the drop-in in use: a reference-side program renders the
// same frame with rlcuts::render_frame (CPU reference library) and with
// rlcuts::b200::render_frame (this repo, via the C-ABI) and compares them.
// Prints "MATCH <lookups> <cells>" when image, statistics, per-pass
// split-collapse counts and per-pass mse against a reference image are
// identical.  `shim_demo session`: rlcuts::b200::Session driven pass by pass
// beside the reference's own HashGrid; its HashGrid accessors (dump_stats,
// memory_records, the keys of touched_slots) must agree.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <exception>
#include <sstream>
#include <tuple>
#include <vector>

#include "rlcuts/render.hpp"
#include "rlcuts/scene_gen.hpp"
#include "rlcuts_b200_shim.hpp"

static int session_demo() {
  rlcuts::Scene scene = rlcuts::gen_cornell_grid(2, 1, 64);
  scene.camera.width = 48;
  scene.camera.height = 36;
  rlcuts::RenderConfig cfg;
  cfg.spp = 3;
  cfg.passes = 3;
  cfg.sampler = rlcuts::SamplerKind::rl_lightcuts;
  cfg.cut.cut_size = 32;
  const rlcuts::RenderContext ctx = rlcuts::build_context(scene, cfg);
  rlcuts::HashConfig hash = cfg.hash;
  hash.base_tile = ctx.base_tile;
  rlcuts::HashGrid grid(hash, rlcuts::init_cut(ctx.tree, cfg.cut.cut_size, cfg.cut.eps_q));
  rlcuts::Framebuffer fb(scene.camera.width, scene.camera.height);
  rlcuts::b200::Session gpu(ctx, cfg);
  for (uint32_t p = 0; p < 2; ++p) {
    rlcuts::render_pass(ctx, cfg, p, &grid, fb);
    rlcuts::end_of_pass_update(grid, ctx.tree, cfg.cut, cfg.workers);
    gpu.render_pass(p);
    gpu.end_of_pass_update();
  }
  rlcuts::render_pass(ctx, cfg, 2, &grid, fb);  // touched slots set, not yet cleared
  gpu.render_pass(2);
  std::ostringstream a, b;
  grid.dump_stats(a);
  gpu.dump_stats(b);
  using K = std::tuple<int32_t, int32_t, int32_t, uint32_t, uint32_t>;
  auto keys = [](auto&& slots, auto&& key_of) {
    std::vector<K> v;
    for (uint32_t s : slots) {
      const rlcuts::CellKey k = key_of(s);
      v.emplace_back(k.qx, k.qy, k.qz, k.qn, k.level);
    }
    std::sort(v.begin(), v.end());
    return v;
  };
  const auto kc = keys(grid.touched_slots(), [&](uint32_t s) { return grid.key_of(s); });
  const auto kg = keys(gpu.touched_slots(), [&](uint32_t s) { return gpu.key_of(s); });
  const bool same = a.str() == b.str() && grid.memory_records() == gpu.memory_records() &&
                    kc == kg && !kc.empty();
  std::printf("%s touched=%zu records=%llu\n", same ? "MATCH" : "DIFFER", kg.size(),
              (unsigned long long)gpu.memory_records());
  return same ? 0 : 1;
}

int main(int argc, char** argv) {
  try {
    if (argc > 1 && std::strcmp(argv[1], "session") == 0) return session_demo();
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
