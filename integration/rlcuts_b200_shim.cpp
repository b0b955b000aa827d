// rlcuts_b200_shim.cpp -- implementation of rlcuts_b200_shim.hpp over the
// C-ABI.  Builds against the reference headers (proj/include) and
// include/rlcuts_b200.h; no reference source is needed.
#include "rlcuts_b200_shim.hpp"

#include <algorithm>
#include <ostream>

#include <chrono>
#include <stdexcept>
#include <string>
#include <vector>

#include "rlcuts_b200.h"

namespace rlcuts::b200 {

namespace {

// Maps an rlc_status back to the reference's exception types.
void check(rlc_status st) {
  if (st == RLC_OK) return;
  const std::string msg = rlc_last_error();
  if (st == RLC_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == RLC_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

rlc_render_config to_c(const RenderConfig& c) {
  rlc_render_config r;
  check(rlc_render_config_default(&r));
  r.spp = c.spp;
  r.passes = c.passes;
  r.max_depth = c.max_depth;
  r.sampler = uint32_t(c.sampler);
  r.cut.cut_size = c.cut.cut_size;
  r.cut.alpha = c.cut.alpha;
  r.cut.split_threshold = c.cut.split_threshold;
  r.cut.eps_q = c.cut.eps_q;
  r.cut.iterations = c.cut.iterations;
  r.cut.alpha_schedule = uint32_t(c.cut.alpha_schedule);
  r.hash.capacity = c.hash.capacity;
  r.hash.base_tile = c.hash.base_tile;
  r.hash.probe_limit = c.hash.probe_limit;
  r.hash.normal_bits = c.hash.normal_bits;
  r.hash.jitter_scale = c.hash.jitter_scale;
  r.seed = c.seed;
  r.workers = c.workers;
  return r;
}

// Flattened rlcuts::Scene (scene.hpp:53-67) kept alive for the descriptor.
struct SceneArrays {
  std::vector<double> vertices, materials;
  std::vector<uint32_t> material_ids;
  rlc_scene_desc desc{};

  explicit SceneArrays(const Scene& s) {
    for (const Triangle& t : s.triangles) {
      for (const Vec3* p : {&t.p0, &t.p1, &t.p2}) {
        vertices.push_back(p->x);
        vertices.push_back(p->y);
        vertices.push_back(p->z);
      }
      material_ids.push_back(t.material_id);
    }
    for (const Material& m : s.materials) {
      for (double v : {m.albedo.x, m.albedo.y, m.albedo.z, m.emission.x, m.emission.y,
                       m.emission.z})
        materials.push_back(v);
    }
    desc.num_triangles = uint32_t(s.triangles.size());
    desc.num_materials = uint32_t(s.materials.size());
    desc.vertices = vertices.data();
    desc.material_ids = material_ids.data();
    desc.materials = materials.data();
    const Camera& c = s.camera;
    const Vec3* cam[3] = {&c.origin, &c.look_at, &c.up};
    double* dst[3] = {desc.cam_origin, desc.cam_look_at, desc.cam_up};
    for (int k = 0; k < 3; ++k) {
      dst[k][0] = cam[k]->x;
      dst[k][1] = cam[k]->y;
      dst[k][2] = cam[k]->z;
    }
    desc.vfov_degrees = c.vfov_degrees;
    desc.width = c.width;
    desc.height = c.height;
  }
};

}  // namespace

struct Session::Impl {
  const RenderContext* ctx = nullptr;
  rlc_render_config cfg{};
  rlc_context* c = nullptr;
  rlc_grid* g = nullptr;
  rlc_framebuffer* fb = nullptr;

  ~Impl() {
    rlc_framebuffer_destroy(fb);
    rlc_grid_destroy(g);
    rlc_context_destroy(c);
  }
};

Session::Session(const RenderContext& ctx, const RenderConfig& config, int device)
    : impl_(std::make_unique<Impl>()) {
  if (ctx.scene == nullptr) throw std::invalid_argument("Session: context without a scene");
  impl_->ctx = &ctx;
  impl_->cfg = to_c(config);
  impl_->cfg.hash.base_tile = ctx.base_tile;  // resolved by build_context (render.cpp:153-155)
  SceneArrays arrays(*ctx.scene);
  check(rlc_context_create(&arrays.desc, &impl_->cfg, device, &impl_->c));
  if (config.sampler == SamplerKind::rl_lightcuts)
    check(rlc_grid_create(impl_->c, &impl_->cfg, &impl_->g));
  check(rlc_framebuffer_create(impl_->c, ctx.scene->camera.width, ctx.scene->camera.height,
                               &impl_->fb));
}

Session::~Session() = default;

void Session::render_pass(uint32_t pass_index) {
  check(rlc_render_pass(impl_->c, &impl_->cfg, pass_index, impl_->g, impl_->fb));
}

void Session::update_scene(const Scene& scene) {
  SceneArrays arrays(scene);
  check(rlc_context_update_scene(impl_->c, &arrays.desc));
}

uint32_t Session::end_of_pass_update() {
  if (impl_->g == nullptr) return 0;
  uint32_t changes = 0;
  check(rlc_end_of_pass_update(impl_->g, impl_->c, &impl_->cfg.cut, &changes));
  return changes;
}

void Session::framebuffer(Framebuffer& out) const {
  const size_t n = size_t(out.width) * size_t(out.height);
  std::vector<double> sum(3 * n);
  std::vector<uint64_t> count(n);
  check(rlc_framebuffer_download(impl_->fb, sum.data(), count.data()));
  for (size_t i = 0; i < n; ++i) {
    out.sum[i] = Vec3{sum[3 * i], sum[3 * i + 1], sum[3 * i + 2]};
    out.count[i] = count[i];
  }
}

uint32_t Session::occupied_count() const {
  rlc_grid_stats s{};
  if (impl_->g) check(rlc_grid_stats_get(impl_->g, &s));
  return s.occupied;
}

uint64_t Session::lookup_count() const {
  rlc_grid_stats s{};
  if (impl_->g) check(rlc_grid_stats_get(impl_->g, &s));
  return s.lookups;
}

uint64_t Session::fallback_hits() const {
  rlc_grid_stats s{};
  if (impl_->g) check(rlc_grid_stats_get(impl_->g, &s));
  return s.fallback_hits;
}

namespace {
struct SlotView {
  std::vector<uint32_t> slot;
  std::vector<rlc_cell_key> key;
  std::vector<uint8_t> touched;
};

SlotView slot_view(rlc_grid* g) {
  SlotView v;
  if (!g) return v;
  uint32_t n = 0;
  check(rlc_grid_slots(g, 0, nullptr, nullptr, nullptr, nullptr, &n));
  v.slot.resize(n);
  v.key.resize(n);
  v.touched.resize(n);
  check(rlc_grid_slots(g, n, v.slot.data(), nullptr, v.key.data(), v.touched.data(), &n));
  return v;
}
}  // namespace

CellKey Session::key_of(uint32_t slot) const {
  const SlotView v = slot_view(impl_->g);
  for (size_t i = 0; i < v.slot.size(); ++i)
    if (v.slot[i] == slot) {
      const rlc_cell_key& k = v.key[i];
      return CellKey{k.qx, k.qy, k.qz, k.qn, k.level};
    }
  return CellKey{};  // an empty slot holds a default key
}

std::vector<uint32_t> Session::touched_slots() const {
  const SlotView v = slot_view(impl_->g);
  std::vector<uint32_t> out;
  for (size_t i = 0; i < v.slot.size(); ++i)
    if (v.touched[i]) out.push_back(v.slot[i]);
  return out;
}

uint64_t Session::memory_records() const {
  rlc_grid_stats s{};
  if (impl_->g) check(rlc_grid_stats_get(impl_->g, &s));
  return uint64_t(s.occupied) * s.cut_size;  // every cut keeps the template's size
}

void Session::dump_stats(std::ostream& out) const {  // hash_grid.cpp:189-202
  rlc_grid_stats s{};
  if (impl_->g) check(rlc_grid_stats_get(impl_->g, &s));
  uint64_t histogram[17] = {};
  for (const rlc_cell_key& k : slot_view(impl_->g).key) ++histogram[std::min<uint32_t>(k.level, 16)];
  out << "occupied,lookups,fallback_hits";
  for (uint32_t level = 0; level <= 16; ++level) out << ",level_" << level;
  out << "\n";
  out << s.occupied << ',' << s.lookups << ',' << s.fallback_hits;
  for (uint32_t level = 0; level <= 16; ++level) out << ',' << histogram[level];
  out << "\n";
}

RenderResult render_frame(const RenderContext& ctx, const RenderConfig& config,
                          const Image* reference) {
  if (config.passes == 0 || config.spp == 0 || config.spp % config.passes != 0)
    throw std::invalid_argument("render_frame: spp must be divisible by passes");
  if (ctx.scene == nullptr) throw std::invalid_argument("render_frame: context without a scene");
  rlc_render_config cfg = to_c(config);
  cfg.hash.base_tile = ctx.base_tile;  // resolved by build_context (render.cpp:153-155)
  SceneArrays arrays(*ctx.scene);
  rlc_context* c = nullptr;
  check(rlc_context_create(&arrays.desc, &cfg, 0, &c));
  struct Guard {
    rlc_context* c;
    ~Guard() { rlc_context_destroy(c); }
  } guard{c};
  const int w = ctx.scene->camera.width, h = ctx.scene->camera.height;
  std::vector<double> img(size_t(w) * size_t(h) * 3);
  std::vector<uint32_t> changes(config.passes);
  std::vector<double> pass_mse(config.passes);
  rlc_render_result r{};
  r.sc_changes = changes.data();
  if (reference != nullptr) {  // scored after every pass on the device path
    std::vector<double> ref;
    ref.reserve(reference->pixels.size() * 3);
    for (const Vec3& p : reference->pixels) {
      ref.push_back(p.x);
      ref.push_back(p.y);
      ref.push_back(p.z);
    }
    check(rlc_render_frame_scored(c, &cfg, ref.data(), reference->width, reference->height,
                                  img.data(), &r, pass_mse.data()));
  } else {
    check(rlc_render_frame(c, &cfg, img.data(), &r));
  }
  RenderResult result;
  result.image = Image(w, h);
  for (size_t i = 0; i < result.image.pixels.size(); ++i)
    result.image.pixels[i] = Vec3{img[3 * i], img[3 * i + 1], img[3 * i + 2]};
  result.wall_ms = r.wall_ms;
  result.occupied_cells = r.occupied_cells;
  result.lookups = r.lookups;
  result.fallback_hits = r.fallback_hits;
  result.sc_changes = changes;
  if (reference != nullptr) result.pass_mse = pass_mse;
  return result;
}

}  // namespace rlcuts::b200
