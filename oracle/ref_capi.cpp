// ref_capi.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A thin extern "C" wrapper around the *unmodified* reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/librlcuts_ref.so).  It lets the Python tests and bench.py's
// CPU-baseline leg drive the reference through its own public API
// (proj/include/rlcuts/*.hpp) with plain arrays, so the reference and the
// CUDA path consume byte-identical scenes.  Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
//
// Nothing here re-implements reference logic: each function marshals arrays
// into rlcuts:: types and calls the reference function named in its comment.

#include <algorithm>
#include <sstream>
#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rlcuts/bvh.hpp"
#include "rlcuts/cut.hpp"
#include "rlcuts/estimators.hpp"
#include "rlcuts/hash_grid.hpp"
#include "rlcuts/image.hpp"
#include "rlcuts/light_tree.hpp"
#include "rlcuts/render.hpp"
#include "rlcuts/rng.hpp"
#include "rlcuts/scene.hpp"
#include "rlcuts_b200.h"  // only for the plain-data config/scene structs

using namespace rlcuts;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return RLC_ERR_INVALID_ARGUMENT;
  if (dynamic_cast<const std::out_of_range*>(&e)) return RLC_ERR_OUT_OF_RANGE;
  if (const auto* io = dynamic_cast<const ImageIoError*>(&e))
    return io->code() == ImageIoErrc::io_error ? RLC_ERR_IO : RLC_ERR_PARSE;
  return RLC_ERR_INTERNAL;
}

Image to_image(const double* px, int w, int h) {
  Image im(w, h);
  for (size_t i = 0; i < im.pixels.size(); ++i)
    im.pixels[i] = Vec3{px[3 * i], px[3 * i + 1], px[3 * i + 2]};
  return im;
}

Scene to_scene(const rlc_scene_desc* d) {
  Scene s;
  s.triangles.resize(d->num_triangles);
  for (uint32_t t = 0; t < d->num_triangles; ++t) {
    const double* v = d->vertices + size_t(t) * 9;
    s.triangles[t].p0 = {v[0], v[1], v[2]};
    s.triangles[t].p1 = {v[3], v[4], v[5]};
    s.triangles[t].p2 = {v[6], v[7], v[8]};
    s.triangles[t].material_id = d->material_ids[t];
  }
  s.materials.resize(d->num_materials);
  for (uint32_t m = 0; m < d->num_materials; ++m) {
    const double* v = d->materials + size_t(m) * 6;
    s.materials[m].albedo = {v[0], v[1], v[2]};
    s.materials[m].emission = {v[3], v[4], v[5]};
  }
  s.camera.origin = {d->cam_origin[0], d->cam_origin[1], d->cam_origin[2]};
  s.camera.look_at = {d->cam_look_at[0], d->cam_look_at[1], d->cam_look_at[2]};
  s.camera.up = {d->cam_up[0], d->cam_up[1], d->cam_up[2]};
  s.camera.vfov_degrees = d->vfov_degrees;
  s.camera.width = d->width;
  s.camera.height = d->height;
  s.derive_emitters();  // proj/src/scene.cpp:33-37
  return s;
}

RenderConfig to_config(const rlc_render_config* c) {
  RenderConfig r;
  r.spp = c->spp;
  r.passes = c->passes;
  r.max_depth = c->max_depth;
  r.sampler = SamplerKind(c->sampler);
  r.cut.cut_size = c->cut.cut_size;
  r.cut.alpha = c->cut.alpha;
  r.cut.split_threshold = c->cut.split_threshold;
  r.cut.eps_q = c->cut.eps_q;
  r.cut.iterations = c->cut.iterations;
  r.cut.alpha_schedule = AlphaSchedule(c->cut.alpha_schedule);
  r.hash.capacity = c->hash.capacity;
  r.hash.base_tile = c->hash.base_tile;
  r.hash.probe_limit = c->hash.probe_limit;
  r.hash.normal_bits = c->hash.normal_bits;
  r.hash.jitter_scale = c->hash.jitter_scale;
  r.seed = c->seed;
  r.workers = c->workers;
  return r;
}

// State of one reference run: the exact loop body of render_frame
// (proj/src/render.cpp:209-224) split into callable passes, so the tests can
// read the HashGrid between passes.
struct RefRun {
  Scene scene;
  RenderConfig cfg;
  RenderContext ctx;
  std::unique_ptr<HashGrid> grid;
  std::unique_ptr<Framebuffer> fb;
};

void fill_cut(const Cut& c, uint32_t m, uint32_t i, uint32_t* node_ids, uint32_t* ends,
              double* q, double* cdf, uint32_t* visits) {
  for (uint32_t j = 0; j < m && j < c.size(); ++j) {
    const size_t o = size_t(i) * m + j;
    if (node_ids) node_ids[o] = c.node_ids[j];
    if (ends) ends[o] = c.ends[j];
    if (q) q[o] = c.q[j];
    if (cdf) cdf[o] = c.cdf[j];
    if (visits) visits[o] = c.visits[j];
  }
}

LightTree tree_from_points(uint32_t n, const double* centroids, const double* energies) {
  std::vector<EmitterRecord> em(n);
  for (uint32_t i = 0; i < n; ++i) {
    em[i].triangle_id = i;
    em[i].centroid = {centroids[3 * i], centroids[3 * i + 1], centroids[3 * i + 2]};
    em[i].energy = energies[i];
  }
  return build_light_tree(em, emitter_centroid_bounds(em));  // light_tree.cpp:50-119
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- counter RNG: proj/include/rlcuts/rng.hpp:12-43 ----
uint64_t ref_mix64(uint64_t x) { return mix64(x); }
void ref_rng_draws(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint32_t n, double* out) {
  RandomSequence r(seed, a, b, c);
  for (uint32_t i = 0; i < n; ++i) out[i] = r.next();
}

// ---- whole-pipeline runs (render.cpp:143-240) ----
void* ref_run_create(const rlc_scene_desc* desc, const rlc_render_config* config, int* status) {
  try {
    auto run = std::make_unique<RefRun>();
    run->scene = to_scene(desc);
    run->cfg = to_config(config);
    run->ctx = build_context(run->scene, run->cfg);  // render.cpp:143
    run->ctx.scene = &run->scene;
    run->ctx.accel.scene = &run->scene;
    if (run->cfg.sampler == SamplerKind::rl_lightcuts) {
      HashConfig hash = run->cfg.hash;
      hash.base_tile = run->ctx.base_tile;
      run->grid = std::make_unique<HashGrid>(
          hash, init_cut(run->ctx.tree, run->cfg.cut.cut_size, run->cfg.cut.eps_q));
    }
    run->fb = std::make_unique<Framebuffer>(run->scene.camera.width, run->scene.camera.height);
    *status = RLC_OK;
    return run.release();
  } catch (const std::exception& e) {
    *status = fail(e);
    return nullptr;
  }
}

void ref_run_destroy(void* h) { delete static_cast<RefRun*>(h); }

// The dynamic-emitter semantics of rlc_context_update_scene, through the
// reference's public API: ctx' = build_context(scene', cfg) with the light
// tree of the run's creation; the HashGrid and the Framebuffer carry over.
int ref_run_update_scene(void* h, const rlc_scene_desc* desc) {
  RefRun* run = static_cast<RefRun*>(h);
  try {
    LightTree tree0 = run->ctx.tree;
    run->scene = to_scene(desc);
    run->ctx = build_context(run->scene, run->cfg);
    run->ctx.scene = &run->scene;
    run->ctx.accel.scene = &run->scene;
    run->ctx.tree = std::move(tree0);
    return RLC_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// render_pass + end_of_pass_update (render.cpp:219-224).  Returns the
// split-collapse change count, or -status on error.
int64_t ref_run_pass(void* h, uint32_t pass_index, double* wall_ms) {
  RefRun* run = static_cast<RefRun*>(h);
  try {
    const auto t0 = std::chrono::steady_clock::now();
    render_pass(run->ctx, run->cfg, pass_index, run->grid.get(), *run->fb);
    uint32_t changes = 0;
    if (run->grid) changes = end_of_pass_update(*run->grid, run->ctx.tree, run->cfg.cut,
                                                run->cfg.workers);
    if (wall_ms)
      *wall_ms = std::chrono::duration<double, std::milli>(
                     std::chrono::steady_clock::now() - t0).count();
    return changes;
  } catch (const std::exception& e) {
    return -int64_t(fail(e));
  }
}

// render_pass alone (render.cpp:159-183).
int ref_run_render_only(void* h, uint32_t pass_index) {
  RefRun* run = static_cast<RefRun*>(h);
  try {
    render_pass(run->ctx, run->cfg, pass_index, run->grid.get(), *run->fb);
    return RLC_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_run_framebuffer(void* h, double* sum, uint64_t* count) {
  const Framebuffer& fb = *static_cast<RefRun*>(h)->fb;
  for (size_t i = 0; i < fb.sum.size(); ++i) {
    if (sum) {
      sum[3 * i] = fb.sum[i].x;
      sum[3 * i + 1] = fb.sum[i].y;
      sum[3 * i + 2] = fb.sum[i].z;
    }
    if (count) count[i] = fb.count[i];
  }
}

// out: occupied, lookups, fallback_hits, cut_size
void ref_run_stats(void* h, uint64_t* out) {
  RefRun* run = static_cast<RefRun*>(h);
  if (!run->grid) {
    out[0] = out[1] = out[2] = out[3] = 0;
    return;
  }
  out[0] = run->grid->occupied_count();
  out[1] = run->grid->lookup_count();
  out[2] = run->grid->fallback_hits();
  out[3] = run->grid->fallback_cut().size();
}

// HashGrid::dump_stats text (into out, NUL-terminated, truncated to cap),
// memory_records, and the keys of touched_slots() in slot order (5 u32 per
// key; returns their count).
uint32_t ref_run_grid_views(void* h, char* out, uint32_t cap, uint64_t* mem_records,
                            uint32_t* touched_keys, uint32_t max_keys) {
  RefRun* run = static_cast<RefRun*>(h);
  if (!run->grid) return 0;
  std::ostringstream os;
  run->grid->dump_stats(os);
  const std::string s = os.str();
  if (out && cap > 0) {
    const size_t n = std::min<size_t>(s.size(), cap - 1);
    std::memcpy(out, s.data(), n);
    out[n] = 0;
  }
  if (mem_records) *mem_records = run->grid->memory_records();
  const std::vector<uint32_t> t = run->grid->touched_slots();
  for (size_t i = 0; i < t.size() && i < max_keys; ++i) {
    const CellKey& k = run->grid->key_of(t[i]);
    touched_keys[5 * i] = uint32_t(k.qx);
    touched_keys[5 * i + 1] = uint32_t(k.qy);
    touched_keys[5 * i + 2] = uint32_t(k.qz);
    touched_keys[5 * i + 3] = k.qn;
    touched_keys[5 * i + 4] = k.level;
  }
  return uint32_t(t.size());
}

// Occupied slots in slot order (HashGrid::key_of per slot, hash_grid.hpp:90):
// slot index and 5 u32 of its CellKey.  Returns the number of occupied slots.
uint32_t ref_run_slots(void* h, uint32_t max_n, uint32_t* slot_out, uint32_t* key_out) {
  RefRun* run = static_cast<RefRun*>(h);
  if (!run->grid) return 0;
  const HashGrid& g = *run->grid;
  uint32_t n = 0;
  for (uint32_t slot = 0; slot < g.config().capacity; ++slot) {
    if (g.cut(CellHandle{slot}).size() == 0) continue;
    if (n < max_n) {
      const CellKey& k = g.key_of(slot);
      slot_out[n] = slot;
      key_out[5 * n] = uint32_t(k.qx);
      key_out[5 * n + 1] = uint32_t(k.qy);
      key_out[5 * n + 2] = uint32_t(k.qz);
      key_out[5 * n + 3] = k.qn;
      key_out[5 * n + 4] = k.level;
    }
    ++n;
  }
  return n;
}

// dout: base_tile, shadow_eps;  uout: triangles, emitters, bvh nodes, tree nodes
void ref_run_info(void* h, double* dout, uint32_t* uout) {
  RefRun* run = static_cast<RefRun*>(h);
  dout[0] = run->ctx.base_tile;
  dout[1] = run->ctx.accel.shadow_eps;
  uout[0] = uint32_t(run->scene.triangles.size());
  uout[1] = uint32_t(run->ctx.emitters.size());
  uout[2] = uint32_t(run->ctx.accel.nodes.size());
  uout[3] = uint32_t(run->ctx.tree.nodes.size());
}

// Occupied cells in slot order (an occupied slot holds a non-empty cut; an
// empty slot holds a default Cut).  Returns the number of cells written.
uint32_t ref_run_export(void* h, uint32_t max_cells, rlc_cell_key* keys, uint32_t* node_ids,
                        uint32_t* ends, double* q, double* cdf, uint32_t* visits) {
  RefRun* run = static_cast<RefRun*>(h);
  if (!run->grid) return 0;
  const HashGrid& g = *run->grid;
  const uint32_t m = g.fallback_cut().size();
  uint32_t n = 0;
  for (uint32_t slot = 0; slot < g.config().capacity; ++slot) {
    const Cut& c = g.cut(CellHandle{slot});
    if (c.size() == 0) continue;
    if (n < max_cells) {
      const CellKey& k = g.key_of(slot);
      if (keys) keys[n] = rlc_cell_key{k.qx, k.qy, k.qz, k.qn, k.level};
      fill_cut(c, m, n, node_ids, ends, q, cdf, visits);
    }
    ++n;
  }
  return n;
}

void ref_run_template(void* h, uint32_t* node_ids, uint32_t* ends, double* q, double* cdf,
                      uint32_t* visits, double* eps_q) {
  RefRun* run = static_cast<RefRun*>(h);
  const Cut& c = run->grid->fallback_cut();
  fill_cut(c, c.size(), 0, node_ids, ends, q, cdf, visits);
  if (eps_q) *eps_q = c.eps_q;
}

// Scene BVH queries (bvh.cpp:124-188) on the run's context.
void ref_run_occluded(void* h, uint32_t n, const double* a, const double* b, uint8_t* out) {
  RefRun* run = static_cast<RefRun*>(h);
  for (uint32_t i = 0; i < n; ++i)
    out[i] = occluded(run->ctx.accel, {a[3 * i], a[3 * i + 1], a[3 * i + 2]},
                      {b[3 * i], b[3 * i + 1], b[3 * i + 2]});
}

void ref_run_intersect(void* h, uint32_t n, const double* org, const double* dir,
                       double t_min, double* t_out, int32_t* tri_out) {
  RefRun* run = static_cast<RefRun*>(h);
  for (uint32_t i = 0; i < n; ++i) {
    Ray r;
    r.origin = {org[3 * i], org[3 * i + 1], org[3 * i + 2]};
    r.dir = {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]};
    r.t_min = t_min;
    const auto hit = intersect(run->ctx.accel, r);
    t_out[i] = hit ? hit->t : -1.0;
    tri_out[i] = hit ? int32_t(hit->triangle_id) : -1;
  }
}

// The stock render_frame (render.cpp:202-240) -- the CPU baseline arm.
// stats: occupied, lookups, fallback_hits.  Returns wall_ms (< 0 on error).
// With `reference` ([h*w*3], the camera's size) pass_mse[passes] is filled.
double ref_render_frame(const rlc_scene_desc* desc, const rlc_render_config* config,
                        double* image, uint64_t* stats, uint32_t* sc_changes,
                        const double* reference, double* pass_mse) {
  try {
    Scene scene = to_scene(desc);
    const RenderConfig cfg = to_config(config);
    const RenderContext ctx = build_context(scene, cfg);
    Image ref_img;
    if (reference) ref_img = to_image(reference, desc->width, desc->height);
    const RenderResult res = render_frame(ctx, cfg, reference ? &ref_img : nullptr);
    if (pass_mse)
      for (size_t i = 0; i < res.pass_mse.size(); ++i) pass_mse[i] = res.pass_mse[i];
    if (image)
      for (size_t i = 0; i < res.image.pixels.size(); ++i) {
        image[3 * i] = res.image.pixels[i].x;
        image[3 * i + 1] = res.image.pixels[i].y;
        image[3 * i + 2] = res.image.pixels[i].z;
      }
    if (stats) {
      stats[0] = res.occupied_cells;
      stats[1] = res.lookups;
      stats[2] = res.fallback_hits;
    }
    if (sc_changes)
      for (size_t i = 0; i < res.sc_changes.size(); ++i) sc_changes[i] = res.sc_changes[i];
    return res.wall_ms;
  } catch (const std::exception& e) {
    fail(e);
    return -1.0;
  }
}

// ---- light tree / cut unit entry points (light_tree.cpp, cut.cpp) ----
// nodes_out: [2n-1][5] = range_begin, range_end, left, right, parent.
uint32_t ref_light_tree(uint32_t n, const double* centroids, const double* energies,
                        uint32_t* order_out, int32_t* nodes_out, double* energy_out) {
  try {
    const LightTree t = tree_from_points(n, centroids, energies);
    for (uint32_t i = 0; i < n; ++i) order_out[i] = t.order[i];
    for (size_t i = 0; i < t.nodes.size(); ++i) {
      nodes_out[5 * i] = int32_t(t.nodes[i].range_begin);
      nodes_out[5 * i + 1] = int32_t(t.nodes[i].range_end);
      nodes_out[5 * i + 2] = t.nodes[i].left;
      nodes_out[5 * i + 3] = t.nodes[i].right;
      nodes_out[5 * i + 4] = t.nodes[i].parent;
      energy_out[i] = t.nodes[i].energy;
    }
    return uint32_t(t.nodes.size());
  } catch (const std::exception& e) {
    fail(e);
    return 0;
  }
}

// init_cut (cut.cpp:27-74); returns the cut size, arrays sized >= min(M, n).
uint32_t ref_init_cut(uint32_t n, const double* centroids, const double* energies, uint32_t M,
                      double eps_q, uint32_t* node_ids, uint32_t* ends, double* q, double* cdf,
                      uint32_t* visits, double* eps_out) {
  try {
    const LightTree t = tree_from_points(n, centroids, energies);
    const Cut c = init_cut(t, M, eps_q);
    fill_cut(c, c.size(), 0, node_ids, ends, q, cdf, visits);
    if (eps_out) *eps_out = c.eps_q;
    return c.size();
  } catch (const std::exception& e) {
    fail(e);
    return 0;
  }
}

// split_collapse (cut.cpp:119-190) on an init_cut(tree, M) whose q (and
// optionally visits) are overwritten first; cut arrays are in/out [m].
// Returns the change count, or -status.
int64_t ref_split_collapse(uint32_t n, const double* centroids, const double* energies,
                           uint32_t M, double eps_q, const double* q_in,
                           const uint32_t* visits_in, double threshold, uint32_t iterations,
                           uint32_t* node_ids, uint32_t* ends, double* q, double* cdf,
                           uint32_t* visits) {
  try {
    const LightTree t = tree_from_points(n, centroids, energies);
    Cut c = init_cut(t, M, eps_q);
    for (uint32_t i = 0; i < c.size(); ++i) {
      c.q[i] = q_in[i];
      if (visits_in) c.visits[i] = visits_in[i];
    }
    rebuild_cdf(c);
    const uint32_t ch = split_collapse(c, t, threshold, iterations);
    fill_cut(c, c.size(), 0, node_ids, ends, q, cdf, visits);
    return ch;
  } catch (const std::exception& e) {
    return -int64_t(fail(e));
  }
}

// A sequence of update_q calls (cut.cpp:76-86) on one cut; q/visits in/out.
int ref_update_q_seq(uint32_t m, double* q, uint32_t* visits, double eps_q, double alpha,
                     uint32_t schedule, uint32_t count, const uint32_t* s, const double* v,
                     double* q_before) {
  try {
    Cut c;
    c.node_ids.assign(m, 0);
    c.q.assign(q, q + m);
    c.visits.assign(visits, visits + m);
    c.eps_q = eps_q;
    CutConfig cfg;
    cfg.alpha = alpha;
    cfg.alpha_schedule = AlphaSchedule(schedule);
    for (uint32_t i = 0; i < count; ++i) {
      if (q_before) q_before[i] = s[i] < m ? c.q[s[i]] : 0.0;
      update_q(c, s[i], v[i], cfg);
    }
    for (uint32_t j = 0; j < m; ++j) {
      q[j] = c.q[j];
      visits[j] = c.visits[j];
    }
    return RLC_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// sample_cluster (cut.cpp:97-106) on given q/cdf arrays.
void ref_sample_cluster(uint32_t m, const double* q, const double* cdf, uint32_t count,
                        const double* u, uint32_t* s_out, double* p_out) {
  Cut c;
  c.q.assign(q, q + m);
  c.cdf.assign(cdf, cdf + m);
  for (uint32_t i = 0; i < count; ++i) {
    const ClusterSample cs = sample_cluster(c, u[i]);
    s_out[i] = cs.index;
    p_out[i] = cs.p;
  }
}

// ---- hash-grid key functions (hash_grid.cpp:27-100) ----
int ref_level_for_footprint(uint32_t n, const double* area_pdf, double base_tile,
                            uint32_t* out) {
  try {
    for (uint32_t i = 0; i < n; ++i) out[i] = level_for_footprint(area_pdf[i], base_tile);
    return RLC_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_make_key(uint32_t n, const double* pos, const double* nrm, const uint32_t* level,
                 const double* ju1, const double* ju2, double base_tile, uint32_t normal_bits,
                 double jitter_scale, rlc_cell_key* out, uint64_t* hash_out) {
  try {
    HashConfig cfg;
    cfg.base_tile = base_tile;
    cfg.normal_bits = normal_bits;
    cfg.jitter_scale = jitter_scale;
    for (uint32_t i = 0; i < n; ++i) {
      const CellKey k = make_key({pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]},
                                 {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]}, level[i],
                                 ju1[i], ju2[i], cfg);
      out[i] = rlc_cell_key{k.qx, k.qy, k.qz, k.qn, k.level};
      if (hash_out) hash_out[i] = hash_key(k);
    }
    return RLC_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_octa_encode(uint32_t n, const double* nrm, double* uv) {
  for (uint32_t i = 0; i < n; ++i) {
    const Vec2 e = octa_encode({nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]});
    uv[2 * i] = e.x;
    uv[2 * i + 1] = e.y;
  }
}

// image module (image.cpp:43-136) through the reference's own functions
int ref_image_write_pfm(const double* px, int w, int h, const char* path) {
  try {
    write_pfm(to_image(px, w, h), path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_image_read_pfm(const char* path, double* px, uint64_t cap, int* w, int* h) {
  try {
    const Image im = read_pfm(path);
    *w = im.width;
    *h = im.height;
    if (px && cap >= im.pixels.size())
      for (size_t i = 0; i < im.pixels.size(); ++i) {
        px[3 * i] = im.pixels[i].x;
        px[3 * i + 1] = im.pixels[i].y;
        px[3 * i + 2] = im.pixels[i].z;
      }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_image_write_ppm(const double* px, int w, int h, const char* path) {
  try {
    write_ppm(to_image(px, w, h), path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_image_mse(const double* a, int wa, int ha, const double* b, int wb, int hb, int relative,
                  double* out) {
  try {
    const Image ia = to_image(a, wa, ha), ib = to_image(b, wb, hb);
    *out = relative ? relative_mse(ia, ib) : mse(ia, ib);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
