// rlcuts_b200_shim.hpp -- the binding a reference maintainer adds to
// proj/include/rlcuts/ to run the per-frame direct-lighting step on a B200.
// Same types and signatures as proj/include/rlcuts/render.hpp:39-69, in
// namespace rlcuts::b200; implemented over the C-ABI in
// include/rlcuts_b200.h (link with -lrlcuts_b200).
#pragma once

#include <cstdint>
#include <memory>
#include <ostream>
#include <vector>

#include "rlcuts/hash_grid.hpp"
#include "rlcuts/image.hpp"
#include "rlcuts/render.hpp"

namespace rlcuts::b200 {

// render_frame (proj/src/render.cpp:202-240): same arguments, same result
// fields (image, wall_ms, occupied_cells, lookups, fallback_hits, pass_mse,
// sc_changes).  Throws std::invalid_argument / std::out_of_range like the
// reference, std::runtime_error for device failures.
RenderResult render_frame(const RenderContext& ctx, const RenderConfig& config,
                          const Image* reference = nullptr);

// The pass-level loop of render_frame for callers that drive passes
// themselves (render_pass + end_of_pass_update, render.cpp:159-200).  The
// learned state and the accumulation buffer stay on the device; framebuffer()
// downloads the running sums into a host Framebuffer.
class Session {
 public:
  Session(const RenderContext& ctx, const RenderConfig& config, int device = 0);
  ~Session();
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  void render_pass(uint32_t pass_index);   // render_pass
  uint32_t end_of_pass_update();           // end_of_pass_update
  // Dynamic emitters (rlc_context_update_scene): render `scene` from now on
  // as build_context(scene) would, keeping the light tree of the session's
  // creation so the learned cuts stay valid.  Same triangles and materials.
  void update_scene(const Scene& scene);
  void framebuffer(Framebuffer& out) const;
  uint32_t occupied_count() const;
  uint64_t lookup_count() const;
  uint64_t fallback_hits() const;
  // HashGrid's host accessors (hash_grid.hpp:87-110) over the device grid:
  // key_of / touched_slots index the device table's slots (positions can
  // differ from a CPU grid's, whose insertion order differs under probing).
  CellKey key_of(uint32_t slot) const;
  std::vector<uint32_t> touched_slots() const;
  uint64_t memory_records() const;
  void dump_stats(std::ostream& out) const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace rlcuts::b200
