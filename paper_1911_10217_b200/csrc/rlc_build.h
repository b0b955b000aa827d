// rlc_build.h -- host-side, once-per-context construction of the structures
// the device path reads: the scene BVH in the reference topology, the
// Morton light tree, emitter records, material flags, camera constants, the
// template cut and the footprint-level thresholds.
#pragma once

#include <stdexcept>
#include <string>
#include <array>
#include <vector>

#include "rlc_common.h"
#include "rlcuts_b200.h"

namespace rlc {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct OutOfRange : std::out_of_range {
  using std::out_of_range::out_of_range;
};

constexpr uint32_t kMaxLevel = 16;  // proj/src/hash_grid.cpp:20

struct HostScene {
  // scene BVH (reference topology, bvh.cpp:64-122)
  std::vector<BvhNode> nodes;
  std::vector<BvhNodeF> nodes_f;  // same topology, fp32 outward-rounded boxes
  std::vector<BvhNodeF> nodes_cam; // same, boxes relative to the camera origin (fl64(c - O))
  std::vector<TriAccel> tris;  // BVH leaf order
  std::vector<Wide4> wide;       // 4-wide conservative tree, DFS order (empty: root is a leaf)
  std::vector<WideQ> wide_q;     // `wide` quantized to 64-byte nodes (RLC_SHADOW_QUANT=0: none)
  std::vector<Wide4> wide_ref;   // the reference tree collapsed, children left to right
  std::vector<Wide4> wide_cam;   // wide_ref with camera-relative boxes
  double coord_bound = 0;        // S: largest |coordinate| of the scene (shadow-tree padding)
  std::vector<uint32_t> tri_leaf; // binary leaf node per leaf-order triangle
  std::vector<double> mat_values; // the scene's materials [m*6] (albedo, emission)
  std::vector<TriAccel> tris_s;   // triangles in the shadow tree's leaf order
  std::vector<uint32_t> tri_leaf_s; // reference leaf node per tris_s entry
  std::vector<BvhNode> shadow_bin;  // binary SAH tree behind `wide` (leaves: tris_s ranges)
  // per `wide` node, the shadow_bin node behind each child (kWideEmpty: none),
  // and per shadow_bin node its tris_s range: a dynamic update recomputes the
  // wide boxes straight from the moved triangles
  std::vector<std::array<uint32_t, kWide>> wide_kids;
  std::vector<uint32_t> bin_first, bin_end;
  // shadow_bin nodes deepest level first, and each level's start in it (the
  // refit's bottom-up order); refit scratch reused from update to update
  std::vector<uint32_t> bin_order, bin_level_start;
  std::vector<double> refit_box;    // [6] per shadow_bin node
  std::vector<uint32_t> refit_leaf; // reference leaf per triangle id
  // dynamic update whose shadow tree is refitted on the device (the host
  // leaves tris_s / tri_leaf_s / wide / wide_q empty; refit_leaf is the input)
  bool gpu_refit = false;
  double scene_lo[3], scene_hi[3];
  double shadow_eps = 0;
  // materials / triangles
  std::vector<MatRec> mats;
  std::vector<uint32_t> tri_mat;  // by triangle id
  std::vector<double> tri_normal; // by triangle id, [3] (triangle_normal)
  // emitters + light tree (light_tree.cpp:30-119)
  std::vector<LightRec> lights;          // by emitter index
  std::vector<uint32_t> emitter_tri;     // emitter index -> triangle id
  std::vector<uint32_t> emitter_mat;     // emitter index -> material id
  std::vector<double> emitter_energy;    // luminance(emission) * area
  std::vector<double> emitter_centroid;  // [3] per emitter
  std::vector<uint32_t> order;           // sorted position -> emitter index
  std::vector<LtNode> lt_nodes;          // preorder ids, root 0
  std::vector<uint32_t> lt_begin;        // range_begin per node
  std::vector<double> lt_energy;
  std::vector<double> energy_cdf;        // estimators.cpp:12-26
  CameraConst cam;
  double base_tile = 0;                  // render.cpp:153-155
  double level_threshold[kMaxLevel + 1]; // see level_thresholds()
};

// Whole-context build (proj/src/render.cpp:143-157).  Throws InvalidArgument
// with the reference's messages for empty scenes / no emitters.
// With `keep` (rlc_context_update_scene / _prepare_scene: the context's
// creation scene, read only, so several updates can be built at once): the
// light tree, emitter list and the shadow tree's topology are those of
// `keep` (not copied into `out`: the device keeps them) and the shadow tree
// is refitted instead of rebuilt; the fp32 copies of the reference tree that
// only deferred closest-hit rays use are not built (the device then runs
// those rays on the fp64 reference tree).  `out` may be a scene recycled
// from an earlier update: its buffers are reused.
// The reference scene BVH alone (build_scene_bvh, bvh.cpp:64-122) into
// out.nodes / out.tris (diagnostics: rlc_debug_host_bvh times it).
void build_reference_bvh(const rlc_scene_desc& d, HostScene& out);
void build_host_scene(const rlc_scene_desc& desc, const rlc_render_config& cfg, HostScene& out,
                      const HostScene* keep = nullptr);

// memcpy on the host build's worker pool (1 MB chunks): moves large device
// downloads out of pinned staging at host memory bandwidth.
void parallel_copy(void* dst, const void* src, size_t bytes);

// Light tree alone over emitter centroids/energies (light_tree.cpp:56-119),
// exposed for the unit-level entry points.
void build_light_tree(const std::vector<double>& centroids, const std::vector<double>& energy,
                      std::vector<uint32_t>& order, std::vector<LtNode>& nodes,
                      std::vector<uint32_t>& node_begin, std::vector<double>& node_energy);

struct HostCut {
  std::vector<uint32_t> node_ids, ends, visits;
  std::vector<double> q, cdf;
  double eps_q = 0;
};
// init_cut (proj/src/cut.cpp:27-74).
HostCut make_template_cut(const std::vector<LtNode>& nodes, const std::vector<uint32_t>& begin,
                          const std::vector<double>& energy, uint32_t light_count, uint32_t M,
                          double eps_q);

// Smallest r with clamp(round(log2(r)), 0, 16) >= k for k = 1..16, found by
// bisection over the doubles with the host libm, so the device reproduces
// level_for_footprint (hash_grid.cpp:34-44) without its own log2.
void level_thresholds(double out[kMaxLevel + 1]);

// ---- image module (rlc_image.cpp; proj/src/image.cpp:43-136) -------------
// ImageIoError (image.hpp:15-28): code is RLC_ERR_IO or RLC_ERR_PARSE.
struct ImageIoError : std::runtime_error {
  ImageIoError(int code, const std::string& msg);
  int code() const { return code_; }

 private:
  int code_;
};
void write_pfm(const double* px, int32_t w, int32_t h, const std::string& path);
void read_pfm(const std::string& path, double* px, uint64_t cap_pixels, int32_t* w, int32_t* h);
void write_ppm(const double* px, int32_t w, int32_t h, const std::string& path);
double mse(const double* a, const double* b, uint64_t npix);
double relative_mse(const double* a, const double* b, uint64_t npix);
// mse's sequential sum over per-pixel terms computed elsewhere (device).
double sum_terms(const double* e, uint64_t n);

}  // namespace rlc
