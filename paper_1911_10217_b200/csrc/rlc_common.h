// rlc_common.h -- FP64 vector math, counter RNG and plain-data layouts shared
// by the host build code (g++, -ffp-contract=off) and the sm_100a kernels
// (nvcc --fmad=false).  Every expression keeps the operand order of the
// reference so that host-precomputed and device-computed values are
// bit-identical to the reference's doubles (contraction
// into FMA changes cell keys).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define RLC_HD __host__ __device__ __forceinline__
#else
#define RLC_HD inline
#include <cmath>
#endif

namespace rlc {

constexpr double kPi = 3.14159265358979323846;  // proj/include/rlcuts/math.hpp:12

// ---- Vec3: proj/include/rlcuts/math.hpp:15-53 ----------------------------
struct V3 {
  double x, y, z;
};
RLC_HD V3 v3(double x, double y, double z) { return V3{x, y, z}; }
RLC_HD V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
RLC_HD V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
RLC_HD V3 operator-(V3 a) { return V3{-a.x, -a.y, -a.z}; }
RLC_HD V3 operator*(V3 a, V3 b) { return V3{a.x * b.x, a.y * b.y, a.z * b.z}; }
RLC_HD V3 operator*(V3 a, double s) { return V3{a.x * s, a.y * s, a.z * s}; }
RLC_HD V3 operator/(V3 a, double s) { return V3{a.x / s, a.y / s, a.z / s}; }
RLC_HD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
RLC_HD V3 cross(V3 a, V3 b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
RLC_HD double length(V3 v) { return sqrt(dot(v, v)); }
RLC_HD V3 normalize(V3 v) { return v / length(v); }
// std::min / std::max argument semantics: min(a,b) = (b < a) ? b : a,
// max(a,b) = (a < b) ? b : a (NaN handling follows from that).
RLC_HD double smin(double a, double b) { return (b < a) ? b : a; }
RLC_HD double smax(double a, double b) { return (a < b) ? b : a; }
RLC_HD double clampd(double v, double lo, double hi) {  // std::clamp
  return v < lo ? lo : (hi < v ? hi : v);
}
// Rec.709 luminance, math.hpp:56
RLC_HD double luminance(V3 c) { return 0.2126 * c.x + 0.7152 * c.y + 0.0722 * c.z; }

// ---- counter RNG: proj/include/rlcuts/rng.hpp:12-43 -----------------------
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
RLC_HD uint64_t mix64(uint64_t x) {
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
RLC_HD uint64_t hash_combine(uint64_t a, uint64_t b) { return mix64(a ^ mix64(b)); }
RLC_HD double to_unit(uint64_t bits) { return double(bits >> 11) * 0x1.0p-53; }
// RandomSequence(seed, a, b, c).key_ with mix64(seed) precomputed.
RLC_HD uint64_t rng_key(uint64_t seed_mixed, uint64_t a, uint64_t b, uint64_t c_mixed) {
  uint64_t k = hash_combine(seed_mixed, a);
  k = hash_combine(k, b);
  return mix64(k ^ c_mixed);  // hash_combine(k, c) with c_mixed = mix64(c)
}
// The d-th draw (d = 1, 2, ...) of the sequence: rng.hpp:37.
RLC_HD double rng_draw(uint64_t key, uint64_t d) { return to_unit(mix64(key + kGolden * d)); }

// Draw indices of one depth-1 path (proj/src/render.cpp:65-66, 90-95).
enum : uint32_t { kDrawJx = 1, kDrawJy = 2, kDrawU1 = 3, kDrawU2 = 4, kDrawU3 = 5,
                  kDrawJu1 = 6, kDrawJu2 = 7 };

// ---- plain-data device layouts ------------------------------------------
// Scene BVH node, reference topology (proj/include/rlcuts/bvh.hpp:16-22),
// 64 B so one node is four 16-byte loads.
struct alignas(64) BvhNode {
  double lo[3];
  double hi[3];
  uint32_t a;      // internal: left child; leaf: first index into the tri arrays
  uint32_t b;      // internal: right child
  uint32_t count;  // 0 for internal nodes
  uint32_t pad;
};

// The same binary node with its box rounded outward to fp32 for the
// closest-hit traversal's fp32 decision tests (exact fp64 only in the rare
// ambiguous band).  32 B: two siblings share one 64-byte line.
constexpr uint32_t kNodeLeaf = 0x80000000u;
struct alignas(32) BvhNodeF {
  float lo[3];
  float hi[3];
  uint32_t a;  // internal: left child (right = a + 1); leaf: kNodeLeaf | first tri
  uint32_t b;  // leaf: triangle count
};

// 4-wide node collapsed from the reference binary BVH for the any-hit shadow
// kernel.  Child boxes are the binary nodes' boxes rounded OUTWARD to fp32,
// so the fp64 slab test on them passes whenever the reference's test on the
// exact box passes (rounding is monotone); a triangle hit found through this
// tree is accepted only after its binary ancestor chain passes the exact
// fp64 test ("Exact any-hit on a conservative wide BVH").
constexpr uint32_t kWideLeaf = 0x80000000u;  // child: leaf flag
constexpr uint32_t kWideEmpty = 0xffffffffu; // child: unused slot
constexpr uint32_t kLeafPure = 0x08000000u;  // leaf: all triangles in one reference leaf
#ifndef RLC_WIDE
#define RLC_WIDE 4
#endif
constexpr int kWide = RLC_WIDE;  // children per node (4 or 8)
struct alignas(128) Wide4 {
  float lo[3][kWide];  // [axis][child]
  float hi[3][kWide];
  uint32_t child[kWide];  // internal: node index; leaf: kWideLeaf | (count - 1) << 28 |
                          // kLeafPure? | first tri (27 bits)
  uint32_t pad[kWide == 8 ? 8 : 4];
};
static_assert(sizeof(Wide4) % 128 == 0, "wide nodes are whole 128-byte lines");

// The shadow tree's 4-wide node quantized to 64 bytes: child box planes are
// origin + q * 2^(e - 127) per axis (q 8-bit).  The host chooses every q so
// the plane lies OUTSIDE the Wide4 node's (already outward-rounded, padded)
// fp32 bound, so a quantized box contains the exact one; k_shadow evaluates
// t = fma(q, 2^e inv, fma(origin, inv, -o inv)) per plane.
struct alignas(64) WideQ {
  float origin[3];
  uint8_t ex[3];          // per-axis scale exponent: scale = 2^(ex - 127)
  uint8_t pad0;
  uint8_t qlo[3][4];      // [axis][child]
  uint8_t qhi[3][4];
  uint32_t child[4];      // as Wide4::child
  uint32_t valid;         // bit c: child[c] is not kWideEmpty
  uint32_t pad1;
};
static_assert(sizeof(WideQ) == 64, "quantized wide nodes are 64 bytes");

// Triangle as the Moller-Trumbore test consumes it (bvh.cpp:44-62): p0 and
// the two edges, precomputed with the reference's own subtraction.  Stored
// in BVH leaf order.  80 B.
struct alignas(16) TriAccel {
  double p0[3];
  double e1[3];
  double e2[3];
  uint32_t tri_id;
  uint32_t pad;
};

// Emitter in reference emitter order (light_tree.cpp:30-42): everything
// sample_triangle_point (scene.cpp:49-59) and nee_estimate
// (estimators.cpp:82-106) read.  128 B, one line.
struct alignas(128) LightRec {
  double p0[3], p1[3], p2[3];
  double n[3];         // triangle_normal (scene.hpp:27)
  double emission[3];  // material emission
  double pdf_area;     // 1 / triangle_area
};

// An emitter at its light-tree position (tree.order[pos], light_tree.hpp):
// the learned sampler's pick reads one record instead of order[] then the
// LightRec.  Built on the device from LightRec and order (k_light_order).
// 80 B, three 32-byte sectors per random pick: the normal and 1 / area are
// recomputed from the vertices with the expressions that built LightRec
// (rlc_build.cpp, emitter()), so they are the same doubles.
struct alignas(16) LightOrd {
  double p0[3], p1[3], p2[3];
  uint32_t mat;      // material (emission)
  uint32_t emitter;  // emitter index (tree.order[pos])
};

// Material flags precomputed with the reference predicates.
struct alignas(16) MatRec {
  double albedo[3];
  double emission[3];
  uint32_t is_emitter;  // luminance(emission) > 0   (scene.hpp:17)
  uint32_t reflective;  // luminance(albedo) > 0     (render.cpp:84)
};

// Light-tree node as split-collapse reads it (light_tree.hpp:29-36).
struct alignas(16) LtNode {
  uint32_t range_end;
  int32_t left;
  int32_t right;
  int32_t parent;
};

// Camera constants precomputed on the host exactly as camera_ray
// (proj/src/scene.cpp:10-23) and pixel_solid_angle (:25-31) do.
struct CameraConst {
  double origin[3];
  double u[3], v[3], w[3];
  double tan_half, aspect;
  double width_d, height_d;
  double pdf_omega;  // 1 / pixel_solid_angle
  int32_t width, height;
};

}  // namespace rlc
