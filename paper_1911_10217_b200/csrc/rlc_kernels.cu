// rlc_kernels.cu -- sm_100a kernels of the per-pass RL-lightcuts path.
//
// Per pass (render_pass + end_of_pass_update, proj/src/render.cpp:159-200):
//   k_primary      camera ray, closest hit, shading point, footprint level,
//                  5-D cell key and hash-grid lookup (find only)  (one thread/path)
//   k_insert,      the pass's new keys into the table in canonical order,
//   k_commit       published with template cuts
//   k_sample       cut sampling from the pass-frozen cdf, emitter point,
//                  NEE geometry, shadow segment, feedback v, the ray
//                  compaction's tile counts                       (one thread/vertex)
//   k_cmp_scatter  stable compaction of the shadow segments
//   k_shadow       any-hit traversal of the segments (persistent warps)
//   radix sort     stable, update records by (cell, cluster)      (beside k_shadow)
//   k_fold         sequential update_q per (cell, cluster) segment in canonical
//                  order -> live q, visits and per-sample q_before
//   k_accumulate   deferred radiance with q_before, Framebuffer::add_sample
//   k_split        split-collapse + ends per touched cell (one warp/cell),
//                  then the serial cdf (one lane/cell)
// Sharded passes add k_write_block, k_classify, k_resolve_pending, k_apply /
// k_apply_entries and k_shard_scatter.
//
// All FP64 arithmetic keeps the reference's operand order and this file is
// compiled with --fmad=false: the path is bit-exact with the reference
// (SURVEY 0 facts 1-6 and Appendix B give the argument).
#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "rlc_kernels.h"
#include "rlc_libm.h"
#include "rlc_sincostab.h"

namespace rlc {

namespace {
std::atomic<uint64_t> g_launches{0};
inline void count_launch(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
constexpr unsigned kFull = 0xffffffffu;
}  // namespace

uint64_t launches() { return g_launches.load(); }
void add_launches(uint64_t k) { count_launch(k); }

// Opt-in traversal statistics (build with EXTRA=-DRLC_TRAV_STATS): per-ray
// node steps and triangle tests of k_shadow [0..2] and closest_sah [3..5]
// (rays, nodes, triangles).  Diagnostics only; zero in the product build.
__device__ unsigned long long g_trav[8];
#ifdef RLC_TRAV_STATS
#define RLC_STAT(i, v) atomicAdd(&g_trav[i], (unsigned long long)(v))
#else
#define RLC_STAT(i, v) ((void)0)
#endif
// Work counters of the dominant kernel (the roofline's own-work bytes,
// bench.py), kept while a context counts (rlc_context_count_work):
// k_shadow's rays traversed by the tree, node steps and triangle tests,
// summed per lane in registers and added once per warp, and the rays queued
// for it.
__device__ unsigned long long g_work[4];
void work_counters(uint64_t out[4], bool reset) {
  cudaMemcpyFromSymbol(out, g_work, sizeof(uint64_t) * 4);
  if (reset) {
    const unsigned long long z[4] = {};
    cudaMemcpyToSymbol(g_work, z, sizeof(z));
  }
}

// L2 read bandwidth probe (the bench's second roofline denominator): every
// block streams the whole L2-resident buffer with 16-byte L2 loads (.cg, no
// L1), `reps` times.
__global__ void __launch_bounds__(256) k_l2_probe(const uint4* __restrict__ buf, size_t n16,
                                                  uint32_t reps, uint32_t* __restrict__ sink) {
  uint32_t acc = 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (uint32_t r = 0; r < reps; ++r)
    for (size_t i = (size_t(blockIdx.x) * blockDim.x + threadIdx.x + r * 4099u) % n16, k = 0;
         k < (n16 + stride - 1) / stride; ++k, i = (i + stride) % n16) {
      const uint4 v = __ldcg(buf + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x9e3779b9u) *sink = acc;  // keeps the loads
}

double measure_l2_gbs(size_t bytes, uint32_t reps) {
  uint4* buf = nullptr;
  uint32_t* sink = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess) return 0;
  cudaMemset(buf, 1, bytes);
  const size_t n16 = bytes / 16;
  const uint32_t blocks = 148 * 8;
  k_l2_probe<<<blocks, 256>>>(buf, n16, 1, sink);  // warm: the buffer into L2
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_l2_probe<<<blocks, 256>>>(buf, n16, reps, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const size_t stride = size_t(blocks) * 256;
  const double moved = double(reps) * double((n16 + stride - 1) / stride) * double(stride) * 16.0;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(sink);
  count_launch(2);
  return ms > 0 ? moved / (ms * 1e-3) / 1e9 : 0;
}

void trav_stats(uint64_t out[8], bool reset) {
  cudaMemcpyFromSymbol(out, g_trav, sizeof(uint64_t) * 8);
  if (reset) {
    const unsigned long long z[8] = {};
    cudaMemcpyToSymbol(g_trav, z, sizeof(z));
  }
}

static inline uint32_t blocks_for(uint32_t n, uint32_t t) { return (n + t - 1) / t; }

// Debug build (EXTRA=-DRLC_DEBUG_CHECKS): device bounds checks on the
// indices the hash grid, cut sampling, shadow queue and fold compute; a
// failure raises kErrCheck, reported by the host as an exception.  (The
// pool's compute-sanitizer is closed; tests/run_checked.sh runs the GPU
// suite against this build.)
#ifdef RLC_DEBUG_CHECKS
#define RLC_CHECK(cond, errp)                                                 \
  do {                                                                        \
    if (!(cond)) atomicOr(reinterpret_cast<unsigned int*>(errp), kErrCheck); \
  } while (0)
#else
#define RLC_CHECK(cond, errp) ((void)0)
#endif

// ---------------------------------------------------------------------------
// geometry helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ V3 ld3(const double* p) { return V3{p[0], p[1], p[2]}; }

// A 16-byte-aligned record of read-only data in 128-bit loads (scattered
// records cost one L1 wavefront per load instruction and lane).
template <typename T>
__device__ __forceinline__ T ldg_vec(const T* p) {
  static_assert(sizeof(T) % 16 == 0 && alignof(T) >= 16, "16-byte records");
  union {
    T t;
    double2 d[sizeof(T) / 16];
  } u;
  const double2* s = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int i = 0; i < int(sizeof(T) / 16); ++i) u.d[i] = __ldg(s + i);
  return u.t;
}

struct NodeView {
  double lo0, lo1, lo2, hi0, hi1, hi2;
  uint32_t a, b, count;
};

__device__ __forceinline__ NodeView load_node(const BvhNode* nodes, uint32_t i) {
  const double2* p = reinterpret_cast<const double2*>(nodes + i);
  const double2 x = __ldg(p), y = __ldg(p + 1), z = __ldg(p + 2);
  const uint4 w = __ldg(reinterpret_cast<const uint4*>(nodes + i) + 3);
  return NodeView{x.x, x.y, y.x, y.y, z.x, z.y, w.x, w.y, w.z};
}

// intersect_aabb, proj/src/bvh.cpp:29-40 (std::max/std::min semantics).
__device__ __forceinline__ bool slab(double lo, double hi, double o, double inv, double& tmin,
                                     double& tmax) {
  double t0 = (lo - o) * inv;
  double t1 = (hi - o) * inv;
  if (inv < 0) {
    const double t = t0;
    t0 = t1;
    t1 = t;
  }
  tmin = smax(tmin, t0);
  tmax = smin(tmax, t1);
  return !(tmax < tmin);
}

__device__ __forceinline__ bool box_hit(const NodeView& n, V3 o, V3 inv, double tmin,
                                        double tmax) {
  if (!slab(n.lo0, n.hi0, o.x, inv.x, tmin, tmax)) return false;
  if (!slab(n.lo1, n.hi1, o.y, inv.y, tmin, tmax)) return false;
  return slab(n.lo2, n.hi2, o.z, inv.z, tmin, tmax);
}

// Moller-Trumbore, proj/src/bvh.cpp:44-62.
__device__ __forceinline__ bool tri_hit(const TriAccel* tris, uint32_t i, V3 o, V3 d,
                                        double tmin, double tmax, double* tout) {
  const double2* p = reinterpret_cast<const double2*>(tris + i);
  const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), e = __ldg(p + 3),
                f = __ldg(p + 4);
  const V3 p0{a.x, a.y, b.x};
  const V3 e1{b.y, c.x, c.y};
  const V3 e2{e.x, e.y, f.x};
  const V3 pv = cross(d, e2);
  const double det = dot(e1, pv);
  if (fabs(det) < 1e-14) return false;
  const double inv_det = 1.0 / det;
  const V3 tv = o - p0;
  const double u = dot(tv, pv) * inv_det;
  if (u < 0 || u > 1) return false;
  const V3 qv = cross(tv, e1);
  const double v = dot(d, qv) * inv_det;
  if (v < 0 || u + v > 1) return false;
  const double t = dot(e2, qv) * inv_det;
  if (t <= tmin || t >= tmax) return false;
  *tout = t;
  return true;
}

constexpr int kStack = 64;  // bvh.cpp:134 uses a 64-entry stack too

// occluded(), proj/src/bvh.cpp:159-188.  The any-hit boolean does not depend
// on traversal order, so any order over the same tree and slab test gives
// the reference's answer.
__device__ __noinline__ bool occluded_ray(const DevScene& sc, V3 a, V3 dir, V3 inv, double tmin, double tmax,
                             uint32_t* err) {
  uint32_t stack[kStack];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    const NodeView n = load_node(sc.nodes, stack[--sp]);
    if (!box_hit(n, a, inv, tmin, tmax)) continue;
    if (n.count > 0) {
      for (uint32_t i = n.a; i < n.a + n.count; ++i) {
        double t;
        if (tri_hit(sc.tris, i, a, dir, tmin, tmax, &t)) return true;
      }
    } else {
      if (sp + 2 > kStack) {
        atomicOr(err, kErrStackOverflow);
        return false;
      }
      stack[sp++] = n.a;
      stack[sp++] = n.b;
    }
  }
  return false;
}


// fp32 decision test of one binary node against the reference's fp64 slab
// test (bvh.cpp:29-40), both sides bounded:
//   outer: box rounded outward and the interval widened by the rounding
//          bound -> if it fails, the reference test fails;
//   inner: the interval narrowed by the rounding bound plus the box rounding
//          (|c| |inv| 2^-22) -> if it passes, the reference test passes.
// Returns 0 (fail), 1 (pass) or 2 (ambiguous: run the exact fp64 test).  The
// inner test is only used when every |inv| is finite and <= 1e30 (ray.fast),
// where no fp32 term can be NaN or overflow.
struct RayDecide {
  float inv[3], b[3], mt[3], mb[3];
  uint32_t neg;
  bool fast;
};

__device__ __forceinline__ RayDecide make_ray_decide(V3 o, V3 inv) {
  RayDecide r;
  const double oa[3] = {o.x, o.y, o.z}, ia[3] = {inv.x, inv.y, inv.z};
  r.neg = 0;
  r.fast = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float of = float(oa[a]), fi = float(ia[a]);
    r.inv[a] = fi;
    r.b[a] = -(of * fi);
    r.mt[a] = fmaf(fabsf(of) * fabsf(fi), 0x1.0p-21f, 1e-30f);
    r.mb[a] = fabsf(fi) * 0x1.0p-22f;
    r.neg |= (ia[a] < 0 ? 1u : 0u) << a;
    r.fast &= fabs(ia[a]) <= 1e30;
  }
  return r;
}

__device__ __forceinline__ int box_decide(const float4& q0, const float4& q1, const RayDecide& r,
                                          float tmin_dn, float tmin_up, float tmax_dn,
                                          float tmax_up) {
  constexpr float K = 0x1.0p-20f;
  const float lo[3] = {q0.x, q0.y, q0.z}, hi[3] = {q0.w, q1.x, q1.y};
  float no = tmin_dn, fo = tmax_up, ni = tmin_up, fi = tmax_dn;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool neg = (r.neg >> a) & 1u;
    const float nc = neg ? hi[a] : lo[a];
    const float fc = neg ? lo[a] : hi[a];
    const float tn = fmaf(nc, r.inv[a], r.b[a]);
    const float tf = fmaf(fc, r.inv[a], r.b[a]);
    const float en = fmaf(fabsf(tn), K, r.mt[a]);
    const float ef = fmaf(fabsf(tf), K, r.mt[a]);
    no = fmaxf(no, tn - en);
    fo = fminf(fo, tf + ef);
    ni = fmaxf(ni, tn + en + fmaf(fabsf(nc), r.mb[a], 1e-37f));
    fi = fminf(fi, tf - ef - fmaf(fabsf(fc), r.mb[a], 1e-37f));
  }
  // reject only when certain: NaN terms (a NaN closest after a NaN-direction
  // "hit", which the reference's !(tmax < tmin) keeps) go to the exact test
  if (no > fo) return 0;
  if (r.fast && ni <= fi) return 1;
  return 2;
}

// Closest hit through the collapsed reference tree (defined with the wide
// traversal helpers below); false in *used when the ray needs the binary path.
// RLC_COLD_NOINLINE=1 moves it out of line (the rare path after the SAH
// closest hit); measured slower: the call spills more registers.
#ifndef RLC_COLD_NOINLINE
#define RLC_COLD_NOINLINE 0  // measured: noinline spills more and is 8% slower on c3
#endif
#if RLC_COLD_NOINLINE
#define RLC_COLD __noinline__
#else
#define RLC_COLD
#endif
__device__ RLC_COLD bool intersect_wide(const DevScene& sc, V3 o, V3 d, double tmin, bool camera,
                               bool* used, double* t_out, uint32_t* tri_out, uint32_t* err);

// Closest hit on the quantized SAH tree (defined below): 0 miss, 1 hit,
// 2 undecided (the caller runs the reference-order traversal).
__device__ int closest_sah(const DevScene& sc, V3 o, V3 d, double tmin, double* t_out,
                           uint32_t* tri_out);

// intersect() exactly as the reference runs it (bvh.cpp:124-157): binary
// tree, fp64 slab tests, right child first.  The path of last resort for
// deferred rays when the context carries no fp32 copies of the reference
// tree (dynamic scene updates build none).
__device__ __noinline__ bool intersect_exact(const DevScene& sc, V3 o, V3 d, double tmin,
                                             double* t_out, uint32_t* tri_out, uint32_t* err) {
  const V3 inv{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
  double closest = HUGE_VAL;
  uint32_t hit = kNoSlot;
  uint32_t stack[kStack];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    const NodeView n = load_node(sc.nodes, stack[--sp]);
    if (!box_hit(n, o, inv, tmin, closest)) continue;
    if (n.count > 0) {
      for (uint32_t k = n.a; k < n.a + n.count; ++k) {
        double t;
        if (tri_hit(sc.tris, k, o, d, tmin, closest, &t)) {
          closest = t;
          hit = k;
        }
      }
    } else {
      if (sp + 2 > kStack) {
        atomicOr(err, kErrStackOverflow);
        break;
      }
      stack[sp++] = n.a;
      stack[sp++] = n.b;
    }
  }
  if (hit == kNoSlot) return false;
  *t_out = closest;
  *tri_out = sc.tris[hit].tri_id;
  return true;
}

// intersect(), proj/src/bvh.cpp:124-157: closest hit in the reference's
// traversal order (pop the right child first), so exact-t ties go to the same
// triangle.  Every box decision equals the reference's (box_decide, exact
// fp64 test in the ambiguous band); triangle tests are the exact fp64
// Moller-Trumbore.
__device__ bool intersect(const DevScene& sc, V3 o, V3 d, double tmin, double* t_out,
                          uint32_t* tri_out, uint32_t* err) {
  const int sah = closest_sah(sc, o, d, tmin, t_out, tri_out);
  if (sah != 2) return sah == 1;
  bool used;
  const bool got = intersect_wide(sc, o, d, tmin, false, &used, t_out, tri_out, err);
  if (used) return got;
  if (sc.nodes_f == nullptr) return intersect_exact(sc, o, d, tmin, t_out, tri_out, err);
  const V3 inv{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
  const RayDecide rd = make_ray_decide(o, inv);
  const float tmin_dn = __double2float_rd(tmin), tmin_up = __double2float_ru(tmin);
  double closest = HUGE_VAL;
  float tmax_dn = HUGE_VALF, tmax_up = HUGE_VALF;
  uint32_t hit = kNoSlot;
  uint32_t stack[kStack];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    const uint32_t i = stack[--sp];
    const float4* np = reinterpret_cast<const float4*>(sc.nodes_f + i);
    const float4 q0 = __ldg(np), q1 = __ldg(np + 1);
    int dcs = box_decide(q0, q1, rd, tmin_dn, tmin_up, tmax_dn, tmax_up);
    if (dcs == 2) dcs = box_hit(load_node(sc.nodes, i), o, inv, tmin, closest) ? 1 : 0;
    if (dcs == 0) continue;
    const uint32_t a = __float_as_uint(q1.z), cnt = __float_as_uint(q1.w);
    if (a & kNodeLeaf) {
      const uint32_t first = a & ~kNodeLeaf;
      for (uint32_t k = first; k < first + cnt; ++k) {
        double t;
        if (tri_hit(sc.tris, k, o, d, tmin, closest, &t)) {
          closest = t;
          hit = k;
          tmax_dn = __double2float_rd(closest);
          tmax_up = __double2float_ru(closest);
        }
      }
    } else {
      if (sp + 2 > kStack) {
        atomicOr(err, kErrStackOverflow);
        break;
      }
      stack[sp++] = a;      // left
      stack[sp++] = a + 1;  // right, popped first (bvh.cpp:147-148)
    }
  }
  if (hit == kNoSlot) return false;
  *t_out = closest;
  *tri_out = sc.tris[hit].tri_id;
  return true;
}

// Camera rays: origin == the camera origin O, so the node boxes can be
// stored as fp32(fl64(c - O)) rounded outward (nodes_cam) and every error of
// the fp32 decision test is relative to the per-axis t (inverse and product
// rounding, box rounding, the reference's own fp64 rounding: < 4 u32 in
// total; K = 8 u32).  Same three outcomes as box_decide; the 1e-30 slack
// covers underflow.
__device__ __forceinline__ int box_decide_cam(const float4& q0, const float4& q1,
                                              const float inv[3], uint32_t neg, bool fast,
                                              float tmin_dn, float tmin_up, float tmax_dn,
                                              float tmax_up) {
  constexpr float K = 0x1.0p-21f;
  const float lo[3] = {q0.x, q0.y, q0.z}, hi[3] = {q0.w, q1.x, q1.y};
  float no = tmin_dn, fo = tmax_up, ni = tmin_up, fi = tmax_dn;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool ng = (neg >> a) & 1u;
    const float tn = (ng ? hi[a] : lo[a]) * inv[a];
    const float tf = (ng ? lo[a] : hi[a]) * inv[a];
    no = fmaxf(no, fmaf(fabsf(tn), -K, tn));
    ni = fmaxf(ni, fmaf(fabsf(tn), K, tn));
    fo = fminf(fo, fmaf(fabsf(tf), K, tf));
    fi = fminf(fi, fmaf(fabsf(tf), -K, tf));
  }
  if (no > fo + 1e-30f) return 0;  // NaN: the exact test decides
  if (fast && ni + 1e-30f <= fi) return 1;
  return 2;
}

// intersect() for camera rays: the reference order and decisions, with the
// camera-relative decision test.
__device__ bool intersect_camera(const DevScene& sc, V3 o, V3 d, double* t_out,
                                 uint32_t* tri_out, uint32_t* err) {
  const int sah = closest_sah(sc, o, d, 0.0, t_out, tri_out);
  if (sah != 2) return sah == 1;
  bool used;
  const bool got = intersect_wide(sc, o, d, 0.0, true, &used, t_out, tri_out, err);
  if (used) return got;
  if (sc.nodes_cam == nullptr) return intersect_exact(sc, o, d, 0.0, t_out, tri_out, err);
  const V3 inv{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
  const double ia[3] = {inv.x, inv.y, inv.z};
  float finv[3];
  uint32_t neg = 0;
  bool fast = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    finv[a] = float(ia[a]);
    neg |= (ia[a] < 0 ? 1u : 0u) << a;
    fast &= fabs(ia[a]) <= 1e30;
  }
  const double tmin = 0.0;
  double closest = HUGE_VAL;
  float tmax_dn = HUGE_VALF, tmax_up = HUGE_VALF;
  uint32_t hit = kNoSlot;
  uint32_t stack[kStack];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    const uint32_t i = stack[--sp];
    const float4* np = reinterpret_cast<const float4*>(sc.nodes_cam + i);
    const float4 q0 = __ldg(np), q1 = __ldg(np + 1);
    int dcs = box_decide_cam(q0, q1, finv, neg, fast, 0.f, 0.f, tmax_dn, tmax_up);
    if (dcs == 2) dcs = box_hit(load_node(sc.nodes, i), o, inv, tmin, closest) ? 1 : 0;
    if (dcs == 0) continue;
    const uint32_t a = __float_as_uint(q1.z), cnt = __float_as_uint(q1.w);
    if (a & kNodeLeaf) {
      const uint32_t first = a & ~kNodeLeaf;
      for (uint32_t k = first; k < first + cnt; ++k) {
        double t;
        if (tri_hit(sc.tris, k, o, d, tmin, closest, &t)) {
          closest = t;
          hit = k;
          tmax_dn = __double2float_rd(closest);
          tmax_up = __double2float_ru(closest);
        }
      }
    } else {
      if (sp + 2 > kStack) {
        atomicOr(err, kErrStackOverflow);
        break;
      }
      stack[sp++] = a;      // left
      stack[sp++] = a + 1;  // right, popped first (bvh.cpp:147-148)
    }
  }
  if (hit == kNoSlot) return false;
  *t_out = closest;
  *tri_out = sc.tris[hit].tri_id;
  return true;
}

// ---------------------------------------------------------------------------
// hash-grid key (proj/src/hash_grid.cpp:27-100)
// ---------------------------------------------------------------------------
struct Key {
  int32_t qx, qy, qz;
  uint32_t qn, level;
};

__device__ __forceinline__ double sign_nz(double v) { return v >= 0 ? 1.0 : -1.0; }

__device__ __forceinline__ Key make_key(V3 p, V3 n, uint32_t level, double ju1, double ju2,
                                        double base_tile, uint32_t bits, double js) {
  const double cell = base_tile * ldexp(1.0, int(level));  // base_tile * exp2(level), exact
  const double offset = js * cell * (ju1 - 0.5);
  Key k;
  k.qx = int32_t(floor((p.x + offset) / cell));
  k.qy = int32_t(floor((p.y + offset) / cell));
  k.qz = int32_t(floor((p.z + offset) / cell));
  k.level = level;
  const uint32_t steps = 1u << bits;
  const double quantum = 1.0 / double(steps);
  const double noffset = js * quantum * (ju2 - 0.5);
  // octa_encode, hash_grid.cpp:50-61
  const double norm = fabs(n.x) + fabs(n.y) + fabs(n.z);
  double ox = n.x / norm;
  double oy = n.y / norm;
  if (n.z < 0) {
    const double tx = (1.0 - fabs(oy)) * sign_nz(ox);
    const double ty = (1.0 - fabs(ox)) * sign_nz(oy);
    ox = tx;
    oy = ty;
  }
  const double eu = ox * 0.5 + 0.5;
  const double ev = oy * 0.5 + 0.5;
  const double top = double(steps - 1);
  const uint32_t qu = uint32_t(clampd(floor((eu + noffset) * double(steps)), 0.0, top));
  const uint32_t qv = uint32_t(clampd(floor((ev + noffset) * double(steps)), 0.0, top));
  k.qn = (qu << bits) | qv;
  return k;
}

__device__ __forceinline__ uint64_t hash_key(const Key& k) {
  const uint64_t w0 = (uint64_t(uint32_t(k.qx)) << 32) | uint64_t(uint32_t(k.qy));
  const uint64_t w1 = (uint64_t(uint32_t(k.qz)) << 32) | (uint64_t(k.qn & 0xffffu) << 16) |
                      uint64_t(k.level & 0xffffu);
  return hash_combine(mix64(w0), w1);
}

// Packed 128-bit slot word: lo = qx | qy << 32, hi = qz | qn << 32 (26 bits)
// | level << 58 (5 bits) | valid << 63.  An all-zero word is an empty slot.
__device__ __forceinline__ void pack_key(const Key& k, uint64_t& lo, uint64_t& hi) {
  lo = uint64_t(uint32_t(k.qx)) | (uint64_t(uint32_t(k.qy)) << 32);
  hi = uint64_t(uint32_t(k.qz)) | (uint64_t(k.qn & 0x3ffffffu) << 32) |
       (uint64_t(k.level & 0x1fu) << 58) | (1ull << 63);
}

__device__ __forceinline__ void cas128(unsigned long long* addr, uint64_t new_lo, uint64_t new_hi,
                                       uint64_t& old_lo, uint64_t& old_hi) {
  asm volatile(
      "{\n\t.reg .b128 d, c, s;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 s, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, s;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}\n"
      : "=l"(old_lo), "=l"(old_hi)
      : "l"(0ull), "l"(0ull), "l"(new_lo), "l"(new_hi), "l"(addr)
      : "memory");
}

__device__ __forceinline__ Key unpack_key(uint64_t lo, uint64_t hi) {
  return Key{int32_t(uint32_t(lo)), int32_t(uint32_t(lo >> 32)), int32_t(uint32_t(hi)),
             uint32_t(hi >> 32) & 0x3ffffffu, uint32_t(hi >> 58) & 0x1fu};
}

// lookup_or_insert (hash_grid.cpp:113-141) is split in two so that the table
// the reference builds -- keys inserted one by one in canonical lookup order
// -- comes out slot for slot, whatever order the threads run in:
//  * during a pass every lookup only reads the table as it stood when the
//    pass began (probe_find); nothing writes it, so plain loads are exact;
//  * keys not found (kPending) are collected once each with the smallest
//    canonical id that looked them up (nk_register), inserted after the
//    lookups in that order (k_insert), and published (k_commit).
// Linear probing from hash % capacity over min(probe_limit, capacity) slots.
// kPending: an empty slot ends the probe (the key is new); kFallback: the
// window is full of other keys (the table only grows, so the reference's
// lookup exhausts it too, hash_grid.cpp:140).
// Slot i of the probe sequence of hash h: (h + i) % capacity in uint64
// arithmetic, as the reference computes it (the sum wraps for h within
// probe_limit of 2^64).
__device__ __forceinline__ uint32_t probe_slot(uint64_t h, uint32_t i, uint64_t cap) {
  return uint32_t((h + i) % cap);
}

__device__ __forceinline__ uint32_t probe_find(const DevGrid& g, uint64_t lo, uint64_t hi,
                                               uint64_t h) {
  const uint32_t probes = min(g.probe_limit, g.capacity);
  const bool wraps = h > ~0ull - probes;
  uint32_t slot = uint32_t(h % uint64_t(g.capacity));
  for (uint32_t i = 0; i < probes; ++i) {
    if (wraps) slot = probe_slot(h, i, g.capacity);
    const ulonglong2 cur = __ldcg(reinterpret_cast<const ulonglong2*>(g.slot_keys + 2 * size_t(slot)));
    if (cur.x == lo && cur.y == hi) return slot;
    if (cur.y == 0) return kPending;  // empty (an occupied word has the valid bit in hi)
    slot = slot + 1 == g.capacity ? 0 : slot + 1;
  }
  return kFallback;
}

// Files a pending key with canonical id `id` in the pass's new-key table
// (128-bit CAS claim, smallest id kept).  Many warps file the same keys
// (a cold table: every lookup misses), so each entry is read first and
// written only when that can change it.  A plain 16-byte read may observe a
// claim half done; the entry is taken as another key's only when a complete
// half differs from ours (a valid hi word, or a non-zero lo word), and as
// ours only when both halves match -- otherwise the CAS decides.
__device__ __forceinline__ void nk_register(const NewKeys& nk, uint64_t lo, uint64_t hi, uint64_t h,
                                            uint32_t id, uint32_t* err) {
  uint32_t e = uint32_t(h ^ (h >> 31)) & nk.mask;
  for (uint32_t i = 0; i <= nk.mask; ++i) {
    const ulonglong2 cur = __ldcg(reinterpret_cast<const ulonglong2*>(nk.keys + 2 * size_t(e)));
    bool mine = cur.x == lo && cur.y == hi;
    const bool other = (cur.y != 0 && cur.y != hi) || (cur.x != 0 && cur.x != lo);
    if (!mine && !other) {
      uint64_t olo, ohi;
      cas128(nk.keys + 2 * size_t(e), lo, hi, olo, ohi);
      if (olo == 0 && ohi == 0) {
        const uint32_t d = atomicAdd(nk.count, 1u);
        nk.list[d] = e;
        atomicMin(nk.id + e, id);
        return;
      }
      mine = olo == lo && ohi == hi;
    }
    if (mine) {
      if (id < __ldcg(nk.id + e)) atomicMin(nk.id + e, id);  // ids only decrease
      return;
    }
    e = (e + 1) & nk.mask;
  }
  atomicOr(err, kErrNewKeyOverflow);
}

// k_insert: the pending keys of the pass into the table as if inserted one
// by one in order of their smallest canonical id.  Ordered linear probing
// (Amble & Knuth): along its probe window a key passes occupied slots and
// slots claimed by earlier keys, claims the first other slot with atomicMin
// on (id << 32 | d), and a later key it displaces carries on from there.  At
// the fixpoint every key sits on the first slot of its window not held by an
// earlier key -- exactly the reference's sequential insertion -- or, if its
// whole window is held by earlier keys, has none (the fallback cut).
__global__ void __launch_bounds__(128) k_insert(DevGrid g, NewKeys nk) {
  const uint32_t n = *nk.count;
  const uint32_t probes = min(g.probe_limit, g.capacity);
  const uint64_t cap = g.capacity;
  for (uint32_t d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    uint32_t e = nk.list[d];
    uint64_t v = (uint64_t(nk.id[e]) << 32) | d;
    uint64_t h = hash_key(unpack_key(nk.keys[2 * size_t(e)], nk.keys[2 * size_t(e) + 1]));
    uint32_t i = 0;
    while (i < probes) {
      const uint64_t s = probe_slot(h, i, cap);
      if (__ldcg(g.slot_keys + 2 * s + 1) != 0) {  // a key of an earlier pass
        ++i;
        continue;
      }
      const uint64_t old = atomicMin(g.claim + s, v);
      if (old == ~0ull) break;  // the slot was free: placed
      if (old < v) {            // held by an earlier key
        ++i;
        continue;
      }
      // displaced a later key: it continues behind this slot
      v = old;
      e = nk.list[uint32_t(old)];
      h = hash_key(unpack_key(nk.keys[2 * size_t(e)], nk.keys[2 * size_t(e) + 1]));
      uint32_t j = 0;  // its position in its own window (it held slot s)
      while (j + 1 < probes && probe_slot(h, j, cap) != uint32_t(s)) ++j;
      i = j + 1u;
    }
  }
}

// k_commit: one warp per new key finds its claimed slot (if any), publishes
// the key and a fresh cell holding the template cut (hash_grid.cpp:121-127),
// and clears the new-key entry for the next pass.
__global__ void __launch_bounds__(256) k_commit(DevGrid g, NewKeys nk) {
  const uint32_t n = *nk.count;
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) atomicAdd(g.counters + kCntNewKeys, (unsigned long long)n);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t probes = min(g.probe_limit, g.capacity);
  const uint64_t cap = g.capacity;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); d < n; d += warps) {
    const uint32_t e = nk.list[d];
    const uint64_t lo = nk.keys[2 * size_t(e)], hi = nk.keys[2 * size_t(e) + 1];
    const uint64_t v = (uint64_t(nk.id[e]) << 32) | d;
    const uint64_t h = hash_key(unpack_key(lo, hi));
    uint32_t slot = kFallback;
    for (uint32_t i0 = 0; i0 < probes && slot == kFallback; i0 += 32) {
      const uint32_t i = i0 + lane;
      bool mine = false;
      uint64_t s = 0;
      if (i < probes) {
        s = probe_slot(h, i, cap);
        // slots of earlier passes keep stale-free claims (cleared below), but
        // the key check first keeps a numerically equal old claim out
        mine = __ldcg(g.slot_keys + 2 * s + 1) == 0 && __ldcg(g.claim + s) == v;
      }
      const unsigned m = __ballot_sync(kFull, mine);
      if (m) slot = probe_slot(h, i0 + uint32_t(__ffs(m) - 1), cap);
    }
    __syncwarp();
    if (lane == 0) {
      nk.keys[2 * size_t(e)] = 0;
      nk.keys[2 * size_t(e) + 1] = 0;
      nk.id[e] = 0xffffffffu;
    }
    if (slot == kFallback) continue;
    uint32_t cid = 0;
    if (lane == 0) {
      cid = uint32_t(atomicAdd(g.counters + kCntCells, 1ull));
      RLC_CHECK(cid < g.capacity && slot < g.capacity, g.counters + kCntErr);
      g.claim[slot] = ~0ull;
      g.slot_keys[2 * size_t(slot)] = lo;
      g.slot_keys[2 * size_t(slot) + 1] = hi;
      g.slot_cell[slot] = cid;
      g.cell_slot[cid] = slot;
      const Key k = unpack_key(lo, hi);
      uint32_t* ck = g.cell_key + size_t(5) * cid;
      ck[0] = uint32_t(k.qx);
      ck[1] = uint32_t(k.qy);
      ck[2] = uint32_t(k.qz);
      ck[3] = k.qn;
      ck[4] = k.level;
      g.touched[cid] = 0;
    }
    cid = __shfl_sync(kFull, cid, 0);
    const size_t row = size_t(cid) * g.M;
    for (uint32_t j = lane; j < g.M; j += 32) {
      g.node_ids[row + j] = g.t_node[j];
      g.ends[row + j] = g.t_ends[j];
      g.q[row + j] = g.t_q[j];
      g.cdf[row + j] = g.t_cdf[j];
      g.visits[row + j] = g.t_visits[j];
    }
  }
}

void launch_insert_new_keys(const DevGrid& g, const NewKeys& nk, cudaStream_t st) {
  static const uint32_t blocks = [] {
    const char* e = std::getenv("RLC_INSERT_BLOCKS");
    return e ? uint32_t(std::max(1, std::atoi(e))) : 2u * 148u;
  }();
  k_insert<<<blocks, 128, 0, st>>>(g, nk);
  k_commit<<<blocks, 256, 0, st>>>(g, nk);
  count_launch(2);
}

// ---------------------------------------------------------------------------
// k_primary: PassRenderer::trace up to the cell lookup (render.cpp:59-99)
// ---------------------------------------------------------------------------
// Thread -> path mapping: with one sample per pixel and pass, each warp
// takes an 8 x 4 pixel tile (coherent camera rays for the packet traversal);
// otherwise consecutive canonical indices.  Results land at the canonical
// index either way.
__device__ __forceinline__ bool path_of_thread(const PassParams& P, uint32_t rows, uint32_t* idx,
                                               uint32_t* px, uint32_t* py, uint32_t* s) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (P.spp_pp == 1) {
    const uint32_t warp = t >> 5, lane = t & 31u;
    const uint32_t tiles_x = (P.width + 7u) / 8u;
    const uint32_t tx = warp % tiles_x, ty = warp / tiles_x;
    const uint32_t x = tx * 8u + (lane & 7u), y = ty * 4u + (lane >> 3);
    *s = 0;
    *px = x;
    *py = P.row_begin + y;
    *idx = y * P.width + x;
    return x < P.width && y < rows;
  }
  *idx = t;
  *s = t % P.spp_pp;
  const uint32_t pix = t / P.spp_pp;
  *px = pix % P.width;
  *py = P.row_begin + pix / P.width;
  return t < P.n;
}

// First RNG dimension of the draws at path vertex `depth` (1-based):
// RandomSequence::next() order of PassRenderer::trace (render.cpp:63-133):
// jx, jy, then per vertex u1 u2 u3 [ju1 ju2 learned] b1 b2.
__device__ __forceinline__ uint32_t draw_base(const PassParams& P, uint32_t depth) {
  return kDrawU1 + (depth - 1u) * (P.sampler == 2u ? 7u : 5u);
}

// Shading of a closest hit at vertex `depth` (render.cpp:74-99, up to the
// cell lookup): G-buffer entry plus the cell key of a learned vertex.
__device__ __forceinline__ void shade_vertex(const DevScene& sc, const DevGrid& g,
                                             const PassParams& P, uint32_t depth, V3 org, V3 dir,
                                             double t, uint32_t tri, double pdf_omega, GBuf& out,
                                             bool& need, Key& key, uint64_t& h, uint32_t* err) {
  const V3 pos = org + dir * t;
  const V3 ng = ld3(sc.tri_normal + size_t(3) * tri);
  const V3 wo = -dir;
  const double cos_facing = dot(ng, wo);
  const uint32_t mat = sc.tri_mat[tri];
  const MatRec& m = sc.mats[mat];
  uint32_t flags = kGHit | mat;
  if (depth == 1 && m.is_emitter && cos_facing > 0) flags |= kGEmit;
  const V3 ns = dot(ng, wo) < 0 ? -ng : ng;  // faceforward, math.hpp:59-61
  out.pos[0] = pos.x;
  out.pos[1] = pos.y;
  out.pos[2] = pos.z;
  out.ns[0] = ns.x;
  out.ns[1] = ns.y;
  out.ns[2] = ns.z;
  if (m.reflective) {
    flags |= kGReflective;
    if (P.sampler == 2u) {
      const double cos_in = fabs(cos_facing);
      const double area_pdf =
          smax(pdf_omega * cos_in / smax(t * t, 1e-24), 1e-12);  // render.cpp:86-88
      if (!(area_pdf > 0)) atomicOr(err, kErrBadAreaPdf);
      // level_for_footprint (hash_grid.cpp:34-44) via host-derived thresholds
      const double r = 1.0 / sqrt(area_pdf) / sc.base_tile;
      uint32_t level = 0;
#pragma unroll
      for (int k = 1; k <= 16; ++k) level += (r >= sc.level_thr[k]) ? 1u : 0u;
      if (fabs(length(ns) - 1.0) > 1e-4) atomicOr(err, kErrNonUnitNormal);
      const uint32_t base = draw_base(P, depth);
      const double ju1 = rng_draw(out.rng, base + 3u);
      const double ju2 = rng_draw(out.rng, base + 4u);
      key = make_key(pos, ns, level, ju1, ju2, sc.base_tile, g.normal_bits, g.jitter_scale);
      h = hash_key(key);
      need = true;
    }
  }
  out.flags = flags;
}

// Warp-cooperative lookup (hash_grid.cpp:113-141 up to the insertion): one
// probe per distinct hash in the warp (all 32 lanes must call).  A key the
// table lacks is filed once with the smallest vertex id of the lanes that
// hold it; the vertex keeps its packed key for the resolution after k_commit.
__device__ __forceinline__ void warp_lookup(const DevGrid& g, const NewKeys& nk,
                                            unsigned long long* __restrict__ pkey, bool need,
                                            const Key& key, uint64_t h, uint32_t vid,
                                            uint32_t lane, uint32_t* slot_out, uint32_t* err,
                                            bool file_new) {
  const unsigned need_mask = __ballot_sync(kFull, need);
  if (!need) return;
  uint64_t lo, hi;
  pack_key(key, lo, hi);
  const unsigned peers = __match_any_sync(need_mask, h) & need_mask;
  const int leader = __ffs(peers) - 1;
  // the lookup's dense cell id (slot_cell of the found slot) or the
  // kPending / kFallback sentinel
  auto cell_of = [&](uint32_t sl) { return sl < kPending ? g.slot_cell[sl] : sl; };
  uint32_t slot = 0;
  if (int(lane) == leader) slot = cell_of(probe_find(g, lo, hi, h));
  slot = __shfl_sync(peers, slot, leader);
  const uint64_t llo = __shfl_sync(peers, lo, leader);
  const uint64_t lhi = __shfl_sync(peers, hi, leader);
  const bool same = llo == lo && lhi == hi;
  const unsigned same_mask = __ballot_sync(peers, same);
  if (same) {
    if (slot == kPending && file_new) {
      const uint32_t first = __reduce_min_sync(same_mask, vid);
      if (int(lane) == leader) nk_register(nk, lo, hi, h, first, err);
    }
  } else {  // 64-bit hash collision inside the warp
    slot = cell_of(probe_find(g, lo, hi, h));
    if (slot == kPending && file_new) nk_register(nk, lo, hi, h, vid, err);
  }
  if (slot == kPending) {
    pkey[2 * size_t(vid)] = lo;
    pkey[2 * size_t(vid) + 1] = hi;
  }
  if (file_new) {
    const unsigned pm = __ballot_sync(need_mask, slot == kPending);
    if (pm && int(lane) == __ffs(pm) - 1)
      atomicAdd(g.counters + kCntPending, (unsigned long long)__popc(pm));
  }
  *slot_out = slot;
  const unsigned fb = __ballot_sync(need_mask, slot == kFallback);
  if (int(lane) == __ffs(need_mask) - 1) {
    atomicAdd(g.counters + kCntLookups, (unsigned long long)__popc(need_mask));
    if (fb) atomicAdd(g.counters + kCntFallback, (unsigned long long)__popc(fb));
  }
}

#ifndef RLC_PRIMARY_BLOCKS
#define RLC_PRIMARY_BLOCKS 8  // blocks per SM (64 registers): measured best on c3
#endif
__global__ void __launch_bounds__(128, RLC_PRIMARY_BLOCKS) k_primary(DevScene sc, DevGrid g, PassParams P,
                                                 GBuf* __restrict__ gbuf, NewKeys nk,
                                                 unsigned long long* __restrict__ pkey) {
  const uint32_t rows = P.n / (P.width * P.spp_pp);
  uint32_t idx, px, py, s;
  const bool active = path_of_thread(P, rows, &idx, &px, &py, &s);
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t* err = reinterpret_cast<uint32_t*>(g.counters + kCntErr);

  bool need = false;
  Key key{};
  uint64_t h = 0;
  GBuf out;
  out.cell = kNoSlot;
  out.flags = 0;
  V3 org{0, 0, 0}, dir{0, 0, 1};
  uint64_t rk = 0;
  if (active) {
    const uint64_t pixel_index = uint64_t(py) * uint64_t(P.width) + px;
    // graph replays: the replay's first pass index in device memory, plus
    // this pass's position in the graph
    const uint32_t pass = P.pass_dev ? *P.pass_dev + P.pass_index : P.pass_index;
    const uint64_t sample_index = uint64_t(pass) * P.spp_pp + s;
    rk = rng_key(P.seed_mixed, pixel_index, sample_index, P.zero_mixed);
    const double jx = rng_draw(rk, kDrawJx);
    const double jy = rng_draw(rk, kDrawJy);
    // camera_ray, scene.cpp:10-23
    const CameraConst& c = sc.cam;
    const double fx = double(px) + jx;
    const double fy = double(py) + jy;
    const double sx = (2.0 * fx / c.width_d - 1.0) * c.tan_half * c.aspect;
    const double sy = (1.0 - 2.0 * fy / c.height_d) * c.tan_half;
    dir = normalize(ld3(c.u) * sx + ld3(c.v) * sy - ld3(c.w));
    org = ld3(c.origin);
  }
  out.rng = rk;
  double t = 0;
  uint32_t tri = 0;
  const bool got = active && (sc.fp32_ok ? intersect_camera(sc, org, dir, &t, &tri, err)
                                         : intersect(sc, org, dir, 0.0, &t, &tri, err));
  if (got) shade_vertex(sc, g, P, 1u, org, dir, t, tri, sc.cam.pdf_omega, out, need, key, h, err);
  warp_lookup(g, nk, pkey, need, key, h, idx * P.depth, lane, &out.cell, err,
              !P.defer_insert);
  if (active) gbuf[size_t(idx) * P.depth] = out;
}

// ---------------------------------------------------------------------------
// k_bounce: the continuation of PassRenderer::trace from vertex depth-1 to
// vertex depth (render.cpp:127-135, then 71-99 for the new hit):
// sample_cosine_hemisphere (math.hpp:101-107) with the host libm's exact
// sin/cos (rlc_libm.h), the closest hit from t_min = shadow_eps in the
// reference traversal order, and the cell lookup of the new vertex.
// ---------------------------------------------------------------------------
__device__ const double kSinCosTab[440] = RLC_SINCOSTAB_INIT;

__device__ __forceinline__ V3 cosine_hemisphere(const DevScene& sc, V3 n, double u1, double u2) {
  const libm::Ctx lc{kSinCosTab, sc.libm_fma != 0};
  const double r = sqrt(u1);
  const double phi = 2.0 * kPi * u2;
  const V3 local{r * libm::cos(lc, phi), r * libm::sin(lc, phi), sqrt(smax(0.0, 1.0 - u1))};
  // Frame (math.hpp:85-99): Duff et al. branchless basis
  const double sign = copysign(1.0, n.z);
  const double a = -1.0 / (sign + n.z);
  const double bb = n.x * n.y * a;
  const V3 t{1.0 + sign * n.x * n.x * a, sign * bb, -sign * n.x};
  const V3 b{bb, sign + n.y * n.y * a, -n.y};
  return t * local.x + b * local.y + n * local.z;
}

#ifndef RLC_BOUNCE_BLOCKS
#define RLC_BOUNCE_BLOCKS 6  // blocks per SM (80 registers): c3 depth 3 5.07 -> 4.75 ms per frame
#endif
__global__ void __launch_bounds__(128, RLC_BOUNCE_BLOCKS) k_bounce(DevScene sc, DevGrid g, PassParams P,
                                                uint32_t depth, GBuf* __restrict__ gbuf,
                                                NewKeys nk, unsigned long long* __restrict__ pkey) {
  const uint32_t path = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = path < P.n;
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t* err = reinterpret_cast<uint32_t*>(g.counters + kCntErr);
  bool need = false;
  Key key{};
  uint64_t h = 0;
  GBuf out;
  out.cell = kNoSlot;
  out.flags = 0;
  out.rng = 0;
  bool go = false;
  V3 org{0, 0, 0}, dir{0, 0, 1};
  double pdf_omega = 0;
  if (active) {
    const GBuf prev = gbuf[size_t(path) * P.depth + depth - 2u];
    out.rng = prev.rng;
    if (prev.flags & kGReflective) {  // render.cpp:127: non-reflective vertices end the path
      const uint32_t base = draw_base(P, depth - 1u) + (P.sampler == 2u ? 5u : 3u);
      const double b1 = rng_draw(prev.rng, base);
      const double b2 = rng_draw(prev.rng, base + 1u);
      const V3 ns = ld3(prev.ns);
      dir = cosine_hemisphere(sc, ns, b1, b2);
      const double cos_theta = dot(ns, dir);
      if (!(cos_theta <= 0)) {
        go = true;
        pdf_omega = cos_theta / kPi;
        org = ld3(prev.pos);
      }
    }
  }
  double t = 0;
  uint32_t tri = 0;
  const bool got = go && intersect(sc, org, dir, sc.shadow_eps, &t, &tri, err);
  if (got) shade_vertex(sc, g, P, depth, org, dir, t, tri, pdf_omega, out, need, key, h, err);
  warp_lookup(g, nk, pkey, need, key, h, path * P.depth + depth - 1u, lane, &out.cell, err,
              !P.defer_insert);
  if (active) gbuf[size_t(path) * P.depth + depth - 1u] = out;
}

// ---------------------------------------------------------------------------
// k_sample: sample_light + nee_estimate (estimators.cpp:28-106)
// ---------------------------------------------------------------------------
// std::upper_bound over the cdf row, clamped to M - 1 (sample_cluster,
// cut.cpp:97-106).  A two-round 16-ary count over the (non-decreasing) row
// was measured slower on c3 (k_sample 0.216 -> 0.249 ms).
__device__ __forceinline__ uint32_t upper_bound_cdf(const double* __restrict__ cdf, uint32_t M,
                                                    double target) {
  uint32_t lo = 0, cnt = M;
  while (cnt > 0) {
    const uint32_t step = cnt >> 1;
    if (!(target < cdf[lo + step])) {
      lo += step + 1;
      cnt -= step + 1;
    } else {
      cnt = step;
    }
  }
  return lo == M ? M - 1 : lo;
}

// stable compaction tiles (k_cmp_*): 256 threads x 8 vertices
constexpr int kCmpThreads = 256, kCmpItems = 8, kCmpTile = kCmpThreads * kCmpItems;

#ifndef RLC_SAMPLE_BLOCKS
#define RLC_SAMPLE_BLOCKS 7  // 72 registers, 7 blocks per SM: c3 0.880 vs 0.886 ms at 84 (6 blocks)
#endif
#ifndef RLC_SORT_COMPACT
#define RLC_SORT_COMPACT 0  // compacting the records first measured slower (its three
                            // launches delay the sort past the shadow rays): c3 1.105 vs 1.089 ms
#endif
__global__ void __launch_bounds__(128, RLC_SAMPLE_BLOCKS) k_sample(DevScene sc, DevGrid g, PassParams P,
                                                const GBuf* __restrict__ gbuf,
                                                SampleRec* __restrict__ srec,
                                                uint8_t* __restrict__ rflag,
                                                uint32_t* __restrict__ keys,
                                                uint32_t* __restrict__ vals,
                                                double* __restrict__ q_before,
                                                ShadowRay* __restrict__ rays,
                                                unsigned int* __restrict__ ray_count,
                                                const unsigned long long* __restrict__ pkey,
                                                uint32_t* __restrict__ emit,
                                                double* __restrict__ vdense,
                                                uint32_t* __restrict__ gflags,
                                                uint32_t* __restrict__ ray_tile_counts) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;  // path vertex
  if (idx >= P.nv) return;
  uint32_t* err = reinterpret_cast<uint32_t*>(g.counters + kCntErr);
  const GBuf gb = ldg_vec(gbuf + idx);
  gflags[idx] = gb.flags;
  keys[idx] = kInvalidKey;
  if (!(gb.flags & kGReflective)) {  // (its sample record is never read: no partial store)
    rflag[idx] = 0;  // read by the compactions
    return;
  }
  const uint32_t base = draw_base(P, idx % P.depth + 1u);
  const double u1 = rng_draw(gb.rng, base);
  const double u2 = rng_draw(gb.rng, base + 1u);
  const double u3 = rng_draw(gb.rng, base + 2u);

  SampleRec r;
  r.flags = 0;
  r.s = 0;
  r.total = 0;
  uint32_t e = 0;
  double frozen_share = 0;      // learned: the cluster's share of the frozen cdf
  uint32_t lpos = 0xffffffffu;  // learned: light-tree position of the pick
  if (P.sampler == 2u) {
    // A key new this pass (kPending) has been inserted in canonical order
    // since the lookups (k_insert / k_commit) or refused (fallback); either
    // way its cut is still the template (a new cell starts as a copy, the
    // fallback cut never changes), so the selection reads the template.
    // Sharded traces (defer_insert) leave the insertion to the fold of all
    // ranks' records.
    uint32_t cell = gb.cell;
    const bool fresh = cell == kPending;
    if (fresh && !P.defer_insert) {
      const uint64_t lo = pkey[2 * size_t(idx)], hi = pkey[2 * size_t(idx) + 1];
      const uint32_t slot = probe_find(g, lo, hi, hash_key(unpack_key(lo, hi)));
      if (slot < kPending) {
        cell = g.slot_cell[slot];
      } else {
        cell = kFallback;
        atomicAdd(g.counters + kCntFallback, 1ull);
      }
    }
    const bool fallback = cell == kFallback;
    const bool tmpl = fallback || fresh;
    const uint32_t M = g.M;
    const size_t row = tmpl ? 0 : size_t(cell) * M;
    const double* cdf = tmpl ? g.t_cdf : g.cdf + row;
    const uint32_t* ends = tmpl ? g.t_ends : g.ends + row;
    // sample_cluster (cut.cpp:97-106): upper_bound of u1 * total.  (A
    // two-round search from a per-cell summary of 8 block maxima -- 24
    // independent loads instead of log2 M dependent ones -- measured slower
    // on c3: 1.117 vs 1.086 ms per frame, same box.)
    const double total = cdf[M - 1];
    const double target = u1 * total;
    const uint32_t s = upper_bound_cdf(cdf, M, target);
    const uint32_t begin = s == 0 ? 0u : ends[s - 1];
    const uint32_t size = ends[s] - begin;
    const double clo = s == 0 ? 0.0 : cdf[s - 1];
    const double span = cdf[s] - clo;
    const double frac = span > 0 ? clampd((u1 * total - clo) / span, 0.0, 1.0) : 0.0;
    if (P.frozen_pdf) frozen_share = span / total;
    const uint32_t offset = min(size - 1, uint32_t(frac * double(size)));
    RLC_CHECK(s < M && size >= 1 && begin + offset < sc.num_lights, err);
    lpos = begin + offset;  // tree.order[begin + offset] is the emitter (lights_ord)
    r.pin = 1.0 / double(size);
    r.total = total;
    r.s = s;
    r.flags = kSLearned;
    if (fallback) {
      q_before[idx] = g.t_q[s];  // the fallback cut is never updated
    } else {
      // carries an update_q record (render.cpp:111-117); a deferred new key
      // is sorted by the sharded fold
      if (cell < kPending) keys[idx] = cell * M + s;
      r.flags |= kSRecord;
    }
  } else if (P.sampler == 0u) {
    const uint32_t n = sc.num_lights;
    e = min(n - 1, uint32_t(u1 * double(n)));
    r.pin = 1.0 / double(n);
  } else {
    const uint32_t n = sc.num_lights;
    const double back = sc.energy_cdf[n - 1];
    const double target = u1 * back;
    uint32_t lo = 0, cnt = n;
    while (cnt > 0) {
      const uint32_t step = cnt >> 1;
      if (!(target < sc.energy_cdf[lo + step])) {
        lo += step + 1;
        cnt -= step + 1;
      } else {
        cnt = step;
      }
    }
    e = lo == n ? n - 1 : lo;
    r.pin = sc.emitter_energy[e] / back;
  }

  V3 p0, p1, p2, nl, emission;
  double pdf_area;
  if (lpos != 0xffffffffu) {  // the pick's record at its tree position (order[] folded in)
    static_assert(sizeof(LightOrd) == 80, "LightOrd layout");
    const LightOrd L = ldg_vec(sc.lights_ord + lpos);  // 5 128-bit loads
    e = L.emitter;
    p0 = ld3(L.p0), p1 = ld3(L.p1), p2 = ld3(L.p2);
    // triangle_normal and 1 / area exactly as LightRec holds them
    const V3 cr = cross(p1 - p0, p2 - p0);
    nl = normalize(cr);
    const double area = 0.5 * length(cr);
    pdf_area = area > 0 ? 1.0 / area : 0.0;
    emission = ld3(sc.mats[L.mat].emission);
  } else {
    RLC_CHECK(e < sc.num_lights, err);
    const LightRec& L = sc.lights[e];
    p0 = ld3(L.p0), p1 = ld3(L.p1), p2 = ld3(L.p2), nl = ld3(L.n);
    pdf_area = L.pdf_area;
    emission = ld3(L.emission);
  }
  if (P.export_samples) emit[idx] = e;
  r.pdf_area = pdf_area;
  if (!(pdf_area > 0)) atomicOr(err, kErrDegenerateLight);
  // sample_triangle_point, scene.cpp:49-59
  const double su = sqrt(u2);
  const double b0 = 1.0 - su;
  const double b1 = u3 * su;
  const V3 point = p0 * b0 + p1 * b1 + p2 * (1.0 - b0 - b1);
  // nee_estimate, estimators.cpp:82-106
  const V3 pos = ld3(gb.pos);
  const V3 ns = ld3(gb.ns);
  r.c[0] = r.c[1] = r.c[2] = 0;
  r.v = 0;
  V3 to_light = point - pos;
  const double d2 = dot(to_light, to_light);
  if (!(d2 < 1e-24)) {
    const double d = sqrt(d2);
    to_light = to_light / d;
    const double cos_x = dot(ns, to_light);
    if (!(cos_x <= 0)) {
      const double cos_y = dot(nl, -to_light);
      if (!(cos_y <= 0)) {
        // Contribution as if visible; k_shadow zeroes it when the segment
        // is occluded (occluded(), bvh.cpp:159-188, is q-independent).
        const MatRec& m = sc.mats[gb.flags & kGMatMask];
        const double geometry = cos_x * cos_y / d2;
        const V3 contrib = ld3(m.albedo) * (1.0 / kPi) * emission * geometry;
        r.c[0] = contrib.x;
        r.c[1] = contrib.y;
        r.c[2] = contrib.z;
        r.flags |= kSNonzero;
        // estimators.cpp:103-104; pdf_in_cluster is 1 for the baselines
        r.v = luminance(contrib) / ((P.sampler == 2u ? r.pin : 1.0) * r.pdf_area);
        if (P.frozen_pdf && (r.flags & kSLearned)) {
          // pdf_mode frozen_cdf: the probability the selection used -- the
          // cluster's share of the frozen cdf -- not the live q;
          // the learning (v, the fold) is unchanged
          r.pin = frozen_share * r.pin;
          r.flags |= kSFrozen;
        }
        // the shadow segment (pos, point) of occluded(): bvh.cpp:160-167
        const V3 dd = point - pos;
        const double len = length(dd);
        if (!(len <= 2 * sc.shadow_eps)) {
          const V3 dir = dd / len;
          ShadowRay ray;
          ray.o[0] = pos.x;
          ray.o[1] = pos.y;
          ray.o[2] = pos.z;
          ray.d[0] = dir.x;
          ray.d[1] = dir.y;
          ray.d[2] = dir.z;
          ray.tmax = len - sc.shadow_eps;
          ray.idx = idx;
          ray.pad = 0;
          rays[idx] = ray;
          r.flags |= kSRay;
        }
      }
    }
  }
  srec[idx] = r;
  vdense[idx] = r.v;
  rflag[idx] = uint8_t(r.flags & (kSNonzero | kSLearned | kSRay | kSRecord));
  // the ray compaction's per-tile counts (k_cmp_count's work): one atomic per
  // group of converged lanes; a warp's 32 vertices lie in one tile
  const unsigned am = __activemask();
  const unsigned rm = __ballot_sync(am, (r.flags & kSRay) != 0);
  if ((threadIdx.x & 31u) == uint32_t(__ffs(am) - 1) && rm)
    atomicAdd(ray_tile_counts + idx / kCmpTile, uint32_t(__popc(rm)));
}

// ---------------------------------------------------------------------------
// k_shadow: any-hit traversal of the queued shadow segments.  Persistent
// warps refill idle lanes from the queue (dynamic ray fetch) so incoherent
// shadow rays keep the SIMT lanes busy; each traversal step reads one
// child-pair record and runs both children's slab tests.
// ---------------------------------------------------------------------------
constexpr int kShadowThreads = 128;
// per-lane stack entries (shared memory); a ray that would overflow it is
// finished on the exact fp64 path (occluded_ray), so the size only trades
// shared memory (hence L1) against how often that happens
#ifndef RLC_SHADOW_STACK
#define RLC_SHADOW_STACK (kWide == 8 ? 64 : 12)  // c3: 12 entries 1.085 ms, 16: 1.092, 32: 1.111, 8: 1.25 (428 exact re-runs per frame)
#endif
constexpr int kShadowStack = RLC_SHADOW_STACK;
constexpr uint32_t kDone = 0x7fffffffu;  // traversal finished (no leaf flag)

// Leaf entries: kWideLeaf | kLeafVerified? | (count - 1) << 28 | kLeafPure? |
// first tri (27 bits).  kLeafVerified (set during traversal) is only ever set
// on pure leaves, whose box lies inside their reference leaf's box.
constexpr uint32_t kLeafVerified = 0x40000000u;
__device__ __forceinline__ uint32_t leaf_first(uint32_t e) { return e & 0x07ffffffu; }
__device__ __forceinline__ uint32_t leaf_count(uint32_t e) { return ((e >> 28) & 3u) + 1u; }

// Exact acceptance of a triangle found through the conservative wide tree.
// The reference reaches a leaf iff every node on its ancestor chain passes
// the fp64 slab test (bvh.cpp:29-40).  That test is monotone under box
// inclusion (a larger box only lowers the entry and raises the exit, and
// rounding is monotone) and every binary parent's box contains its
// children's (exact min/max over a superset of triangles), so the chain
// passes iff the leaf's own box passes: one exact test, skipped entirely
// when the fp32 inner test already proved it (kLeafVerified).
__device__ __forceinline__ bool leaf_reached(const DevScene& sc, uint32_t e, V3 o, V3 inv,
                                             double tmin, double tmax) {
  if (e & kLeafVerified) return true;
  return box_hit(load_node(sc.nodes, __ldg(sc.tri_leaf_s + leaf_first(e))), o, inv, tmin, tmax);
}

// Conservative fp32 slab test of the 4 children of a Wide4 node against one
// ray.  Per axis the reference computes t = fl64(fl64(c - o) * inv) on the
// exact box (bvh.cpp:29-40); here t' = fma(c', inv', -o'inv') on the outward-
// rounded fp32 box, widened by |t'| 2^-20 + |o'||inv'| 2^-21: the box rounding
// only ever moves t' outward and the margin bounds the fp32 rounding of the
// origin, inverse and FMA plus the fp64 reference's own rounding, so the
// interval contains the reference's and the test passes whenever the
// reference's passes.  NaN terms (zero direction components) are ignored by
// fmaxf/fminf, which only drops a constraint.  Rays with |inv| > 1e30 (fp32
// range) take the exact fp64 path instead (ShadowLane::exact).
struct RayF {
  float inv[3], b[3], mt[3], mb[3];
  uint32_t neg;  // bit a: inv[a] < 0 (near plane is hi)
  float tmin, tmax;        // outward-rounded interval (outer test)
  float tmin_in, tmax_in;  // inward-rounded interval (inner test)
  bool fast;               // every |inv| finite and <= 1e30: the inner test is valid
  float margin;            // boxw_s inner margin S max|inv| 2^-19
};

// Shadow rays on the padded shadow tree (boxes grown by S 2^-21, S the
// largest |coordinate| of the scene; rlc_build.cpp build_wide).  For an
// origin within S the fp32 t = fma(c, inv, -(o inv)) differs from
// (c - o) inv by at most 6 S |inv| 2^-24 < S |inv| 2^-21, less than the
// padding moves the planes, so the plain slab test is the outer test.  The
// reference's t lies within S |inv_a| 2^-20 of ours on every axis, so the
// inner test shrinks the per-child interval by the ray constant
// margin = S max|inv| 2^-19 (infinite or NaN, i.e. no inner test, for
// axis-parallel rays, whose NaN slab terms fmaxf/fminf ignore).
__device__ __forceinline__ uint32_t boxw_s(const float (&lo)[3][kWide],
                                           const float (&hi)[3][kWide], const RayF& r,
                                           float (&near_out)[kWide], uint32_t* inner) {
  float nb[kWide], fb[kWide];
#pragma unroll
  for (int c = 0; c < kWide; ++c) {
    nb[c] = r.tmin;
    fb[c] = r.tmax;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool neg = (r.neg >> a) & 1u;
#pragma unroll
    for (int c = 0; c < kWide; ++c) {
      const float n = neg ? hi[a][c] : lo[a][c];
      const float f = neg ? lo[a][c] : hi[a][c];
      nb[c] = fmaxf(nb[c], fmaf(n, r.inv[a], r.b[a]));
      fb[c] = fminf(fb[c], fmaf(f, r.inv[a], r.b[a]));
    }
  }
  uint32_t m = 0, mi = 0;
#pragma unroll
  for (int c = 0; c < kWide; ++c) {
    m |= (nb[c] <= fb[c]) ? (1u << c) : 0u;
    mi |= (fmaxf(nb[c] + r.margin, r.tmin_in) <= fminf(fb[c] - r.margin, r.tmax_in)) ? (1u << c)
                                                                                      : 0u;
    near_out[c] = nb[c];
  }
  *inner = mi & m;
  return m;
}

// Also returns in *inner the children whose fp32 inner test passes (the
// interval narrowed by the rounding bound and the box rounding |c||inv|2^-22),
// i.e. the children whose exact fp64 test certainly passes (see box_decide).
__device__ __forceinline__ uint32_t boxw_f(const float (&lo)[3][kWide],
                                           const float (&hi)[3][kWide], const RayF& r,
                                           float (&near_out)[kWide], uint32_t* inner) {
  constexpr float K = 0x1.0p-20f;
  float nr[kWide], fr[kWide], ni[kWide], fi[kWide];
#pragma unroll
  for (int c = 0; c < kWide; ++c) {
    nr[c] = r.tmin;
    fr[c] = r.tmax;
    ni[c] = r.tmin_in;
    fi[c] = r.tmax_in;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const bool neg = (r.neg >> a) & 1u;
#pragma unroll
    for (int c = 0; c < kWide; ++c) {
      const float nc = neg ? hi[a][c] : lo[a][c];
      const float fc = neg ? lo[a][c] : hi[a][c];
      const float tn = fmaf(nc, r.inv[a], r.b[a]);
      const float tf = fmaf(fc, r.inv[a], r.b[a]);
      const float en = fmaf(fabsf(tn), K, r.mt[a]);
      const float ef = fmaf(fabsf(tf), K, r.mt[a]);
      nr[c] = fmaxf(nr[c], tn - en);
      fr[c] = fminf(fr[c], tf + ef);
      ni[c] = fmaxf(ni[c], tn + en + fmaf(fabsf(nc), r.mb[a], 1e-37f));
      fi[c] = fminf(fi[c], tf - ef - fmaf(fabsf(fc), r.mb[a], 1e-37f));
    }
  }
  uint32_t m = 0, mi = 0;
#pragma unroll
  for (int c = 0; c < kWide; ++c) {
    m |= (nr[c] <= fr[c]) ? (1u << c) : 0u;
    mi |= (ni[c] <= fi[c]) ? (1u << c) : 0u;
    near_out[c] = nr[c];
  }
  *inner = r.fast ? (mi & m) : 0u;
  return m;
}

// Branch-free Moller-Trumbore: the reference's expressions (bvh.cpp:44-62)
// with every early exit folded into one predicate.
// ---------------------------------------------------------------------------
// Closest hit on the collapsed reference tree.  The
// reference's closest hit equals a scan of its leaves in DFS order (right
// subtree first) in which a leaf's triangles are tested iff the leaf's own
// box passes the slab test against the running `closest`: every ancestor was
// tested earlier with a `closest` at least as large, on a box containing the
// leaf's, so it passed whenever the leaf passes (the slab test is monotone in
// both).  wide_ref keeps the binary left-to-right order in every node, so
// pushing the passing children left to right pops them in the reference's
// leaf order.  Internal children are culled conservatively with the `closest`
// of the moment (a failing box fails later too).  A leaf is decided when it
// is popped: by the fp32 inner test made at push time if `closest` has not
// changed since (the stack watermark `fresh`), else by the exact fp64 test
// of its reference box.  Triangle tests are the exact fp64 Moller-Trumbore.
// ---------------------------------------------------------------------------
// Three-input fp32 min / max (sm_100 FMNMX3); like fminf / fmaxf, a NaN
// operand is ignored.
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Camera rays on wide_cam: every stored coordinate is x' = fl32 outward of
// x -/+ 2^-21 |x| (x = fl64(c - O)), so fl32(x' * fl32(inv)) bounds the
// reference's fl64(x * inv) from outside on every axis and the plain slab
// test is the outer test.  The reference's per-axis t exceeds ours by less
// than 2^-20 |t|, and t -> t + |t| kappa is monotone, so the inner test
// (the exact test certainly passes) needs only the per-child near/far
// moved in by kappa = 2^-19.  t_min = 0; 1e-30 covers underflow.
__device__ __forceinline__ uint32_t boxw_cam(const float (&lo)[3][kWide],
                                             const float (&hi)[3][kWide], const float (&inv)[3],
                                             uint32_t neg, float tmax_up, float tmax_dn,
                                             uint32_t* inner) {
  constexpr float kappa = 0x1.0p-19f;
  float nb[kWide], fb[kWide];
#pragma unroll
  for (int c = 0; c < kWide; ++c) {
    float tn[3], tf[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const bool ng = (neg >> a) & 1u;
      tn[a] = (ng ? hi[a][c] : lo[a][c]) * inv[a];
      tf[a] = (ng ? lo[a][c] : hi[a][c]) * inv[a];
    }
    nb[c] = fmaxf(fmax3(0.f, tn[0], tn[1]), tn[2]);  // t_min = 0
    fb[c] = fmin3(tf[0], tf[1], tf[2]);
  }
  uint32_t m = 0, mi = 0;
#pragma unroll
  for (int c = 0; c < kWide; ++c) {
    m |= (nb[c] <= fminf(fb[c], tmax_up) + 1e-30f) ? (1u << c) : 0u;
    const float ni = fmaf(fabsf(nb[c]), kappa, nb[c]) + 1e-30f;
    const float fi = fminf(fmaf(-fabsf(fb[c]), kappa, fb[c]) - 1e-30f, tmax_dn);
    mi |= (ni <= fi) ? (1u << c) : 0u;
  }
  *inner = mi & m;
  return m;
}

template <bool CAM>
__device__ __forceinline__ bool closest_wide(const DevScene& sc, const Wide4* __restrict__ wn,
                                             RayF rf, V3 o, V3 d, V3 inv, double tmin,
                                             double* t_out, uint32_t* tri_out, uint32_t* err) {
  double closest = HUGE_VAL;
  uint32_t hit = kNoSlot;
  uint32_t stack[kStack];
  int sp = 0, fresh = 0;
  // the reference tests the root box first (bvh.cpp:130-134)
  if (!box_hit(load_node(sc.nodes, 0), o, inv, tmin, closest)) return false;
  uint32_t cur = 0;
  bool stale = false;
  while (true) {
    if (cur & kWideLeaf) {
      bool reach = true;
      if (stale || !(cur & kLeafVerified))
        reach = box_hit(load_node(sc.nodes, __ldg(sc.tri_leaf + leaf_first(cur))), o, inv, tmin,
                        closest);
      if (reach) {
        const uint32_t first = leaf_first(cur), cnt = leaf_count(cur);
        for (uint32_t k = first; k < first + cnt; ++k) {
          double t;
          if (tri_hit(sc.tris, k, o, d, tmin, closest, &t)) {
            closest = t;
            hit = k;
            rf.tmax = __double2float_ru(closest);
            rf.tmax_in = __double2float_rd(closest);
            fresh = sp;  // the leaves on the stack were decided with the old closest
          }
        }
      }
    } else {
      const float4* p = reinterpret_cast<const float4*>(wn + cur);
      float lo[3][kWide], hi[3][kWide];
      uint32_t c[kWide];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float4 vl = __ldg(p + a), vh = __ldg(p + 3 + a);
        lo[a][0] = vl.x, lo[a][1] = vl.y, lo[a][2] = vl.z, lo[a][3] = vl.w;
        hi[a][0] = vh.x, hi[a][1] = vh.y, hi[a][2] = vh.z, hi[a][3] = vh.w;
      }
      {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p + 6));
        c[0] = v.x, c[1] = v.y, c[2] = v.z, c[3] = v.w;
      }
      uint32_t mi, m;
      if (CAM) {
        m = boxw_cam(lo, hi, rf.inv, rf.neg, rf.tmax, rf.tmax_in, &mi);
      } else {
        float tn[kWide];
        m = boxw_f(lo, hi, rf, tn, &mi);
      }
      if (sp + kWide > kStack) {
        atomicOr(err, kErrStackOverflow);
        break;
      }
#pragma unroll
      for (int k = 0; k < kWide; ++k) {  // left to right: the rightmost is popped first
        // an empty slot's box (+inf, -inf) never passes the camera test; the
        // general test's error terms can turn it into NaN, which passes
        if (!((m >> k) & 1u) || (!CAM && c[k] == kWideEmpty)) continue;
        uint32_t e = c[k];
        if ((e & kWideLeaf) && (e & kLeafPure) && ((mi >> k) & 1u)) e |= kLeafVerified;
        stack[sp++] = e;
      }
    }
    if (sp == 0) break;
    const int p = --sp;
    cur = stack[p];
    stale = p < fresh;
    if (stale) fresh = p;
  }
  if (hit == kNoSlot) return false;
  *t_out = closest;
  *tri_out = sc.tris[hit].tri_id;
  return true;
}

__device__ RLC_COLD bool intersect_wide(const DevScene& sc, V3 o, V3 d, double tmin, bool camera,
                                        bool* used, double* t_out, uint32_t* tri_out,
                                        uint32_t* err) {
  static_assert(kWide == 4, "closest_wide loads 4-wide nodes");
  const Wide4* wn = camera ? sc.wide_cam : sc.wide_ref;
  const V3 inv{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
  const double ia[3] = {inv.x, inv.y, inv.z}, oa[3] = {o.x, o.y, o.z};
  bool ok = wn != nullptr && sc.fp32_ok;
  RayF rf;
  rf.neg = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ok &= fabs(ia[a]) <= 1e30;  // fp32-representable inverse: the decision bounds hold
    const float fi = float(ia[a]);
    rf.inv[a] = fi;
    if (camera) {  // camera-relative boxes: purely relative errors (box_decide_cam)
      rf.b[a] = 0.f;
      rf.mt[a] = 1e-30f;
    } else {
      const float of = float(oa[a]);
      rf.b[a] = -(of * fi);
      rf.mt[a] = fmaf(fabsf(of) * fabsf(fi), 0x1.0p-21f, 1e-30f);
    }
    rf.mb[a] = fabsf(fi) * 0x1.0p-22f;
    rf.neg |= (ia[a] < 0 ? 1u : 0u) << a;
  }
  *used = ok;
  if (!ok) return false;
  rf.fast = true;
  rf.tmin = __double2float_rd(tmin);
  rf.tmin_in = __double2float_ru(tmin);
  rf.tmax = HUGE_VALF;
  rf.tmax_in = HUGE_VALF;
  return camera ? closest_wide<true>(sc, wn, rf, o, d, inv, tmin, t_out, tri_out, err)
                : closest_wide<false>(sc, wn, rf, o, d, inv, tmin, t_out, tri_out, err);
}

// ---------------------------------------------------------------------------
// Closest hit on the quantized triangle-level SAH tree.  The
// reference's answer is the first triangle, in its leaf scan order, whose
// Moller-Trumbore t is smallest among the triangles its traversal reaches
// (leaf box passes the slab test against the running `closest`).  Let T1 be
// the triangle with the smallest MT t (t1) over ALL triangles, found here by
// any conservative traversal (every triangle with an MT hit below the
// running closest is reached: the same property k_shadow relies on), and
// assume no other triangle's MT t equals t1.  If T1's reference leaf passes
// the exact slab test against t1, then when the reference reaches that leaf
// its `closest` is > t1 (no tie), the test passes (monotone in t_max, and
// the ancestors passed earlier on larger boxes with a larger closest), T1 is
// accepted, and nothing after it can beat t1: the reference returns T1.
// Otherwise (the leaf test fails, or an exact tie) the answer depends on the
// reference's order and the caller runs the ordered traversal.  Nodes are
// culled against fl32_ru(closest); a triangle at t <= closest has a
// conservative box entry <= t, so ties are always seen.
// ---------------------------------------------------------------------------
#ifndef RLC_CLOSEST_SAH
#define RLC_CLOSEST_SAH 1
#endif
#ifndef RLC_SAH_STACK
#define RLC_SAH_STACK 32
#endif
constexpr int kSahStack = RLC_SAH_STACK;  // overflow: the ray is deferred to the ordered path

__device__ __forceinline__ bool tri_t(const TriAccel* tris, uint32_t i, V3 o, V3 d, double* tout) {
  const double2* p = reinterpret_cast<const double2*>(tris + i);
  const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), e = __ldg(p + 3),
                f = __ldg(p + 4);
  const V3 p0{a.x, a.y, b.x};
  const V3 e1{b.y, c.x, c.y};
  const V3 e2{e.x, e.y, f.x};
  const V3 pv = cross(d, e2);
  const double det = dot(e1, pv);
  const double inv_det = 1.0 / det;
  const V3 tv = o - p0;
  const double u = dot(tv, pv) * inv_det;
  const V3 qv = cross(tv, e1);
  const double v = dot(d, qv) * inv_det;
  *tout = dot(e2, qv) * inv_det;
  return !(fabs(det) < 1e-14) & !(u < 0 || u > 1) & !(v < 0 || u + v > 1);
}

__device__ int closest_sah(const DevScene& sc, V3 o, V3 d, double tmin, double* t_out,
                           uint32_t* tri_out) {
  if (!RLC_CLOSEST_SAH || sc.wide_q == nullptr || !sc.fp32_ok || sc.nodes_root_leaf) return 2;
  const V3 inv{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
  const double ia[3] = {inv.x, inv.y, inv.z}, oa[3] = {o.x, o.y, o.z};
  float finv[3], fb0[3];
  uint32_t neg = 0;
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ok &= fabs(ia[a]) <= 1e30;              // finite fp32 inverse (NaN, axis-parallel: no)
    ok &= fabs(oa[a]) <= sc.coord_bound;   // the padding bound of the shadow tree
    finv[a] = float(ia[a]);
    fb0[a] = -(float(oa[a]) * finv[a]);
    neg |= (ia[a] < 0 ? 1u : 0u) << a;
  }
  if (!ok) return 2;
  const float tmin_f = __double2float_rd(tmin);
  double closest = HUGE_VAL;
  float tmax_f = HUGE_VALF;
  uint32_t hit = kNoSlot;
  bool tie = false;
  uint32_t stk_e[kSahStack];
  float stk_t[kSahStack];
  int sp = 0;
  uint32_t cur = 0;
  uint32_t st_nodes = 0, st_tris = 0;
  while (true) {
    if (!(cur & kWideLeaf)) {
      ++st_nodes;
      const uint4* p = reinterpret_cast<const uint4*>(sc.wide_q + cur);
      const uint4 w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2), w3 = __ldg(p + 3);
      const uint32_t ql[3] = {w1.x, w1.y, w1.z}, qh[3] = {w1.w, w2.x, w2.y};
      const float org[3] = {__uint_as_float(w0.x), __uint_as_float(w0.y), __uint_as_float(w0.z)};
      uint32_t c[kWide] = {w2.z, w2.w, w3.x, w3.y};
      float A[3], B[3];
      uint32_t nw[3], fw[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const bool ng = (neg >> a) & 1u;
        nw[a] = ng ? qh[a] : ql[a];
        fw[a] = ng ? ql[a] : qh[a];
        A[a] = __uint_as_float(((w0.w >> (8 * a)) & 255u) << 23) * finv[a];
        B[a] = fmaf(org[a], finv[a], fb0[a]);
      }
      float tn[kWide];
      uint32_t m = 0;
#pragma unroll
      for (int k = 0; k < kWide; ++k) {
        float n3[3], f3[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          n3[a] = fmaf(float((nw[a] >> (8 * k)) & 255u), A[a], B[a]);
          f3[a] = fmaf(float((fw[a] >> (8 * k)) & 255u), A[a], B[a]);
        }
        tn[k] = fmaxf(fmax3(tmin_f, n3[0], n3[1]), n3[2]);
        const float fk = fminf(fmin3(tmax_f, f3[0], f3[1]), f3[2]);
        const bool pass = tn[k] <= fk && ((w3.z >> k) & 1u);  // w3.z: non-empty children
        m |= pass ? (1u << k) : 0u;
        if (!pass) tn[k] = HUGE_VALF;
      }
#define RLC_CSWAP(i, j)                                   \
  if (tn[j] < tn[i]) {                                    \
    const float tt = tn[i]; tn[i] = tn[j]; tn[j] = tt;    \
    const uint32_t cc = c[i]; c[i] = c[j]; c[j] = cc;     \
  }
      RLC_CSWAP(0, 1) RLC_CSWAP(2, 3) RLC_CSWAP(0, 2) RLC_CSWAP(1, 3) RLC_CSWAP(1, 2)
#undef RLC_CSWAP
      const int hits = __popc(m);
      if (hits > 0) {
        if (sp + hits - 1 > kSahStack) return 2;
#pragma unroll
        for (int k = kWide - 1; k >= 1; --k)
          if (k < hits) {
            stk_e[sp] = c[k];
            stk_t[sp] = tn[k];
            ++sp;
          }
        cur = c[0];
        continue;
      }
    } else {
      const uint32_t first = leaf_first(cur), cnt = leaf_count(cur);
      st_tris += cnt;
      for (uint32_t i = first; i < first + cnt; ++i) {
        double t;
        if (tri_t(sc.tris_s, i, o, d, &t) && !(t <= tmin)) {
          if (t < closest) {
            closest = t;
            hit = i;
            tie = false;
            tmax_f = __double2float_ru(closest);
          } else if (!(t > closest)) {
            tie = true;  // an exact tie (or NaN): the reference's order decides
          }
        }
      }
    }
    bool found = false;
    while (sp > 0) {
      --sp;
      if (stk_t[sp] <= tmax_f) {
        cur = stk_e[sp];
        found = true;
        break;
      }
    }
    if (!found) break;
  }
  RLC_STAT(3, 1);
  RLC_STAT(4, st_nodes);
  RLC_STAT(5, st_tris);
  if (hit == kNoSlot) return 0;
  if (tie) {
    RLC_STAT(7, 1);  // deferred to the reference-order traversal: an exact tie
    return 2;
  }
  if (!box_hit(load_node(sc.nodes, __ldg(sc.tri_leaf_s + hit)), o, inv, tmin, closest)) {
    RLC_STAT(7, 1);  // deferred: the reference's own box test misses the hit's leaf
    return 2;
  }
  *t_out = closest;
  *tri_out = sc.tris_s[hit].tri_id;
  return 1;
}

__device__ __forceinline__ bool tri_any(const TriAccel* tris, uint32_t i, V3 o, V3 d, double tmin,
                                        double tmax) {
  const double2* p = reinterpret_cast<const double2*>(tris + i);
  const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), e = __ldg(p + 3),
                f = __ldg(p + 4);
  const V3 p0{a.x, a.y, b.x};
  const V3 e1{b.y, c.x, c.y};
  const V3 e2{e.x, e.y, f.x};
  const V3 pv = cross(d, e2);
  const double det = dot(e1, pv);
  const double inv_det = 1.0 / det;
  const V3 tv = o - p0;
  const double u = dot(tv, pv) * inv_det;
  const V3 qv = cross(tv, e1);
  const double v = dot(d, qv) * inv_det;
  const double t = dot(e2, qv) * inv_det;
  return !(fabs(det) < 1e-14) & !(u < 0 || u > 1) & !(v < 0 || u + v > 1) &
         !(t <= tmin || t >= tmax);
}

// nee_estimate returns the zero result (estimators.cpp:95)
__device__ __forceinline__ void mark_occluded(uint8_t* rflag, double* vdense, uint32_t idx) {
  vdense[idx] = 0.0;
  rflag[idx] |= kROccluded;
}

// Any-hit traversal of the queued shadow segments (occluded(), bvh.cpp:
// 159-188).  Persistent warps refill idle lanes from the queue after every
// leaf round.  Node steps and leaf tests are separated ("while-while") and a
// lane that reaches a leaf postpones it while other lanes still have node
// steps to do (speculative traversal, Aila & Laine 2009), so both phases run
// with as many lanes as possible.
#ifndef RLC_SHADOW_BLOCKS
#define RLC_SHADOW_BLOCKS 8  // blocks per SM (64 registers) with the 12-entry stack: c3 1.058 -> 1.045 ms (c5: 16.4 -> 16.8 ms; 7 was best with 32 entries)
#endif
template <bool QUANT, bool COUNT>
__global__ void __launch_bounds__(kShadowThreads, RLC_SHADOW_BLOCKS) k_shadow(DevScene sc,
                                                           const ShadowRay* __restrict__ rays,
                                                           const uint32_t* __restrict__ order,
                                                           unsigned int* __restrict__ ray_count,
                                                           uint8_t* __restrict__ rflag,
                                                           double* __restrict__ vdense,
                                                           unsigned int* __restrict__ err) {
  const uint32_t lane = threadIdx.x & 31u;
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned n = *reinterpret_cast<volatile unsigned*>(ray_count);
  const double tmin = sc.shadow_eps;
  bool active = false;
  bool exhausted = false;
  V3 o{0, 0, 0}, d{0, 0, 0}, inv{0, 0, 0};
  RayF rf;
  double tmax = 0;
  uint32_t idx = 0;
  uint32_t leaf = 0;    // postponed leaf entry (0: none)
  uint32_t cur = kDone; // current entry: Wide4 index, leaf entry, or kDone
  bool overflow = false; // the stack overflowed: the exact path decides
  const int stack_limit = sc.shadow_stack_limit ? min(kShadowStack, int(sc.shadow_stack_limit))
                                                : kShadowStack;
  // per-lane traversal stack in shared memory, [depth][thread]: conflict-free
  __shared__ uint32_t stack_mem[kShadowStack * kShadowThreads];
  uint32_t* stack = stack_mem + threadIdx.x;
  int sp = 0;
  uint32_t w_rays = 0, w_nodes = 0, w_tris = 0;  // g_work (COUNT instances only)
#define RLC_WORK(x) \
  if constexpr (COUNT) (x)
  while (true) {
    const unsigned need = __ballot_sync(kFull, !active);
    if (need && !exhausted) {
      const int leader = __ffs(need) - 1;
      unsigned base = 0;
      if (int(lane) == leader) base = atomicAdd(ray_count + 1, unsigned(__popc(need)));
      base = __shfl_sync(kFull, base, leader);
      if (base + __popc(need) >= n) exhausted = true;
      if (!active) {
        const unsigned my = base + __popc(need & lt_mask);
        if (my < n) {
          const ShadowRay r = rays[order ? __ldg(order + my) : my];
          o = V3{r.o[0], r.o[1], r.o[2]};
          d = V3{r.d[0], r.d[1], r.d[2]};
          inv = V3{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
          tmax = r.tmax;
          idx = r.idx;
          sp = 0;
          leaf = 0;
          overflow = false;
          const NodeView root = load_node(sc.nodes, 0);
          if (box_hit(root, o, inv, tmin, tmax)) {  // the reference tests the root first
            const double ia[3] = {inv.x, inv.y, inv.z}, oa[3] = {o.x, o.y, o.z};
            bool exact = root.count > 0 || !sc.fp32_ok;
            double maxinv = 0;
            rf.neg = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              exact |= fabs(ia[a]) > 1e30 && isfinite(ia[a]);
              exact |= !(fabs(oa[a]) <= sc.coord_bound);  // origin outside the padding bound
              const float of = float(oa[a]), fi = float(ia[a]);
              rf.inv[a] = fi;
              rf.b[a] = -(of * fi);
              rf.neg |= (ia[a] < 0 ? 1u : 0u) << a;
              maxinv = fmax(maxinv, fabs(ia[a]));
            }
            rf.margin = __double2float_ru(sc.coord_bound * maxinv * 0x1.0p-19) + 1e-30f;
            rf.tmin = __double2float_rd(tmin);
            rf.tmax = __double2float_ru(tmax);
            rf.tmin_in = __double2float_ru(tmin);
            rf.tmax_in = __double2float_rd(tmax);
            if (exact) {  // tiny scene or fp32-range ray: the exact fp64 path
              if (occluded_ray(sc, o, d, inv, tmin, tmax, err)) mark_occluded(rflag, vdense, idx);
            } else {
              cur = 0;
              active = true;
              RLC_WORK(++w_rays);
              RLC_STAT(0, 1);
            }
          }
        }
      }
    }
    if (!__any_sync(kFull, active)) {
      if (exhausted) break;
      continue;
    }
    if (!active) continue;
    // node phase: descend through internal nodes with the current node in a
    // register; the first leaf met is postponed and traversal continues
    // while some lane of the warp has not found a leaf yet
    while (cur != kDone && !(cur & kWideLeaf)) {
      RLC_WORK(++w_nodes);
      RLC_STAT(1, 1);
      float tn[kWide];
      uint32_t mi, m;
      uint32_t c[kWide];
      if constexpr (QUANT) {  // 64-byte quantized node: no inner test (leaves checked exactly)
        const uint4* p = reinterpret_cast<const uint4*>(sc.wide_q + cur);
        const uint4 w0 = __ldg(p), w1 = __ldg(p + 1), w2 = __ldg(p + 2), w3 = __ldg(p + 3);
        const uint32_t ql[3] = {w1.x, w1.y, w1.z}, qh[3] = {w1.w, w2.x, w2.y};
        const float org[3] = {__uint_as_float(w0.x), __uint_as_float(w0.y), __uint_as_float(w0.z)};
        c[0] = w2.z, c[1] = w2.w, c[2] = w3.x, c[3] = w3.y;
        float A[3], B[3];
        uint32_t nw[3], fw[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const bool ng = (rf.neg >> a) & 1u;
          nw[a] = ng ? qh[a] : ql[a];
          fw[a] = ng ? ql[a] : qh[a];
          A[a] = __uint_as_float(((w0.w >> (8 * a)) & 255u) << 23) * rf.inv[a];
          B[a] = fmaf(org[a], rf.inv[a], rf.b[a]);
        }
        float nb[kWide], fb[kWide];
#pragma unroll
        for (int k = 0; k < kWide; ++k) {
          float tn[3], tf[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            tn[a] = fmaf(float((nw[a] >> (8 * k)) & 255u), A[a], B[a]);
            tf[a] = fmaf(float((fw[a] >> (8 * k)) & 255u), A[a], B[a]);
          }
          nb[k] = fmaxf(fmax3(rf.tmin, tn[0], tn[1]), tn[2]);
          fb[k] = fminf(fmin3(rf.tmax, tf[0], tf[1]), tf[2]);
        }
        m = 0;
#pragma unroll
        for (int k = 0; k < kWide; ++k) {
          const bool pass = nb[k] <= fb[k];
          m |= pass ? (1u << k) : 0u;
          tn[k] = pass ? nb[k] : HUGE_VALF;
        }
        m &= w3.z;  // non-empty children
        mi = 0;
      } else {
        constexpr int Q = kWide / 4;  // float4 per [axis] row
        const float4* p = reinterpret_cast<const float4*>(sc.wide + cur);
        float lo[3][kWide], hi[3][kWide];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const float4 vl = __ldg(p + a * Q + q), vh = __ldg(p + (3 + a) * Q + q);
            lo[a][4 * q] = vl.x, lo[a][4 * q + 1] = vl.y, lo[a][4 * q + 2] = vl.z, lo[a][4 * q + 3] = vl.w;
            hi[a][4 * q] = vh.x, hi[a][4 * q + 1] = vh.y, hi[a][4 * q + 2] = vh.z, hi[a][4 * q + 3] = vh.w;
          }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(p + 6 * Q + q));
          c[4 * q] = v.x, c[4 * q + 1] = v.y, c[4 * q + 2] = v.z, c[4 * q + 3] = v.w;
        }
        m = boxw_s(lo, hi, rf, tn, &mi);
      }
      if constexpr (!QUANT) {
#pragma unroll
        for (int k = 0; k < kWide; ++k) {
          if (c[k] == kWideEmpty) m &= ~(1u << k);
          if (((mi >> k) & (c[k] >> 31)) && (c[k] & kLeafPure))
            c[k] |= kLeafVerified;  // leaf proven reached
          if (!(m & (1u << k))) tn[k] = HUGE_VALF;
        }
      }
      if (sp + kWide - 1 > stack_limit) {  // finish this ray on the exact path
        overflow = true;
        m = 0;
        sp = 0;
      }
      // nearest entry first: occluders near the shading point end the ray early
#define RLC_CSWAP(i, j)                                   \
  if (tn[j] < tn[i]) {                                    \
    const float tt = tn[i]; tn[i] = tn[j]; tn[j] = tt;    \
    const uint32_t cc = c[i]; c[i] = c[j]; c[j] = cc;     \
  }
      if constexpr (kWide == 4) {
        RLC_CSWAP(0, 1) RLC_CSWAP(2, 3) RLC_CSWAP(0, 2) RLC_CSWAP(1, 3) RLC_CSWAP(1, 2)
      } else {  // Batcher's 8-input network, 19 comparators
        RLC_CSWAP(0, 1) RLC_CSWAP(2, 3) RLC_CSWAP(4, 5) RLC_CSWAP(6, 7)
        RLC_CSWAP(0, 2) RLC_CSWAP(1, 3) RLC_CSWAP(4, 6) RLC_CSWAP(5, 7)
        RLC_CSWAP(1, 2) RLC_CSWAP(5, 6) RLC_CSWAP(0, 4) RLC_CSWAP(3, 7)
        RLC_CSWAP(1, 5) RLC_CSWAP(2, 6)
        RLC_CSWAP(1, 4) RLC_CSWAP(3, 6)
        RLC_CSWAP(2, 4) RLC_CSWAP(3, 5)
        RLC_CSWAP(3, 4)
      }
#undef RLC_CSWAP
      const int hits = __popc(m);
      if (hits == 0) {
        cur = sp > 0 ? stack[(--sp) * kShadowThreads] : kDone;
      } else {
        cur = c[0];
#pragma unroll
        for (int k = kWide - 1; k >= 1; --k)
          if (k < hits) stack[(sp++) * kShadowThreads] = c[k];
      }
      if (leaf == 0 && cur != kDone && (cur & kWideLeaf)) {
        leaf = cur;
        cur = sp > 0 ? stack[(--sp) * kShadowThreads] : kDone;
      }
      if (!__any_sync(__activemask(), leaf == 0)) break;
    }
    // leaf phase: exact fp64 Moller-Trumbore on the postponed leaf and on
    // every leaf that follows it directly, then the exact ancestor chain
    bool hit = false;
    while (leaf != 0) {
      const uint32_t first = leaf_first(leaf), cnt = leaf_count(leaf);
      RLC_WORK(w_tris += cnt);
      RLC_STAT(2, cnt);
      if (leaf & kLeafPure) {  // one reference leaf: one exact test for the leaf
        for (uint32_t i = first; i < first + cnt; ++i)
          hit |= tri_any(sc.tris_s, i, o, d, tmin, tmax);
        if (hit) hit = leaf_reached(sc, leaf, o, inv, tmin, tmax);
      } else {  // a refitted leaf spanning reference leaves: test each hit's own
        for (uint32_t i = first; i < first + cnt && !hit; ++i)
          hit = tri_any(sc.tris_s, i, o, d, tmin, tmax) &&
                box_hit(load_node(sc.nodes, __ldg(sc.tri_leaf_s + i)), o, inv, tmin, tmax);
      }
      if (hit) break;
      if (cur != kDone && (cur & kWideLeaf)) {
        leaf = cur;
        cur = sp > 0 ? stack[(--sp) * kShadowThreads] : kDone;
      } else {
        leaf = 0;
      }
    }
    if (hit) {
      mark_occluded(rflag, vdense, idx);
      active = false;
    } else if (cur == kDone && leaf == 0) {
      if (overflow) {  // rare: the whole segment again, exactly as the reference
        RLC_STAT(6, 1);
        if (occluded_ray(sc, o, d, inv, tmin, tmax, err)) mark_occluded(rflag, vdense, idx);
        overflow = false;
      }
      active = false;
    }
  }
  if constexpr (!COUNT) return;
  const uint32_t r = __reduce_add_sync(kFull, w_rays), nd = __reduce_add_sync(kFull, w_nodes),
                 tr = __reduce_add_sync(kFull, w_tris);
  if (lane == 0) {
    atomicAdd(&g_work[0], (unsigned long long)r);
    atomicAdd(&g_work[1], (unsigned long long)nd);
    atomicAdd(&g_work[2], (unsigned long long)tr);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_work[3], (unsigned long long)n);
  }
}

// ---------------------------------------------------------------------------
// stable LSD radix sort of (key, val) pairs, 8-bit digits
// ---------------------------------------------------------------------------
// Block size of the record sort.  Sort blocks that fit in the registers the
// 7 shadow blocks per SM leave (8,192: 128 threads x <= 64) run beside
// k_shadow and take its issue slots; 256-thread blocks with 16 keys per
// thread (102 registers) mostly wait for the shadow blocks to retire, and the
// frame is shorter: c3 1.038 vs 1.076 ms per frame, same box.
#ifndef RLC_RS_THREADS
#define RLC_RS_THREADS 256
#endif
#ifndef RLC_RS_MINB
#define RLC_RS_MINB 1  // (8 with 128 threads: rs_scatter at <= 64 registers, beside k_shadow)
#endif
constexpr int kRsThreads = RLC_RS_THREADS;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsItems = int(kSortTile) / kRsThreads;  // per thread

// Tiles of ITEMS keys per thread over the n valid keys (n_dev: a device-side
// count); the per-block digit histograms are laid out [digit][tile].
template <int ITEMS>
__device__ __forceinline__ uint32_t rs_tiles(uint32_t& n, const unsigned* n_dev) {
  if (n_dev) n = min(n, *n_dev);
  constexpr uint32_t tile = kRsThreads * ITEMS;
  return n_dev ? (n + tile - 1) / tile : gridDim.x;
}

template <int ITEMS>
__global__ void __launch_bounds__(kRsThreads) rs_hist(const uint32_t* __restrict__ keys,
                                                      uint32_t n, const unsigned* __restrict__ n_dev,
                                                      int shift, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[256];
  const uint32_t nt = rs_tiles<ITEMS>(n, n_dev);
  if (blockIdx.x >= nt) return;
  for (int d = threadIdx.x; d < 256; d += kRsThreads) h[d] = 0;
  __syncthreads();
  const uint32_t base = blockIdx.x * kRsThreads * ITEMS;
  uint32_t kk[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t j = base + i * kRsThreads + threadIdx.x;
    kk[i] = j < n ? __ldg(keys + j) : 0u;
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t j = base + i * kRsThreads + threadIdx.x;
    if (j < n) atomicAdd(&h[(kk[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += kRsThreads) hist[d * nt + blockIdx.x] = h[d];
}

// Exclusive scan of `total` counters in place, one block of kScanThreads
// (sized to fit beside k_shadow, see kRsThreads).
constexpr uint32_t kScanThreads = 256;
__global__ void __launch_bounds__(kScanThreads) rs_scan(uint32_t* __restrict__ hist, uint32_t total) {
  __shared__ uint32_t warp_sums[32];
  const uint32_t t = threadIdx.x;
  const uint32_t per = (total + kScanThreads - 1u) / kScanThreads;
  const uint32_t b = t * per, e = min(total, b + per);
  uint32_t sum = 0;
  for (uint32_t i = b; i < e; ++i) sum += hist[i];
  // block exclusive scan of `sum`
  uint32_t x = sum;
  const uint32_t lane = t & 31u, w = t >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= uint32_t(o)) x += y;
  }
  if (lane == 31) warp_sums[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t ws = lane < kScanThreads / 32 ? warp_sums[lane] : 0u;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, ws, o);
      if (lane >= uint32_t(o)) ws += y;
    }
    warp_sums[lane] = ws;
  }
  __syncthreads();
  uint32_t run = x - sum + (w > 0 ? warp_sums[w - 1] : 0u);
  for (uint32_t i = b; i < e; ++i) {
    const uint32_t v = hist[i];
    hist[i] = run;
    run += v;
  }
}

// Exclusive scan of one digit's row of per-block counts (hist[d][0..nb)) in
// place; the digit total goes to totals[d].  One block per digit.
template <int ITEMS>
__global__ void __launch_bounds__(256) rs_scan_rows(uint32_t* __restrict__ hist, uint32_t nb,
                                                    uint32_t n, const unsigned* __restrict__ n_dev,
                                                    uint32_t* __restrict__ totals) {
  __shared__ uint32_t ws[8];
  if (n_dev) {  // the tiles of the device count (rs_tiles)
    n = min(n, *n_dev);
    nb = (n + kRsThreads * ITEMS - 1) / (kRsThreads * ITEMS);
  }
  uint32_t* row = hist + size_t(blockIdx.x) * nb;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < nb; base += 256) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < nb ? row[i] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= uint32_t(o)) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (uint32_t q = 0; q < 8; ++q) {
      before += q < w ? ws[q] : 0u;
      total += ws[q];
    }
    if (i < nb) row[i] = carry + before + x - v;
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

template <int ITEMS>
__global__ void __launch_bounds__(kRsThreads, RLC_RS_MINB) rs_scatter(const uint32_t* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin,
                                                         uint32_t* __restrict__ kout,
                                                         uint32_t* __restrict__ vout,
                                                         uint32_t n, const unsigned* __restrict__ n_dev,
                                                         int shift,
                                                         const uint32_t* __restrict__ offs,
                                                         const uint32_t* __restrict__ totals) {
  __shared__ uint32_t wh[kRsWarps][256];
  const uint32_t nt = rs_tiles<ITEMS>(n, n_dev);
  if (blockIdx.x >= nt) return;
  __shared__ uint32_t base_off[256];
  __shared__ uint32_t dsum[kRsWarps];
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  for (int d = lane; d < 256; d += 32) wh[w][d] = 0;
  {  // digit base = exclusive prefix of the digit totals, + this block's row offset
    // (kDpt consecutive digits per thread)
    constexpr uint32_t kDpt = 256 / kRsThreads;
    static_assert(kDpt * kRsThreads == 256, "256 digits over the block");
    const uint32_t d0 = kDpt * threadIdx.x;
    uint32_t tl[kDpt], mine = 0;
#pragma unroll
    for (uint32_t j = 0; j < kDpt; ++j) {
      tl[j] = totals[d0 + j];
      mine += tl[j];
    }
    uint32_t x = mine;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= uint32_t(o)) x += y;
    }
    if (lane == 31) dsum[w] = x;
    __syncthreads();
    uint32_t run = x - mine;
    for (uint32_t q = 0; q < w; ++q) run += dsum[q];
#pragma unroll
    for (uint32_t j = 0; j < kDpt; ++j) {
      base_off[d0 + j] = run + offs[(d0 + j) * nt + blockIdx.x];
      run += tl[j];
    }
  }
  __syncwarp();
  const uint32_t base = blockIdx.x * (kRsThreads * ITEMS) + w * (32 * ITEMS);
  const unsigned lt_mask = (1u << lane) - 1u;
  uint32_t k[ITEMS], v[ITEMS], rank[ITEMS];
  // all of the tile's loads in flight before the ranking (the warp-level
  // ranking's __syncwarp would otherwise serialise one load latency per item)
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint32_t j = base + r * 32 + lane;
    const bool ok = j < n;
    k[r] = ok ? __ldg(kin + j) : 0u;
    v[r] = ok ? (vin ? __ldg(vin + j) : j) : 0u;  // vin null: the identity (vertex ids)
  }
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint32_t j = base + r * 32 + lane;
    const bool ok = j < n;
    const uint32_t d = ok ? (k[r] >> shift) & 255u : 256u + lane;
    const unsigned peers = __match_any_sync(kFull, d);
    const uint32_t before = ok ? wh[w][d] : 0u;
    rank[r] = before + __popc(peers & lt_mask);
    __syncwarp();
    if (ok && (peers & lt_mask) == 0) wh[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < 256; d += kRsThreads) {  // cross-warp exclusive prefix per digit
    uint32_t run = 0;
    for (int ww = 0; ww < kRsWarps; ++ww) {
      const uint32_t c = wh[ww][d];
      wh[ww][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint32_t j = base + r * 32 + lane;
    if (j < n) {
      const uint32_t d = (k[r] >> shift) & 255u;
      const uint32_t pos = base_off[d] + wh[w][d] + rank[r];
      kout[pos] = k[r];
      vout[pos] = v[r];
    }
  }
}

// ---------------------------------------------------------------------------
// k_fold: update_q (cut.cpp:76-86) applied per (cell, cluster) segment in
// canonical order; q_before feeds the deferred radiance.
// ---------------------------------------------------------------------------
// v of record `idx` is at vbase + idx * vstride (sample records or exchanged
// update records); q_before is written per record index, and with seg_n the
// segment's record count at its last record index.
// SEG: 0 the single-GPU fold; 1 (owner mode, per-slot exchange) the
// segment's record count at its last record's index into seg_n; 2 (owner
// mode, per-entry exchange) the entry's final q and record count into
// ent_q / ent_n.
template <int SEG>
__global__ void __launch_bounds__(256) k_fold(DevGrid g, PassParams P,
                                              const uint32_t* __restrict__ keys,
                                              const uint32_t* __restrict__ vals,
                                              const char* __restrict__ vbase, uint32_t vstride,
                                              double* __restrict__ q_before,
                                              const unsigned* __restrict__ n_dev,
                                              uint32_t* __restrict__ seg_n,
                                              double* __restrict__ ent_q = nullptr,
                                              uint32_t* __restrict__ ent_n = nullptr) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (n_dev) P.n = min(P.n, *n_dev);
  if (i >= P.n) return;
  const uint32_t k = keys[i];
  if (k == kInvalidKey) return;
  if (i > 0 && keys[i - 1] == k) return;
  const uint32_t cell = k / g.M;
  RLC_CHECK(cell < g.capacity && cell < uint32_t(g.counters[kCntCells]),
            g.counters + kCntErr);
  const size_t at = size_t(k);
  double q = g.q[at];
  uint32_t vis = g.visits[at];
  // The update chain is sequential (bit-exact order); the record loads are
  // not, so they are issued kBatch at a time ahead of the arithmetic.
  constexpr int kBatch = 8;
  uint32_t j = i, last = 0;
  while (true) {
    uint32_t ids[kBatch];
    int cnt = 0;
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const uint32_t jj = j + b;
      const bool in = cnt == b && jj < P.n && keys[jj] == k;
      if (in) {
        ids[b] = vals[jj];
        ++cnt;
      }
    }
    if (cnt == 0) break;
    double vb[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
      if (b < cnt) vb[b] = *reinterpret_cast<const double*>(vbase + size_t(ids[b]) * vstride);
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      if (b >= cnt) break;
      const double v = vb[b];
      if (!(v >= 0 && isfinite(v)))  // update_q's argument check, cut.cpp:78-80
        atomicOr(reinterpret_cast<unsigned int*>(g.counters + kCntErr), kErrBadValue);
      q_before[ids[b]] = q;
      const double a = P.harmonic ? 1.0 / (1.0 + double(vis)) : P.alpha;
      q = smax((1.0 - a) * q + a * v, g.eps_q);
      ++vis;
      if constexpr (SEG == 1) last = ids[b];
    }
    j += uint32_t(cnt);
    if (cnt < kBatch) break;
  }
  if constexpr (SEG == 1) seg_n[last] = j - i;
  if constexpr (SEG == 2) {  // indexed by table slot: dense cell ids differ between ranks
    const size_t ent = size_t(g.cell_slot[cell]) * g.M + (k - cell * g.M);
    ent_q[ent] = q;
    ent_n[ent] = j - i;
  }
  g.q[at] = q;
  g.visits[at] = vis;
  g.touched[cell] = 1u;
}

// ---------------------------------------------------------------------------
// k_accumulate: deferred radiance (estimators.cpp:100-101 with the live
// q_before of sample_cluster, cut.cpp:105) + Framebuffer::add_sample
// (image.hpp:56-60) in per-pixel sample order.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_accumulate(DevScene sc, PassParams P,
                                                    const uint32_t* __restrict__ gflags,
                                                    const SampleRec* __restrict__ srec,
                                                    const uint8_t* __restrict__ rflag,
                                                    const double* __restrict__ q_before,
                                                    Framebuf fb) {
  const uint32_t pix = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t npix = P.n / P.spp_pp;
  if (pix >= npix) return;
  const uint32_t px = pix % P.width;
  const uint32_t py = P.row_begin + pix / P.width;
  const size_t fi = size_t(py) * P.width + px;
  V3 sum = ld3(fb.sum + 3 * fi);
  unsigned long long cnt = fb.count[fi];
  for (uint32_t s = 0; s < P.spp_pp; ++s) {
    // radiance of PassRenderer::trace (render.cpp:64-137): emission of the
    // primary hit, then throughput-weighted NEE of every reflective vertex
    V3 L{0.0, 0.0, 0.0};
    V3 T{1.0, 1.0, 1.0};
    const size_t v0 = size_t(pix * P.spp_pp + s) * P.depth;
    for (uint32_t d = 0; d < P.depth; ++d) {
      const size_t idx = v0 + d;
      const uint32_t flags = gflags[idx];
      if (!(flags & kGHit)) break;
      const MatRec& m = sc.mats[flags & kGMatMask];
      if (flags & kGEmit) L = L + ld3(m.emission);
      if (!(flags & kGReflective)) break;
      V3 rad{0.0, 0.0, 0.0};
      const uint8_t rf = rflag[idx];  // the sample record only for a visible contribution
      if ((rf & kSNonzero) && !(rf & kROccluded)) {
        const SampleRec r = ldg_vec(srec + idx);
        double pdf_sel;
        if ((r.flags & kSLearned) && !(r.flags & kSFrozen)) {
          const double p = q_before[idx] / r.total;
          pdf_sel = p * r.pin;
        } else {
          pdf_sel = r.pin;
        }
        const double den = pdf_sel * r.pdf_area;
        rad = V3{r.c[0], r.c[1], r.c[2]} / den;
      }
      L = L + T * rad;
      T = T * ld3(m.albedo);  // used only if vertex d + 1 exists (render.cpp:133)
    }
    sum = sum + L;
    cnt += 1;
  }
  fb.sum[3 * fi] = sum.x;
  fb.sum[3 * fi + 1] = sum.y;
  fb.sum[3 * fi + 2] = sum.z;
  fb.count[fi] = cnt;
}

// ---------------------------------------------------------------------------
// k_split: split_collapse (cut.cpp:119-190) + rebuild_ends for every
// touched cell (render.cpp:185-200), one warp per cell, cut rows staged in
// shared memory; then the serial rebuild_cdf, one lane per cell.
// ---------------------------------------------------------------------------
struct WarpArg {
  double val;
  uint32_t idx;  // kNoSlot = none
};

// max val, lowest index on ties (cut.cpp:125-131: strict '>' scanning up)
__device__ __forceinline__ WarpArg warp_argmax(WarpArg a) {
  for (int o = 16; o > 0; o >>= 1) {
    WarpArg b;
    b.val = __shfl_xor_sync(kFull, a.val, o);
    b.idx = __shfl_xor_sync(kFull, a.idx, o);
    if (b.idx != kNoSlot &&
        (a.idx == kNoSlot || b.val > a.val || (b.val == a.val && b.idx < a.idx)))
      a = b;
  }
  return a;
}
// min val, lowest index on ties (cut.cpp:146-151: strict '<' scanning up)
__device__ __forceinline__ WarpArg warp_argmin(WarpArg a) {
  for (int o = 16; o > 0; o >>= 1) {
    WarpArg b;
    b.val = __shfl_xor_sync(kFull, a.val, o);
    b.idx = __shfl_xor_sync(kFull, a.idx, o);
    if (b.idx != kNoSlot &&
        (a.idx == kNoSlot || b.val < a.val || (b.val == a.val && b.idx < a.idx)))
      a = b;
  }
  return a;
}

// The cdf row of a cell from its q row (rebuild_cdf, cut.cpp:88-95).
__device__ __forceinline__ void cdf_row(const DevGrid& g, uint32_t cell) {
  const uint32_t M = g.M;
  const size_t row = size_t(cell) * M;
  double run = 0;
  if ((M & 1u) == 0) {  // rows of 16-byte pairs
    const double2* q2 = reinterpret_cast<const double2*>(g.q + row);
    double2* c2 = reinterpret_cast<double2*>(g.cdf + row);
#pragma unroll 8
    for (uint32_t i = 0; i < M / 2; ++i) {
      const double2 v = q2[i];
      run += v.x;
      const double a = run;
      run += v.y;
      c2[i] = make_double2(a, run);
    }
  } else {
    for (uint32_t i = 0; i < M; ++i) {
      run += g.q[row + i];
      g.cdf[row + i] = run;
    }
  }
}

template <bool GLOBAL_ROWS>
__global__ void k_split(DevScene sc, DevGrid g, double threshold, uint32_t iterations,
                        uint32_t* changes_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t wpb = blockDim.x >> 5;
  const uint32_t M = g.M;
  // per warp: qA, qB (double), nA, nB, vA, vB (u32) -- in shared memory, or
  // for cuts too large for it in the grid's global scratch (same arithmetic)
  // (a compile-time choice, so shared-memory rows use shared-memory accesses)
  unsigned char* base = GLOBAL_ROWS
                            ? g.split_scratch + size_t(blockIdx.x * wpb + wib) * 32 * size_t(M)
                            : smem + size_t(wib) * 16 * size_t(M);
  double* qA = reinterpret_cast<double*>(base);
  double* qB = qA + M;
  uint32_t* nA = GLOBAL_ROWS
                     ? reinterpret_cast<uint32_t*>(qB + M)
                     : reinterpret_cast<uint32_t*>(smem + size_t(wpb) * 16 * size_t(M)) +
                           size_t(wib) * 4 * M;
  uint32_t* nB = nA + M;
  uint32_t* vA = nB + M;
  uint32_t* vB = vA + M;
  const uint32_t ncells = uint32_t(*reinterpret_cast<volatile unsigned long long*>(g.counters + kCntCells));
  const double eps = g.eps_q;
  uint32_t my_changes = 0;
  for (uint32_t cell = blockIdx.x * wpb + wib; cell < ncells; cell += gridDim.x * wpb) {
    if (!g.touched[cell]) continue;  // warp-uniform
    const size_t row = size_t(cell) * M;
    for (uint32_t i0 = 0; i0 < M; i0 += 128) {  // all of a chunk's loads in flight first
      double qv[4];
      uint32_t nv[4], vv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t i = i0 + lane + 32u * k;
        if (i < M) {
          qv[k] = __ldcg(g.q + row + i);
          nv[k] = __ldcg(g.node_ids + row + i);
          vv[k] = __ldcg(g.visits + row + i);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t i = i0 + lane + 32u * k;
        if (i < M) {
          qA[i] = qv[k];
          nA[i] = nv[k];
          vA[i] = vv[k];
        }
      }
    }
    __syncwarp();
    const uint32_t changes_before = my_changes;
    for (uint32_t it = 0; it < iterations; ++it) {
      WarpArg sp{0.0, kNoSlot};
      for (uint32_t i = lane; i < M; i += 32) {
        if (sc.lt[nA[i]].left < 0) continue;   // tree leaf: unsplittable
        if (qA[i] * 0.5 < eps) continue;       // halves would fall below the floor
        if (sp.idx == kNoSlot || qA[i] > sp.val) sp = WarpArg{qA[i], i};
      }
      sp = warp_argmax(sp);
      if (sp.idx == kNoSlot) break;
      const uint32_t split_at = sp.idx;
      // Collapse candidates: adjacent leaves with a common parent.  The
      // parent is a proper ancestor of the split leaf iff the split leaf is
      // one of the pair (cut leaves are disjoint ranges), cut.cpp:133-145.
      WarpArg cp{0.0, kNoSlot};
      for (uint32_t i = lane; i + 1 < M; i += 32) {
        const int32_t pa = sc.lt[nA[i]].parent;
        if (pa < 0 || pa != sc.lt[nA[i + 1]].parent) continue;
        if (i == split_at || i + 1 == split_at) continue;
        const double mass = qA[i] + qA[i + 1];
        if (cp.idx == kNoSlot || mass < cp.val) cp = WarpArg{mass, i};
      }
      cp = warp_argmin(cp);
      if (cp.idx == kNoSlot) break;
      const uint32_t col = cp.idx;
      if (!(qA[split_at] > threshold * cp.val)) break;
      // emit the new leaf sequence (cut.cpp:156-181)
      for (uint32_t i = lane; i < M; i += 32) {
        if (i == col + 1) continue;
        const uint32_t pos = i + (i > split_at ? 1u : 0u) - (i > col + 1 ? 1u : 0u);
        if (i == split_at) {
          const LtNode nd = sc.lt[nA[i]];
          const double half = qA[i] * 0.5;
          nB[pos] = uint32_t(nd.left);
          nB[pos + 1] = uint32_t(nd.right);
          qB[pos] = half;
          qB[pos + 1] = half;
          vB[pos] = vA[i];
          vB[pos + 1] = vA[i];
        } else if (i == col) {
          nB[pos] = uint32_t(sc.lt[nA[i]].parent);
          qB[pos] = qA[i] + qA[i + 1];
          vB[pos] = vA[i] + vA[i + 1];
        } else {
          nB[pos] = nA[i];
          qB[pos] = qA[i];
          vB[pos] = vA[i];
        }
      }
      __syncwarp();
      for (uint32_t i = lane; i < M; i += 32) {
        qA[i] = qB[i];
        nA[i] = nB[i];
        vA[i] = vB[i];
      }
      __syncwarp();
      ++my_changes;
    }
    // write back node ids, q, visits, ends when the cut changed (k_fold
    // already stored the folded q); serial cdf (cut.cpp:88-95) always
    if (my_changes != changes_before) {  // warp-uniform
      for (uint32_t i = lane; i < M; i += 32) {
        g.q[row + i] = qA[i];
        g.node_ids[row + i] = nA[i];
        g.visits[row + i] = vA[i];
        g.ends[row + i] = sc.lt[nA[i]].range_end;
      }
    }
    __syncwarp();  // (the rows are refilled for the next cell)
  }
  // rebuild_cdf (cut.cpp:88-95) of the warp's cells: the serial
  // left-to-right sum, bit-exact, one lane per cell -- the warp's cells at
  // once instead of one lane summing while 31 wait (the serial sum by lane 0
  // was 40% of this kernel's instructions).  The rows this warp wrote are
  // visible to its lanes after the __syncwarp above.
  const uint32_t wstride = gridDim.x * wpb;
  for (uint32_t cell = blockIdx.x * wpb + wib + lane * wstride; cell < ncells;
       cell += 32 * wstride) {
    if (!g.touched[cell]) continue;
    cdf_row(g, cell);
    g.touched[cell] = 0u;
  }
  if (lane == 0 && my_changes) atomicAdd(changes_out, my_changes);
}

// Batch entry points of occluded() / intersect() (bvh.hpp:38-40).
__global__ void k_segments(DevScene sc, uint32_t n, const double* __restrict__ a,
                           const double* __restrict__ b, ShadowRay* __restrict__ rays,
                           unsigned int* __restrict__ ray_count, uint8_t* __restrict__ rflag) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const V3 pa = ld3(a + 3 * size_t(i)), pb = ld3(b + 3 * size_t(i));
  const V3 dd = pb - pa;
  const double len = length(dd);
  rflag[i] = 0;  // k_shadow sets kROccluded
  if (len <= 2 * sc.shadow_eps) return;  // bvh.cpp:162
  const V3 dir = dd / len;
  const unsigned slot = atomicAdd(ray_count, 1u);
  ShadowRay r;
  r.o[0] = pa.x;
  r.o[1] = pa.y;
  r.o[2] = pa.z;
  r.d[0] = dir.x;
  r.d[1] = dir.y;
  r.d[2] = dir.z;
  r.tmax = len - sc.shadow_eps;
  r.idx = i;
  r.pad = 0;
  rays[slot] = r;
}

// occluded: a queued segment k_shadow found blocked (a segment of length
// <= 2 shadow_eps is never queued nor occluded, bvh.cpp:162)
__global__ void k_segments_out(uint32_t n, const uint8_t* __restrict__ rflag,
                               uint8_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = (rflag[i] & kROccluded) ? 1 : 0;
}

__global__ void k_intersect_batch(DevScene sc, uint32_t n, const double* __restrict__ org,
                                  const double* __restrict__ dir, double tmin,
                                  double* __restrict__ t_out, int32_t* __restrict__ tri_out,
                                  unsigned int* err, uint32_t sah_only) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t;
  uint32_t tri;
  if (sah_only) {  // diagnostic: the SAH decision alone, -2 when it defers to the ordered path
    const int r = closest_sah(sc, ld3(org + 3 * size_t(i)), ld3(dir + 3 * size_t(i)), tmin, &t, &tri);
    t_out[i] = r == 1 ? t : -1.0;
    tri_out[i] = r == 1 ? int32_t(tri) : (r == 0 ? -1 : -2);
    return;
  }
  if (intersect(sc, ld3(org + 3 * size_t(i)), ld3(dir + 3 * size_t(i)), tmin, &t, &tri, err)) {
    t_out[i] = t;
    tri_out[i] = int32_t(tri);
  } else {
    t_out[i] = -1.0;
    tri_out[i] = -1;
  }
}

void launch_occluded_batch(const DevScene& sc, uint32_t n, const double* a, const double* b,
                           PassBuffers& pb, unsigned long long* counters, uint8_t* out,
                           cudaStream_t st) {
  if (n == 0) return;
  cudaMemsetAsync(pb.ray_count, 0, 2 * sizeof(unsigned int), st);
  k_segments<<<blocks_for(n, 256), 256, 0, st>>>(sc, n, a, b, pb.rays, pb.ray_count, pb.rflag);
  launch_shadow(sc, pb, nullptr, counters, st);
  k_segments_out<<<blocks_for(n, 256), 256, 0, st>>>(n, pb.rflag, out);
  count_launch(2);
}

void launch_intersect_batch(const DevScene& sc, uint32_t n, const double* org, const double* dir,
                            double tmin, double* t_out, int32_t* tri_out,
                            unsigned long long* counters, cudaStream_t st, bool sah_only) {
  if (n == 0) return;
  k_intersect_batch<<<blocks_for(n, 128), 128, 0, st>>>(
      sc, n, org, dir, tmin, t_out, tri_out, reinterpret_cast<unsigned int*>(counters + kCntErr),
      sah_only ? 1u : 0u);
  count_launch();
}

static void launch_compact(const PassBuffers& b, const uint32_t* order, uint32_t n, uint32_t mask,
                           uint32_t* out, unsigned int* count_out, cudaStream_t st,
                           uint32_t* block_counts = nullptr, const uint32_t* key_src = nullptr,
                           uint32_t* key_out = nullptr, const uint8_t* flags = nullptr);

// ---------------------------------------------------------------------------
// Screen-band sharding with an exact exchange.  Every
// rank traces its band and files its update records (cell, cluster, v) in
// canonical order into a fixed-size block; the blocks of all ranks are
// all-gathered (rank-major = canonical order, bands being consecutive).  The
// tables are identical on every rank, so a record names its cell by table
// slot; only keys new this pass travel as keys, and every rank inserts them
// in canonical order (identical tables again).  The records are folded in
// canonical order per (cell, cluster) -- by every rank (replicated) or by
// the owner of the cell, slot % nranks, whose q_before values and per-entry
// record counts are then summed over the ranks and applied by the others to
// their copies -- so every rank ends with the single-GPU state.
// ---------------------------------------------------------------------------
__global__ void k_write_block(DevGrid g, const GBuf* __restrict__ gbuf,
                              const SampleRec* __restrict__ srec,
                              const double* __restrict__ vdense,
                              const uint32_t* __restrict__ rec_path,
                              const unsigned int* __restrict__ count, uint32_t n,
                              const unsigned long long* __restrict__ pkey, uint32_t cap,
                              ExchangeRecord* __restrict__ block) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t c = min(*count, cap);
  if (k == 0) {
    RecordBlockHeader h{};
    h.count = c;
    *reinterpret_cast<RecordBlockHeader*>(block) = h;
  }
  if (k >= n || k >= c) return;
  const uint32_t idx = rec_path[k];
  const uint32_t cell = gbuf[idx].cell;
  ExchangeRecord r;
  r.cluster = srec[idx].s;
  r.v = vdense[idx];
  if (cell == kPending) {  // new this pass: inserted with all ranks' records
    r.slot = kPending;
    r.klo = pkey[2 * size_t(idx)];
    r.khi = pkey[2 * size_t(idx) + 1];
  } else {
    r.slot = g.cell_slot[cell];
    r.klo = 0;
    r.khi = 0;
  }
  block[1 + k] = r;
}

// k_write_block with the block written into every destination's slot range
// of rank `rank` (stride cap + 1): peer receive buffers over NVLink.  The
// system-scope fence orders the stores before the barrier collective that
// follows on the stream.
__global__ void k_write_block_to(DevGrid g, const GBuf* __restrict__ gbuf,
                                 const SampleRec* __restrict__ srec,
                                 const double* __restrict__ vdense,
                                 const uint32_t* __restrict__ rec_path,
                                 const unsigned int* __restrict__ count, uint32_t n,
                                 const unsigned long long* __restrict__ pkey, uint32_t cap,
                                 PeerDsts dst, uint32_t ndst, uint32_t rank) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t c = min(*count, cap);
  const size_t base = size_t(rank) * (cap + 1);
  if (k == 0) {
    RecordBlockHeader h{};
    h.count = c;
    for (uint32_t d = 0; d < ndst; ++d)
      *reinterpret_cast<RecordBlockHeader*>(dst.p[d] + base) = h;
  }
  if (k < n && k < c) {
    const uint32_t idx = rec_path[k];
    const uint32_t cell = gbuf[idx].cell;
    ExchangeRecord r;
    r.cluster = srec[idx].s;
    r.v = vdense[idx];
    if (cell == kPending) {
      r.slot = kPending;
      r.klo = pkey[2 * size_t(idx)];
      r.khi = pkey[2 * size_t(idx) + 1];
    } else {
      r.slot = g.cell_slot[cell];
      r.klo = 0;
      r.khi = 0;
    }
    for (uint32_t d = 0; d < ndst; ++d) dst.p[d][base + 1 + k] = r;
  }
  __threadfence_system();
}

void launch_export_block_to(const DevGrid& g, const PassBuffers& b, uint32_t n,
                            const PeerDsts& dst, uint32_t ndst, uint32_t rank, uint32_t cap,
                            cudaStream_t st) {
  launch_compact(b, nullptr, n, kSRecord, b.rec_path, b.rec_count, st);
  k_write_block_to<<<blocks_for(n > 0 ? n : 1, 256), 256, 0, st>>>(
      g, b.gbuf, b.srec, b.vdense, b.rec_path, b.rec_count, n, b.pkey, cap, dst, ndst, rank);
  count_launch();
}

void launch_export_block(const DevGrid& g, const PassBuffers& b, uint32_t n, void* block,
                         uint32_t cap, cudaStream_t st) {
  launch_compact(b, nullptr, n, kSRecord, b.rec_path, b.rec_count, st);
  k_write_block<<<blocks_for(n > 0 ? n : 1, 256), 256, 0, st>>>(
      g, b.gbuf, b.srec, b.vdense, b.rec_path, b.rec_count, n, b.pkey, cap,
      static_cast<ExchangeRecord*>(block));
  count_launch();
}

// Each exchange slot t of the gathered blocks: padding (a header slot or
// past its block's count), a record of an existing cell (its cell, owner and
// sort key), or a record whose key was new at trace time -- filed with the
// smallest slot index that holds it (the canonical order in which the
// single-GPU reference inserts keys) and listed for k_resolve_pending.
__global__ void __launch_bounds__(256) k_classify(DevGrid g, uint32_t rank, uint32_t owner_fold,
                                                  ExchangeBuffers x) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t r = t / x.stride, j = t - r * x.stride;
  bool valid = false;
  ExchangeRecord rec{};
  if (r < x.nranks && j > 0) {
    const auto* hdr = reinterpret_cast<const RecordBlockHeader*>(x.rec + size_t(r) * x.stride);
    if (j <= hdr->count) {
      rec = x.rec[t];
      valid = true;
    }
  }
  uint32_t* err = reinterpret_cast<uint32_t*>(g.counters + kCntErr);
  const bool pending = valid && rec.slot == kPending;
  if (valid && !pending) {
    RLC_CHECK(rec.slot < g.capacity, g.counters + kCntErr);
    const uint32_t cell = g.slot_cell[rec.slot];
    const bool owned = !owner_fold || rec.slot % x.nranks == rank;
    x.cellx[t] = cell;
    x.kflag[t] = owned ? uint8_t(kXValid | kXOwned | kXSort) : kXValid;
    if (owned) x.keys[t] = cell * g.M + rec.cluster;
  } else if (r < x.nranks) {
    x.kflag[t] = pending ? uint8_t(kXValid | kXPending) : uint8_t(0);
  }
  if (valid && !(rec.v >= 0 && isfinite(rec.v)))  // update_q's argument check, cut.cpp:78-80
    atomicOr(err, kErrBadValue);
  const unsigned pmask = __ballot_sync(kFull, pending);
  if (!pending) return;
  // list the record for the resolution after the insertion
  const uint32_t leader0 = __ffs(pmask) - 1;
  uint32_t base = 0;
  if (lane == leader0) base = atomicAdd(x.pend_count, uint32_t(__popc(pmask)));
  base = __shfl_sync(pmask, base, leader0);
  x.pend[base + __popc(pmask & ((1u << lane) - 1u))] = t;
  // file the key once per warp (lanes of one key agree on the smallest slot)
  const uint64_t h = hash_key(unpack_key(rec.klo, rec.khi));
  const unsigned peers = __match_any_sync(pmask, h) & pmask;
  const int leader = __ffs(peers) - 1;
  const uint64_t llo = __shfl_sync(peers, rec.klo, leader);
  const uint64_t lhi = __shfl_sync(peers, rec.khi, leader);
  const bool same = llo == rec.klo && lhi == rec.khi;
  const unsigned same_mask = __ballot_sync(peers, same);
  if (same) {
    const uint32_t first = __reduce_min_sync(same_mask, t);
    if (int(lane) == leader) nk_register(x.nk, rec.klo, rec.khi, h, first, err);
  } else {
    nk_register(x.nk, rec.klo, rec.khi, h, t, err);
  }
}

// After the insertion: the cell of each record whose key was new at trace
// time, or the fallback for a refused key (its record updates nothing);
// fallback hits of this rank's own records are counted.
__global__ void k_resolve_pending(DevGrid g, uint32_t rank, uint32_t owner_fold, ExchangeBuffers x) {
  const uint32_t n = *x.pend_count;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t t = x.pend[i];
    const ExchangeRecord rec = x.rec[t];
    const uint32_t slot = probe_find(g, rec.klo, rec.khi, hash_key(unpack_key(rec.klo, rec.khi)));
    if (slot < kPending) {
      const uint32_t cell = g.slot_cell[slot];
      const bool owned = !owner_fold || slot % x.nranks == rank;
      x.cellx[t] = cell;
      x.kflag[t] = owned ? uint8_t(kXValid | kXOwned | kXSort) : kXValid;
      if (owned) x.keys[t] = cell * g.M + rec.cluster;
    } else {  // refused: a full window (hash_grid.cpp:140)
      x.cellx[t] = kFallback;
      x.kflag[t] = kXValid | kXFallback;
      if (t / x.stride == rank) atomicAdd(g.counters + kCntFallback, 1ull);
    }
  }
}

void launch_shard_fold(const DevGrid& g, const PassParams& fold_params, uint32_t rank,
                       bool owner_fold, ExchangeBuffers& x, cudaStream_t st) {
  (void)fold_params;
  const uint32_t total = x.nranks * x.stride;
  if (total == 0) return;
  cudaMemsetAsync(x.nk.count, 0, sizeof(unsigned int), st);
  cudaMemsetAsync(x.pend_count, 0, sizeof(unsigned int), st);
  cudaMemsetAsync(x.q_rec, 0, sizeof(double) * total, st);
  if (owner_fold && x.entry_mode) {
    cudaMemsetAsync(x.ent_q, 0, sizeof(double) * x.entries, st);
    cudaMemsetAsync(x.ent_n, 0, sizeof(uint32_t) * x.entries, st);
  } else if (owner_fold) {
    cudaMemsetAsync(x.seg_n, 0, sizeof(uint32_t) * total, st);
  }
  k_classify<<<blocks_for(total, 256), 256, 0, st>>>(g, rank, owner_fold ? 1u : 0u, x);
  count_launch();
  launch_insert_new_keys(g, x.nk, st);
  k_resolve_pending<<<148, 256, 0, st>>>(g, rank, owner_fold ? 1u : 0u, x);
  count_launch();
}

void launch_shard_sortfold(const DevGrid& g, const PassParams& fold_params, uint32_t key_bits,
                           bool owner_fold, ExchangeBuffers& x, cudaStream_t st) {
  const uint32_t total = x.nranks * x.stride;
  if (total == 0) return;
  // the folded records, compacted in slot (= canonical) order, sorted stably
  // by (cell, cluster) over the device count, folded in canonical order
  PassBuffers cb{};
  launch_compact(cb, nullptr, total, kXSort, x.vals_alt, x.sort_count, st, x.block_counts, x.keys,
                 x.keys_alt, x.kflag);
  uint32_t *k = nullptr, *v = nullptr;
  launch_sort_buffers(x.keys_alt, x.vals_alt, x.keys, x.vals, x.hist, total, key_bits, st, &k, &v,
                      x.sort_count, true);
  PassParams p = fold_params;
  p.n = total;
  const char* vb = reinterpret_cast<const char*>(x.rec) + offsetof(ExchangeRecord, v);
  const uint32_t vs = uint32_t(sizeof(ExchangeRecord));
  if (owner_fold && x.entry_mode)
    k_fold<2><<<blocks_for(total, 256), 256, 0, st>>>(g, p, k, v, vb, vs, x.q_rec, x.sort_count,
                                                      nullptr, x.ent_q, x.ent_n);
  else if (owner_fold)
    k_fold<1><<<blocks_for(total, 256), 256, 0, st>>>(g, p, k, v, vb, vs, x.q_rec, x.sort_count,
                                                      x.seg_n);
  else
    k_fold<0><<<blocks_for(total, 256), 256, 0, st>>>(g, p, k, v, vb, vs, x.q_rec, x.sort_count,
                                                      nullptr);
  count_launch();
}

// Owner mode: the cut entries of the cells other ranks folded, from each
// entry's last record t (seg_n[t] = the entry's record count, summed over
// the ranks with its q_before): q = max((1 - a) q_before + a v, eps), a the
// harmonic weight of that record's visit count, visits += count -- the
// arithmetic of update_q (cut.cpp:76-86) the owner ran record by record.
__global__ void k_apply(DevGrid g, PassParams P, ExchangeBuffers x) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= x.nranks * x.stride) return;
  const uint32_t c = x.seg_n[t];
  if (c == 0 || (x.kflag[t] & kXOwned)) return;
  const uint32_t cell = x.cellx[t];
  const ExchangeRecord rec = x.rec[t];
  const size_t e = size_t(cell) * g.M + rec.cluster;
  g.touched[cell] = 1u;
  const uint32_t vis_before = g.visits[e] + c - 1u;  // visits seen by the last record
  const double a = P.harmonic ? 1.0 / (1.0 + double(vis_before)) : P.alpha;
  g.q[e] = smax((1.0 - a) * x.q_rec[t] + a * rec.v, g.eps_q);
  g.visits[e] = vis_before + 1u;
}

// Owner mode, per-entry exchange: the cut entries other ranks folded take
// the owner's final q (summed over the ranks: one non-zero term) and advance
// their visits by its record count.  Entries are indexed slot * M + cluster:
// table slots are the same on every rank, dense cell ids need not be.
__global__ void k_apply_entries(DevGrid g, uint32_t rank, ExchangeBuffers x) {
  const size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x;  // slot * M + cluster
  if (e >= x.entries) return;
  const uint32_t c = x.ent_n[e];
  if (c == 0) return;
  const uint32_t slot = uint32_t(e / g.M);
  if (slot % x.nranks == rank) return;  // this rank folded it
  const uint32_t cell = g.slot_cell[slot];
  const size_t at = size_t(cell) * g.M + (e - size_t(slot) * g.M);
  g.q[at] = x.ent_q[e];
  g.visits[at] += c;
  g.touched[cell] = 1u;
}

void launch_shard_apply(const DevGrid& g, const PassParams& fold_params, uint32_t rank,
                        ExchangeBuffers& x, cudaStream_t st) {
  const uint32_t total = x.nranks * x.stride;
  if (total == 0) return;
  if (x.entry_mode) {
    k_apply_entries<<<uint32_t((x.entries + 255) / 256), 256, 0, st>>>(g, rank, x);
  } else {
    k_apply<<<blocks_for(total, 256), 256, 0, st>>>(g, fold_params, x);
  }
  count_launch();
}

__global__ void k_shard_scatter(DevGrid g, const uint32_t* __restrict__ rec_path,
                                const unsigned int* __restrict__ count, uint32_t n, uint32_t rank,
                                ExchangeBuffers x, double* __restrict__ q_before) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || k >= *count || k + 1 >= x.stride) return;
  const uint32_t t = rank * x.stride + 1 + k;
  q_before[rec_path[k]] =  // fallback: never updated
      (x.kflag[t] & kXFallback) ? g.t_q[x.rec[t].cluster] : x.q_rec[t];
}

void launch_shard_scatter(const DevGrid& g, const PassBuffers& b, uint32_t n, uint32_t rank,
                          const ExchangeBuffers& x, cudaStream_t st) {
  if (n == 0) return;
  k_shard_scatter<<<blocks_for(n, 256), 256, 0, st>>>(g, b.rec_path, b.rec_count, n, rank, x,
                                                      b.q_before);
  count_launch();
}

__global__ void k_end_pass(const uint32_t* pass_dev, uint32_t offset, uint32_t* changes,
                           uint32_t* hist) {
  if (hist) hist[*pass_dev + offset] = *changes;
  *changes = 0;
}

__global__ void k_add_u32(uint32_t* p, uint32_t v, uint32_t set) { *p = set ? v : *p + v; }

void launch_end_pass(const uint32_t* pass_dev, uint32_t offset, uint32_t* changes, uint32_t* hist,
                     cudaStream_t st) {
  k_end_pass<<<1, 1, 0, st>>>(pass_dev, offset, changes, hist);
  count_launch();
}

void launch_set_u32(uint32_t* p, uint32_t v, cudaStream_t st) {
  k_add_u32<<<1, 1, 0, st>>>(p, v, 1u);
  count_launch();
}

void launch_add_u32(uint32_t* p, uint32_t v, cudaStream_t st) {
  k_add_u32<<<1, 1, 0, st>>>(p, v, 0u);
  count_launch();
}

// rlc_pass_samples: one record per path vertex; radiance as k_accumulate
// forms it (estimators.cpp:100-101 with the live q_before, cut.cpp:105).
__global__ void k_export_samples(PassParams P, const GBuf* __restrict__ gbuf,
                                 const SampleRec* __restrict__ srec,
                                 const uint8_t* __restrict__ rflag,
                                 const double* __restrict__ vdense,
                                 const double* __restrict__ q_before,
                                 const uint32_t* __restrict__ emit, SampleExport* __restrict__ out) {
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P.nv) return;
  SampleExport e{};
  e.vertex = idx;
  if (gbuf[idx].flags & kGReflective) {
    const SampleRec r = srec[idx];
    const bool learned = r.flags & kSLearned;
    const bool nonzero = (r.flags & kSNonzero) && !(rflag[idx] & kROccluded);
    e.flags = 1u | (learned && !(r.flags & kSRecord) ? 2u : 0u) | (r.flags & kSRay ? 4u : 0u) |
              (nonzero ? 8u : 0u) | (learned ? 16u : 0u) | (r.flags & kSFrozen ? 32u : 0u);
    e.cluster = learned ? r.s : 0u;
    e.emitter = P.export_samples ? emit[idx] : 0xffffffffu;
    e.v = vdense[idx];
    e.total = r.total;
    if (learned) e.q_before = q_before[idx];
    if (nonzero) {
      const double pdf_sel =
          learned && !(r.flags & kSFrozen) ? (e.q_before / r.total) * r.pin : r.pin;
      const double den = pdf_sel * r.pdf_area;
      e.radiance[0] = r.c[0] / den;
      e.radiance[1] = r.c[1] / den;
      e.radiance[2] = r.c[2] / den;
    }
  }
  out[idx] = e;
}

void launch_export_samples(const PassParams& p, const PassBuffers& b, SampleExport* out,
                           cudaStream_t st) {
  if (p.nv == 0) return;
  k_export_samples<<<blocks_for(p.nv, 256), 256, 0, st>>>(p, b.gbuf, b.srec, b.rflag, b.vdense,
                                                          b.q_before, b.emit, out);
  count_launch();
}

__global__ void k_resolve(Framebuf fb, uint32_t npix, double* __restrict__ image) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  const unsigned long long c = fb.count[i];
  for (int a = 0; a < 3; ++a) image[3 * i + a] = c > 0 ? fb.sum[3 * i + a] / double(c) : 0.0;
}

// ---------------------------------------------------------------------------
// Device refit of the shadow tree for a dynamic update (the host refit of
// rlc_build.cpp, same arithmetic): shadow-order triangle records and their
// reference leaves, binary node boxes bottom up (the second child to finish
// builds its parent's box), 4-wide child boxes padded by S 2^-21 and rounded
// outward, leaf words with kLeafPure, and the quantized nodes.  Any
// conservative tree is exact.
// ---------------------------------------------------------------------------
__device__ __forceinline__ V3 vtx(const double* v, uint32_t t, int k) {
  return V3{v[size_t(t) * 9 + 3 * k], v[size_t(t) * 9 + 3 * k + 1], v[size_t(t) * 9 + 3 * k + 2]};
}

__global__ void k_refit_tris(RefitTopo t, const double* __restrict__ vertices,
                             const uint32_t* __restrict__ leaf_of_id, TriAccel* __restrict__ tris_s,
                             uint32_t* __restrict__ tri_leaf_s) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t.num_tris) return;
  const uint32_t id = t.tri_ids[i];
  const V3 p0 = vtx(vertices, id, 0), p1 = vtx(vertices, id, 1), p2 = vtx(vertices, id, 2);
  const V3 e1 = p1 - p0, e2 = p2 - p0;
  TriAccel a;
  a.p0[0] = p0.x, a.p0[1] = p0.y, a.p0[2] = p0.z;
  a.e1[0] = e1.x, a.e1[1] = e1.y, a.e1[2] = e1.z;
  a.e2[0] = e2.x, a.e2[1] = e2.y, a.e2[2] = e2.z;
  a.tri_id = id;
  a.pad = 0;
  tris_s[i] = a;
  tri_leaf_s[i] = leaf_of_id[id];
}

__global__ void k_refit_boxes(RefitTopo t, const double* __restrict__ vertices) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= t.num_leaves) return;
  uint32_t k = t.bin_leaves[q];
  double lo[3] = {HUGE_VAL, HUGE_VAL, HUGE_VAL}, hi[3] = {-HUGE_VAL, -HUGE_VAL, -HUGE_VAL};
  const uint32_t a = t.bin_a[k], n = t.bin_count[k];
  for (uint32_t i = a; i < a + n; ++i) {
    const uint32_t id = t.tri_ids[i];
    for (int c = 0; c < 3; ++c) {
      const V3 p = vtx(vertices, id, c);
      lo[0] = smin(lo[0], p.x), lo[1] = smin(lo[1], p.y), lo[2] = smin(lo[2], p.z);
      hi[0] = smax(hi[0], p.x), hi[1] = smax(hi[1], p.y), hi[2] = smax(hi[2], p.z);
    }
  }
  while (true) {
    double* o = t.box + 6 * size_t(k);
    for (int c = 0; c < 3; ++c) {
      o[c] = lo[c];
      o[3 + c] = hi[c];
    }
    const uint32_t p = t.bin_parent[k];
    if (p == 0xffffffffu) return;
    __threadfence();
    if (atomicAdd(t.arrive + p, 1u) == 0) return;  // the sibling builds the parent
    __threadfence();
    const volatile double* ba = t.box + 6 * size_t(t.bin_a[p]);
    const volatile double* bb = t.box + 6 * size_t(t.bin_b[p]);
    for (int c = 0; c < 3; ++c) {
      lo[c] = smin(ba[c], bb[c]);
      hi[c] = smax(ba[3 + c], bb[3 + c]);
    }
    k = p;
  }
}

// quantize_wide (rlc_build.cpp) for one node: the same planes.
__device__ void quantize_node(const Wide4& n, WideQ& q, unsigned int* err) {
  for (int c = 0; c < 4; ++c) {
    q.child[c] = n.child[c];
    q.valid |= n.child[c] != kWideEmpty ? (1u << c) : 0u;
  }
  for (int a = 0; a < 3; ++a) {
    float lo = HUGE_VALF, hi = -HUGE_VALF;
    for (int c = 0; c < 4; ++c)
      if (n.child[c] != kWideEmpty) {
        lo = fminf(lo, n.lo[a][c]);
        hi = fmaxf(hi, n.hi[a][c]);
      }
    if (!(lo <= hi)) lo = hi = 0.f;
    q.origin[a] = lo;
    const double ext = double(hi) - double(lo);
    int e = -126;
    if (ext > 0) {
      frexp(ext / 250.0, &e);
      while (e > -126 && ldexp(250.0, e - 1) >= ext) --e;
      while (e < 127 && ldexp(250.0, e) < ext) ++e;
      e = max(-126, min(127, e));
    }
    q.ex[a] = uint8_t(e + 127);
    const float scale = ldexpf(1.0f, e);
    for (int c = 0; c < 4; ++c) {
      if (n.child[c] == kWideEmpty) {
        q.qlo[a][c] = 255;
        q.qhi[a][c] = 0;
        continue;
      }
      const double L = double(n.lo[a][c]), Hh = double(n.hi[a][c]);
      int ql = int(floor((L - double(lo)) / double(scale)));
      ql = max(0, min(255, ql));
      while (ql > 0 && double(lo) + double(ql) * double(scale) > L) --ql;
      int qh = int(ceil((Hh - double(lo)) / double(scale)));
      qh = max(0, min(255, qh));
      while (qh < 255 && double(lo) + double(qh) * double(scale) < Hh) ++qh;
      if (double(lo) + double(ql) * double(scale) > L || double(lo) + double(qh) * double(scale) < Hh)
        atomicOr(err, kErrCheck);  // (cannot happen: 250 steps span the extent)
      q.qlo[a][c] = uint8_t(ql);
      q.qhi[a][c] = uint8_t(qh);
    }
  }
}

__global__ void k_refit_wide(RefitTopo t, const uint32_t* __restrict__ tri_leaf_s, double pad,
                             Wide4* __restrict__ wide, WideQ* __restrict__ wide_q,
                             unsigned int* err) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= t.num_wide) return;
  Wide4 n{};
  for (int c = 0; c < 4; ++c) {
    const uint32_t b = t.kids[4 * size_t(w) + c];
    if (b == kWideEmpty) {
      n.child[c] = kWideEmpty;
      for (int a = 0; a < 3; ++a) {
        n.lo[a][c] = HUGE_VALF;
        n.hi[a][c] = -HUGE_VALF;
      }
      continue;
    }
    const double* bx = t.box + 6 * size_t(b);
    for (int a = 0; a < 3; ++a) {  // as collapse_wide (no origin, no growth)
      n.lo[a][c] = __double2float_rd(bx[a] - pad);
      n.hi[a][c] = __double2float_ru(bx[3 + a] + pad);
    }
    const uint32_t cnt = t.bin_count[b];
    if (cnt > 0) {
      const uint32_t first = t.bin_a[b];
      bool pure = true;
      for (uint32_t k = 1; k < cnt; ++k) pure &= tri_leaf_s[first + k] == tri_leaf_s[first];
      n.child[c] = kWideLeaf | ((cnt - 1) << 28) | (pure ? kLeafPure : 0u) | first;
    } else {
      n.child[c] = t.base_child[4 * size_t(w) + c];  // internal: the creation numbering
    }
  }
  if (wide) wide[w] = n;
  if (wide_q) {
    WideQ q{};
    quantize_node(n, q, err);
    wide_q[w] = q;
  }
}

void launch_refit_shadow(const RefitTopo& t, const double* vertices, const uint32_t* leaf_of_id,
                         double pad, TriAccel* tris_s, uint32_t* tri_leaf_s, Wide4* wide,
                         WideQ* wide_q, unsigned int* err, cudaStream_t st) {
  cudaMemsetAsync(t.arrive, 0, sizeof(unsigned int) * t.num_bin, st);
  k_refit_tris<<<blocks_for(t.num_tris, 256), 256, 0, st>>>(t, vertices, leaf_of_id, tris_s,
                                                           tri_leaf_s);
  k_refit_boxes<<<blocks_for(t.num_leaves, 128), 128, 0, st>>>(t, vertices);
  k_refit_wide<<<blocks_for(t.num_wide, 128), 128, 0, st>>>(t, tri_leaf_s, pad, wide, wide_q, err);
  count_launch(3);
}

// LightOrd at every light-tree position: the record of emitter order[pos].
__global__ void k_light_order(DevScene sc, LightOrd* __restrict__ out) {
  const uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= sc.num_lights) return;
  const uint32_t e = sc.order[pos];
  const LightRec& L = sc.lights[e];
  LightOrd o{};
  for (int a = 0; a < 3; ++a) {
    o.p0[a] = L.p0[a];
    o.p1[a] = L.p1[a];
    o.p2[a] = L.p2[a];
  }
  o.mat = sc.emitter_mat[e];
  o.emitter = e;
  out[pos] = o;
}

void launch_light_order(const DevScene& sc, LightOrd* out, cudaStream_t st) {
  if (sc.num_lights == 0) return;
  k_light_order<<<blocks_for(sc.num_lights, 256), 256, 0, st>>>(sc, out);
  count_launch();
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
// Shared-memory carve-outs: the kernels without shared memory prefer all of
// the SM's unified memory as L1 (their node, cut and emitter loads hit L1
// 66-82%), and k_shadow the smallest carve-out that holds its 7-8 blocks'
// 6 KB stacks.  The SM settles on a configuration all resident blocks accept,
// so the preferences of kernels running side by side matter: c3 1.049 ->
// 1.029 ms per frame (same box).  RLC_CARVEOUT / RLC_CARVEOUT_SHADOW
// (percent) override them; -1 leaves the driver's default.
static void set_carveouts() {
  static bool done = false;
  if (done) return;
  done = true;
  const char* e = std::getenv("RLC_CARVEOUT");
  const char* e2 = std::getenv("RLC_CARVEOUT_SHADOW");
  const int pct = e ? std::atoi(e) : 0, pct_shadow = e2 ? std::atoi(e2) : 25;
  if (pct >= 0)
    for (const void* f : {reinterpret_cast<const void*>(k_primary), reinterpret_cast<const void*>(k_sample),
                          reinterpret_cast<const void*>(k_bounce), reinterpret_cast<const void*>(k_fold<0>),
                          reinterpret_cast<const void*>(k_accumulate)})
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  if (pct_shadow >= 0)
    for (const void* f : {reinterpret_cast<const void*>(k_shadow<true, false>),
                          reinterpret_cast<const void*>(k_shadow<true, true>),
                          reinterpret_cast<const void*>(k_shadow<false, false>),
                          reinterpret_cast<const void*>(k_shadow<false, true>)})
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct_shadow);
  cudaGetLastError();
}

void launch_primary(const DevScene& sc, const DevGrid& g, const PassParams& p,
                    const PassBuffers& b, cudaStream_t st) {
  set_carveouts();
  if (p.n == 0) return;
  uint32_t blocks = blocks_for(p.n, 128);
  if (p.spp_pp == 1) {  // 8 x 4 pixel tiles per warp (path_of_thread)
    const uint32_t rows = p.n / p.width;
    const uint32_t warps = ((p.width + 7u) / 8u) * ((rows + 3u) / 4u);
    blocks = (warps + 3u) / 4u;
  }
  k_primary<<<blocks, 128, 0, st>>>(sc, g, p, b.gbuf, b.nk, b.pkey);
  count_launch();
}

void launch_bounce(const DevScene& sc, const DevGrid& g, const PassParams& p, uint32_t depth,
                   const PassBuffers& b, cudaStream_t st) {
  if (p.n == 0) return;
  k_bounce<<<blocks_for(p.n, 128), 128, 0, st>>>(sc, g, p, depth, b.gbuf, b.nk, b.pkey);
  count_launch();
}

void launch_sample(const DevScene& sc, const DevGrid& g, const PassParams& p,
                   const PassBuffers& b, cudaStream_t st) {
  if (p.nv == 0) return;
  cudaMemsetAsync(b.ray_count, 0, 2 * sizeof(unsigned int), st);
  cudaMemsetAsync(b.block_counts, 0, sizeof(uint32_t) * blocks_for(p.nv, kCmpTile), st);
  k_sample<<<blocks_for(p.nv, 128), 128, 0, st>>>(sc, g, p, b.gbuf, b.srec, b.rflag, b.keys, b.vals,
                                                  b.q_before, b.rays, b.ray_count, b.pkey,
                                                  b.emit, b.vdense, b.gflags, b.block_counts);
  count_launch();
}

// ---- stable compaction of ray-bearing paths -------------------------------

__device__ __forceinline__ bool has_flag(const uint8_t* rflag, const uint32_t* order, uint32_t j,
                                         uint32_t mask) {
  const uint32_t i = order ? order[j] : j;
  return i != kNoSlot && (rflag[i] & mask);
}

__global__ void __launch_bounds__(kCmpThreads) k_cmp_count(const uint8_t* __restrict__ rflag,
                                                           const uint32_t* __restrict__ order,
                                                           uint32_t n, uint32_t mask,
                                                           uint32_t* __restrict__ counts) {
  __shared__ uint32_t ws[kCmpThreads / 32];
  uint32_t c = 0;
  for (int k = 0; k < kCmpItems; ++k) {
    const uint32_t j = blockIdx.x * kCmpTile + k * kCmpThreads + threadIdx.x;
    if (j < n && has_flag(rflag, order, j, mask)) ++c;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kCmpThreads / 32; ++w) t += ws[w];
    counts[blockIdx.x] = t;
  }
}

// counts[] holds exclusive block offsets (rs_scan) on entry.
__global__ void __launch_bounds__(kCmpThreads) k_cmp_scatter(const uint8_t* __restrict__ rflag,
                                                             const uint32_t* __restrict__ order,
                                                             uint32_t n, uint32_t mask,
                                                             const uint32_t* __restrict__ offs,
                                                             uint32_t* __restrict__ out,
                                                             unsigned int* __restrict__ count_out,
                                                             const uint32_t* __restrict__ key_src,
                                                             uint32_t* __restrict__ key_out) {
  __shared__ uint32_t wsum[kCmpThreads / 32];
  __shared__ uint32_t base;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = offs[blockIdx.x];
  __syncthreads();
  for (int k = 0; k < kCmpItems; ++k) {
    const uint32_t j = blockIdx.x * kCmpTile + k * kCmpThreads + threadIdx.x;
    const bool f = j < n && has_flag(rflag, order, j, mask);
    const unsigned b = __ballot_sync(kFull, f);
    if (lane == 0) wsum[w] = __popc(b);
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (uint32_t q = 0; q < kCmpThreads / 32; ++q) {
      before += q < w ? wsum[q] : 0u;
      total += wsum[q];
    }
    if (f) {
      const uint32_t at = base + before + __popc(b & ((1u << lane) - 1u));
      const uint32_t i = order ? order[j] : j;
      out[at] = i;
      if (key_out) key_out[at] = key_src[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) base += total;
    __syncthreads();
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    count_out[0] = base;
    count_out[1] = 0;  // fetch cursor of the persistent consumer
  }
}

// Stable compaction of the vertices whose rflag has `mask`, in the order of
// `order` (canonical when null), into out[]; the count goes to count_out[0].
// With key_out, key_src[vertex] is gathered alongside.  block_counts: a
// scratch of its own per concurrent stream (null: b.block_counts).
static void launch_compact(const PassBuffers& b, const uint32_t* order, uint32_t n, uint32_t mask,
                           uint32_t* out, unsigned int* count_out, cudaStream_t st,
                           uint32_t* block_counts, const uint32_t* key_src, uint32_t* key_out,
                           const uint8_t* flags) {
  const uint32_t nb = blocks_for(n > 0 ? n : 1, kCmpTile);
  uint32_t* bc = block_counts ? block_counts : b.block_counts;
  const uint8_t* fl = flags ? flags : b.rflag;
  k_cmp_count<<<nb, kCmpThreads, 0, st>>>(fl, order, n, mask, bc);
  rs_scan<<<1, kScanThreads, 0, st>>>(bc, nb);
  k_cmp_scatter<<<nb, kCmpThreads, 0, st>>>(fl, order, n, mask, bc, out, count_out, key_src,
                                            key_out);
  count_launch(3);
}

// k_sample counted the rays of every tile (b.block_counts): scan and scatter
void launch_ray_compact(const PassBuffers& b, const uint32_t* order, uint32_t n, cudaStream_t st) {
  if (order) {
    launch_compact(b, order, n, kSRay, b.ray_order, b.ray_count, st);
    return;
  }
  const uint32_t nb = blocks_for(n > 0 ? n : 1, kCmpTile);
  rs_scan<<<1, kScanThreads, 0, st>>>(b.block_counts, nb);
  k_cmp_scatter<<<nb, kCmpThreads, 0, st>>>(b.rflag, nullptr, n, kSRay, b.block_counts, b.ray_order,
                                            b.ray_count, nullptr, nullptr);
  count_launch(2);
}

void launch_shadow(const DevScene& sc, const PassBuffers& b, const uint32_t* order,
                   unsigned long long* counters, cudaStream_t st, bool leave_room) {
  static int per_sm = 0, sms = 0;
  if (per_sm == 0) {
    int dev = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_shadow<true, false>, kShadowThreads, 0);
    if (const char* e = getenv("RLC_SHADOW_BLOCKS_PER_SM"))  // tuning knob (co-residency)
      if (atoi(e) > 0 && atoi(e) < per_sm) per_sm = atoi(e);
    if (per_sm < 1) per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 148;
  }
  // with the update-record sort running beside it, one block slot per SM is
  // left to the sort (measured: 1.69 vs 1.71 ms per c3 frame)
  static const int room = [] {  // RLC_SHADOW_ROOM: block slots per SM left to the sort
    const char* e = getenv("RLC_SHADOW_ROOM");
    return e ? atoi(e) : 1;
  }();
  const int use = leave_room && per_sm > room ? per_sm - room : per_sm;
  // the work-counting instances run only while the context counts (the
  // bench's roofline frames); counting costs ~1.5% of a c3 frame
  auto kern = sc.count_work ? (sc.wide_q ? k_shadow<true, true> : k_shadow<false, true>)
                            : (sc.wide_q ? k_shadow<true, false> : k_shadow<false, false>);
  kern<<<use * sms, kShadowThreads, 0, st>>>(
      sc, b.rays, order, b.ray_count, b.rflag, b.vdense,
      reinterpret_cast<unsigned int*>(counters + kCntErr));
  count_launch();
}

template <int ITEMS>
static void sort_passes(uint32_t*& ka, uint32_t*& va, uint32_t*& kb, uint32_t*& vb,
                        uint32_t* hist, uint32_t n, uint32_t key_bits, cudaStream_t st,
                        const unsigned* n_dev, bool identity_vals) {
  const uint32_t nb = blocks_for(n, kRsThreads * ITEMS);
  for (uint32_t shift = 0; shift < key_bits; shift += 8) {
    rs_hist<ITEMS><<<nb, kRsThreads, 0, st>>>(ka, n, n_dev, int(shift), hist);
    uint32_t* totals = hist + size_t(nb) * 256u;
    rs_scan_rows<ITEMS><<<256, 256, 0, st>>>(hist, nb, n, n_dev, totals);
    const uint32_t* vin = identity_vals && shift == 0 ? nullptr : va;
    rs_scatter<ITEMS><<<nb, kRsThreads, 0, st>>>(ka, vin, kb, vb, n, n_dev, int(shift), hist, totals);
    count_launch(3);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
}

void launch_sort_buffers(uint32_t* ka, uint32_t* va, uint32_t* kb, uint32_t* vb, uint32_t* hist,
                         uint32_t n, uint32_t key_bits, cudaStream_t st, uint32_t** keys_out,
                         uint32_t** vals_out, const unsigned* n_dev, bool small_tiles,
                         bool identity_vals) {
  if (n > 1) {
    if (small_tiles)
      sort_passes<int(kSortTileSmall) / kRsThreads>(ka, va, kb, vb, hist, n, key_bits, st, n_dev,
                                                     identity_vals);
    else
      sort_passes<kRsItems>(ka, va, kb, vb, hist, n, key_bits, st, n_dev, identity_vals);
  }
  *keys_out = ka;
  *vals_out = va;
}


void launch_sort(PassBuffers& b, uint32_t n, uint32_t key_bits, cudaStream_t st,
                 uint32_t** keys_out, uint32_t** vals_out) {
  // RLC_SORT_COMPACT: only the vertices that carry an update record are
  // sorted (c3: 1.48M of 2.07M), gathered by a stable compaction, the digit
  // passes reading the count on the device
#if RLC_SORT_COMPACT
  launch_compact(b, nullptr, n, kSRecord, b.vals_alt, b.sort_count, st, b.block_counts2, b.keys,
                 b.keys_alt);
  launch_sort_buffers(b.keys_alt, b.vals_alt, b.keys, b.vals, b.sort_hist, n, key_bits, st,
                      keys_out, vals_out, b.sort_count);
#else  // every vertex (invalid keys sort last; the values start as the vertex ids)
  launch_sort_buffers(b.keys, b.vals, b.keys_alt, b.vals_alt, b.sort_hist, n, key_bits, st,
                      keys_out, vals_out, nullptr, false, true);
#endif
}

void launch_fold(const DevGrid& g, const PassParams& p, const uint32_t* keys,
                 const uint32_t* vals, const PassBuffers& b, cudaStream_t st) {
  if (p.nv == 0) return;
  PassParams q = p;
  q.n = p.nv;  // k_fold runs over the update records of all path vertices
  k_fold<0><<<blocks_for(q.n, 256), 256, 0, st>>>(
      g, q, keys, vals, reinterpret_cast<const char*>(b.vdense), uint32_t(sizeof(double)),
      b.q_before, RLC_SORT_COMPACT ? b.sort_count : nullptr, nullptr);
  count_launch();
}

void launch_accumulate(const DevScene& sc, const PassParams& p, const PassBuffers& b,
                       const Framebuf& fb, cudaStream_t st) {
  const uint32_t npix = p.spp_pp ? p.n / p.spp_pp : 0;
  if (npix == 0) return;
  k_accumulate<<<blocks_for(npix, 256), 256, 0, st>>>(sc, p, b.gflags, b.srec, b.rflag,
                                                      b.q_before, fb);
  count_launch();
}

void launch_split_collapse(const DevScene& sc, const DevGrid& g, double threshold,
                           uint32_t iterations, uint32_t* changes_out, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_split<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  const size_t per_warp = size_t(g.M) * 32;  // 2 doubles + 4 u32 per entry
  if (g.split_scratch) {  // rows in global memory: kSplitGlobalWarps warps
    k_split<true><<<kSplitGlobalWarps / 4, 128, 0, st>>>(sc, g, threshold, iterations,
                                                        changes_out);
    count_launch();
    return;
  }
  // At most 32 KB of shared memory per block: split-collapse runs beside the
  // next pass's primary rays, and a larger carve-out shrinks their L1 (40 KB
  // blocks made the whole c3 frame 7% slower: 1.109 vs 1.040 ms).
  uint32_t wpb = uint32_t(32 * 1024 / per_warp);
  if (wpb > 8) wpb = 8;
  if (wpb < 1) wpb = 1;
  const size_t smem = per_warp * wpb;
  k_split<false><<<148 * 4, wpb * 32, smem, st>>>(sc, g, threshold, iterations, changes_out);
  count_launch();
}

__global__ void k_libm_sincos(DevScene sc, uint32_t n, const double* __restrict__ x,
                              double* __restrict__ s, double* __restrict__ c) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const libm::Ctx lc{kSinCosTab, sc.libm_fma != 0};
  s[i] = libm::sin(lc, x[i]);
  c[i] = libm::cos(lc, x[i]);
}

void launch_libm_sincos(const DevScene& sc, uint32_t n, const double* x, double* s, double* c,
                        cudaStream_t st) {
  if (n == 0) return;
  k_libm_sincos<<<blocks_for(n, 256), 256, 0, st>>>(sc, n, x, s, c);
  count_launch();
}

// d = resolve() - ref per pixel (image.cpp:35-41, 117-121)
__global__ void k_pixel_err(Framebuf fb, uint32_t npix, const double* __restrict__ ref,
                            double* __restrict__ err) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  const unsigned long long c = fb.count[i];
  double a[3];
  for (int k = 0; k < 3; ++k) a[k] = c > 0 ? fb.sum[3 * i + k] / double(c) : 0.0;
  const double dx = a[0] - ref[3 * i], dy = a[1] - ref[3 * i + 1], dz = a[2] - ref[3 * i + 2];
  err[i] = dx * dx + dy * dy + dz * dz;
}

void launch_pixel_err(const Framebuf& fb, uint32_t npix, const double* ref, double* err,
                      cudaStream_t st) {
  if (npix == 0) return;
  k_pixel_err<<<blocks_for(npix, 256), 256, 0, st>>>(fb, npix, ref, err);
  count_launch();
}

void launch_resolve(const Framebuf& fb, uint32_t npix, double* image, cudaStream_t st) {
  if (npix == 0) return;
  k_resolve<<<blocks_for(npix, 256), 256, 0, st>>>(fb, npix, image);
  count_launch();
}

}  // namespace rlc
