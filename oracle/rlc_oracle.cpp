// rlc_oracle.cpp -- TEST INFRASTRUCTURE: CPU restatement of the RL-lightcuts
// per-pass path (arXiv 1911.10217 reference, /root/reference/proj), used only
// as the checker of the CUDA path.  Not linked into, loaded by or called from
// the product.
//
// It restates the reference algorithm as the *deferred fold* the GPU path
// implements: per pass, every path is traced and its
// light sample drawn from the pass-frozen cut cdf; update records are then
// stably ordered by (cell, cluster, canonical id) and folded with update_q's
// exact arithmetic, which yields each sample's q_before (the live q that
// sample_cluster's pdf reads, proj/src/cut.cpp:105) and the final q.  Radiance
// is formed afterwards from q_before.  Pinned bit-exact against the compiled
// reference (tests/test_oracle.py) and the reference's known-answer vectors
// (tests/golden/).
//
// Third-party algorithm: the scene BVH split uses libstdc++'s (GCC 13.3)
// std::nth_element, exactly as proj/src/bvh.cpp:103-107 does; light-tree and
// cut ordering use total orders, so any sort gives the same result.
//
// Build: oracle/Makefile (-ffp-contract=off, no -march).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "rlcuts_b200.h"  // plain-data scene/config structs only

namespace orc {

thread_local std::string g_err;

// ---- proj/include/rlcuts/math.hpp:15-61 ----------------------------------
struct V {
  double x = 0, y = 0, z = 0;
};
static inline V operator+(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
static inline V operator-(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
static inline V operator-(V a) { return {-a.x, -a.y, -a.z}; }
static inline V operator*(V a, V b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
static inline V operator*(V a, double s) { return {a.x * s, a.y * s, a.z * s}; }
static inline V operator/(V a, double s) { return {a.x / s, a.y / s, a.z / s}; }
static inline double dot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline V cross(V a, V b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
static inline double len(V v) { return std::sqrt(dot(v, v)); }
static inline V unit(V v) { return v / len(v); }
static inline double at(V v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); }
static inline double lum(V c) { return 0.2126 * c.x + 0.7152 * c.y + 0.0722 * c.z; }
static inline V vmin(V a, V b) { return {std::min(a.x, b.x), std::min(a.y, b.y), std::min(a.z, b.z)}; }
static inline V vmax(V a, V b) { return {std::max(a.x, b.x), std::max(a.y, b.y), std::max(a.z, b.z)}; }

struct Box {  // AABB, math.hpp:66-83
  V lo{HUGE_VAL, HUGE_VAL, HUGE_VAL}, hi{-HUGE_VAL, -HUGE_VAL, -HUGE_VAL};
  void add(V p) { lo = vmin(lo, p); hi = vmax(hi, p); }
  void add(const Box& b) { lo = vmin(lo, b.lo); hi = vmax(hi, b.hi); }
  V ext() const { return hi - lo; }
  int axis() const {
    const V e = ext();
    if (e.x >= e.y && e.x >= e.z) return 0;
    return e.y >= e.z ? 1 : 2;
  }
};

// ---- counter RNG, proj/include/rlcuts/rng.hpp:12-43 ----------------------
static inline uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
static inline uint64_t combine(uint64_t a, uint64_t b) { return mix(a ^ mix(b)); }
struct Rng {
  uint64_t key, dim = 0;
  Rng(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    key = combine(combine(combine(mix(seed), a), b), c);
  }
  double next() { return double(mix(key + 0x9e3779b97f4a7c15ull * ++dim) >> 11) * 0x1.0p-53; }
};

// ---- scene (proj/include/rlcuts/scene.hpp, proj/src/scene.cpp) ----------
struct Tri {
  V p0, p1, p2;
  uint32_t mat;
};
struct Mat {
  V albedo, emission;
};
struct Scene {
  std::vector<Tri> tris;
  std::vector<Mat> mats;
  V org, look, up;
  double vfov = 45;
  int w = 0, h = 0;
};

// ---- scene BVH (proj/src/bvh.cpp) ----------------------------------------
struct Node {
  Box b;
  uint32_t l = 0, r = 0, begin = 0, count = 0;
};
struct Bvh {
  std::vector<Node> nodes;
  std::vector<uint32_t> order;
  double eps = 0;
};

static Box tri_box(const Tri& t) {
  Box b;
  b.add(t.p0);
  b.add(t.p1);
  b.add(t.p2);
  return b;
}

// bvh.cpp:64-122: median split on the longest centroid axis, leaves <= 4
static Bvh build_bvh(const Scene& s) {
  const uint32_t n = uint32_t(s.tris.size());
  if (n == 0) throw std::invalid_argument("build_scene_bvh: empty scene");
  std::vector<Box> tb(n);
  std::vector<V> c(n);
  for (uint32_t i = 0; i < n; ++i) {
    tb[i] = tri_box(s.tris[i]);
    c[i] = (tb[i].lo + tb[i].hi) * 0.5;
  }
  Bvh B;
  B.order.resize(n);
  std::iota(B.order.begin(), B.order.end(), 0u);
  B.nodes.emplace_back();
  struct E {
    uint32_t node, b, e;
  };
  std::vector<E> st{{0, 0, n}};
  while (!st.empty()) {
    const E e = st.back();
    st.pop_back();
    Box bx, cb;
    for (uint32_t i = e.b; i < e.e; ++i) {
      bx.add(tb[B.order[i]]);
      cb.add(c[B.order[i]]);
    }
    B.nodes[e.node].b = bx;
    const uint32_t cnt = e.e - e.b;
    if (cnt <= 4) {
      B.nodes[e.node].begin = e.b;
      B.nodes[e.node].count = cnt;
      continue;
    }
    const int ax = cb.axis();
    const uint32_t mid = e.b + cnt / 2;
    std::nth_element(B.order.begin() + e.b, B.order.begin() + mid, B.order.begin() + e.e,
                     [&](uint32_t a, uint32_t b) { return at(c[a], ax) < at(c[b], ax); });
    const uint32_t l = uint32_t(B.nodes.size());
    B.nodes.emplace_back();
    B.nodes.emplace_back();
    B.nodes[e.node].l = l;
    B.nodes[e.node].r = l + 1;
    st.push_back({l, e.b, mid});
    st.push_back({l + 1, mid, e.e});
  }
  B.eps = 1e-4 * len(B.nodes[0].b.ext());
  return B;
}

// bvh.cpp:29-40
static bool slab_test(const Box& b, V o, V inv, double t0m, double t1m) {
  for (int a = 0; a < 3; ++a) {
    double t0 = (at(b.lo, a) - at(o, a)) * at(inv, a);
    double t1 = (at(b.hi, a) - at(o, a)) * at(inv, a);
    if (at(inv, a) < 0) std::swap(t0, t1);
    t0m = std::max(t0m, t0);
    t1m = std::min(t1m, t1);
    if (t1m < t0m) return false;
  }
  return true;
}

// bvh.cpp:44-62
static bool mt(const Tri& t, V o, V d, double tmin, double tmax, double* out) {
  const V e1 = t.p1 - t.p0, e2 = t.p2 - t.p0;
  const V pv = cross(d, e2);
  const double det = dot(e1, pv);
  if (std::abs(det) < 1e-14) return false;
  const double inv = 1.0 / det;
  const V tv = o - t.p0;
  const double u = dot(tv, pv) * inv;
  if (u < 0 || u > 1) return false;
  const V qv = cross(tv, e1);
  const double v = dot(d, qv) * inv;
  if (v < 0 || u + v > 1) return false;
  const double tt = dot(e2, qv) * inv;
  if (tt <= tmin || tt >= tmax) return false;
  *out = tt;
  return true;
}

// Traversal work counters (nodes box-tested, triangles tested) used to derive
// the algorithmic bytes of the visibility kernels.
struct Trav {
  uint64_t rays = 0, nodes = 0, tris = 0;
  uint64_t max_nodes = 0, hist[8] = {};  // per-ray node-count histogram (powers of 4)
  uint64_t cur = 0;
  void begin() { ++rays; cur = 0; }
  void end() {
    max_nodes = cur > max_nodes ? cur : max_nodes;
    int b = 0;
    for (uint64_t c = cur; c >= 4 && b < 7; c /= 4) ++b;
    ++hist[b];
  }
};

// bvh.cpp:124-157
static bool closest(const Scene& s, const Bvh& B, V o, V d, double tmin, double* t, uint32_t* tri,
                    Trav* tv = nullptr) {
  const V inv{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
  double best = HUGE_VAL;
  int64_t hit = -1;
  std::vector<uint32_t> st{0};
  if (tv) tv->begin();
  while (!st.empty()) {
    const Node& n = B.nodes[st.back()];
    st.pop_back();
    if (tv) ++tv->nodes, ++tv->cur;
    if (!slab_test(n.b, o, inv, tmin, best)) continue;
    if (n.count) {
      if (tv) tv->tris += n.count;
      for (uint32_t i = n.begin; i < n.begin + n.count; ++i) {
        double tt;
        if (mt(s.tris[B.order[i]], o, d, tmin, best, &tt)) {
          best = tt;
          hit = B.order[i];
        }
      }
    } else {
      st.push_back(n.l);
      st.push_back(n.r);
    }
  }
  if (tv) tv->end();
  if (hit < 0) return false;
  *t = best;
  *tri = uint32_t(hit);
  return true;
}

// bvh.cpp:159-188
static bool blocked(const Scene& s, const Bvh& B, V a, V b, Trav* tv = nullptr) {
  const V dd = b - a;
  const double L = len(dd);
  if (L <= 2 * B.eps) return false;
  if (tv) tv->begin();
  const V d = dd / L;
  const double tmax = L - B.eps;
  const V inv{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
  std::vector<uint32_t> st{0};
  while (!st.empty()) {
    const Node& n = B.nodes[st.back()];
    st.pop_back();
    if (tv) ++tv->nodes, ++tv->cur;
    if (!slab_test(n.b, a, inv, B.eps, tmax)) continue;
    if (n.count) {
      for (uint32_t i = n.begin; i < n.begin + n.count; ++i) {
        double tt;
        if (tv) ++tv->tris;
        if (mt(s.tris[B.order[i]], a, d, B.eps, tmax, &tt)) {
          if (tv) tv->end();
          return true;
        }
      }
    } else {
      st.push_back(n.l);
      st.push_back(n.r);
    }
  }
  if (tv) tv->end();
  return false;
}

// ---- light tree (proj/src/light_tree.cpp) -------------------------------
struct LNode {
  uint32_t b = 0, e = 0;
  int32_t l = -1, r = -1, p = -1;
  double energy = 0;
};
struct LTree {
  std::vector<uint32_t> order;
  std::vector<LNode> nodes;
};

static uint32_t spread(uint32_t x) {  // light_tree.cpp:14-21
  x &= 0x3ff;
  x = (x | (x << 16)) & 0x030000ff;
  x = (x | (x << 8)) & 0x0300f00f;
  x = (x | (x << 4)) & 0x030c30c3;
  x = (x | (x << 2)) & 0x09249249;
  return x;
}

// light_tree.cpp:56-119
static LTree build_tree(const std::vector<V>& cen, const std::vector<double>& en) {
  const uint32_t n = uint32_t(cen.size());
  if (n == 0) throw std::invalid_argument("build_light_tree: no emitters");
  Box bb;
  for (const V& c : cen) bb.add(c);
  const V lo = bb.lo - V{1e-6, 1e-6, 1e-6};
  const V ex = vmax(bb.ext() + V{2e-6, 2e-6, 2e-6}, V{1e-12, 1e-12, 1e-12});
  std::vector<std::pair<uint32_t, uint32_t>> s(n);
  for (uint32_t i = 0; i < n; ++i) {
    const V rel = cen[i] - lo;
    uint32_t q[3];
    for (int a = 0; a < 3; ++a)
      q[a] = uint32_t(std::min(1023.0, std::max(0.0, at(rel, a) / at(ex, a) * 1024.0)));
    s[i] = {spread(q[0]) | (spread(q[1]) << 1) | (spread(q[2]) << 2), i};
  }
  std::sort(s.begin(), s.end());
  LTree T;
  for (auto& p : s) T.order.push_back(p.second);
  // recursive preorder build
  struct Rec {
    static uint32_t go(LTree& T, const std::vector<std::pair<uint32_t, uint32_t>>& s,
                       const std::vector<double>& en, uint32_t b, uint32_t e, int32_t par) {
      const uint32_t id = uint32_t(T.nodes.size());
      T.nodes.push_back(LNode{b, e, -1, -1, par, 0});
      if (e - b == 1) {
        T.nodes[id].energy = en[T.order[b]];
        return id;
      }
      const uint32_t f = s[b].first, l = s[e - 1].first;
      uint32_t mid;
      if (f == l) {
        mid = b + (e - b) / 2;
      } else {
        const int bit = 31 - __builtin_clz(f ^ l);
        const uint32_t th = (f & ~((1u << (bit + 1)) - 1u)) | (1u << bit);
        mid = b;
        while (mid < e && s[mid].first < th) ++mid;
      }
      const uint32_t lc = go(T, s, en, b, mid, int32_t(id));
      const uint32_t rc = go(T, s, en, mid, e, int32_t(id));
      T.nodes[id].l = int32_t(lc);
      T.nodes[id].r = int32_t(rc);
      T.nodes[id].energy = T.nodes[lc].energy + T.nodes[rc].energy;
      return id;
    }
  };
  Rec::go(T, s, en, 0, n, -1);
  return T;
}

// ---- cuts (proj/src/cut.cpp) ---------------------------------------------
struct Cut {
  std::vector<uint32_t> node, ends, visits;
  std::vector<double> q, cdf;
  double eps = 0;
};

static void cdf_of(Cut& c) {  // cut.cpp:88-95, serial left-to-right
  c.cdf.resize(c.q.size());
  double run = 0;
  for (size_t i = 0; i < c.q.size(); ++i) c.cdf[i] = (run += c.q[i]);
}

static void ends_of(Cut& c, const LTree& T) {  // cut.cpp:18-23
  c.ends.resize(c.node.size());
  for (size_t i = 0; i < c.node.size(); ++i) c.ends[i] = T.nodes[c.node[i]].e;
}

static Cut init_cut(const LTree& T, uint32_t M, double eps) {  // cut.cpp:27-74
  if (M == 0) throw std::invalid_argument("init_cut: cut size must be positive");
  const uint32_t target = std::min<uint32_t>(M, uint32_t(T.order.size()));
  std::deque<uint32_t> q{0};
  std::vector<uint32_t> f;
  uint32_t count = 1;
  while (count < target && !q.empty()) {
    const uint32_t id = q.front();
    q.pop_front();
    if (T.nodes[id].l < 0) {
      f.push_back(id);
    } else {
      q.push_back(uint32_t(T.nodes[id].l));
      q.push_back(uint32_t(T.nodes[id].r));
      ++count;
    }
  }
  f.insert(f.end(), q.begin(), q.end());
  std::sort(f.begin(), f.end(), [&](uint32_t a, uint32_t b) { return T.nodes[a].b < T.nodes[b].b; });
  Cut c;
  c.node = f;
  c.eps = eps < 0 ? 1e-4 / double(f.size()) : eps;
  ends_of(c, T);
  double tot = 0;
  for (uint32_t id : f) tot += T.nodes[id].energy;
  for (uint32_t id : f)
    c.q.push_back(std::max(tot > 0 ? T.nodes[id].energy / tot : 1.0 / double(f.size()), c.eps));
  c.visits.assign(f.size(), 1);
  cdf_of(c);
  return c;
}

// cut.cpp:76-86
static void update(Cut& c, uint32_t s, double v, double alpha, bool harmonic) {
  if (s >= c.q.size()) throw std::out_of_range("update_q: cluster index out of range");
  if (!(v >= 0) || !std::isfinite(v))
    throw std::invalid_argument("update_q: value must be finite and non-negative");
  const double a = harmonic ? 1.0 / (1.0 + double(c.visits[s])) : alpha;
  c.q[s] = std::max((1.0 - a) * c.q[s] + a * v, c.eps);
  ++c.visits[s];
}

// cut.cpp:97-106 (index only; the pdf is formed from q_before later)
static uint32_t pick_cluster(const Cut& c, double u) {
  const double target = u * c.cdf.back();
  const auto it = std::upper_bound(c.cdf.begin(), c.cdf.end(), target);
  return it == c.cdf.end() ? uint32_t(c.cdf.size() - 1) : uint32_t(it - c.cdf.begin());
}

// cut.cpp:119-190
static uint32_t split_collapse(Cut& c, const LTree& T, double thr, uint32_t iters) {
  uint32_t changes = 0;
  for (uint32_t r = 0; r < iters; ++r) {
    int sp = -1;
    for (size_t i = 0; i < c.node.size(); ++i) {
      if (T.nodes[c.node[i]].l < 0) continue;
      if (c.q[i] * 0.5 < c.eps) continue;
      if (sp < 0 || c.q[i] > c.q[size_t(sp)]) sp = int(i);
    }
    if (sp < 0) break;
    std::vector<int32_t> anc;
    for (int32_t p = T.nodes[c.node[size_t(sp)]].p; p >= 0; p = T.nodes[p].p) anc.push_back(p);
    int cp = -1;
    double cm = 0;
    for (size_t i = 0; i + 1 < c.node.size(); ++i) {
      const int32_t pa = T.nodes[c.node[i]].p;
      if (pa < 0 || pa != T.nodes[c.node[i + 1]].p) continue;
      if (std::find(anc.begin(), anc.end(), pa) != anc.end()) continue;
      const double m = c.q[i] + c.q[i + 1];
      if (cp < 0 || m < cm) {
        cp = int(i);
        cm = m;
      }
    }
    if (cp < 0) break;
    if (!(c.q[size_t(sp)] > thr * cm)) break;
    Cut d;
    d.eps = c.eps;
    for (size_t i = 0; i < c.node.size(); ++i) {
      if (int(i) == sp) {
        const LNode& nd = T.nodes[c.node[i]];
        d.node.push_back(uint32_t(nd.l));
        d.node.push_back(uint32_t(nd.r));
        d.q.push_back(c.q[i] * 0.5);
        d.q.push_back(c.q[i] * 0.5);
        d.visits.push_back(c.visits[i]);
        d.visits.push_back(c.visits[i]);
      } else if (int(i) == cp) {
        d.node.push_back(uint32_t(T.nodes[c.node[i]].p));
        d.q.push_back(c.q[i] + c.q[i + 1]);
        d.visits.push_back(c.visits[i] + c.visits[i + 1]);
        ++i;
      } else {
        d.node.push_back(c.node[i]);
        d.q.push_back(c.q[i]);
        d.visits.push_back(c.visits[i]);
      }
    }
    ends_of(d, T);
    cdf_of(d);
    c = std::move(d);
    ++changes;
  }
  return changes;
}

// ---- hash grid keys (proj/src/hash_grid.cpp:27-100) ----------------------
struct Key {
  int32_t qx = 0, qy = 0, qz = 0;
  uint32_t qn = 0, level = 0;
  bool operator==(const Key& o) const {
    return qx == o.qx && qy == o.qy && qz == o.qz && qn == o.qn && level == o.level;
  }
};

static uint64_t hkey(const Key& k) {
  const uint64_t w0 = (uint64_t(uint32_t(k.qx)) << 32) | uint64_t(uint32_t(k.qy));
  const uint64_t w1 = (uint64_t(uint32_t(k.qz)) << 32) | (uint64_t(k.qn & 0xffffu) << 16) |
                      uint64_t(k.level & 0xffffu);
  return combine(mix(w0), w1);
}

static uint32_t level_of(double area_pdf, double base) {
  if (!(area_pdf > 0)) throw std::invalid_argument("level_for_footprint: area pdf must be positive");
  if (!(base > 0)) throw std::invalid_argument("level_for_footprint: base tile must be positive");
  const double l = std::round(std::log2((1.0 / std::sqrt(area_pdf)) / base));
  return uint32_t(std::clamp(l, 0.0, 16.0));
}

static double sgn(double v) { return v >= 0 ? 1.0 : -1.0; }

static void octa(V n, double* u, double* v) {
  const double norm = std::abs(n.x) + std::abs(n.y) + std::abs(n.z);
  double ox = n.x / norm, oy = n.y / norm;
  if (n.z < 0) {
    const double tx = (1.0 - std::abs(oy)) * sgn(ox);
    const double ty = (1.0 - std::abs(ox)) * sgn(oy);
    ox = tx;
    oy = ty;
  }
  *u = ox * 0.5 + 0.5;
  *v = oy * 0.5 + 0.5;
}

static Key make_key(V p, V n, uint32_t level, double j1, double j2, double base, uint32_t bits,
                    double js) {
  if (std::abs(len(n) - 1.0) > 1e-4) throw std::invalid_argument("make_key: normal must be unit length");
  const double cell = base * std::exp2(double(level));
  const double off = js * cell * (j1 - 0.5);
  Key k;
  k.qx = int32_t(std::floor((p.x + off) / cell));
  k.qy = int32_t(std::floor((p.y + off) / cell));
  k.qz = int32_t(std::floor((p.z + off) / cell));
  k.level = level;
  const uint32_t steps = 1u << bits;
  const double noff = js * (1.0 / double(steps)) * (j2 - 0.5);
  double u, v;
  octa(n, &u, &v);
  auto qz = [&](double c) {
    return uint32_t(std::clamp(std::floor((c + noff) * double(steps)), 0.0, double(steps - 1)));
  };
  k.qn = (qz(u) << bits) | qz(v);
  return k;
}

// ---- one oracle run ------------------------------------------------------
struct Sample {  // one light sample of the pass (one per reflective path vertex)
  uint64_t canon;    // (py*W + px)*spp_pp + s
  uint32_t pixel;
  uint32_t slot;     // UINT32_MAX: fallback
  uint32_t cluster;
  uint32_t emitter;
  uint32_t size;
  double total, pdf_area, v, q_before;
  V contrib, radiance;
  V thr;             // path throughput at the vertex (render.cpp:110, 133)
  bool nonzero;
};

struct Run {
  Scene s;
  rlc_render_config cfg{};
  Bvh bvh;
  std::vector<uint32_t> em_tri;
  std::vector<double> em_energy, energy_cdf;
  LTree tree;
  double base = 0, pdf_omega = 0;
  // hash grid (hash_grid.cpp:102-141), sequential canonical-order insertion
  std::vector<uint8_t> used, touched;
  std::vector<Key> keys;
  std::vector<Cut> cuts;
  Cut tmpl;
  uint64_t lookups = 0, fallbacks = 0;
  uint32_t occupied = 0;
  // framebuffer
  std::vector<V> sum;
  std::vector<uint64_t> count;
  std::vector<Sample> last;  // samples of the last pass (debug / golden dumps)
  Trav prim, shadow;         // traversal work over all passes

  uint32_t lookup(const Key& k) {
    ++lookups;
    const uint64_t h = hkey(k);
    const uint32_t cap = cfg.hash.capacity;
    const uint32_t probes = std::min(cfg.hash.probe_limit, cap);
    for (uint32_t i = 0; i < probes; ++i) {
      const uint32_t slot = uint32_t((h + i) % cap);
      if (!used[slot]) {
        used[slot] = 1;
        keys[slot] = k;
        cuts[slot] = tmpl;
        ++occupied;
        return slot;
      }
      if (keys[slot] == k) return slot;
    }
    ++fallbacks;
    return UINT32_MAX;
  }

  // lookup_or_insert without the lookup counter (keys received from other ranks)
  uint32_t insert(const Key& k) {
    const uint64_t l0 = lookups, f0 = fallbacks;
    const uint32_t slot = lookup(k);
    lookups = l0;
    fallbacks = f0;
    return slot;
  }

  const Cut& cut_of(uint32_t slot) const { return slot == UINT32_MAX ? tmpl : cuts[slot]; }

  // render_pass, proj/src/render.cpp:59-138 and 159-183, as a deferred fold
  // Current band of the pass being traced: rows [r0, r1).
  std::vector<Sample> cur;
  std::vector<V> emitted;
  std::vector<size_t> first_of;  // samples of path canon: [first_of[canon], first_of[canon + 1])
  uint32_t band_r0 = 0, band_spp = 1;

  // render_pass (render.cpp:159-183) = trace + fold_local.
  void pass(uint32_t pass_index) {
    trace(pass_index, 0, uint32_t(s.h));
    fold_local();
  }

  // PassRenderer::trace (render.cpp:59-137) without update_q for every path
  // of rows [r0, r1), canonical order: light samples of all path vertices in
  // (path, depth) order, each with the path throughput it is weighted by.
  void trace(uint32_t pass_index, uint32_t r0, uint32_t r1) {
    if (cfg.passes == 0 || cfg.spp % cfg.passes != 0)
      throw std::invalid_argument("render_pass: spp must be divisible by passes");
    const uint32_t spp_pp = cfg.spp / cfg.passes;
    const bool rl = cfg.sampler == RLC_SAMPLER_RL_LIGHTCUTS;
    const V w = unit(s.org - s.look), u = unit(cross(s.up, w)), vv = cross(w, u);
    const double tan_half = std::tan(0.5 * s.vfov * 3.14159265358979323846 / 180.0);
    const double aspect = double(s.w) / double(s.h);
    const uint32_t n_em = uint32_t(em_tri.size());
    if (r1 > uint32_t(s.h) || r0 > r1) throw std::invalid_argument("oracle: bad row band");
    std::vector<Sample>& samples = cur;
    samples.clear();
    band_r0 = r0;
    band_spp = spp_pp;
    emitted.assign(size_t(s.w) * (r1 - r0) * spp_pp, V{});
    first_of.assign(emitted.size() + 1, 0);
    for (uint32_t py = r0; py < r1; ++py)
      for (uint32_t px = 0; px < uint32_t(s.w); ++px)
        for (uint32_t k = 0; k < spp_pp; ++k) {
          const uint64_t canon = (uint64_t(py - r0) * s.w + px) * spp_pp + k;
          first_of[canon] = samples.size();
          Rng rng(cfg.seed, uint64_t(py) * s.w + px, uint64_t(pass_index) * spp_pp + k, 0);
          const double jx = rng.next(), jy = rng.next();
          const double sx = (2.0 * (double(px) + jx) / s.w - 1.0) * tan_half * aspect;
          const double sy = (1.0 - 2.0 * (double(py) + jy) / s.h) * tan_half;
          V org = s.org, dir = unit(u * sx + vv * sy - w);
          double tmin = 0.0, pdf_om = pdf_omega;
          V thr{1, 1, 1};
          for (uint32_t depth = 1; depth <= cfg.max_depth; ++depth) {
            double t;
            uint32_t tri;
            if (!closest(s, bvh, org, dir, tmin, &t, &tri, depth == 1 ? &prim : nullptr)) break;
            const V pos = org + dir * t;
            const Tri& T = s.tris[tri];
            const V ng = unit(cross(T.p1 - T.p0, T.p2 - T.p0));
            const V wo = -dir;
            const double cf = dot(ng, wo);
            const Mat& m = s.mats[T.mat];
            if (depth == 1 && lum(m.emission) > 0 && cf > 0) emitted[canon] = V{} + m.emission;
            const V ns = dot(ng, wo) < 0 ? -ng : ng;
            if (!(lum(m.albedo) > 0)) break;
            const double area_pdf =
                std::max(pdf_om * std::abs(cf) / std::max(t * t, 1e-24), 1e-12);
            const double u1 = rng.next(), u2 = rng.next(), u3 = rng.next();
            Sample sm{};
            sm.canon = canon;
            sm.pixel = py * s.w + px;
            sm.thr = thr;
            uint32_t e = 0;
            double pdf_sel_base = 0;
            if (rl) {
              const double j1 = rng.next(), j2 = rng.next();
              const Key key = make_key(pos, ns, level_of(area_pdf, base), j1, j2, base,
                                       cfg.hash.normal_bits, cfg.hash.jitter_scale);
              sm.slot = lookup(key);
              const Cut& c = cut_of(sm.slot);  // cdf and ends are frozen for the pass
              const uint32_t sidx = pick_cluster(c, u1);
              const uint32_t b = sidx == 0 ? 0 : c.ends[sidx - 1];
              sm.size = c.ends[sidx] - b;
              const double lo = sidx == 0 ? 0.0 : c.cdf[sidx - 1];
              const double span = c.cdf[sidx] - lo;
              const double frac =
                  span > 0 ? std::clamp((u1 * c.cdf.back() - lo) / span, 0.0, 1.0) : 0.0;
              e = tree.order[b + std::min(sm.size - 1, uint32_t(frac * double(sm.size)))];
              sm.cluster = sidx;
              sm.total = c.cdf.back();
            } else if (cfg.sampler == RLC_SAMPLER_UNIFORM) {
              e = std::min(n_em - 1, uint32_t(u1 * double(n_em)));
              pdf_sel_base = 1.0 / double(n_em);
            } else {
              const double target = u1 * energy_cdf.back();
              const auto it = std::upper_bound(energy_cdf.begin(), energy_cdf.end(), target);
              e = it == energy_cdf.end() ? n_em - 1 : uint32_t(it - energy_cdf.begin());
              pdf_sel_base = em_energy[e] / energy_cdf.back();
            }
            sm.emitter = e;
            // sample_triangle_point, scene.cpp:49-59
            const Tri& L = s.tris[em_tri[e]];
            const double area = 0.5 * len(cross(L.p1 - L.p0, L.p2 - L.p0));
            if (area <= 0) throw std::invalid_argument("sample_triangle_point: degenerate triangle");
            const double su = std::sqrt(u2), b0 = 1.0 - su, b1 = u3 * su;
            const V pt = L.p0 * b0 + L.p1 * b1 + L.p2 * (1.0 - b0 - b1);
            sm.pdf_area = 1.0 / area;
            const double pin = rl ? 1.0 / double(sm.size) : 1.0;
            // nee_estimate, estimators.cpp:82-106 (radiance deferred)
            V tl = pt - pos;
            const double d2 = dot(tl, tl);
            if (!(d2 < 1e-24)) {
              tl = tl / std::sqrt(d2);
              const double cx = dot(ns, tl);
              const double cy = dot(unit(cross(L.p1 - L.p0, L.p2 - L.p0)), -tl);
              if (!(cx <= 0) && !(cy <= 0) && !blocked(s, bvh, pos, pt, &shadow)) {
                sm.contrib = m.albedo * (1.0 / 3.14159265358979323846) * s.mats[L.mat].emission *
                             (cx * cy / d2);
                sm.nonzero = true;
                sm.v = lum(sm.contrib) / (pin * sm.pdf_area);
              }
            }
            if (!rl && sm.nonzero) sm.radiance = sm.contrib / (pdf_sel_base * sm.pdf_area);
            samples.push_back(sm);
            if (depth == cfg.max_depth) break;
            // the bounce, render.cpp:128-135: sample_cosine_hemisphere
            // (math.hpp:101-107) with the host libm's std::cos / std::sin
            const double b1u = rng.next(), b2u = rng.next();
            const double r = std::sqrt(b1u), phi = 2.0 * 3.14159265358979323846 * b2u;
            const V local{r * std::cos(phi), r * std::sin(phi), std::sqrt(std::max(0.0, 1.0 - b1u))};
            const double sign = std::copysign(1.0, ns.z);  // Frame, math.hpp:85-99
            const double a = -1.0 / (sign + ns.z);
            const double bb = ns.x * ns.y * a;
            const V tx{1.0 + sign * ns.x * ns.x * a, sign * bb, -sign * ns.x};
            const V by{bb, sign + ns.y * ns.y * a, -ns.y};
            const V nd = tx * local.x + by * local.y + ns * local.z;
            const double cos_theta = dot(ns, nd);
            if (cos_theta <= 0) break;
            thr = thr * m.albedo;
            pdf_om = cos_theta / 3.14159265358979323846;
            org = pos;
            dir = nd;
            tmin = bvh.eps;
          }
        }
    first_of[emitted.size()] = samples.size();
  }

  // The deferred fold of the band's own update records.
  void fold_local() {
    std::vector<Sample>& samples = cur;
    const bool rl = cfg.sampler == RLC_SAMPLER_RL_LIGHTCUTS;
    if (rl) {
      // deferred fold: stable order by (fallback, slot, cluster, canonical id)
      std::vector<uint32_t> idx(samples.size());
      std::iota(idx.begin(), idx.end(), 0u);
      std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) {
        const Sample &x = samples[a], &y = samples[b];
        if (x.slot != y.slot) return x.slot < y.slot;
        return x.cluster < y.cluster;
      });
      for (uint32_t i : idx) {
        Sample& sm = samples[i];
        const bool fb = sm.slot == UINT32_MAX;
        Cut& c = fb ? tmpl : cuts[sm.slot];
        sm.q_before = c.q[sm.cluster];
        if (sm.nonzero) {
          const double pdf_sel = (sm.q_before / sm.total) * (1.0 / double(sm.size));
          sm.radiance = sm.contrib / (pdf_sel * sm.pdf_area);
        }
        if (!fb) {
          update(c, sm.cluster, sm.v, cfg.cut.alpha, cfg.cut.alpha_schedule == RLC_ALPHA_HARMONIC);
          touched[sm.slot] = 1;
        }
      }
    }
    accumulate();
  }

  // Framebuffer::add_sample in canonical order (image.hpp:56-60)
  void accumulate() {
    std::vector<Sample>& samples = cur;
    for (size_t canon = 0; canon < emitted.size(); ++canon) {
      V L = emitted[canon];
      for (size_t i = first_of[canon]; i < first_of[canon + 1]; ++i)
        L = L + samples[i].thr * samples[i].radiance;
      const size_t pix = size_t(band_r0) * s.w + canon / band_spp;
      sum[pix] = sum[pix] + L;
      count[pix] += 1;
    }
    last = samples;
  }

  // This band's update records in canonical order (sharded passes).
  std::vector<rlc_update_record> records() const {
    std::vector<rlc_update_record> out;
    if (cfg.sampler != RLC_SAMPLER_RL_LIGHTCUTS) return out;
    for (const Sample& sm : cur) {
      if (sm.slot == UINT32_MAX) continue;
      const Key& k = keys[sm.slot];
      out.push_back(rlc_update_record{k.qx, k.qy, k.qz, k.qn, k.level, sm.cluster, sm.v});
    }
    return out;
  }

  // Sharded pass: folds the records of all ranks (rank-major, which is
  // canonical order because ranks own consecutive row bands), then forms the
  // radiance of this band's samples from their q_before and accumulates it.
  void fold_records(const rlc_update_record* all, const uint64_t* counts, uint32_t nranks,
                    uint32_t rank, uint64_t stride) {
    struct R {
      uint32_t slot, cluster;
      double v;
    };
    std::vector<R> recs;
    uint64_t own_offset = 0;
    for (uint32_t r = 0; r < nranks; ++r) {
      if (r < rank) own_offset += counts[r];
      for (uint64_t k = 0; k < counts[r]; ++k) {
        const rlc_update_record& u = all[r * stride + k];
        const Key key{u.qx, u.qy, u.qz, u.qn, u.level};
        const uint32_t slot = insert(key);
        if (slot == UINT32_MAX) throw std::runtime_error("oracle: sharded key overflow");
        recs.push_back(R{slot, u.cluster, u.v});
      }
    }
    std::vector<uint32_t> idx(recs.size());
    std::iota(idx.begin(), idx.end(), 0u);
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) {
      if (recs[a].slot != recs[b].slot) return recs[a].slot < recs[b].slot;
      return recs[a].cluster < recs[b].cluster;
    });
    std::vector<double> qb(recs.size());
    for (uint32_t i : idx) {
      Cut& c = cuts[recs[i].slot];
      qb[i] = c.q[recs[i].cluster];
      update(c, recs[i].cluster, recs[i].v, cfg.cut.alpha,
             cfg.cut.alpha_schedule == RLC_ALPHA_HARMONIC);
      touched[recs[i].slot] = 1;
    }
    uint64_t k = own_offset;
    for (Sample& sm : cur) {
      if (sm.slot == UINT32_MAX) sm.q_before = tmpl.q[sm.cluster];
      else sm.q_before = qb[k++];
      if (sm.nonzero) {
        const double pdf_sel = (sm.q_before / sm.total) * (1.0 / double(sm.size));
        sm.radiance = sm.contrib / (pdf_sel * sm.pdf_area);
      }
    }
    accumulate();
  }

  // end_of_pass_update, proj/src/render.cpp:185-200
  uint32_t end_of_pass() {
    uint32_t ch = 0;
    for (size_t i = 0; i < cuts.size(); ++i) {
      if (!used[i] || !touched[i]) continue;
      ch += split_collapse(cuts[i], tree, cfg.cut.split_threshold, cfg.cut.iterations);
      cdf_of(cuts[i]);
      touched[i] = 0;
    }
    return ch;
  }
};

static Scene to_scene(const rlc_scene_desc* d) {
  Scene s;
  for (uint32_t t = 0; t < d->num_triangles; ++t) {
    const double* v = d->vertices + size_t(t) * 9;
    s.tris.push_back(Tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}, d->material_ids[t]});
  }
  for (uint32_t m = 0; m < d->num_materials; ++m) {
    const double* v = d->materials + size_t(m) * 6;
    s.mats.push_back(Mat{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}});
  }
  s.org = {d->cam_origin[0], d->cam_origin[1], d->cam_origin[2]};
  s.look = {d->cam_look_at[0], d->cam_look_at[1], d->cam_look_at[2]};
  s.up = {d->cam_up[0], d->cam_up[1], d->cam_up[2]};
  s.vfov = d->vfov_degrees;
  s.w = d->width;
  s.h = d->height;
  return s;
}

static int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return RLC_ERR_INVALID_ARGUMENT;
  if (dynamic_cast<const std::out_of_range*>(&e)) return RLC_ERR_OUT_OF_RANGE;
  return RLC_ERR_INTERNAL;
}

static LTree tree_from(uint32_t n, const double* c, const double* e) {
  std::vector<V> cen(n);
  std::vector<double> en(e, e + n);
  for (uint32_t i = 0; i < n; ++i) cen[i] = {c[3 * i], c[3 * i + 1], c[3 * i + 2]};
  return build_tree(cen, en);
}

static void put_cut(const Cut& c, uint32_t m, uint32_t row, uint32_t* node, uint32_t* ends,
                    double* q, double* cdf, uint32_t* visits) {
  for (uint32_t j = 0; j < m && j < c.q.size(); ++j) {
    const size_t o = size_t(row) * m + j;
    if (node) node[o] = c.node[j];
    if (ends) ends[o] = c.ends[j];
    if (q) q[o] = c.q[j];
    if (cdf) cdf[o] = c.cdf[j];
    if (visits) visits[o] = c.visits[j];
  }
}

}  // namespace orc

using namespace orc;

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void* orc_run_create(const rlc_scene_desc* d, const rlc_render_config* cfg, int* status) {
  try {
    auto r = std::make_unique<Run>();
    r->s = to_scene(d);
    r->cfg = *cfg;
    r->bvh = build_bvh(r->s);  // render.cpp:145
    std::vector<V> cen;
    for (uint32_t t = 0; t < r->s.tris.size(); ++t) {  // collect_emitters, light_tree.cpp:30-42
      const Tri& T = r->s.tris[t];
      const Mat& m = r->s.mats[T.mat];
      if (!(lum(m.emission) > 0)) continue;
      r->em_tri.push_back(t);
      cen.push_back((T.p0 + T.p1 + T.p2) / 3.0);
      r->em_energy.push_back(lum(m.emission) * (0.5 * len(cross(T.p1 - T.p0, T.p2 - T.p0))));
    }
    if (r->em_tri.empty()) throw std::invalid_argument("build_context: scene has no emitters");
    r->tree = build_tree(cen, r->em_energy);
    double run = 0;
    for (double e : r->em_energy) r->energy_cdf.push_back(run += e);
    if (!(r->energy_cdf.back() > 0))
      throw std::invalid_argument("build_energy_cdf: total emitter energy must be positive");
    r->base = cfg->hash.base_tile > 0 ? cfg->hash.base_tile : len(r->bvh.nodes[0].b.ext()) / 256.0;
    const double th = std::tan(0.5 * r->s.vfov * 3.14159265358979323846 / 180.0);
    const double ph = 2.0 * th, pw = ph * (double(r->s.w) / double(r->s.h));
    r->pdf_omega = 1.0 / ((pw / r->s.w) * (ph / r->s.h));
    if (cfg->sampler == RLC_SAMPLER_RL_LIGHTCUTS) {
      if (cfg->hash.capacity < 1) throw std::invalid_argument("HashGrid: capacity must be at least 1");
      r->tmpl = init_cut(r->tree, cfg->cut.cut_size, cfg->cut.eps_q);
      r->used.assign(cfg->hash.capacity, 0);
      r->touched.assign(cfg->hash.capacity, 0);
      r->keys.resize(cfg->hash.capacity);
      r->cuts.resize(cfg->hash.capacity);
    }
    r->sum.assign(size_t(r->s.w) * r->s.h, V{});
    r->count.assign(size_t(r->s.w) * r->s.h, 0);
    *status = RLC_OK;
    return r.release();
  } catch (const std::exception& e) {
    *status = fail(e);
    return nullptr;
  }
}

void orc_run_destroy(void* h) { delete static_cast<Run*>(h); }

int64_t orc_run_pass(void* h, uint32_t pass_index) {
  Run* r = static_cast<Run*>(h);
  try {
    r->pass(pass_index);
    return r->cfg.sampler == RLC_SAMPLER_RL_LIGHTCUTS ? int64_t(r->end_of_pass()) : 0;
  } catch (const std::exception& e) {
    return -int64_t(fail(e));
  }
}

// Sharded pass (oracle model of the replicated protocol of rlc_shard_trace / rlc_shard_fold:
// records exchanged between ranks, every rank folding all of them).
int64_t orc_run_trace(void* h, uint32_t pass_index, uint32_t r0, uint32_t r1) {
  Run* r = static_cast<Run*>(h);
  try {
    r->trace(pass_index, r0, r1);
    return int64_t(r->records().size());
  } catch (const std::exception& e) {
    return -int64_t(fail(e));
  }
}

void orc_run_records(void* h, rlc_update_record* out) {
  const std::vector<rlc_update_record> v = static_cast<Run*>(h)->records();
  std::copy(v.begin(), v.end(), out);
}

int orc_run_fold(void* h, const rlc_update_record* all, const uint64_t* counts, uint32_t nranks,
                 uint32_t rank, uint64_t stride) {
  Run* r = static_cast<Run*>(h);
  try {
    r->fold_records(all, counts, nranks, rank, stride);
    return RLC_OK;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int64_t orc_run_end_of_pass(void* h) { return static_cast<Run*>(h)->end_of_pass(); }

void orc_run_framebuffer(void* h, double* sum, uint64_t* count) {
  Run* r = static_cast<Run*>(h);
  for (size_t i = 0; i < r->sum.size(); ++i) {
    if (sum) {
      sum[3 * i] = r->sum[i].x;
      sum[3 * i + 1] = r->sum[i].y;
      sum[3 * i + 2] = r->sum[i].z;
    }
    if (count) count[i] = r->count[i];
  }
}

void orc_run_stats(void* h, uint64_t* out) {
  Run* r = static_cast<Run*>(h);
  out[0] = r->occupied;
  out[1] = r->lookups;
  out[2] = r->fallbacks;
  out[3] = r->tmpl.q.size();
}

uint32_t orc_run_export(void* h, uint32_t max_cells, rlc_cell_key* keys, uint32_t* node,
                        uint32_t* ends, double* q, double* cdf, uint32_t* visits) {
  Run* r = static_cast<Run*>(h);
  const uint32_t m = uint32_t(r->tmpl.q.size());
  uint32_t n = 0;
  for (size_t i = 0; i < r->cuts.size(); ++i) {
    if (!r->used[i]) continue;
    if (n < max_cells) {
      const Key& k = r->keys[i];
      if (keys) keys[n] = rlc_cell_key{k.qx, k.qy, k.qz, k.qn, k.level};
      put_cut(r->cuts[i], m, n, node, ends, q, cdf, visits);
    }
    ++n;
  }
  return n;
}

// Per-sample records of the last pass, in canonical order:
// u32 out [n][4] = pixel, cluster, emitter, fallback; f64 out [n][6] =
// q_before, v, radiance rgb, total.  Returns the sample count.
uint32_t orc_run_samples(void* h, uint32_t max_n, uint32_t* u32_out, double* f64_out) {
  Run* r = static_cast<Run*>(h);
  const uint32_t n = uint32_t(r->last.size());
  for (uint32_t i = 0; i < n && i < max_n; ++i) {
    const Sample& s = r->last[i];
    u32_out[4 * i] = s.pixel;
    u32_out[4 * i + 1] = s.cluster;
    u32_out[4 * i + 2] = s.emitter;
    u32_out[4 * i + 3] = s.slot == UINT32_MAX ? 1u : 0u;
    f64_out[6 * i] = s.q_before;
    f64_out[6 * i + 1] = s.v;
    f64_out[6 * i + 2] = s.radiance.x;
    f64_out[6 * i + 3] = s.radiance.y;
    f64_out[6 * i + 4] = s.radiance.z;
    f64_out[6 * i + 5] = s.total;
  }
  return n;
}

// out[6]: primary rays, nodes, tris; shadow rays, nodes, tris
void orc_run_trav_stats(void* h, uint64_t* out) {
  Run* r = static_cast<Run*>(h);
  out[0] = r->prim.rays;
  out[1] = r->prim.nodes;
  out[2] = r->prim.tris;
  out[3] = r->shadow.rays;
  out[4] = r->shadow.nodes;
  out[5] = r->shadow.tris;
}

// shadow rays: max nodes per ray and histogram of node counts in bins
// [1,4),[4,16),...,[4^7,inf)
void orc_run_trav_hist(void* h, uint64_t* out) {
  Run* r = static_cast<Run*>(h);
  out[0] = r->shadow.max_nodes;
  for (int i = 0; i < 8; ++i) out[1 + i] = r->shadow.hist[i];
}

void orc_run_occluded(void* h, uint32_t n, const double* a, const double* b, uint8_t* out) {
  Run* r = static_cast<Run*>(h);
  for (uint32_t i = 0; i < n; ++i)
    out[i] = blocked(r->s, r->bvh, {a[3 * i], a[3 * i + 1], a[3 * i + 2]},
                     {b[3 * i], b[3 * i + 1], b[3 * i + 2]});
}

// ---- unit-level entry points (for the golden vectors) --------------------
uint32_t orc_light_tree(uint32_t n, const double* c, const double* e, uint32_t* order_out,
                        int32_t* nodes_out, double* energy_out) {
  try {
    const LTree T = tree_from(n, c, e);
    for (uint32_t i = 0; i < n; ++i) order_out[i] = T.order[i];
    for (size_t i = 0; i < T.nodes.size(); ++i) {
      nodes_out[5 * i] = int32_t(T.nodes[i].b);
      nodes_out[5 * i + 1] = int32_t(T.nodes[i].e);
      nodes_out[5 * i + 2] = T.nodes[i].l;
      nodes_out[5 * i + 3] = T.nodes[i].r;
      nodes_out[5 * i + 4] = T.nodes[i].p;
      energy_out[i] = T.nodes[i].energy;
    }
    return uint32_t(T.nodes.size());
  } catch (const std::exception& ex) {
    fail(ex);
    return 0;
  }
}

uint32_t orc_init_cut(uint32_t n, const double* c, const double* e, uint32_t M, double eps,
                      uint32_t* node, uint32_t* ends, double* q, double* cdf, uint32_t* visits,
                      double* eps_out) {
  try {
    const Cut k = init_cut(tree_from(n, c, e), M, eps);
    put_cut(k, uint32_t(k.q.size()), 0, node, ends, q, cdf, visits);
    if (eps_out) *eps_out = k.eps;
    return uint32_t(k.q.size());
  } catch (const std::exception& ex) {
    fail(ex);
    return 0;
  }
}

int64_t orc_split_collapse(uint32_t n, const double* c, const double* e, uint32_t M, double eps,
                           const double* q_in, const uint32_t* visits_in, double thr,
                           uint32_t iters, uint32_t* node, uint32_t* ends, double* q, double* cdf,
                           uint32_t* visits) {
  try {
    const LTree T = tree_from(n, c, e);
    Cut k = init_cut(T, M, eps);
    for (size_t i = 0; i < k.q.size(); ++i) {
      k.q[i] = q_in[i];
      if (visits_in) k.visits[i] = visits_in[i];
    }
    cdf_of(k);
    const uint32_t ch = split_collapse(k, T, thr, iters);
    put_cut(k, uint32_t(k.q.size()), 0, node, ends, q, cdf, visits);
    return ch;
  } catch (const std::exception& ex) {
    return -int64_t(fail(ex));
  }
}

int orc_update_q_seq(uint32_t m, double* q, uint32_t* visits, double eps, double alpha,
                     uint32_t schedule, uint32_t count, const uint32_t* s, const double* v,
                     double* q_before) {
  try {
    Cut k;
    k.q.assign(q, q + m);
    k.visits.assign(visits, visits + m);
    k.eps = eps;
    for (uint32_t i = 0; i < count; ++i) {
      if (q_before) q_before[i] = s[i] < m ? k.q[s[i]] : 0.0;
      update(k, s[i], v[i], alpha, schedule == RLC_ALPHA_HARMONIC);
    }
    std::copy(k.q.begin(), k.q.end(), q);
    std::copy(k.visits.begin(), k.visits.end(), visits);
    return RLC_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

void orc_sample_cluster(uint32_t m, const double* q, const double* cdf, uint32_t count,
                        const double* u, uint32_t* s_out, double* p_out) {
  Cut k;
  k.q.assign(q, q + m);
  k.cdf.assign(cdf, cdf + m);
  for (uint32_t i = 0; i < count; ++i) {
    s_out[i] = pick_cluster(k, u[i]);
    p_out[i] = k.q[s_out[i]] / k.cdf.back();
  }
}

int orc_level_for_footprint(uint32_t n, const double* pdf, double base, uint32_t* out) {
  try {
    for (uint32_t i = 0; i < n; ++i) out[i] = level_of(pdf[i], base);
    return RLC_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

int orc_make_key(uint32_t n, const double* pos, const double* nrm, const uint32_t* level,
                 const double* j1, const double* j2, double base, uint32_t bits, double js,
                 rlc_cell_key* out, uint64_t* hash_out) {
  try {
    for (uint32_t i = 0; i < n; ++i) {
      const Key k = make_key({pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]},
                             {nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]}, level[i], j1[i], j2[i],
                             base, bits, js);
      out[i] = rlc_cell_key{k.qx, k.qy, k.qz, k.qn, k.level};
      if (hash_out) hash_out[i] = hkey(k);
    }
    return RLC_OK;
  } catch (const std::exception& ex) {
    return fail(ex);
  }
}

void orc_octa_encode(uint32_t n, const double* nrm, double* uv) {
  for (uint32_t i = 0; i < n; ++i)
    octa({nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2]}, &uv[2 * i], &uv[2 * i + 1]);
}

uint64_t orc_mix64(uint64_t x) { return mix(x); }

void orc_rng_draws(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint32_t n, double* out) {
  Rng r(seed, a, b, c);
  for (uint32_t i = 0; i < n; ++i) out[i] = r.next();
}

}  // extern "C"
