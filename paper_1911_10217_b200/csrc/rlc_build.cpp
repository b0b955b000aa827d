// rlc_build.cpp -- host construction of everything the device path reads.
//
// The scene BVH is built with the reference's splitting rule (median of the
// centroids on the longest centroid axis via std::nth_element, leaves of at
// most four triangles; proj/src/bvh.cpp:64-122).  std::nth_element is the
// libstdc++ (GCC 13.3) introselect; calling it on the same array state with
// the same ordering predicate reproduces the reference's leaf partition,
// which is what closest-hit tie breaking (bvh.cpp:139-142) depends on.
//
// The light tree follows proj/src/light_tree.cpp:56-119: 10-bit Morton
// codes, a total order on (code, emitter index), preorder node ids, split at
// the highest differing code bit (median when a range shares one code).
#include "rlc_build.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <array>
#include <cmath>
#include <cstring>
#include <deque>
#include <mutex>
#include <memory>
#include <functional>
#include <condition_variable>
#include <thread>
#include <atomic>
#include <future>
#include <limits>
#include <numeric>
#include <cstdlib>
#include <string>

namespace rlc {

namespace {

// A process-wide pool of hardware_concurrency - 1 persistent workers (host
// builds run many short parallel loops, several of them concurrently from
// the build's own tasks: thread creation per loop and oversubscription cost
// more than the loops).  A submitter works on its own batch too, so nested
// and concurrent submissions cannot deadlock.
class WorkerPool {
 public:
  static WorkerPool& get() {
    static WorkerPool pool;
    return pool;
  }
  unsigned threads() const { return unsigned(workers_.size()) + 1; }
  // Runs job(c) for c in [0, chunks); returns when all are done.
  // Submissions from a thread that set low priority (background work beside
  // a critical path, e.g. the shadow-tree refit beside the reference BVH)
  // are taken by the workers only when no normal batch has chunks left.
  static int& priority() {
    thread_local int p = 1;
    return p;
  }
  void run(size_t chunks, const std::function<void(size_t)>& job) {
    auto batch = std::make_shared<Batch>();
    batch->job = &job;
    batch->chunks = chunks;
    batch->prio = priority();
    {
      std::lock_guard<std::mutex> lk(m_);
      queue_.push_back(batch);
      has_work_.store(true, std::memory_order_release);
    }
    cv_.notify_all();
    work(*batch);  // the submitter takes chunks too
    // the last chunks are usually short: spin briefly on the count, then sleep
    // (several builds share the pool: a spinning submitter would hold a core
    // the other builds' chunks need)
    for (int i = 0; i < 2000 && batch->done.load(std::memory_order_acquire) != batch->chunks; ++i)
      cpu_relax();
    if (batch->done.load(std::memory_order_acquire) != batch->chunks) {
      std::unique_lock<std::mutex> lk(batch->m);
      batch->cv.wait(lk, [&] { return batch->done.load() == batch->chunks; });
    }
    if (batch->error) std::rethrow_exception(batch->error);
  }
  ~WorkerPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (std::thread& t : workers_) t.join();
  }

 private:
  struct Batch {
    const std::function<void(size_t)>* job = nullptr;
    size_t chunks = 0;
    std::atomic<size_t> next{0};
    std::atomic<size_t> done{0};
    int prio = 1;
    std::exception_ptr error;  // under m
    std::mutex m;
    std::condition_variable cv;
  };
  static void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#else
    std::this_thread::yield();
#endif
  }
  WorkerPool() {
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    for (unsigned i = 0; i + 1 < hw; ++i) workers_.emplace_back([this] { loop(); });
  }
  static void work(Batch& b) {
    for (size_t c; (c = b.next.fetch_add(1)) < b.chunks;) {
      try {
        (*b.job)(c);
      } catch (...) {
        std::lock_guard<std::mutex> lk(b.m);
        if (!b.error) b.error = std::current_exception();
      }
      if (b.done.fetch_add(1, std::memory_order_acq_rel) + 1 == b.chunks) {
        std::lock_guard<std::mutex> lk(b.m);
        b.cv.notify_all();
      }
    }
  }
  void loop() {
    while (true) {
      // per-frame scene updates submit loops back to back: spin ~50 us for
      // the next batch before sleeping on the condition variable (longer
      // spins steal the cores of the build's own threads)
      const auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; !has_work_.load(std::memory_order_acquire); ++i) {
        cpu_relax();
        if ((i & 63) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(50))
          break;
      }
      std::shared_ptr<Batch> b;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || !queue_.empty(); });
        if (stop_) return;
        // retire fully claimed batches, then take the first of the highest priority
        for (auto it = queue_.begin(); it != queue_.end();)
          it = (*it)->next.load() >= (*it)->chunks ? queue_.erase(it) : std::next(it);
        if (queue_.empty()) {
          has_work_.store(false, std::memory_order_release);
          continue;
        }
        b = queue_.front();
        for (const auto& c : queue_)
          if (c->prio > b->prio) {
            b = c;
            break;
          }
      }
      work(*b);
    }
  }
  std::vector<std::thread> workers_;
  std::deque<std::shared_ptr<Batch>> queue_;
  std::atomic<bool> has_work_{false};
  std::mutex m_;
  std::condition_variable cv_;
  bool stop_ = false;
};

// Runs fn(i) for i in [0, n) on the worker pool in contiguous chunks.  The
// iterations must write disjoint data; exceptions propagate to the caller.
template <class F>
void parallel_for(size_t n, const F& fn, size_t min_chunk = 2048) {
  WorkerPool& pool = WorkerPool::get();
  const size_t chunks = std::min<size_t>(pool.threads(), (n + min_chunk - 1) / min_chunk);
  if (chunks <= 1) {
    for (size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  const std::function<void(size_t)> job = [&](size_t c) {
    const size_t b = n * c / chunks, e = n * (c + 1) / chunks;
    for (size_t i = b; i < e; ++i) fn(i);
  };
  pool.run(chunks, job);
}

struct Box {
  V3 lo{HUGE_VAL, HUGE_VAL, HUGE_VAL};
  V3 hi{-HUGE_VAL, -HUGE_VAL, -HUGE_VAL};
  void grow(V3 p) {  // AABB::extend, math.hpp:71
    lo = V3{smin(lo.x, p.x), smin(lo.y, p.y), smin(lo.z, p.z)};
    hi = V3{smax(hi.x, p.x), smax(hi.y, p.y), smax(hi.z, p.z)};
  }
  void grow(const Box& b) {
    lo = V3{smin(lo.x, b.lo.x), smin(lo.y, b.lo.y), smin(lo.z, b.lo.z)};
    hi = V3{smax(hi.x, b.hi.x), smax(hi.y, b.hi.y), smax(hi.z, b.hi.z)};
  }
  V3 extent() const { return hi - lo; }
  V3 center() const { return (lo + hi) * 0.5; }
  int longest_axis() const {  // math.hpp:78-82
    const V3 e = extent();
    if (e.x >= e.y && e.x >= e.z) return 0;
    return e.y >= e.z ? 1 : 2;
  }
};

double comp(V3 v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); }

V3 vert(const rlc_scene_desc& d, uint32_t t, int k) {
  const double* p = d.vertices + size_t(t) * 9 + size_t(k) * 3;
  return V3{p[0], p[1], p[2]};
}

// RLC_BUILD_TIMING=1: per-phase host build times on stderr (diagnostics).
struct PhaseTimer {
  bool on = std::getenv("RLC_BUILD_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void lap(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "build %-16s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t0).count());
  }
};

void put3(double* dst, V3 v) {
  dst[0] = v.x;
  dst[1] = v.y;
  dst[2] = v.z;
}

uint32_t spread10(uint32_t x) {  // 10 bits -> every third bit
  x &= 0x3ffu;
  x = (x | (x << 16)) & 0x030000ffu;
  x = (x | (x << 8)) & 0x0300f00fu;
  x = (x | (x << 4)) & 0x030c30c3u;
  x = (x | (x << 2)) & 0x09249249u;
  return x;
}

// Scene BVH over all triangles (build_scene_bvh, bvh.cpp:64-122): median
// split on the longest centroid axis with libstdc++ std::nth_element, leaves
// of <= 4 triangles.  A node's split depends only on the index range it owns,
// so subtrees below n/64 triangles are built concurrently into private node
// arrays and spliced in afterwards: the topology, left/right order, leaf
// membership and triangle order are those of the sequential build (only the
// internal node numbering differs; siblings stay adjacent).
void build_bvh(const rlc_scene_desc& d, HostScene& out) {
  PhaseTimer pt;
  pt.on = std::getenv("RLC_BVH_TIMING") != nullptr;
  const uint32_t n = d.num_triangles;
  // scratch kept per thread across builds (per-frame rebuilds touch no
  // fresh pages)
  // (local references: the worker threads' lambdas must see this thread's
  // instances, not their own thread_local ones)
  thread_local std::vector<Box> tl_tb;
  thread_local std::vector<V3> tl_cen;
  thread_local std::vector<double> tl_ckey[3];
  thread_local std::vector<uint32_t> tl_perm;
  std::vector<Box>& tb = tl_tb;
  std::vector<V3>& cen = tl_cen;
  // centroid coordinates per axis, contiguous: the nth_element comparator
  // reads 8-byte keys instead of a strided V3 and an axis switch (the same
  // doubles, so the same comparisons and the same permutation)
  std::vector<double>(&ckey)[3] = tl_ckey;
  tb.resize(n);
  cen.resize(n);
  for (auto& k : ckey) k.resize(n);
  pt.lap("bvh scratch");
  parallel_for(n, [&](size_t i) {
    Box b;
    b.grow(vert(d, uint32_t(i), 0));
    b.grow(vert(d, uint32_t(i), 1));
    b.grow(vert(d, uint32_t(i), 2));
    tb[i] = b;
    cen[i] = b.center();
    ckey[0][i] = cen[i].x;
    ckey[1][i] = cen[i].y;
    ckey[2][i] = cen[i].z;
  });
  std::vector<uint32_t>& perm = tl_perm;
  perm.resize(n);
  std::iota(perm.begin(), perm.end(), 0u);
  pt.lap("bvh centroids");

  struct Todo {
    uint32_t node, begin, end;
  };
  // Builds the subtree of `root` (already allocated in `nodes`) over
  // perm[begin, end); new nodes are appended to `nodes`.
  auto build = [&](std::vector<BvhNode>& nodes, uint32_t root, uint32_t begin, uint32_t end,
                   uint32_t defer_below, std::vector<Todo>* deferred) {
    std::vector<Todo> todo{{root, begin, end}};
    while (!todo.empty()) {
      const Todo t = todo.back();
      todo.pop_back();
      const uint32_t count = t.end - t.begin;
      if (deferred && count < defer_below && count > 4) {
        deferred->push_back(t);
        continue;
      }
      Box bounds, cb;
      for (uint32_t i = t.begin; i < t.end; ++i) {
        bounds.grow(tb[perm[i]]);
        cb.grow(cen[perm[i]]);
      }
      BvhNode& nd = nodes[t.node];
      put3(nd.lo, bounds.lo);
      put3(nd.hi, bounds.hi);
      if (count <= 4) {
        nd.a = t.begin;
        nd.b = 0;
        nd.count = count;
        continue;
      }
      const int axis = cb.longest_axis();
      const uint32_t mid = t.begin + count / 2;
      const double* key = ckey[axis].data();
      std::nth_element(perm.begin() + t.begin, perm.begin() + mid, perm.begin() + t.end,
                       [key](uint32_t x, uint32_t y) { return key[x] < key[y]; });
      const uint32_t child = uint32_t(nodes.size());
      nodes.push_back(BvhNode{});
      nodes.push_back(BvhNode{});
      nodes[t.node].a = child;
      nodes[t.node].b = child + 1;
      nodes[t.node].count = 0;
      todo.push_back({child, t.begin, mid});
      todo.push_back({child + 1, mid, t.end});
    }
  };
  std::vector<BvhNode>& nodes = out.nodes;
  nodes.clear();
  nodes.reserve(size_t(2) * n);
  nodes.push_back(BvhNode{});
  std::vector<Todo> deferred;
  const uint32_t cut = std::max<uint32_t>(n / 64, 2048);
  // The top levels breadth first, the nodes of a level split concurrently
  // (disjoint perm ranges; children numbered in level order afterwards), so
  // the sequential nth_element work on the critical path is ~2n instead of
  // n per level.  Below `cut` whole subtrees are built in parallel.
  {
    std::vector<Todo> level{{0, 0, n}};
    while (!level.empty()) {
      std::vector<std::array<uint32_t, 3>> split(level.size());  // mid, leaf?, count
      parallel_for(level.size(), [&](size_t k) {
        const Todo t = level[k];
        const uint32_t count = t.end - t.begin;
        Box bounds, cb;
        if (count >= 32768) {  // min/max: chunked in parallel, exactly the same boxes
          constexpr uint32_t kChunk = 4096;
          const uint32_t nc = (count + kChunk - 1) / kChunk;
          std::vector<Box> pb(nc), pc(nc);
          parallel_for(nc, [&](size_t c) {
            const uint32_t b0 = t.begin + uint32_t(c) * kChunk, b1 = std::min(t.end, b0 + kChunk);
            for (uint32_t i = b0; i < b1; ++i) {
              pb[c].grow(tb[perm[i]]);
              pc[c].grow(cen[perm[i]]);
            }
          }, 1);
          for (uint32_t c = 0; c < nc; ++c) {
            bounds.grow(pb[c]);
            cb.grow(pc[c]);
          }
        } else {
          for (uint32_t i = t.begin; i < t.end; ++i) {
            bounds.grow(tb[perm[i]]);
            cb.grow(cen[perm[i]]);
          }
        }
        BvhNode& nd = nodes[t.node];
        put3(nd.lo, bounds.lo);
        put3(nd.hi, bounds.hi);
        if (count <= 4) {
          nd.a = t.begin;
          nd.b = 0;
          nd.count = count;
          split[k] = {0u, 1u, count};
          return;
        }
        const int axis = cb.longest_axis();
        const uint32_t mid = t.begin + count / 2;
        const double* key = ckey[axis].data();
        std::nth_element(perm.begin() + t.begin, perm.begin() + mid, perm.begin() + t.end,
                         [key](uint32_t x, uint32_t y) { return key[x] < key[y]; });
        split[k] = {mid, 0u, count};
      }, 1);
      std::vector<Todo> next;
      for (size_t k = 0; k < level.size(); ++k) {
        if (split[k][1]) continue;
        const Todo t = level[k];
        const uint32_t child = uint32_t(nodes.size());
        nodes.push_back(BvhNode{});
        nodes.push_back(BvhNode{});
        nodes[t.node].a = child;
        nodes[t.node].b = child + 1;
        nodes[t.node].count = 0;
        for (const Todo c : {Todo{child, t.begin, split[k][0]}, Todo{child + 1, split[k][0], t.end}}) {
          if (c.end - c.begin < cut && c.end - c.begin > 4) deferred.push_back(c);
          else next.push_back(c);
        }
      }
      level.swap(next);
      pt.lap("bvh level");
    }
  }
  if (!deferred.empty()) {
    // subtrees in parallel, each into a private array whose element 0 is the
    // subtree root (a node already allocated in `nodes`)
    std::vector<std::vector<BvhNode>> local(deferred.size());
    parallel_for(deferred.size(), [&](size_t k) {  // on the persistent worker pool
      std::vector<BvhNode>& L = local[k];
      L.reserve(size_t(2) * (deferred[k].end - deferred[k].begin));
      L.push_back(BvhNode{});
      build(L, 0, deferred[k].begin, deferred[k].end, 0, nullptr);
    }, 1);
    for (size_t k = 0; k < deferred.size(); ++k) {
      const std::vector<BvhNode>& L = local[k];
      const uint32_t base = uint32_t(nodes.size()) - 1;  // local index i >= 1 -> base + i
      auto remap = [&](const BvhNode& y) {
        BvhNode x = y;
        if (x.count == 0) {
          x.a += base;
          x.b += base;
        }
        return x;
      };
      nodes[deferred[k].node] = remap(L[0]);
      for (size_t i = 1; i < L.size(); ++i) nodes.push_back(remap(L[i]));
    }
  }
  pt.lap("bvh subtrees");
  out.tris.resize(n);
  parallel_for(n, [&](size_t i) {
    const uint32_t id = perm[i];
    const V3 p0 = vert(d, id, 0), p1 = vert(d, id, 1), p2 = vert(d, id, 2);
    TriAccel& ta = out.tris[i];
    put3(ta.p0, p0);
    put3(ta.e1, p1 - p0);
    put3(ta.e2, p2 - p0);
    ta.tri_id = id;
    ta.pad = 0;
  });
  for (int a = 0; a < 3; ++a) {
    out.scene_lo[a] = nodes[0].lo[a];
    out.scene_hi[a] = nodes[0].hi[a];
  }
  const V3 ext = V3{nodes[0].hi[0], nodes[0].hi[1], nodes[0].hi[2]} -
                 V3{nodes[0].lo[0], nodes[0].lo[1], nodes[0].lo[2]};
  out.shadow_eps = 1e-4 * length(ext);  // bvh.cpp:120
}

// The next float toward -inf / +inf (bit stepping; std::nextafter's libm
// call dominated the tree collapses).
inline float float_down(float f) {
  if (f != f || f == -HUGE_VALF) return f;
  if (f == 0.0f) return -std::numeric_limits<float>::denorm_min();
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u = f > 0 ? u - 1 : u + 1;
  std::memcpy(&f, &u, 4);
  return f;
}
inline float float_up(float f) { return -float_down(-f); }

float round_down(double x) {
  float f = float(x);
  if (double(f) > x) f = float_down(f);
  return f;
}
float round_up(double x) {
  float f = float(x);
  if (double(f) < x) f = float_up(f);
  return f;
}

double surface(const BvhNode& n) {
  const double dx = n.hi[0] - n.lo[0], dy = n.hi[1] - n.lo[1], dz = n.hi[2] - n.lo[2];
  return dx * dy + dy * dz + dz * dx;
}

// Binned-SAH binary tree whose leaves are exactly the reference BVH's leaves
// (same triangle ranges, same exact boxes).  Every node box is the exact
// union of the leaf boxes below it, so it contains them: traversing this
// tree with a conservative test reaches every leaf whose exact slab test
// passes, which is all the exact any-hit acceptance needs.
std::vector<BvhNode> sah_over_leaves(const std::vector<BvhNode>& ref) {
  struct Prim {
    Box b;
    V3 c;
    uint32_t node;
  };
  std::vector<Prim> prims;
  for (uint32_t i = 0; i < ref.size(); ++i) {
    if (ref[i].count == 0) continue;
    Box b;
    b.lo = V3{ref[i].lo[0], ref[i].lo[1], ref[i].lo[2]};
    b.hi = V3{ref[i].hi[0], ref[i].hi[1], ref[i].hi[2]};
    prims.push_back(Prim{b, b.center(), i});
  }
  auto area = [](const Box& b) {
    const V3 e = b.extent();
    return e.x * e.y + e.y * e.z + e.z * e.x;
  };
  std::vector<BvhNode> out;
  out.reserve(2 * prims.size());
  out.push_back(BvhNode{});
  struct Todo {
    uint32_t node, begin, end;
  };
  std::vector<Todo> todo{{0, 0, uint32_t(prims.size())}};
  constexpr int kBins = 16;
  while (!todo.empty()) {
    const Todo t = todo.back();
    todo.pop_back();
    Box bounds, cb;
    for (uint32_t i = t.begin; i < t.end; ++i) {
      bounds.grow(prims[i].b);
      cb.grow(prims[i].c);
    }
    BvhNode& nd = out[t.node];
    put3(nd.lo, bounds.lo);
    put3(nd.hi, bounds.hi);
    if (t.end - t.begin == 1) {
      const BvhNode& leaf = ref[prims[t.begin].node];
      nd.a = leaf.a;
      nd.b = 0;
      nd.count = leaf.count;
      continue;
    }
    int best_axis = -1, best_split = 0;
    double best_cost = HUGE_VAL;
    for (int a = 0; a < 3; ++a) {
      const double lo = comp(cb.lo, a), ext = comp(cb.hi, a) - lo;
      if (!(ext > 0)) continue;
      Box bb[kBins];
      uint32_t cnt[kBins] = {};
      for (uint32_t i = t.begin; i < t.end; ++i) {
        int k = int((comp(prims[i].c, a) - lo) / ext * kBins);
        k = k < 0 ? 0 : (k >= kBins ? kBins - 1 : k);
        bb[k].grow(prims[i].b);
        ++cnt[k];
      }
      Box right[kBins];
      uint32_t rc[kBins] = {};
      Box acc;
      uint32_t n = 0;
      for (int k = kBins - 1; k > 0; --k) {
        acc.grow(bb[k]);
        n += cnt[k];
        right[k] = acc;
        rc[k] = n;
      }
      Box left;
      uint32_t nl = 0;
      for (int k = 1; k < kBins; ++k) {
        left.grow(bb[k - 1]);
        nl += cnt[k - 1];
        if (nl == 0 || rc[k] == 0) continue;
        const double cost = area(left) * nl + area(right[k]) * rc[k];
        if (cost < best_cost) {
          best_cost = cost;
          best_axis = a;
          best_split = k;
        }
      }
    }
    uint32_t mid;
    if (best_axis < 0) {
      mid = t.begin + (t.end - t.begin) / 2;
    } else {
      const double lo = comp(cb.lo, best_axis), ext = comp(cb.hi, best_axis) - lo;
      const auto it = std::partition(prims.begin() + t.begin, prims.begin() + t.end,
                                     [&](const Prim& p) {
                                       int k = int((comp(p.c, best_axis) - lo) / ext * kBins);
                                       k = k < 0 ? 0 : (k >= kBins ? kBins - 1 : k);
                                       return k < best_split;
                                     });
      mid = uint32_t(it - prims.begin());
      if (mid == t.begin || mid == t.end) mid = t.begin + (t.end - t.begin) / 2;
    }
    const uint32_t child = uint32_t(out.size());
    out.push_back(BvhNode{});
    out.push_back(BvhNode{});
    out[t.node].a = child;
    out[t.node].b = child + 1;
    out[t.node].count = 0;
    todo.push_back({child, t.begin, mid});
    todo.push_back({child + 1, mid, t.end});
  }
  return out;
}

// Binned-SAH binary tree over single triangles for the any-hit shadow rays
// (DESIGN.md 5.3).  Prims are the leaf-order triangles (positions of
// out.tris) with their exact vertex boxes; a leaf holds at most 4 triangles
// of ONE reference leaf, so its exact box lies inside that reference leaf's
// box and a passing (inner) test on it proves the reference leaf test.  The
// returned leaves index `perm` (a permutation of leaf-order positions).
std::vector<BvhNode> sah_over_tris(const rlc_scene_desc& d, const HostScene& hs,
                                   std::vector<uint32_t>& perm) {
  const uint32_t n = uint32_t(hs.tris.size());
  std::vector<Box> tb(n);
  std::vector<V3> cen(n);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t id = hs.tris[i].tri_id;
    Box b;
    b.grow(vert(d, id, 0));
    b.grow(vert(d, id, 1));
    b.grow(vert(d, id, 2));
    tb[i] = b;
    cen[i] = b.center();
  }
  perm.resize(n);
  std::iota(perm.begin(), perm.end(), 0u);
  auto area = [](const Box& b) {
    const V3 e = b.extent();
    return e.x * e.y + e.y * e.z + e.z * e.x;
  };
  std::vector<BvhNode> out;
  out.reserve(size_t(2) * n);
  out.push_back(BvhNode{});
  struct Todo {
    uint32_t node, begin, end;
  };
  std::vector<Todo> todo{{0, 0, n}};
  constexpr int kBins = 16;
  while (!todo.empty()) {
    const Todo t = todo.back();
    todo.pop_back();
    Box bounds, cb;
    for (uint32_t i = t.begin; i < t.end; ++i) {
      bounds.grow(tb[perm[i]]);
      cb.grow(cen[perm[i]]);
    }
    BvhNode& nd = out[t.node];
    put3(nd.lo, bounds.lo);
    put3(nd.hi, bounds.hi);
    const uint32_t count = t.end - t.begin;
    bool pure = true;
    for (uint32_t i = t.begin + 1; i < t.end; ++i)
      pure &= hs.tri_leaf[perm[i]] == hs.tri_leaf[perm[t.begin]];
    int best_axis = -1, best_split = 0;
    double best_cost = HUGE_VAL;
    if (count > 1) {
      for (int a = 0; a < 3; ++a) {
        const double lo = comp(cb.lo, a), ext = comp(cb.hi, a) - lo;
        if (!(ext > 0)) continue;
        Box bb[kBins];
        uint32_t cnt[kBins] = {};
        for (uint32_t i = t.begin; i < t.end; ++i) {
          int k = int((comp(cen[perm[i]], a) - lo) / ext * kBins);
          k = k < 0 ? 0 : (k >= kBins ? kBins - 1 : k);
          bb[k].grow(tb[perm[i]]);
          ++cnt[k];
        }
        Box right[kBins];
        uint32_t rc[kBins] = {};
        Box acc;
        uint32_t m = 0;
        for (int k = kBins - 1; k > 0; --k) {
          acc.grow(bb[k]);
          m += cnt[k];
          right[k] = acc;
          rc[k] = m;
        }
        Box left;
        uint32_t nl = 0;
        for (int k = 1; k < kBins; ++k) {
          left.grow(bb[k - 1]);
          nl += cnt[k - 1];
          if (nl == 0 || rc[k] == 0) continue;
          const double cost = area(left) * nl + area(right[k]) * rc[k];
          if (cost < best_cost) {
            best_cost = cost;
            best_axis = a;
            best_split = k;
          }
        }
      }
    }
    // leaf: one triangle, or up to 4 of one reference leaf when splitting
    // does not pay (SAH, traversal cost 1 per box against tri_cost per
    // triangle; RLC_SAH_TRI_COST, default 1)
    static const double tri_cost = [] {
      const char* e = std::getenv("RLC_SAH_TRI_COST");
      return e ? std::atof(e) : 1.0;
    }();
    const double a_node = area(bounds);
    const bool can_leaf = count == 1 || (count <= 4 && pure);
    if (can_leaf && (best_axis < 0 || !(a_node > 0) ||
                     tri_cost * double(count) <= 1.0 + tri_cost * best_cost / a_node)) {
      nd.a = t.begin;
      nd.b = 0;
      nd.count = count;
      continue;
    }
    uint32_t mid;
    if (best_axis < 0) {  // coincident centroids: split the list (keeps leaves pure)
      std::stable_sort(perm.begin() + t.begin, perm.begin() + t.end,
                       [&](uint32_t x, uint32_t y) { return hs.tri_leaf[x] < hs.tri_leaf[y]; });
      mid = t.begin + count / 2;
    } else {
      const double lo = comp(cb.lo, best_axis), ext = comp(cb.hi, best_axis) - lo;
      const auto it = std::partition(perm.begin() + t.begin, perm.begin() + t.end,
                                     [&](uint32_t x) {
                                       int k = int((comp(cen[x], best_axis) - lo) / ext * kBins);
                                       k = k < 0 ? 0 : (k >= kBins ? kBins - 1 : k);
                                       return k < best_split;
                                     });
      mid = uint32_t(it - perm.begin());
      if (mid == t.begin || mid == t.end) mid = t.begin + count / 2;
    }
    const uint32_t child = uint32_t(out.size());
    out.push_back(BvhNode{});
    out.push_back(BvhNode{});
    out[t.node].a = child;
    out[t.node].b = child + 1;
    out[t.node].count = 0;
    todo.push_back({child, t.begin, mid});
    todo.push_back({child + 1, mid, t.end});
  }
  return out;
}

// Collapses a binary tree to 4-wide nodes: every wide node stands for one
// binary internal node and lists up to four of its descendants (children
// expanded largest-surface-first, in place, so the list keeps the binary
// tree's left-to-right order); child boxes are rounded outward to fp32, taken
// relative to `origin` when given (x = fl64(c - O)) and then enlarged by
// |x| * grow + pad before the outward rounding.
// Leaves get kLeafPure when all their triangles lie in one reference leaf
// (leaf_of[i]: reference leaf of triangle position i; null: always).
std::vector<Wide4> collapse_wide(const std::vector<BvhNode>& nodes, const double* origin,
                                 double grow = 0.0, double pad = 0.0,
                                 const std::vector<uint32_t>* leaf_of = nullptr,
                                 std::vector<std::array<uint32_t, kWide>>* kids_out = nullptr) {
  std::vector<uint32_t> wid(nodes.size(), kWideEmpty);
  std::vector<std::array<uint32_t, kWide>> kids;
  kids.reserve(nodes.size() / 2 + 1);
  // breadth-first numbering: the internal children of a node get consecutive
  // indices, so siblings share cache lines (two 64-byte quantized nodes per
  // 128-byte line)
  std::vector<uint32_t> todo{0};
  todo.reserve(nodes.size() / 2 + 1);
  std::vector<uint32_t> order;
  for (size_t head = 0; head < todo.size(); ++head) {
    const uint32_t b = todo[head];
    wid[b] = uint32_t(order.size());
    order.push_back(b);
    std::array<uint32_t, kWide> L;
    L.fill(kWideEmpty);
    L[0] = nodes[b].a;
    L[1] = nodes[b].b;
    int nl = 2;
    while (nl < kWide) {
      int best = -1;
      for (int k = 0; k < nl; ++k)
        if (nodes[L[k]].count == 0 && (best < 0 || surface(nodes[L[k]]) > surface(nodes[L[best]])))
          best = k;
      if (best < 0) break;
      const uint32_t x = L[best];
      for (int k = nl; k > best + 1; --k) L[k] = L[k - 1];  // keep left-to-right order
      L[best] = nodes[x].a;
      L[best + 1] = nodes[x].b;
      ++nl;
    }
    kids.push_back(L);
    for (int k = 0; k < nl; ++k)
      if (nodes[L[k]].count == 0) todo.push_back(L[k]);
  }
  std::vector<Wide4> wide(order.size());
  parallel_for(order.size(), [&](size_t w) {
    Wide4& n = wide[w];
    std::memset(&n, 0, sizeof(n));
    for (int c = 0; c < kWide; ++c) {
      const uint32_t b = kids[w][c];
      if (b == kWideEmpty) {
        n.child[c] = kWideEmpty;
        for (int a = 0; a < 3; ++a) {
          n.lo[a][c] = HUGE_VALF;
          n.hi[a][c] = -HUGE_VALF;
        }
        continue;
      }
      const BvhNode& bn = nodes[b];
      for (int a = 0; a < 3; ++a) {
        const double lo = origin ? bn.lo[a] - origin[a] : bn.lo[a];
        const double hi = origin ? bn.hi[a] - origin[a] : bn.hi[a];
        n.lo[a][c] = round_down(lo - std::fabs(lo) * grow - pad);
        n.hi[a][c] = round_up(hi + std::fabs(hi) * grow + pad);
      }
      bool pure = true;
      if (bn.count > 0 && leaf_of)
        for (uint32_t k = 1; k < bn.count; ++k) pure &= (*leaf_of)[bn.a + k] == (*leaf_of)[bn.a];
      n.child[c] = bn.count > 0 ? (kWideLeaf | ((bn.count - 1) << 28) | (pure ? kLeafPure : 0u) |
                                   bn.a)
                                : wid[b];
    }
  });
  if (kids_out) *kids_out = std::move(kids);
  return wide;
}

// Quantizes wide nodes to WideQ (rlc_common.h): per node and axis the origin
// is the smallest child bound and the scale the smallest power of two that
// spans the node in 250 steps; each bound is then moved outward until the
// exact plane origin + q * scale encloses the fp32 bound.
void quantize_wide(const std::vector<Wide4>& w, std::vector<WideQ>& out) {
  out.resize(w.size());
  parallel_for(w.size(), [&](size_t i) {
    const Wide4& n = w[i];
    WideQ& q = out[i];
    std::memset(&q, 0, sizeof(q));
    for (int c = 0; c < 4; ++c) {
      q.child[c] = n.child[c];
      if (n.child[c] != kWideEmpty) q.valid |= 1u << c;
    }
    for (int a = 0; a < 3; ++a) {
      float lo = HUGE_VALF, hi = -HUGE_VALF;
      for (int c = 0; c < 4; ++c)
        if (n.child[c] != kWideEmpty) {
          lo = std::min(lo, n.lo[a][c]);
          hi = std::max(hi, n.hi[a][c]);
        }
      if (!(lo <= hi)) lo = hi = 0.f;  // no children
      q.origin[a] = lo;
      const double ext = double(hi) - double(lo);
      // scale 2^e: the smallest with ext / scale <= 250
      int e = -126;
      if (ext > 0) {
        std::frexp(ext / 250.0, &e);  // ext / 250 < 2^e
        while (e > -126 && std::ldexp(250.0, e - 1) >= ext) --e;
        while (e < 127 && std::ldexp(250.0, e) < ext) ++e;
        e = std::max(-126, std::min(127, e));
      }
      q.ex[a] = uint8_t(e + 127);
      const float scale = std::ldexp(1.0f, e);
      for (int c = 0; c < 4; ++c) {
        if (n.child[c] == kWideEmpty) {
          q.qlo[a][c] = 255;
          q.qhi[a][c] = 0;
          continue;
        }
        // the device evaluates the exact plane origin + q * scale (k_shadow)
        auto plane = [&](int qv) { return double(lo) + double(qv) * double(scale); };
        int ql = int(std::floor((double(n.lo[a][c]) - double(lo)) / double(scale)));
        ql = std::max(0, std::min(255, ql));
        while (ql > 0 && plane(ql) > double(n.lo[a][c])) --ql;
        int qh = int(std::ceil((double(n.hi[a][c]) - double(lo)) / double(scale)));
        qh = std::max(0, std::min(255, qh));
        while (qh < 255 && plane(qh) < double(n.hi[a][c])) ++qh;
        if (plane(ql) > double(n.lo[a][c]) || plane(qh) < double(n.hi[a][c]))
          throw std::runtime_error("quantize_wide: bound not representable");
        q.qlo[a][c] = uint8_t(ql);
        q.qhi[a][c] = uint8_t(qh);
      }
    }
  });
}

// The wide trees of the traversal kernels:
//  * `wide`: any-hit shadow rays -- a binned-SAH tree over the reference
//    BVH's leaves (default) or the reference tree itself
//    (RLC_SHADOW_TREE=reference), collapsed;
//  * `wide_ref`: closest-hit rays -- the reference tree collapsed with its
//    children in left-to-right order, so the reference's leaf order (right
//    subtree first) is a plain stack traversal; `wide_cam` (camera-relative
//    boxes) is filled in with the camera constants.
// Per binary node of a tree whose leaves are [a, a + count) ranges in DFS
// order (children after their parent): the [first, end) range it covers.
void node_ranges(const std::vector<BvhNode>& bin, std::vector<uint32_t>& first,
                 std::vector<uint32_t>& end) {
  first.assign(bin.size(), 0);
  end.assign(bin.size(), 0);
  for (size_t k = bin.size(); k-- > 0;) {
    const BvhNode& nd = bin[k];
    if (nd.count > 0) {
      first[k] = nd.a;
      end[k] = nd.a + nd.count;
    } else {
      first[k] = std::min(first[nd.a], first[nd.b]);
      end[k] = std::max(end[nd.a], end[nd.b]);
    }
  }
}

// shadow_bin's nodes grouped by depth, deepest first (children after their
// parent in the array, so depths come from one forward pass).
void bin_levels(const std::vector<BvhNode>& bin, std::vector<uint32_t>& order,
                std::vector<uint32_t>& level_start) {
  std::vector<uint32_t> depth(bin.size(), 0);
  uint32_t maxd = 0;
  for (size_t k = 0; k < bin.size(); ++k) {
    maxd = std::max(maxd, depth[k]);
    if (bin[k].count == 0) depth[bin[k].a] = depth[bin[k].b] = depth[k] + 1;
  }
  std::vector<uint32_t> cnt(maxd + 2, 0);
  for (uint32_t dd : depth) ++cnt[maxd - dd + 1];
  level_start.assign(maxd + 2, 0);
  for (uint32_t l = 1; l < maxd + 2; ++l) level_start[l] = level_start[l - 1] + cnt[l];
  order.assign(bin.size(), 0);
  std::vector<uint32_t> at(level_start.begin(), level_start.end() - 1);
  for (size_t k = 0; k < bin.size(); ++k) order[at[maxd - depth[k]]++] = uint32_t(k);
}

// Dynamic update, phase A (no reference BVH needed, so it runs beside its
// build): the creation SAH topology refitted to the moved triangles (any
// conservative tree is exact) -- shadow-order triangle
// records, binary node boxes bottom up by levels (leaves from their
// triangles' vertices, internal nodes from their children), every wide child
// box padded by S 2^-21 and rounded outward, and the quantized nodes.
// Leaf words keep the previous frame's kLeafPure bits until phase B.
void refit_shadow_boxes(const rlc_scene_desc& d, HostScene& out, const HostScene& base) {
  PhaseTimer pt;
  double S = 0;  // = max |coordinate| of the reference BVH's root box
  {
    std::vector<double> part(64, 0.0);
    const size_t nv = size_t(d.num_triangles) * 9;
    parallel_for(64, [&](size_t c) {
      double m = 0;
      for (size_t i = nv * c / 64; i < nv * (c + 1) / 64; ++i) m = std::max(m, std::fabs(d.vertices[i]));
      part[c] = m;
    }, 1);
    for (double m : part) S = std::max(S, m);
  }
  out.coord_bound = S;
  const size_t nt = base.tris_s.size();
  if (out.tris_s.size() != nt) out.tris_s = base.tris_s;  // triangle ids of the creation order
  parallel_for(nt, [&](size_t i) {
    TriAccel& ta = out.tris_s[i];
    const uint32_t id = ta.tri_id;
    const V3 p0 = vert(d, id, 0), p1 = vert(d, id, 1), p2 = vert(d, id, 2);
    put3(ta.p0, p0);
    put3(ta.e1, p1 - p0);
    put3(ta.e2, p2 - p0);
  });
  pt.lap("refit tris");
  const auto& kids = base.wide_kids;  // the creation topology
  const auto& bin = base.shadow_bin;
  std::vector<double>& nb = out.refit_box;  // scratch of this output scene
  nb.resize(6 * bin.size());
  const auto& order = base.bin_order;
  const auto& lstart = base.bin_level_start;
  for (size_t l = 0; l + 1 < lstart.size(); ++l) {
    const uint32_t l0 = lstart[l], l1 = lstart[l + 1];
    parallel_for(l1 - l0, [&](size_t q) {
      const uint32_t k = order[l0 + q];
      const BvhNode& nd = bin[k];
      Box bx;
      if (nd.count > 0) {
        for (uint32_t i = nd.a; i < nd.a + nd.count; ++i) {
          const uint32_t id = out.tris_s[i].tri_id;
          bx.grow(vert(d, id, 0));
          bx.grow(vert(d, id, 1));
          bx.grow(vert(d, id, 2));
        }
      } else {
        for (const uint32_t ch : {nd.a, nd.b}) {
          const double* c = &nb[6 * size_t(ch)];
          bx.grow(V3{c[0], c[1], c[2]});
          bx.grow(V3{c[3], c[4], c[5]});
        }
      }
      double* o = &nb[6 * size_t(k)];
      o[0] = bx.lo.x, o[1] = bx.lo.y, o[2] = bx.lo.z, o[3] = bx.hi.x, o[4] = bx.hi.y, o[5] = bx.hi.z;
    }, 512);
  }
  pt.lap("refit boxes");
  const double pad = S * 0x1.0p-21;
  // internal child words: the creation numbering; boxes rewritten below, leaf
  // words in phase B
  if (out.wide.size() != base.wide.size()) out.wide = base.wide;
  parallel_for(kids.size(), [&](size_t w) {
    Wide4& n = out.wide[w];
    for (int c = 0; c < kWide; ++c) {
      const uint32_t b = kids[w][c];
      if (b == kWideEmpty) {
        n.child[c] = kWideEmpty;
        for (int a = 0; a < 3; ++a) {
          n.lo[a][c] = HUGE_VALF;
          n.hi[a][c] = -HUGE_VALF;
        }
        continue;
      }
      const double* bx = &nb[6 * size_t(b)];
      for (int a = 0; a < 3; ++a) {  // as collapse_wide (no origin, no growth)
        n.lo[a][c] = round_down(bx[a] - pad);
        n.hi[a][c] = round_up(bx[3 + a] + pad);
      }
    }
  }, 512);
  pt.lap("wide refit");
  const char* q = std::getenv("RLC_SHADOW_QUANT");
  if (q && std::string(q) == "0") out.wide_q.clear();
  else quantize_wide(out.wide, out.wide_q);
  pt.lap("quantize");
}

// Phase B, after the reference BVH: the reference leaf of every shadow-order
// triangle, and kLeafPure on the leaves whose triangles all lie in one
// reference leaf (patched into the wide and the quantized nodes).
void refit_shadow_leaves(HostScene& out, const HostScene& base) {
  std::vector<uint32_t>& leaf_of_id = out.refit_leaf;  // scratch reused across updates
  leaf_of_id.resize(out.tris.size());
  parallel_for(out.tris.size(), [&](size_t j) { leaf_of_id[out.tris[j].tri_id] = out.tri_leaf[j]; });
  const size_t nt = out.tris_s.size();
  out.tri_leaf_s.resize(nt);
  parallel_for(nt, [&](size_t i) { out.tri_leaf_s[i] = leaf_of_id[out.tris_s[i].tri_id]; });
  const auto& kids = base.wide_kids;
  const auto& bin = base.shadow_bin;
  const bool quant = !out.wide_q.empty();
  parallel_for(kids.size(), [&](size_t w) {
    for (int c = 0; c < kWide; ++c) {
      const uint32_t b = kids[w][c];
      if (b == kWideEmpty) continue;
      const BvhNode& bn = bin[b];
      if (bn.count == 0) continue;  // internal: the creation numbering, already in place
      bool pure = true;
      for (uint32_t k = 1; k < bn.count; ++k) pure &= out.tri_leaf_s[bn.a + k] == out.tri_leaf_s[bn.a];
      const uint32_t word = kWideLeaf | ((bn.count - 1) << 28) | (pure ? kLeafPure : 0u) | bn.a;
      out.wide[w].child[c] = word;
      if (quant) out.wide_q[w].child[c] = word;
    }
  }, 512);
}

void build_wide(const rlc_scene_desc& d, HostScene& out, const HostScene* keep, bool refit) {
  PhaseTimer pt;
  if (!refit) out.wide.clear();  // (refit: the boxes of refit_shadow_boxes)
  out.wide_ref.clear();
  out.tri_leaf.assign(out.tris.size(), 0);
  parallel_for(out.nodes.size(), [&](size_t i) {
    for (uint32_t t = out.nodes[i].a; out.nodes[i].count > 0 && t < out.nodes[i].a + out.nodes[i].count; ++t)
      out.tri_leaf[t] = uint32_t(i);
  });
  pt.lap("tri_leaf");
  if (out.nodes.empty() || out.nodes[0].count > 0) {  // a leaf root: exact paths only
    out.tris_s = out.tris;
    out.tri_leaf_s = out.tri_leaf;
    return;
  }
  if (out.tris.size() >= (1u << 27)) throw InvalidArgument("build_scene_bvh: too many triangles");
  // the closest-hit trees depend only on the reference BVH: built beside the shadow tree
  auto f_ref = std::async(std::launch::async, [&] {
    if (keep == nullptr) out.wide_ref = collapse_wide(out.nodes, nullptr);
  });
  // shadow tree: SAH over triangles (default), over the reference leaves
  // (RLC_SHADOW_TREE=leaves) or the reference tree (=reference)
  const char* env = std::getenv("RLC_SHADOW_TREE");
  const std::string mode = env ? env : "tris";
  const bool use_ref = mode == "reference";
  // Shadow-tree boxes are padded by S 2^-21 (S = the largest |coordinate| of
  // the scene): more than the fp32 error of t = fma(c, inv, -(o inv)) for any
  // origin within S, so k_shadow's plain slab test is conservative.
  double S = 0;
  for (int a = 0; a < 3; ++a)
    S = std::max(S, std::max(std::fabs(out.nodes[0].lo[a]), std::fabs(out.nodes[0].hi[a])));
  out.coord_bound = S;
  if (mode == "reference" || mode == "leaves") {
    out.tris_s = out.tris;
    out.tri_leaf_s = out.tri_leaf;
    out.wide = collapse_wide(use_ref ? out.nodes : sah_over_leaves(out.nodes), nullptr, 0.0,
                             S * 0x1.0p-21);
  } else if (refit && out.gpu_refit) {
    // the device refits the tree (launch_refit_shadow): it needs the reference
    // leaf of every triangle id
    out.refit_leaf.resize(out.tris.size());
    parallel_for(out.tris.size(), [&](size_t j) { out.refit_leaf[out.tris[j].tri_id] = out.tri_leaf[j]; });
    out.tris_s.clear();
    out.tri_leaf_s.clear();
    out.wide.clear();
    out.wide_q.clear();
  } else if (refit) {
    refit_shadow_leaves(out, *keep);  // the boxes were refitted beside the reference BVH
  } else {
    std::vector<uint32_t> perm;
    out.tris_s.resize(out.tris.size());
    out.tri_leaf_s.resize(out.tris.size());
    out.shadow_bin = sah_over_tris(d, out, perm);
    for (size_t i = 0; i < perm.size(); ++i) {
      out.tris_s[i] = out.tris[perm[i]];
      out.tri_leaf_s[i] = out.tri_leaf[perm[i]];
    }
    out.wide = collapse_wide(out.shadow_bin, nullptr, 0.0, S * 0x1.0p-21, &out.tri_leaf_s,
                             &out.wide_kids);
    node_ranges(out.shadow_bin, out.bin_first, out.bin_end);
    bin_levels(out.shadow_bin, out.bin_order, out.bin_level_start);
  }
  f_ref.get();
  pt.lap("wide_ref");
  if (refit) return;  // quantized in refit_shadow_boxes, leaf bits patched above
  const char* q = std::getenv("RLC_SHADOW_QUANT");
  if (q && std::string(q) == "0") out.wide_q.clear();
  if (!(q && std::string(q) == "0")) quantize_wide(out.wide, out.wide_q);
  pt.lap("quantize");
}

}  // namespace

void build_light_tree(const std::vector<double>& centroids, const std::vector<double>& energy,
                      std::vector<uint32_t>& order, std::vector<LtNode>& nodes,
                      std::vector<uint32_t>& node_begin, std::vector<double>& node_energy) {
  const uint32_t n = uint32_t(energy.size());
  if (n == 0) throw InvalidArgument("build_light_tree: no emitters");
  Box cb;  // emitter_centroid_bounds, light_tree.cpp:50-54
  for (uint32_t i = 0; i < n; ++i)
    cb.grow(V3{centroids[3 * i], centroids[3 * i + 1], centroids[3 * i + 2]});
  const V3 lo = cb.lo - V3{1e-6, 1e-6, 1e-6};
  const V3 e0 = cb.extent() + V3{2e-6, 2e-6, 2e-6};
  const V3 ext{smax(e0.x, 1e-12), smax(e0.y, 1e-12), smax(e0.z, 1e-12)};

  std::vector<uint64_t> keyed(n);  // (code << 32) | emitter: the total order
  for (uint32_t i = 0; i < n; ++i) {
    const V3 rel = V3{centroids[3 * i], centroids[3 * i + 1], centroids[3 * i + 2]} - lo;
    uint32_t qa[3];
    for (int a = 0; a < 3; ++a) {
      const double s = comp(rel, a) / comp(ext, a) * 1024.0;
      qa[a] = uint32_t(smin(1023.0, smax(0.0, s)));
    }
    const uint32_t code = spread10(qa[0]) | (spread10(qa[1]) << 1) | (spread10(qa[2]) << 2);
    keyed[i] = (uint64_t(code) << 32) | i;
  }
  std::sort(keyed.begin(), keyed.end());
  order.resize(n);
  std::vector<uint32_t> code(n);
  for (uint32_t i = 0; i < n; ++i) {
    order[i] = uint32_t(keyed[i]);
    code[i] = uint32_t(keyed[i] >> 32);
  }

  nodes.assign(0, LtNode{});
  nodes.reserve(size_t(2) * n);
  node_begin.clear();
  node_begin.reserve(size_t(2) * n);
  struct Todo {
    uint32_t begin, end;
    int32_t parent;
    int side;  // 0 left child of parent, 1 right child
  };
  std::vector<Todo> todo{{0, n, -1, 0}};
  while (!todo.empty()) {  // preorder: node, then left subtree, then right subtree
    const Todo t = todo.back();
    todo.pop_back();
    const int32_t id = int32_t(nodes.size());
    nodes.push_back(LtNode{t.end, -1, -1, t.parent});
    node_begin.push_back(t.begin);
    if (t.parent >= 0) {
      if (t.side == 0) nodes[size_t(t.parent)].left = id;
      else nodes[size_t(t.parent)].right = id;
    }
    if (t.end - t.begin == 1) continue;
    const uint32_t first = code[t.begin], last = code[t.end - 1];
    uint32_t mid;
    if (first == last) {
      mid = t.begin + (t.end - t.begin) / 2;
    } else {
      const int bit = 31 - __builtin_clz(first ^ last);
      const uint32_t cut = (first & ~((1u << (bit + 1)) - 1u)) | (1u << bit);
      mid = uint32_t(std::lower_bound(code.begin() + t.begin, code.begin() + t.end, cut) -
                     code.begin());
    }
    todo.push_back({mid, t.end, id, 1});
    todo.push_back({t.begin, mid, id, 0});
  }
  node_energy.assign(nodes.size(), 0.0);
  for (size_t k = nodes.size(); k-- > 0;) {  // children carry larger preorder ids
    if (nodes[k].left < 0) node_energy[k] = energy[order[node_begin[k]]];
    else node_energy[k] = node_energy[size_t(nodes[k].left)] + node_energy[size_t(nodes[k].right)];
  }
}

HostCut make_template_cut(const std::vector<LtNode>& nodes, const std::vector<uint32_t>& begin,
                          const std::vector<double>& energy, uint32_t light_count, uint32_t M,
                          double eps_q) {
  if (M == 0) throw InvalidArgument("init_cut: cut size must be positive");
  const uint32_t target = std::min(M, light_count);
  std::deque<uint32_t> frontier_q{0u};
  std::vector<uint32_t> done;
  uint32_t count = 1;
  while (count < target && !frontier_q.empty()) {  // breadth-first, cut.cpp:36-50
    const uint32_t id = frontier_q.front();
    frontier_q.pop_front();
    if (nodes[id].left < 0) {
      done.push_back(id);
    } else {
      frontier_q.push_back(uint32_t(nodes[id].left));
      frontier_q.push_back(uint32_t(nodes[id].right));
      ++count;
    }
  }
  done.insert(done.end(), frontier_q.begin(), frontier_q.end());
  std::sort(done.begin(), done.end(), [&](uint32_t a, uint32_t b) { return begin[a] < begin[b]; });

  HostCut c;
  const uint32_t m = uint32_t(done.size());
  c.node_ids = done;
  c.eps_q = eps_q < 0 ? 1e-4 / double(m) : eps_q;
  c.ends.resize(m);
  c.q.resize(m);
  c.cdf.resize(m);
  c.visits.assign(m, 1u);
  double total = 0;
  for (uint32_t i = 0; i < m; ++i) {
    c.ends[i] = nodes[done[i]].range_end;
    total += energy[done[i]];
  }
  double run = 0;
  for (uint32_t i = 0; i < m; ++i) {
    const double e = energy[done[i]];
    const double share = total > 0 ? e / total : 1.0 / double(m);
    c.q[i] = smax(share, c.eps_q);
    run += c.q[i];
    c.cdf[i] = run;
  }
  return c;
}

void level_thresholds(double out[kMaxLevel + 1]) {
  auto level_of = [](double r) {
    const double l = std::round(std::log2(r));
    return uint32_t(clampd(l, 0.0, double(kMaxLevel)));
  };
  out[0] = 0.0;
  for (uint32_t k = 1; k <= kMaxLevel; ++k) {
    uint64_t lo = 1, hi = 0x7fefffffffffffffull;  // level(lo) < k <= level(hi)
    while (hi - lo > 1) {
      const uint64_t mid = lo + (hi - lo) / 2;
      double r;
      std::memcpy(&r, &mid, 8);
      if (level_of(r) >= k) hi = mid;
      else lo = mid;
    }
    std::memcpy(&out[k], &hi, 8);
  }
}

void build_reference_bvh(const rlc_scene_desc& d, HostScene& out) { build_bvh(d, out); }

void build_host_scene(const rlc_scene_desc& d, const rlc_render_config& cfg, HostScene& out,
                      const HostScene* keep) {
  PhaseTimer pt;
  if (d.num_triangles == 0 || d.vertices == nullptr || d.material_ids == nullptr)
    throw InvalidArgument("build_scene_bvh: empty scene");
  if (d.num_materials == 0 || d.materials == nullptr)
    throw InvalidArgument("build_context: scene has no materials");
  if (d.width <= 0 || d.height <= 0) throw InvalidArgument("build_context: empty camera raster");
  for (uint32_t t = 0; t < d.num_triangles; ++t)
    if (d.material_ids[t] >= d.num_materials)
      throw OutOfRange("build_context: material id out of range");

  // A dynamic update (keep = the context's creation scene, read only) writes
  // into `out`'s own buffers: an output scene recycled from an earlier update
  // touches no fresh pages, and several updates can be built at once.
  out.mat_values.assign(d.materials, d.materials + size_t(d.num_materials) * 6);
  out.mats.resize(d.num_materials);
  for (uint32_t m = 0; m < d.num_materials; ++m) {
    const double* v = d.materials + size_t(m) * 6;
    MatRec& r = out.mats[m];
    for (int a = 0; a < 3; ++a) {
      r.albedo[a] = v[a];
      r.emission[a] = v[3 + a];
    }
    r.is_emitter = luminance(V3{v[3], v[4], v[5]}) > 0 ? 1u : 0u;
    r.reflective = luminance(V3{v[0], v[1], v[2]}) > 0 ? 1u : 0u;
  }
  out.tri_mat.assign(d.material_ids, d.material_ids + d.num_triangles);
  out.tri_normal.resize(size_t(3) * d.num_triangles);
  parallel_for(d.num_triangles, [&](size_t t) {
    const V3 p0 = vert(d, uint32_t(t), 0);
    put3(&out.tri_normal[3 * t],
         normalize(cross(vert(d, uint32_t(t), 1) - p0, vert(d, uint32_t(t), 2) - p0)));
  });
  pt.lap("normals");
  // A dynamic update refits the creation shadow tree; its boxes do not
  // depend on the reference BVH, so they are refitted beside its build.
  const char* tree_env = std::getenv("RLC_SHADOW_TREE");
  const bool refit = keep != nullptr && !keep->shadow_bin.empty() && !keep->wide_kids.empty() &&
                     !(tree_env && (std::string(tree_env) == "reference" ||
                                    std::string(tree_env) == "leaves"));
  // RLC_HOST_REFIT=1: the shadow tree refitted here instead of on the device
  const bool host_refit = std::getenv("RLC_HOST_REFIT") != nullptr;
  out.gpu_refit = refit && !host_refit;
  std::future<void> f_boxes;
  if (refit && !out.gpu_refit) {
    f_boxes = std::async(std::launch::async, [&] {
      WorkerPool::priority() = 0;  // the reference BVH's loops go first
      refit_shadow_boxes(d, out, *keep);
    });
  }
  build_bvh(d, out);  // render.cpp:145
  pt.lap("reference bvh");
  if (refit && !out.gpu_refit) f_boxes.get();
  pt.lap("refit join");
  // The rest depends only on the scene and the reference BVH and writes
  // disjoint parts of `out`: the traversal trees, the emitters and light
  // tree, and the camera-relative copies run concurrently.
  auto f_wide = std::async(std::launch::async, [&] { build_wide(d, out, keep, refit); });
  auto f_emit = std::async(std::launch::async, [&] {
    if (keep == nullptr) {  // fp32 reference-tree copy: deferred closest-hit rays only
      out.nodes_f.resize(out.nodes.size());
      for (size_t i = 0; i < out.nodes.size(); ++i) {
        const BvhNode& n = out.nodes[i];
        BvhNodeF& f = out.nodes_f[i];
        for (int a = 0; a < 3; ++a) {
          f.lo[a] = round_down(n.lo[a]);
          f.hi[a] = round_up(n.hi[a]);
        }
        if (n.count > 0) {
          f.a = kNodeLeaf | n.a;
          f.b = n.count;
        } else {
          if (n.b != n.a + 1) throw std::runtime_error("build_scene_bvh: siblings must be adjacent");
          f.a = n.a;
          f.b = 0;
        }
      }
    }

    // collect_emitters (light_tree.cpp:30-42) over derive_emitters order;
    // a dynamic update keeps the materials, hence the emitter list
    auto emitter = [&](uint32_t t, size_t k) {
      const MatRec& m = out.mats[d.material_ids[t]];
      const V3 p0 = vert(d, t, 0), p1 = vert(d, t, 1), p2 = vert(d, t, 2);
      const V3 cr = cross(p1 - p0, p2 - p0);
      const double area = 0.5 * length(cr);
      const V3 c = (p0 + p1 + p2) / 3.0;
      LightRec& lr = out.lights[k];
      lr = LightRec{};
      put3(lr.p0, p0);
      put3(lr.p1, p1);
      put3(lr.p2, p2);
      put3(lr.n, normalize(cr));
      for (int a = 0; a < 3; ++a) lr.emission[a] = m.emission[a];
      // sample_triangle_point throws on area <= 0 (scene.cpp:50-51); the
      // device checks pdf_area <= 0 and raises the same error when drawn.
      lr.pdf_area = area > 0 ? 1.0 / area : 0.0;
      out.emitter_energy[k] = luminance(V3{m.emission[0], m.emission[1], m.emission[2]}) * area;
      out.emitter_centroid[3 * k] = c.x;
      out.emitter_centroid[3 * k + 1] = c.y;
      out.emitter_centroid[3 * k + 2] = c.z;
    };
    if (keep != nullptr) {
      out.emitter_tri = keep->emitter_tri;
    } else {
      out.emitter_tri.clear();
      for (uint32_t t = 0; t < d.num_triangles; ++t)
        if (out.mats[d.material_ids[t]].is_emitter) out.emitter_tri.push_back(t);
    }
    const size_t ne = out.emitter_tri.size();
    out.emitter_mat.resize(ne);
    for (size_t k = 0; k < ne; ++k) out.emitter_mat[k] = d.material_ids[out.emitter_tri[k]];
    out.lights.resize(ne);
    out.emitter_energy.resize(ne);
    out.emitter_centroid.resize(3 * ne);
    parallel_for(ne, [&](size_t k) { emitter(out.emitter_tri[k], k); });
    if (out.lights.empty()) throw InvalidArgument("build_context: scene has no emitters");
    if (!keep) {  // (a dynamic update moves the creation light tree over at the end)
      build_light_tree(out.emitter_centroid, out.emitter_energy, out.order, out.lt_nodes,
                       out.lt_begin, out.lt_energy);
    }

    out.energy_cdf.resize(out.emitter_energy.size());  // estimators.cpp:12-26
    double run = 0;
    for (size_t i = 0; i < out.emitter_energy.size(); ++i) {
      run += out.emitter_energy[i];
      out.energy_cdf[i] = run;
    }
    if (!(out.energy_cdf.back() > 0))
      throw InvalidArgument("build_energy_cdf: total emitter energy must be positive");
    pt.lap("emitters");

  });
  const V3 ext = V3{out.scene_hi[0], out.scene_hi[1], out.scene_hi[2]} -
                 V3{out.scene_lo[0], out.scene_lo[1], out.scene_lo[2]};
  out.base_tile = cfg.hash.base_tile > 0 ? cfg.hash.base_tile : length(ext) / 256.0;

  // camera_ray / pixel_solid_angle constants (scene.cpp:10-31)
  CameraConst& cam = out.cam;
  const V3 org{d.cam_origin[0], d.cam_origin[1], d.cam_origin[2]};
  const V3 look{d.cam_look_at[0], d.cam_look_at[1], d.cam_look_at[2]};
  const V3 up{d.cam_up[0], d.cam_up[1], d.cam_up[2]};
  const V3 w = normalize(org - look);
  const V3 u = normalize(cross(up, w));
  const V3 v = cross(w, u);
  put3(cam.origin, org);
  put3(cam.u, u);
  put3(cam.v, v);
  put3(cam.w, w);
  cam.tan_half = std::tan(0.5 * d.vfov_degrees * kPi / 180.0);
  cam.aspect = double(d.width) / double(d.height);
  cam.width = d.width;
  cam.height = d.height;
  cam.width_d = double(d.width);
  cam.height_d = double(d.height);
  const double plane_h = 2.0 * cam.tan_half;
  const double plane_w = plane_h * cam.aspect;
  cam.pdf_omega = 1.0 / ((plane_w / d.width) * (plane_h / d.height));

  level_thresholds(out.level_threshold);

  // Camera-relative copy for the primary rays, whose origin is exactly the
  // camera origin O: the reference's per-axis term fl64(c - O) rounded
  // outward to fp32, so every fp32 error of the decision test is relative.
  if (keep == nullptr) out.nodes_cam.resize(out.nodes.size());
  if (keep == nullptr) parallel_for(out.nodes.size(), [&](size_t i) {
    const BvhNode& n = out.nodes[i];
    BvhNodeF& f = out.nodes_cam[i];
    for (int a = 0; a < 3; ++a) {
      f.lo[a] = round_down(n.lo[a] - cam.origin[a]);
      f.hi[a] = round_up(n.hi[a] - cam.origin[a]);
    }
    f.a = n.count > 0 ? (kNodeLeaf | n.a) : n.a;
    f.b = n.count > 0 ? n.count : 0;
  });
  // The wide copy for camera rays is enlarged by 2^-21 |x| per coordinate,
  // more than the whole relative gap between fl32(x' * fl32(inv)) and the
  // reference's fl64(x * inv) (< 2^-23): its plain slab test is conservative
  // (DESIGN.md 5.4).
  out.wide_cam.clear();
  if (out.nodes[0].count == 0 && keep == nullptr)
    out.wide_cam = collapse_wide(out.nodes, cam.origin, 0x1.0p-21);
  pt.lap("camera copies");
  f_wide.get();
  pt.lap("wide join");
  f_emit.get();
  pt.lap("emit join");
}

void parallel_copy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kChunk = size_t(1) << 20;
  const size_t n = (bytes + kChunk - 1) / kChunk;
  parallel_for(n, [&](size_t i) {
    const size_t b = i * kChunk, e = std::min(bytes, b + kChunk);
    std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
  }, 1);
}

}  // namespace rlc
