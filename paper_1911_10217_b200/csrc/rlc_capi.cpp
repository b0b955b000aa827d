// rlc_capi.cpp -- the C-ABI drop-in boundary (include/rlcuts_b200.h) and the
// host runtime behind it: device-resident context, hash grid and framebuffer,
// and the per-pass launch sequence.  There is no CPU fallback: without an
// sm_100 device every create call fails with RLC_ERR_NO_DEVICE.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <future>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "rlc_build.h"
#include "rlc_kernels.h"
#include "rlc_libm.h"
#include "rlc_sincostab.h"
#include "rlcuts_b200.h"

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define RLC_CK(x)                                                                       \
  do {                                                                                  \
    const cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess)                                                              \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                 \
  } while (0)

template <class F>
rlc_status guarded(F&& f) {
  try {
    f();
    return RLC_OK;
  } catch (const NoDevice& e) {
    g_err = e.what();
    return RLC_ERR_NO_DEVICE;
  } catch (const rlc::ImageIoError& e) {
    g_err = e.what();
    return rlc_status(e.code());
  } catch (const CudaError& e) {
    g_err = e.what();
    return RLC_ERR_CUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RLC_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return RLC_ERR_OUT_OF_RANGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RLC_ERR_INTERNAL;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) throw rlc::InvalidArgument(msg);
}

// Owns a set of device allocations.
struct DeviceArena {
  std::vector<void*> ptrs;
  uint64_t bytes = 0;
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    const size_t b = count * sizeof(T) > 0 ? count * sizeof(T) : 16;
    RLC_CK(cudaMalloc(&p, b));
    ptrs.push_back(p);
    bytes += b;
    return static_cast<T*>(p);
  }
  // ordered on stream st; the caller synchronizes st before freeing v
  template <class T>
  T* upload(const std::vector<T>& v, cudaStream_t st) {
    T* p = alloc<T>(v.size());
    if (!v.empty())
      RLC_CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return p;
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
    bytes = 0;
  }
  ~DeviceArena() { release(); }
};

// A pass's new-key table (rlc::NewKeys) for up to n lookups: 2^k >= 2n
// entries, cleared once here and then by k_commit after every pass.
rlc::NewKeys alloc_new_keys(DeviceArena& A, uint64_t n, cudaStream_t st) {
  uint64_t cap = 1024;
  while (cap < 2 * n) cap <<= 1;
  rlc::NewKeys nk{};
  nk.keys = A.alloc<unsigned long long>(2 * cap);
  nk.id = A.alloc<uint32_t>(cap);
  nk.list = A.alloc<uint32_t>(cap);
  nk.count = A.alloc<unsigned int>(1);
  nk.mask = uint32_t(cap - 1);
  RLC_CK(cudaMemsetAsync(nk.keys, 0, 16 * cap, st));
  RLC_CK(cudaMemsetAsync(nk.id, 0xff, 4 * cap, st));
  RLC_CK(cudaMemsetAsync(nk.count, 0, 4, st));
  return nk;
}

// The scene arrays of a context: one device buffer per array, in the fixed
// order of upload_scene, reused by rlc_context_update_scene while the new
// contents fit (a frame's arrays have nearly the same sizes), so a scene
// update is a copy, not a reallocation.
struct SceneBuffers {
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  std::vector<Buf> bufs;
  size_t next = 0;
  uint64_t bytes = 0;
  // Dynamic scene updates write into recycled host scenes (one per update in
  // flight), whose buffers keep their addresses from one update to the next:
  // the large ones are page-locked once each (cudaHostRegister) and then
  // DMA'd at full rate instead of being staged by the driver.
  bool pin = false;
  cudaStream_t stream = nullptr;  // the context stream the copies are ordered on
  std::vector<std::pair<const void*, size_t>> pinned;
  void begin(cudaStream_t st, bool pin_sources = false) {
    next = 0;
    stream = st;
    pin = pin_sources;
  }
  void ensure_pinned(const void* src, size_t n) {
    for (auto& pr : pinned) {
      if (pr.first != src) continue;
      if (pr.second >= n) return;
      cudaHostUnregister(const_cast<void*>(pr.first));  // grown in place: re-register
      cudaGetLastError();
      pr.second = 0;
      if (cudaHostRegister(const_cast<void*>(src), n, cudaHostRegisterDefault) == cudaSuccess)
        pr.second = n;
      else
        cudaGetLastError();
      return;
    }
    if (cudaHostRegister(const_cast<void*>(src), n, cudaHostRegisterDefault) == cudaSuccess)
      pinned.emplace_back(src, n);
    else
      cudaGetLastError();  // not pinnable: the pageable copy still works
  }
  // copy = false: the contents are known unchanged since the last upload
  // into this slot (a dynamic scene update's frozen arrays)
  template <class T>
  T* put(const std::vector<T>& v, bool copy = true) {
    if (next == bufs.size()) bufs.emplace_back();
    Buf& b = bufs[next++];
    const size_t need = v.size() * sizeof(T) > 0 ? v.size() * sizeof(T) : 16;
    if (need > b.cap) {
      copy = true;
      if (b.p) RLC_CK(cudaFree(b.p));
      b.p = nullptr;
      bytes -= b.cap;
      const size_t cap = need + need / 8;  // headroom for the next frame
      RLC_CK(cudaMalloc(&b.p, cap));
      b.cap = cap;
      bytes += cap;
    }
    if (copy && !v.empty()) {
      const size_t n = v.size() * sizeof(T);
      if (pin && n >= (size_t(1) << 20)) ensure_pinned(v.data(), n);
      RLC_CK(cudaMemcpyAsync(b.p, v.data(), n, cudaMemcpyHostToDevice, stream));
    }
    return static_cast<T*>(b.p);
  }
  // host memory pinned for this context must be released before it is freed
  void unpin_all() {
    for (auto& pr : pinned) cudaHostUnregister(const_cast<void*>(pr.first));
    cudaGetLastError();
    pinned.clear();
  }
  ~SceneBuffers() {
    unpin_all();
    for (Buf& b : bufs)
      if (b.p) cudaFree(b.p);
  }
};

void check_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw NoDevice("no CUDA device: the rlcuts_b200 path has no CPU fallback");
  }
  if (device < 0 || device >= n) throw rlc::InvalidArgument("rlc_context_create: bad device index");
  cudaDeviceProp prop;
  RLC_CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    throw NoDevice("rlcuts_b200 is built for sm_100a (B200); device " + std::string(prop.name) +
                   " is not supported");
  RLC_CK(cudaSetDevice(device));
}

const double kSinCosTabHost[440] = RLC_SINCOSTAB_INIT;

// The x86-64 glibc build of sin/cos the host libm dispatches to (rlc_libm.h):
// the host restatement of each build is compared with std::sin / std::cos on
// angles that separate the two builds and on 4096 sampler angles 2 pi u.
// kUnknown if neither matches everywhere (then bounce directions cannot be
// reproduced and max_depth > 1 is refused).
int probe_libm_variant() {
  static const int variant = [] {
    std::vector<double> xs = {0x1.47750e7b60563p+0, 0x1.de8813a4f28cap+0, 0x1.2ce0bf964b8acp+1,
                              0x1.68e5b478ea497p+0};
    uint64_t st = 0x243f6a8885a308d3ull;
    for (int i = 0; i < 4096; ++i) {
      st = rlc::mix64(st + 0x9e3779b97f4a7c15ull);
      xs.push_back(2.0 * rlc::kPi * (double(st >> 11) * 0x1.0p-53));
    }
    for (const int cand : {rlc::libm::kFma, rlc::libm::kSse2}) {
      const rlc::libm::Ctx c{kSinCosTabHost, cand == rlc::libm::kFma};
      bool ok = true;
      for (const double x : xs) {
        volatile double vx = x;  // a runtime libm call, never a compile-time fold
        const double hs = std::sin(vx), hc = std::cos(vx);
        if (hs != rlc::libm::sin(c, x) || hc != rlc::libm::cos(c, x)) {
          ok = false;
          break;
        }
      }
      if (ok) return cand;
    }
    return int(rlc::libm::kUnknown);
  }();
  return variant;
}

const char* device_error_message(uint32_t bits) {
  if (bits & rlc::kErrNonUnitNormal) return "make_key: normal must be unit length";
  if (bits & rlc::kErrBadValue) return "update_q: value must be finite and non-negative";
  if (bits & rlc::kErrDegenerateLight) return "sample_triangle_point: degenerate triangle";
  if (bits & rlc::kErrBadAreaPdf) return "level_for_footprint: area pdf must be positive";
  if (bits & rlc::kErrStackOverflow) return "scene BVH deeper than the 64-entry traversal stack";
  if (bits & rlc::kErrNewKeyOverflow) return "hash grid: new-key table of the pass overflowed";
  if (bits & rlc::kErrCheck) return "device bounds check failed (RLC_DEBUG_CHECKS build)";
  return "device error";
}

}  // namespace

struct PassParamsHolder {
  rlc::PassParams p{};
  rlc::DevGrid g{};
  uint32_t n = 0;
  uint32_t nv = 0;
  const rlc_grid* grid = nullptr;
  bool valid = false;
};

struct rlc_context {
  // Grids and framebuffers keep their context alive: the caller's reference
  // plus one per live child, so destroying the context before its children
  // (any order a garbage collector picks) defers the teardown to the last
  // child.  The render_frame cache's own grid/framebuffer hold no reference.
  std::atomic<int> refs{1};
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  rlc::HostScene host;
  rlc::DevScene dev{};
  rlc_render_config create_cfg{};  // build_context's config (rlc_context_update_scene)
  // dynamic updates built ahead (rlc_context_prepare_scene): each builds on a
  // worker thread from its own copy of the vertices, against the creation
  // scene `host` (read only), into its own recycled output scene
  struct FrameScene {
    rlc::HostScene h;
    std::vector<double> vertices;
    rlc_scene_desc desc{};
    std::future<void> build;
    uint64_t token = 0;
    bool busy = false;
  };
  std::vector<std::unique_ptr<FrameScene>> frame_scenes;
  // device refit of the shadow tree for dynamic updates: the creation
  // topology (uploaded at the first update) and the refitted arrays
  DeviceArena refit_arena;
  rlc::RefitTopo refit{};
  rlc::TriAccel* refit_tris_s = nullptr;
  uint32_t* refit_tri_leaf_s = nullptr;
  rlc::Wide4* refit_wide = nullptr;
  rlc::WideQ* refit_wide_q = nullptr;
  void ensure_refit_topology() {
    if (refit.num_wide) return;
    const rlc::HostScene& h = host;
    const uint32_t nb = uint32_t(h.shadow_bin.size()), nw = uint32_t(h.wide_kids.size());
    const uint32_t nt = uint32_t(h.tris_s.size());
    std::vector<uint32_t> a(nb), b(nb), cnt(nb), parent(nb, 0xffffffffu), leaves;
    for (uint32_t k = 0; k < nb; ++k) {
      const rlc::BvhNode& n = h.shadow_bin[k];
      a[k] = n.a;
      b[k] = n.b;
      cnt[k] = n.count;
      if (n.count > 0) {
        leaves.push_back(k);
      } else {
        parent[n.a] = k;
        parent[n.b] = k;
      }
    }
    std::vector<uint32_t> kids(4 * size_t(nw)), base(4 * size_t(nw)), ids(nt);
    for (uint32_t w = 0; w < nw; ++w)
      for (int c = 0; c < 4; ++c) {
        kids[4 * size_t(w) + c] = h.wide_kids[w][c];
        base[4 * size_t(w) + c] = h.wide[w].child[c];
      }
    for (uint32_t i = 0; i < nt; ++i) ids[i] = h.tris_s[i].tri_id;
    DeviceArena& A = refit_arena;
    refit.bin_a = A.upload(a, stream);
    refit.bin_b = A.upload(b, stream);
    refit.bin_count = A.upload(cnt, stream);
    refit.bin_parent = A.upload(parent, stream);
    refit.bin_leaves = A.upload(leaves, stream);
    refit.num_bin = nb;
    refit.num_leaves = uint32_t(leaves.size());
    refit.kids = A.upload(kids, stream);
    refit.base_child = A.upload(base, stream);
    refit.tri_ids = A.upload(ids, stream);
    refit.num_tris = nt;
    refit.box = A.alloc<double>(6 * size_t(nb));
    refit.arrive = A.alloc<unsigned int>(nb);
    refit_tris_s = A.alloc<rlc::TriAccel>(nt);
    refit_tri_leaf_s = A.alloc<uint32_t>(nt);
    if (h.wide_q.empty()) refit_wide = A.alloc<rlc::Wide4>(nw);
    else refit_wide_q = A.alloc<rlc::WideQ>(nw);
    RLC_CK(cudaStreamSynchronize(stream));  // the host vectors above go out of scope
    refit.num_wide = nw;
  }
  uint64_t next_scene_token = 1;
  SceneBuffers scene_bufs;  // the device scene (upload_scene)
  DeviceArena lights_ord_arena;  // dev.lights_ord, rebuilt on the device after every upload
  size_t lights_ord_cap = 0;
  void build_light_order() {
    if (dev.num_lights > lights_ord_cap) {
      lights_ord_arena.release();
      dev.lights_ord = lights_ord_arena.alloc<rlc::LightOrd>(dev.num_lights);
      lights_ord_cap = dev.num_lights;
    }
    rlc::launch_light_order(dev, const_cast<rlc::LightOrd*>(dev.lights_ord), stream);
    RLC_CK(cudaGetLastError());
  }
  DeviceArena arena;
  unsigned long long* counters = nullptr;  // error bits for grid-less passes
  // primary rays of the next pass overlap the tail of the current one: they
  // run on `pstream` into the other G-buffer slot
  cudaStream_t pstream = nullptr;
  cudaStream_t sstream = nullptr;  // the record sort beside the shadow rays, the
                                   // framebuffer accumulation beside split-collapse
  cudaEvent_t ev_sample_done = nullptr, ev_sort_done = nullptr;
  cudaEvent_t ev_fold_done = nullptr, ev_acc_done = nullptr;
  bool acc_pending = false;  // an accumulation on sstream the main stream has not joined
  // Orders every later main-stream operation after the side-stream
  // accumulation (framebuffer and pass-buffer readers/writers call this).
  void join_acc() {
    if (!acc_pending) return;
    RLC_CK(cudaStreamWaitEvent(stream, ev_acc_done, 0));
    acc_pending = false;
  }
  bool overlap = true;  // primary rays of the next pass on a side stream (RLC_OVERLAP=0: off)
  cudaEvent_t ev_prim_done = nullptr;
  // Orders all later side-stream work after everything enqueued on the main
  // stream so far.  The next pass's primary rays wait only for their G-buffer
  // slot, so a main-stream write they read (a grid reset, a fresh grid's
  // slots, a scene upload) must be followed by this fence.
  cudaEvent_t ev_main_fence = nullptr;
  cudaEvent_t ev_commit = nullptr;  // the last pass's new keys are in the table
  void fence_side() {
    RLC_CK(cudaEventRecord(ev_main_fence, stream));
    if (pstream) RLC_CK(cudaStreamWaitEvent(pstream, ev_main_fence, 0));
    if (sstream) RLC_CK(cudaStreamWaitEvent(sstream, ev_main_fence, 0));
  }
  // G-buffer slots (passes in flight): RLC_GSLOTS, 2 (default) or 3
  static constexpr int kMaxSlots = 3;
  int nslots = 2;
  int slot_of(uint32_t pass) const { return int(pass % uint32_t(nslots)); }
  cudaEvent_t ev_gbuf_free[kMaxSlots] = {nullptr, nullptr, nullptr};
  rlc::GBuf* gslot[kMaxSlots] = {nullptr, nullptr, nullptr};
  unsigned long long* pkey_slot[kMaxSlots] = {};  // pending keys, per G-buffer slot
  // sample records and q_before per G-buffer slot: pass p's accumulation
  // (side stream) reads them while pass p + 1 samples and folds
  rlc::SampleRec* srec_slot[kMaxSlots] = {};
  uint8_t* rflag_slot[kMaxSlots] = {};  // (the occluded bits k_accumulate reads)
  uint32_t* gflags_slot[kMaxSlots] = {};
  double* qb_slot[kMaxSlots] = {};
  void sync_all() {
    RLC_CK(cudaStreamSynchronize(stream));
    if (pstream) RLC_CK(cudaStreamSynchronize(pstream));
    if (sstream) RLC_CK(cudaStreamSynchronize(sstream));
    acc_pending = false;
  }
  // per-stage CUDA-event timing (rlc_context_enable_timing)
  bool timing = false;
  struct Mark {
    int stage;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<Mark> marks;
  cudaEvent_t take_event() {  // pooled timing events
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      RLC_CK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  // Brackets the launches of one stage with events on the stream they use.
  template <class F>
  void stage_on(cudaStream_t s, int id, F&& launch) {
    if (!timing || marks.size() >= 200000) {
      launch();
      return;
    }
    const cudaEvent_t a = take_event(), b = take_event();
    RLC_CK(cudaEventRecord(a, s));
    launch();
    RLC_CK(cudaEventRecord(b, s));
    marks.push_back(Mark{id, a, b});
  }
  template <class F>
  void stage(int id, F&& launch) {
    stage_on(stream, id, static_cast<F&&>(launch));
  }
  ~rlc_context() {
    if (h_stage) cudaFreeHost(h_stage);
    if (graph.exec) cudaGraphExecDestroy(graph.exec);
    if (shard_graph.exec) cudaGraphExecDestroy(shard_graph.exec);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    if (ev_prim_done) cudaEventDestroy(ev_prim_done);
    if (ev_main_fence) cudaEventDestroy(ev_main_fence);
    if (ev_commit) cudaEventDestroy(ev_commit);
    if (ev_sample_done) cudaEventDestroy(ev_sample_done);
    if (ev_fold_done) cudaEventDestroy(ev_fold_done);
    if (ev_acc_done) cudaEventDestroy(ev_acc_done);
    if (ev_sort_done) cudaEventDestroy(ev_sort_done);
    if (sstream) cudaStreamDestroy(sstream);
    for (cudaEvent_t e : ev_gbuf_free)
      if (e) cudaEventDestroy(e);
    if (pstream) cudaStreamDestroy(pstream);
  }
  // sharded pass state (rlc_shard_trace -> rlc_shard_fold -> rlc_shard_finish)
  PassParamsHolder shard;
  bool shard_folded = false;
  DeviceArena xarena;
  rlc::ExchangeBuffers xb{};
  // sharded passes (rlc_shard_*): this rank's record block and the buffers
  // of the fold over nranks x cap gathered record slots
  DeviceArena blockarena;
  void* block = nullptr;
  uint64_t block_cap = 0;    // record slots of this pass's block (the caller's cap)
  uint64_t block_alloc = 0;  // record slots allocated
  uint64_t xb_slots = 0;
  // block bytes: a header slot and cap record slots of 32 B
  uint64_t block_bytes() const { return (block_cap + 1) * sizeof(rlc::ExchangeRecord); }
  void ensure_block(uint64_t cap) {
    block_cap = cap;
    if (cap <= block_alloc && block) return;
    sync_all();
    blockarena.release();
    block = blockarena.alloc<rlc::ExchangeRecord>(cap + 1);
    block_alloc = cap;
  }
  // exchange slots of nranks blocks of cap + 1 slots (header + records)
  void ensure_exchange(uint32_t nranks, uint32_t cap) {
    const uint64_t slots = uint64_t(nranks) * (uint64_t(cap) + 1);
    xb.nranks = nranks;
    xb.stride = cap + 1;
    if (slots <= xb_slots) return;
    sync_all();
    xarena.release();
    const uint64_t n = slots;
    xb.rec = nullptr;
    xb.cellx = xarena.alloc<uint32_t>(n);
    xb.kflag = xarena.alloc<uint8_t>(n);
    xb.keys = xarena.alloc<uint32_t>(n);
    xb.vals = xarena.alloc<uint32_t>(n);
    xb.keys_alt = xarena.alloc<uint32_t>(n);
    xb.vals_alt = xarena.alloc<uint32_t>(n);
    xb.hist = xarena.alloc<uint32_t>((size_t(n) / rlc::kSortTileSmall + 2) * 256);
    xb.block_counts = xarena.alloc<uint32_t>(n / 2048 + 2);
    xb.sort_count = xarena.alloc<unsigned int>(2);
    xb.q_rec = xarena.alloc<double>(n);
    xb.seg_n = xarena.alloc<uint32_t>(n);
    xb.pend = xarena.alloc<uint32_t>(n);
    xb.pend_count = xarena.alloc<unsigned int>(1);
    xb.nk = alloc_new_keys(xarena, n, stream);
    xb_slots = n;
  }
  // per-entry arrays of the owner-mode entry exchange (capacity * M entries)
  DeviceArena entarena;
  uint64_t ent_cap = 0;
  void ensure_entries(uint64_t entries) {
    xb.entries = entries;
    if (entries <= ent_cap) return;
    sync_all();
    entarena.release();
    xb.ent_q = entarena.alloc<double>(entries);
    xb.ent_n = entarena.alloc<uint32_t>(entries);
    ent_cap = entries;
  }
  // render_frame cache (prepare_frame_cache)
  rlc_grid* frame_grid = nullptr;
  rlc_framebuffer* frame_fb = nullptr;
  rlc_render_config frame_cfg{};
  DeviceArena frame_hist_arena;
  uint32_t* frame_hist = nullptr;
  uint32_t frame_hist_cap = 0;
  // per-pass scratch, grown on demand
  DeviceArena scratch;
  rlc::PassBuffers pb{};
  uint32_t pb_cap = 0;
  uint32_t pb_gen = 0;  // bumped when the pass buffers move (invalidates captured graphs)
  // CUDA graph of one whole pass (render_pass + end_of_pass_update) for
  // launch-bound frames, replayed by run_passes
  struct PassGraph {
    cudaGraphExec_t exec = nullptr;
    rlc_render_config cfg{};
    const void* grid = nullptr;
    const void* fb = nullptr;
    const void* hist = nullptr;
    double alpha = 0;
    uint32_t pb_gen = 0, scene_gen = 0;
    uint64_t launches = 0;  // kernels per replay
  } graph;
  uint32_t scene_gen = 0;       // bumped by rlc_context_update_scene
  // CUDA graph of two sharded frames (rlc_shard_frames), NCCL calls included
  struct ShardGraph {
    cudaGraphExec_t exec = nullptr;
    rlc_render_config cfg{};
    const void *grid = nullptr, *fb = nullptr, *comm = nullptr, *gathered = nullptr,
               *block = nullptr, *peer_recv = nullptr;
    uint32_t r0 = 0, r1 = 0;
    uint64_t cap = 0;
    int owner = 0;
    uint32_t pb_gen = 0, scene_gen = 0;
    uint64_t launches = 0;
  } shard_graph;
  const uint32_t* graph_pass_dev = nullptr;  // set while capturing: setup_pass reads it
  uint32_t* d_pass = nullptr;     // device pass index of graph replays
  // pinned staging for large downloads (download_to_host)
  void* h_stage = nullptr;
  size_t h_stage_cap = 0;
  uint32_t* d_changes = nullptr;  // device change count of graph replays
  // rlc_pass_samples: the last pass's parameters and G-buffer slot
  bool export_samples = false;
  bool frozen_pdf = false;  // rlc_context_set_pdf_mode
  rlc::PassParams last_pass{};
  rlc::PassBuffers last_pb{};
  bool last_valid = false;

  void ensure_scratch(uint32_t n) {
    if (n <= pb_cap) return;
    sync_all();
    ++pb_gen;
    scratch.release();
    const uint32_t cap = n;
    for (int k = 0; k < nslots; ++k) {
      gslot[k] = scratch.alloc<rlc::GBuf>(cap);
      pkey_slot[k] = scratch.alloc<unsigned long long>(2 * size_t(cap));
      srec_slot[k] = scratch.alloc<rlc::SampleRec>(cap);
      gflags_slot[k] = scratch.alloc<uint32_t>(cap);
      rflag_slot[k] = scratch.alloc<uint8_t>(cap);
      qb_slot[k] = scratch.alloc<double>(cap);
    }
    pb.gbuf = gslot[0];
    pb.pkey = pkey_slot[0];
    pb.nk = alloc_new_keys(scratch, cap, stream);
    pb.emit = scratch.alloc<uint32_t>(cap);
    pb.srec = srec_slot[0];
    pb.vdense = scratch.alloc<double>(cap);
    pb.gflags = gflags_slot[0];
    pb.rflag = rflag_slot[0];
    pb.keys = scratch.alloc<uint32_t>(cap);
    pb.vals = scratch.alloc<uint32_t>(cap);
    pb.keys_alt = scratch.alloc<uint32_t>(cap);
    pb.vals_alt = scratch.alloc<uint32_t>(cap);
    pb.q_before = qb_slot[0];
    pb.rays = scratch.alloc<rlc::ShadowRay>(cap);
    pb.ray_count = scratch.alloc<unsigned int>(2);
    pb.ray_order = scratch.alloc<uint32_t>(cap);
    pb.rec_path = scratch.alloc<uint32_t>(cap);
    pb.rec_count = scratch.alloc<unsigned int>(2);
    pb.block_counts = scratch.alloc<uint32_t>(cap / 2048 + 2);
    pb.block_counts2 = scratch.alloc<uint32_t>(cap / 2048 + 2);
    pb.sort_count = scratch.alloc<unsigned int>(2);
    pb.sort_hist_cap = ((cap + rlc::kSortTile - 1u) / rlc::kSortTile + 2u) * 256u;  // rows + digit totals
    pb.sort_hist = scratch.alloc<uint32_t>(pb.sort_hist_cap);
    pb_cap = cap;
  }
};

struct rlc_grid {
  const rlc_context* ctx = nullptr;
  bool holds_ref = false;  // false for the context's own render_frame cache
  rlc::DevGrid dev{};
  rlc::HostCut tmpl;
  uint32_t key_bits = 0;
  DeviceArena arena;
  uint32_t* d_changes = nullptr;
  double alpha = 0.2;
  uint32_t harmonic = 0;
};

struct rlc_framebuffer {
  const rlc_context* ctx = nullptr;
  bool holds_ref = false;  // false for the context's own render_frame cache
  int32_t width = 0, height = 0;
  DeviceArena arena;
  rlc::Framebuf fb{};
  double* d_image = nullptr;
};

namespace {

uint32_t read_and_clear_err(cudaStream_t st, unsigned long long* counters) {
  unsigned long long e = 0;
  RLC_CK(cudaMemcpyAsync(&e, counters + rlc::kCntErr, sizeof(e), cudaMemcpyDeviceToHost, st));
  RLC_CK(cudaStreamSynchronize(st));
  if (e) RLC_CK(cudaMemsetAsync(counters + rlc::kCntErr, 0, sizeof(e), st));
  return uint32_t(e);
}

void throw_device_error(uint32_t bits) {
  if (bits & (rlc::kErrStackOverflow | rlc::kErrNewKeyOverflow | rlc::kErrCheck))
    throw std::runtime_error(device_error_message(bits));
  throw rlc::InvalidArgument(device_error_message(bits));
}

// Validated launch parameters of one pass over rows [r0, r1).
struct PassSetup {
  rlc::PassParams p{};
  rlc::DevGrid g{};
  uint32_t n = 0;   // paths
  uint32_t nv = 0;  // path vertices n * max_depth
};

PassSetup setup_pass(rlc_context* ctx, const rlc_render_config* cfg, uint32_t pass_index,
                     rlc_grid* grid, rlc_framebuffer* fb, bool need_fb, uint32_t r0, uint32_t r1) {
  require(cfg->passes != 0 && cfg->spp % cfg->passes == 0,
          "render_pass: spp must be divisible by passes");
  require(!(cfg->sampler == RLC_SAMPLER_RL_LIGHTCUTS && grid == nullptr),
          "render_pass: learned sampler needs a hash grid");
  require(cfg->sampler <= RLC_SAMPLER_RL_LIGHTCUTS, "render_pass: unknown sampler");
  if (cfg->max_depth > 1 && probe_libm_variant() == rlc::libm::kUnknown)
    throw std::runtime_error(
        "render_pass: max_depth > 1 needs the host libm's sin/cos, which this build does not "
        "reproduce (rlc_libm.h)");
  require(!need_fb || (fb != nullptr && fb->width == ctx->host.cam.width &&
                       fb->height == ctx->host.cam.height),
          "render_pass: framebuffer size must match the camera");
  require(r0 <= r1 && r1 <= uint32_t(ctx->host.cam.height), "render_pass: bad row range");
  require(grid == nullptr || grid->ctx == ctx, "render_pass: grid belongs to another context");
  // no join with the previous pass's accumulation: it reads only its own
  // G-buffer slot's buffers (the next pass's primary rays wait for them)
  PassSetup S;
  const uint32_t spp_pp = cfg->spp / cfg->passes;
  const uint64_t n64 = uint64_t(r1 - r0) * uint64_t(ctx->host.cam.width) * spp_pp;
  require(n64 * cfg->max_depth < (1ull << 31), "render_pass: too many path vertices for one launch");
  S.n = uint32_t(n64);
  S.nv = uint32_t(n64 * cfg->max_depth);
  S.p.width = uint32_t(ctx->host.cam.width);
  S.p.row_begin = r0;
  S.p.spp_pp = spp_pp;
  S.p.pass_index = pass_index;
  S.p.n = S.n;
  S.p.depth = cfg->max_depth;
  S.p.nv = S.nv;
  S.p.sampler = cfg->sampler;
  S.p.seed_mixed = rlc::mix64(cfg->seed);
  S.p.zero_mixed = rlc::mix64(0);
  S.p.alpha = grid ? grid->alpha : cfg->cut.alpha;
  S.p.harmonic = grid ? grid->harmonic : 0u;
  S.p.pass_dev = ctx->graph_pass_dev;
  S.p.export_samples = ctx->export_samples ? 1u : 0u;
  S.p.frozen_pdf = ctx->frozen_pdf ? 1u : 0u;
  if (grid) S.g = grid->dev;
  else S.g.counters = ctx->counters;
  if (S.nv > 0) ctx->ensure_scratch(S.nv);
  return S;
}

// Primary rays, cut samples and shadow rays of one pass (render.cpp:59-99,
// estimators.cpp:28-106).  Returns the update records sorted by
// (cell, cluster) in *k / *v for the learned sampler.
void enqueue_trace(rlc_context* ctx, const PassSetup& S, rlc_grid* grid, uint32_t** k,
                   uint32_t** v) {
  cudaStream_t st = ctx->stream;
  // Primary rays do not read the learned state, only the hash table's keys
  // (new cells get fresh ids with touched = 0, which the running
  // split-collapse skips), so they run on the side stream as soon as their
  // G-buffer slot is free and overlap the previous pass's tail.
  const int slot = ctx->slot_of(S.p.pass_index);
  ctx->pb.gbuf = ctx->gslot[slot];
  ctx->pb.pkey = ctx->pkey_slot[slot];
  ctx->pb.srec = ctx->srec_slot[slot];
  ctx->pb.rflag = ctx->rflag_slot[slot];
  ctx->pb.gflags = ctx->gflags_slot[slot];
  ctx->pb.q_before = ctx->qb_slot[slot];
  const bool rl = S.p.sampler == RLC_SAMPLER_RL_LIGHTCUTS;
  // The pass's new keys go in after all its lookups, in canonical order
  // (k_insert / k_commit, the reference's sequential insertion), right behind
  // the primary rays (one vertex per path) or behind the last bounce; k_sample
  // then finds them.  Side-stream placements that keep the two small launches
  // off the critical path (a resolve kernel ahead of the record sort) measured
  // slower: the sort, already level with the shadow rays, then waits for them
  // (c3 1.108 vs 1.042 ms per frame, same box).
  const bool insert = rl && !S.p.defer_insert;
  const cudaStream_t ps = ctx->overlap ? ctx->pstream : st;
  auto insert_new_keys = [&](cudaStream_t s) {
    ctx->stage_on(s, 7, [&] { rlc::launch_insert_new_keys(S.g, ctx->pb.nk, s); });
  };
  // the slot's buffers are free once pass - 2's accumulation has read them
  RLC_CK(cudaStreamWaitEvent(ps, ctx->ev_gbuf_free[slot], 0));
  if (rl) RLC_CK(cudaMemsetAsync(ctx->pb.nk.count, 0, sizeof(unsigned int), ps));
  ctx->stage_on(ps, 0, [&] { rlc::launch_primary(ctx->dev, S.g, S.p, ctx->pb, ps); });
  if (insert && S.p.depth == 1) insert_new_keys(ps);
  if (ctx->overlap) {
    RLC_CK(cudaEventRecord(ctx->ev_prim_done, ps));
    RLC_CK(cudaStreamWaitEvent(st, ctx->ev_prim_done, 0));
  }
  // Multi-bounce paths (max_depth > 1): one launch per further vertex; the
  // vertices of all depths then share the sample / sort / shadow / fold
  // launches below, in canonical (path, depth) order.
  for (uint32_t d = 2; d <= S.p.depth; ++d)
    ctx->stage(0, [&] { rlc::launch_bounce(ctx->dev, S.g, S.p, d, ctx->pb, st); });
  if (insert && S.p.depth > 1) {
    insert_new_keys(st);
    // the next pass's lookups (primary stream) read the table and reuse the
    // new-key table
    if (ps != st) {
      RLC_CK(cudaEventRecord(ctx->ev_commit, st));
      RLC_CK(cudaStreamWaitEvent(ps, ctx->ev_commit, 0));
    }
  }
  ctx->stage(1, [&] { rlc::launch_sample(ctx->dev, S.g, S.p, ctx->pb, st); });
  // The update records are sorted by (cell, cluster) for the fold on the
  // side stream while the shadow rays are traced, in canonical (pixel)
  // order: neighbouring pixels give coherent origins, and on the
  // triangle-level shadow tree that beats the sorted order (0.55 vs 0.62 ms
  // on c3).  The any-hit result does not depend on the order.
  *k = nullptr;
  *v = nullptr;
  if (rl && !S.p.defer_insert) {  // (a sharded trace sorts all ranks' records in rlc_shard_fold)
    RLC_CK(cudaEventRecord(ctx->ev_sample_done, st));
    RLC_CK(cudaStreamWaitEvent(ctx->sstream, ctx->ev_sample_done, 0));
    ctx->stage_on(ctx->sstream, 2, [&] {
      rlc::launch_sort(ctx->pb, S.nv, grid->key_bits, ctx->sstream, k, v);
    });
    RLC_CK(cudaEventRecord(ctx->ev_sort_done, ctx->sstream));
  }
  ctx->stage(8, [&] { rlc::launch_ray_compact(ctx->pb, nullptr, S.nv, st); });
  ctx->stage(6, [&] {
    rlc::launch_shadow(ctx->dev, ctx->pb, ctx->pb.ray_order, S.g.counters, st, rl);
  });
  if (rl && !S.p.defer_insert) RLC_CK(cudaStreamWaitEvent(st, ctx->ev_sort_done, 0));
}

// render_pass body (proj/src/render.cpp:159-183) for rows [r0, r1).
void enqueue_pass(const rlc_context* cctx, const rlc_render_config* cfg, uint32_t pass_index,
                  rlc_grid* grid, rlc_framebuffer* fb, uint32_t r0, uint32_t r1) {
  rlc_context* ctx = const_cast<rlc_context*>(cctx);
  const PassSetup S = setup_pass(ctx, cfg, pass_index, grid, fb, true, r0, r1);
  if (S.n == 0) return;
  uint32_t *k = nullptr, *v = nullptr;
  if (S.nv > 0) enqueue_trace(ctx, S, grid, &k, &v);  // max_depth 0: empty paths
  ctx->last_pass = S.p;
  ctx->last_pb = ctx->pb;
  ctx->last_valid = true;
  cudaStream_t st = ctx->stream;
  if (cfg->sampler == RLC_SAMPLER_RL_LIGHTCUTS && S.nv > 0) {
    ctx->stage(3, [&] { rlc::launch_fold(S.g, S.p, k, v, ctx->pb, st); });
    // The framebuffer accumulation reads only pass buffers; the
    // end_of_pass_update that follows touches only cut rows: run the former
    // on the side stream beside the latter, joined by the next reader.
    RLC_CK(cudaEventRecord(ctx->ev_fold_done, st));
    RLC_CK(cudaStreamWaitEvent(ctx->sstream, ctx->ev_fold_done, 0));
    ctx->stage_on(ctx->sstream, 4, [&] {
      rlc::launch_accumulate(ctx->dev, S.p, ctx->pb, fb->fb, ctx->sstream);
    });
    RLC_CK(cudaEventRecord(ctx->ev_acc_done, ctx->sstream));
    RLC_CK(cudaEventRecord(ctx->ev_gbuf_free[ctx->slot_of(S.p.pass_index)], ctx->sstream));
    ctx->acc_pending = true;
  } else {
    ctx->stage(4, [&] { rlc::launch_accumulate(ctx->dev, S.p, ctx->pb, fb->fb, st); });
    RLC_CK(cudaEventRecord(ctx->ev_gbuf_free[ctx->slot_of(S.p.pass_index)], st));  // last G-buffer reader
  }
  RLC_CK(cudaGetLastError());
}

void finish_sync(const rlc_context* cctx, rlc_grid* grid) {
  rlc_context* ctx = const_cast<rlc_context*>(cctx);
  ctx->join_acc();
  const uint32_t bits =
      read_and_clear_err(ctx->stream, grid ? grid->dev.counters : ctx->counters);
  if (bits) throw_device_error(bits);
}

void prepare_frame_cache(rlc_context* ctx, const rlc_render_config* config);

void enqueue_eop(rlc_grid* grid, const rlc_context* ctx, const rlc_cut_config* cut,
                 uint32_t* d_changes) {
  require(grid != nullptr && ctx != nullptr && cut != nullptr,
          "end_of_pass_update: null argument");
  require(grid->ctx == ctx, "end_of_pass_update: grid belongs to another context");
  rlc_context* c = const_cast<rlc_context*>(ctx);
  c->stage(5, [&] {
    rlc::launch_split_collapse(ctx->dev, grid->dev, cut->split_threshold, cut->iterations,
                               d_changes, ctx->stream);
  });
  RLC_CK(cudaGetLastError());
}

// Uploads the device view of a host scene into arena A.
// update = true: a dynamic scene update (rlc_context_update_scene), whose
// materials, material ids and light tree are those of the previous upload.
void upload_scene(const rlc::HostScene& h, SceneBuffers& A, rlc::DevScene& d, cudaStream_t st,
                  bool update = false) {
  A.begin(st, update);
  d.nodes = A.put(h.nodes);
  d.nodes_f = A.put(h.nodes_f);
  d.nodes_cam = A.put(h.nodes_cam);
  // the unquantized shadow tree is read only when there is no quantized one
  static const std::vector<rlc::Wide4> kNoWide;
  d.wide = A.put(h.wide_q.empty() ? h.wide : kNoWide);
  d.wide_q = A.put(h.wide_q);
  d.wide_ref = A.put(h.wide_ref);
  d.wide_cam = A.put(h.wide_cam);
  if (h.nodes_f.empty()) d.nodes_f = nullptr;
  if (h.nodes_cam.empty()) d.nodes_cam = nullptr;
  if (h.wide.empty() || !h.wide_q.empty()) d.wide = nullptr;
  if (h.wide_q.empty()) d.wide_q = nullptr;
  if (h.wide_ref.empty()) d.wide_ref = nullptr;
  if (h.wide_cam.empty()) d.wide_cam = nullptr;
  d.tri_leaf = A.put(h.tri_leaf);
  d.tris_s = A.put(h.tris_s);
  d.tri_leaf_s = A.put(h.tri_leaf_s);
  d.tris = A.put(h.tris);
  d.mats = A.put(h.mats, !update);
  d.tri_mat = A.put(h.tri_mat, !update);
  d.tri_normal = A.put(h.tri_normal);
  d.lights = A.put(h.lights);
  d.order = A.put(h.order, !update);
  d.lt = A.put(h.lt_nodes, !update);
  d.energy_cdf = A.put(h.energy_cdf);
  d.emitter_mat = A.put(h.emitter_mat, !update);
  d.emitter_energy = A.put(h.emitter_energy);
  d.num_lights = uint32_t(h.lights.size());
  d.num_tris = uint32_t(h.tri_mat.size());
  d.fp32_ok = 1;
  for (int a = 0; a < 3; ++a)
    if (!(std::fabs(h.scene_lo[a]) <= 1e8 && std::fabs(h.scene_hi[a]) <= 1e8)) d.fp32_ok = 0;
  d.nodes_root_leaf = h.nodes.empty() || h.nodes[0].count > 0 ? 1u : 0u;
  d.shadow_stack_limit = 0;
  if (const char* e = std::getenv("RLC_SHADOW_STACK_LIMIT")) d.shadow_stack_limit = uint32_t(std::atoi(e));
  d.shadow_eps = h.shadow_eps;
  d.coord_bound = h.coord_bound;
  d.libm_fma = probe_libm_variant() == rlc::libm::kFma ? 1u : 0u;
  d.base_tile = h.base_tile;
  for (int k = 0; k <= 16; ++k) d.level_thr[k] = h.level_threshold[k];
  d.cam = h.cam;
}

}  // namespace

extern "C" {

const char* rlc_last_error(void) { return g_err.c_str(); }
int rlc_abi_version(void) { return RLC_ABI_VERSION; }
uint64_t rlc_kernel_launches(void) { return rlc::launches(); }

rlc_status rlc_render_config_default(rlc_render_config* c) {
  return guarded([&] {
    require(c != nullptr, "rlc_render_config_default: null config");
    std::memset(c, 0, sizeof(*c));
    c->spp = 16;  // render.hpp:18-25
    c->passes = 4;
    c->max_depth = 1;
    c->sampler = RLC_SAMPLER_UNIFORM;
    c->cut.cut_size = 128;  // cut.hpp:22-27
    c->cut.alpha = 0.2;
    c->cut.split_threshold = 4.0;
    c->cut.eps_q = -1;
    c->cut.iterations = 1;
    c->cut.alpha_schedule = RLC_ALPHA_FIXED;
    c->hash.capacity = 1u << 16;  // hash_grid.hpp:18-22
    c->hash.base_tile = 0;
    c->hash.probe_limit = 32;
    c->hash.normal_bits = 4;
    c->hash.jitter_scale = 0;
    c->seed = 1;
    c->workers = 1;
  });
}

rlc_status rlc_context_create(const rlc_scene_desc* scene, const rlc_render_config* config,
                              int device, rlc_context** out) {
  return guarded([&] {
    require(scene != nullptr && config != nullptr && out != nullptr,
            "rlc_context_create: null argument");
    *out = nullptr;
    check_device(device);
    auto ctx = std::make_unique<rlc_context>();
    ctx->device = device;
    if (const char* e = std::getenv("RLC_GSLOTS"))  // G-buffer slots: 2 or 3 (A/B)
      ctx->nslots = std::min(rlc_context::kMaxSlots, std::max(2, std::atoi(e)));
    ctx->create_cfg = *config;
    rlc::build_host_scene(*scene, *config, ctx->host);
    RLC_CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    upload_scene(ctx->host, ctx->scene_bufs, ctx->dev, ctx->stream);
    ctx->build_light_order();
    ctx->counters = ctx->arena.alloc<unsigned long long>(rlc::kCntNum);
    RLC_CK(cudaMemsetAsync(ctx->counters, 0, sizeof(unsigned long long) * rlc::kCntNum, ctx->stream));
    RLC_CK(cudaStreamCreateWithFlags(&ctx->pstream, cudaStreamNonBlocking));
    ctx->overlap = true;  // measured faster on c3 (1.51 vs 1.56 ms per frame)
    if (const char* e = std::getenv("RLC_OVERLAP")) ctx->overlap = std::string(e) != "0";
    RLC_CK(cudaEventCreateWithFlags(&ctx->ev_prim_done, cudaEventDisableTiming));
    RLC_CK(cudaEventCreateWithFlags(&ctx->ev_main_fence, cudaEventDisableTiming));
    RLC_CK(cudaEventCreateWithFlags(&ctx->ev_commit, cudaEventDisableTiming));
    RLC_CK(cudaStreamCreateWithFlags(&ctx->sstream, cudaStreamNonBlocking));
    RLC_CK(cudaEventCreateWithFlags(&ctx->ev_sample_done, cudaEventDisableTiming));
    RLC_CK(cudaEventCreateWithFlags(&ctx->ev_fold_done, cudaEventDisableTiming));
    RLC_CK(cudaEventCreateWithFlags(&ctx->ev_acc_done, cudaEventDisableTiming));
    RLC_CK(cudaEventCreateWithFlags(&ctx->ev_sort_done, cudaEventDisableTiming));
    for (cudaEvent_t& e : ctx->ev_gbuf_free) {
      RLC_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      RLC_CK(cudaEventRecord(e, ctx->stream));
    }
    // render_frame's grid, framebuffer and pass buffers for this config;
    // best effort: build_context does not validate the hash/cut config
    // (render.cpp:143-157), render_frame reports it
    try {
      prepare_frame_cache(ctx.get(), config);
    } catch (const std::invalid_argument&) {
    }
    RLC_CK(cudaStreamSynchronize(ctx->stream));
    *out = ctx.release();
  });
}

namespace {

// rlc_context_update_scene's argument checks (the reference's build_context
// has no such call; DESIGN.md 5.10 defines the semantics).
void check_update(const rlc_context* ctx, const rlc_scene_desc* scene) {
  require(ctx != nullptr && scene != nullptr, "rlc_context_update_scene: null argument");
  const rlc::HostScene& old = ctx->host;
  require(scene->num_triangles == old.tri_mat.size() &&
              scene->num_materials * 6 == old.mat_values.size() &&
              scene->width == old.cam.width && scene->height == old.cam.height,
          "rlc_context_update_scene: triangle count, materials and resolution must not change");
  require(scene->vertices != nullptr, "rlc_context_update_scene: null vertices");
  for (uint32_t t = 0; t < scene->num_triangles; ++t)
    require(scene->material_ids[t] == old.tri_mat[t],
            "rlc_context_update_scene: material ids must not change");
  for (size_t i = 0; i < old.mat_values.size(); ++i)
    require(scene->materials[i] == old.mat_values[i],
            "rlc_context_update_scene: materials must not change");
}

// build_context(scene) (render.cpp:143-157) with the light tree of the
// context's creation (same emitter order, topology and node energies), on a
// worker thread; returns its token.
uint64_t prepare_scene(rlc_context* ctx, const rlc_scene_desc* scene) {
  check_update(ctx, scene);
  rlc_context::FrameScene* f = nullptr;
  for (auto& p : ctx->frame_scenes)
    if (!p->busy) {
      f = p.get();
      break;
    }
  if (!f) {
    require(ctx->frame_scenes.size() < 8, "rlc_context_prepare_scene: at most 8 scenes in flight");
    ctx->frame_scenes.push_back(std::make_unique<rlc_context::FrameScene>());
    f = ctx->frame_scenes.back().get();
  }
  f->vertices.assign(scene->vertices, scene->vertices + size_t(scene->num_triangles) * 9);
  f->desc = *scene;
  f->desc.vertices = f->vertices.data();
  f->desc.material_ids = ctx->host.tri_mat.data();  // validated equal, frozen
  f->desc.materials = ctx->host.mat_values.data();
  f->token = ctx->next_scene_token++;
  f->busy = true;
  const rlc_render_config cfg = ctx->create_cfg;
  const rlc::HostScene* base = &ctx->host;
  f->build = std::async(std::launch::async,
                        [f, cfg, base] { rlc::build_host_scene(f->desc, cfg, f->h, base); });
  return f->token;
}

void commit_scene(rlc_context* ctx, uint64_t token) {
  rlc_context::FrameScene* f = nullptr;
  for (auto& p : ctx->frame_scenes)
    if (p->busy && p->token == token) f = p.get();
  require(f != nullptr, "rlc_context_commit_scene: no prepared scene with this token");
  const bool report = std::getenv("RLC_UPDATE_TIMING") != nullptr;
  auto t = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!report) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "update_scene %s %.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  };
  try {
    f->build.get();
  } catch (...) {
    f->busy = false;
    throw;
  }
  lap("host build wait");
  RLC_CK(cudaSetDevice(ctx->device));
  ctx->sync_all();  // the previous frame's kernels read the buffers
  lap("sync");
  rlc::DevScene d{};
  d.count_work = ctx->dev.count_work;
  d.lights_ord = ctx->dev.lights_ord;
  upload_scene(f->h, ctx->scene_bufs, d, ctx->stream, true);
  if (f->h.gpu_refit) {  // the shadow tree refitted on the device
    ctx->ensure_refit_topology();
    const double* verts = ctx->scene_bufs.put(f->vertices);
    const uint32_t* leaf_of_id = ctx->scene_bufs.put(f->h.refit_leaf);
    rlc::launch_refit_shadow(ctx->refit, verts, leaf_of_id, f->h.coord_bound * 0x1.0p-21,
                             ctx->refit_tris_s, ctx->refit_tri_leaf_s, ctx->refit_wide,
                             ctx->refit_wide_q,
                             reinterpret_cast<unsigned int*>(ctx->counters + rlc::kCntErr),
                             ctx->stream);
    RLC_CK(cudaGetLastError());
    d.tris_s = ctx->refit_tris_s;
    d.tri_leaf_s = ctx->refit_tri_leaf_s;
    d.wide = ctx->refit_wide;
    d.wide_q = ctx->refit_wide_q;
  }
  ctx->dev = d;
  ctx->build_light_order();
  // the copies complete before the output scene is recycled and before any
  // stream reads the new scene
  RLC_CK(cudaStreamSynchronize(ctx->stream));
  f->busy = false;
  ++ctx->scene_gen;  // captured pass graphs hold the old scene's pointers
  lap("upload");
}

}  // namespace

rlc_status rlc_context_update_scene(rlc_context* ctx, const rlc_scene_desc* scene) {
  return guarded([&] {
    RLC_CK(cudaSetDevice(ctx ? ctx->device : 0));
    commit_scene(ctx, prepare_scene(ctx, scene));
  });
}

rlc_status rlc_context_prepare_scene(rlc_context* ctx, const rlc_scene_desc* scene,
                                     uint64_t* token) {
  return guarded([&] {
    require(token != nullptr, "rlc_context_prepare_scene: null token");
    *token = prepare_scene(ctx, scene);
  });
}

rlc_status rlc_context_commit_scene(rlc_context* ctx, uint64_t token) {
  return guarded([&] {
    require(ctx != nullptr, "rlc_context_commit_scene: null context");
    commit_scene(ctx, token);
  });
}

namespace {
void context_release(const rlc_context* cctx) {
  rlc_context* ctx = const_cast<rlc_context*>(cctx);
  if (ctx->refs.fetch_sub(1) != 1) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->pstream) cudaStreamSynchronize(ctx->pstream);
  if (ctx->sstream) cudaStreamSynchronize(ctx->sstream);
  rlc_grid_destroy(ctx->frame_grid);
  rlc_framebuffer_destroy(ctx->frame_fb);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}
}  // namespace

rlc_status rlc_context_destroy(rlc_context* ctx) {
  return guarded([&] {
    if (!ctx) return;
    context_release(ctx);
  });
}

rlc_status rlc_context_info_get(const rlc_context* ctx, rlc_context_info* info) {
  return guarded([&] {
    require(ctx != nullptr && info != nullptr, "rlc_context_info_get: null argument");
    info->num_triangles = uint32_t(ctx->host.tri_mat.size());
    info->num_emitters = uint32_t(ctx->host.lights.size());
    info->bvh_nodes = uint32_t(ctx->host.nodes.size());
    info->light_tree_nodes = uint32_t(ctx->host.lt_nodes.size());
    info->base_tile = ctx->host.base_tile;
    info->shadow_eps = ctx->host.shadow_eps;
    info->device_bytes = ctx->arena.bytes + ctx->scene_bufs.bytes + ctx->scratch.bytes;
  });
}

rlc_status rlc_context_set_stream(rlc_context* ctx, void* stream) {
  return guarded([&] {
    require(ctx != nullptr, "rlc_context_set_stream: null context");
    ctx->sync_all();
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  });
}

rlc_status rlc_context_synchronize(rlc_context* ctx) {
  return guarded([&] {
    require(ctx != nullptr, "rlc_context_synchronize: null context");
    ctx->sync_all();
  });
}

rlc_status rlc_context_enable_timing(rlc_context* ctx, int enable) {
  return guarded([&] {
    require(ctx != nullptr, "rlc_context_enable_timing: null context");
    ctx->timing = enable != 0;
  });
}

rlc_status rlc_context_stage_times(rlc_context* ctx, double* ms, uint32_t* counts) {
  return guarded([&] {
    require(ctx != nullptr, "rlc_context_stage_times: null context");
    ctx->sync_all();
    double acc[RLC_NUM_STAGES] = {};
    uint32_t cnt[RLC_NUM_STAGES] = {};
    for (const auto& m : ctx->marks) {
      float t = 0;
      RLC_CK(cudaEventElapsedTime(&t, m.a, m.b));
      acc[m.stage] += t;
      cnt[m.stage] += 1;
    }
    ctx->marks.clear();
    ctx->ev_used = 0;
    for (int i = 0; i < RLC_NUM_STAGES; ++i) {
      if (ms) ms[i] = acc[i];
      if (counts) counts[i] = cnt[i];
    }
  });
}

rlc_status rlc_context_stage_marks(rlc_context* ctx, uint32_t max_marks, double* out,
                                   uint32_t* n_out) {
  return guarded([&] {
    require(ctx != nullptr && n_out != nullptr, "rlc_context_stage_marks: null argument");
    ctx->sync_all();
    *n_out = uint32_t(ctx->marks.size());
    if (!out || ctx->marks.empty()) return;
    const cudaEvent_t t0 = ctx->marks.front().a;
    for (size_t i = 0; i < ctx->marks.size() && i < max_marks; ++i) {
      float a = 0, b = 0;
      RLC_CK(cudaEventElapsedTime(&a, t0, ctx->marks[i].a));
      RLC_CK(cudaEventElapsedTime(&b, t0, ctx->marks[i].b));
      out[3 * i] = ctx->marks[i].stage;
      out[3 * i + 1] = a;
      out[3 * i + 2] = b;
    }
  });
}

rlc_status rlc_debug_trav_stats(int32_t reset, uint64_t* out8) {
  return guarded([&] {
    require(out8 != nullptr, "rlc_debug_trav_stats: null argument");
    rlc::trav_stats(out8, reset != 0);
  });
}

rlc_status rlc_context_count_work(rlc_context* ctx, int enable) {
  return guarded([&] {
    require(ctx != nullptr, "rlc_context_count_work: null context");
    ctx->dev.count_work = enable ? 1u : 0u;
    ++ctx->scene_gen;  // captured pass graphs hold the old kernel choice
  });
}

rlc_status rlc_debug_host_bvh(const rlc_scene_desc* scene, uint32_t reps, double* ms_out,
                              uint32_t* nodes_out) {
  return guarded([&] {
    require(scene != nullptr && ms_out != nullptr && reps > 0, "rlc_debug_host_bvh: bad argument");
    rlc::HostScene h;
    double total = 0;
    for (uint32_t r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      rlc::build_reference_bvh(*scene, h);
      total += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    *ms_out = total / reps;
    if (nodes_out) *nodes_out = uint32_t(h.nodes.size());
  });
}

rlc_status rlc_work_counters(int32_t reset, uint64_t* out4) {
  return guarded([&] {
    require(out4 != nullptr, "rlc_work_counters: null argument");
    rlc::work_counters(out4, reset != 0);
  });
}

rlc_status rlc_measure_l2_bandwidth(int device, double* gbs) {
  return guarded([&] {
    require(gbs != nullptr, "rlc_measure_l2_bandwidth: null argument");
    check_device(device);
    *gbs = rlc::measure_l2_gbs(size_t(48) << 20, 40);
    RLC_CK(cudaGetLastError());
  });
}

rlc_status rlc_libm_variant(int32_t* variant) {
  return guarded([&] {
    require(variant != nullptr, "rlc_libm_variant: null argument");
    *variant = probe_libm_variant();
  });
}

rlc_status rlc_libm_sincos_host(int32_t variant, uint64_t n, const double* x, double* s,
                                double* c) {
  return guarded([&] {
    require(variant == rlc::libm::kFma || variant == rlc::libm::kSse2,
            "rlc_libm_sincos_host: unknown variant");
    require(n == 0 || (x && s && c), "rlc_libm_sincos_host: null argument");
    const rlc::libm::Ctx lc{kSinCosTabHost, variant == rlc::libm::kFma};
    for (uint64_t i = 0; i < n; ++i) {
      s[i] = rlc::libm::sin(lc, x[i]);
      c[i] = rlc::libm::cos(lc, x[i]);
    }
  });
}

rlc_status rlc_libm_sincos(const rlc_context* cctx, uint32_t n, const double* x, double* s,
                           double* c) {
  return guarded([&] {
    require(cctx != nullptr && (n == 0 || (x && s && c)), "rlc_libm_sincos: null argument");
    if (n == 0) return;
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    RLC_CK(cudaSetDevice(ctx->device));
    DeviceArena tmp;
    double* dx = tmp.alloc<double>(n);
    double* ds = tmp.alloc<double>(n);
    double* dc = tmp.alloc<double>(n);
    RLC_CK(cudaMemcpyAsync(dx, x, 8 * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    rlc::launch_libm_sincos(ctx->dev, n, dx, ds, dc, ctx->stream);
    RLC_CK(cudaGetLastError());
    RLC_CK(cudaMemcpyAsync(s, ds, 8 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    RLC_CK(cudaMemcpyAsync(c, dc, 8 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    RLC_CK(cudaStreamSynchronize(ctx->stream));
  });
}

rlc_status rlc_occluded_batch(const rlc_context* cctx, uint32_t n, const double* a,
                              const double* b, uint8_t* out) {
  return guarded([&] {
    require(cctx != nullptr && (n == 0 || (a && b && out)), "occluded: null argument");
    if (n == 0) return;
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    RLC_CK(cudaSetDevice(ctx->device));
    ctx->join_acc();  // the shadow queue and sample records are reused below
    ctx->ensure_scratch(n);
    DeviceArena tmp;
    double* da = tmp.alloc<double>(3 * size_t(n));
    double* db = tmp.alloc<double>(3 * size_t(n));
    uint8_t* dout = tmp.alloc<uint8_t>(n);
    RLC_CK(cudaMemcpyAsync(da, a, 24 * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    RLC_CK(cudaMemcpyAsync(db, b, 24 * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    rlc::launch_occluded_batch(ctx->dev, n, da, db, ctx->pb, ctx->counters, dout, ctx->stream);
    RLC_CK(cudaMemcpyAsync(out, dout, n, cudaMemcpyDeviceToHost, ctx->stream));
    finish_sync(ctx, nullptr);
  });
}

namespace {
void intersect_batch(const rlc_context* cctx, uint32_t n, const double* origins,
                     const double* dirs, double t_min, double* t_out, int32_t* tri_out,
                     bool sah_only) {
    require(cctx != nullptr && (n == 0 || (origins && dirs && t_out && tri_out)),
            "intersect: null argument");
    if (n == 0) return;
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    RLC_CK(cudaSetDevice(ctx->device));
    DeviceArena tmp;
    double* dorg = tmp.alloc<double>(3 * size_t(n));
    double* ddir = tmp.alloc<double>(3 * size_t(n));
    double* dt = tmp.alloc<double>(n);
    int32_t* dtri = tmp.alloc<int32_t>(n);
    RLC_CK(cudaMemcpyAsync(dorg, origins, 24 * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    RLC_CK(cudaMemcpyAsync(ddir, dirs, 24 * size_t(n), cudaMemcpyHostToDevice, ctx->stream));
    rlc::launch_intersect_batch(ctx->dev, n, dorg, ddir, t_min, dt, dtri, ctx->counters,
                                ctx->stream, sah_only);
    RLC_CK(cudaMemcpyAsync(t_out, dt, 8 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    RLC_CK(cudaMemcpyAsync(tri_out, dtri, 4 * size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    finish_sync(ctx, nullptr);
}
}  // namespace

rlc_status rlc_intersect_batch(const rlc_context* ctx, uint32_t n, const double* origins,
                               const double* dirs, double t_min, double* t_out,
                               int32_t* tri_out) {
  return guarded([&] { intersect_batch(ctx, n, origins, dirs, t_min, t_out, tri_out, false); });
}

rlc_status rlc_intersect_batch_sah(const rlc_context* ctx, uint32_t n, const double* origins,
                                   const double* dirs, double t_min, double* t_out,
                                   int32_t* tri_out) {
  return guarded([&] { intersect_batch(ctx, n, origins, dirs, t_min, t_out, tri_out, true); });
}

rlc_status rlc_grid_create(const rlc_context* ctx, const rlc_render_config* cfg, rlc_grid** out) {
  return guarded([&] {
    require(ctx != nullptr && cfg != nullptr && out != nullptr, "rlc_grid_create: null argument");
    *out = nullptr;
    RLC_CK(cudaSetDevice(ctx->device));
    require(cfg->hash.capacity >= 1, "HashGrid: capacity must be at least 1");
    require(ctx->host.base_tile > 0, "HashGrid: base tile must be resolved before build");
    require(cfg->hash.normal_bits <= 13,
            "HashGrid: the device key packs at most 13 octahedral bits per component");
    require(cfg->cut.alpha_schedule <= RLC_ALPHA_HARMONIC, "CutConfig: unknown alpha schedule");
    auto g = std::make_unique<rlc_grid>();
    g->ctx = ctx;
    const rlc::HostScene& h = ctx->host;
    g->tmpl = rlc::make_template_cut(h.lt_nodes, h.lt_begin, h.lt_energy,
                                     uint32_t(h.lights.size()), cfg->cut.cut_size, cfg->cut.eps_q);
    const uint32_t M = uint32_t(g->tmpl.q.size());
    const uint64_t cap = cfg->hash.capacity;
    require(cap * M < 0xffffffffull, "HashGrid: capacity * cut size exceeds 32-bit segment keys");
    uint32_t bits = 8;
    while (bits < 32 && (cap * M) >= ((1ull << bits) - 1)) bits += 8;
    g->key_bits = bits;
    DeviceArena& A = g->arena;
    rlc::DevGrid& d = g->dev;
    const cudaStream_t st = ctx->stream;
    d.slot_keys = A.alloc<unsigned long long>(2 * cap);
    RLC_CK(cudaMemsetAsync(d.slot_keys, 0, 16 * cap, st));
    d.slot_cell = A.alloc<uint32_t>(cap);
    d.capacity = uint32_t(cap);
    d.probe_limit = cfg->hash.probe_limit;
    d.normal_bits = cfg->hash.normal_bits;
    d.M = M;
    d.jitter_scale = cfg->hash.jitter_scale;
    d.node_ids = A.alloc<uint32_t>(cap * M);
    d.ends = A.alloc<uint32_t>(cap * M);
    d.q = A.alloc<double>(cap * M);
    d.cdf = A.alloc<double>(cap * M);
    d.visits = A.alloc<uint32_t>(cap * M);
    d.cell_key = A.alloc<uint32_t>(5 * cap);
    d.cell_slot = A.alloc<uint32_t>(cap);
    d.touched = A.alloc<uint32_t>(cap);
    // cuts too large for k_split's shared-memory rows work in global scratch
    d.split_scratch = size_t(M) * 32 > rlc::kSplitSmemMax
                          ? A.alloc<unsigned char>(size_t(rlc::kSplitGlobalWarps) * 32 * M)
                          : nullptr;
    RLC_CK(cudaMemsetAsync(d.touched, 0, 4 * cap, st));
    d.t_node = A.upload(g->tmpl.node_ids, st);
    d.t_ends = A.upload(g->tmpl.ends, st);
    d.t_q = A.upload(g->tmpl.q, st);
    d.t_cdf = A.upload(g->tmpl.cdf, st);
    d.t_visits = A.upload(g->tmpl.visits, st);
    d.eps_q = g->tmpl.eps_q;
    d.counters = A.alloc<unsigned long long>(rlc::kCntNum);
    RLC_CK(cudaMemsetAsync(d.counters, 0, sizeof(unsigned long long) * rlc::kCntNum, st));
    d.claim = A.alloc<unsigned long long>(cap);
    RLC_CK(cudaMemsetAsync(d.claim, 0xff, 8 * cap, st));
    g->d_changes = A.alloc<uint32_t>(1);
    RLC_CK(cudaMemsetAsync(g->d_changes, 0, 4, st));
    // initialised before this call returns: any stream of the context may use it
    RLC_CK(cudaStreamSynchronize(st));
    g->alpha = cfg->cut.alpha;
    g->harmonic = cfg->cut.alpha_schedule == RLC_ALPHA_HARMONIC ? 1u : 0u;
    g->holds_ref = true;
    const_cast<rlc_context*>(ctx)->refs.fetch_add(1);
    *out = g.release();
  });
}

rlc_status rlc_grid_destroy(rlc_grid* grid) {
  return guarded([&] {
    if (!grid) return;
    const rlc_context* ctx = grid->ctx;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    const bool release = grid->holds_ref;
    delete grid;
    if (release) context_release(ctx);
  });
}

rlc_status rlc_grid_stats_get(const rlc_grid* grid, rlc_grid_stats* stats) {
  return guarded([&] {
    require(grid != nullptr && stats != nullptr, "rlc_grid_stats_get: null argument");
    unsigned long long c[rlc::kCntNum];
    const_cast<rlc_context*>(grid->ctx)->sync_all();
    RLC_CK(cudaMemcpy(c, grid->dev.counters, sizeof(c), cudaMemcpyDeviceToHost));
    stats->occupied = uint32_t(c[rlc::kCntCells]);
    stats->cut_size = grid->dev.M;
    stats->lookups = c[rlc::kCntLookups];
    stats->fallback_hits = c[rlc::kCntFallback];
    stats->pending_lookups = c[rlc::kCntPending];
    stats->new_keys = c[rlc::kCntNewKeys];
  });
}

rlc_status rlc_grid_export(const rlc_grid* grid, uint32_t max_cells, rlc_cell_key* keys,
                           uint32_t* node_ids, uint32_t* ends, double* q, double* cdf,
                           uint32_t* visits, uint32_t* num_cells) {
  return guarded([&] {
    require(grid != nullptr, "rlc_grid_export: null grid");
    const_cast<rlc_context*>(grid->ctx)->sync_all();
    unsigned long long nc = 0;
    RLC_CK(cudaMemcpy(&nc, grid->dev.counters + rlc::kCntCells, 8, cudaMemcpyDeviceToHost));
    if (num_cells) *num_cells = uint32_t(nc);
    const size_t n = std::min<size_t>(nc, max_cells);
    const size_t M = grid->dev.M;
    if (n == 0) return;
    if (keys) {
      std::vector<uint32_t> k(5 * n);
      RLC_CK(cudaMemcpy(k.data(), grid->dev.cell_key, 20 * n, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < n; ++i)
        keys[i] = rlc_cell_key{int32_t(k[5 * i]), int32_t(k[5 * i + 1]), int32_t(k[5 * i + 2]),
                               k[5 * i + 3], k[5 * i + 4]};
    }
    if (node_ids) RLC_CK(cudaMemcpy(node_ids, grid->dev.node_ids, 4 * n * M, cudaMemcpyDeviceToHost));
    if (ends) RLC_CK(cudaMemcpy(ends, grid->dev.ends, 4 * n * M, cudaMemcpyDeviceToHost));
    if (q) RLC_CK(cudaMemcpy(q, grid->dev.q, 8 * n * M, cudaMemcpyDeviceToHost));
    if (cdf) RLC_CK(cudaMemcpy(cdf, grid->dev.cdf, 8 * n * M, cudaMemcpyDeviceToHost));
    if (visits) RLC_CK(cudaMemcpy(visits, grid->dev.visits, 4 * n * M, cudaMemcpyDeviceToHost));
  });
}

rlc_status rlc_grid_slots(const rlc_grid* grid, uint32_t max_slots, uint32_t* slot_out,
                          uint32_t* cell_out, rlc_cell_key* key_out, uint8_t* touched_out,
                          uint32_t* count_out) {
  return guarded([&] {
    require(grid != nullptr && count_out != nullptr, "rlc_grid_slots: null argument");
    const_cast<rlc_context*>(grid->ctx)->sync_all();
    const rlc::DevGrid& g = grid->dev;
    const size_t cap = g.capacity;
    unsigned long long nc = 0;
    RLC_CK(cudaMemcpy(&nc, g.counters + rlc::kCntCells, 8, cudaMemcpyDeviceToHost));
    std::vector<unsigned long long> sk(2 * cap);
    std::vector<uint32_t> sc(cap), ck(5 * static_cast<size_t>(nc)), tch(static_cast<size_t>(nc));
    RLC_CK(cudaMemcpy(sk.data(), g.slot_keys, 16 * cap, cudaMemcpyDeviceToHost));
    RLC_CK(cudaMemcpy(sc.data(), g.slot_cell, 4 * cap, cudaMemcpyDeviceToHost));
    if (nc > 0) {
      RLC_CK(cudaMemcpy(ck.data(), g.cell_key, 20 * size_t(nc), cudaMemcpyDeviceToHost));
      RLC_CK(cudaMemcpy(tch.data(), g.touched, 4 * size_t(nc), cudaMemcpyDeviceToHost));
    }
    uint32_t n = 0;
    for (size_t s = 0; s < cap; ++s) {
      if (sk[2 * s] == 0 && sk[2 * s + 1] == 0) continue;  // empty slot
      const uint32_t c = sc[s];
      if (c >= nc) continue;  // (cannot happen between calls: claims publish their cell)
      if (n < max_slots) {
        if (slot_out) slot_out[n] = uint32_t(s);
        if (cell_out) cell_out[n] = c;
        if (key_out)
          key_out[n] = rlc_cell_key{int32_t(ck[5 * c]), int32_t(ck[5 * c + 1]),
                                    int32_t(ck[5 * c + 2]), ck[5 * c + 3], ck[5 * c + 4]};
        if (touched_out) touched_out[n] = tch[c] ? 1 : 0;
      }
      ++n;
    }
    *count_out = n;
  });
}

rlc_status rlc_grid_template(const rlc_grid* grid, uint32_t* node_ids, uint32_t* ends, double* q,
                             double* cdf, uint32_t* visits, double* eps_q) {
  return guarded([&] {
    require(grid != nullptr, "rlc_grid_template: null grid");
    const rlc::HostCut& t = grid->tmpl;
    const size_t M = t.q.size();
    if (node_ids) std::memcpy(node_ids, t.node_ids.data(), 4 * M);
    if (ends) std::memcpy(ends, t.ends.data(), 4 * M);
    if (q) std::memcpy(q, t.q.data(), 8 * M);
    if (cdf) std::memcpy(cdf, t.cdf.data(), 8 * M);
    if (visits) std::memcpy(visits, t.visits.data(), 4 * M);
    if (eps_q) *eps_q = t.eps_q;
  });
}

rlc_status rlc_framebuffer_create(const rlc_context* ctx, int32_t width, int32_t height,
                                  rlc_framebuffer** out) {
  return guarded([&] {
    require(ctx != nullptr && out != nullptr, "rlc_framebuffer_create: null argument");
    require(width > 0 && height > 0, "rlc_framebuffer_create: empty raster");
    *out = nullptr;
    RLC_CK(cudaSetDevice(ctx->device));
    auto fb = std::make_unique<rlc_framebuffer>();
    fb->ctx = ctx;
    fb->width = width;
    fb->height = height;
    const size_t npix = size_t(width) * size_t(height);
    fb->fb.sum = fb->arena.alloc<double>(3 * npix);
    fb->fb.count = fb->arena.alloc<unsigned long long>(npix);
    fb->fb.width = uint32_t(width);
    fb->d_image = fb->arena.alloc<double>(3 * npix);
    RLC_CK(cudaMemsetAsync(fb->fb.sum, 0, 24 * npix, ctx->stream));
    RLC_CK(cudaMemsetAsync(fb->fb.count, 0, 8 * npix, ctx->stream));
    RLC_CK(cudaStreamSynchronize(ctx->stream));
    fb->holds_ref = true;
    const_cast<rlc_context*>(ctx)->refs.fetch_add(1);
    *out = fb.release();
  });
}

rlc_status rlc_framebuffer_destroy(rlc_framebuffer* fb) {
  return guarded([&] {
    if (!fb) return;
    const rlc_context* ctx = fb->ctx;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->sstream) cudaStreamSynchronize(ctx->sstream);  // a pending accumulation
    const bool release = fb->holds_ref;
    delete fb;
    if (release) context_release(ctx);
  });
}

rlc_status rlc_framebuffer_clear(rlc_framebuffer* fb) {
  return guarded([&] {
    require(fb != nullptr, "rlc_framebuffer_clear: null framebuffer");
    const_cast<rlc_context*>(fb->ctx)->join_acc();
    const size_t npix = size_t(fb->width) * size_t(fb->height);
    RLC_CK(cudaMemsetAsync(fb->fb.sum, 0, 24 * npix, fb->ctx->stream));
    RLC_CK(cudaMemsetAsync(fb->fb.count, 0, 8 * npix, fb->ctx->stream));
  });
}

rlc_status rlc_framebuffer_download(const rlc_framebuffer* fb, double* sum, uint64_t* count) {
  return guarded([&] {
    require(fb != nullptr, "rlc_framebuffer_download: null framebuffer");
    const_cast<rlc_context*>(fb->ctx)->join_acc();
    const size_t npix = size_t(fb->width) * size_t(fb->height);
    RLC_CK(cudaStreamSynchronize(fb->ctx->stream));
    if (sum) RLC_CK(cudaMemcpy(sum, fb->fb.sum, 24 * npix, cudaMemcpyDeviceToHost));
    if (count) RLC_CK(cudaMemcpy(count, fb->fb.count, 8 * npix, cudaMemcpyDeviceToHost));
  });
}

rlc_status rlc_framebuffer_resolve(const rlc_framebuffer* fb, double* image) {
  return guarded([&] {
    require(fb != nullptr && image != nullptr, "rlc_framebuffer_resolve: null argument");
    const_cast<rlc_context*>(fb->ctx)->join_acc();
    const uint32_t npix = uint32_t(size_t(fb->width) * size_t(fb->height));
    rlc::launch_resolve(fb->fb, npix, fb->d_image, fb->ctx->stream);
    RLC_CK(cudaMemcpyAsync(image, fb->d_image, 24 * size_t(npix), cudaMemcpyDeviceToHost,
                           fb->ctx->stream));
    RLC_CK(cudaStreamSynchronize(fb->ctx->stream));
  });
}

rlc_status rlc_render_pass(const rlc_context* ctx, const rlc_render_config* config,
                           uint32_t pass_index, rlc_grid* grid, rlc_framebuffer* fb) {
  return guarded([&] {
    require(ctx != nullptr && config != nullptr, "render_pass: null argument");
    enqueue_pass(ctx, config, pass_index, grid, fb, 0, uint32_t(ctx->host.cam.height));
    finish_sync(ctx, grid);
  });
}

rlc_status rlc_render_pass_rows(const rlc_context* ctx, const rlc_render_config* config,
                                uint32_t pass_index, rlc_grid* grid, rlc_framebuffer* fb,
                                uint32_t row_begin, uint32_t row_end) {
  return guarded([&] {
    require(ctx != nullptr && config != nullptr, "render_pass: null argument");
    enqueue_pass(ctx, config, pass_index, grid, fb, row_begin, row_end);
    finish_sync(ctx, grid);
  });
}

rlc_status rlc_render_pass_async(const rlc_context* ctx, const rlc_render_config* config,
                                 uint32_t pass_index, rlc_grid* grid, rlc_framebuffer* fb) {
  return guarded([&] {
    require(ctx != nullptr && config != nullptr, "render_pass: null argument");
    enqueue_pass(ctx, config, pass_index, grid, fb, 0, uint32_t(ctx->host.cam.height));
  });
}

namespace {

void shard_trace(rlc_context* ctx, const rlc_render_config* config, uint32_t pass_index,
                 rlc_grid* grid, uint32_t row_begin, uint32_t row_end, uint64_t cap,
                 const rlc::PeerDsts* dsts = nullptr, uint32_t ndst = 0, uint32_t rank = 0) {
  require(config->sampler == RLC_SAMPLER_RL_LIGHTCUTS && grid != nullptr,
          "rlc_shard_trace: the sharded pass is the learned sampler's");
  require(cap > 0 && cap < (1ull << 31), "rlc_shard_trace: bad record capacity");
  RLC_CK(cudaSetDevice(ctx->device));
  PassSetup S = setup_pass(ctx, config, pass_index, grid, nullptr, false, row_begin, row_end);
  require(S.nv <= cap, "rlc_shard_trace: the band has more path vertices than the record capacity");
  S.p.defer_insert = 1;  // new keys go in with all ranks' records (rlc_shard_fold)
  ctx->shard = PassParamsHolder{S.p, S.g, S.n, S.nv, grid, true};
  ctx->shard_folded = false;
  ctx->ensure_block(cap);
  if (S.nv > 0) {
    uint32_t *k, *v;
    enqueue_trace(ctx, S, grid, &k, &v);
  }
  ctx->last_pass = S.p;
  ctx->last_pb = ctx->pb;
  ctx->last_valid = true;
  if (dsts)  // the records straight into the gathered buffers (peer memory)
    rlc::launch_export_block_to(S.g, ctx->pb, S.nv, *dsts, ndst, rank, uint32_t(cap), ctx->stream);
  else
    rlc::launch_export_block(S.g, ctx->pb, S.nv, ctx->block, uint32_t(cap), ctx->stream);
  RLC_CK(cudaGetLastError());
}

void shard_fold(rlc_context* ctx, const rlc_render_config* config, rlc_grid* grid,
                const void* blocks, uint32_t nranks, uint32_t rank, int owner_fold) {
  require(nranks > 0 && rank < nranks, "rlc_shard_fold: bad rank");
  require(ctx->shard.valid && ctx->shard.grid == grid && !ctx->shard_folded,
          "rlc_shard_fold: no matching rlc_shard_trace on this grid");
  require(blocks != nullptr, "rlc_shard_fold: null blocks");
  (void)config;
  RLC_CK(cudaSetDevice(ctx->device));
  const PassParamsHolder& S = ctx->shard;
  ctx->ensure_exchange(nranks, uint32_t(ctx->block_cap));
  ctx->xb.rec = static_cast<const rlc::ExchangeRecord*>(blocks);
  // Owner mode exchanges either per-slot values (q_before and the entry's
  // record count at its last record: 12 B per slot, all-reduced) or, when
  // the records far outnumber the cut entries (c5), per-entry final values
  // (12 B per entry, all-reduced) plus q_before reduce-scattered to each
  // band: the one with fewer bytes per rank.  RLC_SHARD_ENTRY=0/1 forces it.
  {
    const uint64_t S = uint64_t(nranks) * ctx->xb.stride;
    const uint64_t E = uint64_t(grid->dev.capacity) * grid->dev.M;
    bool entry = owner_fold != 0 && nranks > 1 && 3 * E < 2 * S;
    if (const char* e = std::getenv("RLC_SHARD_ENTRY")) entry = owner_fold != 0 && std::atoi(e) != 0;
    ctx->xb.entry_mode = entry ? 1u : 0u;
    if (entry) ctx->ensure_entries(E);
  }
  ctx->stage(9, [&] {
    rlc::launch_shard_fold(S.g, S.p, rank, owner_fold != 0, ctx->xb, ctx->stream);
  });
  // the next pass's lookups (its primary rays on the side stream) must see
  // this pass's new keys
  if (ctx->overlap && ctx->pstream) {
    RLC_CK(cudaEventRecord(ctx->ev_commit, ctx->stream));
    RLC_CK(cudaStreamWaitEvent(ctx->pstream, ctx->ev_commit, 0));
  }
  ctx->stage(3, [&] {
    rlc::launch_shard_sortfold(S.g, S.p, grid->key_bits, owner_fold != 0, ctx->xb, ctx->stream);
  });
  ctx->shard_folded = true;
  RLC_CK(cudaGetLastError());
}

void shard_finish(rlc_context* ctx, rlc_grid* grid, rlc_framebuffer* fb, uint32_t rank,
                  int owner_fold) {
  require(ctx->shard.valid && ctx->shard.grid == grid && ctx->shard_folded,
          "rlc_shard_finish: no matching rlc_shard_fold on this grid");
  require(fb != nullptr && fb->width == ctx->host.cam.width && fb->height == ctx->host.cam.height,
          "render_pass: framebuffer size must match the camera");
  RLC_CK(cudaSetDevice(ctx->device));
  const PassParamsHolder S = ctx->shard;
  ctx->shard.valid = false;
  cudaStream_t st = ctx->stream;
  if (owner_fold) ctx->stage(3, [&] { rlc::launch_shard_apply(S.g, S.p, rank, ctx->xb, st); });
  rlc::launch_shard_scatter(S.g, ctx->pb, S.nv, rank, ctx->xb, st);
  if (S.n > 0) ctx->stage(4, [&] { rlc::launch_accumulate(ctx->dev, S.p, ctx->pb, fb->fb, st); });
  RLC_CK(cudaEventRecord(ctx->ev_gbuf_free[ctx->slot_of(S.p.pass_index)], st));
  RLC_CK(cudaGetLastError());
}

}  // namespace

rlc_status rlc_shard_trace(const rlc_context* cctx, const rlc_render_config* config,
                           uint32_t pass_index, rlc_grid* grid, uint32_t row_begin,
                           uint32_t row_end, uint64_t cap_records, void** block,
                           uint64_t* block_bytes) {
  return guarded([&] {
    require(cctx != nullptr && config != nullptr && block != nullptr && block_bytes != nullptr,
            "rlc_shard_trace: null argument");
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    shard_trace(ctx, config, pass_index, grid, row_begin, row_end, cap_records);
    *block = ctx->block;
    *block_bytes = ctx->block_bytes();
  });
}

rlc_status rlc_shard_trace_to(const rlc_context* cctx, const rlc_render_config* config,
                              uint32_t pass_index, rlc_grid* grid, uint32_t row_begin,
                              uint32_t row_end, uint64_t cap_records, uint32_t rank,
                              void* const* dst_buffers, uint32_t ndst) {
  return guarded([&] {
    require(cctx != nullptr && config != nullptr && dst_buffers != nullptr,
            "rlc_shard_trace_to: null argument");
    require(ndst >= 1 && ndst <= rlc::kMaxPeers, "rlc_shard_trace_to: bad destination count");
    rlc::PeerDsts d{};
    for (uint32_t k = 0; k < ndst; ++k) {
      require(dst_buffers[k] != nullptr, "rlc_shard_trace_to: null destination");
      d.p[k] = static_cast<rlc::ExchangeRecord*>(dst_buffers[k]);
    }
    shard_trace(const_cast<rlc_context*>(cctx), config, pass_index, grid, row_begin, row_end,
                cap_records, &d, ndst, rank);
  });
}

rlc_status rlc_shard_fold(const rlc_context* cctx, const rlc_render_config* config,
                          rlc_grid* grid, const void* blocks, uint32_t nranks, uint32_t rank,
                          int owner_fold, double** q_before_slots, uint32_t** seg_counts,
                          uint64_t* slots) {
  return guarded([&] {
    require(cctx != nullptr && config != nullptr, "rlc_shard_fold: null argument");
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    shard_fold(ctx, config, grid, blocks, nranks, rank, owner_fold);
    if (q_before_slots) *q_before_slots = ctx->xb.q_rec;
    if (seg_counts) *seg_counts = ctx->xb.entry_mode ? nullptr : ctx->xb.seg_n;
    if (slots) *slots = uint64_t(nranks) * ctx->xb.stride;
  });
}

rlc_status rlc_shard_entry_arrays(const rlc_context* cctx, double** entry_q,
                                  uint32_t** entry_counts, uint64_t* entries) {
  return guarded([&] {
    require(cctx != nullptr, "rlc_shard_entry_arrays: null context");
    const bool on = cctx->xb.entry_mode != 0;
    if (entry_q) *entry_q = on ? cctx->xb.ent_q : nullptr;
    if (entry_counts) *entry_counts = on ? cctx->xb.ent_n : nullptr;
    if (entries) *entries = on ? cctx->xb.entries : 0;
  });
}

rlc_status rlc_shard_finish(const rlc_context* cctx, rlc_grid* grid, rlc_framebuffer* fb,
                            uint32_t rank, int owner_fold) {
  return guarded([&] {
    require(cctx != nullptr, "rlc_shard_finish: null argument");
    shard_finish(const_cast<rlc_context*>(cctx), grid, fb, rank, owner_fold);
  });
}

rlc_status rlc_shard_sync(const rlc_context* cctx, rlc_grid* grid) {
  return guarded([&] {
    require(cctx != nullptr, "rlc_shard_sync: null argument");
    finish_sync(cctx, grid);
  });
}

// ---- NCCL data plane of sharded frames -----------------------------------
// libnccl is loaded at the first communicator (dlopen of the soname torch
// also uses, so one process shares one NCCL): single-GPU use needs no NCCL.
namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                 ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.init_rank = reinterpret_cast<decltype(a.init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.reduce_scatter =
        reinterpret_cast<decltype(a.reduce_scatter)>(dlsym(h, "ncclReduceScatter"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    return a;
  }();
  if (!api.init_rank || !api.all_gather || !api.all_reduce)
    throw std::runtime_error("rlcuts_b200: libnccl.so.2 could not be loaded (multi-GPU frames)");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string(what) + ": " +
                             (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}
}  // namespace

struct rlc_comm {
  ncclComm_t comm = nullptr;
  uint32_t nranks = 1, rank = 0;
  int device = 0;
  DeviceArena arena;
  void* gathered = nullptr;  // nranks record blocks
  uint64_t gathered_bytes = 0;
  // peer exchange (rlc_comm_enable_peer_exchange): this rank's receive buffer
  // (its own cudaMalloc, exported by CUDA IPC) and every rank's, opened here
  bool peer = false;
  uint64_t peer_cap = 0;
  void* peer_recv = nullptr;
  rlc::PeerDsts peer_dst{};
  int* barrier = nullptr;  // one int all-reduced after the stores
  void release_peer() {
    for (uint32_t r = 0; r < nranks && r < rlc::kMaxPeers; ++r)
      if (r != rank && peer_dst.p[r]) cudaIpcCloseMemHandle(peer_dst.p[r]);
    if (peer_recv) cudaFree(peer_recv);
    if (barrier) cudaFree(barrier);
    peer_recv = nullptr;
    barrier = nullptr;
    peer_dst = {};
    peer = false;
  }
  ~rlc_comm() {
    release_peer();
    if (comm) nccl().destroy(comm);
  }
};

rlc_status rlc_comm_unique_id(uint8_t* id128) {
  return guarded([&] {
    require(id128 != nullptr, "rlc_comm_unique_id: null argument");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id128, &id, sizeof(id));
  });
}

rlc_status rlc_comm_create(int device, uint32_t nranks, uint32_t rank, const uint8_t* id128,
                           rlc_comm** out) {
  return guarded([&] {
    require(id128 != nullptr && out != nullptr && nranks > 0 && rank < nranks,
            "rlc_comm_create: bad argument");
    *out = nullptr;
    check_device(device);
    auto c = std::make_unique<rlc_comm>();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    nccl_check(nccl().init_rank(&c->comm, int(nranks), id, int(rank)), "ncclCommInitRank");
    *out = c.release();
  });
}

rlc_status rlc_comm_destroy(rlc_comm* comm) {
  return guarded([&] { delete comm; });
}

rlc_status rlc_comm_enable_peer_exchange(rlc_comm* comm, uint64_t cap_records, int enable) {
  return guarded([&] {
    require(comm != nullptr, "rlc_comm_enable_peer_exchange: null communicator");
    require(comm->nranks <= rlc::kMaxPeers, "rlc_comm_enable_peer_exchange: too many ranks");
    RLC_CK(cudaSetDevice(comm->device));
    RLC_CK(cudaDeviceSynchronize());
    comm->release_peer();
    if (!enable) return;
    require(cap_records > 0, "rlc_comm_enable_peer_exchange: bad record capacity");
    // two halves by pass parity: a rank writes pass p + 1's records while
    // the others may still read pass p's (the per-pass barrier then orders
    // pass p + 2's writes after every rank's reads of pass p)
    const size_t bytes =
        2 * size_t(comm->nranks) * (cap_records + 1) * sizeof(rlc::ExchangeRecord);
    RLC_CK(cudaMalloc(&comm->peer_recv, bytes));
    RLC_CK(cudaMemset(comm->peer_recv, 0, bytes));
    RLC_CK(cudaMalloc(&comm->barrier, sizeof(int)));
    RLC_CK(cudaMemset(comm->barrier, 0, sizeof(int)));
    comm->peer_dst.p[comm->rank] = static_cast<rlc::ExchangeRecord*>(comm->peer_recv);
    if (comm->nranks > 1) {  // every rank's IPC handle to every rank (setup, synchronizing)
      cudaIpcMemHandle_t mine;
      RLC_CK(cudaIpcGetMemHandle(&mine, comm->peer_recv));
      const size_t hb = sizeof(cudaIpcMemHandle_t);
      unsigned char* dev = nullptr;
      RLC_CK(cudaMalloc(&dev, hb * (comm->nranks + 1)));
      RLC_CK(cudaMemcpy(dev + hb * comm->nranks, &mine, hb, cudaMemcpyHostToDevice));
      nccl_check(nccl().all_gather(dev + hb * comm->nranks, dev, hb, ncclUint8, comm->comm, 0),
                 "ncclAllGather");
      std::vector<cudaIpcMemHandle_t> all(comm->nranks);
      RLC_CK(cudaMemcpy(all.data(), dev, hb * comm->nranks, cudaMemcpyDeviceToHost));
      cudaFree(dev);
      for (uint32_t r = 0; r < comm->nranks; ++r) {
        if (r == comm->rank) continue;
        void* p = nullptr;
        RLC_CK(cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess));
        comm->peer_dst.p[r] = static_cast<rlc::ExchangeRecord*>(p);
      }
    }
    comm->peer_cap = cap_records;
    comm->peer = true;
  });
}

namespace {
// One sharded frame on the context stream (rlc_shard_frame): the band's
// trace, the NCCL exchange, the exact fold and split-collapse.
void shard_frame_body(rlc_context* ctx, const rlc_render_config* config, uint32_t pass_index,
                      rlc_grid* grid, rlc_framebuffer* fb, rlc_comm* comm, uint32_t row_begin,
                      uint32_t row_end, uint64_t cap_records, int owner_fold) {
  cudaStream_t st = ctx->stream;
  if (comm->peer) {
    // the records stored straight into every rank's receive buffer over
    // NVLink, then one all-reduce of an int as the barrier: each rank's
    // stores precede its part of the collective on its stream
    require(cap_records == comm->peer_cap,
            "rlc_shard_frame: record capacity differs from the peer exchange's");
    const size_t half = size_t(pass_index & 1u) * comm->nranks * (cap_records + 1);
    rlc::PeerDsts d = comm->peer_dst;
    for (uint32_t r = 0; r < comm->nranks; ++r) d.p[r] += half;
    shard_trace(ctx, config, pass_index, grid, row_begin, row_end, cap_records, &d, comm->nranks,
                comm->rank);
    if (comm->nranks > 1)
      nccl_check(nccl().all_reduce(comm->barrier, comm->barrier, 1, ncclInt32, ncclSum, comm->comm,
                                   st),
                 "ncclAllReduce");
    shard_fold(ctx, config, grid, static_cast<rlc::ExchangeRecord*>(comm->peer_recv) + half,
               comm->nranks, comm->rank, owner_fold);
  } else {
  shard_trace(ctx, config, pass_index, grid, row_begin, row_end, cap_records);
  const uint64_t bb = ctx->block_bytes();
  if (comm->gathered_bytes < bb * comm->nranks) {
    ctx->sync_all();
    comm->arena.release();
    comm->gathered = comm->arena.alloc<unsigned char>(bb * comm->nranks);
    comm->gathered_bytes = bb * comm->nranks;
  }
  // the exchange: every rank's block to every rank (fixed size: no host count)
  nccl_check(nccl().all_gather(ctx->block, comm->gathered, bb, ncclUint8, comm->comm, st),
             "ncclAllGather");
  shard_fold(ctx, config, grid, comm->gathered, comm->nranks, comm->rank, owner_fold);
  }
  if (owner_fold && comm->nranks > 1 && ctx->xb.entry_mode) {
    // each band's q_before from the owners (reduce-scatter, in place: this
    // rank's block of slots), every entry's final q and count (all-reduce)
    const size_t stride = ctx->xb.stride;
    require(nccl().reduce_scatter != nullptr, "rlc_shard_frame: libnccl lacks ncclReduceScatter");
    nccl_check(nccl().reduce_scatter(ctx->xb.q_rec, ctx->xb.q_rec + size_t(comm->rank) * stride,
                                     stride, ncclFloat64, ncclSum, comm->comm, st),
               "ncclReduceScatter");
    nccl_check(nccl().all_reduce(ctx->xb.ent_q, ctx->xb.ent_q, ctx->xb.entries, ncclFloat64,
                                 ncclSum, comm->comm, st),
               "ncclAllReduce");
    nccl_check(nccl().all_reduce(ctx->xb.ent_n, ctx->xb.ent_n, ctx->xb.entries, ncclUint32,
                                 ncclSum, comm->comm, st),
               "ncclAllReduce");
  } else if (owner_fold && comm->nranks > 1) {  // q_before and entry counts from the cells' owners
    const size_t slots = size_t(comm->nranks) * ctx->xb.stride;
    nccl_check(nccl().all_reduce(ctx->xb.q_rec, ctx->xb.q_rec, slots, ncclFloat64, ncclSum,
                                 comm->comm, st),
               "ncclAllReduce");
    nccl_check(nccl().all_reduce(ctx->xb.seg_n, ctx->xb.seg_n, slots, ncclUint32, ncclSum,
                                 comm->comm, st),
               "ncclAllReduce");
  }
  shard_finish(ctx, grid, fb, comm->rank, owner_fold);
  RLC_CK(cudaMemsetAsync(grid->d_changes, 0, 4, st));
  enqueue_eop(grid, ctx, &config->cut, grid->d_changes);  // split-collapse: identical on every rank
}
}  // namespace

rlc_status rlc_shard_frame(const rlc_context* cctx, const rlc_render_config* config,
                           uint32_t pass_index, rlc_grid* grid, rlc_framebuffer* fb,
                           rlc_comm* comm, uint32_t row_begin, uint32_t row_end,
                           uint64_t cap_records, int owner_fold) {
  return guarded([&] {
    require(cctx != nullptr && config != nullptr && comm != nullptr && grid != nullptr,
            "rlc_shard_frame: null argument");
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    require(comm->device == ctx->device, "rlc_shard_frame: communicator on another device");
    shard_frame_body(ctx, config, pass_index, grid, fb, comm, row_begin, row_end, cap_records,
                     owner_fold);
  });
}

rlc_status rlc_shard_frames(const rlc_context* cctx, const rlc_render_config* config,
                            uint32_t first_pass, uint32_t count, rlc_grid* grid,
                            rlc_framebuffer* fb, rlc_comm* comm, uint32_t row_begin,
                            uint32_t row_end, uint64_t cap_records, int owner_fold,
                            int use_graph) {
  return guarded([&] {
    require(cctx != nullptr && config != nullptr && comm != nullptr && grid != nullptr,
            "rlc_shard_frames: null argument");
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    require(comm->device == ctx->device, "rlc_shard_frames: communicator on another device");
    auto single = [&](uint32_t p) {
      shard_frame_body(ctx, config, p, grid, fb, comm, row_begin, row_end, cap_records,
                       owner_fold);
    };
    constexpr uint32_t kFrames = 2;  // one frame per G-buffer slot
    if (!use_graph || ctx->timing || count < kFrames) {
      for (uint32_t p = first_pass; p < first_pass + count; ++p) single(p);
      return;
    }
    cudaStream_t st = ctx->stream;
    if (!ctx->d_pass) {
      ctx->d_pass = ctx->arena.alloc<uint32_t>(2);
      ctx->d_changes = ctx->d_pass + 1;
      RLC_CK(cudaMemsetAsync(ctx->d_pass, 0, 8, st));
    }
    // every allocation outside the capture: one frame run directly sizes the
    // pass, block, exchange and gather buffers
    single(first_pass);
    ++first_pass;
    --count;
    auto& G = ctx->shard_graph;
    const bool same = G.exec && std::memcmp(&G.cfg, config, sizeof(*config)) == 0 &&
                      G.grid == grid && G.fb == fb && G.comm == comm && G.r0 == row_begin &&
                      G.r1 == row_end && G.cap == cap_records && G.owner == owner_fold &&
                      G.pb_gen == ctx->pb_gen && G.scene_gen == ctx->scene_gen &&
                      G.gathered == comm->gathered && G.block == ctx->block &&
                      G.peer_recv == comm->peer_recv;
    if (!same) {
      if (G.exec) {
        RLC_CK(cudaGraphExecDestroy(G.exec));
        G.exec = nullptr;
      }
      ctx->graph_pass_dev = ctx->d_pass;
      const uint64_t l0 = rlc::launches();
      cudaGraph_t graph = nullptr;
      RLC_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
      try {
        for (cudaEvent_t e : ctx->ev_gbuf_free) RLC_CK(cudaEventRecord(e, st));
        for (uint32_t i = 0; i < kFrames; ++i) single(i);  // slot i; pass *d_pass + i
        if (ctx->overlap && ctx->pstream) {  // join the side stream's last wait
          RLC_CK(cudaEventRecord(ctx->ev_prim_done, ctx->pstream));
          RLC_CK(cudaStreamWaitEvent(st, ctx->ev_prim_done, 0));
        }
        rlc::launch_add_u32(ctx->d_pass, kFrames, st);
      } catch (...) {
        cudaStreamEndCapture(st, &graph);
        if (graph) cudaGraphDestroy(graph);
        ctx->graph_pass_dev = nullptr;
        throw;
      }
      RLC_CK(cudaStreamEndCapture(st, &graph));
      ctx->graph_pass_dev = nullptr;
      G.launches = rlc::launches() - l0;
      const cudaError_t e = cudaGraphInstantiate(&G.exec, graph, 0);
      cudaGraphDestroy(graph);
      RLC_CK(e);
      G.cfg = *config;
      G.grid = grid;
      G.fb = fb;
      G.comm = comm;
      G.r0 = row_begin;
      G.r1 = row_end;
      G.cap = cap_records;
      G.owner = owner_fold;
      G.pb_gen = ctx->pb_gen;
      G.scene_gen = ctx->scene_gen;
      G.gathered = comm->gathered;
      G.peer_recv = comm->peer_recv;
      G.block = ctx->block;
    }
    const uint32_t replays = count / kFrames;
    rlc::launch_set_u32(ctx->d_pass, first_pass, st);
    for (uint32_t r = 0; r < replays; ++r) RLC_CK(cudaGraphLaunch(G.exec, st));
    rlc::add_launches(G.launches * replays);
    for (cudaEvent_t e : ctx->ev_gbuf_free) RLC_CK(cudaEventRecord(e, st));
    for (uint32_t p = first_pass + replays * kFrames; p < first_pass + count; ++p) single(p);
  });
}

rlc_status rlc_context_set_pdf_mode(rlc_context* ctx, int mode) {
  return guarded([&] {
    require(ctx != nullptr, "rlc_context_set_pdf_mode: null context");
    require(mode == RLC_PDF_LIVE_Q || mode == RLC_PDF_FROZEN_CDF, "rlc_context_set_pdf_mode: bad mode");
    ctx->frozen_pdf = mode == RLC_PDF_FROZEN_CDF;
    ++ctx->scene_gen;  // captured pass graphs hold the old pass parameters
  });
}

rlc_status rlc_context_enable_sample_export(rlc_context* ctx, int enable) {
  return guarded([&] {
    require(ctx != nullptr, "rlc_context_enable_sample_export: null context");
    ctx->export_samples = enable != 0;
  });
}

rlc_status rlc_pass_samples(const rlc_context* cctx, uint64_t max_n, rlc_sample_record* out,
                            uint64_t* n_out) {
  return guarded([&] {
    require(cctx != nullptr && n_out != nullptr, "rlc_pass_samples: null argument");
    static_assert(sizeof(rlc_sample_record) == sizeof(rlc::SampleExport), "record layout");
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    const rlc::PassParams& p = ctx->last_pass;
    *n_out = p.nv;
    if (out == nullptr || max_n == 0 || p.nv == 0 || !ctx->last_valid) return;
    RLC_CK(cudaSetDevice(ctx->device));
    ctx->sync_all();
    const uint64_t n = std::min<uint64_t>(max_n, p.nv);
    DeviceArena tmp;
    rlc::SampleExport* d = tmp.alloc<rlc::SampleExport>(p.nv);
    rlc::launch_export_samples(p, ctx->last_pb, d, ctx->stream);
    RLC_CK(cudaGetLastError());
    RLC_CK(cudaMemcpyAsync(out, d, n * sizeof(rlc_sample_record), cudaMemcpyDeviceToHost,
                           ctx->stream));
    RLC_CK(cudaStreamSynchronize(ctx->stream));
  });
}

rlc_status rlc_end_of_pass_update(rlc_grid* grid, const rlc_context* ctx,
                                  const rlc_cut_config* cut, uint32_t* changes) {
  return guarded([&] {
    require(grid != nullptr, "end_of_pass_update: null grid");
    RLC_CK(cudaMemsetAsync(grid->d_changes, 0, 4, ctx->stream));
    enqueue_eop(grid, ctx, cut, grid->d_changes);
    uint32_t c = 0;
    RLC_CK(cudaMemcpyAsync(&c, grid->d_changes, 4, cudaMemcpyDeviceToHost, ctx->stream));
    finish_sync(ctx, grid);
    if (changes) *changes = c;
  });
}

rlc_status rlc_end_of_pass_update_async(rlc_grid* grid, const rlc_context* ctx,
                                        const rlc_cut_config* cut) {
  return guarded([&] {
    require(grid != nullptr, "end_of_pass_update: null grid");
    RLC_CK(cudaMemsetAsync(grid->d_changes, 0, 4, ctx->stream));
    enqueue_eop(grid, ctx, cut, grid->d_changes);
  });
}

rlc_status rlc_grid_last_changes(const rlc_grid* grid, uint32_t* changes) {
  return guarded([&] {
    require(grid != nullptr && changes != nullptr, "rlc_grid_last_changes: null argument");
    RLC_CK(cudaMemcpyAsync(changes, grid->d_changes, 4, cudaMemcpyDeviceToHost, grid->ctx->stream));
    RLC_CK(cudaStreamSynchronize(grid->ctx->stream));
  });
}

}  // extern "C"

namespace {

bool same_grid_config(const rlc_render_config& a, const rlc_render_config& b) {
  return a.hash.capacity == b.hash.capacity && a.hash.probe_limit == b.hash.probe_limit &&
         a.hash.normal_bits == b.hash.normal_bits && a.hash.jitter_scale == b.hash.jitter_scale &&
         a.cut.cut_size == b.cut.cut_size && a.cut.eps_q == b.cut.eps_q &&
         a.cut.alpha == b.cut.alpha && a.cut.alpha_schedule == b.cut.alpha_schedule;
}

// A fresh HashGrid in place: empty slots, no cells, zeroed counters.  Cut
// rows need no reset (a row is written from the template when its cell is
// inserted, src/hash_grid.cpp:126).
void reset_grid(rlc_grid* g, cudaStream_t st) {
  const size_t cap = g->dev.capacity;
  RLC_CK(cudaMemsetAsync(g->dev.slot_keys, 0, 16 * cap, st));
  RLC_CK(cudaMemsetAsync(g->dev.claim, 0xff, 8 * cap, st));
  RLC_CK(cudaMemsetAsync(g->dev.touched, 0, 4 * cap, st));
  RLC_CK(cudaMemsetAsync(g->dev.counters, 0, sizeof(unsigned long long) * rlc::kCntNum, st));
  RLC_CK(cudaMemsetAsync(g->d_changes, 0, 4, st));
}

// The context's reusable render_frame state (grid, framebuffer, per-pass
// change counts), allocated once -- at context creation for the creation
// config -- so render_frame itself performs no device allocation.
void prepare_frame_cache(rlc_context* ctx, const rlc_render_config* config) {
  if (config->sampler == RLC_SAMPLER_RL_LIGHTCUTS) {
    if (ctx->frame_grid == nullptr || !same_grid_config(ctx->frame_cfg, *config)) {
      if (ctx->frame_grid) {
        rlc_grid_destroy(ctx->frame_grid);
        ctx->frame_grid = nullptr;
      }
      rlc_grid* g = nullptr;
      const rlc_status st = rlc_grid_create(ctx, config, &g);
      if (st == RLC_ERR_INVALID_ARGUMENT) throw rlc::InvalidArgument(g_err);
      if (st != RLC_OK) throw std::runtime_error(g_err);
      g->holds_ref = false;  // owned by the context itself
      ctx->refs.fetch_sub(1);
      ctx->frame_grid = g;
      ctx->frame_cfg = *config;
    }
  }
  if (ctx->frame_fb == nullptr) {
    rlc_framebuffer* fb = nullptr;
    if (rlc_framebuffer_create(ctx, ctx->host.cam.width, ctx->host.cam.height, &fb) != RLC_OK)
      throw std::runtime_error(g_err);
    fb->holds_ref = false;  // owned by the context itself
    ctx->refs.fetch_sub(1);
    ctx->frame_fb = fb;
    // render_frame's image download staging (download_to_host), allocated
    // with the rest of the frame cache so render_frame allocates nothing
    const size_t img = size_t(24) * size_t(fb->width) * size_t(fb->height);
    if (img >= (size_t(4) << 20) && ctx->h_stage_cap < img) {
      if (ctx->h_stage) RLC_CK(cudaFreeHost(ctx->h_stage));
      ctx->h_stage = nullptr;
      ctx->h_stage_cap = 0;
      RLC_CK(cudaMallocHost(&ctx->h_stage, img));
      ctx->h_stage_cap = img;
    }
  }
  if (config->passes > ctx->frame_hist_cap) {
    ctx->frame_hist_arena.release();
    ctx->frame_hist = ctx->frame_hist_arena.alloc<uint32_t>(config->passes);
    ctx->frame_hist_cap = config->passes;
  }
  if (config->passes != 0 && config->spp % config->passes == 0)
    ctx->ensure_scratch(uint32_t(ctx->host.cam.width) * uint32_t(ctx->host.cam.height) *
                        (config->spp / config->passes));
}

}  // namespace

extern "C" {

namespace {

// Pinned host staging for the per-pixel error terms of render_frame_scored.
// Device -> caller host memory, synchronously on stream st: large copies go
// through the context's pinned staging buffer (full-rate DMA) and are fanned
// out to the caller's pageable memory by the worker pool; a pageable
// cudaMemcpy is staged by the driver at a fraction of that rate.
void download_to_host(rlc_context* ctx, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes < (size_t(4) << 20)) {
    RLC_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    RLC_CK(cudaStreamSynchronize(st));
    return;
  }
  if (bytes > ctx->h_stage_cap) {
    RLC_CK(cudaStreamSynchronize(st));
    if (ctx->h_stage) RLC_CK(cudaFreeHost(ctx->h_stage));
    ctx->h_stage = nullptr;
    ctx->h_stage_cap = 0;
    RLC_CK(cudaMallocHost(&ctx->h_stage, bytes));
    ctx->h_stage_cap = bytes;
  }
  RLC_CK(cudaMemcpyAsync(ctx->h_stage, src, bytes, cudaMemcpyDeviceToHost, st));
  RLC_CK(cudaStreamSynchronize(st));
  rlc::parallel_copy(dst, ctx->h_stage, bytes);
}

struct PinnedBuf {
  double* p = nullptr;
  explicit PinnedBuf(size_t n) { RLC_CK(cudaMallocHost(&p, n * sizeof(double))); }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

// render_frame (render.cpp:202-240), optionally scored against a reference
// image after every pass (render.cpp:226-228).
// Passes [first, first + count) of render_pass + end_of_pass_update
// (render.cpp:218-224), per-pass change counts into d_hist[pass] when given.
// With RLC_GRAPHS=1, small frames (at most kGraphMaxPaths paths, no stage
// timing) replay a captured CUDA graph of kGraphPasses passes, the
// next pass's primary rays overlapping each pass's tail inside the graph as
// on the streams.  The replay's first pass index lives in device memory
// (k_primary adds its position in the graph; a one-thread kernel files each
// pass's change count and one advances the index), so a replay needs no host
// work.  Larger frames, and the passes left over, are enqueued pass by pass.
// Opt-in because it measured no faster: c1 (65k paths per frame) runs 0.133
// ms per pass from the graph against 0.128 ms from the streams -- the small
// frames are bound by the dependent kernels' ramp-up, not by host launches.
constexpr uint64_t kGraphMaxPaths = 1u << 19;
constexpr uint32_t kGraphPasses = 8;

void run_passes(rlc_context* ctx, const rlc_render_config* cfg, rlc_grid* grid,
                rlc_framebuffer* fb, uint32_t first, uint32_t count, uint32_t* d_hist) {
  const uint32_t H = uint32_t(ctx->host.cam.height);
  const uint64_t paths = uint64_t(ctx->host.cam.width) * H * (cfg->passes ? cfg->spp / cfg->passes : 0);
  const char* env = std::getenv("RLC_GRAPHS");
  const bool use_graph = env && std::string(env) == "1" && !ctx->timing && paths > 0 && paths <= kGraphMaxPaths &&
                         cfg->max_depth >= 1 && count >= kGraphPasses;
  auto single = [&](uint32_t p) {
    enqueue_pass(ctx, cfg, p, grid, fb, 0, H);
    if (grid) enqueue_eop(grid, ctx, &cfg->cut, d_hist ? d_hist + p : grid->d_changes);
  };
  if (!use_graph) {
    for (uint32_t p = first; p < first + count; ++p) single(p);
    return;
  }
  cudaStream_t st = ctx->stream;
  if (!ctx->d_pass) {
    ctx->d_pass = ctx->arena.alloc<uint32_t>(2);
    ctx->d_changes = ctx->d_pass + 1;
    RLC_CK(cudaMemsetAsync(ctx->d_pass, 0, 8, st));
  }
  // validation and buffer sizing outside the capture (setup_pass allocates)
  setup_pass(ctx, cfg, first, grid, fb, true, 0, H);
  auto& G = ctx->graph;
  const bool same = G.exec && std::memcmp(&G.cfg, cfg, sizeof(*cfg)) == 0 && G.grid == grid &&
                    G.fb == fb && G.hist == d_hist && G.pb_gen == ctx->pb_gen &&
                    G.scene_gen == ctx->scene_gen && (!grid || G.alpha == grid->alpha);
  ctx->join_acc();
  if (!same) {
    if (G.exec) {
      RLC_CK(cudaGraphExecDestroy(G.exec));
      G.exec = nullptr;
    }
    ctx->graph_pass_dev = ctx->d_pass;
    const uint64_t l0 = rlc::launches();
    cudaGraph_t graph = nullptr;
    RLC_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    try {
      // both G-buffer slots are free when a replay starts (stream order)
      for (cudaEvent_t e : ctx->ev_gbuf_free) RLC_CK(cudaEventRecord(e, st));
      for (uint32_t i = 0; i < kGraphPasses; ++i) {
        enqueue_pass(ctx, cfg, i, grid, fb, 0, H);  // slot i & 1; pass *d_pass + i
        if (grid) enqueue_eop(grid, ctx, &cfg->cut, ctx->d_changes);
        rlc::launch_end_pass(ctx->d_pass, i, ctx->d_changes, grid ? d_hist : nullptr, st);
      }
      ctx->join_acc();
      rlc::launch_add_u32(ctx->d_pass, kGraphPasses, st);
    } catch (...) {
      cudaStreamEndCapture(st, &graph);
      if (graph) cudaGraphDestroy(graph);
      ctx->graph_pass_dev = nullptr;
      ctx->acc_pending = false;
      throw;
    }
    RLC_CK(cudaStreamEndCapture(st, &graph));
    ctx->graph_pass_dev = nullptr;
    G.launches = rlc::launches() - l0;
    const cudaError_t e = cudaGraphInstantiate(&G.exec, graph, 0);
    cudaGraphDestroy(graph);
    RLC_CK(e);
    G.cfg = *cfg;
    G.grid = grid;
    G.fb = fb;
    G.hist = d_hist;
    G.alpha = grid ? grid->alpha : 0.0;
    G.pb_gen = ctx->pb_gen;
    G.scene_gen = ctx->scene_gen;
  }
  const uint32_t replays = count / kGraphPasses;
  rlc::launch_set_u32(ctx->d_pass, first, st);
  for (uint32_t r = 0; r < replays; ++r) RLC_CK(cudaGraphLaunch(G.exec, st));
  rlc::add_launches(G.launches * replays);
  // later overlapped passes start their primary rays once the G-buffer slot
  // is free: both slots are free when the replays are done
  for (cudaEvent_t e : ctx->ev_gbuf_free) RLC_CK(cudaEventRecord(e, st));
  for (uint32_t p = first + replays * kGraphPasses; p < first + count; ++p) single(p);
}

void render_frame_impl(rlc_context* ctx, const rlc_render_config* config, const double* reference,
                       double* image_out, rlc_render_result* result, double* pass_mse) {
  require(config->passes != 0 && config->spp != 0 && config->spp % config->passes == 0,
          "render_frame: spp must be divisible by passes");
  const auto t0 = std::chrono::steady_clock::now();
  RLC_CK(cudaSetDevice(ctx->device));
  prepare_frame_cache(ctx, config);
  rlc_grid* grid = config->sampler == RLC_SAMPLER_RL_LIGHTCUTS ? ctx->frame_grid : nullptr;
  rlc_framebuffer* fb = ctx->frame_fb;
  cudaStream_t st = ctx->stream;
  if (grid) {
    grid->alpha = config->cut.alpha;
    reset_grid(grid, st);
  }
  const size_t npix = size_t(fb->width) * size_t(fb->height);
  RLC_CK(cudaMemsetAsync(fb->fb.sum, 0, 24 * npix, st));
  RLC_CK(cudaMemsetAsync(fb->fb.count, 0, 8 * npix, st));
  uint32_t* d_hist = ctx->frame_hist;
  RLC_CK(cudaMemsetAsync(d_hist, 0, 4 * size_t(config->passes), st));
  // the first pass's primary rays (side stream) insert into the reset table
  ctx->fence_side();
  // scoring: the reference on the device, per-pixel terms double-buffered to
  // pinned host memory, the ordered sum of pass p - 1 while pass p runs
  DeviceArena tmp;
  std::unique_ptr<PinnedBuf> h_err[2];
  double* d_ref = nullptr;
  double* d_err[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int k = 0; k < 2; ++k)
        if (e[k]) cudaEventDestroy(e[k]);
    }
  } ev_guard{ev};
  if (reference) {
    d_ref = tmp.alloc<double>(3 * npix);
    RLC_CK(cudaMemcpyAsync(d_ref, reference, 24 * npix, cudaMemcpyHostToDevice, st));
    for (int k = 0; k < 2; ++k) {
      d_err[k] = tmp.alloc<double>(npix);
      h_err[k] = std::make_unique<PinnedBuf>(npix);
      RLC_CK(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
    }
  }
  auto score = [&](uint32_t pass) {
    const int k = int(pass & 1u);
    RLC_CK(cudaEventSynchronize(ev[k]));
    pass_mse[pass] = rlc::sum_terms(h_err[k]->p, npix) / (3.0 * double(npix));
  };
  if (!reference) run_passes(ctx, config, grid, fb, 0, config->passes, d_hist);
  for (uint32_t pass = 0; reference && pass < config->passes; ++pass) {
    enqueue_pass(ctx, config, pass, grid, fb, 0, uint32_t(ctx->host.cam.height));
    if (grid) enqueue_eop(grid, ctx, &config->cut, d_hist + pass);
    {
      const int k = int(pass & 1u);
      ctx->join_acc();
      rlc::launch_pixel_err(fb->fb, uint32_t(npix), d_ref, d_err[k], st);
      RLC_CK(cudaMemcpyAsync(h_err[k]->p, d_err[k], 8 * npix, cudaMemcpyDeviceToHost, st));
      RLC_CK(cudaEventRecord(ev[k], st));
      if (pass > 0) score(pass - 1);
    }
  }
  if (reference) score(config->passes - 1);
  ctx->join_acc();
  if (image_out) {
    rlc::launch_resolve(fb->fb, uint32_t(npix), fb->d_image, st);
    download_to_host(ctx, image_out, fb->d_image, 24 * npix, st);
  }
  std::vector<uint32_t> h(config->passes);
  RLC_CK(cudaMemcpyAsync(h.data(), d_hist, 4 * h.size(), cudaMemcpyDeviceToHost, st));
  unsigned long long c[rlc::kCntNum] = {};
  if (grid)
    RLC_CK(cudaMemcpyAsync(c, grid->dev.counters, sizeof(c), cudaMemcpyDeviceToHost, st));
  finish_sync(ctx, grid);
  if (result) {
    result->num_passes = config->passes;
    if (result->sc_changes) std::memcpy(result->sc_changes, h.data(), 4 * h.size());
    result->occupied_cells = uint32_t(c[rlc::kCntCells]);
    result->lookups = c[rlc::kCntLookups];
    result->fallback_hits = c[rlc::kCntFallback];
    result->wall_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
}

void check_image(const double* px, int32_t w, int32_t h, const char* what) {
  require(px != nullptr && w > 0 && h > 0, what);
}

}  // namespace

rlc_status rlc_render_frame(const rlc_context* cctx, const rlc_render_config* config,
                            double* image_out, rlc_render_result* result) {
  return guarded([&] {
    require(cctx != nullptr && config != nullptr, "render_frame: null argument");
    render_frame_impl(const_cast<rlc_context*>(cctx), config, nullptr, image_out, result, nullptr);
  });
}

rlc_status rlc_render_passes_async(const rlc_context* cctx, const rlc_render_config* config,
                                   uint32_t first_pass, uint32_t count, rlc_grid* grid,
                                   rlc_framebuffer* fb) {
  return guarded([&] {
    require(cctx != nullptr && config != nullptr, "render_pass: null argument");
    require(config->sampler != RLC_SAMPLER_RL_LIGHTCUTS || grid != nullptr,
            "render_pass: learned sampler needs a hash grid");
    rlc_context* ctx = const_cast<rlc_context*>(cctx);
    RLC_CK(cudaSetDevice(ctx->device));
    if (count == 0) return;
    run_passes(ctx, config, grid, fb, first_pass, count, nullptr);
  });
}

rlc_status rlc_render_frame_scored(const rlc_context* cctx, const rlc_render_config* config,
                                   const double* reference, int32_t ref_width,
                                   int32_t ref_height, double* image_out,
                                   rlc_render_result* result, double* pass_mse) {
  return guarded([&] {
    require(cctx != nullptr && config != nullptr, "render_frame: null argument");
    require(reference == nullptr || pass_mse != nullptr, "render_frame: null pass_mse");
    if (reference)
      require(ref_width == cctx->host.cam.width && ref_height == cctx->host.cam.height,
              "mse: image dimensions disagree");
    render_frame_impl(const_cast<rlc_context*>(cctx), config, reference, image_out, result,
                      pass_mse);
  });
}

rlc_status rlc_image_write_pfm(const double* pixels, int32_t width, int32_t height,
                               const char* path) {
  return guarded([&] {
    require(path != nullptr, "write_pfm: null path");
    check_image(pixels, width, height, "write_pfm: bad image");
    rlc::write_pfm(pixels, width, height, path);
  });
}

rlc_status rlc_image_read_pfm(const char* path, double* pixels, uint64_t max_pixels,
                              int32_t* width, int32_t* height) {
  return guarded([&] {
    require(path != nullptr && width != nullptr && height != nullptr, "read_pfm: null argument");
    rlc::read_pfm(path, pixels, max_pixels, width, height);
  });
}

rlc_status rlc_image_write_ppm(const double* pixels, int32_t width, int32_t height,
                               const char* path) {
  return guarded([&] {
    require(path != nullptr, "write_ppm: null path");
    check_image(pixels, width, height, "write_ppm: bad image");
    rlc::write_ppm(pixels, width, height, path);
  });
}

rlc_status rlc_image_mse(const double* a, int32_t wa, int32_t ha, const double* b, int32_t wb,
                         int32_t hb, double* out) {
  return guarded([&] {
    require(out != nullptr, "mse: null output");
    require(wa == wb && ha == hb, "mse: image dimensions disagree");
    check_image(a, wa, ha, "mse: bad image");
    check_image(b, wb, hb, "mse: bad image");
    *out = rlc::mse(a, b, uint64_t(wa) * uint64_t(ha));
  });
}

rlc_status rlc_image_relative_mse(const double* a, int32_t wa, int32_t ha, const double* b,
                                  int32_t wb, int32_t hb, double* out) {
  return guarded([&] {
    require(out != nullptr, "relative_mse: null output");
    require(wa == wb && ha == hb, "mse: image dimensions disagree");
    check_image(a, wa, ha, "mse: bad image");
    check_image(b, wb, hb, "mse: bad image");
    *out = rlc::relative_mse(a, b, uint64_t(wa) * uint64_t(ha));
  });
}

}  // extern "C"
