// rlc_kernels.h -- device-side views and the launchers the host runtime calls.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "rlc_common.h"

namespace rlc {

constexpr uint32_t kNoSlot = 0xffffffffu;    // path without an RL lookup
constexpr uint32_t kFallback = 0xfffffffeu;  // probe exhaustion -> fallback cut
// a key not in the table when the pass started, inserted (or refused) in
// canonical order after the lookups (k_insert / k_commit); its cut is the
// template until then
constexpr uint32_t kPending = 0xfffffffdu;
constexpr uint32_t kInvalidKey = 0xffffffffu;

// G-buffer flags (per path)
enum : uint32_t {
  kGHit = 1u << 29,
  kGEmit = 1u << 30,        // primary hit on the emitting side (render.cpp:79-81)
  kGReflective = 1u << 31,  // NEE vertex (render.cpp:84)
  kGMatMask = (1u << 29) - 1,
};
// Sample-record flags
// kSRay: rays[idx] valid; kSRecord: the sample carries an update_q record
enum : uint32_t { kSNonzero = 1u, kSLearned = 2u, kSRay = 4u, kSRecord = 8u, kSFrozen = 16u };
// kSFrozen (pdf_mode frozen_cdf): srec.pin holds the whole selection pdf,
// (cdf[s] - cdf[s - 1]) / total * pin, instead of the live q_before's
// rflag bit set by k_shadow for an occluded segment (srec keeps the visible
// contribution; its v is zeroed in vdense): a byte in a 2 MB array instead of
// a read-modify-write of the 64-byte sample record
constexpr uint8_t kROccluded = 0x80;

// Device error bits (mapped to the reference's exceptions by the host).
enum : uint32_t {
  kErrNonUnitNormal = 1u,     // make_key, hash_grid.cpp:78-80
  kErrBadValue = 2u,          // update_q, cut.cpp:78-80
  kErrDegenerateLight = 4u,   // sample_triangle_point, scene.cpp:50-51
  kErrBadAreaPdf = 8u,        // level_for_footprint, hash_grid.cpp:35-37
  kErrStackOverflow = 16u,    // BVH deeper than the traversal stack
  kErrNewKeyOverflow = 32u,   // more distinct new keys in one pass than the dedup table holds
  kErrCheck = 64u,            // a device bounds check failed (RLC_DEBUG_CHECKS builds)
};

// Counters block (u64 each).
enum : uint32_t { kCntCells = 0, kCntLookups = 1, kCntFallback = 2, kCntChanges = 3,
                  kCntErr = 4, kCntPending = 5, kCntNewKeys = 6, kCntNum = 8 };

struct alignas(16) GBuf {  // 64 B per path vertex
  double pos[3];
  double ns[3];
  uint64_t rng;
  uint32_t cell;   // dense cell id of the vertex's lookup, or kPending / kFallback / kNoSlot
  uint32_t flags;
};

struct alignas(16) SampleRec {  // 64 B per path
  double c[3];      // contribution (estimators.cpp:100-101)
  double pdf_area;
  double pin;       // learned: pdf_in_cluster; baselines: pdf_light_selection
  double total;     // learned: frozen cdf total of the cell cut
  double v;         // feedback value
  uint32_t s;       // cluster index
  uint32_t flags;
};

// One shadow segment of nee_estimate (estimators.cpp:95 -> bvh.cpp:159-188),
// queued by k_sample and traced by k_shadow.  64 B.
struct alignas(16) ShadowRay {
  double o[3];
  double d[3];
  double tmax;  // len - shadow_eps
  uint32_t idx; // path index
  uint32_t pad;
};

// One update_q record as exchanged between ranks (32 B): the cell named by
// its table slot -- the tables are identical on every rank, slot for slot --
// or kPending with the packed CellKey for a key new this pass.
struct alignas(16) ExchangeRecord {
  uint32_t slot;     // table slot, or kPending (key in klo/khi)
  uint32_t cluster;
  double v;
  unsigned long long klo, khi;  // packed CellKey (pending records only)
};

struct DevScene {
  const BvhNode* nodes;
  const BvhNodeF* nodes_f;  // fp32 outward-rounded copy for the decision tests
  const BvhNodeF* nodes_cam; // camera-relative fp32 copy (primary rays)
  const Wide4* wide;        // conservative 4-wide tree (null if the root is a leaf)
  const WideQ* wide_q;      // the same tree quantized (null: k_shadow reads `wide`)
  const Wide4* wide_ref;    // reference tree collapsed in its leaf order (closest hit)
  const Wide4* wide_cam;    // same, camera-relative boxes (primary rays)
  const uint32_t* tri_leaf; // binary leaf per leaf-order triangle
  const TriAccel* tris_s;   // triangles in the shadow tree's leaf order
  const uint32_t* tri_leaf_s; // reference leaf per tris_s entry
  const TriAccel* tris;
  const MatRec* mats;
  const uint32_t* tri_mat;
  const double* tri_normal;
  const LightRec* lights;
  const LightOrd* lights_ord;  // emitters in light-tree order (order[] folded in)
  const uint32_t* emitter_mat; // material id per emitter (emission of lights_ord)
  const uint32_t* order;
  const LtNode* lt;
  const double* energy_cdf;
  const double* emitter_energy;
  uint32_t num_lights;
  uint32_t num_tris;
  uint32_t fp32_ok;  // scene coordinates within 1e8: the fp32 shadow pre-test is valid
  uint32_t nodes_root_leaf;  // the reference BVH is a single leaf (no wide trees apply)
  uint32_t shadow_stack_limit;  // test knob RLC_SHADOW_STACK_LIMIT: a smaller k_shadow stack (0: full)
  uint32_t libm_fma; // host libm build whose sin/cos the bounce sampler restates (rlc_libm.h)
  uint32_t count_work;  // k_shadow's counting instance (rlc_context_count_work)
  double shadow_eps;
  double coord_bound;  // S: k_shadow's lean test holds for ray origins within S
  double base_tile;
  double level_thr[17];
  CameraConst cam;
};

struct DevGrid {
  unsigned long long* slot_keys;  // [capacity][2] packed CellKey (0 = empty)
  uint32_t* slot_cell;            // [capacity]
  uint32_t capacity;
  uint32_t probe_limit;
  uint32_t normal_bits;
  uint32_t M;                     // cut size (cluster count)
  double jitter_scale;
  // per-cell cut rows [cell][M]
  uint32_t* node_ids;
  uint32_t* ends;
  double* q;
  double* cdf;
  uint32_t* visits;
  uint32_t* cell_key;             // [cell][5]
  uint32_t* cell_slot;            // [cell] its table slot
  uint32_t* touched;              // [cell]
  // template cut == fallback cut [M]
  const uint32_t* t_node;
  const uint32_t* t_ends;
  const double* t_q;
  const double* t_cdf;
  const uint32_t* t_visits;
  double eps_q;
  unsigned long long* counters;   // kCnt*
  // insertion claims [capacity]: (canonical id << 32 | new-key index) of the
  // pending key holding an empty slot during k_insert; ~0 = none
  unsigned long long* claim;
  unsigned char* split_scratch;   // k_split rows in global memory for cuts too large
                                  // for shared memory (kSplitGlobalWarps * 32 M bytes)
};

struct PassParams {
  uint32_t width;
  uint32_t row_begin;
  uint32_t spp_pp;
  uint32_t pass_index;
  uint32_t n;           // paths in this launch: rows * width * spp_pp
  uint32_t depth;       // max_depth D: path vertices per path
  uint32_t nv;          // vertices n * D; vertex (path, d) is path * D + d - 1
  uint32_t sampler;
  uint64_t seed_mixed;  // mix64(seed)
  uint64_t zero_mixed;  // mix64(0): the c component of the RNG key
  double alpha;
  uint32_t harmonic;
  const uint32_t* pass_dev;  // non-null (CUDA-graph replays): the pass index is read here
  uint32_t defer_insert;     // sharded trace: new keys are inserted by the fold of all ranks
  uint32_t export_samples;   // k_sample files each vertex's emitter index (rlc_pass_samples)
  uint32_t frozen_pdf;       // radiance with the pass-frozen cdf's pdf (non-parity, unbiased)
};

// The distinct keys missing from the table in one pass, each with the
// smallest canonical id that looked it up (the reference's insertion order,
// hash_grid.cpp:113-141): an open-addressing table of 2^k entries, cleared
// entry by entry by k_commit after use.
struct NewKeys {
  unsigned long long* keys;  // [cap][2] packed CellKey, 0 = empty
  uint32_t* id;              // [cap] smallest canonical id, ~0 = empty
  uint32_t* list;            // [cap] entry index of the d-th distinct key
  unsigned int* count;       // distinct keys this pass
  uint32_t mask;             // cap - 1
};

struct PassBuffers {
  GBuf* gbuf;
  unsigned long long* pkey;  // [vertex][2] packed key of a kPending lookup (per G-buffer slot)
  NewKeys nk;
  uint32_t* emit;            // [vertex] emitter index (P.export_samples)
  SampleRec* srec;
  double* vdense;        // [vertex] srec's v, dense: the fold's gathers stay in L2
  uint32_t* gflags;      // [vertex] the G-buffer flags, dense (k_accumulate; per slot)
  uint8_t* rflag;        // per vertex: srec's kSNonzero | kSLearned | kSRay | kSRecord bits (compaction
                         // input), kROccluded; per slot
  uint32_t* keys;
  uint32_t* vals;
  uint32_t* keys_alt;
  uint32_t* vals_alt;
  double* q_before;
  ShadowRay* rays;
  unsigned int* ray_count;  // [0] queued rays, [1] fetch cursor
  uint32_t* ray_order;      // path indices with a shadow ray, in trace order
  uint32_t* rec_path;       // path index of each update record (canonical order)
  unsigned int* rec_count;  // [0] update records of the pass
  uint32_t* block_counts;   // compaction scratch
  uint32_t* block_counts2;  // compaction scratch of the record sort (side stream)
  unsigned int* sort_count; // update records of the pass (the record sort's device count)
  uint32_t* sort_hist;
  uint32_t sort_hist_cap;  // entries
};

// A rank's update records of one sharded pass, as all-gathered: cap + 1
// slots of 32 B, slot 0 the header (the record count), record k in slot
// k + 1.  Every rank's block has the same size, so the gather needs no count
// on the host, and the gathered blocks are one array of exchange slots
// t = rank * (cap + 1) + 1 + k in canonical order.
struct alignas(16) RecordBlockHeader {
  unsigned long long count;
  unsigned long long pad[3];
};
static_assert(sizeof(RecordBlockHeader) == sizeof(ExchangeRecord), "block slot size");

// Buffers of the sharded fold, for nranks * (cap + 1) exchange slots.
struct ExchangeBuffers {
  const ExchangeRecord* rec;  // [t] the gathered blocks (header slots included)
  uint32_t* cellx;       // [t] the record's dense cell id (kFallback: refused key)
  uint8_t* kflag;        // [t] kXValid | kXFallback | kXOwned | kXSort | kXPending
  uint32_t* keys;        // [t] sort key (cell * M + cluster) of the records this rank folds
  uint32_t* keys_alt;
  uint32_t* vals;
  uint32_t* vals_alt;
  uint32_t* hist;
  uint32_t* block_counts;
  unsigned int* sort_count;
  double* q_rec;         // [t] q_before of record t (the all-reduced array in owner mode)
  uint32_t* seg_n;       // [t] records of the cut entry at its last record t, else 0 (owner mode)
  double* ent_q;         // [slot * M + cluster] the owner's final q (owner mode, entry exchange)
  uint32_t* ent_n;       // [slot * M + cluster] its record count (zero: not folded this pass)
  uint64_t entries;      // capacity * M
  uint32_t entry_mode;   // owner mode exchanges per-entry finals instead of per-slot counts
  uint32_t* pend;        // slots of the records whose key was new at trace time
  unsigned int* pend_count;
  NewKeys nk;
  uint32_t stride;       // exchange slots per rank block (cap + 1)
  uint32_t nranks;
};
enum : uint8_t { kXValid = 1, kXFallback = 2, kXOwned = 4, kXSort = 8, kXPending = 16 };

// == rlc_sample_record (include/rlcuts_b200.h)
struct alignas(8) SampleExport {
  uint32_t vertex, cluster, emitter, flags;
  double q_before, v, total;
  double radiance[3];
};

struct Framebuf {
  double* sum;                // [h*w*3]
  unsigned long long* count;  // [h*w]
  uint32_t width;
};

// Each launcher adds its kernel launches to a process-wide counter.
uint64_t launches();
void add_launches(uint64_t k);
// End of pass `offset` of a graph replay: hist[*pass_dev + offset] = *changes
// (hist may be null), *changes = 0.
void launch_end_pass(const uint32_t* pass_dev, uint32_t offset, uint32_t* changes, uint32_t* hist,
                     cudaStream_t st);
void launch_set_u32(uint32_t* p, uint32_t v, cudaStream_t st);  // *p = v
void launch_add_u32(uint32_t* p, uint32_t v, cudaStream_t st);  // *p += v
void trav_stats(uint64_t out[8], bool reset);
void work_counters(uint64_t out[4], bool reset);  // k_shadow rays, node steps, triangle tests
// Measured L2 read bandwidth (GB/s) over an L2-resident buffer of `bytes`.
double measure_l2_gbs(size_t bytes, uint32_t reps);

void launch_primary(const DevScene& sc, const DevGrid& g, const PassParams& p,
                    const PassBuffers& b, cudaStream_t st);
// Bounce to vertex `depth` (2..D) of every path: cosine-hemisphere
// direction, closest hit, cell lookup (render.cpp:127-135 then 71-99).
void launch_bounce(const DevScene& sc, const DevGrid& g, const PassParams& p, uint32_t depth,
                   const PassBuffers& b, cudaStream_t st);
void launch_sample(const DevScene& sc, const DevGrid& g, const PassParams& p,
                   const PassBuffers& b, cudaStream_t st);
// The pass's new keys into the table in canonical order (k_insert), then
// published with fresh cells holding the template cut (k_commit).
void launch_insert_new_keys(const DevGrid& g, const NewKeys& nk, cudaStream_t st);
// Sorts (keys, vals) by key; returns which buffer pair holds the result.
// Stable compaction of the paths that carry a shadow ray, in the order of
// `order` (sorted update records) or canonical order when it is null.
void launch_ray_compact(const PassBuffers& b, const uint32_t* order, uint32_t n, cudaStream_t st);
// leave_room: one block slot per SM stays free for concurrent work (the sort).
void launch_shadow(const DevScene& sc, const PassBuffers& b, const uint32_t* order,
                   unsigned long long* counters, cudaStream_t st, bool leave_room = false);
void launch_sort(PassBuffers& b, uint32_t n, uint32_t key_bits, cudaStream_t st,
                 uint32_t** keys_out, uint32_t** vals_out);
// Keys per block of the record sort (its per-block digit histograms hold
// 256 x ceil(n / kSortTile) counters).
#ifndef RLC_SORT_TILE
#define RLC_SORT_TILE 4096
#endif
constexpr uint32_t kSortTile = RLC_SORT_TILE;
// Keys per block of the sharded fold's sort (a rank folds a fraction of the
// gathered records, so smaller tiles keep the SMs busy).
constexpr uint32_t kSortTileSmall = 1024;
// n_dev (may be null): a device-side count <= n of the valid entries; the
// digit passes then cover ceil(*n_dev / tile) tiles only.  small_tiles:
// kSortTileSmall keys per block instead of kSortTile.  identity_vals: va is
// not read, the values start as 0 .. n - 1.
void launch_sort_buffers(uint32_t* ka, uint32_t* va, uint32_t* kb, uint32_t* vb, uint32_t* hist,
                         uint32_t n, uint32_t key_bits, cudaStream_t st, uint32_t** keys_out,
                         uint32_t** vals_out, const unsigned* n_dev, bool small_tiles = false,
                         bool identity_vals = false);
// Sharded passes.  The rank's update records of the
// traced band, in canonical order, into `block` (header slot + cap slots).
void launch_export_block(const DevGrid& g, const PassBuffers& b, uint32_t n, void* block,
                         uint32_t cap, cudaStream_t st);
// The same records stored straight into `ndst` (<= kMaxPeers) gathered
// buffers at block `rank` -- peers' receive buffers over NVLink (CUDA IPC) or,
// for emulated ranks, buffers on this device: only the records that exist
// cross, then one barrier collective orders them before the fold.
constexpr uint32_t kMaxPeers = 16;
struct PeerDsts {
  ExchangeRecord* p[kMaxPeers];
};
void launch_export_block_to(const DevGrid& g, const PassBuffers& b, uint32_t n,
                            const PeerDsts& dst, uint32_t ndst, uint32_t rank, uint32_t cap,
                            cudaStream_t st);
// The fold of all ranks' gathered blocks (x.rec: nranks x x.stride slots,
// valid until the pass's launch_shard_scatter): the pass's new keys inserted
// in canonical order (identical tables on every rank), then each record's
// cell and owner -- this rank for every record (owner_fold = 0), else the
// rank slot % nranks of its table slot.
void launch_shard_fold(const DevGrid& g, const PassParams& fold_params, uint32_t rank,
                       bool owner_fold, ExchangeBuffers& x, cudaStream_t st);
// update_q for the records this rank folds, per cut entry in canonical
// order: q_before per record slot into x.q_rec and, in owner mode, the
// entry's record count at its last record into x.seg_n (zero elsewhere).
void launch_shard_sortfold(const DevGrid& g, const PassParams& fold_params, uint32_t key_bits,
                           bool owner_fold, ExchangeBuffers& x, cudaStream_t st);
// Owner mode, after x.q_rec and x.seg_n were summed over the ranks: the cut
// entries other ranks folded, advanced to the state their last record leaves
// (q from its q_before and v, visits by the record count), touched flags.
// Entry exchange (x.entry_mode): the entries other ranks folded take the
// summed final q and record counts of x.ent_q / x.ent_n instead.
void launch_shard_apply(const DevGrid& g, const PassParams& fold_params, uint32_t rank,
                        ExchangeBuffers& x, cudaStream_t st);
// q_before of this rank's own records (fallback: the template's) for the
// accumulation of its band.
void launch_shard_scatter(const DevGrid& g, const PassBuffers& b, uint32_t n, uint32_t rank,
                          const ExchangeBuffers& x, cudaStream_t st);
void launch_fold(const DevGrid& g, const PassParams& p, const uint32_t* keys,
                 const uint32_t* vals, const PassBuffers& b, cudaStream_t st);
void launch_accumulate(const DevScene& sc, const PassParams& p, const PassBuffers& b,
                       const Framebuf& fb, cudaStream_t st);
// Cut sizes whose k_split rows (32 M bytes per warp) exceed this stage in
// global memory (DevGrid::split_scratch, kSplitGlobalWarps warps).
constexpr size_t kSplitSmemMax = 200 * 1024;
constexpr uint32_t kSplitGlobalWarps = 148 * 8;
void launch_split_collapse(const DevScene& sc, const DevGrid& g, double threshold,
                           uint32_t iterations, uint32_t* changes_out, cudaStream_t st);
void launch_occluded_batch(const DevScene& sc, uint32_t n, const double* a, const double* b,
                           PassBuffers& pb, unsigned long long* counters, uint8_t* out,
                           cudaStream_t st);
void launch_intersect_batch(const DevScene& sc, uint32_t n, const double* org, const double* dir,
                            double tmin, double* t_out, int32_t* tri_out,
                            unsigned long long* counters, cudaStream_t st, bool sah_only = false);
void launch_resolve(const Framebuf& fb, uint32_t npix, double* image, cudaStream_t st);
// Dynamic updates: the creation shadow tree refitted on the device to the
// moved triangles.  Topology arrays are the creation's.
struct RefitTopo {
  const uint32_t* bin_a;       // [bin node] leaf: first tris_s position; internal: left child
  const uint32_t* bin_b;       // internal: right child
  const uint32_t* bin_count;   // leaf: triangles (> 0); internal: 0
  const uint32_t* bin_parent;  // parent bin node (0xffffffff: the root)
  const uint32_t* bin_leaves;  // the leaf bin nodes
  uint32_t num_bin, num_leaves;
  const uint32_t* kids;        // [wide node][4] bin node of each child, or kWideEmpty
  const uint32_t* base_child;  // [wide node][4] the creation's child words
  uint32_t num_wide;
  const uint32_t* tri_ids;     // [tris_s position] triangle id (creation order)
  uint32_t num_tris;
  double* box;                 // [bin node][6] scratch
  unsigned int* arrive;        // [bin node] scratch (zeroed by the launcher)
};
void launch_refit_shadow(const RefitTopo& t, const double* vertices, const uint32_t* leaf_of_id,
                         double pad, TriAccel* tris_s, uint32_t* tri_leaf_s, Wide4* wide,
                         WideQ* wide_q, unsigned int* err, cudaStream_t st);
// sc.lights_ord from sc.lights, sc.order and sc.emitter_mat.
void launch_light_order(const DevScene& sc, LightOrd* out, cudaStream_t st);
// Per-vertex parity records of the pass in `p` (rlc_pass_samples).
void launch_export_samples(const PassParams& p, const PassBuffers& b, SampleExport* out,
                           cudaStream_t st);
// Per-pixel squared error of the resolved framebuffer against `ref`
// (mse's summand, image.cpp:119-121), for the ordered host sum.
void launch_pixel_err(const Framebuf& fb, uint32_t npix, const double* ref, double* err,
                      cudaStream_t st);
// Device sin/cos of the bounce sampler (rlc_libm.h) for the parity tests.
void launch_libm_sincos(const DevScene& sc, uint32_t n, const double* x, double* s, double* c,
                        cudaStream_t st);

}  // namespace rlc
