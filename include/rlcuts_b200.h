/*
 * rlcuts_b200.h -- C-ABI drop-in boundary of the B200-native RL-lightcuts
 * direct-lighting path.
 *
 * The reference (`/root/reference/proj`, CPU C++20 `rlcuts`) exposes the
 * per-frame direct-lighting step as C++ functions in proj/include/rlcuts/.
 * Every entry point below replaces one of them; the citation on each line is
 * the reference interface it stands in for.  Plain pointers and sizes only:
 * no C++ or torch types cross this boundary.
 *
 * Error convention: every call returns an rlc_status.  The reference throws
 * C++ exceptions; RLC_ERR_INVALID_ARGUMENT stands for std::invalid_argument
 * and RLC_ERR_OUT_OF_RANGE for std::out_of_range (e.g.
 * proj/src/render.cpp:161-166, proj/src/cut.cpp:77-80).  rlc_last_error()
 * returns the thread-local message of the last failing call.
 *
 * Threading: calls are synchronous with respect to the host unless noted
 * (the reference fans out and joins std::threads inside each call,
 * proj/src/render.cpp:23-38).  Device work is issued on the context stream
 * (rlc_context_set_stream), and a call returns after that stream drained,
 * except rlc_render_pass_async / rlc_end_of_pass_update_async.
 *
 * There is no CPU fallback: on a host without a usable sm_100 device every
 * create call fails with RLC_ERR_NO_DEVICE.
 */
#ifndef RLCUTS_B200_H
#define RLCUTS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RLC_ABI_VERSION 1

typedef enum rlc_status {
  RLC_OK = 0,
  RLC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  RLC_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range in the reference */
  RLC_ERR_CUDA = 3,             /* CUDA runtime / kernel failure */
  RLC_ERR_NO_DEVICE = 4,        /* no sm_100 device: there is no CPU fallback */
  RLC_ERR_INTERNAL = 5,
  RLC_ERR_IO = 6,               /* ImageIoError io_error (image.hpp:15-28) */
  RLC_ERR_PARSE = 7             /* ImageIoError parse_error */
} rlc_status;

/* proj/include/rlcuts/estimators.hpp:16-20 (SamplerKind) */
enum { RLC_SAMPLER_UNIFORM = 0, RLC_SAMPLER_ENERGY = 1, RLC_SAMPLER_RL_LIGHTCUTS = 2 };
/* proj/include/rlcuts/cut.hpp:16-19 (AlphaSchedule) */
enum { RLC_ALPHA_FIXED = 0, RLC_ALPHA_HARMONIC = 1 };

/* proj/include/rlcuts/cut.hpp:21-28 (CutConfig) */
typedef struct rlc_cut_config {
  uint32_t cut_size;       /* M; clamped to the light count */
  uint32_t iterations;     /* split-collapse repeats per pass */
  double alpha;            /* learning rate in (0,1] */
  double split_threshold;  /* T */
  double eps_q;            /* < 0 resolves to 1e-4 / M */
  uint32_t alpha_schedule; /* RLC_ALPHA_* */
  uint32_t _pad;
} rlc_cut_config;

/* proj/include/rlcuts/hash_grid.hpp:17-23 (HashConfig) */
typedef struct rlc_hash_config {
  uint32_t capacity;
  uint32_t probe_limit;
  uint32_t normal_bits;
  uint32_t _pad;
  double base_tile;    /* <= 0: derive from scene (diag / 256) */
  double jitter_scale; /* 0 keeps key derivation a pure function */
} rlc_hash_config;

/* proj/include/rlcuts/render.hpp:17-26 (RenderConfig) */
typedef struct rlc_render_config {
  uint32_t spp;
  uint32_t passes;
  uint32_t max_depth;
  uint32_t sampler; /* RLC_SAMPLER_* */
  rlc_cut_config cut;
  rlc_hash_config hash;
  uint64_t seed;
  uint32_t workers; /* accepted for interface parity; the device ignores it */
  uint32_t _pad;
} rlc_render_config;

/* proj/include/rlcuts/scene.hpp:13-67 (Material, Triangle, Camera, Scene),
 * flattened: vertices[t*9 + v*3 + axis] = triangles[t].p{v}[axis],
 * materials[m*6 + 0..2] = albedo, materials[m*6 + 3..5] = emission. */
typedef struct rlc_scene_desc {
  uint32_t num_triangles;
  uint32_t num_materials;
  const double* vertices;
  const uint32_t* material_ids;
  const double* materials;
  double cam_origin[3];
  double cam_look_at[3];
  double cam_up[3];
  double vfov_degrees;
  int32_t width;
  int32_t height;
} rlc_scene_desc;

/* proj/include/rlcuts/hash_grid.hpp:26-34 (CellKey) */
typedef struct rlc_cell_key {
  int32_t qx, qy, qz;
  uint32_t qn;
  uint32_t level;
} rlc_cell_key;

/* proj/include/rlcuts/render.hpp:56-64 (RenderResult, minus the image) */
typedef struct rlc_render_result {
  double wall_ms;
  uint32_t occupied_cells;
  uint32_t num_passes;
  uint64_t lookups;
  uint64_t fallback_hits;
  uint32_t* sc_changes; /* optional caller array [passes] */
} rlc_render_result;

/* proj/include/rlcuts/hash_grid.hpp:101-103 (occupied_count, lookup_count,
 * fallback_hits) */
typedef struct rlc_grid_stats {
  uint32_t occupied;
  uint32_t cut_size;
  uint64_t lookups;
  uint64_t fallback_hits;
  /* lookups whose key was not in the table when their pass began, and the
   * distinct such keys (each inserted, or refused by a full probe window,
   * in canonical order after the pass's lookups) */
  uint64_t pending_lookups;
  uint64_t new_keys;
} rlc_grid_stats;

typedef struct rlc_context_info {
  uint32_t num_triangles;
  uint32_t num_emitters;
  uint32_t bvh_nodes;
  uint32_t light_tree_nodes;
  double base_tile;  /* resolved, proj/src/render.cpp:153-155 */
  double shadow_eps; /* proj/src/bvh.cpp:120 */
  uint64_t device_bytes;
} rlc_context_info;

typedef struct rlc_context rlc_context;         /* RenderContext, render.hpp:28-37 */
typedef struct rlc_grid rlc_grid;               /* HashGrid, hash_grid.hpp:80-133 */
typedef struct rlc_framebuffer rlc_framebuffer; /* Framebuffer, image.hpp:47-63 */

/* ---- library ---------------------------------------------------------- */
const char* rlc_last_error(void);
int rlc_abi_version(void);
/* Number of kernel launches this process issued so far (bench evidence). */
uint64_t rlc_kernel_launches(void);
/* Reference defaults: render.hpp:17-26, cut.hpp:21-28, hash_grid.hpp:17-23 */
rlc_status rlc_render_config_default(rlc_render_config* config);

/* ---- context: build_context (proj/src/render.cpp:143-157) ------------- */
rlc_status rlc_context_create(const rlc_scene_desc* scene, const rlc_render_config* config,
                              int device, rlc_context** out);
rlc_status rlc_context_destroy(rlc_context* ctx);
/* Dynamic emitters (the reference has no such call):
 * after this call the context renders `scene` exactly as
 *     ctx' = build_context(scene, creation config); ctx'.tree = ctx.tree;
 * would (render.cpp:143-157) -- a fresh scene BVH, emitter records and
 * energy cdf, but the light tree of the context's creation (emitter order,
 * topology and node energies), so the learned cuts of every hash grid of
 * this context stay valid across frames.  Vertices and the camera pose may
 * change; the triangle count, material ids, materials and the camera
 * resolution must not (RLC_ERR_INVALID_ARGUMENT).  Synchronizes. */
rlc_status rlc_context_update_scene(rlc_context* ctx, const rlc_scene_desc* scene);
/* rlc_context_update_scene in two steps, so the host builds of later frames
 * overlap this frame's GPU work and each other: prepare copies the scene's
 * vertices and starts its host build on a worker thread (at most 8 in
 * flight), *token identifies it; commit waits for that build, uploads it
 * and makes it the context's scene (synchronizes).  Tokens are committed in
 * any order; update_scene = prepare + commit. */
rlc_status rlc_context_prepare_scene(rlc_context* ctx, const rlc_scene_desc* scene,
                                     uint64_t* token);
rlc_status rlc_context_commit_scene(rlc_context* ctx, uint64_t token);
rlc_status rlc_context_info_get(const rlc_context* ctx, rlc_context_info* info);
/* Issue device work on `stream` (a cudaStream_t); NULL = the context's own. */
rlc_status rlc_context_set_stream(rlc_context* ctx, void* stream);
rlc_status rlc_context_synchronize(rlc_context* ctx);

/* Per-stage device timing with CUDA events on the context stream (bench
 * evidence).  Stages: 0 primary, 1 sample, 2 sort, 3 fold, 4 accumulate,
 * 5 split-collapse, 6 shadow (any-hit traversal), 7 insert (the pass's new
 * hash-grid keys, in canonical order), 8 ray compaction, 9 the sharded fold's
 * gather of all ranks' records and key insertion (stage 3 of a sharded pass:
 * its sort and update_q).  Stage 0 includes the
 * bounce rays of max_depth > 1.  rlc_context_stage_times synchronizes,
 * returns accumulated milliseconds and launch counts per stage since the
 * last call, and resets them. */
#define RLC_NUM_STAGES 10
rlc_status rlc_context_enable_timing(rlc_context* ctx, int enable);
rlc_status rlc_context_stage_times(rlc_context* ctx, double* ms, uint32_t* counts);
/* The timeline behind rlc_context_stage_times (call it first): per stage
 * launch, out[3i..3i+2] = stage, start, end in ms from the first mark, on
 * the stream the stage ran on (the overlap of the streams made visible).
 * *n_out = marks recorded; synchronizes.  Marks are kept until the next
 * rlc_context_stage_times. */
rlc_status rlc_context_stage_marks(rlc_context* ctx, uint32_t max_marks, double* out,
                                   uint32_t* n_out);

/* ---- scene visibility, batched ---------------------------------------- */
/* occluded (proj/include/rlcuts/bvh.hpp:38-40, proj/src/bvh.cpp:159-188):
 * a, b [n*3] host arrays, out [n] = 1 iff the open segment is blocked. */
rlc_status rlc_occluded_batch(const rlc_context* ctx, uint32_t n, const double* a,
                              const double* b, uint8_t* out);
/* intersect (bvh.hpp:35-36, bvh.cpp:124-157): closest hit with
 * t in (t_min, inf); t_out = -1 and tri_out = -1 on a miss. */
rlc_status rlc_intersect_batch(const rlc_context* ctx, uint32_t n, const double* origins,
                               const double* dirs, double t_min, double* t_out,
                               int32_t* tri_out);
/* Diagnostic: traversal counters of a build with -DRLC_TRAV_STATS (zeros
 * otherwise): out8[0..2] shadow rays / node steps / triangle tests of
 * k_shadow, out8[3..5] rays / node steps / triangle tests of the SAH closest
 * hit, out8[6] shadow rays finished on the exact path after a stack
 * overflow.  reset != 0 clears them after reading. */
rlc_status rlc_debug_trav_stats(int32_t reset, uint64_t* out8);
/* Work counters (the bench's own-work roofline bytes), kept while a
 * context counts (rlc_context_count_work: k_shadow's counting instance,
 * ~1.5% slower on c3): out4[0..2] = shadow rays traversed by k_shadow's tree, its node steps
 * (64-byte nodes) and triangle tests (80-byte triangles), out4[3] = shadow
 * rays queued, summed over the process since the last reset.  reset != 0
 * clears them. */
rlc_status rlc_work_counters(int32_t reset, uint64_t* out4);
rlc_status rlc_context_count_work(rlc_context* ctx, int enable);
/* Diagnostic, host only (no device needed): the reference scene BVH build
 * (build_scene_bvh, bvh.cpp:64-122) of `scene`, `reps` times; *ms_out =
 * mean milliseconds, *nodes_out = node count (may be NULL). */
rlc_status rlc_debug_host_bvh(const rlc_scene_desc* scene, uint32_t reps, double* ms_out,
                              uint32_t* nodes_out);
/* Measured L2 read bandwidth of `device` in GB/s (16-byte L2 loads over a
 * 48 MB L2-resident buffer): the bench's second roofline denominator. */
rlc_status rlc_measure_l2_bandwidth(int device, double* gbs);
/* Diagnostic (parity tests): the closest-hit decision of the SAH tree alone
 * (DESIGN.md 5.4): as rlc_intersect_batch, but tri_out = -2 where the SAH
 * traversal defers to the reference-order traversal (exact tie, or the hit's
 * reference leaf fails the exact slab test, or a ray outside its bounds). */
rlc_status rlc_intersect_batch_sah(const rlc_context* ctx, uint32_t n, const double* origins,
                                   const double* dirs, double t_min, double* t_out,
                                   int32_t* tri_out);

/* ---- bounce sampler trigonometry ---------------------------------------
 * sample_cosine_hemisphere (proj/include/rlcuts/math.hpp:101-107) calls
 * std::cos / std::sin, which glibc does not round correctly; the device
 * restates the host libm's build exactly (paper_1911_10217_b200/csrc/
 * rlc_libm.h).  rlc_libm_variant: 1 = glibc FMA build, 0 = SSE2 build,
 * -1 = unrecognised (max_depth > 1 then fails with RLC_ERR_INTERNAL).
 * rlc_libm_sincos runs the device restatement on host arrays (parity tests);
 * rlc_libm_sincos_host runs the same code on the host (no device needed). */
rlc_status rlc_libm_variant(int32_t* variant);
rlc_status rlc_libm_sincos(const rlc_context* ctx, uint32_t n, const double* x, double* s,
                           double* c);
rlc_status rlc_libm_sincos_host(int32_t variant, uint64_t n, const double* x, double* s,
                                double* c);

/* ---- hash grid: HashGrid(hash, init_cut(tree, M, eps))
 *      (proj/src/render.cpp:211-216, proj/src/hash_grid.cpp:102-111,
 *       proj/src/cut.cpp:27-74) --------------------------------------- */
rlc_status rlc_grid_create(const rlc_context* ctx, const rlc_render_config* config,
                           rlc_grid** out);
rlc_status rlc_grid_destroy(rlc_grid* grid);
rlc_status rlc_grid_stats_get(const rlc_grid* grid, rlc_grid_stats* stats);
/* Parity export keyed by CellKey (slot ids are insertion-order dependent,
 * SURVEY 0 fact 9).  Arrays are [max_cells] / [max_cells * cut_size]; any
 * pointer may be NULL.  *num_cells receives the occupied count. */
/* HashGrid's slot view (hash_grid.hpp:87-110: key_of, touched_slots,
 * dump_stats, memory_records are built on it by the mirrors): the occupied
 * slots in slot order with their dense cell, CellKey and touched flag (set by
 * render_pass, cleared by end_of_pass_update).  *count_out = occupied slots;
 * at most max_slots entries are written, every output array optional. */
rlc_status rlc_grid_slots(const rlc_grid* grid, uint32_t max_slots, uint32_t* slot_out,
                          uint32_t* cell_out, rlc_cell_key* key_out, uint8_t* touched_out,
                          uint32_t* count_out);
rlc_status rlc_grid_export(const rlc_grid* grid, uint32_t max_cells, rlc_cell_key* keys,
                           uint32_t* node_ids, uint32_t* ends, double* q, double* cdf,
                           uint32_t* visits, uint32_t* num_cells);
/* The template cut every new cell starts from (init_cut, cut.cpp:27-74). */
rlc_status rlc_grid_template(const rlc_grid* grid, uint32_t* node_ids, uint32_t* ends,
                             double* q, double* cdf, uint32_t* visits, double* eps_q);

/* ---- framebuffer: Framebuffer (proj/include/rlcuts/image.hpp:47-63) ---- */
rlc_status rlc_framebuffer_create(const rlc_context* ctx, int32_t width, int32_t height,
                                  rlc_framebuffer** out);
rlc_status rlc_framebuffer_destroy(rlc_framebuffer* fb);
rlc_status rlc_framebuffer_clear(rlc_framebuffer* fb);
/* sum: [h*w*3] doubles, count: [h*w]; either may be NULL. */
rlc_status rlc_framebuffer_download(const rlc_framebuffer* fb, double* sum, uint64_t* count);
/* Framebuffer::resolve (proj/src/image.cpp:35-41): image [h*w*3]. */
rlc_status rlc_framebuffer_resolve(const rlc_framebuffer* fb, double* image);

/* ---- per-frame step ---------------------------------------------------- */
/* render_pass (proj/src/render.cpp:159-183). */
rlc_status rlc_render_pass(const rlc_context* ctx, const rlc_render_config* config,
                           uint32_t pass_index, rlc_grid* grid, rlc_framebuffer* fb);
/* Same, restricted to image rows [row_begin, row_end) (screen-band sharding). */
rlc_status rlc_render_pass_rows(const rlc_context* ctx, const rlc_render_config* config,
                                uint32_t pass_index, rlc_grid* grid, rlc_framebuffer* fb,
                                uint32_t row_begin, uint32_t row_end);
/* end_of_pass_update (proj/src/render.cpp:185-200); *changes may be NULL. */
rlc_status rlc_end_of_pass_update(rlc_grid* grid, const rlc_context* ctx,
                                  const rlc_cut_config* cut, uint32_t* changes);
/* Asynchronous variants: enqueue on the context stream and return; the
 * change count stays on the device (read it with rlc_grid_last_changes). */
rlc_status rlc_render_pass_async(const rlc_context* ctx, const rlc_render_config* config,
                                 uint32_t pass_index, rlc_grid* grid, rlc_framebuffer* fb);
/* Passes [first_pass, first_pass + count) of render_frame's loop
 * (render.cpp:218-224): for each, render_pass and -- with the learned
 * sampler -- end_of_pass_update, enqueued without synchronizing (errors
 * surface at the next synchronizing call).  Launch-bound frames (at most 2^19
 * paths per pass) replay one captured CUDA graph per pass. */
rlc_status rlc_render_passes_async(const rlc_context* ctx, const rlc_render_config* config,
                                   uint32_t first_pass, uint32_t count, rlc_grid* grid,
                                   rlc_framebuffer* fb);
rlc_status rlc_end_of_pass_update_async(rlc_grid* grid, const rlc_context* ctx,
                                        const rlc_cut_config* cut);
rlc_status rlc_grid_last_changes(const rlc_grid* grid, uint32_t* changes);
/* ---- screen-band sharding: one learned update -----------------------------
 * One update_q call of render.cpp:111-117 -- the cell key, the cluster and
 * the feedback value, 32 B -- as the CPU model of the exchange
 * (oracle/restate.py, rlcuts.RECORD_DTYPE) files it.  The device blocks of
 * rlc_shard_trace carry the same update naming the cell by its table slot
 * (the tables are identical on every rank) and the key only for cells new
 * in the pass; their layout is the library's. */
typedef struct rlc_update_record {
  int32_t qx, qy, qz;
  uint32_t qn, level, cluster;
  double v;
} rlc_update_record;
/* ---- sharded frames (multi-GPU) -------------------
 * Rank `rank` of `nranks` renders rows [row_begin, row_end) of a pass; the
 * bands are consecutive in rank order.  The learned state stays identical
 * on every rank and equal to a single render_pass over all rows.  All calls
 * enqueue on the context stream and return without a host synchronization.
 *
 * 1. rlc_shard_trace: traces the band and files its update records in
 *    canonical order into a device block of *block_bytes = 32 (cap_records
 *    + 1) bytes (a 32-byte header slot with the count, then `cap_records`
 *    32-byte record slots; cap_records >= the band's path vertices, the
 *    same on every rank).
 * 2. the caller all-gathers the blocks of all ranks, rank-major (NCCL
 *    ncclAllGather of block_bytes, or any transport), into device memory
 *    that stays valid until rlc_shard_finish;
 * 3. rlc_shard_fold: inserts the pass's new keys in canonical order and
 *    folds, in canonical order per cut entry, the records of every cell
 *    (owner_fold = 0) or of the cells this rank owns (table slot % nranks
 *    == rank).  Per exchange slot (*slots of them, device arrays):
 *    *q_before_slots, the record's q_before, and *seg_counts, at the last
 *    record of each cut entry the entry's record count -- both zero for the
 *    records other ranks fold;
 * 4. owner_fold: the caller sums q_before_slots and seg_counts over the
 *    ranks (ncclAllReduce);
 * 5. rlc_shard_finish: advances the cut entries other ranks folded to the
 *    state their last record leaves (owner_fold) and accumulates the band's
 *    radiance;
 * 6. rlc_end_of_pass_update(_async): split-collapse, identical on every rank.
 * rlc_shard_frame does 1-6 with NCCL on the context stream (one call per
 * frame per rank, no host synchronization; errors surface at the next
 * synchronizing call, e.g. rlc_shard_sync). */
typedef struct rlc_comm rlc_comm;
rlc_status rlc_shard_trace(const rlc_context* ctx, const rlc_render_config* config,
                           uint32_t pass_index, rlc_grid* grid, uint32_t row_begin,
                           uint32_t row_end, uint64_t cap_records, void** block,
                           uint64_t* block_bytes);
/* rlc_shard_trace with the block stored straight into ndst (<= 16) gathered
 * buffers of nranks * block_bytes each, at block `rank` -- every rank's
 * receive buffer (peer memory over NVLink, or buffers of emulated ranks):
 * only the records that exist are written.  The caller orders the stores
 * before any rank's rlc_shard_fold (a barrier collective) and keeps a buffer
 * unwritten until its readers' rlc_shard_finish. */
rlc_status rlc_shard_trace_to(const rlc_context* ctx, const rlc_render_config* config,
                              uint32_t pass_index, rlc_grid* grid, uint32_t row_begin,
                              uint32_t row_end, uint64_t cap_records, uint32_t rank,
                              void* const* dst_buffers, uint32_t ndst);
rlc_status rlc_shard_fold(const rlc_context* ctx, const rlc_render_config* config, rlc_grid* grid,
                          const void* blocks, uint32_t nranks, uint32_t rank, int owner_fold,
                          double** q_before_slots, uint32_t** seg_counts, uint64_t* slots);
/* Owner mode's entry exchange, chosen by rlc_shard_fold when the records far
 * outnumber the cut entries (3 * capacity * M < 2 * slots; RLC_SHARD_ENTRY=0/1
 * forces it): *seg_counts is then null, and the caller instead sums these
 * per-entry arrays over the ranks -- each entry's final q and record count
 * from its owner, zero elsewhere -- while each rank needs only its own band's
 * block of q_before_slots summed (ncclReduceScatter).  Null / 0 in the
 * per-slot mode. */
rlc_status rlc_shard_entry_arrays(const rlc_context* ctx, double** entry_q,
                                  uint32_t** entry_counts, uint64_t* entries);
rlc_status rlc_shard_finish(const rlc_context* ctx, rlc_grid* grid, rlc_framebuffer* fb,
                            uint32_t rank, int owner_fold);
/* Waits for the context's work and reports device errors of the grid. */
rlc_status rlc_shard_sync(const rlc_context* ctx, rlc_grid* grid);
/* NCCL communicator of a rank (libnccl.so.2 loaded on first use): id128 is
 * ncclGetUniqueId's 128 bytes from rank 0, shared by the caller. */
rlc_status rlc_comm_unique_id(uint8_t* id128);
rlc_status rlc_comm_create(int device, uint32_t nranks, uint32_t rank, const uint8_t* id128,
                           rlc_comm** out);
rlc_status rlc_comm_destroy(rlc_comm* comm);
/* Collective (every rank calls it): rlc_shard_frame then moves the records
 * by peer memory instead of ncclAllGather -- each rank stores its band's
 * records straight into every rank's receive buffer (CUDA IPC handles over
 * NVLink; two halves by pass parity), then one int all-reduce is the
 * barrier.  cap_records as rlc_shard_frame's; enable = 0 returns to NCCL. */
rlc_status rlc_comm_enable_peer_exchange(rlc_comm* comm, uint64_t cap_records, int enable);
rlc_status rlc_shard_frame(const rlc_context* ctx, const rlc_render_config* config,
                           uint32_t pass_index, rlc_grid* grid, rlc_framebuffer* fb,
                           rlc_comm* comm, uint32_t row_begin, uint32_t row_end,
                           uint64_t cap_records, int owner_fold);
/* Frames first_pass .. first_pass + count - 1 of rlc_shard_frame.  use_graph:
 * after one direct frame (which sizes every buffer), a CUDA graph of two
 * frames -- kernels and NCCL collectives, the pass index read from device
 * memory -- is captured once and replayed; the results equal the direct
 * frames bit for bit. */
rlc_status rlc_shard_frames(const rlc_context* ctx, const rlc_render_config* config,
                            uint32_t first_pass, uint32_t count, rlc_grid* grid,
                            rlc_framebuffer* fb, rlc_comm* comm, uint32_t row_begin,
                            uint32_t row_end, uint64_t cap_records, int owner_fold,
                            int use_graph);

/* ---- per-sample parity export (SURVEY 8(b) "opt-in per-sample record
 * dump") ---------------------------------------------------------------
 * One record per path vertex of the context's last render_pass / sharded
 * pass (rows of that call, canonical order: pixel, sample, depth).  A vertex
 * that drew a light sample (sample_light, proj/src/estimators.cpp:28-80)
 * has RLC_SAMPLE_VALID; `emitter` is the selected emitter index (the
 * north star's bit-exact light selection), `cluster` the cut entry
 * (sample_cluster, proj/src/cut.cpp:97-106), `q_before` the live q the
 * reference's pdf reads (cut.cpp:105), `v` the update_q value
 * (estimators.cpp:103-104, 0 when occluded), `total` the frozen cdf total,
 * `radiance` nee_estimate's radiance (estimators.cpp:100-101).  Emitter
 * indices are filed only while rlc_context_enable_sample_export is on. */
enum {
  RLC_SAMPLE_VALID = 1,      /* a light sample was drawn at this vertex */
  RLC_SAMPLE_FALLBACK = 2,   /* the cell lookup fell back (hash_grid.cpp:140) */
  RLC_SAMPLE_RAY = 4,        /* a shadow segment was traced (bvh.cpp:159-188) */
  RLC_SAMPLE_NONZERO = 8,    /* unoccluded, front-facing: nonzero contribution */
  RLC_SAMPLE_LEARNED = 16,   /* drawn from a cut (rl_lightcuts) */
  RLC_SAMPLE_FROZEN = 32     /* radiance weighted by the frozen-cdf pdf (rlc_context_set_pdf_mode) */
};
typedef struct rlc_sample_record {
  uint32_t vertex;  /* canonical index within the pass's rows */
  uint32_t cluster;
  uint32_t emitter;
  uint32_t flags;   /* RLC_SAMPLE_* */
  double q_before;
  double v;
  double total;
  double radiance[3];
} rlc_sample_record;
rlc_status rlc_context_enable_sample_export(rlc_context* ctx, int enable);
/* ---- pdf mode (SURVEY 8 notes, 0 fact 2) --------------------------------
 * The reference weights a learned sample's radiance by the LIVE q of its
 * cluster at the moment its update lands (cut.cpp:105: q_before), while the
 * cluster was drawn from the pass-frozen cdf -- the estimator is biased.
 * RLC_PDF_FROZEN_CDF (a non-parity mode) weights it by the probability the
 * selection used, the cluster's share of the frozen cdf; selection and
 * learning are unchanged.  Default RLC_PDF_LIVE_Q (bit-exact with the
 * reference).  Samples exported in the frozen mode carry RLC_SAMPLE_FROZEN. */
enum { RLC_PDF_LIVE_Q = 0, RLC_PDF_FROZEN_CDF = 1 };
rlc_status rlc_context_set_pdf_mode(rlc_context* ctx, int mode);
/* out [max_n] may be NULL (count only); *n_out = path vertices of the pass. */
rlc_status rlc_pass_samples(const rlc_context* ctx, uint64_t max_n, rlc_sample_record* out,
                            uint64_t* n_out);

/* render_frame (proj/src/render.cpp:202-240): image_out [h*w*3] host,
 * resolved; result may be NULL. */
rlc_status rlc_render_frame(const rlc_context* ctx, const rlc_render_config* config,
                            double* image_out, rlc_render_result* result);
/* render_frame with a reference image (render.cpp:226-228): reference
 * [ref_height*ref_width*3] host, linear RGB, top row first; pass_mse [passes]
 * receives mse(framebuffer.resolve(), reference) after every pass, identical
 * to the reference's sequential sum (per-pixel terms on the device, the
 * ordered sum on the host while the next pass runs).  Dimensions other than
 * the camera's fail like mse (RLC_ERR_INVALID_ARGUMENT). */
rlc_status rlc_render_frame_scored(const rlc_context* ctx, const rlc_render_config* config,
                                   const double* reference, int32_t ref_width,
                                   int32_t ref_height, double* image_out,
                                   rlc_render_result* result, double* pass_mse);

/* ---- image module (proj/include/rlcuts/image.hpp:65-78,
 *      proj/src/image.cpp:43-136); host code, images are [h*w*3] doubles,
 *      linear RGB, top row first ----------------------------------------- */
/* write_pfm: float32 RGB, little-endian (scale -1), bottom row first. */
rlc_status rlc_image_write_pfm(const double* pixels, int32_t width, int32_t height,
                               const char* path);
/* read_pfm: *width / *height always set; pixels filled when max_pixels
 * >= width * height (pixels may be NULL to query the size). */
rlc_status rlc_image_read_pfm(const char* path, double* pixels, uint64_t max_pixels,
                              int32_t* width, int32_t* height);
/* write_ppm: 8-bit gamma-2.2 preview. */
rlc_status rlc_image_write_ppm(const double* pixels, int32_t width, int32_t height,
                               const char* path);
/* mse / relative_mse (b is the reference). */
rlc_status rlc_image_mse(const double* a, int32_t wa, int32_t ha, const double* b, int32_t wb,
                         int32_t hb, double* out);
rlc_status rlc_image_relative_mse(const double* a, int32_t wa, int32_t ha, const double* b,
                                  int32_t wb, int32_t hb, double* out);

#ifdef __cplusplus
}
#endif

#endif /* RLCUTS_B200_H */
