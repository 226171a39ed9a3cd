/*
 * edx.h — C ABI of the B200-native embedding-sample dispatch path
 * (libedx.so, built from paper_2512_21615_b200/csrc/).
 *
 * Drop-in boundary for the reference's header-only C++ API in
 * /root/reference/proj/include/embdispatch/.  The reference has no ABI of
 * its own (proj/CMakeLists.txt:13-17: an INTERFACE library of inline
 * functions), so every entry point below names the reference declaration it
 * replaces.  The C++ drop-in headers in include/embdispatch/ forward to these
 * functions and turn status codes back into the reference's exception types
 * with the same messages (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - Plain pointers and sizes; no CUDA or torch types.  Unless a parameter
 *    says "device", every pointer is host memory.
 *  - Every function returns an edx_status.  On failure edx_last_error()
 *    returns the message of the last failing call on this thread.
 *  - Samples are CSR: ids[offsets[i] .. offsets[i+1]) are sample i's
 *    embedding ids in order (EmbeddingSample::ids, types.hpp:37-42).
 *  - Matrices are row-major doubles, rows = samples, cols = workers
 *    (CostMatrix, cost.hpp:52-60).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with EDX_CUDA_ERROR.
 */
#ifndef EDX_H
#define EDX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum edx_status {
  EDX_OK = 0,
  EDX_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  EDX_LOGIC_ERROR = 2,      /* std::logic_error */
  EDX_RUNTIME_ERROR = 3,    /* std::runtime_error */
  EDX_CUDA_ERROR = 4        /* device failure; no reference counterpart */
} edx_status;

/* Message of the last failing call on this thread ("" if none). */
const char* edx_last_error(void);
/* ABI version, bumped on any incompatible change. */
int edx_abi_version(void);

/* embdispatch::ClusterConfig — types.hpp:71-82. */
typedef struct edx_cluster_config {
  int32_t n;                    /* worker count */
  int32_t m;                    /* samples per worker per iteration */
  const double* bandwidths_bps; /* n_bandwidths entries */
  int32_t n_bandwidths;
  int32_t reserved;
  uint64_t d_tran_bytes; /* one embedding transfer */
  uint64_t cache_capacity;
  double alpha; /* exact-solver fraction of EcoMix */
} edx_cluster_config;

/* embdispatch::IterationReport — sim.hpp:38-50 (counts and realised cost).
 * The four per-worker arrays are caller-owned with n entries each. */
typedef struct edx_report {
  uint64_t iteration;
  uint64_t miss_pull, update_push, evict_push;
  uint64_t hits, lookups;
  double cost_s;
  uint64_t* miss_pull_w;
  uint64_t* update_push_w;
  uint64_t* evict_push_w;
  double* cost_w;
} edx_report;

/* validate(const ClusterConfig&, size_t max_sample_len) — types.hpp:87-108. */
int edx_validate_config(const edx_cluster_config* cfg, uint64_t max_sample_len);
/* unit_cost(cfg, j).seconds for every worker — types.hpp:112-120. */
int edx_unit_costs(const edx_cluster_config* cfg, double* out);

/* ------------------------------------------------------------------ engine
 * One engine = one embdispatch::SimState (sim.hpp:54-268) whose global
 * per-embedding state and per-worker caches live in device memory, plus the
 * device buffers of the current batch.  Calls on one engine are ordered on
 * its own CUDA stream; distinct engines may run concurrently. */
typedef struct edx_engine edx_engine;

typedef struct edx_engine_options {
  int32_t device;          /* CUDA ordinal */
  int32_t reserved0;
  uint64_t id_space;       /* ids must be < id_space (dense device state) */
  uint64_t max_batch_ids;  /* capacity of one batch's id stream (sum of lengths) */
  /* multi-GPU row sharding of the cost build; world_size 1 = off */
  int32_t rank;
  int32_t world_size;
  const void* nccl_unique_id; /* 128-byte ncclUniqueId from rank 0, world_size > 1 */
} edx_engine_options;

/* 128-byte ncclUniqueId for a multi-GPU engine group (call on rank 0 and
 * share the bytes with the other ranks, e.g. through torch.distributed). */
int edx_nccl_unique_id(void* out, uint64_t len);

/* The multi-GPU exchange steps over a caller's transport (host buffers).
 * The engine runs exactly this bookkeeping -- which rank builds which rows,
 * who sends what to whom, what is broadcast -- over NCCL on device memory;
 * these entry points let a host harness (tests: torch.distributed gloo)
 * drive it without a GPU.  Callbacks return 0 on success. */
typedef struct edx_transport {
  void* ctx;
  int (*send)(void* ctx, const void* buf, uint64_t bytes, int32_t peer);
  int (*recv)(void* ctx, void* buf, uint64_t bytes, int32_t peer);
  int (*broadcast)(void* ctx, void* buf, uint64_t bytes, int32_t root);
} edx_transport;

/* Row shard [lo[r], hi[r]) of every rank r < world (the cost build's split). */
int edx_shard_rows(uint64_t rows, int32_t world, uint64_t* lo, uint64_t* hi);
/* The engine's gather: every rank holds its shard of the rows x n row-major
 * matrix at its rows' place; afterwards the root holds all of it. */
int edx_exchange_gather_rows(const edx_transport* t, double* matrix, uint64_t rows, int32_t n,
                             int32_t world, int32_t rank, int32_t root);
/* The engine's decision broadcast (one int32 per sample) from the root. */
int edx_exchange_broadcast_decision(const edx_transport* t, int32_t* decision, uint64_t rows,
                                    int32_t root);

/* SimState::SimState(const ClusterConfig&) — sim.hpp:56-59.  With world_size
 * > 1 every rank holds a replica of the state; edx_engine_build computes this
 * rank's row shard and gathers the matrix to rank 0 over NCCL, rank 0 solves
 * and broadcasts the decision, and every rank applies the step. */
int edx_engine_create(const edx_cluster_config* cfg, const edx_engine_options* opt,
                      edx_engine** out);
void edx_engine_destroy(edx_engine* e);

/* Stages one iteration's samples (the std::vector<EmbeddingSample> argument of
 * build_matrix / step, cost.hpp:105 / sim.hpp:87).  on_device != 0 means
 * ids/offsets are device pointers already resident in HBM. */
int edx_engine_load_batch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                          uint64_t num_samples, int on_device);
/* A batch already in device memory whose id count the caller knows: no host
 * round trip (edx_engine_load_batch with on_device=1 reads the offsets back).
 * offsets[0] == 0 and offsets[num_samples] == total_ids are checked on the
 * device and reported by the next synchronising call. */
int edx_engine_load_device_batch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                                 uint64_t num_samples, uint64_t total_ids);
/* build_matrix(samples, snapshot(), cfg) — cost.hpp:105-125 over the live
 * device state (SimState::snapshot, sim.hpp:71-82, costs nothing here).
 * matrix_out (rows*n doubles) may be NULL to keep the matrix on device. */
int edx_engine_build(edx_engine* e, double* matrix_out);
/* ecomix(matrix, cfg) — assign.hpp:247-285 on the engine's matrix, and
 * decision_cost(matrix, decision) — assign.hpp:288-298.  alpha < 0 uses the
 * configured alpha.  Either output may be NULL. */
int edx_engine_dispatch(edx_engine* e, double alpha, int32_t* decision_out,
                        double* expected_cost_out);
/* baseline_hitgreedy(samples, snapshot, cfg) — assign.hpp:346-392 (the
 * paper's relevance-score / LAIA-proxy baseline, dispatch_with kHitGreedy,
 * sim.hpp:390-391) on the loaded batch and the engine's live state.  The
 * decision stays on device for edx_engine_step(e, NULL, ...); decision_out
 * may be NULL.  EDX_INVALID_ARGUMENT "sample count must be m*n". */
int edx_engine_dispatch_hitgreedy(edx_engine* e, int32_t* decision_out);
/* SimState::step(samples, decision) — sim.hpp:87-218.  decision NULL = the
 * engine's last dispatch (already on device). */
int edx_engine_step(edx_engine* e, const int32_t* decision, edx_report* rep);
/* One run() iteration (sim.hpp:421-441): load, build, dispatch, step. */
int edx_engine_iterate(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                       uint64_t num_samples, int on_device, int32_t* decision_out,
                       double* expected_cost_out, edx_report* rep);

/* The engine's CUDA stream (a cudaStream_t) so callers can order their own
 * work and timing events after the engine's. */
int edx_engine_stream(edx_engine* e, void** stream);

/* edx_engine_iterate for a batch already in device memory whose id count the
 * caller knows (see edx_engine_load_device_batch): the batch is staged into the
 * engine's own buffers and the iteration runs as one CUDA graph replay when the
 * engine allows it (one GPU, caches of <= 12,288 entries, profiling off). */
int edx_engine_iterate_device(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                              uint64_t num_samples, uint64_t total_ids, int32_t* decision_out,
                              double* expected_cost_out, edx_report* rep);
/* Input prefetch (the paper's pipelined batch loading; SURVEY
 * 8f item 2): starts the host->device copy of a HOST batch on the engine's
 * copy stream into one of two device slots and returns.  A later
 * edx_engine_iterate / edx_engine_load_batch with the same (ids, offsets,
 * num_samples) host pointers uses the prefetched copy instead of copying
 * again.  The host buffers must stay unchanged until that call (pinned memory
 * makes the copy asynchronous).  Offsets are validated here, with the same
 * messages as edx_engine_load_batch. */
int edx_engine_prefetch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                        uint64_t num_samples);
/* edx_engine_iterate on a host batch (used from the prefetch slot when it was
 * prefetched) that, once the iteration is launched and before waiting for it,
 * prefetches the NEXT host batch (next_ids may be NULL): the steady-state loop
 * of a pipelined caller, copy of batch i+1 overlapping iteration i. */
int edx_engine_iterate_prefetch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                                uint64_t num_samples, const uint32_t* next_ids,
                                const uint64_t* next_offsets, uint64_t next_num_samples,
                                int32_t* decision_out, double* expected_cost_out, edx_report* rep);
/* SimState::seed_entry — sim.hpp:252-261 (test hook). */
int edx_engine_seed_entry(edx_engine* e, uint32_t id, int32_t worker, int latest, int owner);
/* SimState::state_of — sim.hpp:64-67. */
int edx_engine_state_of(edx_engine* e, uint32_t id, uint64_t* owners, uint64_t* latest,
                        uint64_t* resident);
/* SimState::validate_consistency — sim.hpp:222-248. */
int edx_engine_validate_consistency(edx_engine* e);
/* SimState::clock — sim.hpp:61. */
uint64_t edx_engine_clock(edx_engine* e);
/* Counter bumped by every state mutation (step, seed_entry, the imports): a
 * Snapshot view of the device state is current while it is unchanged. */
uint64_t edx_engine_state_version(edx_engine* e);
/* Waits for the work enqueued on the engine (e.g. an edx_engine_build without
 * matrix_out) and reports device-side errors. */
int edx_engine_synchronize(edx_engine* e);
/* decision_cost(matrix, decision) — assign.hpp:288-298 — of the last
 * dispatch (computed on a side stream; this call waits for it). */
int edx_engine_expected_cost(edx_engine* e, double* out);

/* Parity exports (SimState::cache(j).entries(), cache.hpp:180-182, and the
 * global map).  Global: ids with any non-zero mask, ascending id; call with
 * cap = 0 to get the count. */
int edx_engine_export_global(edx_engine* e, uint32_t* ids, uint64_t* owners, uint64_t* latest,
                             uint64_t* resident, uint64_t cap, uint64_t* count);
int edx_engine_cache_size(edx_engine* e, int32_t worker, uint64_t* size);
/* Entries of worker j's cache, ascending id (CacheEntry, cache.hpp:36-42). */
int edx_engine_export_cache(edx_engine* e, int32_t worker, uint32_t* ids, uint8_t* version,
                            uint32_t* mark, uint32_t* freq, uint64_t* last_access);
/* WorkerCache::current_mark and the at-current-mark count (cache.hpp:90,237). */
int edx_engine_cache_marks(edx_engine* e, int32_t worker, uint32_t* current_mark,
                           uint64_t* at_current_mark);
/* Replaces the global masks with a host Snapshot (cost.hpp:39-48) for the
 * const Snapshot& overload of build_matrix; caches are left untouched. */
int edx_engine_import_snapshot(edx_engine* e, const uint32_t* ids, const uint64_t* owners,
                               const uint64_t* latest, const uint64_t* resident,
                               uint64_t count);

/* Replaces the whole SimState (the parity hook SURVEY §8(b) sketches as
 * edx_import_state): the clock (sim.hpp:267), every global_ entry
 * (sim.hpp:266; g_* arrays, ids unique) and every worker's cache
 * (cache.hpp:233-239): worker j's entries are e_*[entry_off[j] ..
 * entry_off[j+1]) (CacheEntry fields, cache.hpp:36-42), plus current_mark_ and
 * at_current_mark_ per worker.  e_version may be NULL; when given it must equal
 * bit j of the entry's `latest` mask (EDX_LOGIC_ERROR "version flag diverged
 * from global state").  The result is checked with
 * edx_engine_validate_consistency (its errors are returned). */
int edx_engine_import_state(edx_engine* e, uint64_t clock, uint64_t g_count, const uint32_t* g_ids,
                            const uint64_t* g_owners, const uint64_t* g_latest,
                            const uint64_t* g_resident, const uint64_t* entry_off,
                            const uint32_t* e_ids, const uint8_t* e_version, const uint32_t* e_mark,
                            const uint32_t* e_freq, const uint64_t* e_last,
                            const uint32_t* current_mark, const uint64_t* at_current_mark);

/* Per-phase device times of the calls since the last reset, measured with CUDA
 * events on the engine stream when profiling is on.  Phases (ms):
 * [0] build  [1] gap+sort  [2] exact solve  [3] greedy  [4] step  [5] whole dispatch
 * counts: [0] launches of own kernels, [1] Hungarian Dijkstra steps (last solve). */
#define EDX_NUM_PHASES 6
int edx_engine_set_profiling(edx_engine* e, int on);
int edx_engine_phase_times(edx_engine* e, double* ms, uint64_t* counts, int reset);

/* Names of the kernels the engine's last cost build, exact solve and greedy
 * launched ("" = none; static strings), for measurement labels. */
int edx_engine_last_kernels(edx_engine* e, const char** build, const char** solver,
                            const char** greedy);

/* Counters of the last exact solve (engine e, or the stateless context when
 * e is NULL): [0] Dijkstra steps [1] cycles in steps [2] cycles applying
 * potentials [3] cycles augmenting [4] cycles re-keying column blocks
 * [5] augmenting-path hops [6] columns re-keyed [7] total solver cycles. */
int edx_solver_stats(edx_engine* e, uint64_t* out);

/* --------------------------------------------------- stateless matrix API
 * Run on a process-wide default device context (device 0 or the current
 * device).  Inputs/outputs are host memory. */

/* build_matrix(samples, snapshot, cfg) — cost.hpp:105-125 with an explicit
 * host Snapshot given as parallel arrays (ids unique). */
int edx_build_matrix(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                     const uint64_t* snap_owners, const uint64_t* snap_latest,
                     const uint64_t* snap_resident, uint64_t snap_count, const uint32_t* ids,
                     const uint64_t* offsets, uint64_t num_samples, double* out);
/* baseline_hitgreedy — assign.hpp:346-392 on a snapshot ({owners, latest}
 * per id; residency is not consulted).  decision: num_samples entries. */
int edx_hitgreedy(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                  const uint64_t* snap_owners, const uint64_t* snap_latest, uint64_t snap_count,
                  const uint32_t* ids, const uint64_t* offsets, uint64_t num_samples,
                  int32_t* decision);
/* expected_cost(sample, j, snapshot, cfg) for every j and every given sample
 * (cost.hpp:81-100) — build_matrix without the m*n sample-count check. */
int edx_expected_costs(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                       const uint64_t* snap_owners, const uint64_t* snap_latest,
                       uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                       uint64_t num_samples, double* out);
/* build_matrix / expected_cost with a SizeLookupFn (cost.hpp:64-73,81-125):
 * sizes[t] = size_of(ids[t]) in bytes for every id position t of the batch
 * (parallel to ids, same offsets); each add is then bytes * 8.0 / bw_j of
 * that id instead of the uniform d_tran unit cost. */
int edx_build_matrix_sized(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                           const uint64_t* snap_owners, const uint64_t* snap_latest,
                           uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                           uint64_t num_samples, const uint64_t* sizes, double* out);
int edx_expected_costs_sized(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                             const uint64_t* snap_owners, const uint64_t* snap_latest,
                             uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                             uint64_t num_samples, const uint64_t* sizes, double* out);
/* row_gap_key — cost.hpp:130-146. */
int edx_row_gap_key(uint64_t rows, uint64_t cols, const double* values, uint64_t row,
                    double* out);
/* rows_by_gap — assign.hpp:197-207. */
int edx_rows_by_gap(uint64_t rows, uint64_t cols, const double* values, uint64_t* order);
/* hungarian(const SquareCost&) — assign.hpp:80-157.  total may be NULL. */
int edx_hungarian(uint64_t k, const double* values, uint64_t* col_of_row, double* total);
/* Hungarian on a column-expanded EcoMix block without materialising it:
 * expand_columns(matrix, rows, mult) (assign.hpp:223-241) then hungarian. */
int edx_hungarian_blocks(uint64_t rows, uint64_t cols, const double* values,
                         const uint64_t* block_rows, int32_t mult, uint64_t* col_of_row,
                         double* total);
/* greedy_dispatch — assign.hpp:162-192; outputs n_order (row, worker) pairs. */
int edx_greedy_dispatch(uint64_t rows, uint64_t cols, const double* values,
                        const uint64_t* order, uint64_t n_order, const int32_t* capacity,
                        uint64_t* out_rows, int32_t* out_workers);
/* ecomix — assign.hpp:247-285.  row_ids may be NULL (identity). */
int edx_ecomix(const edx_cluster_config* cfg, uint64_t rows, uint64_t cols,
               const double* values, const uint64_t* row_ids, int32_t* decision);
/* decision_cost — assign.hpp:288-298. */
int edx_decision_cost(uint64_t rows, uint64_t cols, const double* values,
                      const int32_t* decision, double* out);

/* --------------------------------------------------- standalone WorkerCache
 * cache.hpp:73-240, one device-resident cache driven entry by entry (SimState
 * updates its caches a batch at a time inside edx_engine_step instead).
 * policy: 0 = VictimPolicy::kMarkVersion, 1 = kPriorityRatio.  footprint is
 * the FootprintFn value of the id (1.0 without one), used by kPriorityRatio. */
typedef struct edx_cache edx_cache;
/* WorkerCache(capacity, policy, footprint) — cache.hpp:79-84 */
int edx_cache_create(uint64_t capacity, int policy, int device, edx_cache** out);
void edx_cache_destroy(edx_cache* c);
/* touch(id, latest, now) — cache.hpp:102-122 */
int edx_cache_touch(edx_cache* c, uint32_t id, int latest, uint64_t now, double footprint);
/* set_version(id, latest) — cache.hpp:126-135 */
int edx_cache_set_version(edx_cache* c, uint32_t id, int latest);
/* erase(id) — cache.hpp:174-180 */
int edx_cache_erase(edx_cache* c, uint32_t id);
/* find(id) — cache.hpp:94-97; *found = 0 when absent */
int edx_cache_find(edx_cache* c, uint32_t id, int* found, int* version_latest, uint32_t* mark,
                   uint32_t* frequency, uint64_t* last_access);
/* select_victim() — cache.hpp:141-148 */
int edx_cache_select_victim(edx_cache* c, uint32_t* victim);
/* evict_for(needed, needs_push, pinned) — cache.hpp:152-170: the evicted ids
 * in eviction order (at most capacity); needs_push is applied by the caller. */
int edx_cache_evict_for(edx_cache* c, uint64_t needed, const uint32_t* pinned, uint64_t n_pinned,
                        uint32_t* victims, uint64_t* n_victims);
/* size(), current_mark() and the at-current-mark count — cache.hpp:86-91 */
int edx_cache_info(edx_cache* c, uint64_t* size, uint32_t* current_mark, uint64_t* at_current_mark);
/* entries() — cache.hpp:180-182, as parallel arrays (count first with ids NULL) */
int edx_cache_export(edx_cache* c, uint32_t* ids, uint8_t* version, uint32_t* mark,
                     uint32_t* frequency, uint64_t* last_access, uint64_t cap_out, uint64_t* count);

/* ------------------------------------------------- synthetic input stream
 * ZipfStream (workload.hpp:94-133): the benchmark's input producer, host side. */
typedef struct edx_zipf edx_zipf;
int edx_zipf_create(uint64_t total_embeddings, uint64_t sample_len, double zipf_s,
                    uint64_t iterations, uint64_t seed, uint64_t samples_per_iteration,
                    edx_zipf** out);
/* Fills samples_per_iteration*sample_len ids; returns 1, or 0 at the end. */
int edx_zipf_next(edx_zipf* z, uint32_t* ids);
void edx_zipf_reset(edx_zipf* z);
/* ZipfSampler (workload.hpp:54-79): ids in [0, population) with P(id) ∝
 * (id+1)^-s, drawn from std::mt19937_64(seed) by inverse CDF; free with
 * edx_zipf_destroy.  edx_zipf_draw returns the next `count` draws. */
int edx_zipf_sampler_create(uint64_t population, double zipf_s, uint64_t seed, edx_zipf** out);
int edx_zipf_draw(edx_zipf* z, uint64_t count, uint32_t* out);
void edx_zipf_destroy(edx_zipf* z);

/* ------------------------------------------------------------ trace input
 * TraceStream (workload.hpp:176-268): a plain-text trace, one sample per line,
 * read once and held as per-iteration CSR (offsets rebased to 0) for the
 * engine's batch entry points.  table_sizes = NULL: no schema; otherwise the
 * schema's n_tables table sizes and names (TraceSchema, workload.hpp:137-150).  Errors
 * are EDX_RUNTIME_ERROR with the reference's messages; the dropped trailing
 * partial iteration is reported by edx_trace_info (the caller warns). */
typedef struct edx_trace edx_trace;
int edx_trace_load(const char* path, uint64_t n_tables, const uint64_t* table_sizes,
                   const char* const* table_names, uint64_t samples_per_iteration,
                   uint64_t cache_capacity, uint64_t m, edx_trace** out);
void edx_trace_info(const edx_trace* t, uint64_t* iterations, uint64_t* dropped,
                    uint64_t* max_sample_len, uint64_t* samples);
/* Iteration it (< iterations): ids, offsets[samples_per_iteration + 1] and the
 * id count, pointing into the trace (valid until edx_trace_destroy). */
int edx_trace_iteration(const edx_trace* t, uint64_t it, const uint32_t** ids,
                        const uint64_t** offsets, uint64_t* num_ids);
void edx_trace_destroy(edx_trace* t);

#ifdef __cplusplus
}
#endif

#endif /* EDX_H */
