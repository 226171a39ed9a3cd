/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference embdispatch hot path
 * (/root/reference/proj/include/embdispatch/{types,cost,assign,cache,sim,workload}.hpp)
 * used as the CPU checker for the CUDA product in paper_2512_21615_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It is never on the product path.
 *
 * The same `orc_*` ABI is exported by oracle/ref_shim.cpp, which compiles the
 * UNMODIFIED reference headers into oracle/_ref/libedx_ref.so, so every test
 * can run one binding against either library.  Parity of this restatement
 * against the compiled reference is pinned by tests/test_oracle_vs_ref.py
 * (here, where /root/reference exists) and by the committed fixtures under
 * tests/golden/ (generated from oracle/_ref by tests/golden/make_golden.py).
 *
 * Build: cc -O2 -ffp-contract=off (the reference engine has no contractible
 * a*b+c, but the flag keeps the oracle bit-stable on every host).
 */
#ifndef EDX_ORACLE_H
#define EDX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the reference's exception classes. */
#define ORC_OK 0
#define ORC_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define ORC_LOGIC_ERROR 2      /* std::logic_error */
#define ORC_RUNTIME_ERROR 3    /* std::runtime_error */

/* Same layout as edx_cluster_config in include/edx.h (types.hpp:71-82). */
typedef struct orc_cluster_config {
  int32_t n;
  int32_t m;
  const double* bandwidths_bps;
  int32_t n_bandwidths;
  int32_t reserved;
  uint64_t d_tran_bytes;
  uint64_t cache_capacity;
  double alpha;
} orc_cluster_config;

/* Same layout as edx_report in include/edx.h (IterationReport, sim.hpp:38-50).
 * The per-worker arrays are caller-owned, n entries each. */
typedef struct orc_report {
  uint64_t iteration;
  uint64_t miss_pull, update_push, evict_push;
  uint64_t hits, lookups;
  double cost_s;
  uint64_t* miss_pull_w;
  uint64_t* update_push_w;
  uint64_t* evict_push_w;
  double* cost_w;
} orc_report;

const char* orc_last_error(void);

int orc_validate_config(const orc_cluster_config* cfg, uint64_t max_sample_len);
int orc_unit_costs(const orc_cluster_config* cfg, double* out);

/* ---- workload (workload.hpp:54-133) ---- */
typedef struct orc_zipf orc_zipf;
int orc_zipf_create(uint64_t total_embeddings, uint64_t sample_len, double zipf_s,
                    uint64_t iterations, uint64_t seed, uint64_t samples_per_iteration,
                    orc_zipf** out);
void orc_zipf_destroy(orc_zipf* z);
/* Fills ids[samples_per_iteration*sample_len]; returns 1 if produced, 0 at end. */
int orc_zipf_next(orc_zipf* z, uint32_t* ids);
void orc_zipf_reset(orc_zipf* z);
/* cmd_bench matrix (experiment.hpp:217-223): k*k uniform [0,1) doubles. */
void orc_bench_matrix(uint64_t k, double* out);

/* ---- matrix-level API (cost.hpp, assign.hpp) ---- */
int orc_build_matrix_snapshot(const orc_cluster_config* cfg, const uint32_t* snap_ids,
                              const uint64_t* snap_owners, const uint64_t* snap_latest,
                              const uint64_t* snap_resident, uint64_t snap_count,
                              const uint32_t* ids, const uint64_t* offsets,
                              uint64_t num_samples, double* out);
/* expected_cost (cost.hpp:81-100) of every (sample, worker) with a
 * SizeLookupFn (cost.hpp:64-73): sizes[t] = size_of(ids[t]) bytes per id
 * position; no sample-count check (build_matrix adds only that). */
int orc_expected_costs_sized(const orc_cluster_config* cfg, const uint32_t* snap_ids,
                             const uint64_t* snap_owners, const uint64_t* snap_latest,
                             uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                             uint64_t num_samples, const uint64_t* sizes, double* out);
/* baseline_hitgreedy — assign.hpp:346-392 on a snapshot (owners/latest). */
int orc_hitgreedy_snapshot(const orc_cluster_config* cfg, const uint32_t* snap_ids,
                           const uint64_t* snap_owners, const uint64_t* snap_latest,
                           uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                           uint64_t num_samples, int32_t* decision);
int orc_row_gap_key(uint64_t rows, uint64_t cols, const double* values, uint64_t row,
                    double* out);
int orc_rows_by_gap(uint64_t rows, uint64_t cols, const double* values, uint64_t* order);
int orc_hungarian(uint64_t k, const double* values, uint64_t* col_of_row, double* total);
int orc_greedy_dispatch(uint64_t rows, uint64_t cols, const double* values,
                        const uint64_t* order, uint64_t n_order, const int32_t* capacity,
                        uint64_t* out_rows, int32_t* out_workers);
int orc_ecomix(const orc_cluster_config* cfg, uint64_t rows, uint64_t cols,
               const double* values, const uint64_t* row_ids, int32_t* decision);
int orc_decision_cost(uint64_t rows, uint64_t cols, const double* values,
                      const int32_t* decision, double* out);

/* ---- engine (sim.hpp SimState + cache.hpp WorkerCache) ---- */
typedef struct orc_sim orc_sim;
int orc_sim_create(const orc_cluster_config* cfg, orc_sim** out);
void orc_sim_destroy(orc_sim* s);
int orc_sim_build_matrix(orc_sim* s, const uint32_t* ids, const uint64_t* offsets,
                         uint64_t num_samples, double* out);
/* baseline_hitgreedy on the simulator's live state (its snapshot). */
int orc_sim_hitgreedy(orc_sim* s, const uint32_t* ids, const uint64_t* offsets,
                      uint64_t num_samples, int32_t* decision);
int orc_sim_step(orc_sim* s, const uint32_t* ids, const uint64_t* offsets,
                 uint64_t num_samples, const int32_t* decision, orc_report* rep);
int orc_sim_seed_entry(orc_sim* s, uint32_t id, int32_t worker, int latest, int owner);
int orc_sim_validate_consistency(orc_sim* s);
uint64_t orc_sim_clock(orc_sim* s);
uint64_t orc_sim_global_count(orc_sim* s);
void orc_sim_export_global(orc_sim* s, uint32_t* ids, uint64_t* owners, uint64_t* latest,
                           uint64_t* resident);
uint64_t orc_sim_cache_size(orc_sim* s, int32_t worker);
void orc_sim_export_cache(orc_sim* s, int32_t worker, uint32_t* ids, uint8_t* version,
                          uint32_t* mark, uint32_t* freq, uint64_t* last_access);
void orc_sim_cache_marks(orc_sim* s, int32_t worker, uint32_t* current_mark,
                         uint64_t* at_current_mark);
/* Replaces the whole simulator state (parity hook, the counterpart of
 * edx_engine_import_state): the clock, every global_ entry (sim.hpp:266) and
 * every worker's cache entries (cache.hpp:233-239), current_mark_ and
 * at_current_mark_.  Worker j's entries are e_*[entry_off[j] .. entry_off[j+1]). */
int orc_sim_import_state(orc_sim* s, uint64_t clock, uint64_t g_count, const uint32_t* g_ids,
                         const uint64_t* g_owners, const uint64_t* g_latest,
                         const uint64_t* g_resident, const uint64_t* entry_off,
                         const uint32_t* e_ids, const uint8_t* e_version, const uint32_t* e_mark,
                         const uint32_t* e_freq, const uint64_t* e_last,
                         const uint32_t* current_mark, const uint64_t* at_current_mark);

/* One full reference iteration timed like run() (sim.hpp:421-441):
 * snapshot -> build_matrix -> ecomix -> step, plus decision_cost.  times_s
 * receives {snapshot, build, decide, step} seconds; threads > 1 partitions
 * the build rows over host threads (bit-identical: rows are independent). */
int orc_ref_iteration(orc_sim* s, const uint32_t* ids, const uint64_t* offsets,
                      uint64_t num_samples, int threads, int32_t* decision,
                      double* expected_cost, orc_report* rep, double* times_s);

/* ---- standalone WorkerCache (cache.hpp:73-240) ----
 * policy 0 = kMarkVersion, 1 = kPriorityRatio; footprint = FootprintFn(id)
 * of the touched id (kept per id, 1.0 for ids never given one). */
typedef struct orc_cache orc_cache;
int orc_cache_create(uint64_t capacity, int policy, orc_cache** out);
void orc_cache_destroy(orc_cache* c);
int orc_cache_touch(orc_cache* c, uint32_t id, int latest, uint64_t now, double footprint);
int orc_cache_set_version(orc_cache* c, uint32_t id, int latest);
int orc_cache_erase(orc_cache* c, uint32_t id);
int orc_cache_select_victim(orc_cache* c, uint32_t* victim);
int orc_cache_evict_for(orc_cache* c, uint64_t needed, const uint32_t* pinned, uint64_t n_pinned,
                        uint32_t* victims, uint64_t* n_victims);
void orc_cache_info(orc_cache* c, uint64_t* size, uint32_t* current_mark);
/* entries sorted by id */
void orc_cache_export(orc_cache* c, uint32_t* ids, uint8_t* version, uint32_t* mark,
                      uint32_t* freq, uint64_t* last_access);

/* ---- report formats (report_io.hpp; compiled reference only) ---- */
typedef struct orc_iter_report {
  uint64_t iteration;
  const char* mechanism;
  uint64_t miss_pull, update_push, evict_push, hits, lookups;
  double cost_s, decision_s, matrix_s, expected_cost_s;
  int32_t has_expected, n;
  const uint64_t *miss_pull_w, *update_push_w, *evict_push_w;
  const double* cost_w;
} orc_iter_report;
typedef struct orc_run_summary {
  const char* mechanism;
  uint64_t iterations, measured_iterations, miss_pull, update_push, evict_push, hits, lookups;
  double cost_s, expected_cost_s, decision_s_total, decision_s_max, matrix_s_total;
  int32_t has_expected, n;
  uint64_t budget_violations;
  const uint64_t *miss_pull_w, *update_push_w, *evict_push_w, *ops_w;
} orc_run_summary;
/* report_jsonl (report_io.hpp:35-55); *len = bytes needed (out may be NULL) */
int orc_report_jsonl(const orc_iter_report* rep, char* out, uint64_t cap, uint64_t* len);
/* comparison_csv (report_io.hpp:89-146) */
int orc_comparison_csv(const orc_run_summary* runs, uint64_t count, const char* reference,
                       const orc_cluster_config* cfg, char* out, uint64_t cap, uint64_t* len);

/* TraceStream dump (workload.hpp:176-268; compiled reference only):
 * "iterations I dropped D max M\n", kept samples one per line, warnings. */
int orc_trace_dump(const char* path, const char* schema_path, int32_t n, int32_t m,
                   uint64_t capacity, char* out, uint64_t cap, uint64_t* len);

/* Cross-check counters: total Dijkstra steps of the last orc_hungarian call. */
uint64_t orc_last_hungarian_steps(void);

#ifdef __cplusplus
}
#endif

#endif
