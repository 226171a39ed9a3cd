// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference headers (/root/reference/proj/include,
// read in place through -I, never copied) behind the same `orc_*` C ABI as
// oracle/edx_oracle.c, so tests can run the identical binding against the
// real reference.  Built by oracle/Makefile into oracle/_ref/libedx_ref.so.
//
// It also exports orc_ref_iteration(), the reference's own per-iteration
// sequence (SimState::snapshot -> build_matrix -> ecomix -> decision_cost ->
// SimState::step; sim.hpp:421-441) timed phase by phase with steady_clock,
// exactly where run() times it (sim.hpp:423-432).  bench.py --impl reference
// and the cpu_baseline leg drive that entry point.  The optional row-parallel
// build partitions rows over std::threads, each calling the reference's
// expected_cost (cost.hpp:81); rows are independent, so it is bit-identical
// ("all host cores" variant).

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <set>
#include <unordered_map>
#include <vector>

#include "embdispatch/assign.hpp"
#include "embdispatch/cost.hpp"
#include "embdispatch/report_io.hpp"
#include "embdispatch/sim.hpp"
#include "embdispatch/workload.hpp"

#include "edx_oracle.h"

using namespace embdispatch;

namespace {

thread_local std::string g_err;
thread_local std::uint64_t g_steps = 0;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORC_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return ORC_LOGIC_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_RUNTIME_ERROR;
  }
}

ClusterConfig to_cfg(const orc_cluster_config* c) {
  ClusterConfig cfg;
  cfg.n = c->n;
  cfg.m = c->m;
  cfg.bandwidths_bps.assign(c->bandwidths_bps, c->bandwidths_bps + c->n_bandwidths);
  cfg.d_tran_bytes = c->d_tran_bytes;
  cfg.cache_capacity = static_cast<std::size_t>(c->cache_capacity);
  cfg.alpha = c->alpha;
  return cfg;
}

std::vector<EmbeddingSample> to_samples(const uint32_t* ids, const uint64_t* offsets,
                                        uint64_t R) {
  std::vector<EmbeddingSample> out(R);
  for (uint64_t i = 0; i < R; ++i) out[i].ids.assign(ids + offsets[i], ids + offsets[i + 1]);
  return out;
}

CostMatrix to_matrix(uint64_t rows, uint64_t cols, const double* values) {
  CostMatrix m;
  m.rows = rows;
  m.cols = cols;
  m.values.assign(values, values + rows * cols);
  m.row_ids.resize(rows);
  for (uint64_t i = 0; i < rows; ++i) m.row_ids[i] = i;
  return m;
}

void copy_report(const IterationReport& r, int n, orc_report* out) {
  out->iteration = r.iteration;
  out->miss_pull = r.miss_pull;
  out->update_push = r.update_push;
  out->evict_push = r.evict_push;
  out->hits = r.hits;
  out->lookups = r.lookups;
  out->cost_s = r.cost_s;
  for (int j = 0; j < n; ++j) {
    out->miss_pull_w[j] = r.miss_pull_w[j];
    out->update_push_w[j] = r.update_push_w[j];
    out->evict_push_w[j] = r.evict_push_w[j];
    out->cost_w[j] = r.cost_w[j];
  }
}

}  // namespace

struct orc_zipf {
  WorkloadSpec spec;
  ClusterConfig cfg;
  ZipfStream stream;
  std::vector<EmbeddingSample> buf;
  orc_zipf(const WorkloadSpec& s, const ClusterConfig& c) : spec(s), cfg(c), stream(s, c) {}
};

struct orc_sim {
  ClusterConfig cfg;
  SimState state;
  explicit orc_sim(const ClusterConfig& c) : cfg(c), state(c) {}
};

namespace {

// Parity import (orc_sim_import_state): the reference keeps SimState's and
// WorkerCache's state private and has no setter.  An explicit template
// instantiation may name private members ([temp.spec.general]), so a friend
// defined inside one hands out the member pointer -- the reference headers
// stay unmodified and are still compiled in place.
template <class Tag, typename Tag::type M>
struct Rob {
  friend typename Tag::type get(Tag) { return M; }
};
#define EDX_ROB(NAME, CLASS, TYPE, MEMBER)                   \
  struct NAME {                                              \
    using type = TYPE CLASS::*;                              \
    friend type get(NAME);                                   \
  };                                                         \
  template struct Rob<NAME, &CLASS::MEMBER>;
using GlobalMap = std::unordered_map<EmbeddingId, EmbeddingState>;
using EntryMap = std::unordered_map<EmbeddingId, CacheEntry>;
EDX_ROB(RobCaches, SimState, std::vector<WorkerCache>, caches_)
EDX_ROB(RobGlobal, SimState, GlobalMap, global_)
EDX_ROB(RobClock, SimState, std::uint64_t, clock_)
EDX_ROB(RobEntries, WorkerCache, EntryMap, entries_)
EDX_ROB(RobOrder, WorkerCache, std::set<VictimKey>, order_)
EDX_ROB(RobMark, WorkerCache, std::uint32_t, current_mark_)
EDX_ROB(RobAtMark, WorkerCache, std::size_t, at_current_mark_)
#undef EDX_ROB

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_validate_config(const orc_cluster_config* c, uint64_t max_len) {
  return guarded([&] { validate(to_cfg(c), static_cast<std::size_t>(max_len)); });
}

int orc_unit_costs(const orc_cluster_config* c, double* out) {
  return guarded([&] {
    const ClusterConfig cfg = to_cfg(c);
    for (int j = 0; j < cfg.n; ++j) out[j] = unit_cost(cfg, j).seconds;
  });
}

int orc_zipf_create(uint64_t total, uint64_t sample_len, double zipf_s, uint64_t iterations,
                    uint64_t seed, uint64_t per_iteration, orc_zipf** out) {
  return guarded([&] {
    WorkloadSpec spec;
    spec.total_embeddings = total;
    spec.sample_len = sample_len;
    spec.zipf_s = zipf_s;
    spec.iterations = iterations;
    spec.seed = seed;
    ClusterConfig cfg;
    cfg.n = 1;
    cfg.m = static_cast<int>(per_iteration);
    *out = new orc_zipf(spec, cfg);
  });
}

void orc_zipf_destroy(orc_zipf* z) { delete z; }

int orc_zipf_next(orc_zipf* z, uint32_t* ids) {
  if (!z->stream.next_iteration(z->buf)) return 0;
  std::size_t off = 0;
  for (const auto& s : z->buf) {
    std::memcpy(ids + off, s.ids.data(), s.ids.size() * sizeof(uint32_t));
    off += s.ids.size();
  }
  return 1;
}

void orc_zipf_reset(orc_zipf* z) { z->stream.reset(); }

void orc_bench_matrix(uint64_t k, double* out) {
  std::mt19937_64 rng(0x5eedULL ^ k);
  for (uint64_t i = 0; i < k * k; ++i) out[i] = static_cast<double>(rng() >> 11) * 0x1.0p-53;
}

int orc_build_matrix_snapshot(const orc_cluster_config* c, const uint32_t* snap_ids,
                              const uint64_t* owners, const uint64_t* latest,
                              const uint64_t* resident, uint64_t count, const uint32_t* ids,
                              const uint64_t* offsets, uint64_t R, double* out) {
  return guarded([&] {
    Snapshot snap;
    for (uint64_t s = 0; s < count; ++s) {
      EmbeddingState& st = snap.states[snap_ids[s]];
      st.owners = owners[s];
      st.latest = latest[s];
      st.resident = resident ? resident[s] : 0;
    }
    const CostMatrix m = build_matrix(to_samples(ids, offsets, R), snap, to_cfg(c));
    std::memcpy(out, m.values.data(), m.values.size() * sizeof(double));
  });
}

int orc_expected_costs_sized(const orc_cluster_config* c, const uint32_t* snap_ids,
                             const uint64_t* owners, const uint64_t* latest, uint64_t count,
                             const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                             const uint64_t* sizes, double* out) {
  return guarded([&] {
    Snapshot snap;
    for (uint64_t s = 0; s < count; ++s) {
      EmbeddingState& st = snap.states[snap_ids[s]];
      st.owners = owners[s];
      st.latest = latest[s];
    }
    std::unordered_map<EmbeddingId, std::uint64_t> table;
    for (uint64_t t = offsets[0]; t < offsets[R]; ++t) table[ids[t]] = sizes[t];
    const SizeLookupFn size_of = [&table](EmbeddingId id) { return table.at(id); };
    const ClusterConfig cfg = to_cfg(c);
    const auto samples = to_samples(ids, offsets, R);
    for (uint64_t i = 0; i < R; ++i)
      for (int j = 0; j < cfg.n; ++j)
        out[i * static_cast<uint64_t>(cfg.n) + static_cast<uint64_t>(j)] =
            expected_cost(samples[i], j, snap, cfg, size_of);
  });
}

int orc_row_gap_key(uint64_t rows, uint64_t cols, const double* values, uint64_t row,
                    double* out) {
  return guarded([&] { *out = row_gap_key(to_matrix(rows, cols, values), row); });
}

int orc_rows_by_gap(uint64_t rows, uint64_t cols, const double* values, uint64_t* order) {
  return guarded([&] {
    const auto o = rows_by_gap(to_matrix(rows, cols, values));
    for (uint64_t i = 0; i < rows; ++i) order[i] = o[i];
  });
}

int orc_hungarian(uint64_t k, const double* values, uint64_t* col_of_row, double* total) {
  return guarded([&] {
    SquareCost sq;
    sq.order = k;
    sq.values.assign(values, values + k * k);
    const AssignmentResult r = hungarian(sq);
    for (uint64_t i = 0; i < k; ++i) col_of_row[i] = r.col_of_row[i];
    if (total) *total = r.total_cost;
  });
}

int orc_hitgreedy_snapshot(const orc_cluster_config* c, const uint32_t* snap_ids,
                           const uint64_t* owners, const uint64_t* latest, uint64_t count,
                           const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                           int32_t* decision) {
  return guarded([&] {
    Snapshot snap;
    for (uint64_t s = 0; s < count; ++s) {
      EmbeddingState& st = snap.states[snap_ids[s]];
      st.owners = owners[s];
      st.latest = latest[s];
    }
    const DispatchDecision d = baseline_hitgreedy(to_samples(ids, offsets, R), snap, to_cfg(c));
    for (std::size_t i = 0; i < d.worker_of_sample.size(); ++i) decision[i] = d.worker_of_sample[i];
  });
}

int orc_greedy_dispatch(uint64_t rows, uint64_t cols, const double* values,
                        const uint64_t* order, uint64_t n_order, const int32_t* capacity,
                        uint64_t* out_rows, int32_t* out_workers) {
  return guarded([&] {
    std::vector<std::size_t> o(order, order + n_order);
    std::vector<int> cap(capacity, capacity + cols);
    const auto part = greedy_dispatch(to_matrix(rows, cols, values), o, cap);
    for (std::size_t t = 0; t < part.size(); ++t) {
      out_rows[t] = part[t].first;
      out_workers[t] = part[t].second;
    }
  });
}

int orc_ecomix(const orc_cluster_config* c, uint64_t rows, uint64_t cols, const double* values,
               const uint64_t* row_ids, int32_t* decision) {
  return guarded([&] {
    CostMatrix m = to_matrix(rows, cols, values);
    if (row_ids)
      for (uint64_t i = 0; i < rows; ++i) m.row_ids[i] = row_ids[i];
    const DispatchDecision d = ecomix(m, to_cfg(c));
    for (uint64_t i = 0; i < rows; ++i) decision[i] = d.worker_of_sample[i];
  });
}

int orc_decision_cost(uint64_t rows, uint64_t cols, const double* values,
                      const int32_t* decision, double* out) {
  return guarded([&] {
    DispatchDecision d;
    d.worker_of_sample.assign(decision, decision + rows);
    *out = decision_cost(to_matrix(rows, cols, values), d);
  });
}

int orc_sim_create(const orc_cluster_config* c, orc_sim** out) {
  return guarded([&] { *out = new orc_sim(to_cfg(c)); });
}

void orc_sim_destroy(orc_sim* s) { delete s; }

int orc_sim_build_matrix(orc_sim* s, const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                         double* out) {
  return guarded([&] {
    const Snapshot snap = s->state.snapshot();
    const CostMatrix m = build_matrix(to_samples(ids, offsets, R), snap, s->cfg);
    std::memcpy(out, m.values.data(), m.values.size() * sizeof(double));
  });
}

int orc_sim_hitgreedy(orc_sim* s, const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                      int32_t* decision) {
  return guarded([&] {
    const Snapshot snap = s->state.snapshot();
    const DispatchDecision d = baseline_hitgreedy(to_samples(ids, offsets, R), snap, s->cfg);
    for (std::size_t i = 0; i < d.worker_of_sample.size(); ++i) decision[i] = d.worker_of_sample[i];
  });
}

int orc_sim_step(orc_sim* s, const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                 const int32_t* decision, orc_report* rep) {
  return guarded([&] {
    DispatchDecision d;
    d.worker_of_sample.assign(decision, decision + R);
    const IterationReport r = s->state.step(to_samples(ids, offsets, R), d);
    copy_report(r, s->cfg.n, rep);
  });
}

int orc_sim_seed_entry(orc_sim* s, uint32_t id, int32_t worker, int latest, int owner) {
  return guarded([&] { s->state.seed_entry(id, worker, latest != 0, owner != 0); });
}

int orc_sim_validate_consistency(orc_sim* s) {
  return guarded([&] { s->state.validate_consistency(); });
}

uint64_t orc_sim_clock(orc_sim* s) { return s->state.clock(); }

uint64_t orc_sim_global_count(orc_sim* s) { return s->state.snapshot().states.size(); }

void orc_sim_export_global(orc_sim* s, uint32_t* ids, uint64_t* owners, uint64_t* latest,
                           uint64_t* resident) {
  const Snapshot snap = s->state.snapshot();
  std::size_t t = 0;
  for (const auto& [id, st] : snap.states) {
    ids[t] = id;
    owners[t] = st.owners;
    latest[t] = st.latest;
    resident[t] = st.resident;
    ++t;
  }
}

uint64_t orc_sim_cache_size(orc_sim* s, int32_t worker) { return s->state.cache(worker).size(); }

void orc_sim_export_cache(orc_sim* s, int32_t worker, uint32_t* ids, uint8_t* version,
                          uint32_t* mark, uint32_t* freq, uint64_t* last_access) {
  std::size_t t = 0;
  for (const auto& [id, e] : s->state.cache(worker).entries()) {
    ids[t] = id;
    version[t] = e.version_latest ? 1 : 0;
    mark[t] = e.mark;
    freq[t] = e.frequency;
    last_access[t] = e.last_access;
    ++t;
  }
}

int orc_sim_import_state(orc_sim* s, uint64_t clock, uint64_t g_count, const uint32_t* g_ids,
                         const uint64_t* g_owners, const uint64_t* g_latest,
                         const uint64_t* g_resident, const uint64_t* entry_off,
                         const uint32_t* e_ids, const uint8_t* e_version, const uint32_t* e_mark,
                         const uint32_t* e_freq, const uint64_t* e_last,
                         const uint32_t* current_mark, const uint64_t* at_current_mark) {
  return guarded([&] {
    SimState& st = s->state;
    st.*get(RobClock{}) = clock;
    GlobalMap& g = st.*get(RobGlobal{});
    g.clear();
    g.reserve(g_count);
    for (uint64_t t = 0; t < g_count; ++t)
      g[g_ids[t]] = EmbeddingState{g_owners[t], g_latest[t], g_resident[t]};
    std::vector<WorkerCache>& caches = st.*get(RobCaches{});
    for (int j = 0; j < s->cfg.n; ++j) {
      WorkerCache& c = caches[j];
      EntryMap& em = c.*get(RobEntries{});
      std::set<VictimKey>& order = c.*get(RobOrder{});
      em.clear();
      order.clear();
      const uint64_t a = entry_off[j], b = entry_off[j + 1];
      if (b - a > c.capacity()) throw std::invalid_argument("imported cache exceeds its capacity");
      em.reserve(b - a);
      for (uint64_t t = a; t < b; ++t) {
        const CacheEntry e{e_ids[t], e_version[t] != 0, e_mark[t], e_freq[t], e_last[t]};
        em.emplace(e.id, e);
        order.insert(victim_key(e));
      }
      c.*get(RobMark{}) = current_mark[j];
      c.*get(RobAtMark{}) = static_cast<std::size_t>(at_current_mark[j]);
    }
  });
}

void orc_sim_cache_marks(orc_sim* s, int32_t worker, uint32_t* current_mark,
                         uint64_t* at_current_mark) {
  const WorkerCache& c = s->state.cache(worker);
  *current_mark = c.current_mark();
  // at_current_mark_ is private in the reference; count it from the entries
  // (cache.hpp:111,116,175 keep it equal to #entries with mark == current).
  uint64_t at = 0;
  for (const auto& [id, e] : c.entries())
    if (e.mark == c.current_mark()) ++at;
  *at_current_mark = at;
}

uint64_t orc_last_hungarian_steps(void) { return g_steps; }

// Standalone WorkerCache: the reference class itself; the footprint callback
// reads the value recorded for the id at its touches.
struct orc_cache {
  std::unordered_map<EmbeddingId, double> fp;
  WorkerCache cache;
  orc_cache(uint64_t cap, int policy)
      : cache(cap, policy ? VictimPolicy::kPriorityRatio : VictimPolicy::kMarkVersion,
              [this](EmbeddingId id) {
                auto it = fp.find(id);
                return it == fp.end() ? 1.0 : it->second;
              }) {}
};

int orc_cache_create(uint64_t capacity, int policy, orc_cache** out) {
  return guarded([&] { *out = new orc_cache(capacity, policy); });
}
void orc_cache_destroy(orc_cache* c) { delete c; }
int orc_cache_touch(orc_cache* c, uint32_t id, int latest, uint64_t now, double footprint) {
  return guarded([&] {
    if (!c->cache.resident(id) && !c->cache.full()) c->fp[id] = footprint;
    c->cache.touch(id, latest != 0, now);
  });
}
int orc_cache_set_version(orc_cache* c, uint32_t id, int latest) {
  return guarded([&] { c->cache.set_version(id, latest != 0); });
}
int orc_cache_erase(orc_cache* c, uint32_t id) {
  return guarded([&] { c->cache.erase(id); });
}
int orc_cache_select_victim(orc_cache* c, uint32_t* victim) {
  return guarded([&] { *victim = c->cache.select_victim(); });
}
int orc_cache_evict_for(orc_cache* c, uint64_t needed, const uint32_t* pinned, uint64_t n_pinned,
                        uint32_t* victims, uint64_t* n_victims) {
  return guarded([&] {
    WorkerCache::PinnedSet pins(pinned, pinned + n_pinned);
    const auto ev = c->cache.evict_for(needed, nullptr, n_pinned ? &pins : nullptr);
    *n_victims = ev.size();
    for (std::size_t t = 0; t < ev.size(); ++t) victims[t] = ev[t].first;
  });
}
void orc_cache_info(orc_cache* c, uint64_t* size, uint32_t* current_mark) {
  *size = c->cache.size();
  *current_mark = c->cache.current_mark();
}
void orc_cache_export(orc_cache* c, uint32_t* ids, uint8_t* version, uint32_t* mark,
                      uint32_t* freq, uint64_t* last_access) {
  std::vector<CacheEntry> es;
  for (const auto& [id, e] : c->cache.entries()) es.push_back(e);
  std::sort(es.begin(), es.end(), [](const CacheEntry& a, const CacheEntry& b) { return a.id < b.id; });
  for (std::size_t t = 0; t < es.size(); ++t) {
    ids[t] = es[t].id;
    version[t] = es[t].version_latest;
    mark[t] = es[t].mark;
    freq[t] = es[t].frequency;
    last_access[t] = es[t].last_access;
  }
}

// One reference iteration, timed like run() (sim.hpp:421-441).  times_s gets
// {snapshot, build, decide, step}; `threads` > 1 partitions build rows.
int orc_ref_iteration(orc_sim* s, const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                      int threads, int32_t* decision, double* expected_out, orc_report* rep,
                      double* times_s) {
  return guarded([&] {
    using clk = std::chrono::steady_clock;
    const auto samples = to_samples(ids, offsets, R);
    const auto t0 = clk::now();
    const Snapshot snap = s->state.snapshot();
    const auto t1 = clk::now();
    CostMatrix matrix;
    if (threads <= 1) {
      matrix = build_matrix(samples, snap, s->cfg);
    } else {
      if (samples.size() != s->cfg.samples_per_iteration())
        throw std::invalid_argument("expected m*n samples");
      matrix.rows = samples.size();
      matrix.cols = static_cast<std::size_t>(s->cfg.n);
      matrix.values.resize(matrix.rows * matrix.cols);
      matrix.row_ids.resize(matrix.rows);
      std::vector<std::thread> pool;
      const std::size_t chunk = (matrix.rows + threads - 1) / threads;
      for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
          const std::size_t lo = t * chunk, hi = std::min(matrix.rows, lo + chunk);
          for (std::size_t i = lo; i < hi; ++i) {
            matrix.row_ids[i] = i;
            for (WorkerId j = 0; j < s->cfg.n; ++j)
              matrix.at(i, j) = embdispatch::expected_cost(samples[i], j, snap, s->cfg);
          }
        });
      }
      for (auto& th : pool) th.join();
    }
    const auto t2 = clk::now();
    const DispatchDecision d = ecomix(matrix, s->cfg);
    const auto t3 = clk::now();
    const IterationReport r = s->state.step(samples, d);
    const auto t4 = clk::now();
    if (expected_out) *expected_out = decision_cost(matrix, d);
    if (decision)
      for (uint64_t i = 0; i < R; ++i) decision[i] = d.worker_of_sample[i];
    if (rep) copy_report(r, s->cfg.n, rep);
    if (times_s) {
      times_s[0] = std::chrono::duration<double>(t1 - t0).count();
      times_s[1] = std::chrono::duration<double>(t2 - t1).count();
      times_s[2] = std::chrono::duration<double>(t3 - t2).count();
      times_s[3] = std::chrono::duration<double>(t4 - t3).count();
    }
  });
}

}  // extern "C"

// report_io.hpp over POD copies of IterationReport / RunSummary.
namespace {
void put_string(const std::string& s, char* out, uint64_t cap, uint64_t* len) {
  *len = s.size();
  if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
}
}  // namespace

int orc_report_jsonl(const orc_iter_report* r, char* out, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    IterationReport rep;
    rep.iteration = r->iteration;
    rep.mechanism = r->mechanism;
    rep.miss_pull = r->miss_pull;
    rep.update_push = r->update_push;
    rep.evict_push = r->evict_push;
    rep.hits = r->hits;
    rep.lookups = r->lookups;
    rep.cost_s = r->cost_s;
    rep.decision_s = r->decision_s;
    rep.matrix_s = r->matrix_s;
    rep.expected_cost_s = r->expected_cost_s;
    rep.has_expected = r->has_expected != 0;
    rep.miss_pull_w.assign(r->miss_pull_w, r->miss_pull_w + r->n);
    rep.update_push_w.assign(r->update_push_w, r->update_push_w + r->n);
    rep.evict_push_w.assign(r->evict_push_w, r->evict_push_w + r->n);
    rep.cost_w.assign(r->cost_w, r->cost_w + r->n);
    put_string(report_jsonl(rep), out, cap, len);
  });
}

int orc_comparison_csv(const orc_run_summary* runs, uint64_t count, const char* reference,
                       const orc_cluster_config* c, char* out, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    std::vector<RunResult> results(count);
    for (uint64_t k = 0; k < count; ++k) {
      const orc_run_summary& r = runs[k];
      RunSummary& s = results[k].summary;
      s.mechanism = r.mechanism;
      s.iterations = r.iterations;
      s.measured_iterations = r.measured_iterations;
      s.miss_pull = r.miss_pull;
      s.update_push = r.update_push;
      s.evict_push = r.evict_push;
      s.hits = r.hits;
      s.lookups = r.lookups;
      s.cost_s = r.cost_s;
      s.expected_cost_s = r.expected_cost_s;
      s.has_expected = r.has_expected != 0;
      s.decision_s_total = r.decision_s_total;
      s.decision_s_max = r.decision_s_max;
      s.matrix_s_total = r.matrix_s_total;
      s.budget_violations = r.budget_violations;
      s.miss_pull_w.assign(r.miss_pull_w, r.miss_pull_w + r.n);
      s.update_push_w.assign(r.update_push_w, r.update_push_w + r.n);
      s.evict_push_w.assign(r.evict_push_w, r.evict_push_w + r.n);
      s.ops_w.assign(r.ops_w, r.ops_w + r.n);
    }
    put_string(comparison_csv(results, reference, to_cfg(c)), out, cap, len);
  });
}

/* TraceStream / load_schema (workload.hpp:152-268) through the reference:
 * "iterations I dropped D max M\n", one line per kept sample, then the
 * warning text the reference wrote. */
int orc_trace_dump(const char* path, const char* schema_path, int32_t n, int32_t m,
                   uint64_t capacity, char* out, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    ClusterConfig cfg;
    cfg.n = n;
    cfg.m = m;
    cfg.cache_capacity = capacity;
    TraceSchema schema;
    if (schema_path) schema = load_schema(schema_path);
    std::ostringstream warn;
    TraceStream ts(path, cfg, schema_path ? &schema : nullptr, &warn);
    std::ostringstream os;
    os << "iterations " << ts.iterations() << " dropped " << ts.dropped_samples() << " max "
       << ts.max_sample_len() << "\n";
    std::vector<EmbeddingSample> batch;
    while (ts.next_iteration(batch))
      for (const auto& smp : batch) {
        for (std::size_t i = 0; i < smp.ids.size(); ++i) os << (i ? " " : "") << smp.ids[i];
        os << "\n";
      }
    os << warn.str();
    put_string(os.str(), out, cap, len);
  });
}
