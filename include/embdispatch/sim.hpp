// Drop-in for the reference's sim.hpp: IterationReport, SimState and the
// run() loop for the EcoMix mechanism.  SimState owns an edx_engine: the
// global per-embedding state and every worker's cache stay resident on the
// GPU, step() is the device cache update (libedx step.cu), and
// snapshot()/cache()/state_of() materialise host copies for callers that
// inspect them.  run() drives the engine directly (no host snapshot, no
// matrix round trip), timing the reference's regions (sim.hpp:423-432).
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "embdispatch/assign.hpp"
#include "embdispatch/cache.hpp"
#include "embdispatch/cost.hpp"
#include "embdispatch/workload.hpp"

namespace embdispatch {

// sim.hpp:38-50.
struct IterationReport {
  std::size_t iteration = 0;
  std::string mechanism;
  std::vector<std::uint64_t> miss_pull_w, update_push_w, evict_push_w;
  std::vector<double> cost_w;
  std::uint64_t miss_pull = 0, update_push = 0, evict_push = 0;
  double cost_s = 0.0;
  std::uint64_t hits = 0, lookups = 0;
  double decision_s = 0.0;
  double matrix_s = 0.0;
  double expected_cost_s = 0.0;
  bool has_expected = false;
};

// Device sizing of a SimState (no reference counterpart: the reference grows
// hash maps on demand).  Defaults can be overridden with EDX_ID_SPACE /
// EDX_MAX_BATCH_IDS.
struct EngineOptions {
  int device = 0;
  std::uint64_t id_space = 0;       // ids must be < id_space; 0 = env or 2^20
  std::uint64_t max_batch_ids = 0;  // ids per iteration; 0 = env or 2^20
};

namespace edxc {
inline std::uint64_t env_or(const char* name, std::uint64_t dflt) {
  const char* v = std::getenv(name);
  return v ? std::strtoull(v, nullptr, 10) : dflt;
}

struct Report {
  std::vector<uint64_t> mp, up, ep;
  std::vector<double> cw;
  edx_report c{};
  explicit Report(int n) : mp(n), up(n), ep(n), cw(n) {
    c.miss_pull_w = mp.data();
    c.update_push_w = up.data();
    c.evict_push_w = ep.data();
    c.cost_w = cw.data();
  }
  IterationReport to_report() const {
    IterationReport r;
    r.iteration = c.iteration;
    r.miss_pull_w = mp;
    r.update_push_w = up;
    r.evict_push_w = ep;
    r.cost_w = cw;
    r.miss_pull = c.miss_pull;
    r.update_push = c.update_push;
    r.evict_push = c.evict_push;
    r.cost_s = c.cost_s;
    r.hits = c.hits;
    r.lookups = c.lookups;
    return r;
  }
};
}  // namespace edxc

// sim.hpp:54-268.
class SimState {
 public:
  explicit SimState(const ClusterConfig& cfg, EngineOptions opt = {}) : cfg_(cfg) {
    edx_engine_options o{};
    o.device = opt.device;
    o.id_space = opt.id_space ? opt.id_space : edxc::env_or("EDX_ID_SPACE", 1ULL << 20);
    o.max_batch_ids = opt.max_batch_ids ? opt.max_batch_ids : edxc::env_or("EDX_MAX_BATCH_IDS", 1ULL << 20);
    o.world_size = 1;
    const edx_cluster_config c = edxc::to_c(cfg_);
    edxc::check(edx_engine_create(&c, &o, &e_));
  }
  SimState(const SimState&) = delete;
  SimState& operator=(const SimState&) = delete;
  SimState(SimState&& o) noexcept : cfg_(std::move(o.cfg_)), e_(o.e_) { o.e_ = nullptr; }
  ~SimState() { edx_engine_destroy(e_); }

  const ClusterConfig& config() const { return cfg_; }
  std::uint64_t clock() const { return edx_engine_clock(e_); }
  edx_engine* engine() const { return e_; }

  EmbeddingState state_of(EmbeddingId id) const {
    EmbeddingState st;
    edxc::check(edx_engine_state_of(e_, id, &st.owners, &st.latest, &st.resident));
    return st;
  }

  // A host copy of one worker's cache (read-only view).
  const WorkerCache& cache(WorkerId j) const {
    if (j < 0 || j >= cfg_.n) throw std::out_of_range("worker out of range");
    uint64_t size = 0;
    edxc::check(edx_engine_cache_size(e_, j, &size));
    std::vector<uint32_t> ids(size), mark(size), freq(size);
    std::vector<uint8_t> ver(size);
    std::vector<uint64_t> last(size);
    edxc::check(edx_engine_export_cache(e_, j, ids.data(), ver.data(), mark.data(), freq.data(),
                                        last.data()));
    uint32_t cur = 1;
    uint64_t at = 0;
    edxc::check(edx_engine_cache_marks(e_, j, &cur, &at));
    std::unordered_map<EmbeddingId, CacheEntry> entries;
    for (uint64_t t = 0; t < size; ++t)
      entries[ids[t]] = CacheEntry{ids[t], ver[t] != 0, mark[t], freq[t], last[t]};
    views_.resize(static_cast<std::size_t>(cfg_.n));
    views_[static_cast<std::size_t>(j)] = WorkerCache(cfg_.cache_capacity, cur, std::move(entries));
    return views_[static_cast<std::size_t>(j)];
  }

  // sim.hpp:71-82: the full state as a host Snapshot, tagged with the engine
  // so that build_matrix can use the live device state instead.
  Snapshot snapshot() const {
    Snapshot s = device_snapshot();
    uint64_t count = 0;
    edxc::check(edx_engine_export_global(e_, nullptr, nullptr, nullptr, nullptr, 0, &count));
    std::vector<uint32_t> ids(count);
    std::vector<uint64_t> ow(count), la(count), re(count);
    edxc::check(edx_engine_export_global(e_, ids.data(), ow.data(), la.data(), re.data(), count,
                                         &count));
    s.resident_ids.resize(static_cast<std::size_t>(cfg_.n));
    for (uint64_t t = 0; t < count; ++t) {
      s.states[ids[t]] = EmbeddingState{ow[t], la[t], re[t]};
      for (WorkerMask r = re[t]; r; r &= r - 1)
        s.resident_ids[static_cast<std::size_t>(__builtin_ctzll(r))].push_back(ids[t]);
    }
    return s;
  }

  // Zero-copy: valid for build_matrix until the next step().
  Snapshot device_snapshot() const {
    Snapshot s;
    s.engine = e_;
    s.engine_clock = clock();
    return s;
  }

  // sim.hpp:87-218.
  IterationReport step(const std::vector<EmbeddingSample>& samples, const DispatchDecision& decision) {
    decision.validate(cfg_);
    if (samples.size() != cfg_.samples_per_iteration())
      throw std::invalid_argument("expected m*n samples");
    const edxc::Csr csr(samples);
    edxc::check(edx_engine_load_batch(e_, csr.ids.data(), csr.offsets.data(), samples.size(), 0));
    std::vector<int32_t> dec(decision.worker_of_sample.begin(), decision.worker_of_sample.end());
    edxc::Report rep(cfg_.n);
    edxc::check(edx_engine_step(e_, dec.data(), &rep.c));
    return rep.to_report();
  }

  // sim.hpp:222-248.
  void validate_consistency() const { edxc::check(edx_engine_validate_consistency(e_)); }

  // sim.hpp:252-261.
  void seed_entry(EmbeddingId id, WorkerId worker, bool latest, bool owner) {
    edxc::check(edx_engine_seed_entry(e_, id, worker, latest ? 1 : 0, owner ? 1 : 0));
  }

 private:
  ClusterConfig cfg_;
  edx_engine* e_ = nullptr;
  mutable std::vector<WorkerCache> views_;
};

// sim.hpp:271-318 for the mechanisms on the device path: EcoMix and the
// hit-greedy baseline (random / round-robin are outside it).
struct Mechanism {
  enum class Kind { kEcoMix, kHitGreedy };
  Kind kind = Kind::kEcoMix;
  double alpha = 1.0;
  std::string name() const {
    return kind == Kind::kHitGreedy ? std::string("hitgreedy") : "ecomix:" + detail::format_double(alpha);
  }
  bool needs_snapshot() const { return true; }
  bool needs_matrix() const { return kind == Kind::kEcoMix; }
  static Mechanism parse(const std::string& text) {
    Mechanism mech;
    if (text == "hitgreedy") {
      mech.kind = Kind::kHitGreedy;
      return mech;
    }
    if (text == "ecomix" || text.rfind("ecomix:", 0) == 0) {
      if (text.size() > 7) {
        try {
          mech.alpha = std::stod(text.substr(7));
        } catch (const std::exception&) {
          throw std::invalid_argument("bad alpha in mechanism '" + text + "'");
        }
      }
      if (mech.alpha < 0.0 || mech.alpha > 1.0) throw std::invalid_argument("alpha must lie in [0, 1]");
      return mech;
    }
    throw std::invalid_argument("unknown mechanism '" + text +
                                "' (the device path runs ecomix and hitgreedy)");
  }
};

struct RunOptions {
  std::size_t warmup = 10;
  double training_budget_s = 0.0;
  bool validate_state = false;
  std::uint64_t random_seed = 1;
};

struct RunSummary {
  std::string mechanism;
  std::size_t iterations = 0, measured_iterations = 0;
  std::uint64_t miss_pull = 0, update_push = 0, evict_push = 0, hits = 0, lookups = 0;
  double cost_s = 0.0, expected_cost_s = 0.0;
  bool has_expected = false;
  double decision_s_total = 0.0, decision_s_max = 0.0, matrix_s_total = 0.0;
  std::size_t budget_violations = 0;
  std::vector<std::uint64_t> miss_pull_w, update_push_w, evict_push_w, ops_w;
  double hit_ratio() const {
    return lookups == 0 ? 0.0 : static_cast<double>(hits) / static_cast<double>(lookups);
  }
  std::uint64_t ops_total() const { return miss_pull + update_push + evict_push; }
};

struct RunResult {
  Mechanism mechanism;
  std::vector<IterationReport> reports;
  RunSummary summary;
};

// sim.hpp:400-478 on the engine: build (matrix_s), dispatch (decision_s),
// device step, decision_cost; summaries accumulated in the reference's order.
inline RunResult run(SampleStream& stream, const Mechanism& mech, const ClusterConfig& cfg,
                     const RunOptions& opt, EngineOptions eopt = {}) {
  using clk = std::chrono::steady_clock;
  RunResult result;
  result.mechanism = mech;
  RunSummary& s = result.summary;
  s.mechanism = mech.name();
  s.miss_pull_w.assign(static_cast<std::size_t>(cfg.n), 0);
  s.update_push_w.assign(static_cast<std::size_t>(cfg.n), 0);
  s.evict_push_w.assign(static_cast<std::size_t>(cfg.n), 0);
  s.ops_w.assign(static_cast<std::size_t>(cfg.n), 0);
  ClusterConfig tuned = cfg;
  tuned.alpha = mech.alpha;
  if (!eopt.max_batch_ids) eopt.max_batch_ids = tuned.samples_per_iteration() * stream.max_sample_len();
  SimState state(tuned, eopt);
  edx_engine* e = state.engine();
  std::vector<EmbeddingSample> samples;
  std::size_t iteration = 0;
  while (stream.next_iteration(samples)) {
    if (samples.size() != cfg.samples_per_iteration())
      throw std::invalid_argument("stream underrun: iteration is short of samples");
    const edxc::Csr csr(samples);
    edxc::check(edx_engine_load_batch(e, csr.ids.data(), csr.offsets.data(), samples.size(), 0));
    const bool hybrid = mech.needs_matrix();
    const auto t0 = clk::now();
    if (hybrid) edxc::check(edx_engine_build(e, nullptr));
    const auto t1 = clk::now();
    double expected = 0.0;
    std::vector<int32_t> dec(samples.size());
    if (hybrid) edxc::check(edx_engine_dispatch(e, mech.alpha, dec.data(), &expected));
    else edxc::check(edx_engine_dispatch_hitgreedy(e, dec.data()));
    const auto t2 = clk::now();
    edxc::Report raw(cfg.n);
    edxc::check(edx_engine_step(e, nullptr, &raw.c));
    IterationReport rep = raw.to_report();
    rep.mechanism = mech.name();
    rep.matrix_s = hybrid ? std::chrono::duration<double>(t1 - t0).count() : 0.0;
    rep.decision_s = std::chrono::duration<double>(t2 - t1).count();
    rep.expected_cost_s = expected;
    rep.has_expected = hybrid;
    if (opt.validate_state) state.validate_consistency();
    if (iteration >= opt.warmup) {
      ++s.measured_iterations;
      s.miss_pull += rep.miss_pull;
      s.update_push += rep.update_push;
      s.evict_push += rep.evict_push;
      s.hits += rep.hits;
      s.lookups += rep.lookups;
      s.cost_s += rep.cost_s;
      s.expected_cost_s += rep.expected_cost_s;
      s.has_expected = hybrid;
      s.matrix_s_total += rep.matrix_s;
      for (std::size_t j = 0; j < static_cast<std::size_t>(cfg.n); ++j) {
        s.miss_pull_w[j] += rep.miss_pull_w[j];
        s.update_push_w[j] += rep.update_push_w[j];
        s.evict_push_w[j] += rep.evict_push_w[j];
        s.ops_w[j] += rep.miss_pull_w[j] + rep.update_push_w[j] + rep.evict_push_w[j];
      }
    }
    s.decision_s_total += rep.decision_s;
    s.decision_s_max = std::max(s.decision_s_max, rep.decision_s);
    if (opt.training_budget_s > 0.0 && rep.decision_s > opt.training_budget_s) ++s.budget_violations;
    result.reports.push_back(std::move(rep));
    ++iteration;
  }
  s.iterations = iteration;
  return result;
}

}  // namespace embdispatch
