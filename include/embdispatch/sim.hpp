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
// hash maps on demand).  id_space > 0 selects the dense fast path (every id
// < id_space, tables indexed by id); 0 (the default, or EDX_ID_SPACE) accepts
// any uint32 id through the device's open-addressing id table, which grows as
// new ids arrive.  max_batch_ids bounds one iteration's id stream (0 = env
// EDX_MAX_BATCH_IDS or 2^20; run() sizes it from the stream).
struct EngineOptions {
  int device = 0;
  std::uint64_t id_space = 0;
  std::uint64_t max_batch_ids = 0;
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
    o.id_space = opt.id_space ? opt.id_space : edxc::env_or("EDX_ID_SPACE", 0);
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

  // sim.hpp:71-82.  The reference copies the whole global map; here the
  // Snapshot is a view of the device state (nothing is copied unless the
  // caller reads `states` / `resident_ids`), and build_matrix /
  // baseline_hitgreedy read the device tables directly while it is current.
  Snapshot snapshot() const { return Snapshot::of_engine(e_, cfg_.n); }
  Snapshot device_snapshot() const { return snapshot(); }

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

// sim.hpp:271-318.  EcoMix and the hit-greedy baseline run on the device;
// random and round-robin are the data-free controls (host, assign.hpp).
struct Mechanism {
  enum class Kind { kEcoMix, kRandom, kRoundRobin, kHitGreedy };
  Kind kind = Kind::kEcoMix;
  double alpha = 1.0;

  std::string name() const {
    switch (kind) {
      case Kind::kRandom: return "random";
      case Kind::kRoundRobin: return "roundrobin";
      case Kind::kHitGreedy: return "hitgreedy";
      case Kind::kEcoMix: break;
    }
    return "ecomix:" + detail::format_double(alpha);
  }
  bool needs_snapshot() const { return kind == Kind::kEcoMix || kind == Kind::kHitGreedy; }
  bool needs_matrix() const { return kind == Kind::kEcoMix; }

  // "ecomix:<alpha>", "ecomix", "random", "roundrobin", "hitgreedy"
  static Mechanism parse(const std::string& text) {
    Mechanism mech;
    if (text == "random") {
      mech.kind = Kind::kRandom;
    } else if (text == "roundrobin") {
      mech.kind = Kind::kRoundRobin;
    } else if (text == "hitgreedy") {
      mech.kind = Kind::kHitGreedy;
    } else if (text == "ecomix" || text.rfind("ecomix:", 0) == 0) {
      if (text.size() > 7) {
        try {
          mech.alpha = std::stod(text.substr(7));
        } catch (const std::exception&) {
          throw std::invalid_argument("bad alpha in mechanism '" + text + "'");
        }
      }
      if (mech.alpha < 0.0 || mech.alpha > 1.0) throw std::invalid_argument("alpha must lie in [0, 1]");
    } else {
      throw std::invalid_argument("unknown mechanism '" + text + "'");
    }
    return mech;
  }
};

namespace detail {
// sim.hpp:360-366: the random baseline's per-iteration seed (one splitmix64
// step of seed ^ iteration * golden ratio).
inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t iteration) {
  std::uint64_t z = (seed ^ (iteration * 0x9e3779b97f4a7c15ull)) + 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
}  // namespace detail

// sim.hpp:373-395: one decision of `mech`.  The matrix is read only by
// EcoMix, the snapshot only by the snapshot-aware mechanisms.
inline DispatchDecision dispatch_with(const Mechanism& mech,
                                      const std::vector<EmbeddingSample>& samples,
                                      const Snapshot& snap, const CostMatrix& matrix,
                                      const ClusterConfig& cfg, std::uint64_t iteration,
                                      std::uint64_t random_seed) {
  switch (mech.kind) {
    case Mechanism::Kind::kEcoMix: {
      ClusterConfig tuned = cfg;
      tuned.alpha = mech.alpha;
      return ecomix(matrix, tuned);
    }
    case Mechanism::Kind::kRandom:
      return baseline_random(samples.size(), cfg, detail::mix_seed(random_seed, iteration));
    case Mechanism::Kind::kRoundRobin:
      return baseline_roundrobin(samples.size(), cfg);
    case Mechanism::Kind::kHitGreedy:
      return baseline_hitgreedy(samples, snap, cfg);
  }
  throw std::logic_error("unreachable");
}

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

// sim.hpp:400-478 on the engine: build (matrix_s, synchronised), dispatch
// (decision_s), device step, decision_cost; summaries accumulated in the
// reference's order.
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
  if (!eopt.max_batch_ids) eopt.max_batch_ids = cfg.samples_per_iteration() * stream.max_sample_len();
  if (!eopt.id_space)  // a Zipf stream's ids are dense: the direct-indexed fast path
    if (const auto* z = dynamic_cast<const ZipfStream*>(&stream)) eopt.id_space = z->spec().total_embeddings;
  ClusterConfig tuned = cfg;
  if (mech.kind == Mechanism::Kind::kEcoMix) tuned.alpha = mech.alpha;
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
    // matrix_s: the build alone, synchronised (sim.hpp:423-425)
    double matrix_s = 0.0;
    if (hybrid) {
      const auto t0 = clk::now();
      edxc::check(edx_engine_build(e, nullptr));
      edxc::check(edx_engine_synchronize(e));
      matrix_s = std::chrono::duration<double>(clk::now() - t0).count();
    }
    // decision_s: the dispatcher alone, until its decision is on the host
    // (sim.hpp:428-432); decision_cost runs on a side stream outside it
    std::vector<int32_t> dec(samples.size());
    const auto t1 = clk::now();
    bool device_decision = true;
    switch (mech.kind) {
      case Mechanism::Kind::kEcoMix:
        edxc::check(edx_engine_dispatch(e, mech.alpha, dec.data(), nullptr));
        break;
      case Mechanism::Kind::kHitGreedy:
        edxc::check(edx_engine_dispatch_hitgreedy(e, dec.data()));
        break;
      default: {
        const DispatchDecision d = dispatch_with(mech, samples, Snapshot{}, CostMatrix{}, cfg,
                                                 iteration, opt.random_seed);
        dec.assign(d.worker_of_sample.begin(), d.worker_of_sample.end());
        device_decision = false;
      }
    }
    const double decision_s = std::chrono::duration<double>(clk::now() - t1).count();
    edxc::Report raw(cfg.n);
    edxc::check(edx_engine_step(e, device_decision ? nullptr : dec.data(), &raw.c));
    IterationReport rep = raw.to_report();
    rep.mechanism = mech.name();
    rep.matrix_s = matrix_s;
    rep.decision_s = decision_s;
    if (hybrid) {  // decision_cost (sim.hpp:437-440), computed beside the step
      edxc::check(edx_engine_expected_cost(e, &rep.expected_cost_s));
      rep.has_expected = true;
    }
    if (opt.validate_state) state.validate_consistency();
    if (iteration >= opt.warmup) {
      ++s.measured_iterations;
      s.miss_pull += rep.miss_pull;
      s.update_push += rep.update_push;
      s.evict_push += rep.evict_push;
      s.hits += rep.hits;
      s.lookups += rep.lookups;
      s.cost_s += rep.cost_s;
      if (rep.has_expected) {
        s.expected_cost_s += rep.expected_cost_s;
        s.has_expected = true;
      }
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
