// Drop-in for the reference's types.hpp (ids, samples, cluster config, unit
// costs, worker masks, per-embedding state).  Validation and unit costs run
// through libedx so the two sides can never disagree on a message or a bit.
#pragma once

#include <cstdint>
#include <string>
#include <unordered_set>
#include <vector>

#include "embdispatch/bridge.hpp"

namespace embdispatch {

using EmbeddingId = std::uint32_t;  // flat id over all tables (types.hpp:30)
using WorkerId = int;

// The ordered, duplicate-free ids one sample touches (types.hpp:37-42).
struct EmbeddingSample {
  std::vector<EmbeddingId> ids;
  bool empty() const { return ids.empty(); }
  std::size_t size() const { return ids.size(); }
};

// First occurrence wins; empty input is rejected (types.hpp:46-60).
inline EmbeddingSample make_sample(const std::vector<EmbeddingId>& raw_ids) {
  if (raw_ids.empty()) throw std::invalid_argument("embedding sample must contain at least one id");
  EmbeddingSample s;
  std::unordered_set<EmbeddingId> seen;
  for (EmbeddingId id : raw_ids)
    if (seen.insert(id).second) s.ids.push_back(id);
  return s;
}

struct TransmitCost {
  double seconds = 0.0;
};

// types.hpp:71-82.
struct ClusterConfig {
  int n = 8;
  int m = 128;
  std::vector<double> bandwidths_bps;
  std::uint64_t d_tran_bytes = 2048;
  std::size_t cache_capacity = 0;
  double alpha = 1.0;
  std::size_t samples_per_iteration() const {
    return static_cast<std::size_t>(n) * static_cast<std::size_t>(m);
  }
};

namespace edxc {
inline edx_cluster_config to_c(const ClusterConfig& c) {
  edx_cluster_config r{};
  r.n = c.n;
  r.m = c.m;
  r.bandwidths_bps = c.bandwidths_bps.data();
  r.n_bandwidths = static_cast<int32_t>(c.bandwidths_bps.size());
  r.d_tran_bytes = c.d_tran_bytes;
  r.cache_capacity = c.cache_capacity;
  r.alpha = c.alpha;
  return r;
}
}  // namespace edxc

// types.hpp:87-108 (edx_validate_config).
inline void validate(const ClusterConfig& cfg, std::size_t max_sample_len) {
  const edx_cluster_config c = edxc::to_c(cfg);
  edxc::check(edx_validate_config(&c, max_sample_len));
}

// types.hpp:112-120 (edx_unit_costs).
inline TransmitCost unit_cost(const ClusterConfig& cfg, WorkerId worker) {
  if (worker < 0 || worker >= cfg.n || static_cast<std::size_t>(worker) >= cfg.bandwidths_bps.size())
    throw std::invalid_argument("worker id " + std::to_string(worker) + " out of range");
  std::vector<double> u(static_cast<std::size_t>(cfg.n));
  const edx_cluster_config c = edxc::to_c(cfg);
  edxc::check(edx_unit_costs(&c, u.data()));
  return TransmitCost{u[static_cast<std::size_t>(worker)]};
}

using WorkerMask = std::uint64_t;  // n <= 64 (types.hpp:89,124)
inline WorkerMask worker_bit(WorkerId w) { return WorkerMask{1} << w; }
inline int mask_count(WorkerMask m) { return __builtin_popcountll(m); }
inline bool mask_has(WorkerMask m, WorkerId w) { return (m & worker_bit(w)) != 0; }

// types.hpp:139-156.
struct EmbeddingState {
  WorkerMask owners = 0;
  WorkerMask latest = 0;
  WorkerMask resident = 0;
  bool owned_by(WorkerId w) const { return mask_has(owners, w); }
  bool latest_on(WorkerId w) const { return mask_has(latest, w); }
  bool resident_on(WorkerId w) const { return mask_has(resident, w); }
  bool consistent() const {
    return (owners & ~latest) == 0 && (latest & ~resident) == 0 && !(owners != 0 && latest != owners);
  }
};

}  // namespace embdispatch
