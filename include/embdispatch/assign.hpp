// Drop-in for the reference's assign.hpp hot path: the exact solver, the
// capacity-bounded greedy, the gap order and the EcoMix hybrid, all executed
// by libedx kernels (hungarian.cu, dispatch.cu), and the hit-greedy baseline
// (hitgreedy.cu).  The random / round-robin controls are data-free host code.
#pragma once

#include <algorithm>
#include <cmath>
#include <numeric>
#include <ostream>
#include <random>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "embdispatch/cost.hpp"

namespace embdispatch {

// assign.hpp:38-58.
struct DispatchDecision {
  std::vector<WorkerId> worker_of_sample;

  void validate(const ClusterConfig& cfg) const {
    if (worker_of_sample.size() != cfg.samples_per_iteration())
      throw std::invalid_argument("decision does not cover m*n samples");
    std::vector<int> load(static_cast<std::size_t>(cfg.n), 0);
    for (WorkerId w : worker_of_sample) {
      if (w < 0 || w >= cfg.n) throw std::invalid_argument("worker id out of range");
      ++load[static_cast<std::size_t>(w)];
    }
    for (WorkerId j = 0; j < cfg.n; ++j)
      if (load[static_cast<std::size_t>(j)] != cfg.m)
        throw std::invalid_argument("worker " + std::to_string(j) + " received " +
                                    std::to_string(load[static_cast<std::size_t>(j)]) +
                                    " samples, expected " + std::to_string(cfg.m));
  }
};

// assign.hpp:62-68.
struct SquareCost {
  std::size_t order = 0;
  std::vector<double> values;
  std::vector<WorkerId> col_to_worker;
  double at(std::size_t r, std::size_t c) const { return values[r * order + c]; }
};

struct AssignmentResult {
  std::vector<std::size_t> col_of_row;
  double total_cost = 0.0;
};

// assign.hpp:80-157 (edx_hungarian: K5 dense e-maxx on the device).
inline AssignmentResult hungarian(const SquareCost& sq) {
  if (sq.order < 1) throw std::invalid_argument("solver needs at least one row");
  if (sq.values.size() != sq.order * sq.order) throw std::invalid_argument("cost matrix must be square");
  AssignmentResult r;
  std::vector<uint64_t> cols(sq.order);
  edxc::check(edx_hungarian(sq.order, sq.values.data(), cols.data(), &r.total_cost));
  r.col_of_row.assign(cols.begin(), cols.end());
  return r;
}

// assign.hpp:162-192 (edx_greedy_dispatch: K4 rounds kernel).
inline std::vector<std::pair<std::size_t, WorkerId>> greedy_dispatch(
    const CostMatrix& matrix, const std::vector<std::size_t>& rows, std::vector<int> capacity) {
  if (capacity.size() != matrix.cols) throw std::invalid_argument("need one capacity per worker");
  std::vector<uint64_t> order(rows.begin(), rows.end()), out_rows(rows.size());
  std::vector<int32_t> cap(capacity.begin(), capacity.end()), out_w(rows.size());
  edxc::check(edx_greedy_dispatch(matrix.rows, matrix.cols, matrix.values.data(), order.data(),
                                  order.size(), cap.data(), out_rows.data(), out_w.data()));
  std::vector<std::pair<std::size_t, WorkerId>> part(rows.size());
  for (std::size_t t = 0; t < rows.size(); ++t) part[t] = {out_rows[t], out_w[t]};
  return part;
}

// assign.hpp:197-207 (gap keys + stable radix sort on the device).
inline std::vector<std::size_t> rows_by_gap(const CostMatrix& matrix) {
  std::vector<uint64_t> order(matrix.rows);
  edxc::check(edx_rows_by_gap(matrix.rows, matrix.cols, matrix.values.data(), order.data()));
  return std::vector<std::size_t>(order.begin(), order.end());
}

namespace detail {
// assign.hpp:213-216.
inline int exact_multiplicity(int m, double alpha) {
  return std::clamp(static_cast<int>(std::floor(m * alpha + 1e-9)), 0, m);
}
}  // namespace detail

// assign.hpp:223-241.  Materialised on the host only for callers that want
// the square matrix; ecomix never builds it (the device solver is collapsed).
inline SquareCost expand_columns(const CostMatrix& matrix, const std::vector<std::size_t>& rows,
                                 int mult) {
  SquareCost sq;
  sq.order = rows.size();
  if (sq.order != matrix.cols * static_cast<std::size_t>(mult))
    throw std::invalid_argument("row count must equal cols * multiplicity");
  sq.col_to_worker.resize(sq.order);
  for (std::size_t c = 0; c < sq.order; ++c)
    sq.col_to_worker[c] = static_cast<WorkerId>(c / static_cast<std::size_t>(mult));
  sq.values.resize(sq.order * sq.order);
  for (std::size_t r = 0; r < sq.order; ++r)
    for (std::size_t c = 0; c < sq.order; ++c)
      sq.values[r * sq.order + c] = matrix.at(rows[r], static_cast<std::size_t>(sq.col_to_worker[c]));
  return sq;
}

// assign.hpp:247-285 (edx_ecomix: gap sort, collapsed Hungarian, greedy).
inline DispatchDecision ecomix(const CostMatrix& matrix, const ClusterConfig& cfg) {
  DispatchDecision d;
  d.worker_of_sample.resize(matrix.rows);
  std::vector<uint64_t> rid(matrix.row_ids.begin(), matrix.row_ids.end());
  std::vector<int32_t> dec(matrix.rows);
  const edx_cluster_config c = edxc::to_c(cfg);
  edxc::check(edx_ecomix(&c, matrix.rows, matrix.cols, matrix.values.data(),
                         rid.empty() ? nullptr : rid.data(), dec.data()));
  d.worker_of_sample.assign(dec.begin(), dec.end());
  return d;
}

// assign.hpp:346-392 (edx_hitgreedy / edx_engine_dispatch_hitgreedy): the
// relevance-score baseline on the snapshot -- the live device state when the
// snapshot is the engine's current one.
inline DispatchDecision baseline_hitgreedy(const std::vector<EmbeddingSample>& samples,
                                           const Snapshot& snap, const ClusterConfig& cfg) {
  if (samples.size() != cfg.samples_per_iteration())
    throw std::invalid_argument("sample count must be m*n");
  std::vector<int32_t> dec(samples.size());
  const edxc::Csr csr(samples);
  if (edx_engine* e = snap.device_view()) {
    edxc::check(edx_engine_load_batch(e, csr.ids.data(), csr.offsets.data(), samples.size(), 0));
    edxc::check(edx_engine_dispatch_hitgreedy(e, dec.data()));
  } else {
    const edxc::SnapArrays a(snap);
    const edx_cluster_config c = edxc::to_c(cfg);
    edxc::check(edx_hitgreedy(&c, a.ids.data(), a.owners.data(), a.latest.data(), a.ids.size(),
                              csr.ids.data(), csr.offsets.data(), samples.size(), dec.data()));
  }
  DispatchDecision d;
  d.worker_of_sample.assign(dec.begin(), dec.end());
  return d;
}

// assign.hpp:300-326: the random control -- a uniformly random balanced
// assignment.  Data-free host code (no state, no matrix): sample perm[p]
// goes to worker p / m, perm from an explicit Fisher-Yates pass over
// std::mt19937_64(seed) (draw j = rng() % (i + 1) for i = R-1 .. 1), so the
// decisions replay bit-identically from the seed.
inline DispatchDecision baseline_random(std::size_t sample_count, const ClusterConfig& cfg,
                                        std::uint64_t seed) {
  if (sample_count != cfg.samples_per_iteration())
    throw std::invalid_argument("sample count must be m*n");
  std::vector<std::size_t> perm(sample_count);
  std::iota(perm.begin(), perm.end(), std::size_t{0});
  std::mt19937_64 rng(seed);
  for (std::size_t i = sample_count; i-- > 1;)
    std::swap(perm[i], perm[static_cast<std::size_t>(rng() % (i + 1))]);
  DispatchDecision d;
  d.worker_of_sample.assign(sample_count, -1);
  const std::size_t m = static_cast<std::size_t>(cfg.m);
  for (std::size_t p = 0; p < sample_count; ++p)
    d.worker_of_sample[perm[p]] = static_cast<WorkerId>(p / m);
  d.validate(cfg);
  return d;
}

// assign.hpp:329-341: the round-robin control, sample i to worker i mod n.
inline DispatchDecision baseline_roundrobin(std::size_t sample_count, const ClusterConfig& cfg) {
  if (sample_count != cfg.samples_per_iteration())
    throw std::invalid_argument("sample count must be m*n");
  DispatchDecision d;
  d.worker_of_sample.resize(sample_count);
  for (std::size_t i = 0; i < sample_count; ++i)
    d.worker_of_sample[i] = static_cast<WorkerId>(i % static_cast<std::size_t>(cfg.n));
  d.validate(cfg);
  return d;
}

// assign.hpp:288-298.
inline double decision_cost(const CostMatrix& matrix, const DispatchDecision& decision) {
  if (decision.worker_of_sample.size() != matrix.rows)
    throw std::invalid_argument("decision and matrix disagree on sample count");
  std::vector<int32_t> dec(decision.worker_of_sample.begin(), decision.worker_of_sample.end());
  double out = 0.0;
  edxc::check(edx_decision_cost(matrix.rows, matrix.cols, matrix.values.data(), dec.data(), &out));
  return out;
}

// assign.hpp:396-403.
inline void write_decision(std::ostream& os, const DispatchDecision& decision,
                           double total_expected_cost) {
  for (std::size_t i = 0; i < decision.worker_of_sample.size(); ++i)
    os << i << ' ' << decision.worker_of_sample[i] << '\n';
  os << "total_expected_cost " << detail::format_double(total_expected_cost) << '\n';
}

}  // namespace embdispatch
