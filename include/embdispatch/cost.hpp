// Drop-in for the reference's cost.hpp: Snapshot, CostMatrix, expected_cost,
// build_matrix, row_gap_key and the matrix text format.  The costs are built
// by the K1 kernel (libedx cost.cu), bit-identical to the reference's
// left-to-right fp64 chains.
#pragma once

#include <charconv>
#include <cmath>
#include <functional>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "embdispatch/types.hpp"

namespace embdispatch {

// cost.hpp:39-48.  `engine`/`engine_clock` are an addition: a snapshot taken
// from a device-backed SimState remembers it, and build_matrix reads the live
// device state directly while that state is unchanged (no upload).
struct Snapshot {
  std::unordered_map<EmbeddingId, EmbeddingState> states;
  std::vector<std::vector<EmbeddingId>> resident_ids;
  edx_engine* engine = nullptr;
  std::uint64_t engine_clock = 0;

  EmbeddingState state_of(EmbeddingId id) const {
    auto it = states.find(id);
    return it == states.end() ? EmbeddingState{} : it->second;
  }
};

// cost.hpp:52-60.
struct CostMatrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<double> values;
  std::vector<std::size_t> row_ids;
  double at(std::size_t r, std::size_t c) const { return values[r * cols + c]; }
  double& at(std::size_t r, std::size_t c) { return values[r * cols + c]; }
};

// cost.hpp:64.  Optional per-embedding transfer size in bytes; the device
// build evaluates it once per id position and charges bytes * 8.0 / bw_j
// (cost.hpp:68-73) for each add.
using SizeLookupFn = std::function<std::uint64_t(EmbeddingId)>;

namespace edxc {

struct SnapArrays {
  std::vector<uint32_t> ids;
  std::vector<uint64_t> owners, latest, resident;
  explicit SnapArrays(const Snapshot& s) {
    if (s.engine && s.states.empty()) {  // a device view: read the live state back
      uint64_t count = 0;
      check(edx_engine_export_global(s.engine, nullptr, nullptr, nullptr, nullptr, 0, &count));
      ids.resize(count);
      owners.resize(count);
      latest.resize(count);
      resident.resize(count);
      check(edx_engine_export_global(s.engine, ids.data(), owners.data(), latest.data(),
                                     resident.data(), count, &count));
      return;
    }
    ids.reserve(s.states.size());
    for (const auto& [id, st] : s.states) {
      ids.push_back(id);
      owners.push_back(st.owners);
      latest.push_back(st.latest);
      resident.push_back(st.resident);
    }
  }
};

struct Csr {
  std::vector<uint32_t> ids;
  std::vector<uint64_t> offsets{0};
  explicit Csr(const std::vector<EmbeddingSample>& samples) {
    for (const auto& s : samples) {
      ids.insert(ids.end(), s.ids.begin(), s.ids.end());
      offsets.push_back(ids.size());
    }
  }
};

inline std::vector<uint64_t> sizes_of(const std::vector<uint32_t>& ids, const SizeLookupFn& f) {
  std::vector<uint64_t> out(ids.size());
  for (std::size_t t = 0; t < ids.size(); ++t) out[t] = f(ids[t]);
  return out;
}

}  // namespace edxc

// cost.hpp:81-100 — one cell.
inline double expected_cost(const EmbeddingSample& sample, WorkerId worker, const Snapshot& snap,
                            const ClusterConfig& cfg, const SizeLookupFn& size_of = nullptr) {
  if (worker < 0 || worker >= cfg.n) throw std::invalid_argument("worker id out of range");
  const edxc::SnapArrays a(snap);
  const uint64_t off[2] = {0, sample.ids.size()};
  std::vector<double> row(static_cast<std::size_t>(cfg.n));
  const edx_cluster_config c = edxc::to_c(cfg);
  if (size_of) {
    const auto sz = edxc::sizes_of(sample.ids, size_of);
    edxc::check(edx_expected_costs_sized(&c, a.ids.data(), a.owners.data(), a.latest.data(),
                                         a.ids.size(), sample.ids.data(), off, 1, sz.data(),
                                         row.data()));
  } else {
    edxc::check(edx_expected_costs(&c, a.ids.data(), a.owners.data(), a.latest.data(),
                                   a.ids.size(), sample.ids.data(), off, 1, row.data()));
  }
  return row[static_cast<std::size_t>(worker)];
}

// cost.hpp:105-125.
inline CostMatrix build_matrix(const std::vector<EmbeddingSample>& samples, const Snapshot& snap,
                               const ClusterConfig& cfg, const SizeLookupFn& size_of = nullptr) {
  if (samples.size() != cfg.samples_per_iteration())
    throw std::invalid_argument("expected " + std::to_string(cfg.samples_per_iteration()) +
                                " samples, got " + std::to_string(samples.size()));
  CostMatrix m;
  m.rows = samples.size();
  m.cols = static_cast<std::size_t>(cfg.n);
  m.values.resize(m.rows * m.cols);
  m.row_ids.resize(m.rows);
  for (std::size_t i = 0; i < m.rows; ++i) m.row_ids[i] = i;
  const edxc::Csr csr(samples);
  if (!size_of && snap.engine && edx_engine_clock(snap.engine) == snap.engine_clock) {
    edxc::check(edx_engine_load_batch(snap.engine, csr.ids.data(), csr.offsets.data(), m.rows, 0));
    edxc::check(edx_engine_build(snap.engine, m.values.data()));
    return m;
  }
  const edxc::SnapArrays a(snap);
  const edx_cluster_config c = edxc::to_c(cfg);
  if (size_of) {
    const auto sz = edxc::sizes_of(csr.ids, size_of);
    edxc::check(edx_build_matrix_sized(&c, a.ids.data(), a.owners.data(), a.latest.data(),
                                       a.ids.size(), csr.ids.data(), csr.offsets.data(), m.rows,
                                       sz.data(), m.values.data()));
    return m;
  }
  edxc::check(edx_build_matrix(&c, a.ids.data(), a.owners.data(), a.latest.data(),
                               a.resident.data(), a.ids.size(), csr.ids.data(), csr.offsets.data(),
                               m.rows, m.values.data()));
  return m;
}

// cost.hpp:130-146.
inline double row_gap_key(const CostMatrix& matrix, std::size_t row) {
  double out = 0.0;
  edxc::check(edx_row_gap_key(matrix.rows, matrix.cols, matrix.values.data(), row, &out));
  return out;
}

namespace detail {
inline std::string format_double(double v) {
  char buf[64];
  auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), v);
  if (ec != std::errc{}) throw std::runtime_error("failed to format double");
  return std::string(buf, ptr);
}
}  // namespace detail

// Plain-text matrix files (cost.hpp:162-195): header `rows cols`, then
// shortest-round-trip doubles.
inline void write_matrix(std::ostream& os, const CostMatrix& matrix) {
  os << matrix.rows << ' ' << matrix.cols << '\n';
  for (std::size_t r = 0; r < matrix.rows; ++r) {
    for (std::size_t c = 0; c < matrix.cols; ++c) os << (c ? " " : "") << detail::format_double(matrix.at(r, c));
    os << '\n';
  }
}

inline CostMatrix read_matrix(std::istream& is) {
  CostMatrix m;
  if (!(is >> m.rows >> m.cols)) throw std::runtime_error("matrix file: missing 'rows cols' header");
  if (m.rows == 0 || m.cols == 0) throw std::runtime_error("matrix file: dimensions must be positive");
  m.values.resize(m.rows * m.cols);
  for (std::size_t i = 0; i < m.values.size(); ++i) {
    if (!(is >> m.values[i]))
      throw std::runtime_error("matrix file: expected " + std::to_string(m.values.size()) +
                               " values, got " + std::to_string(i));
    if (!std::isfinite(m.values[i]) || m.values[i] < 0.0)
      throw std::runtime_error("matrix file: values must be finite and non-negative");
  }
  m.row_ids.resize(m.rows);
  for (std::size_t i = 0; i < m.rows; ++i) m.row_ids[i] = i;
  return m;
}

}  // namespace embdispatch
