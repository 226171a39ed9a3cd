// Drop-in for the reference's cost.hpp: Snapshot, CostMatrix, expected_cost,
// build_matrix, row_gap_key and the matrix text format.  The costs are built
// by the K1 kernel (libedx cost.cu), bit-identical to the reference's
// left-to-right fp64 chains.
#pragma once

#include <charconv>
#include <cmath>
#include <functional>
#include <istream>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "embdispatch/types.hpp"

namespace embdispatch {

namespace edxc {

using StateMap = std::unordered_map<EmbeddingId, EmbeddingState>;

// What a Snapshot taken from a device-backed SimState holds until something
// reads it: the engine and its state version (edx_engine_state_version).  The
// first read materialises the host copy from the device; a read after the
// engine's state has changed (step, seed_entry, import) throws instead of
// returning the newer state.
struct SnapPayload {
  edx_engine* engine = nullptr;
  std::uint64_t version = 0;
  int n = 0;
  bool ready = false;
  StateMap states;
  std::vector<std::vector<EmbeddingId>> resident_ids;

  void materialize() {
    if (ready) return;
    if (edx_engine_state_version(engine) != version)
      throw std::logic_error(
          "snapshot read after its SimState changed (step/seed_entry/import); read it before "
          "mutating the SimState");
    uint64_t count = 0;
    check(edx_engine_export_global(engine, nullptr, nullptr, nullptr, nullptr, 0, &count));
    std::vector<uint32_t> ids(count);
    std::vector<uint64_t> ow(count), la(count), re(count);
    check(edx_engine_export_global(engine, ids.data(), ow.data(), la.data(), re.data(), count,
                                   &count));
    states.reserve(count);
    resident_ids.assign(static_cast<std::size_t>(n), {});
    for (uint64_t t = 0; t < count; ++t) {
      states[ids[t]] = EmbeddingState{ow[t], la[t], re[t]};
      for (WorkerMask r = re[t]; r; r &= r - 1)
        resident_ids[static_cast<std::size_t>(__builtin_ctzll(r))].push_back(ids[t]);
    }
    ready = true;
  }
};

}  // namespace edxc

// Snapshot::states (cost.hpp:40): a host map, or -- in a snapshot from
// SimState::snapshot() -- a view of the live device state that is copied to
// the host only when read.  Reads keep the view current for build_matrix's
// device path; a non-const access detaches it into a plain host map (which
// build_matrix then uploads, as the reference's Snapshot is a value copy).
class SnapshotStates {
 public:
  using map_type = edxc::StateMap;
  using iterator = map_type::iterator;
  using const_iterator = map_type::const_iterator;
  using value_type = map_type::value_type;
  using key_type = map_type::key_type;
  using mapped_type = map_type::mapped_type;
  using size_type = map_type::size_type;

  SnapshotStates() = default;
  SnapshotStates(const map_type& m) : own_(m) {}
  SnapshotStates& operator=(const map_type& m) {
    view_.reset();
    own_ = m;
    return *this;
  }
  explicit SnapshotStates(std::shared_ptr<edxc::SnapPayload> v) : view_(std::move(v)) {}

  const map_type& map() const {
    if (!view_) return own_;
    view_->materialize();
    return view_->states;
  }
  map_type& map() {
    if (view_) {
      view_->materialize();
      own_ = view_->states;
      view_.reset();
    }
    return own_;
  }
  operator const map_type&() const { return map(); }

  // the device view, while it is unread-or-const-read and current
  edx_engine* engine_view() const {
    return view_ && edx_engine_state_version(view_->engine) == view_->version ? view_->engine
                                                                              : nullptr;
  }
  bool is_view() const { return static_cast<bool>(view_); }

  EmbeddingState& operator[](EmbeddingId id) { return map()[id]; }
  EmbeddingState& at(EmbeddingId id) { return map().at(id); }
  const EmbeddingState& at(EmbeddingId id) const { return map().at(id); }
  const_iterator find(EmbeddingId id) const { return map().find(id); }
  iterator find(EmbeddingId id) { return map().find(id); }
  size_type count(EmbeddingId id) const { return map().count(id); }
  bool contains(EmbeddingId id) const { return map().count(id) != 0; }
  size_type size() const { return map().size(); }
  bool empty() const { return map().empty(); }
  const_iterator begin() const { return map().begin(); }
  const_iterator end() const { return map().end(); }
  const_iterator cbegin() const { return map().begin(); }
  const_iterator cend() const { return map().end(); }
  iterator begin() { return map().begin(); }
  iterator end() { return map().end(); }
  void clear() { map().clear(); }
  void reserve(size_type k) { map().reserve(k); }
  size_type erase(EmbeddingId id) { return map().erase(id); }
  template <class... A>
  std::pair<iterator, bool> emplace(A&&... a) { return map().emplace(std::forward<A>(a)...); }
  std::pair<iterator, bool> insert(const value_type& v) { return map().insert(v); }
  template <class... A>
  std::pair<iterator, bool> try_emplace(EmbeddingId id, A&&... a) {
    return map().try_emplace(id, std::forward<A>(a)...);
  }

 private:
  std::shared_ptr<edxc::SnapPayload> view_;
  map_type own_;
};

// Snapshot::resident_ids (cost.hpp:41): the same lazy view (no consumer in
// the reference reads it; it is materialised only on access).
class SnapshotResidents {
 public:
  using vec_type = std::vector<std::vector<EmbeddingId>>;
  SnapshotResidents() = default;
  SnapshotResidents(const vec_type& v) : own_(v) {}
  SnapshotResidents& operator=(const vec_type& v) {
    view_.reset();
    own_ = v;
    return *this;
  }
  explicit SnapshotResidents(std::shared_ptr<edxc::SnapPayload> v) : view_(std::move(v)) {}
  const vec_type& vec() const {
    if (!view_) return own_;
    view_->materialize();
    return view_->resident_ids;
  }
  vec_type& vec() {
    if (view_) {
      view_->materialize();
      own_ = view_->resident_ids;
      view_.reset();
    }
    return own_;
  }
  operator const vec_type&() const { return vec(); }
  const std::vector<EmbeddingId>& operator[](std::size_t j) const { return vec()[j]; }
  std::vector<EmbeddingId>& operator[](std::size_t j) { return vec()[j]; }
  std::size_t size() const { return vec().size(); }
  bool empty() const { return vec().empty(); }
  void resize(std::size_t k) { vec().resize(k); }
  vec_type::const_iterator begin() const { return vec().begin(); }
  vec_type::const_iterator end() const { return vec().end(); }

 private:
  std::shared_ptr<edxc::SnapPayload> view_;
  vec_type own_;
};

// cost.hpp:39-48.  A default Snapshot is a host value as in the reference;
// SimState::snapshot() returns a lazy device view (see SnapshotStates).
struct Snapshot {
  SnapshotStates states;
  SnapshotResidents resident_ids;

  EmbeddingState state_of(EmbeddingId id) const {
    auto it = states.find(id);
    return it == states.end() ? EmbeddingState{} : it->second;
  }
  // The engine whose current state this snapshot still views (build_matrix
  // and baseline_hitgreedy then read the device directly), else nullptr.
  edx_engine* device_view() const { return states.engine_view(); }

  static Snapshot of_engine(edx_engine* e, int n) {
    auto p = std::make_shared<edxc::SnapPayload>();
    p->engine = e;
    p->version = edx_engine_state_version(e);
    p->n = n;
    Snapshot s;
    s.states = SnapshotStates(p);
    s.resident_ids = SnapshotResidents(p);
    return s;
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
  if (edx_engine* e = snap.device_view(); e && !size_of) {
    edxc::check(edx_engine_load_batch(e, csr.ids.data(), csr.offsets.data(), m.rows, 0));
    edxc::check(edx_engine_build(e, m.values.data()));
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
