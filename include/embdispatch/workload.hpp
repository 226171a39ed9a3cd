// Drop-in for the reference's synthetic input stream (workload.hpp:36-133):
// WorkloadSpec, SampleStream and ZipfStream over libedx's host generator
// (bit-identical ids), and trace ingestion (workload.hpp:137-300): TraceSchema,
// load_schema, TraceStream and write_trace, the file parsed by libedx into the
// engine's CSR batch layout (edx_trace_*).
#pragma once

#include <cstdint>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "embdispatch/types.hpp"

namespace embdispatch {

struct WorkloadSpec {
  std::size_t total_embeddings = 50000;
  std::size_t sample_len = 26;
  double zipf_s = 1.05;
  std::size_t iterations = 200;
  std::uint64_t seed = 42;
};

// workload.hpp:44-50 (same messages).
inline void validate(const WorkloadSpec& spec) {
  if (spec.sample_len < 1) throw std::invalid_argument("sample_len must be >= 1");
  if (!(spec.zipf_s > 0.0)) throw std::invalid_argument("zipf_s must be positive");
  if (spec.total_embeddings < spec.sample_len)
    throw std::invalid_argument("sample_len exceeds the embedding population");
}

// workload.hpp:54-79: ids in [0, n) with P(id) proportional to (id+1)^-s,
// inverse-CDF over std::mt19937_64(seed) -- the same draws, produced by
// libedx's guide-table sampler (workload.cpp) a block at a time.
class ZipfSampler {
 public:
  ZipfSampler(std::size_t n, double s, std::uint64_t seed) {
    edx_zipf* z = nullptr;
    edxc::check(edx_zipf_sampler_create(n, s, seed, &z));
    z_.reset(z);
  }
  EmbeddingId draw() {
    if (pos_ == buf_.size()) {
      buf_.resize(4096);
      edxc::check(edx_zipf_draw(z_.get(), buf_.size(), buf_.data()));
      pos_ = 0;
    }
    return buf_[pos_++];
  }

 private:
  struct Del {
    void operator()(edx_zipf* z) const { edx_zipf_destroy(z); }
  };
  std::unique_ptr<edx_zipf, Del> z_;
  std::vector<std::uint32_t> buf_;
  std::size_t pos_ = 0;
};

class SampleStream {
 public:
  virtual ~SampleStream() = default;
  virtual bool next_iteration(std::vector<EmbeddingSample>& out) = 0;
  virtual void reset() = 0;
  virtual std::size_t max_sample_len() const = 0;
};

class ZipfStream final : public SampleStream {
 public:
  ZipfStream(const WorkloadSpec& spec, const ClusterConfig& cfg)
      : spec_(spec), per_iteration_(cfg.samples_per_iteration()) {
    edx_zipf* z = nullptr;
    edxc::check(edx_zipf_create(spec.total_embeddings, spec.sample_len, spec.zipf_s,
                                spec.iterations, spec.seed, per_iteration_, &z));
    z_.reset(z);
    buf_.resize(per_iteration_ * spec.sample_len);
  }
  bool next_iteration(std::vector<EmbeddingSample>& out) override {
    if (!edx_zipf_next(z_.get(), buf_.data())) return false;
    out.resize(per_iteration_);
    for (std::size_t i = 0; i < per_iteration_; ++i)
      out[i].ids.assign(buf_.begin() + static_cast<std::ptrdiff_t>(i * spec_.sample_len),
                        buf_.begin() + static_cast<std::ptrdiff_t>((i + 1) * spec_.sample_len));
    return true;
  }
  void reset() override { edx_zipf_reset(z_.get()); }
  std::size_t max_sample_len() const override { return spec_.sample_len; }
  const WorkloadSpec& spec() const { return spec_; }

 private:
  struct Del {
    void operator()(edx_zipf* z) const { edx_zipf_destroy(z); }
  };
  WorkloadSpec spec_;
  std::size_t per_iteration_;
  std::unique_ptr<edx_zipf, Del> z_;
  std::vector<uint32_t> buf_;
};

// Tables of a multi-table trace; row ids flatten into one id space by the
// cumulative table sizes (workload.hpp:137-150).
struct TraceSchema {
  struct Table {
    std::string name;
    std::size_t size = 0;
  };
  std::vector<Table> tables;

  std::size_t total_embeddings() const {
    std::size_t sum = 0;
    for (const Table& t : tables) sum += t.size;
    return sum;
  }
};

// "name size" per line, blank lines skipped (workload.hpp:152-172).
inline TraceSchema load_schema(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open schema file: " + path);
  TraceSchema schema;
  std::string text;
  for (std::size_t line_no = 1; std::getline(in, text); ++line_no) {
    std::istringstream fields(text);
    TraceSchema::Table t;
    if (!(fields >> t.name)) continue;
    if (!(fields >> t.size) || t.size == 0)
      throw std::runtime_error(path + ":" + std::to_string(line_no) +
                               ": expected 'table_name size'");
    schema.tables.push_back(std::move(t));
  }
  if (schema.tables.empty()) throw std::runtime_error("schema file declares no tables: " + path);
  return schema;
}

// One sample per line of whitespace-separated decimal ids, m*n samples per
// iteration, a trailing partial iteration dropped with a warning
// (workload.hpp:176-268).  The file is parsed once by libedx (all host
// threads) into per-iteration CSR; batch_csr() hands that layout straight to
// the engine's edx_engine_load_batch / edx_engine_iterate / edx_engine_prefetch.
class TraceStream final : public SampleStream {
 public:
  TraceStream(const std::string& path, const ClusterConfig& cfg,
              const TraceSchema* schema = nullptr, std::ostream* warnings = &std::cerr) {
    std::vector<std::uint64_t> sizes;
    std::vector<const char*> names;
    if (schema != nullptr)
      for (const auto& t : schema->tables) {
        sizes.push_back(t.size);
        names.push_back(t.name.c_str());
      }
    edx_trace* t = nullptr;
    static const std::uint64_t kNoTables = 0;  // a schema without tables is still a schema
    const std::uint64_t* sizes_p =
        schema == nullptr ? nullptr : (sizes.empty() ? &kNoTables : sizes.data());
    edxc::check(edx_trace_load(path.c_str(), sizes.size(), sizes_p, names.data(),
                               cfg.samples_per_iteration(), cfg.cache_capacity,
                               static_cast<std::uint64_t>(cfg.m), &t));
    t_.reset(t);
    std::uint64_t it = 0, dropped = 0, max_len = 0;
    edx_trace_info(t, &it, &dropped, &max_len, nullptr);
    iterations_ = it;
    dropped_ = dropped;
    max_sample_len_ = max_len;
    per_iteration_ = cfg.samples_per_iteration();
    if (dropped_ != 0 && warnings != nullptr)
      *warnings << "warning: " << path << ": dropping " << dropped_
                << " trailing sample(s) of a partial iteration\n";
  }

  bool next_iteration(std::vector<EmbeddingSample>& out) override {
    if (cursor_ >= iterations_) return false;
    const BatchCsr b = batch_csr(cursor_++);
    out.resize(per_iteration_);
    for (std::size_t i = 0; i < per_iteration_; ++i)
      out[i].ids.assign(b.ids + b.offsets[i], b.ids + b.offsets[i + 1]);
    return true;
  }

  void reset() override { cursor_ = 0; }
  std::size_t max_sample_len() const override { return max_sample_len_; }
  std::size_t iterations() const { return iterations_; }
  std::size_t dropped_samples() const { return dropped_; }

  // Iteration `it` in the engine's batch layout (no copies).
  struct BatchCsr {
    const std::uint32_t* ids;
    const std::uint64_t* offsets;  // per_iteration + 1 entries, offsets[0] == 0
    std::uint64_t num_ids;
  };
  BatchCsr batch_csr(std::size_t it) const {
    BatchCsr b{};
    edxc::check(edx_trace_iteration(t_.get(), it, &b.ids, &b.offsets, &b.num_ids));
    return b;
  }

 private:
  struct Del {
    void operator()(edx_trace* t) const { edx_trace_destroy(t); }
  };
  std::unique_ptr<edx_trace, Del> t_;
  std::size_t per_iteration_ = 0, iterations_ = 0, dropped_ = 0, cursor_ = 0, max_sample_len_ = 0;
};

// Writes the stream from its current position, one sample per line
// (workload.hpp:272-289); returns the line count.
inline std::size_t write_trace(std::ostream& os, SampleStream& stream) {
  std::vector<EmbeddingSample> batch;
  std::size_t lines = 0;
  while (stream.next_iteration(batch))
    for (const EmbeddingSample& s : batch) {
      const char* sep = "";
      for (EmbeddingId id : s.ids) {
        os << sep << id;
        sep = " ";
      }
      os << '\n';
      ++lines;
    }
  return lines;
}

}  // namespace embdispatch
