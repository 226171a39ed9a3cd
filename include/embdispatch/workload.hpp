// Drop-in for the reference's synthetic input stream (workload.hpp:36-133):
// WorkloadSpec, SampleStream and ZipfStream over libedx's host generator
// (bit-identical ids).  Trace ingestion is outside the device path.
#pragma once

#include <cstdint>
#include <memory>
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

 private:
  struct Del {
    void operator()(edx_zipf* z) const { edx_zipf_destroy(z); }
  };
  WorkloadSpec spec_;
  std::size_t per_iteration_;
  std::unique_ptr<edx_zipf, Del> z_;
  std::vector<uint32_t> buf_;
};

}  // namespace embdispatch
