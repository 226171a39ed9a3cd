// Synthetic input stream for the benchmark: ZipfStream (workload.hpp:94-133).
// Host-side input producer (out of the hot path); it must emit the same ids
// as the reference so both arms of bench.py dispatch identical batches.
// std::mt19937_64 is fully specified by the standard and std::pow/upper_bound
// are the same libm/libstdc++ calls, so the stream is identical by
// construction; tests/test_workload.py pins it against the reference.
#include <algorithm>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "edx.h"

extern "C" void edx_set_error(int code, const char* msg);

struct edx_zipf {
  std::vector<double> cdf;
  std::mt19937_64 rng;
  uint64_t sample_len, iterations, emitted = 0, seed, per_iteration;
};

namespace {

void seed_cdf(edx_zipf* z, uint64_t total, double s) {
  // P(id) ~ (id+1)^-s, normalised; the last entry pinned to 1 (workload.hpp:56-66)
  z->cdf.resize(total);
  double acc = 0.0;
  for (uint64_t r = 0; r < total; ++r) {
    acc += std::pow(static_cast<double>(r + 1), -s);
    z->cdf[r] = acc;
  }
  for (double& c : z->cdf) c /= acc;
  z->cdf.back() = 1.0;
}

uint32_t draw(edx_zipf* z) {
  const double u = static_cast<double>(z->rng() >> 11) * 0x1.0p-53;  // workload.hpp:70-71
  return static_cast<uint32_t>(std::upper_bound(z->cdf.begin(), z->cdf.end(), u) - z->cdf.begin());
}

}  // namespace

extern "C" {

int edx_zipf_create(uint64_t total, uint64_t sample_len, double zipf_s, uint64_t iterations,
                    uint64_t seed, uint64_t per_iteration, edx_zipf** out) {
  if (sample_len < 1) {
    edx_set_error(EDX_INVALID_ARGUMENT, "sample_len must be >= 1");
    return EDX_INVALID_ARGUMENT;
  }
  if (!(zipf_s > 0.0)) {
    edx_set_error(EDX_INVALID_ARGUMENT, "zipf_s must be positive");
    return EDX_INVALID_ARGUMENT;
  }
  if (total < sample_len) {
    edx_set_error(EDX_INVALID_ARGUMENT, "sample_len exceeds the embedding population");
    return EDX_INVALID_ARGUMENT;
  }
  auto* z = new edx_zipf;
  z->sample_len = sample_len;
  z->iterations = iterations;
  z->seed = seed;
  z->per_iteration = per_iteration;
  seed_cdf(z, total, zipf_s);
  z->rng.seed(seed);
  *out = z;
  return EDX_OK;
}

int edx_zipf_next(edx_zipf* z, uint32_t* ids) {
  if (z->emitted >= z->iterations) return 0;
  for (uint64_t i = 0; i < z->per_iteration; ++i) {
    uint32_t* row = ids + i * z->sample_len;
    uint64_t have = 0;
    while (have < z->sample_len) {  // distinct ids by rejection (workload.hpp:109-115)
      const uint32_t id = draw(z);
      if (std::find(row, row + have, id) == row + have) row[have++] = id;
    }
  }
  ++z->emitted;
  return 1;
}

void edx_zipf_reset(edx_zipf* z) {
  z->rng.seed(z->seed);
  z->emitted = 0;
}

void edx_zipf_destroy(edx_zipf* z) { delete z; }

}  // extern "C"
