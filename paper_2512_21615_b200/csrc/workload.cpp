// Synthetic input stream: ZipfStream (workload.hpp:94-133) -- the host-side
// input producer of run() and of bench.py (input pipeline).
//
// It must emit exactly the reference's ids.  The reference draws
// u = (rng() >> 11) * 2^-53 from std::mt19937_64 and maps it with
// std::upper_bound over the Zipf CDF (built with std::pow, accumulated in id
// order), rejecting ids already in the sample.  This version produces the
// same stream much faster:
//  * CDF: the pow terms are computed on all host threads, the fp64 prefix sum
//    stays sequential in id order (the same adds, so the same bits).
//  * mapping: a guide table over the top K bits of u's 53-bit integer gives,
//    for each bucket, the first index upper_bound can return there, so the
//    search runs on [guide[b], guide[b+1]] -- the same upper_bound, a handful
//    of probes instead of ~log2(V) cache misses.
//  * draws: the RNG stream is consumed in chunks (sequential, cheap), the
//    chunk is mapped on all host threads, then samples are assembled in draw
//    order with duplicates rejected through a small per-sample hash set
//    (the same membership test as the reference's std::find).
//  * pipeline: a producer thread builds batch t+1 while the caller works on
//    batch t (edx_zipf_next hands over the finished batch and restarts it).
// tests/test_host.py pins the stream against the reference generator.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "edx.h"

extern "C" void edx_set_error(int code, const char* msg);

namespace {

unsigned host_threads() {
  const unsigned t = std::thread::hardware_concurrency();
  return t == 0 ? 1u : std::min(t, 64u);
}

// Runs f(begin, end) over [0, count) split across the host threads.
template <class F>
void parallel_for(uint64_t count, uint64_t min_chunk, F&& f) {
  const unsigned nt = host_threads();
  const uint64_t parts = std::min<uint64_t>(nt, std::max<uint64_t>(1, count / min_chunk));
  if (parts <= 1) {
    f(0, count);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(parts - 1);
  const uint64_t step = (count + parts - 1) / parts;
  for (uint64_t p = 1; p < parts; ++p) {
    const uint64_t b = p * step, e = std::min(count, b + step);
    if (b < e) th.emplace_back([&f, b, e] { f(b, e); });
  }
  f(0, std::min(count, step));
  for (auto& t : th) t.join();
}

}  // namespace

struct edx_zipf {
  std::vector<double> cdf;
  std::vector<uint32_t> guide;  // guide[b] = upper_bound(cdf, b * 2^-K), b in [0, 2^K]
  int kbits = 0;
  std::mt19937_64 rng;
  uint64_t sample_len = 0, iterations = 0, seed = 0, per_iteration = 0;
  uint64_t produced = 0, emitted = 0;

  // mapped draws not yet consumed (the RNG stream is consumed in order)
  std::vector<uint64_t> raw;
  std::vector<uint32_t> drawn;
  size_t drawn_pos = 0;

  // producer pipeline
  std::vector<uint32_t> batch[2];
  int ready = -1;  // buffer holding the next batch, -1 = none yet
  bool busy = false, stop = false;
  std::thread producer;
  std::mutex mu;
  std::condition_variable cv;

  ~edx_zipf() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    if (producer.joinable()) producer.join();
  }

  uint32_t map_one(uint64_t x) const {  // x = rng() >> 11 (53 bits)
    const double u = static_cast<double>(x) * 0x1.0p-53;  // workload.hpp:70-71
    const uint64_t b = x >> (53 - kbits);
    const auto lo = cdf.begin() + guide[b];
    const auto hi = cdf.begin() + guide[b + 1];
    return static_cast<uint32_t>(std::upper_bound(lo, hi, u) - cdf.begin());
  }

  void refill() {
    const size_t chunk = std::max<size_t>(1 << 16, per_iteration * sample_len / 4);
    raw.resize(chunk);
    drawn.resize(chunk);
    for (size_t t = 0; t < chunk; ++t) raw[t] = rng() >> 11;
    parallel_for(chunk, 1 << 14, [this](uint64_t b, uint64_t e) {
      // Tail draws miss the caches twice (guide entry, then the CDF line), so
      // the guide entry is prefetched 16 draws ahead and the CDF line 8 ahead.
      constexpr uint64_t kG = 16, kC = 8;
      const int sh = 53 - kbits;
      for (uint64_t t = b; t < e; ++t) {
        if (t + kG < e) __builtin_prefetch(&guide[raw[t + kG] >> sh]);
        if (t + kC < e) __builtin_prefetch(&cdf[guide[raw[t + kC] >> sh]]);
        drawn[t] = map_one(raw[t]);
      }
    });
    drawn_pos = 0;
  }

  uint32_t next_draw() {
    if (drawn_pos == drawn.size()) refill();
    return drawn[drawn_pos++];
  }

  // One iteration of m*n samples of sample_len distinct ids (workload.hpp:104-117).
  void produce(uint32_t* ids) {
    // per-sample set of the ids drawn so far: open addressing, stamp-cleared
    size_t cap = 64;
    while (cap < 4 * sample_len) cap <<= 1;
    std::vector<uint32_t> key(cap), stamp(cap, 0);
    uint32_t epoch = 0;
    for (uint64_t i = 0; i < per_iteration; ++i) {
      uint32_t* row = ids + i * sample_len;
      if (++epoch == 0) {
        std::fill(stamp.begin(), stamp.end(), 0);
        epoch = 1;
      }
      uint64_t have = 0;
      while (have < sample_len) {
        const uint32_t id = next_draw();
        size_t h = (id * 0x9E3779B1u) & (cap - 1);
        bool dup = false;
        while (stamp[h] == epoch) {
          if (key[h] == id) {
            dup = true;
            break;
          }
          h = (h + 1) & (cap - 1);
        }
        if (dup) continue;  // already in the sample: rejected (workload.hpp:111-114)
        stamp[h] = epoch;
        key[h] = id;
        row[have++] = id;
      }
    }
  }

  void start_producer() {
    producer = std::thread([this] {
      std::unique_lock<std::mutex> lk(mu);
      for (;;) {
        cv.wait(lk, [this] { return stop || (busy && ready < 0); });
        if (stop) return;
        const int buf = static_cast<int>(produced & 1);
        lk.unlock();
        produce(batch[buf].data());
        lk.lock();
        ++produced;
        ready = buf;
        busy = false;
        cv.notify_all();
      }
    });
  }

  void request() {  // caller holds mu
    if (produced < iterations && !busy && ready < 0) {
      busy = true;
      cv.notify_all();
    }
  }

  void reset_stream() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return !busy; });
    rng.seed(seed);
    drawn.clear();
    drawn_pos = 0;
    produced = emitted = 0;
    ready = -1;
    request();
  }
};

namespace {

void build_cdf(edx_zipf* z, uint64_t total, double s) {
  // P(id) ~ (id+1)^-s, accumulated in id order and normalised, the last entry
  // pinned to 1 (workload.hpp:56-66)
  z->cdf.resize(total);
  double* c = z->cdf.data();
  parallel_for(total, 1 << 16, [c, s](uint64_t b, uint64_t e) {
    for (uint64_t r = b; r < e; ++r) c[r] = std::pow(static_cast<double>(r + 1), -s);
  });
  double acc = 0.0;
  for (uint64_t r = 0; r < total; ++r) {
    acc += c[r];
    c[r] = acc;
  }
  parallel_for(total, 1 << 16, [c, acc](uint64_t b, uint64_t e) {
    for (uint64_t r = b; r < e; ++r) c[r] /= acc;
  });
  z->cdf.back() = 1.0;
  // guide table: about one bucket per id, at most 2^24 buckets
  int k = 1;
  while (k < 24 && (1ULL << k) < total) ++k;
  z->kbits = k;
  const uint64_t nb = 1ULL << k;
  z->guide.resize(nb + 1);
  uint32_t* g = z->guide.data();
  parallel_for(nb + 1, 1 << 14, [z, g, k](uint64_t b, uint64_t e) {
    // one search at the range start, then a monotone walk (bucket starts increase)
    const double scale = std::ldexp(1.0, -k);
    const double* c = z->cdf.data();
    const uint64_t n = z->cdf.size();
    uint64_t idx = static_cast<uint64_t>(
        std::upper_bound(z->cdf.begin(), z->cdf.end(), static_cast<double>(b) * scale) - z->cdf.begin());
    for (uint64_t x = b; x < e; ++x) {
      const double u = static_cast<double>(x) * scale;  // bucket start, exact
      while (idx < n && c[idx] <= u) ++idx;             // first index with cdf > u
      g[x] = static_cast<uint32_t>(idx);
    }
  });
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
  if (total > 0xFFFFFFFFull) {
    edx_set_error(EDX_INVALID_ARGUMENT, "population exceeds 32-bit ids");
    return EDX_INVALID_ARGUMENT;
  }
  auto* z = new edx_zipf;
  z->sample_len = sample_len;
  z->iterations = iterations;
  z->seed = seed;
  z->per_iteration = per_iteration;
  build_cdf(z, total, zipf_s);
  z->rng.seed(seed);
  z->batch[0].resize(per_iteration * sample_len);
  z->batch[1].resize(per_iteration * sample_len);
  z->start_producer();
  {
    std::lock_guard<std::mutex> lk(z->mu);
    z->request();
  }
  *out = z;
  return EDX_OK;
}

int edx_zipf_next(edx_zipf* z, uint32_t* ids) {
  std::unique_lock<std::mutex> lk(z->mu);
  if (z->emitted >= z->iterations) return 0;
  z->cv.wait(lk, [z] { return z->ready >= 0; });
  const int buf = z->ready;
  std::memcpy(ids, z->batch[buf].data(), z->batch[buf].size() * sizeof(uint32_t));
  z->ready = -1;
  ++z->emitted;
  z->request();  // start the next batch while the caller works on this one
  return 1;
}

void edx_zipf_reset(edx_zipf* z) { z->reset_stream(); }

int edx_zipf_sampler_create(uint64_t population, double zipf_s, uint64_t seed, edx_zipf** out) {
  if (population == 0) {
    edx_set_error(EDX_INVALID_ARGUMENT, "population must be positive");
    return EDX_INVALID_ARGUMENT;
  }
  if (population > 0xFFFFFFFFull) {
    edx_set_error(EDX_INVALID_ARGUMENT, "population exceeds 32-bit ids");
    return EDX_INVALID_ARGUMENT;
  }
  auto* z = new edx_zipf;  // no stream: iterations = 0, no producer thread
  z->sample_len = 1;
  z->seed = seed;
  build_cdf(z, population, zipf_s);
  z->rng.seed(seed);
  *out = z;
  return EDX_OK;
}

int edx_zipf_draw(edx_zipf* z, uint64_t count, uint32_t* out) {
  if (z->producer.joinable()) {
    edx_set_error(EDX_INVALID_ARGUMENT, "edx_zipf_draw needs a sampler (edx_zipf_sampler_create)");
    return EDX_INVALID_ARGUMENT;
  }
  for (uint64_t t = 0; t < count; ++t) out[t] = z->next_draw();
  return EDX_OK;
}

void edx_zipf_destroy(edx_zipf* z) { delete z; }

}  // extern "C"
