// Report formats of the drop-in (include/embdispatch/report_io.hpp) against
// the compiled reference's report_io.hpp (oracle/_ref/libedx_ref.so, loaded
// at run time) on randomized RunResults: every JSON line and the comparison
// CSV byte for byte.  Host formatting only -- no device needed.
// Usage: report_test <path to libedx_ref.so>
#include <dlfcn.h>

#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "embdispatch/report_io.hpp"
extern "C" {
#include "edx_oracle.h"
}

using namespace embdispatch;

static int failures = 0;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  void* h = dlopen(argv[1], RTLD_NOW);
  if (!h) {
    std::printf("SKIP %s\n", dlerror());
    return 0;
  }
  auto jsonl = reinterpret_cast<decltype(&orc_report_jsonl)>(dlsym(h, "orc_report_jsonl"));
  auto csv = reinterpret_cast<decltype(&orc_comparison_csv)>(dlsym(h, "orc_comparison_csv"));
  std::mt19937_64 rng(20251221);
  auto u = [&](std::uint64_t hi) { return rng() % hi; };
  auto d = [&] {  // mixes integers, tiny and huge magnitudes, exact zeros
    switch (rng() % 5) {
      case 0: return 0.0;
      case 1: return static_cast<double>(rng() % 1000);
      case 2: return std::ldexp(static_cast<double>(rng() >> 11), -53 - static_cast<int>(rng() % 40));
      case 3: return static_cast<double>(rng() >> 11) * 1e-9;
      default: return std::ldexp(static_cast<double>(rng() >> 11), static_cast<int>(rng() % 30));
    }
  };
  for (int trial = 0; trial < 200; ++trial) {
    const int n = 1 + static_cast<int>(u(9));
    ClusterConfig cfg;
    cfg.n = n;
    cfg.m = 1;
    const double speeds[4] = {5e9, 5e8, 1.25e9, 2.5e10};
    for (int j = 0; j < n; ++j) cfg.bandwidths_bps.push_back(speeds[u(1 + trial % 4)]);
    std::vector<RunResult> runs(1 + u(3));
    const std::uint64_t iters = 1 + u(50), lookups = u(100000);
    const char* names[] = {"hitgreedy", "ecomix:0.5", "ecomix:1", "ecomix:0.25"};
    for (std::size_t k = 0; k < runs.size(); ++k) {
      RunSummary& s = runs[k].summary;
      s.mechanism = names[k];
      s.iterations = iters;
      s.measured_iterations = u(iters + 1);
      s.lookups = lookups;
      s.hits = u(lookups + 1);
      s.miss_pull = u(5000);
      s.update_push = u(5000);
      s.evict_push = trial % 7 == 0 ? 0 : u(5000);
      s.cost_s = trial % 11 == 0 ? 0.0 : d();
      s.expected_cost_s = d();
      s.has_expected = rng() & 1;
      s.decision_s_total = d();
      s.decision_s_max = d();
      s.matrix_s_total = d();
      s.budget_violations = u(3);
      for (int j = 0; j < n; ++j) {
        s.miss_pull_w.push_back(u(900));
        s.update_push_w.push_back(u(900));
        s.evict_push_w.push_back(u(900));
        s.ops_w.push_back(u(2700));
      }
      IterationReport rep;
      rep.iteration = u(1000);
      rep.mechanism = names[k];
      rep.miss_pull = u(9999);
      rep.update_push = u(9999);
      rep.evict_push = u(9999);
      rep.hits = u(9999);
      rep.lookups = u(99999);
      rep.cost_s = d();
      rep.decision_s = d();
      rep.matrix_s = d();
      rep.expected_cost_s = d();
      rep.has_expected = rng() & 1;
      rep.miss_pull_w = s.miss_pull_w;
      rep.update_push_w = s.update_push_w;
      rep.evict_push_w = s.evict_push_w;
      for (int j = 0; j < n; ++j) rep.cost_w.push_back(d());
      orc_iter_report o{rep.iteration, rep.mechanism.c_str(), rep.miss_pull, rep.update_push,
                        rep.evict_push, rep.hits, rep.lookups, rep.cost_s, rep.decision_s,
                        rep.matrix_s, rep.expected_cost_s, rep.has_expected, n,
                        rep.miss_pull_w.data(), rep.update_push_w.data(),
                        rep.evict_push_w.data(), rep.cost_w.data()};
      std::vector<char> buf(1 << 16);
      std::uint64_t len = 0;
      jsonl(&o, buf.data(), buf.size(), &len);
      const std::string mine = report_jsonl(rep);
      if (mine != std::string(buf.data(), len)) {
        ++failures;
        std::printf("FAIL jsonl\n  ours %s\n  ref  %s\n", mine.c_str(), buf.data());
      }
    }
    std::vector<orc_run_summary> pod;
    for (const RunResult& r : runs) {
      const RunSummary& s = r.summary;
      pod.push_back(orc_run_summary{s.mechanism.c_str(), s.iterations, s.measured_iterations,
                                    s.miss_pull, s.update_push, s.evict_push, s.hits, s.lookups,
                                    s.cost_s, s.expected_cost_s, s.decision_s_total,
                                    s.decision_s_max, s.matrix_s_total, s.has_expected, n,
                                    s.budget_violations, s.miss_pull_w.data(),
                                    s.update_push_w.data(), s.evict_push_w.data(), s.ops_w.data()});
    }
    orc_cluster_config oc{n, 1, cfg.bandwidths_bps.data(), n, 0, 2048, 16, 1.0};
    std::vector<char> buf(1 << 20);
    std::uint64_t len = 0;
    const std::string ref_name = names[u(runs.size())];
    csv(pod.data(), pod.size(), ref_name.c_str(), &oc, buf.data(), buf.size(), &len);
    const std::string mine = comparison_csv(runs, ref_name, cfg);
    if (mine != std::string(buf.data(), len)) {
      ++failures;
      std::printf("FAIL csv\n--- ours\n%s--- ref\n%s", mine.c_str(), buf.data());
    }
    (void)fast_class_ops_fraction(runs[0].summary, cfg);
  }
  // error paths carry the reference's messages
  ClusterConfig cfg;
  cfg.n = 1;
  cfg.bandwidths_bps = {5e9};
  try {
    comparison_csv({}, "x", cfg);
    ++failures;
  } catch (const std::invalid_argument& e) {
    if (std::string(e.what()) != "no runs to compare") ++failures;
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
