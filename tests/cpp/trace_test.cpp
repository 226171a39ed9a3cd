// Trace ingestion through the drop-in C++ headers (include/embdispatch/
// workload.hpp): the reference's trace tests (tests/test_workload.cpp:179-281)
// written against the same API, plus the CSR view the engine consumes.  Host
// only -- no device needed.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "embdispatch/workload.hpp"

using namespace embdispatch;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
      ++failures;                                                  \
    }                                                              \
  } while (0)

struct TempFile {
  std::filesystem::path path;
  TempFile(const std::string& name, const std::string& text)
      : path(std::filesystem::temp_directory_path() / name) {
    std::ofstream(path) << text;
  }
  ~TempFile() { std::filesystem::remove(path); }
};

static ClusterConfig tiny(int n, int m, std::size_t cap = 64) {
  ClusterConfig c;
  c.n = n;
  c.m = m;
  c.bandwidths_bps.assign(n, 5e9);
  c.cache_capacity = cap;
  return c;
}

static std::vector<std::vector<EmbeddingSample>> drain(SampleStream& s) {
  std::vector<std::vector<EmbeddingSample>> out;
  std::vector<EmbeddingSample> b;
  while (s.next_iteration(b)) out.push_back(b);
  return out;
}

template <class F>
static std::string what_of(F&& f) {
  try {
    f();
  } catch (const std::runtime_error& e) {
    return e.what();
  }
  return "";
}

int main() {
  {
    TempFile f("edx_trace_a.txt", "1 2 3\n4 5 6\n");
    TraceStream s(f.path.string(), tiny(2, 1));
    auto b = drain(s);
    CHECK(b.size() == 1 && b[0].size() == 2);
    CHECK((b[0][0].ids == std::vector<EmbeddingId>{1, 2, 3}));
    CHECK((b[0][1].ids == std::vector<EmbeddingId>{4, 5, 6}));
    CHECK(s.dropped_samples() == 0 && s.max_sample_len() == 3);
    const auto csr = s.batch_csr(0);
    CHECK(csr.num_ids == 6 && csr.offsets[0] == 0 && csr.offsets[1] == 3 && csr.offsets[2] == 6);
  }
  {
    TempFile f("edx_trace_b.txt", "3 3 7\n8 9 10\n");
    TraceStream s(f.path.string(), tiny(2, 1));
    CHECK((drain(s)[0][0].ids == std::vector<EmbeddingId>{3, 7}));
  }
  {
    TempFile f("edx_trace_c.txt", "1\n2\n3\n");
    std::ostringstream w;
    TraceStream s(f.path.string(), tiny(2, 1), nullptr, &w);
    CHECK(drain(s).size() == 1 && s.dropped_samples() == 1);
    CHECK(w.str().find("dropping 1 trailing") != std::string::npos);
  }
  {
    TempFile f("edx_trace_d.txt", "1 2\nx 4\n");
    const std::string w = what_of([&] { TraceStream s(f.path.string(), tiny(2, 1)); });
    CHECK(w.find(":2:") != std::string::npos && w.find("x") != std::string::npos);
  }
  {
    TempFile f("edx_trace_e.txt", "");
    CHECK(!what_of([&] { TraceStream s(f.path.string(), tiny(2, 1)); }).empty());
  }
  {
    TempFile sf("edx_schema.txt", "users 10\nitems 20\nads 5\n");
    const TraceSchema schema = load_schema(sf.path.string());
    CHECK(schema.total_embeddings() == 35);
    TempFile f("edx_trace_f.txt", "1 2 3\n9 19 4\n");
    TraceStream s(f.path.string(), tiny(2, 1), &schema);
    auto b = drain(s);
    CHECK((b[0][0].ids == std::vector<EmbeddingId>{1, 12, 33}));
    CHECK((b[0][1].ids == std::vector<EmbeddingId>{9, 29, 34}));
    TempFile g("edx_trace_g.txt", "10 0 0\n0 0 0\n");
    CHECK(!what_of([&] { TraceStream t(g.path.string(), tiny(2, 1), &schema); }).empty());
    TempFile h("edx_trace_h.txt", "1 2\n3 4\n");
    CHECK(!what_of([&] { TraceStream t(h.path.string(), tiny(2, 1), &schema); }).empty());
  }
  {
    TempFile f("edx_trace_i.txt", "1 2 3\n4 5 6\n7 8 9\n10 11 12\n");
    CHECK(!what_of([&] { TraceStream s(f.path.string(), tiny(2, 2, 4)); }).empty());
  }
  {
    WorkloadSpec spec;
    spec.total_embeddings = 300;
    spec.sample_len = 4;
    spec.iterations = 3;
    spec.seed = 17;
    const ClusterConfig cfg = tiny(2, 2);
    ZipfStream source(spec, cfg);
    const auto path = std::filesystem::temp_directory_path() / "edx_roundtrip.txt";
    {
      std::ofstream out(path);
      CHECK(write_trace(out, source) == 12);
    }
    TraceStream parsed(path.string(), cfg);
    source.reset();
    auto want = drain(source), got = drain(parsed);
    CHECK(got.size() == want.size());
    for (std::size_t i = 0; i < want.size() && i < got.size(); ++i)
      for (std::size_t s = 0; s < want[i].size(); ++s) CHECK(got[i][s].ids == want[i][s].ids);
    std::filesystem::remove(path);
  }
  if (failures == 0) std::printf("OK\n");
  return failures == 0 ? 0 : 1;
}
