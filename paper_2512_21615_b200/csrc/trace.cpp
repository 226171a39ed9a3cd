// Trace ingestion: TraceStream (workload.hpp:176-268) -- the file-driven input
// producer of run(), host side.
//
// The reference reads the trace line by line through std::getline +
// istringstream + std::stoull, collapses duplicates with make_sample, and keeps
// one std::vector per sample.  This loader reads the file in one pass into
// memory, parses newline-aligned chunks on all host threads, and stores the
// result as the engine's CSR layout: per iteration, `ids` plus `offsets`
// rebased to start at 0, ready for edx_engine_load_batch / edx_engine_iterate /
// edx_engine_prefetch with no per-sample repacking.
//
// Behaviour follows the reference exactly:
//  * tokens are maximal runs of non-isspace bytes ("C" locale); a token is an
//    id iff std::stoull(token) consumes all of it: [+-]?[0-9]+ with a
//    magnitude < 2^64 (a leading '-' wraps modulo 2^64, as strtoull does),
//    then truncated to a 32-bit EmbeddingId;
//  * blank lines are skipped but counted; the last line needs no '\n';
//  * with a schema, field i must be < table i's size and is shifted by the
//    sizes of the tables before it (32-bit wrap, as the reference's cast);
//  * duplicates collapse, first occurrence wins (make_sample, types.hpp:46);
//  * a sample longer than cache_capacity / m (when that is > 0) is rejected;
//  * the first failing line in file order wins, with the reference's message;
//  * samples group into iterations of samples_per_iteration; a trailing partial
//    iteration is dropped (the count is returned; the caller prints the warning
//    the reference writes).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "edx.h"

extern "C" void edx_set_error(int code, const char* msg);

struct edx_trace {
  uint64_t per_iteration = 0, iterations = 0, dropped = 0, max_len = 0, samples = 0;
  std::vector<uint32_t> ids;         // every kept sample's ids, in file order
  std::vector<uint64_t> ids_start;   // per iteration: first id index
  std::vector<uint64_t> offsets;     // iterations * (per_iteration + 1), rebased to 0
};

namespace {

inline bool is_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// std::stoull(token) with a full-consumption check (workload.hpp:206-214).
bool parse_id(const char* b, const char* e, uint64_t* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) neg = (*b++ == '-');
  if (b == e) return false;
  uint64_t v = 0;
  for (; b < e; ++b) {
    const unsigned d = static_cast<unsigned char>(*b) - '0';
    if (d > 9) return false;
    if (v > (UINT64_MAX - d) / 10) return false;  // out_of_range
    v = v * 10 + d;
  }
  *out = neg ? (0 - v) : v;
  return true;
}

struct Error {
  enum Kind { kNone, kMalformed, kFieldCount, kRowRange, kTooLong } kind = kNone;
  uint64_t line = 0;  // local (0-based) line within the chunk
  std::string token;
  uint64_t a = 0, b = 0;
};

struct Chunk {
  const char* begin;
  const char* end;
  uint64_t lines = 0;
  std::vector<uint32_t> ids;
  std::vector<uint64_t> lens;
  uint64_t max_len = 0;
  Error err;
};

struct Params {
  bool schema;  // table_sizes != NULL: a schema, possibly with no tables
  uint64_t n_tables;
  const uint64_t* table_sizes;
  std::vector<uint64_t> table_offsets;
  uint64_t max_allowed;
};

void parse_chunk(Chunk& c, const Params& p) {
  std::vector<uint32_t> raw;
  std::unordered_set<uint32_t> seen;
  const char* s = c.begin;
  while (s < c.end) {
    const char* nl = static_cast<const char*>(std::memchr(s, '\n', c.end - s));
    const char* le = nl ? nl : c.end;
    const uint64_t line = c.lines++;
    raw.clear();
    for (const char* t = s; t < le;) {
      while (t < le && is_space(*t)) ++t;
      if (t == le) break;
      const char* te = t;
      while (te < le && !is_space(*te)) ++te;
      uint64_t v;
      if (!parse_id(t, te, &v)) {
        c.err.kind = Error::kMalformed;
        c.err.line = line;
        c.err.token.assign(t, te);
        return;
      }
      raw.push_back(static_cast<uint32_t>(v));
      t = te;
    }
    s = nl ? nl + 1 : c.end;
    if (raw.empty()) continue;
    if (p.schema) {
      if (raw.size() != p.n_tables) {
        c.err = {Error::kFieldCount, line, {}, p.n_tables, raw.size()};
        return;
      }
      for (uint64_t i = 0; i < raw.size(); ++i) {
        if (raw[i] >= p.table_sizes[i]) {
          c.err = {Error::kRowRange, line, {}, raw[i], i};
          return;
        }
        raw[i] = static_cast<uint32_t>(raw[i] + p.table_offsets[i]);
      }
    }
    const uint64_t first = c.ids.size();
    if (raw.size() <= 64) {
      for (uint32_t id : raw) {
        bool dup = false;
        for (uint64_t k = first; k < c.ids.size(); ++k) dup |= (c.ids[k] == id);
        if (!dup) c.ids.push_back(id);
      }
    } else {
      seen.clear();
      for (uint32_t id : raw)
        if (seen.insert(id).second) c.ids.push_back(id);
    }
    const uint64_t len = c.ids.size() - first;
    if (p.max_allowed > 0 && len > p.max_allowed) {
      c.err = {Error::kTooLong, line, {}, len, 0};
      return;
    }
    c.max_len = std::max(c.max_len, len);
    c.lens.push_back(len);
  }
}

int fail(const std::string& msg) {
  edx_set_error(EDX_RUNTIME_ERROR, msg.c_str());
  return EDX_RUNTIME_ERROR;
}

}  // namespace

extern "C" {

int edx_trace_load(const char* path, uint64_t n_tables, const uint64_t* table_sizes,
                   const char* const* table_names, uint64_t samples_per_iteration,
                   uint64_t cache_capacity, uint64_t m, edx_trace** out) {
  const std::string spath = path ? path : "";
  if (samples_per_iteration == 0 || m == 0) {
    edx_set_error(EDX_INVALID_ARGUMENT, "samples_per_iteration and m must be >= 1");
    return EDX_INVALID_ARGUMENT;
  }
  FILE* f = std::fopen(spath.c_str(), "rb");
  if (!f) return fail("cannot open trace file: " + spath);
  std::string buf;
  {
    char tmp[1 << 16];
    size_t got;
    while ((got = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.append(tmp, got);
    std::fclose(f);
  }

  Params p{table_sizes != nullptr, n_tables, table_sizes, {}, cache_capacity / m};
  uint64_t acc = 0;
  for (uint64_t i = 0; i < n_tables; ++i) {
    p.table_offsets.push_back(acc);
    acc += table_sizes[i];
  }

  // newline-aligned chunks, one per host thread (small files: one chunk)
  const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  const uint64_t parts = std::max<uint64_t>(1, std::min<uint64_t>(hw, buf.size() >> 20));
  std::vector<Chunk> chunks;
  const char* base = buf.data();
  const char* end = base + buf.size();
  const char* s = base;
  for (uint64_t k = 0; k < parts && s < end; ++k) {
    const char* e = (k + 1 == parts) ? end : base + buf.size() * (k + 1) / parts;
    if (e < s) e = s;
    const char* nl = e < end ? static_cast<const char*>(std::memchr(e, '\n', end - e)) : nullptr;
    e = (k + 1 == parts || !nl) ? end : nl + 1;
    chunks.push_back(Chunk{s, e});
    s = e;
  }
  {
    std::vector<std::thread> th;
    for (size_t k = 1; k < chunks.size(); ++k)
      th.emplace_back([&chunks, &p, k] { parse_chunk(chunks[k], p); });
    if (!chunks.empty()) parse_chunk(chunks[0], p);
    for (auto& t : th) t.join();
  }

  uint64_t line_base = 0, samples = 0, total_ids = 0, max_len = 0;
  for (const Chunk& c : chunks) {
    if (c.err.kind != Error::kNone) {
      const std::string where = spath + ":" + std::to_string(line_base + c.err.line + 1) + ": ";
      switch (c.err.kind) {
        case Error::kMalformed:
          return fail(where + "malformed id '" + c.err.token + "'");
        case Error::kFieldCount:
          return fail(where + "expected " + std::to_string(c.err.a) +
                      " fields per schema, got " + std::to_string(c.err.b));
        case Error::kRowRange:
          return fail(where + "row id " + std::to_string(c.err.a) + " exceeds table '" +
                      std::string(table_names && table_names[c.err.b] ? table_names[c.err.b]
                                                                      : "") + "'");
        default:
          return fail(where + "sample of " + std::to_string(c.err.a) +
                      " ids cannot fit the per-worker cache (capacity " +
                      std::to_string(cache_capacity) + ", m " + std::to_string(m) + ")");
      }
    }
    line_base += c.lines;
    samples += c.lens.size();
    total_ids += c.ids.size();
    max_len = std::max(max_len, c.max_len);
  }
  if (samples == 0) return fail("trace file holds no samples: " + spath);

  auto* t = new edx_trace;
  t->samples = samples;
  t->per_iteration = samples_per_iteration;
  t->iterations = samples / samples_per_iteration;
  t->dropped = samples - t->iterations * samples_per_iteration;
  t->max_len = max_len;
  t->ids.reserve(total_ids);
  std::vector<uint64_t> lens;
  lens.reserve(samples);
  for (Chunk& c : chunks) {
    t->ids.insert(t->ids.end(), c.ids.begin(), c.ids.end());
    lens.insert(lens.end(), c.lens.begin(), c.lens.end());
    std::vector<uint32_t>().swap(c.ids);
  }
  const uint64_t P = samples_per_iteration;
  t->offsets.resize(t->iterations * (P + 1));
  t->ids_start.resize(t->iterations + 1);
  uint64_t pos = 0;
  for (uint64_t it = 0; it < t->iterations; ++it) {
    t->ids_start[it] = pos;
    uint64_t* o = &t->offsets[it * (P + 1)];
    o[0] = 0;
    for (uint64_t r = 0; r < P; ++r) o[r + 1] = o[r] + lens[it * P + r];
    pos += o[P];
  }
  t->ids_start[t->iterations] = pos;
  t->ids.resize(pos);  // the dropped tail's ids are never handed out
  *out = t;
  return EDX_OK;
}

void edx_trace_info(const edx_trace* t, uint64_t* iterations, uint64_t* dropped,
                    uint64_t* max_sample_len, uint64_t* samples) {
  if (iterations) *iterations = t->iterations;
  if (dropped) *dropped = t->dropped;
  if (max_sample_len) *max_sample_len = t->max_len;
  if (samples) *samples = t->samples;
}

int edx_trace_iteration(const edx_trace* t, uint64_t it, const uint32_t** ids,
                        const uint64_t** offsets, uint64_t* num_ids) {
  if (it >= t->iterations) {
    edx_set_error(EDX_INVALID_ARGUMENT, "trace iteration out of range");
    return EDX_INVALID_ARGUMENT;
  }
  *ids = t->ids.data() + t->ids_start[it];
  *offsets = t->offsets.data() + it * (t->per_iteration + 1);
  *num_ids = t->ids_start[it + 1] - t->ids_start[it];
  return EDX_OK;
}

void edx_trace_destroy(edx_trace* t) { delete t; }

}  // extern "C"
