/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see edx_oracle.h).
 *
 * A sequential, deliberately plain restatement of the reference algorithms.
 * Every function names the reference lines it follows.  Nothing here is
 * optimised: victims are found by a linear scan, the Hungarian is the dense
 * O(k^3) e-maxx loop, and the state is an explicit per-id record.  The CUDA
 * product never links or calls this file.
 */
#define _GNU_SOURCE
#include "edx_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ errors */

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

/* ------------------------------------------------------------- config/unit */

/* validate(ClusterConfig, max_len) — types.hpp:87-108 */
int orc_validate_config(const orc_cluster_config* cfg, uint64_t max_sample_len) {
  if (cfg->n < 1) return fail(ORC_INVALID_ARGUMENT, "worker count must be >= 1");
  if (cfg->n > 64) return fail(ORC_INVALID_ARGUMENT, "at most 64 workers supported");
  if (cfg->m < 1) return fail(ORC_INVALID_ARGUMENT, "batch size per worker must be >= 1");
  if (cfg->n_bandwidths != cfg->n)
    return fail(ORC_INVALID_ARGUMENT, "need one bandwidth per worker");
  for (int j = 0; j < cfg->n; ++j)
    if (!(cfg->bandwidths_bps[j] > 0.0))
      return fail(ORC_INVALID_ARGUMENT, "bandwidths must be positive");
  if (cfg->d_tran_bytes == 0) return fail(ORC_INVALID_ARGUMENT, "d_tran must be positive");
  if (cfg->alpha < 0.0 || cfg->alpha > 1.0)
    return fail(ORC_INVALID_ARGUMENT, "alpha must lie in [0, 1]");
  uint64_t micro = (uint64_t)cfg->m * max_sample_len;
  if (cfg->cache_capacity < micro)
    return fail(ORC_INVALID_ARGUMENT,
                "cache capacity %llu cannot hold one micro-batch of %llu embeddings",
                (unsigned long long)cfg->cache_capacity, (unsigned long long)micro);
  return ORC_OK;
}

/* unit_cost — types.hpp:112-120; detail::transfer_seconds — cost.hpp:68-73 */
static double unit(const orc_cluster_config* cfg, int w) {
  return (double)cfg->d_tran_bytes * 8.0 / cfg->bandwidths_bps[w];
}

int orc_unit_costs(const orc_cluster_config* cfg, double* out) {
  for (int j = 0; j < cfg->n; ++j) out[j] = unit(cfg, j);
  return ORC_OK;
}

/* ------------------------------------------------------------ mt19937_64 */
/* std::mt19937_64 as fixed by [rand.predef]; the reference draws all its
 * randomness from it (workload.hpp:54-79, experiment.hpp:220). */

typedef struct {
  uint64_t s[312];
  int i;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->s[0] = seed;
  for (int k = 1; k < 312; ++k)
    g->s[k] = 6364136223846793005ULL * (g->s[k - 1] ^ (g->s[k - 1] >> 62)) + (uint64_t)k;
  g->i = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      uint64_t y = (g->s[k] & 0xFFFFFFFF80000000ULL) | (g->s[(k + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = g->s[(k + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
      g->s[k] = v;
    }
    g->i = 0;
  }
  uint64_t x = g->s[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* ------------------------------------------------------------ Zipf stream */

struct orc_zipf {
  double* cdf;
  uint64_t n, sample_len, iterations, emitted, seed, per_iteration;
  double s;
  mt64 rng;
};

/* ZipfSampler ctor — workload.hpp:56-66 */
static void zipf_init(orc_zipf* z) {
  double acc = 0.0;
  for (uint64_t r = 0; r < z->n; ++r) {
    acc += pow((double)(r + 1), -z->s);
    z->cdf[r] = acc;
  }
  for (uint64_t r = 0; r < z->n; ++r) z->cdf[r] /= acc;
  z->cdf[z->n - 1] = 1.0;
  mt64_seed(&z->rng, z->seed);
}

/* ZipfSampler::draw — workload.hpp:68-74 (upper_bound over the CDF) */
static uint32_t zipf_draw(orc_zipf* z) {
  double u = (double)(mt64_next(&z->rng) >> 11) * 0x1.0p-53;
  uint64_t lo = 0, hi = z->n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (z->cdf[mid] > u) hi = mid;
    else lo = mid + 1;
  }
  return (uint32_t)lo;
}

int orc_zipf_create(uint64_t total, uint64_t sample_len, double zipf_s, uint64_t iterations,
                    uint64_t seed, uint64_t per_iteration, orc_zipf** out) {
  /* validate(WorkloadSpec) — workload.hpp:44-50 */
  if (sample_len < 1) return fail(ORC_INVALID_ARGUMENT, "sample_len must be >= 1");
  if (!(zipf_s > 0.0)) return fail(ORC_INVALID_ARGUMENT, "zipf_s must be positive");
  if (total < sample_len)
    return fail(ORC_INVALID_ARGUMENT, "sample_len exceeds the embedding population");
  orc_zipf* z = (orc_zipf*)calloc(1, sizeof *z);
  z->cdf = (double*)malloc(sizeof(double) * total);
  z->n = total;
  z->sample_len = sample_len;
  z->iterations = iterations;
  z->seed = seed;
  z->s = zipf_s;
  z->per_iteration = per_iteration;
  zipf_init(z);
  *out = z;
  return ORC_OK;
}

void orc_zipf_destroy(orc_zipf* z) {
  if (!z) return;
  free(z->cdf);
  free(z);
}

/* ZipfStream::next_iteration — workload.hpp:103-119 (distinct ids by rejection) */
int orc_zipf_next(orc_zipf* z, uint32_t* ids) {
  if (z->emitted >= z->iterations) return 0;
  for (uint64_t i = 0; i < z->per_iteration; ++i) {
    uint32_t* row = ids + i * z->sample_len;
    uint64_t have = 0;
    while (have < z->sample_len) {
      uint32_t id = zipf_draw(z);
      int dup = 0;
      for (uint64_t t = 0; t < have; ++t)
        if (row[t] == id) { dup = 1; break; }
      if (!dup) row[have++] = id;
    }
  }
  ++z->emitted;
  return 1;
}

/* ZipfStream::reset — workload.hpp:121-124 */
void orc_zipf_reset(orc_zipf* z) {
  mt64_seed(&z->rng, z->seed);
  z->emitted = 0;
}

/* cmd_bench input — experiment.hpp:217-223 */
void orc_bench_matrix(uint64_t k, double* out) {
  mt64 g;
  mt64_seed(&g, 0x5eedULL ^ k);
  for (uint64_t i = 0; i < k * k; ++i) out[i] = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
}

/* --------------------------------------------------- id -> index hash map */
/* Open addressing with tombstones; a plain container, no reference
 * counterpart beyond std::unordered_map. */

typedef struct {
  uint32_t* keys;
  int32_t* vals; /* -1 empty, -2 tombstone */
  uint64_t cap, used, live;
} idmap;

static uint64_t hmix(uint32_t k) {
  uint64_t x = (uint64_t)k * 0x9E3779B97F4A7C15ULL;
  return x ^ (x >> 29);
}

static void idmap_init(idmap* m, uint64_t cap) {
  uint64_t c = 16;
  while (c < cap * 2) c <<= 1;
  m->cap = c;
  m->keys = (uint32_t*)malloc(sizeof(uint32_t) * c);
  m->vals = (int32_t*)malloc(sizeof(int32_t) * c);
  for (uint64_t i = 0; i < c; ++i) m->vals[i] = -1;
  m->used = m->live = 0;
}

static void idmap_free(idmap* m) {
  free(m->keys);
  free(m->vals);
}

static int32_t idmap_get(const idmap* m, uint32_t k) {
  uint64_t mask = m->cap - 1, i = hmix(k) & mask;
  for (;;) {
    int32_t v = m->vals[i];
    if (v == -1) return -1;
    if (v >= 0 && m->keys[i] == k) return v;
    i = (i + 1) & mask;
  }
}

static void idmap_put(idmap* m, uint32_t k, int32_t val);

static void idmap_grow(idmap* m) {
  idmap n;
  idmap_init(&n, m->live * 2 + 16);
  for (uint64_t i = 0; i < m->cap; ++i)
    if (m->vals[i] >= 0) idmap_put(&n, m->keys[i], m->vals[i]);
  idmap_free(m);
  *m = n;
}

/* insert or overwrite */
static void idmap_put(idmap* m, uint32_t k, int32_t val) {
  if ((m->used + 1) * 4 > m->cap * 3) idmap_grow(m);
  uint64_t mask = m->cap - 1, i = hmix(k) & mask;
  int64_t tomb = -1;
  for (;;) {
    int32_t v = m->vals[i];
    if (v == -1) break;
    if (v == -2) {
      if (tomb < 0) tomb = (int64_t)i;
    } else if (m->keys[i] == k) {
      m->vals[i] = val;
      return;
    }
    i = (i + 1) & mask;
  }
  if (tomb >= 0) i = (uint64_t)tomb;
  else ++m->used;
  m->keys[i] = k;
  m->vals[i] = val;
  ++m->live;
}

static void idmap_del(idmap* m, uint32_t k) {
  uint64_t mask = m->cap - 1, i = hmix(k) & mask;
  for (;;) {
    int32_t v = m->vals[i];
    if (v == -1) return;
    if (v >= 0 && m->keys[i] == k) {
      m->vals[i] = -2;
      --m->live;
      return;
    }
    i = (i + 1) & mask;
  }
}

/* -------------------------------------------------------------- snapshot */
/* Snapshot::state_of — cost.hpp:39-48: unknown ids are {0,0,0}. */

typedef struct {
  idmap map;
  uint32_t* ids;
  uint64_t *owners, *latest, *resident;
  uint64_t count, cap;
} gstate;

static void gstate_init(gstate* g, uint64_t cap) {
  if (cap < 16) cap = 16;
  idmap_init(&g->map, cap);
  g->cap = cap;
  g->count = 0;
  g->ids = (uint32_t*)malloc(sizeof(uint32_t) * cap);
  g->owners = (uint64_t*)malloc(sizeof(uint64_t) * cap);
  g->latest = (uint64_t*)malloc(sizeof(uint64_t) * cap);
  g->resident = (uint64_t*)malloc(sizeof(uint64_t) * cap);
}

static void gstate_free(gstate* g) {
  idmap_free(&g->map);
  free(g->ids);
  free(g->owners);
  free(g->latest);
  free(g->resident);
}

/* global_[id] with default insertion (sim.hpp:169, 179, 195); never erased */
static int64_t gstate_ref(gstate* g, uint32_t id) {
  int32_t x = idmap_get(&g->map, id);
  if (x >= 0) return x;
  if (g->count == g->cap) {
    g->cap *= 2;
    g->ids = (uint32_t*)realloc(g->ids, sizeof(uint32_t) * g->cap);
    g->owners = (uint64_t*)realloc(g->owners, sizeof(uint64_t) * g->cap);
    g->latest = (uint64_t*)realloc(g->latest, sizeof(uint64_t) * g->cap);
    g->resident = (uint64_t*)realloc(g->resident, sizeof(uint64_t) * g->cap);
  }
  int64_t i = (int64_t)g->count++;
  g->ids[i] = id;
  g->owners[i] = g->latest[i] = g->resident[i] = 0;
  idmap_put(&g->map, id, (int32_t)i);
  return i;
}

/* ------------------------------------------------------------- cost build */

/* expected_cost — cost.hpp:81-100: left-to-right fp64 chain, pull on the
 * worker, then one push per other owner in ascending worker order. */
static double expected_cost(const orc_cluster_config* cfg, const gstate* g,
                            const uint32_t* ids, uint64_t len, int j) {
  double cost = 0.0;
  for (uint64_t t = 0; t < len; ++t) {
    int32_t x = idmap_get(&g->map, ids[t]);
    uint64_t owners = x >= 0 ? g->owners[x] : 0, latest = x >= 0 ? g->latest[x] : 0;
    if ((latest >> j) & 1ULL) continue;
    cost += unit(cfg, j);
    uint64_t others = owners & ~(1ULL << j);
    while (others) {
      int o = __builtin_ctzll(others);
      others &= others - 1;
      cost += unit(cfg, o);
    }
  }
  return cost;
}

/* build_matrix — cost.hpp:105-125 */
static int build_matrix(const orc_cluster_config* cfg, const gstate* g, const uint32_t* ids,
                        const uint64_t* offsets, uint64_t R, double* out) {
  uint64_t want = (uint64_t)cfg->n * (uint64_t)cfg->m;
  if (R != want)
    return fail(ORC_INVALID_ARGUMENT, "expected %llu samples, got %llu",
                (unsigned long long)want, (unsigned long long)R);
  for (uint64_t i = 0; i < R; ++i)
    for (int j = 0; j < cfg->n; ++j)
      out[i * (uint64_t)cfg->n + (uint64_t)j] =
          expected_cost(cfg, g, ids + offsets[i], offsets[i + 1] - offsets[i], j);
  return ORC_OK;
}

int orc_build_matrix_snapshot(const orc_cluster_config* cfg, const uint32_t* snap_ids,
                              const uint64_t* snap_owners, const uint64_t* snap_latest,
                              const uint64_t* snap_resident, uint64_t snap_count,
                              const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                              double* out) {
  gstate g;
  gstate_init(&g, snap_count + 16);
  for (uint64_t s = 0; s < snap_count; ++s) {
    int64_t x = gstate_ref(&g, snap_ids[s]);
    g.owners[x] = snap_owners[s];
    g.latest[x] = snap_latest[s];
    g.resident[x] = snap_resident ? snap_resident[s] : 0;
  }
  int rc = build_matrix(cfg, &g, ids, offsets, R, out);
  gstate_free(&g);
  return rc;
}

/* detail::transfer_seconds with a SizeLookupFn (cost.hpp:68-73):
 * bytes * 8.0 / bw, mul then div; expected_cost's chain is unchanged. */
int orc_expected_costs_sized(const orc_cluster_config* cfg, const uint32_t* snap_ids,
                             const uint64_t* snap_owners, const uint64_t* snap_latest,
                             uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                             uint64_t R, const uint64_t* sizes, double* out) {
  gstate g;
  gstate_init(&g, snap_count + 16);
  for (uint64_t s = 0; s < snap_count; ++s) {
    int64_t x = gstate_ref(&g, snap_ids[s]);
    g.owners[x] = snap_owners[s];
    g.latest[x] = snap_latest[s];
  }
  for (uint64_t i = 0; i < R; ++i) {
    for (int j = 0; j < cfg->n; ++j) {
      double cost = 0.0;
      for (uint64_t t = offsets[i]; t < offsets[i + 1]; ++t) {
        int32_t x = idmap_get(&g.map, ids[t]);
        uint64_t owners = x >= 0 ? g.owners[x] : 0, latest = x >= 0 ? g.latest[x] : 0;
        if ((latest >> j) & 1ULL) continue;
        const double bytes = (double)sizes[t];
        cost += bytes * 8.0 / cfg->bandwidths_bps[j];
        uint64_t others = owners & ~(1ULL << j);
        while (others) {
          int o = __builtin_ctzll(others);
          others &= others - 1;
          cost += bytes * 8.0 / cfg->bandwidths_bps[o];
        }
      }
      out[i * (uint64_t)cfg->n + (uint64_t)j] = cost;
    }
  }
  gstate_free(&g);
  return ORC_OK;
}

/* baseline_hitgreedy — assign.hpp:346-392.  A sample scores worker j by how
 * many of its ids have their latest copy on j; samples commit in order of
 * best score (desc), index (asc); each takes its best-scoring worker with
 * workload left, ties to the larger remaining workload, then the lower index
 * (strict comparisons over ascending j). */
typedef struct {
  int best;
  uint64_t index;
} hg_key;

static int hg_cmp(const void* a, const void* b) {
  const hg_key* x = (const hg_key*)a;
  const hg_key* y = (const hg_key*)b;
  if (x->best != y->best) return x->best > y->best ? -1 : 1;
  return x->index < y->index ? -1 : (x->index > y->index ? 1 : 0);
}

static int hitgreedy(const orc_cluster_config* cfg, const gstate* g, const uint32_t* ids,
                     const uint64_t* offsets, uint64_t R, int32_t* decision) {
  if (R != (uint64_t)cfg->n * (uint64_t)cfg->m)
    return fail(ORC_INVALID_ARGUMENT, "sample count must be m*n");
  const int n = cfg->n;
  int* score = (int*)calloc(R * (uint64_t)n + 1, sizeof(int));
  hg_key* order = (hg_key*)malloc(sizeof(hg_key) * (R ? R : 1));
  int* remaining = (int*)malloc(sizeof(int) * (uint64_t)n);
  for (uint64_t i = 0; i < R; ++i) {
    int* sc = score + i * (uint64_t)n;
    for (uint64_t t = offsets[i]; t < offsets[i + 1]; ++t) {
      int32_t x = idmap_get(&g->map, ids[t]);
      uint64_t holders = x >= 0 ? g->latest[x] : 0;
      while (holders) {
        ++sc[__builtin_ctzll(holders)];
        holders &= holders - 1;
      }
    }
    int best = sc[0];
    for (int j = 1; j < n; ++j)
      if (sc[j] > best) best = sc[j];
    order[i].best = best;
    order[i].index = i;
  }
  qsort(order, R, sizeof(hg_key), hg_cmp); /* total order: index breaks ties */
  for (int j = 0; j < n; ++j) remaining[j] = cfg->m;
  for (uint64_t t = 0; t < R; ++t) {
    const uint64_t i = order[t].index;
    const int* sc = score + i * (uint64_t)n;
    int best = -1;
    for (int j = 0; j < n; ++j) {
      if (remaining[j] <= 0) continue;
      if (best < 0 || sc[j] > sc[best] || (sc[j] == sc[best] && remaining[j] > remaining[best]))
        best = j;
    }
    --remaining[best];
    decision[i] = best;
  }
  free(score);
  free(order);
  free(remaining);
  return ORC_OK;
}

int orc_hitgreedy_snapshot(const orc_cluster_config* cfg, const uint32_t* snap_ids,
                           const uint64_t* snap_owners, const uint64_t* snap_latest,
                           uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                           uint64_t R, int32_t* decision) {
  gstate g;
  gstate_init(&g, snap_count + 16);
  for (uint64_t s = 0; s < snap_count; ++s) {
    int64_t x = gstate_ref(&g, snap_ids[s]);
    g.owners[x] = snap_owners[s];
    g.latest[x] = snap_latest[s];
  }
  int rc = hitgreedy(cfg, &g, ids, offsets, R, decision);
  gstate_free(&g);
  return rc;
}

/* row_gap_key — cost.hpp:130-146 */
static double gap_of(uint64_t cols, const double* row) {
  if (cols == 1) return 0.0;
  double smallest = INFINITY, second = INFINITY;
  for (uint64_t c = 0; c < cols; ++c) {
    double v = row[c];
    if (v < smallest) {
      second = smallest;
      smallest = v;
    } else if (v < second) {
      second = v;
    }
  }
  return second - smallest;
}

int orc_row_gap_key(uint64_t rows, uint64_t cols, const double* values, uint64_t row,
                    double* out) {
  if (cols == 0) return fail(ORC_INVALID_ARGUMENT, "row is empty");
  if (row >= rows) return fail(ORC_INVALID_ARGUMENT, "row index out of range");
  *out = gap_of(cols, values + row * cols);
  return ORC_OK;
}

/* rows_by_gap — assign.hpp:197-207: gap descending, index ascending */
static int gap_cmp(const void* a, const void* b, void* ctx) {
  const double* gap = (const double*)ctx;
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  if (gap[x] != gap[y]) return gap[x] > gap[y] ? -1 : 1;
  return x < y ? -1 : (x > y ? 1 : 0);
}

int orc_rows_by_gap(uint64_t rows, uint64_t cols, const double* values, uint64_t* order) {
  if (cols == 0 && rows > 0) return fail(ORC_INVALID_ARGUMENT, "row is empty");
  double* gap = (double*)malloc(sizeof(double) * (rows ? rows : 1));
  for (uint64_t r = 0; r < rows; ++r) {
    gap[r] = gap_of(cols, values + r * cols);
    order[r] = r;
  }
  qsort_r(order, rows, sizeof(uint64_t), gap_cmp, gap);
  free(gap);
  return ORC_OK;
}

/* ---------------------------------------------------------------- solver */

static __thread uint64_t g_hung_steps;
uint64_t orc_last_hungarian_steps(void) { return g_hung_steps; }

/* hungarian — assign.hpp:80-157: integer-scaled e-maxx shortest augmenting
 * paths; rows 1..k in order, strict '<' keeps the lowest column on ties. */
static int hungarian_core(uint64_t k, const double* values, uint64_t* col_of_row,
                          double* total) {
  if (k < 1) return fail(ORC_INVALID_ARGUMENT, "solver needs at least one row");
  for (uint64_t i = 0; i < k * k; ++i)
    if (!isfinite(values[i]) || values[i] < 0.0)
      return fail(ORC_INVALID_ARGUMENT, "costs must be finite and non-negative");
  const int64_t kInf = INT64_MAX;
  const int64_t cap = kInf / (8 * (int64_t)(k + 1));
  int64_t* cost = (int64_t*)malloc(sizeof(int64_t) * k * k);
  for (uint64_t i = 0; i < k * k; ++i) {
    int64_t scaled = (int64_t)llround(values[i] * 1e12);
    cost[i] = scaled < cap ? scaled : cap;
  }
  int64_t* u = (int64_t*)calloc(k + 1, sizeof(int64_t));
  int64_t* v = (int64_t*)calloc(k + 1, sizeof(int64_t));
  uint64_t* p = (uint64_t*)calloc(k + 1, sizeof(uint64_t));
  uint64_t* way = (uint64_t*)calloc(k + 1, sizeof(uint64_t));
  int64_t* minv = (int64_t*)malloc(sizeof(int64_t) * (k + 1));
  char* used = (char*)malloc(k + 1);
  uint64_t steps = 0;
  for (uint64_t i = 1; i <= k; ++i) {
    p[0] = i;
    uint64_t j0 = 0;
    for (uint64_t j = 0; j <= k; ++j) {
      minv[j] = kInf;
      used[j] = 0;
    }
    do {
      ++steps;
      used[j0] = 1;
      uint64_t i0 = p[j0], j1 = 0;
      int64_t delta = kInf;
      const int64_t* row = cost + (i0 - 1) * k;
      for (uint64_t j = 1; j <= k; ++j) {
        if (used[j]) continue;
        int64_t cur = row[j - 1] - u[i0] - v[j];
        if (cur < minv[j]) {
          minv[j] = cur;
          way[j] = j0;
        }
        if (minv[j] < delta) {
          delta = minv[j];
          j1 = j;
        }
      }
      for (uint64_t j = 0; j <= k; ++j) {
        if (used[j]) {
          u[p[j]] += delta;
          v[j] -= delta;
        } else if (minv[j] != kInf) {
          minv[j] -= delta;
        }
      }
      j0 = j1;
    } while (p[j0] != 0);
    do {
      uint64_t j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    } while (j0 != 0);
  }
  for (uint64_t j = 1; j <= k; ++j) col_of_row[p[j] - 1] = j - 1;
  double t = 0.0;
  for (uint64_t i = 0; i < k; ++i) t += values[i * k + col_of_row[i]];
  if (total) *total = t;
  g_hung_steps = steps;
  free(cost);
  free(u);
  free(v);
  free(p);
  free(way);
  free(minv);
  free(used);
  return ORC_OK;
}

int orc_hungarian(uint64_t k, const double* values, uint64_t* col_of_row, double* total) {
  return hungarian_core(k, values, col_of_row, total);
}

/* greedy_dispatch — assign.hpp:162-192 */
int orc_greedy_dispatch(uint64_t rows, uint64_t cols, const double* values,
                        const uint64_t* order, uint64_t n_order, const int32_t* capacity_in,
                        uint64_t* out_rows, int32_t* out_workers) {
  long total = 0;
  for (uint64_t j = 0; j < cols; ++j) total += capacity_in[j];
  if (total != (long)n_order)
    return fail(ORC_INVALID_ARGUMENT, "capacities must sum to the number of rows");
  int32_t* capacity = (int32_t*)malloc(sizeof(int32_t) * (cols ? cols : 1));
  memcpy(capacity, capacity_in, sizeof(int32_t) * cols);
  for (uint64_t t = 0; t < n_order; ++t) {
    uint64_t row = order[t];
    if (row >= rows) {
      free(capacity);
      return fail(ORC_INVALID_ARGUMENT, "row index out of range");
    }
    int32_t best = -1;
    double best_cost = INFINITY;
    for (uint64_t j = 0; j < cols; ++j) {
      if (capacity[j] <= 0) continue;
      double c = values[row * cols + j];
      if (c < best_cost) {
        best_cost = c;
        best = (int32_t)j;
      }
    }
    if (best < 0) {
      free(capacity);
      return fail(ORC_LOGIC_ERROR, "capacities exhausted before rows");
    }
    --capacity[best];
    out_rows[t] = row;
    out_workers[t] = best;
  }
  free(capacity);
  return ORC_OK;
}

/* detail::exact_multiplicity — assign.hpp:213-216 */
static int exact_multiplicity(int m, double alpha) {
  int mult = (int)floor(m * alpha + 1e-9);
  if (mult < 0) mult = 0;
  if (mult > m) mult = m;
  return mult;
}

/* DispatchDecision::validate — assign.hpp:41-57 */
static int validate_decision(const orc_cluster_config* cfg, const int32_t* w, uint64_t count) {
  if (count != (uint64_t)cfg->n * (uint64_t)cfg->m)
    return fail(ORC_INVALID_ARGUMENT, "decision does not cover m*n samples");
  int* load = (int*)calloc((size_t)cfg->n, sizeof(int));
  for (uint64_t i = 0; i < count; ++i) {
    if (w[i] < 0 || w[i] >= cfg->n) {
      free(load);
      return fail(ORC_INVALID_ARGUMENT, "worker id out of range");
    }
    ++load[w[i]];
  }
  for (int j = 0; j < cfg->n; ++j)
    if (load[j] != cfg->m) {
      int got = load[j];
      free(load);
      return fail(ORC_INVALID_ARGUMENT, "worker %d received %d samples, expected %d", j, got,
                  cfg->m);
    }
  free(load);
  return ORC_OK;
}

/* ecomix — assign.hpp:247-285 (with expand_columns, assign.hpp:223-241) */
int orc_ecomix(const orc_cluster_config* cfg, uint64_t rows, uint64_t cols,
               const double* values, const uint64_t* row_ids, int32_t* decision) {
  if (rows != (uint64_t)cfg->n * (uint64_t)cfg->m || cols != (uint64_t)cfg->n)
    return fail(ORC_INVALID_ARGUMENT, "matrix shape does not match cluster config");
  uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * rows);
  orc_rows_by_gap(rows, cols, values, order);
  int mult = exact_multiplicity(cfg->m, cfg->alpha);
  uint64_t exact_rows = (uint64_t)cfg->n * (uint64_t)mult;
  for (uint64_t i = 0; i < rows; ++i) decision[i] = -1;
  int rc = ORC_OK;
  if (mult > 0) {
    uint64_t k = exact_rows;
    double* sq = (double*)malloc(sizeof(double) * k * k);
    for (uint64_t r = 0; r < k; ++r)
      for (uint64_t c = 0; c < k; ++c) sq[r * k + c] = values[order[r] * cols + c / (uint64_t)mult];
    uint64_t* col_of_row = (uint64_t*)malloc(sizeof(uint64_t) * k);
    rc = hungarian_core(k, sq, col_of_row, NULL);
    if (rc == ORC_OK)
      for (uint64_t r = 0; r < k; ++r) {
        uint64_t s = row_ids ? row_ids[order[r]] : order[r];
        decision[s] = (int32_t)(col_of_row[r] / (uint64_t)mult);
      }
    free(sq);
    free(col_of_row);
  }
  if (rc == ORC_OK && exact_rows < rows) {
    uint64_t nrest = rows - exact_rows;
    int32_t* capacity = (int32_t*)malloc(sizeof(int32_t) * cols);
    for (uint64_t j = 0; j < cols; ++j) capacity[j] = cfg->m - mult;
    uint64_t* orows = (uint64_t*)malloc(sizeof(uint64_t) * nrest);
    int32_t* oworkers = (int32_t*)malloc(sizeof(int32_t) * nrest);
    rc = orc_greedy_dispatch(rows, cols, values, order + exact_rows, nrest, capacity, orows,
                             oworkers);
    if (rc == ORC_OK)
      for (uint64_t t = 0; t < nrest; ++t) {
        uint64_t s = row_ids ? row_ids[orows[t]] : orows[t];
        decision[s] = oworkers[t];
      }
    free(capacity);
    free(orows);
    free(oworkers);
  }
  free(order);
  if (rc == ORC_OK) rc = validate_decision(cfg, decision, rows);
  return rc;
}

/* decision_cost — assign.hpp:288-298 */
int orc_decision_cost(uint64_t rows, uint64_t cols, const double* values,
                      const int32_t* decision, double* out) {
  double total = 0.0;
  for (uint64_t i = 0; i < rows; ++i) total += values[i * cols + (uint64_t)decision[i]];
  *out = total;
  return ORC_OK;
}

/* ----------------------------------------------------------- worker cache */
/* WorkerCache (kMarkVersion policy) — cache.hpp:73-240.  The std::set of
 * VictimKeys is replaced by a linear scan for the least key; the victim is
 * the same because the key order (cache.hpp:47-58) is total. */

typedef struct {
  uint64_t capacity, size;
  uint32_t current_mark;
  uint64_t at_current;
  idmap map; /* id -> slot */
  uint32_t* id;
  uint8_t* version;
  uint32_t *mark, *freq;
  uint64_t* last;
  double* fp; /* standalone caches only: FootprintFn(id) per slot */
} wcache;

static void wcache_init(wcache* c, uint64_t capacity) {
  c->capacity = capacity;
  c->size = 0;
  c->current_mark = 1;
  c->at_current = 0;
  idmap_init(&c->map, capacity < (1u << 20) ? capacity : (1u << 20));
  c->id = (uint32_t*)malloc(sizeof(uint32_t) * capacity);
  c->version = (uint8_t*)malloc(capacity);
  c->mark = (uint32_t*)malloc(sizeof(uint32_t) * capacity);
  c->freq = (uint32_t*)malloc(sizeof(uint32_t) * capacity);
  c->last = (uint64_t*)malloc(sizeof(uint64_t) * capacity);
  c->fp = NULL;
}

static void wcache_free(wcache* c) {
  idmap_free(&c->map);
  free(c->id);
  free(c->version);
  free(c->mark);
  free(c->freq);
  free(c->last);
  free(c->fp);
}

/* touch — cache.hpp:102-122 */
static int wcache_touch(wcache* c, uint32_t id, int latest, uint64_t now) {
  int32_t s = idmap_get(&c->map, id);
  if (s < 0) {
    if (c->size == c->capacity)
      return fail(ORC_LOGIC_ERROR, "touch would insert into a full cache; evict first");
    uint64_t t = c->size++;
    c->id[t] = id;
    c->version[t] = (uint8_t)(latest != 0);
    c->mark[t] = c->current_mark;
    c->freq[t] = 1;
    c->last[t] = now;
    idmap_put(&c->map, id, (int32_t)t);
    ++c->at_current;
    return ORC_OK;
  }
  if (c->mark[s] != c->current_mark) ++c->at_current;
  c->mark[s] = c->current_mark;
  c->freq[s] += 1;
  c->last[s] = now;
  c->version[s] = (uint8_t)(latest != 0);
  return ORC_OK;
}

/* set_version — cache.hpp:126-135 */
static int wcache_set_version(wcache* c, uint32_t id, int latest) {
  int32_t s = idmap_get(&c->map, id);
  if (s < 0) return fail(ORC_INVALID_ARGUMENT, "set_version on non-resident embedding");
  c->version[s] = (uint8_t)(latest != 0);
  return ORC_OK;
}

/* erase — cache.hpp:172-178 */
static void wcache_erase(wcache* c, uint32_t id) {
  int32_t s = idmap_get(&c->map, id);
  if (s < 0) return;
  if (c->mark[s] == c->current_mark) --c->at_current;
  idmap_del(&c->map, id);
  uint64_t last = c->size - 1;
  if ((uint64_t)s != last) {
    c->id[s] = c->id[last];
    c->version[s] = c->version[last];
    c->mark[s] = c->mark[last];
    c->freq[s] = c->freq[last];
    c->last[s] = c->last[last];
    if (c->fp) c->fp[s] = c->fp[last];
    idmap_put(&c->map, c->id[s], s);
  }
  --c->size;
}

/* VictimKey order — cache.hpp:47-58 */
static int key_less(const wcache* c, uint64_t a, uint64_t b) {
  if (c->version[a] != c->version[b]) return c->version[a] < c->version[b];
  if (c->mark[a] != c->mark[b]) return c->mark[a] < c->mark[b];
  if (c->freq[a] != c->freq[b]) return c->freq[a] < c->freq[b];
  if (c->last[a] != c->last[b]) return c->last[a] < c->last[b];
  return c->id[a] < c->id[b];
}

/* pick_victim (kMarkVersion) — cache.hpp:194-201: least key not pinned */
static int64_t wcache_pick(const wcache* c, const idmap* pinned) {
  int64_t best = -1;
  for (uint64_t s = 0; s < c->size; ++s) {
    if (pinned && idmap_get(pinned, c->id[s]) >= 0) continue;
    if (best < 0 || key_less(c, s, (uint64_t)best)) best = (int64_t)s;
  }
  return best;
}

/* ---------------------------------------------- standalone WorkerCache */

struct orc_cache {
  wcache w;
  int policy;
};

int orc_cache_create(uint64_t capacity, int policy, orc_cache** out) {
  if (capacity == 0) return fail(ORC_INVALID_ARGUMENT, "cache capacity must be positive");
  orc_cache* c = (orc_cache*)calloc(1, sizeof *c);
  wcache_init(&c->w, capacity);
  c->w.fp = (double*)malloc(sizeof(double) * capacity);
  c->policy = policy;
  *out = c;
  return ORC_OK;
}

void orc_cache_destroy(orc_cache* c) {
  if (!c) return;
  wcache_free(&c->w);
  free(c);
}

int orc_cache_touch(orc_cache* c, uint32_t id, int latest, uint64_t now, double footprint) {
  int inserting = idmap_get(&c->w.map, id) < 0;
  int rc = wcache_touch(&c->w, id, latest, now);
  if (rc == ORC_OK && inserting) c->w.fp[c->w.size - 1] = footprint;
  return rc;
}

int orc_cache_set_version(orc_cache* c, uint32_t id, int latest) {
  return wcache_set_version(&c->w, id, latest);
}

int orc_cache_erase(orc_cache* c, uint32_t id) {
  wcache_erase(&c->w, id);
  return ORC_OK;
}

/* pick_victim (kPriorityRatio) — cache.hpp:203-230: least
 * (version ? 2 : 1) * mark * frequency / footprint, then last access, then id */
static int64_t wcache_pick_ratio(const wcache* c, const idmap* pinned) {
  int64_t best = -1;
  double bp = 0.0;
  for (uint64_t s = 0; s < c->size; ++s) {
    if (pinned && idmap_get(pinned, c->id[s]) >= 0) continue;
    const double num = (c->version[s] ? 2.0 : 1.0) * (double)c->mark[s] * (double)c->freq[s];
    const double pr = num / c->fp[s];
    int better = best < 0 || pr < bp ||
                 (pr == bp && (c->last[s] < c->last[best] ||
                               (c->last[s] == c->last[best] && c->id[s] < c->id[best])));
    if (better) {
      best = (int64_t)s;
      bp = pr;
    }
  }
  return best;
}

static int64_t cache_pick(const orc_cache* c, const idmap* pinned) {
  return c->policy ? wcache_pick_ratio(&c->w, pinned) : wcache_pick(&c->w, pinned);
}

/* select_victim — cache.hpp:141-148 */
int orc_cache_select_victim(orc_cache* c, uint32_t* victim) {
  if (c->w.size != c->w.capacity)
    return fail(ORC_LOGIC_ERROR, "select_victim requires a full cache");
  int64_t s = cache_pick(c, NULL);
  if (s < 0) return fail(ORC_LOGIC_ERROR, "no evictable entry");
  *victim = c->w.id[s];
  return ORC_OK;
}

/* evict_for — cache.hpp:152-170 (maybe_advance_mark :187-192 first) */
int orc_cache_evict_for(orc_cache* c, uint64_t needed, const uint32_t* pinned, uint64_t n_pinned,
                        uint32_t* victims, uint64_t* n_victims) {
  wcache* w = &c->w;
  *n_victims = 0;
  if (needed > w->capacity)
    return fail(ORC_INVALID_ARGUMENT, "cannot free more slots than the capacity");
  if (w->capacity - w->size >= needed) return ORC_OK;
  if (w->size == w->capacity && w->at_current == w->size) {
    ++w->current_mark;
    w->at_current = 0;
  }
  idmap pins;
  idmap_init(&pins, n_pinned + 16);
  for (uint64_t q = 0; q < n_pinned; ++q) idmap_put(&pins, pinned[q], 1);
  int rc = ORC_OK;
  while (w->capacity - w->size < needed) {
    int64_t s = cache_pick(c, &pins);
    if (s < 0) {
      rc = fail(ORC_LOGIC_ERROR, "every cache entry is pinned; cannot evict");
      break;
    }
    victims[(*n_victims)++] = w->id[s];
    wcache_erase(w, w->id[s]);
  }
  idmap_free(&pins);
  return rc;
}

void orc_cache_info(orc_cache* c, uint64_t* size, uint32_t* current_mark) {
  *size = c->w.size;
  *current_mark = c->w.current_mark;
}

static const wcache* g_sort_cache;
static int slot_by_id(const void* a, const void* b) {
  uint32_t x = g_sort_cache->id[*(const uint64_t*)a], y = g_sort_cache->id[*(const uint64_t*)b];
  return x < y ? -1 : (x > y ? 1 : 0);
}

void orc_cache_export(orc_cache* c, uint32_t* ids, uint8_t* version, uint32_t* mark,
                      uint32_t* freq, uint64_t* last_access) {
  const wcache* w = &c->w;
  uint64_t* ord = (uint64_t*)malloc(sizeof(uint64_t) * (w->size + 1));
  for (uint64_t s = 0; s < w->size; ++s) ord[s] = s;
  g_sort_cache = w;
  qsort(ord, w->size, sizeof(uint64_t), slot_by_id);
  for (uint64_t t = 0; t < w->size; ++t) {
    ids[t] = w->id[ord[t]];
    version[t] = w->version[ord[t]];
    mark[t] = w->mark[ord[t]];
    freq[t] = w->freq[ord[t]];
    last_access[t] = w->last[ord[t]];
  }
  free(ord);
}

/* ------------------------------------------------------------ the engine */

struct orc_sim {
  orc_cluster_config cfg;
  double* bw;
  gstate g;
  wcache* caches;
  uint64_t clock;
};

int orc_sim_create(const orc_cluster_config* cfg, orc_sim** out) {
  if (cfg->n < 1 || cfg->n > 64) return fail(ORC_INVALID_ARGUMENT, "worker count out of range");
  if (cfg->cache_capacity == 0)
    return fail(ORC_INVALID_ARGUMENT, "cache capacity must be positive");
  orc_sim* s = (orc_sim*)calloc(1, sizeof *s);
  s->cfg = *cfg;
  s->bw = (double*)malloc(sizeof(double) * (size_t)cfg->n);
  memcpy(s->bw, cfg->bandwidths_bps, sizeof(double) * (size_t)cfg->n);
  s->cfg.bandwidths_bps = s->bw;
  gstate_init(&s->g, 1024);
  s->caches = (wcache*)calloc((size_t)cfg->n, sizeof(wcache));
  for (int j = 0; j < cfg->n; ++j) wcache_init(&s->caches[j], cfg->cache_capacity);
  *out = s;
  return ORC_OK;
}

void orc_sim_destroy(orc_sim* s) {
  if (!s) return;
  for (int j = 0; j < s->cfg.n; ++j) wcache_free(&s->caches[j]);
  free(s->caches);
  gstate_free(&s->g);
  free(s->bw);
  free(s);
}

uint64_t orc_sim_clock(orc_sim* s) { return s->clock; }

int orc_sim_build_matrix(orc_sim* s, const uint32_t* ids, const uint64_t* offsets,
                         uint64_t R, double* out) {
  return build_matrix(&s->cfg, &s->g, ids, offsets, R, out);
}

int orc_sim_hitgreedy(orc_sim* s, const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                      int32_t* decision) {
  return hitgreedy(&s->cfg, &s->g, ids, offsets, R, decision);
}

/* seed_entry — sim.hpp:252-261 */
int orc_sim_seed_entry(orc_sim* s, uint32_t id, int32_t worker, int latest, int owner) {
  if (owner && !latest) return fail(ORC_INVALID_ARGUMENT, "an owner's copy is always latest");
  if (worker < 0 || worker >= s->cfg.n) return fail(ORC_INVALID_ARGUMENT, "worker out of range");
  int rc = wcache_touch(&s->caches[worker], id, latest, s->clock);
  if (rc) return rc;
  int64_t x = gstate_ref(&s->g, id);
  s->g.resident[x] |= 1ULL << worker;
  if (latest) s->g.latest[x] |= 1ULL << worker;
  if (owner) s->g.owners[x] |= 1ULL << worker;
  return ORC_OK;
}

/* SimState::step — sim.hpp:87-218 */
int orc_sim_step(orc_sim* s, const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                 const int32_t* decision, orc_report* rep) {
  const orc_cluster_config* cfg = &s->cfg;
  const int n = cfg->n;
  int rc = validate_decision(cfg, decision, R);
  if (rc) return rc;
  uint64_t total = offsets[R] - offsets[0];

  rep->iteration = s->clock;
  rep->miss_pull = rep->update_push = rep->evict_push = rep->hits = rep->lookups = 0;
  rep->cost_s = 0.0;
  for (int j = 0; j < n; ++j) {
    rep->miss_pull_w[j] = rep->update_push_w[j] = rep->evict_push_w[j] = 0;
    rep->cost_w[j] = 0.0;
  }

  /* needs — sim.hpp:103-117: per-worker first-occurrence order + counts,
   * per-id trainer masks.  uniq lists ids in first appearance order. */
  idmap* need = (idmap*)calloc((size_t)n, sizeof(idmap));
  uint32_t** need_order = (uint32_t**)calloc((size_t)n, sizeof(uint32_t*));
  uint64_t* need_len = (uint64_t*)calloc((size_t)n, sizeof(uint64_t));
  uint32_t** need_cnt = (uint32_t**)calloc((size_t)n, sizeof(uint32_t*));
  for (int j = 0; j < n; ++j) {
    idmap_init(&need[j], total / (uint64_t)n + 16);
    need_order[j] = (uint32_t*)malloc(sizeof(uint32_t) * (total + 1));
    need_cnt[j] = (uint32_t*)malloc(sizeof(uint32_t) * (total + 1));
  }
  idmap tmap;
  idmap_init(&tmap, total + 16);
  uint32_t* uniq = (uint32_t*)malloc(sizeof(uint32_t) * (total + 1));
  uint64_t* umask = (uint64_t*)malloc(sizeof(uint64_t) * (total + 1));
  uint64_t nuniq = 0;
  for (uint64_t i = 0; i < R; ++i) {
    int j = decision[i];
    for (uint64_t t = offsets[i]; t < offsets[i + 1]; ++t) {
      uint32_t id = ids[t];
      ++rep->lookups;
      int32_t x = idmap_get(&need[j], id);
      if (x >= 0) {
        ++need_cnt[j][x];
        continue;
      }
      uint64_t pos = need_len[j]++;
      need_order[j][pos] = id;
      need_cnt[j][pos] = 1;
      idmap_put(&need[j], id, (int32_t)pos);
      int32_t u = idmap_get(&tmap, id);
      if (u < 0) {
        u = (int32_t)nuniq++;
        uniq[u] = id;
        umask[u] = 0;
        idmap_put(&tmap, id, u);
      }
      umask[u] |= 1ULL << j;
    }
  }

  /* Phase 1: on-demand update push — sim.hpp:119-153 */
  for (uint64_t u = 0; u < nuniq && rc == ORC_OK; ++u) {
    int32_t x = idmap_get(&s->g.map, uniq[u]);
    if (x < 0 || s->g.owners[x] == 0) continue;
    uint64_t need_mask = umask[u], pushers = 0, owners = s->g.owners[x];
    while (owners) {
      int w = __builtin_ctzll(owners);
      owners &= owners - 1;
      if ((need_mask & ~(1ULL << w)) != 0) pushers |= 1ULL << w;
    }
    if (!pushers) continue;
    for (uint64_t it = pushers; it; it &= it - 1) ++rep->update_push_w[__builtin_ctzll(it)];
    s->g.owners[x] &= ~pushers;
    if (s->g.owners[x] != 0) {
      for (uint64_t st = s->g.latest[x] & ~s->g.owners[x]; st && rc == ORC_OK; st &= st - 1)
        rc = wcache_set_version(&s->caches[__builtin_ctzll(st)], uniq[u], 0);
      s->g.latest[x] = s->g.owners[x];
    }
  }

  /* Phase 2: per-worker lookups, evictions, miss pulls — sim.hpp:155-190 */
  for (int j = 0; j < n && rc == ORC_OK; ++j) {
    wcache* c = &s->caches[j];
    const uint64_t bit = 1ULL << j;
    for (uint64_t t = 0; t < need_len[j] && rc == ORC_OK; ++t) {
      uint32_t id = need_order[j][t];
      int64_t x = gstate_ref(&s->g, id);
      if (s->g.latest[x] & bit) {
        rep->hits += need_cnt[j][t];
        rc = wcache_touch(c, id, 1, s->clock);
        continue;
      }
      if (!(s->g.resident[x] & bit) && c->size == c->capacity) {
        /* evict_for(1, owner_is_self, &pinned) — cache.hpp:152-170 */
        if (c->at_current == c->size) { /* maybe_advance_mark — cache.hpp:187-192 */
          ++c->current_mark;
          c->at_current = 0;
        }
        int64_t v = wcache_pick(c, &need[j]);
        if (v < 0) {
          rc = fail(ORC_LOGIC_ERROR, "every cache entry is pinned; cannot evict");
          break;
        }
        uint32_t victim = c->id[v];
        int64_t vx = gstate_ref(&s->g, victim);
        x = gstate_ref(&s->g, id); /* arrays may have moved */
        if (s->g.owners[vx] & bit) ++rep->evict_push_w[j];
        wcache_erase(c, victim);
        s->g.owners[vx] &= ~bit;
        s->g.latest[vx] &= ~bit;
        s->g.resident[vx] &= ~bit;
      }
      ++rep->miss_pull_w[j];
      rc = wcache_touch(c, id, 1, s->clock);
      s->g.latest[x] |= bit;
      s->g.resident[x] |= bit;
    }
  }

  /* Phase 3: ownership hand-over — sim.hpp:192-204 */
  for (uint64_t u = 0; u < nuniq && rc == ORC_OK; ++u) {
    int64_t x = gstate_ref(&s->g, uniq[u]);
    uint64_t mask = umask[u];
    for (uint64_t st = s->g.latest[x] & ~mask; st && rc == ORC_OK; st &= st - 1)
      rc = wcache_set_version(&s->caches[__builtin_ctzll(st)], uniq[u], 0);
    s->g.owners[x] = mask;
    s->g.latest[x] = mask;
  }

  if (rc == ORC_OK) {
    ++s->clock; /* sim.hpp:206 */
    /* per-worker totals and realised cost, j order — sim.hpp:208-216 */
    for (int j = 0; j < n; ++j) {
      rep->miss_pull += rep->miss_pull_w[j];
      rep->update_push += rep->update_push_w[j];
      rep->evict_push += rep->evict_push_w[j];
      uint64_t ops = rep->miss_pull_w[j] + rep->update_push_w[j] + rep->evict_push_w[j];
      rep->cost_w[j] = (double)ops * unit(cfg, j);
      rep->cost_s += rep->cost_w[j];
    }
  }

  for (int j = 0; j < n; ++j) {
    idmap_free(&need[j]);
    free(need_order[j]);
    free(need_cnt[j]);
  }
  free(need);
  free(need_order);
  free(need_len);
  free(need_cnt);
  idmap_free(&tmap);
  free(uniq);
  free(umask);
  return rc;
}

/* validate_consistency — sim.hpp:222-248 */
int orc_sim_validate_consistency(orc_sim* s) {
  for (int j = 0; j < s->cfg.n; ++j) {
    wcache* c = &s->caches[j];
    for (uint64_t t = 0; t < c->size; ++t) {
      int32_t x = idmap_get(&s->g.map, c->id[t]);
      uint64_t res = x >= 0 ? s->g.resident[x] : 0, lat = x >= 0 ? s->g.latest[x] : 0;
      if (!((res >> j) & 1ULL))
        return fail(ORC_LOGIC_ERROR, "cache entry missing from global resident set");
      if ((int)c->version[t] != (int)((lat >> j) & 1ULL))
        return fail(ORC_LOGIC_ERROR, "version flag diverged from global state");
    }
  }
  for (uint64_t x = 0; x < s->g.count; ++x) {
    uint64_t o = s->g.owners[x], l = s->g.latest[x], r = s->g.resident[x];
    int ok = ((o & ~l) == 0) && ((l & ~r) == 0) && !(o != 0 && l != o);
    if (!ok)
      return fail(ORC_LOGIC_ERROR, "embedding state invariant violated for id %u", s->g.ids[x]);
    for (uint64_t it = r; it; it &= it - 1)
      if (idmap_get(&s->caches[__builtin_ctzll(it)].map, s->g.ids[x]) < 0)
        return fail(ORC_LOGIC_ERROR, "global resident bit without a cache entry");
  }
  return ORC_OK;
}

uint64_t orc_sim_global_count(orc_sim* s) { return s->g.count; }

void orc_sim_export_global(orc_sim* s, uint32_t* ids, uint64_t* owners, uint64_t* latest,
                           uint64_t* resident) {
  for (uint64_t x = 0; x < s->g.count; ++x) {
    ids[x] = s->g.ids[x];
    owners[x] = s->g.owners[x];
    latest[x] = s->g.latest[x];
    resident[x] = s->g.resident[x];
  }
}

uint64_t orc_sim_cache_size(orc_sim* s, int32_t worker) { return s->caches[worker].size; }

void orc_sim_export_cache(orc_sim* s, int32_t worker, uint32_t* ids, uint8_t* version,
                          uint32_t* mark, uint32_t* freq, uint64_t* last_access) {
  wcache* c = &s->caches[worker];
  for (uint64_t t = 0; t < c->size; ++t) {
    ids[t] = c->id[t];
    version[t] = c->version[t];
    mark[t] = c->mark[t];
    freq[t] = c->freq[t];
    last_access[t] = c->last[t];
  }
}

void orc_sim_cache_marks(orc_sim* s, int32_t worker, uint32_t* current_mark,
                         uint64_t* at_current_mark) {
  *current_mark = s->caches[worker].current_mark;
  *at_current_mark = s->caches[worker].at_current;
}

/* Parity import: replaces the clock, the global table and every cache. */
int orc_sim_import_state(orc_sim* s, uint64_t clock, uint64_t g_count, const uint32_t* g_ids,
                         const uint64_t* g_owners, const uint64_t* g_latest,
                         const uint64_t* g_resident, const uint64_t* entry_off,
                         const uint32_t* e_ids, const uint8_t* e_version, const uint32_t* e_mark,
                         const uint32_t* e_freq, const uint64_t* e_last,
                         const uint32_t* current_mark, const uint64_t* at_current_mark) {
  for (int j = 0; j < s->cfg.n; ++j)
    if (entry_off[j + 1] - entry_off[j] > s->cfg.cache_capacity)
      return fail(ORC_INVALID_ARGUMENT, "imported cache exceeds its capacity");
  gstate_free(&s->g);
  gstate_init(&s->g, g_count + 16);
  for (uint64_t t = 0; t < g_count; ++t) {
    const int64_t x = gstate_ref(&s->g, g_ids[t]);
    s->g.owners[x] = g_owners[t];
    s->g.latest[x] = g_latest[t];
    s->g.resident[x] = g_resident[t];
  }
  for (int j = 0; j < s->cfg.n; ++j) {
    wcache* c = &s->caches[j];
    wcache_free(c);
    wcache_init(c, s->cfg.cache_capacity);
    for (uint64_t t = entry_off[j]; t < entry_off[j + 1]; ++t) {
      const uint64_t k = c->size++;
      c->id[k] = e_ids[t];
      c->version[k] = e_version[t] ? 1 : 0;
      c->mark[k] = e_mark[t];
      c->freq[k] = e_freq[t];
      c->last[k] = e_last[t];
      idmap_put(&c->map, e_ids[t], (int32_t)k);
    }
    c->current_mark = current_mark[j];
    c->at_current = at_current_mark[j];
  }
  s->clock = clock;
  return ORC_OK;
}

/* One iteration of run() — sim.hpp:421-441 — for the "port" CPU baseline
 * when oracle/_ref is absent.  The snapshot is free here (the build reads the
 * live state), so times_s[0] is 0. */
#include <pthread.h>
#include <time.h>

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct {
  orc_sim* s;
  const uint32_t* ids;
  const uint64_t* offsets;
  uint64_t lo, hi;
  double* out;
} build_job;

static void* build_rows(void* arg) {
  build_job* b = (build_job*)arg;
  for (uint64_t i = b->lo; i < b->hi; ++i)
    for (int j = 0; j < b->s->cfg.n; ++j)
      b->out[i * (uint64_t)b->s->cfg.n + (uint64_t)j] = expected_cost(
          &b->s->cfg, &b->s->g, b->ids + b->offsets[i], b->offsets[i + 1] - b->offsets[i], j);
  return NULL;
}

int orc_ref_iteration(orc_sim* s, const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                      int threads, int32_t* decision, double* expected_cost_out,
                      orc_report* rep, double* times_s) {
  const int n = s->cfg.n;
  if (R != (uint64_t)n * (uint64_t)s->cfg.m)
    return fail(ORC_INVALID_ARGUMENT, "expected %llu samples, got %llu",
                (unsigned long long)((uint64_t)n * (uint64_t)s->cfg.m), (unsigned long long)R);
  double* matrix = (double*)malloc(sizeof(double) * R * (uint64_t)n);
  int32_t* dec = decision ? decision : (int32_t*)malloc(sizeof(int32_t) * R);
  double t1 = now_s();
  if (threads <= 1) {
    build_job b = {s, ids, offsets, 0, R, matrix};
    build_rows(&b);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    build_job* jobs = (build_job*)malloc(sizeof(build_job) * (size_t)threads);
    uint64_t chunk = (R + (uint64_t)threads - 1) / (uint64_t)threads;
    for (int t = 0; t < threads; ++t) {
      uint64_t lo = (uint64_t)t * chunk, hi = lo + chunk < R ? lo + chunk : R;
      if (lo > hi) lo = hi;
      jobs[t] = (build_job){s, ids, offsets, lo, hi, matrix};
      pthread_create(&th[t], NULL, build_rows, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
  }
  double t2 = now_s();
  int rc = orc_ecomix(&s->cfg, R, (uint64_t)n, matrix, NULL, dec);
  double t3 = now_s();
  uint64_t mp[64], up[64], ep[64];
  double cw[64];
  orc_report local = {0, 0, 0, 0, 0, 0, 0.0, mp, up, ep, cw};
  if (rc == ORC_OK) rc = orc_sim_step(s, ids, offsets, R, dec, rep ? rep : &local);
  double t4 = now_s();
  if (rc == ORC_OK && expected_cost_out)
    orc_decision_cost(R, (uint64_t)n, matrix, dec, expected_cost_out);
  if (times_s) {
    times_s[0] = 0.0;
    times_s[1] = t2 - t1;
    times_s[2] = t3 - t2;
    times_s[3] = t4 - t3;
  }
  if (!decision) free(dec);
  free(matrix);
  return rc;
}
