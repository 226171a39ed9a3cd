// C ABI of libedx (include/edx.h): the engine (SimState on device) and the
// stateless matrix-level API.  Host code here only validates arguments,
// moves buffers and sequences kernels on the engine's stream; every
// reference computation runs in the CUDA kernels of cost.cu, dispatch.cu,
// hungarian.cu and step.cu.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include "engine.h"
#include "nccl_comm.h"
#include "step.h"

using edx::DevBuf;
using edx::Error;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return EDX_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return EDX_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EDX_RUNTIME_ERROR;
  }
}

}  // namespace

void edx::set_last_error(const char* m) { g_err = m; }

namespace {

constexpr int kT = 256;
unsigned grid_for(uint64_t n) { return static_cast<unsigned>(std::max<uint64_t>(1, (n + kT - 1) / kT)); }

// ---------------------------------------------------------------- config
// validate(const ClusterConfig&, size_t) — types.hpp:87-108, same messages.
void validate_cfg(const edx_cluster_config* c, uint64_t max_len) {
  if (!c) edx::invalid("null cluster config");
  if (c->n < 1) edx::invalid("worker count must be >= 1");
  if (c->n > 64) edx::invalid("at most 64 workers supported");
  if (c->m < 1) edx::invalid("batch size per worker must be >= 1");
  if (c->n_bandwidths != c->n) edx::invalid("need one bandwidth per worker");
  for (int j = 0; j < c->n; ++j)
    if (!(c->bandwidths_bps[j] > 0.0)) edx::invalid("bandwidths must be positive");
  if (c->d_tran_bytes == 0) edx::invalid("d_tran must be positive");
  if (c->alpha < 0.0 || c->alpha > 1.0) edx::invalid("alpha must lie in [0, 1]");
  const uint64_t micro = static_cast<uint64_t>(c->m) * max_len;
  if (c->cache_capacity < micro)
    edx::invalid("cache capacity " + std::to_string(c->cache_capacity) +
                 " cannot hold one micro-batch of " + std::to_string(micro) + " embeddings");
}

// unit_cost — types.hpp:112-120: d_tran * 8.0 / bw, one direction.
std::vector<double> unit_costs(const edx_cluster_config* c) {
  std::vector<double> u(static_cast<size_t>(c->n));
  for (int j = 0; j < c->n; ++j) u[j] = static_cast<double>(c->d_tran_bytes) * 8.0 / c->bandwidths_bps[j];
  return u;
}

void check_flags_host(const int* f) {
  if (f[edx::kFlagIdOutOfRange]) edx::invalid("embedding id outside the engine's id_space");
  if (f[edx::kFlagBadCost]) edx::invalid("costs must be finite and non-negative");
  if (f[edx::kFlagPinned]) edx::logic("every cache entry is pinned; cannot evict");
  if (f[edx::kFlagUnbalanced]) edx::logic("capacities exhausted before rows");
  if (f[edx::kFlagInternal]) throw Error(EDX_RUNTIME_ERROR, "internal error: solver shared-memory layout");
  if (f[edx::kFlagKeyRange])
    throw Error(EDX_RUNTIME_ERROR, "victim key fields exceed the 57-bit device packing");
  if (f[edx::kFlagBadBatch])
    edx::invalid("device offsets must start at 0 and end at the declared id count");
}

// device batch with a declared id count: offsets[0] == 0 and offsets[R] == total,
// checked on the device (no host round trip), reported at the next sync
__global__ void k_check_batch(const uint64_t* __restrict__ offsets, uint64_t R, uint64_t total,
                              int* flags) {
  if (offsets[0] != 0 || offsets[R] != total) atomicOr(flags + edx::kFlagBadBatch, 1);
}

// ------------------------------------------------------- small kernels
__global__ void k_import(const uint32_t* __restrict__ ids, const unsigned long long* __restrict__ ow,
                         const unsigned long long* __restrict__ la,
                         const unsigned long long* __restrict__ re, uint64_t count,
                         uint64_t id_space, ulonglong2* __restrict__ ol,
                         unsigned long long* __restrict__ res, int* flags) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x >= count) return;
  const uint32_t id = ids[x];
  if (id >= id_space) {
    atomicOr(flags + edx::kFlagIdOutOfRange, 1);
    return;
  }
  ol[id] = make_ulonglong2(ow[x], la[x]);
  if (res) res[id] = re ? re[x] : 0ULL;
}

__global__ void k_export_global(const ulonglong2* __restrict__ ol,
                                const unsigned long long* __restrict__ res, uint64_t id_space,
                                const uint32_t* __restrict__ slot2id,
                                uint32_t* __restrict__ ids, unsigned long long* __restrict__ out,
                                uint64_t cap, unsigned long long* __restrict__ count) {
  const uint64_t id = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (id >= id_space) return;
  const ulonglong2 st = ol[id];
  const unsigned long long r = res[id];
  if ((st.x | st.y | r) == 0) return;
  const unsigned long long at = atomicAdd(count, 1ULL);
  if (at < cap) {
    ids[at] = slot2id ? slot2id[id] : static_cast<uint32_t>(id);
    out[3 * at] = st.x;
    out[3 * at + 1] = st.y;
    out[3 * at + 2] = r;
  }
}

// WorkerCache::touch (cache.hpp:102-122) + the mask updates of seed_entry
// (sim.hpp:252-261), one entry.
__global__ void k_seed_entry(uint32_t id, int j, int latest, int owner, uint32_t clock,
                             uint64_t capacity, uint64_t id_space, ulonglong2* ol,
                             unsigned long long* res, int32_t* slot_of, uint32_t* sid,
                             uint32_t* smark, uint32_t* sfreq, uint32_t* slast, uint32_t* size,
                             const uint32_t* cur_mark, unsigned long long* at_cur, int* status) {
  const uint64_t so = static_cast<uint64_t>(j) * id_space + id;
  int32_t s = slot_of[so];
  const uint32_t cm = cur_mark[j];
  if (s < 0) {
    if (size[j] == capacity) {
      *status = 1;  // touch would insert into a full cache
      return;
    }
    s = static_cast<int32_t>(size[j]++);
    const uint64_t g = static_cast<uint64_t>(j) * capacity + s;
    slot_of[so] = s;
    sid[g] = id;
    smark[g] = cm;
    sfreq[g] = 1;
    slast[g] = clock;
    at_cur[j] += 1;
  } else {
    const uint64_t g = static_cast<uint64_t>(j) * capacity + s;
    if (smark[g] != cm) at_cur[j] += 1;
    smark[g] = cm;
    sfreq[g] += 1;
    slast[g] = clock;
  }
  const unsigned long long bit = 1ULL << j;
  res[id] |= bit;
  if (latest) ol[id].y |= bit;
  if (owner) ol[id].x |= bit;
  *status = 0;
}

__global__ void k_fill_slots(int32_t* p, uint64_t n) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x < n) p[x] = -1;
}

__global__ void k_fill_value(int32_t* p, uint64_t n, int32_t v) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x < n) p[x] = v;
}

// Parity import of worker j's cache entries into slots [0, count): the slot
// arrays, the id -> slot index, and a check that each entry's version flag
// equals bit j of the imported `latest` mask (sim.hpp:229-231).
__global__ void k_import_entries(int j, uint64_t count, uint64_t capacity, uint64_t id_space,
                                 const uint32_t* __restrict__ ids, const uint8_t* __restrict__ ver,
                                 const uint32_t* __restrict__ mark, const uint32_t* __restrict__ freq,
                                 const uint64_t* __restrict__ last, const ulonglong2* __restrict__ ol,
                                 int32_t* __restrict__ slot_of, uint32_t* __restrict__ sid,
                                 uint32_t* __restrict__ smark, uint32_t* __restrict__ sfreq,
                                 uint32_t* __restrict__ slast, int* __restrict__ status) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x >= count) return;
  const uint32_t id = ids[x];
  if (id >= id_space) {
    atomicOr(status + 0, 1);
    return;
  }
  if (last[x] > 0xFFFFFFFFull) atomicOr(status + 1, 1);
  if (ver && static_cast<uint64_t>(ver[x] != 0) != ((ol[id].y >> j) & 1ULL)) atomicOr(status + 2, 1);
  int32_t* so = slot_of + static_cast<uint64_t>(j) * id_space + id;
  if (atomicCAS(so, -1, static_cast<int32_t>(x)) != -1) atomicOr(status + 3, 1);  // duplicate id
  const uint64_t g = static_cast<uint64_t>(j) * capacity + x;
  sid[g] = id;
  smark[g] = mark[x];
  sfreq[g] = freq[x];
  slast[g] = static_cast<uint32_t>(last[x]);
}

// validate_consistency (sim.hpp:222-248) over the device tables.
// status: [0] entry without resident bit, [1] invariant violated (+id in [3]),
// [2] resident bit without entry, [4] at_current_mark drift
__global__ void k_validate_slots(int n, uint64_t capacity, uint64_t id_space,
                                 const uint32_t* __restrict__ size, const uint32_t* __restrict__ sid,
                                 const unsigned long long* __restrict__ res,
                                 const int32_t* __restrict__ slot_of, const uint32_t* smark,
                                 const uint32_t* cur_mark, unsigned long long* at_count,
                                 int* status) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x >= static_cast<uint64_t>(n) * capacity) return;
  const int j = static_cast<int>(x / capacity);
  const uint32_t s = static_cast<uint32_t>(x - static_cast<uint64_t>(j) * capacity);
  if (s >= size[j]) return;
  const uint32_t id = sid[x];
  if (!((res[id] >> j) & 1ULL) || slot_of[static_cast<uint64_t>(j) * id_space + id] != static_cast<int32_t>(s))
    atomicOr(status + 0, 1);
  if (smark[x] == cur_mark[j]) atomicAdd(at_count + j, 1ULL);
}

__global__ void k_validate_ids(int n, uint64_t id_space, const ulonglong2* __restrict__ ol,
                               const unsigned long long* __restrict__ res,
                               const int32_t* __restrict__ slot_of,
                               const uint32_t* __restrict__ slot2id, int* status) {
  const uint64_t id = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (id >= id_space) return;
  const ulonglong2 st = ol[id];
  const unsigned long long r = res[id];
  const bool ok = ((st.x & ~st.y) == 0) && ((st.y & ~r) == 0) && !(st.x != 0 && st.y != st.x);
  if (!ok) {
    if (atomicOr(status + 1, 1) == 0)
      status[3] = static_cast<int>(slot2id ? slot2id[id] : static_cast<uint32_t>(id));
  }
  for (unsigned long long it = r; it; it &= it - 1) {
    const int w = __ffsll(static_cast<long long>(it)) - 1;
    if (w >= n || slot_of[static_cast<uint64_t>(w) * id_space + id] < 0) atomicOr(status + 2, 1);
  }
}

__global__ void k_export_cache(int j, uint64_t capacity, uint32_t count,
                               const uint32_t* __restrict__ sid, const ulonglong2* __restrict__ ol,
                               const uint32_t* __restrict__ slot2id, uint8_t* __restrict__ ver,
                               uint32_t* __restrict__ ids) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  const uint32_t slot = sid[static_cast<uint64_t>(j) * capacity + s];
  ver[s] = static_cast<uint8_t>((ol[slot].y >> j) & 1ULL);
  ids[s] = slot2id ? slot2id[slot] : slot;
}

// sum_i values[i*stride + col[i]] left to right (hungarian total, assign.hpp:153-155)
__global__ void k_seq_gather_sum(const double* __restrict__ values, uint64_t k,
                                 const uint64_t* __restrict__ col, double* out) {
  double t = 0.0;
  for (uint64_t i = 0; i < k; ++i) t = __dadd_rn(t, values[i * k + col[i]]);
  *out = t;
}

__global__ void k_seq_gather_sum_blocks(const double* __restrict__ matrix, int n,
                                        const uint64_t* __restrict__ rows, uint64_t k, int mult,
                                        const uint64_t* __restrict__ col, double* out) {
  double t = 0.0;
  for (uint64_t i = 0; i < k; ++i)
    t = __dadd_rn(t, matrix[rows[i] * n + col[i] / static_cast<uint64_t>(mult)]);
  *out = t;
}

__global__ void k_u64_to_u32(const uint64_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ b) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x < n) b[x] = static_cast<uint32_t>(a[x]);
}

__global__ void k_u32_to_u64(const uint32_t* __restrict__ a, uint64_t n, uint64_t* __restrict__ b) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x < n) b[x] = a[x];
}

__global__ void k_pair_rows(const uint64_t* __restrict__ order, uint64_t n, uint64_t* __restrict__ rows) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x < n) rows[x] = order[x];
}

// -------------------------------------------------- process default context
struct DefaultCtx {
  std::mutex mu;
  int device = -1;
  cudaStream_t stream = nullptr;
  edx::DispatchScratch disp;
  edx::HitScratch hit;
  DevBuf<double> values;
  DevBuf<uint32_t> ids, u32a, u32b;
  DevBuf<uint64_t> offsets, u64a, u64b;
  DevBuf<int32_t> i32a, i32b;
  DevBuf<unsigned long long> snapA, snapB, snapC;
  DevBuf<ulonglong2> ol;
  DevBuf<double> ucost, scalar, bw;
  DevBuf<uint64_t> sizes;
  DevBuf<int> flags;

  void init() {
    if (device >= 0) return;
    int count = 0;
    EDX_CUDA(cudaGetDeviceCount(&count));
    if (count <= 0) throw Error(EDX_CUDA_ERROR, "no CUDA device");
    EDX_CUDA(cudaGetDevice(&device));
    EDX_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    flags.ensure(edx::kFlagCount);
    scalar.ensure(4);
  }
  void reset_flags() { EDX_CUDA(cudaMemsetAsync(flags.p, 0, edx::kFlagCount * sizeof(int), stream)); }
  void sync_and_check() {
    int f[edx::kFlagCount];
    EDX_CUDA(cudaMemcpyAsync(f, flags.p, sizeof f, cudaMemcpyDeviceToHost, stream));
    EDX_CUDA(cudaStreamSynchronize(stream));
    check_flags_host(f);
  }
};

DefaultCtx& dctx() {
  static DefaultCtx* c = new DefaultCtx;  // never destroyed: outlives CUDA teardown ordering
  return *c;
}

// ------------------------------------------------------------ engine helpers
void engine_sync_check(edx_engine* e) {
  EDX_CUDA(cudaMemcpyAsync(e->h_flags, e->flags.p, edx::kFlagCount * sizeof(int),
                           cudaMemcpyDeviceToHost, e->stream));
  EDX_CUDA(cudaStreamSynchronize(e->stream));
  int f[edx::kFlagCount];
  std::memcpy(f, e->h_flags, sizeof f);
  if (std::any_of(f, f + edx::kFlagCount, [](int v) { return v != 0; })) {
    EDX_CUDA(cudaMemsetAsync(e->flags.p, 0, edx::kFlagCount * sizeof(int), e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    check_flags_host(f);
  }
  if (e->profiling) {
    auto acc = [&](int a, int b, int phase) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, e->ev[a], e->ev[b]) == cudaSuccess) e->phase_ms[phase] += ms;
    };
    if (e->pending_build) acc(0, 1, 0);
    if (e->pending_dispatch) {
      acc(2, 3, 1);
      acc(4, 5, 2);
      if (e->pending_greedy) acc(6, 7, 3);
      acc(10, 11, 5);
    }
    if (e->pending_step) acc(8, 9, 4);
  }
  e->pending_build = e->pending_dispatch = e->pending_step = e->pending_greedy = false;
  cudaGetLastError();
}

void rec(edx_engine* e, int idx, cudaStream_t s) {
  if (e->profiling) EDX_CUDA(cudaEventRecord(e->ev[idx], s));
}

void engine_load(edx_engine* e, const uint32_t* ids, const uint64_t* offsets, uint64_t R,
                 int on_device, uint64_t declared_total = UINT64_MAX) {
  if (R == 0) edx::invalid("batch holds no samples");
  uint64_t total;
  if (on_device && declared_total != UINT64_MAX) {
    total = declared_total;
    k_check_batch<<<1, 1, 0, e->stream>>>(offsets, R, total, e->flags.p);
    EDX_LAUNCHED();
    e->cur_ids = ids;
    e->cur_offsets = offsets;
  } else if (on_device) {
    uint64_t ends[2];
    EDX_CUDA(cudaMemcpyAsync(&ends[0], offsets, sizeof(uint64_t), cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(&ends[1], offsets + R, sizeof(uint64_t), cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    if (ends[0] != 0) edx::invalid("device offsets must start at 0");
    total = ends[1];
    e->cur_ids = ids;
    e->cur_offsets = offsets;
  } else {
    const uint64_t base = offsets[0];
    for (uint64_t i = 0; i < R; ++i)
      if (offsets[i + 1] < offsets[i]) edx::invalid("sample offsets must be non-decreasing");
    total = offsets[R] - base;
    if (total > e->max_ids)
      edx::invalid("batch holds " + std::to_string(total) + " ids; engine max_batch_ids is " +
                   std::to_string(e->max_ids));
    e->h_offsets.assign(offsets, offsets + R + 1);
    if (base)
      for (auto& o : e->h_offsets) o -= base;
    e->offsets.ensure(R + 1);
    EDX_CUDA(cudaMemcpyAsync(e->ids.p, ids + base, total * sizeof(uint32_t), cudaMemcpyHostToDevice,
                             e->stream));
    EDX_CUDA(cudaMemcpyAsync(e->offsets.p, e->h_offsets.data(), (R + 1) * sizeof(uint64_t),
                             cudaMemcpyHostToDevice, e->stream));
    e->cur_ids = e->ids.p;
    e->cur_offsets = e->offsets.p;
  }
  if (total > e->max_ids)
    edx::invalid("batch holds " + std::to_string(total) + " ids; engine max_batch_ids is " +
                 std::to_string(e->max_ids));
  e->rows = R;
  e->total_ids = total;
  e->built = e->dispatched = e->expected_ready = false;
  e->cur_raw = e->cur_ids;
  if (e->hashed) {  // kernels read the slot stream, translated before first use
    e->cur_ids = e->kslots.p;
    e->translated = false;
  }
}

// ---------------------------------------------------- arbitrary ids (ids.cu)
// Reallocates the slot-indexed tables (global masks, per-worker cache index,
// the step's first-occurrence table) for `cap` slots, keeping the first
// `used` slots, and rebuilds the id table.  Between iterations only.
void grow_slots(edx_engine* e, uint64_t need) {
  const uint64_t kMax = 0xFFFFFFF0ull;
  if (need > kMax) edx::invalid("more than 2^32 - 16 distinct embedding ids");
  const uint64_t old = e->id_space, used = e->idt.used;
  const uint64_t cap = std::min(kMax, std::max(4 * old, 2 * need));
  EDX_CUDA(cudaStreamSynchronize(e->step_side));
  EDX_CUDA(cudaStreamSynchronize(e->stream));
  const int n = e->n;
  DevBuf<ulonglong2> ol;
  DevBuf<unsigned long long> res;
  DevBuf<int32_t> so, fp;
  ol.ensure(cap);
  res.ensure(cap);
  so.ensure(static_cast<uint64_t>(n) * cap);
  fp.ensure(cap);
  EDX_CUDA(cudaMemsetAsync(ol.p, 0, cap * sizeof(ulonglong2), e->stream));
  EDX_CUDA(cudaMemsetAsync(res.p, 0, cap * sizeof(unsigned long long), e->stream));
  k_fill_slots<<<grid_for(static_cast<uint64_t>(n) * cap), kT, 0, e->stream>>>(so.p, static_cast<uint64_t>(n) * cap);
  k_fill_value<<<grid_for(cap), kT, 0, e->stream>>>(fp.p, cap, INT_MAX);
  EDX_LAUNCHED();
  if (used) {
    EDX_CUDA(cudaMemcpyAsync(ol.p, e->ol.p, used * sizeof(ulonglong2), cudaMemcpyDeviceToDevice, e->stream));
    EDX_CUDA(cudaMemcpyAsync(res.p, e->res.p, used * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, e->stream));
    EDX_CUDA(cudaMemcpy2DAsync(so.p, cap * sizeof(int32_t), e->cache.slot_of.p, old * sizeof(int32_t),
                               used * sizeof(int32_t), n, cudaMemcpyDeviceToDevice, e->stream));
  }
  e->ol.swap(ol);
  e->res.swap(res);
  e->cache.slot_of.swap(so);
  e->step.first_pos.swap(fp);
  edx::id_table_grow(e->idt, cap, e->stream);
  e->id_space = cap;
}

// Makes room for `T` new ids before a translation (exact count read back
// only when the running bound says the table might be short).
void reserve_slots(edx_engine* e, uint64_t T) {
  if (e->used_bound + T <= e->idt.cap) return;
  if (e->capturing) edx::invalid("id table full during graph capture");
  EDX_CUDA(cudaStreamSynchronize(e->stream));
  unsigned long long used = 0;
  EDX_CUDA(cudaMemcpy(&used, e->idt.count.p, sizeof used, cudaMemcpyDeviceToHost));
  e->idt.used = used;
  e->used_bound = used;
  if (used + T > e->idt.cap) grow_slots(e, used + T);
}

// Translates the loaded batch to slots (hashed mode) before its first consumer.
void ensure_translated(edx_engine* e) {
  if (!e->hashed || e->translated) return;
  const edx::NvtxRange nv("edx.translate (ids.cu)");
  reserve_slots(e, e->total_ids);
  edx::id_table_translate(e->idt, e->cur_raw, e->total_ids, e->kslots.p, true, e->flags.p,
                          e->stream);
  e->used_bound += e->total_ids;
  e->translated = true;
  e->launches += 1;
}

// Slots of host ids (dense mode: the ids), inserting new ids when `insert`;
// absent ids map to 0xFFFFFFFF when not inserting.
std::vector<uint32_t> host_slots(edx_engine* e, const uint32_t* ids, uint64_t count, bool insert) {
  std::vector<uint32_t> out(ids, ids + count);
  if (!e->hashed || count == 0) return out;
  if (insert) reserve_slots(e, count);
  DevBuf<uint32_t> din, dout;
  din.ensure(count);
  dout.ensure(count);
  EDX_CUDA(cudaMemcpyAsync(din.p, ids, count * 4, cudaMemcpyHostToDevice, e->stream));
  edx::id_table_translate(e->idt, din.p, count, dout.p, insert, e->flags.p, e->stream);
  EDX_CUDA(cudaMemcpyAsync(out.data(), dout.p, count * 4, cudaMemcpyDeviceToHost, e->stream));
  engine_sync_check(e);
  if (insert) e->used_bound += count;
  return out;
}

void engine_build(edx_engine* e) {
  const edx::NvtxRange nv("edx.build (K1 cost.hpp:105-125)");
  const uint64_t want = static_cast<uint64_t>(e->n) * static_cast<uint64_t>(e->m);
  if (!e->cur_ids) edx::invalid("no batch loaded");
  ensure_translated(e);
  if (e->rows != want)
    edx::invalid("expected " + std::to_string(want) + " samples, got " + std::to_string(e->rows));
  e->matrix.ensure(e->rows * e->n);
  e->disp.gap_keys.ensure(e->rows);
  e->disp.row_index.ensure(e->rows);
  if (!e->capturing) EDX_CUDA(cudaStreamWaitEvent(e->stream, e->cost_done, 0));
  rec(e, 0, e->stream);
  if (e->world == 1) {
    edx::launch_cost_build(e->cur_ids, e->cur_offsets, e->rows, e->n, e->ol.p, e->id_space,
                           e->ucost.p, e->matrix.p, e->disp.gap_keys.p, e->disp.row_index.p,
                           e->flags.p, e->stream);
    e->gap_ready = true;
    e->kname[edx::kKBuild] = edx::g_kernel_name[edx::kKBuild];
  } else {
    // row shards (samples are independent, cost.hpp:102-104), gathered to rank 0
    std::vector<uint64_t> lo(e->world), hi(e->world);
    edx::shard_rows(e->rows, e->world, lo.data(), hi.data());
    const uint64_t a = lo[e->rank], b = hi[e->rank];
    if (b > a)
      edx::launch_cost_build(e->cur_ids, e->cur_offsets + a, b - a, e->n, e->ol.p, e->id_space,
                             e->ucost.p, e->matrix.p + a * e->n, nullptr, nullptr, e->flags.p,
                             e->stream);
    e->kname[edx::kKBuild] = edx::g_kernel_name[edx::kKBuild];
    edx::NcclTransport tr(e->comm, e->stream);
    edx::gather_rows(tr, e->matrix.p, lo.data(), hi.data(), e->world, e->rank, 0, e->n);
    e->gap_ready = false;
  }
  rec(e, 1, e->stream);
  e->launches += 1;
  e->pending_build = e->profiling;
  e->built = true;
}

void engine_dispatch(edx_engine* e, double alpha) {
  const edx::NvtxRange nv("edx.dispatch (ecomix assign.hpp:247-285)");
  if (!e->built) edx::invalid("build the cost matrix before dispatching");
  if (alpha < 0.0) alpha = e->alpha;
  if (alpha > 1.0) edx::invalid("alpha must lie in [0, 1]");
  e->decision.ensure(e->rows + 2);
  e->expected.ensure(1);
  edx::PhaseEvents pe;
  if (e->profiling) {
    pe.sort0 = e->ev[2];
    pe.sort1 = e->ev[3];
    pe.exact0 = e->ev[4];
    pe.exact1 = e->ev[5];
    pe.greedy0 = e->ev[6];
    pe.greedy1 = e->ev[7];
  }
  int launches = 0;
  rec(e, 10, e->stream);
  if (e->rank == 0) {
    edx::g_kernel_name[edx::kKSolver] = edx::g_kernel_name[edx::kKGreedy] = "";
    edx::run_ecomix(e->disp, e->matrix.p, e->rows, e->n, e->m, alpha, e->gap_ready,
                    e->decision.p, e->flags.p, e->stream, e->device, e->profiling ? &pe : nullptr,
                    &launches);
    e->kname[edx::kKSolver] = edx::g_kernel_name[edx::kKSolver];
    e->kname[edx::kKGreedy] = edx::g_kernel_name[edx::kKGreedy];
  }
  rec(e, 11, e->stream);
  if (e->world == 1) {
    // decision_cost is only reported (sim.hpp:439): overlap it with the step.
    EDX_CUDA(cudaEventRecord(e->disp.fork, e->stream));
    EDX_CUDA(cudaStreamWaitEvent(e->disp.side, e->disp.fork, 0));
    edx::launch_decision_cost(e->matrix.p, e->decision.p, e->rows, e->n, e->expected.p,
                              e->disp.side);
    EDX_CUDA(cudaEventRecord(e->cost_done, e->disp.side));
  } else {
    // the decision goes out first; rank 0 (the only rank holding the gathered
    // matrix) computes decision_cost on its side stream, overlapping the step,
    // and the expected cost is broadcast only when a caller asks for it
    edx::NcclTransport tr(e->comm, e->stream);
    edx::broadcast_decision(tr, e->decision.p, e->rows, 0);
    if (e->rank == 0) {
      EDX_CUDA(cudaEventRecord(e->disp.fork, e->stream));
      EDX_CUDA(cudaStreamWaitEvent(e->disp.side, e->disp.fork, 0));
      edx::launch_decision_cost(e->matrix.p, e->decision.p, e->rows, e->n, e->expected.p,
                                e->disp.side);
      EDX_CUDA(cudaEventRecord(e->cost_done, e->disp.side));
    } else {
      EDX_CUDA(cudaEventRecord(e->cost_done, e->stream));
    }
  }
  e->launches += launches + 1;
  const int mult = edx::exact_multiplicity(e->m, alpha);
  e->pending_greedy = e->profiling && static_cast<uint64_t>(e->n) * mult < e->rows;
  e->pending_dispatch = e->profiling;
  e->dispatched = e->expected_ready = true;
}

// DispatchDecision::validate — assign.hpp:41-57, same messages.
void validate_decision_host(const int32_t* w, uint64_t count, int n, int m) {
  if (count != static_cast<uint64_t>(n) * static_cast<uint64_t>(m))
    edx::invalid("decision does not cover m*n samples");
  std::vector<int> load(static_cast<size_t>(n), 0);
  for (uint64_t i = 0; i < count; ++i) {
    if (w[i] < 0 || w[i] >= n) edx::invalid("worker id out of range");
    ++load[w[i]];
  }
  for (int j = 0; j < n; ++j)
    if (load[j] != m)
      edx::invalid("worker " + std::to_string(j) + " received " + std::to_string(load[j]) +
                   " samples, expected " + std::to_string(m));
}

// The iteration's expected_cost_s (decision_cost, sim.hpp:439) on the host;
// multi-GPU engines broadcast rank 0's value (every rank must call this).
double fetch_expected(edx_engine* e) {
  EDX_CUDA(cudaStreamWaitEvent(e->stream, e->cost_done, 0));
  if (e->world > 1) {
    edx::NcclTransport tr(e->comm, e->stream);
    edx::broadcast_cost(tr, e->expected.p, 0);
  }
  EDX_CUDA(cudaMemcpyAsync(e->h_expected, e->expected.p, sizeof(double), cudaMemcpyDeviceToHost,
                           e->stream));
  EDX_CUDA(cudaStreamSynchronize(e->stream));
  return *e->h_expected;
}

// Enqueues the step for the current batch and decision (no sync).
void step_enqueue(edx_engine* e, const int32_t* decision) {
  const edx::NvtxRange nv("edx.step (K7 sim.hpp:87-218)");
  if (!e->cur_ids) edx::invalid("no batch loaded");
  ensure_translated(e);
  if (decision) {
    validate_decision_host(decision, e->rows, e->n, e->m);
    e->decision.ensure(e->rows);
    EDX_CUDA(cudaMemcpyAsync(e->decision.p, decision, e->rows * sizeof(int32_t),
                             cudaMemcpyHostToDevice, e->stream));
  } else {
    if (!e->dispatched) edx::invalid("no dispatch decision to step with");
    if (e->rows != static_cast<uint64_t>(e->n) * e->m) edx::invalid("decision does not cover m*n samples");
  }
  if (e->clock >= 0xFFFFFFFFull) throw Error(EDX_RUNTIME_ERROR, "clock exceeds 2^32 iterations");
  edx::StepResult sr;
  rec(e, 8, e->stream);
  edx::step_run(e, e->decision.p, &sr);
  if (e->hashed)  // the slots in use, read back with the iteration's counters
    EDX_CUDA(cudaMemcpyAsync(e->h_used, e->idt.count.p, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, e->stream));
  rec(e, 9, e->stream);
  e->launches += sr.launches;
  e->pending_step = e->profiling;
}

// Waits for the iteration and assembles its IterationReport.
void step_finish(edx_engine* e, edx_report* rep) {
  engine_sync_check(e);
  if (e->hashed) e->used_bound = e->idt.used = *e->h_used;
  // IterationReport totals and realised cost, worker order (sim.hpp:206-216)
  const int n = e->n;
  const unsigned long long* c = e->h_counters;
  rep->iteration = e->clock;
  rep->miss_pull = rep->update_push = rep->evict_push = 0;
  rep->hits = c[3 * n];
  rep->lookups = e->total_ids;
  rep->cost_s = 0.0;
  for (int j = 0; j < n; ++j) {
    rep->miss_pull_w[j] = c[j];
    rep->update_push_w[j] = c[n + j];
    rep->evict_push_w[j] = c[2 * n + j];
    rep->miss_pull += c[j];
    rep->update_push += c[n + j];
    rep->evict_push += c[2 * n + j];
    const uint64_t ops = c[j] + c[n + j] + c[2 * n + j];
    rep->cost_w[j] = static_cast<double>(ops) * e->ucost_h[j];
    rep->cost_s += rep->cost_w[j];
  }
  ++e->clock;
  ++e->state_version;
  e->dispatched = false;
}

void engine_step(edx_engine* e, const int32_t* decision, edx_report* rep) {
  step_enqueue(e, decision);
  step_finish(e, rep);
}

// One fused iteration (build -> dispatch -> step) for an already-loaded
// batch.  With device-decided victims and profiling off it runs as
// a CUDA graph captured on first use and replayed while (rows, ids, alpha)
// stay the same -- the ~40 launches of an iteration become one.  Any capture
// failure disables graphs for the engine and the iteration runs eagerly.
// build -> dispatch -> step enqueue, with the step's decision-independent
// head on the side stream overlapping the dispatch
void iterate_enqueue(edx_engine* e, double alpha) {
  if (!e->cur_ids) edx::invalid("no batch loaded");
  ensure_translated(e);
  static const bool overlap = [] {  // EDX_HEAD_OVERLAP=0: the head runs inside the step (A/B)
    const char* v = std::getenv("EDX_HEAD_OVERLAP");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  try {
    engine_build(e);
    // forked after the build, so it overlaps the dispatch, for batches up to
    // 2^20 ids (C1 0.271 -> 0.265 ms per iteration); on larger batches it
    // runs inside the step (C5: 1.148 ms overlapped against 1.109 inside;
    // 1.128 against 1.096 even when forked only after the greedy's
    // preference lists, beside the one-CTA sweep)
    if (!e->profiling && overlap && e->total_ids <= (1ULL << 20)) edx::step_head(e);
    engine_dispatch(e, alpha);
    step_enqueue(e, nullptr);
  } catch (...) {
    edx::step_head_abandon(e);
    throw;
  }
}

void engine_iterate_core(edx_engine* e, double alpha) {
  if (e->graph_mode < 0) {
    const char* v = std::getenv("EDX_GRAPH");
    e->graph_mode = (v && std::strcmp(v, "0") == 0) ? 0 : 1;
    // sharded engines can capture their NCCL gather / broadcast into the graph
    // too (EDX_MULTI_GRAPH=1; every rank replays the same collective sequence).
    // Parity-green at 2 and 4 ranks, but within noise of eager (C2 / C5 at
    // N = 2, 4: +0.0..0.8%), so eager stays the default there.
    const char* mv = std::getenv("EDX_MULTI_GRAPH");
    if (e->world > 1 && !(mv && std::strcmp(mv, "1") == 0)) e->graph_mode = 0;
  }
  const bool eligible = e->graph_mode == 1 && !e->profiling &&
                        edx::step_device_only(e) && e->cur_raw == e->ids.p;
  if (!eligible) {
    iterate_enqueue(e, alpha);
    return;
  }
  const double a = alpha < 0.0 ? e->alpha : alpha;
  if (e->hashed) reserve_slots(e, e->total_ids);  // the graph translates in-stream
  const unsigned long long epoch = edx::g_alloc_epoch.load(std::memory_order_relaxed);
  if (!e->gexec || e->g_rows != e->rows || e->g_total != e->total_ids || e->g_alpha != a ||
      e->g_epoch != epoch) {
    if (e->gexec) {
      cudaGraphExecDestroy(e->gexec);
      e->gexec = nullptr;
    }
    // first iteration of a shape runs eagerly: every scratch buffer reaches its
    // final size before the capture (no allocation is recorded)
    if (e->g_rows != e->rows || e->g_total != e->total_ids || e->g_alpha != a) {
      e->g_rows = e->rows;
      e->g_total = e->total_ids;
      e->g_alpha = a;
      iterate_enqueue(e, a);
      return;
    }
    const uint64_t l0 = e->launches;
    cudaGraph_t g = nullptr;
    EDX_CUDA(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeRelaxed));
    e->capturing = true;
    bool ok = true;
    try {
      iterate_enqueue(e, a);
      EDX_CUDA(cudaStreamWaitEvent(e->stream, e->cost_done, 0));  // join decision_cost
    } catch (...) {
      ok = false;
    }
    e->capturing = false;
    const cudaError_t ec = cudaStreamEndCapture(e->stream, &g);
    if (ok && ec == cudaSuccess && g) ok = cudaGraphInstantiate(&e->gexec, g, 0) == cudaSuccess;
    else ok = false;
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    if (!ok) {  // not capturable here: eager from now on
      e->gexec = nullptr;
      e->graph_mode = 0;
      e->launches = l0;
      iterate_enqueue(e, a);
      return;
    }
    e->g_launches = e->launches - l0;
    e->launches = l0;
    e->g_epoch = edx::g_alloc_epoch.load(std::memory_order_relaxed);
  }
  // host-side inputs the graph reads at replay time (pinned; the previous
  // iteration's copy has completed: every iteration ends with a sync)
  *e->h_clock = static_cast<uint32_t>(e->clock);
  EDX_CUDA(cudaGraphLaunch(e->gexec, e->stream));
  EDX_CUDA(cudaEventRecord(e->cost_done, e->stream));
  e->launches += e->g_launches;
  if (e->hashed) {
    e->used_bound += e->total_ids;
    e->translated = true;
  }
  e->built = e->gap_ready = e->dispatched = e->expected_ready = true;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

void edx_set_error(int code, const char* msg) {
  (void)code;
  g_err = msg ? msg : "";
}

const char* edx_last_error(void) { return g_err.c_str(); }

int edx_abi_version(void) { return 1; }

int edx_validate_config(const edx_cluster_config* cfg, uint64_t max_sample_len) {
  return guard([&] { validate_cfg(cfg, max_sample_len); });
}

int edx_unit_costs(const edx_cluster_config* cfg, double* out) {
  return guard([&] {
    if (!cfg || cfg->n < 1 || cfg->n_bandwidths < cfg->n) edx::invalid("worker id out of range");
    const auto u = unit_costs(cfg);
    std::copy(u.begin(), u.end(), out);
  });
}

int edx_engine_create(const edx_cluster_config* cfg, const edx_engine_options* opt,
                      edx_engine** out) {
  return guard([&] {
    *out = nullptr;
    if (!cfg || !opt) edx::invalid("null argument");
    if (cfg->n < 1) edx::invalid("worker count must be >= 1");
    if (cfg->n > 64) edx::invalid("at most 64 workers supported");
    if (cfg->m < 1) edx::invalid("batch size per worker must be >= 1");
    if (cfg->n_bandwidths != cfg->n) edx::invalid("need one bandwidth per worker");
    for (int j = 0; j < cfg->n; ++j)
      if (!(cfg->bandwidths_bps[j] > 0.0)) edx::invalid("bandwidths must be positive");
    if (cfg->cache_capacity == 0) edx::invalid("cache capacity must be positive");
    if (cfg->alpha < 0.0 || cfg->alpha > 1.0) edx::invalid("alpha must lie in [0, 1]");
    if (opt->id_space > (1ULL << 32)) edx::invalid("id_space must be at most 2^32 (0 = any uint32 id)");
    if (opt->max_batch_ids == 0 || opt->max_batch_ids >= (1ULL << 31))
      edx::invalid("max_batch_ids must be in [1, 2^31)");
    if (opt->world_size > 1) {
      if (!opt->nccl_unique_id) edx::invalid("world_size > 1 needs the rank-0 nccl_unique_id");
      if (opt->rank < 0 || opt->rank >= opt->world_size) edx::invalid("rank out of range");
    }
    int count = 0;
    EDX_CUDA(cudaGetDeviceCount(&count));
    if (opt->device < 0 || opt->device >= count) edx::invalid("CUDA device ordinal out of range");
    EDX_CUDA(cudaSetDevice(opt->device));
    auto e = std::make_unique<edx_engine>();
    e->device = opt->device;
    e->n = cfg->n;
    e->m = cfg->m;
    e->alpha = cfg->alpha;
    e->capacity = cfg->cache_capacity;
    e->d_tran = cfg->d_tran_bytes;
    e->bw.assign(cfg->bandwidths_bps, cfg->bandwidths_bps + cfg->n);
    e->ucost_h = unit_costs(cfg);
    e->max_ids = opt->max_batch_ids;
    // id_space 0: any uint32 id through the device id table, starting with
    // room for 16 batches of new ids (the tables grow 4x on demand)
    e->hashed = opt->id_space == 0;
    e->id_space = e->hashed ? std::min<uint64_t>(0xFFFFFFF0ull, std::max<uint64_t>(1ULL << 16, 16 * e->max_ids))
                            : opt->id_space;
    e->rank = opt->rank;
    e->world = opt->world_size < 1 ? 1 : opt->world_size;
    EDX_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    for (auto& ev : e->ev) EDX_CUDA(cudaEventCreate(&ev));
    EDX_CUDA(cudaEventCreateWithFlags(&e->cost_done, cudaEventDisableTiming));
    EDX_CUDA(cudaStreamCreateWithFlags(&e->step_side, cudaStreamNonBlocking));
    EDX_CUDA(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    for (auto& f : e->pf) {
      EDX_CUDA(cudaEventCreateWithFlags(&f.ready, cudaEventDisableTiming));
      EDX_CUDA(cudaEventCreateWithFlags(&f.free, cudaEventDisableTiming));
    }
    EDX_CUDA(cudaEventCreateWithFlags(&e->head_fork, cudaEventDisableTiming));
    EDX_CUDA(cudaEventCreateWithFlags(&e->head_done, cudaEventDisableTiming));
    e->ol.ensure(e->id_space);
    e->res.ensure(e->id_space);
    EDX_CUDA(cudaMemsetAsync(e->ol.p, 0, e->id_space * sizeof(ulonglong2), e->stream));
    EDX_CUDA(cudaMemsetAsync(e->res.p, 0, e->id_space * sizeof(unsigned long long), e->stream));
    e->ucost.ensure(e->n);
    EDX_CUDA(cudaMemcpyAsync(e->ucost.p, e->ucost_h.data(), e->n * sizeof(double),
                             cudaMemcpyHostToDevice, e->stream));
    e->ids.ensure(e->max_ids);
    e->flags.ensure(edx::kFlagCount);
    EDX_CUDA(cudaMemsetAsync(e->flags.p, 0, edx::kFlagCount * sizeof(int), e->stream));
    EDX_CUDA(cudaMallocHost(&e->h_flags, edx::kFlagCount * sizeof(int)));
    EDX_CUDA(cudaMallocHost(&e->h_counters, (3 * 64 + 8) * sizeof(unsigned long long)));
    EDX_CUDA(cudaMallocHost(&e->h_expected, sizeof(double)));
    EDX_CUDA(cudaMallocHost(&e->h_clock, sizeof(uint32_t)));
    e->d_clock.ensure(1);
    if (e->hashed) {
      edx::id_table_init(e->idt, e->id_space, e->stream);
      e->kslots.ensure(e->max_ids);
      EDX_CUDA(cudaMallocHost(&e->h_used, sizeof(unsigned long long)));
      *e->h_used = 0;
    }
    e->disp.init(e->device);
    edx::step_init_state(e.get());
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    if (e->world > 1) e->comm = edx::nccl_comm_create(opt->nccl_unique_id, e->world, e->rank);
    *out = e.release();
  });
}

void edx_engine_destroy(edx_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->stream);
  for (auto& ev : e->ev)
    if (ev) cudaEventDestroy(ev);
  if (e->cost_done) cudaEventDestroy(e->cost_done);
  if (e->head_fork) cudaEventDestroy(e->head_fork);
  if (e->head_done) cudaEventDestroy(e->head_done);
  if (e->step_side) {
    cudaStreamSynchronize(e->step_side);
    cudaStreamDestroy(e->step_side);
  }
  if (e->copy_stream) {
    cudaStreamSynchronize(e->copy_stream);
    cudaStreamDestroy(e->copy_stream);
  }
  for (auto& f : e->pf) {
    if (f.ready) cudaEventDestroy(f.ready);
    if (f.free) cudaEventDestroy(f.free);
    if (f.h_offsets) cudaFreeHost(f.h_offsets);
  }
  if (e->h_flags) cudaFreeHost(e->h_flags);
  if (e->h_counters) cudaFreeHost(e->h_counters);
  if (e->h_clock) cudaFreeHost(e->h_clock);
  if (e->gexec) cudaGraphExecDestroy(e->gexec);
  if (e->h_expected) cudaFreeHost(e->h_expected);
  if (e->h_used) cudaFreeHost(e->h_used);
  cudaStream_t s = e->stream;
  if (e->comm) edx::nccl_comm_destroy(e->comm);
  delete e;
  if (s) cudaStreamDestroy(s);
}

namespace {

// Host batch validation shared by the load and prefetch paths (same messages);
// returns the id count.
uint64_t check_host_offsets(const edx_engine* e, const uint64_t* offsets, uint64_t R) {
  if (R == 0) edx::invalid("batch holds no samples");
  for (uint64_t i = 0; i < R; ++i)
    if (offsets[i + 1] < offsets[i]) edx::invalid("sample offsets must be non-decreasing");
  const uint64_t total = offsets[R] - offsets[0];
  if (total > e->max_ids)
    edx::invalid("batch holds " + std::to_string(total) + " ids; engine max_batch_ids is " +
                 std::to_string(e->max_ids));
  return total;
}

// A host batch prefetched by edx_engine_prefetch: wait for its copy, stage it
// into the engine's own buffers (fixed pointers for the graph) and load it.
bool load_prefetched(edx_engine* e, const uint32_t* ids, const uint64_t* offsets, uint64_t R) {
  // only the most recent prefetch can be consumed (the steady-state pairing of
  // edx_engine_iterate_prefetch); every other load invalidates the slots
  {
    auto& f = e->pf[e->pf_next ^ 1];
    const bool match = f.valid && f.host_ids == ids && f.host_offsets == offsets && f.rows == R;
    for (auto& g : e->pf) g.valid = false;
    if (!match) return false;
    EDX_CUDA(cudaStreamWaitEvent(e->stream, f.ready, 0));
    e->offsets.ensure(R + 1);
    if (f.total)
      EDX_CUDA(cudaMemcpyAsync(e->ids.p, f.ids.p, f.total * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                               e->stream));
    EDX_CUDA(cudaMemcpyAsync(e->offsets.p, f.offsets.p, (R + 1) * sizeof(uint64_t),
                             cudaMemcpyDeviceToDevice, e->stream));
    EDX_CUDA(cudaEventRecord(f.free, e->stream));
    engine_load(e, e->ids.p, e->offsets.p, R, 1, f.total);
    return true;
  }
}

void drop_prefetched(edx_engine* e) {
  for (auto& f : e->pf) f.valid = false;
}

}  // namespace

int edx_engine_load_batch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                          uint64_t num_samples, int on_device) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    drop_prefetched(e);
    engine_load(e, ids, offsets, num_samples, on_device);
  });
}

void engine_prefetch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                     uint64_t num_samples) {
  {
    const uint64_t R = num_samples;
    const uint64_t total = check_host_offsets(e, offsets, R);
    const uint64_t base = offsets[0];
    auto& f = e->pf[e->pf_next];
    e->pf_next ^= 1;
    // the slot's previous copy has finished before its pinned offsets are rewritten
    EDX_CUDA(cudaEventSynchronize(f.ready));
    f.valid = false;
    if (f.h_cap < R + 1) {
      if (f.h_offsets) EDX_CUDA(cudaFreeHost(f.h_offsets));
      f.h_offsets = nullptr;
      f.h_cap = 0;
      EDX_CUDA(cudaMallocHost(&f.h_offsets, (R + 1) * sizeof(uint64_t)));
      f.h_cap = R + 1;
    }
    for (uint64_t i = 0; i <= R; ++i) f.h_offsets[i] = offsets[i] - base;
    f.ids.ensure(e->max_ids);
    f.offsets.ensure(R + 1);
    // the previous batch of this slot has been staged out of it
    EDX_CUDA(cudaStreamWaitEvent(e->copy_stream, f.free, 0));
    if (total)
      EDX_CUDA(cudaMemcpyAsync(f.ids.p, ids + base, total * sizeof(uint32_t), cudaMemcpyHostToDevice,
                               e->copy_stream));
    EDX_CUDA(cudaMemcpyAsync(f.offsets.p, f.h_offsets, (R + 1) * sizeof(uint64_t),
                             cudaMemcpyHostToDevice, e->copy_stream));
    EDX_CUDA(cudaEventRecord(f.ready, e->copy_stream));
    f.host_ids = ids;
    f.host_offsets = offsets;
    f.rows = R;
    f.total = total;
    f.valid = true;
  }
}

int edx_engine_prefetch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                        uint64_t num_samples) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    engine_prefetch(e, ids, offsets, num_samples);
  });
}

int edx_engine_load_device_batch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                                 uint64_t num_samples, uint64_t total_ids) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    drop_prefetched(e);
    engine_load(e, ids, offsets, num_samples, 1, total_ids);
  });
}

int edx_engine_build(edx_engine* e, double* matrix_out) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    engine_build(e);
    if (matrix_out) {
      EDX_CUDA(cudaMemcpyAsync(matrix_out, e->matrix.p, e->rows * e->n * sizeof(double),
                               cudaMemcpyDeviceToHost, e->stream));
      engine_sync_check(e);
    }
  });
}

int edx_engine_dispatch(edx_engine* e, double alpha, int32_t* decision_out,
                        double* expected_cost_out) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    engine_dispatch(e, alpha);
    if (decision_out)
      EDX_CUDA(cudaMemcpyAsync(decision_out, e->decision.p, e->rows * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, e->stream));
    if (decision_out || expected_cost_out) engine_sync_check(e);
    if (expected_cost_out) *expected_cost_out = fetch_expected(e);
  });
}

int edx_engine_dispatch_hitgreedy(edx_engine* e, int32_t* decision_out) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    if (e->rows == 0) edx::invalid("load a batch before dispatching");
    if (e->rows != static_cast<uint64_t>(e->n) * static_cast<uint64_t>(e->m))
      edx::invalid("sample count must be m*n");
    if (e->m >= (1 << 26)) edx::invalid("at most 2^26 samples per worker");
    e->decision.ensure(e->rows + 2);
    ensure_translated(e);
    // every rank holds the same replica, so every rank decides identically
    edx::launch_hitgreedy(e->hit, e->cur_ids, e->cur_offsets, e->rows, e->n, e->m, e->ol.p,
                          e->id_space, e->decision.p, e->flags.p, e->stream);
    e->launches += 3;
    e->dispatched = true;
    e->expected_ready = false;
    if (decision_out) {
      EDX_CUDA(cudaMemcpyAsync(decision_out, e->decision.p, e->rows * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, e->stream));
      engine_sync_check(e);
    }
  });
}

int edx_engine_step(edx_engine* e, const int32_t* decision, edx_report* rep) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    engine_step(e, decision, rep);
  });
}

int edx_engine_iterate(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                       uint64_t num_samples, int on_device, int32_t* decision_out,
                       double* expected_cost_out, edx_report* rep) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    drop_prefetched(e);
    engine_load(e, ids, offsets, num_samples, on_device);
    engine_iterate_core(e, -1.0);
    if (decision_out)
      EDX_CUDA(cudaMemcpyAsync(decision_out, e->decision.p, e->rows * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, e->stream));
    step_finish(e, rep);
    if (expected_cost_out) *expected_cost_out = fetch_expected(e);
  });
}

int edx_engine_iterate_prefetch(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                                uint64_t num_samples, const uint32_t* next_ids,
                                const uint64_t* next_offsets, uint64_t next_num_samples,
                                int32_t* decision_out, double* expected_cost_out, edx_report* rep) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    // the next batch is validated before this iteration is launched: a bad
    // next batch must not leave a launched, unfinished iteration behind
    if (next_ids && next_offsets) check_host_offsets(e, next_offsets, next_num_samples);
    if (!load_prefetched(e, ids, offsets, num_samples)) engine_load(e, ids, offsets, num_samples, 0);
    engine_iterate_core(e, -1.0);
    // the next batch's copy is issued while this iteration runs
    if (next_ids && next_offsets) engine_prefetch(e, next_ids, next_offsets, next_num_samples);
    if (decision_out)
      EDX_CUDA(cudaMemcpyAsync(decision_out, e->decision.p, e->rows * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, e->stream));
    step_finish(e, rep);
    if (expected_cost_out) *expected_cost_out = fetch_expected(e);
  });
}

int edx_engine_iterate_device(edx_engine* e, const uint32_t* ids, const uint64_t* offsets,
                              uint64_t num_samples, uint64_t total_ids, int32_t* decision_out,
                              double* expected_cost_out, edx_report* rep) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    if (total_ids > e->max_ids)
      edx::invalid("batch holds " + std::to_string(total_ids) + " ids; engine max_batch_ids is " +
                   std::to_string(e->max_ids));
    drop_prefetched(e);
    // stage into the engine's own batch buffers: fixed pointers for the graph
    e->offsets.ensure(num_samples + 1);
    if (total_ids)
      EDX_CUDA(cudaMemcpyAsync(e->ids.p, ids, total_ids * sizeof(uint32_t), cudaMemcpyDeviceToDevice,
                               e->stream));
    EDX_CUDA(cudaMemcpyAsync(e->offsets.p, offsets, (num_samples + 1) * sizeof(uint64_t),
                             cudaMemcpyDeviceToDevice, e->stream));
    engine_load(e, e->ids.p, e->offsets.p, num_samples, 1, total_ids);
    engine_iterate_core(e, -1.0);
    if (decision_out)
      EDX_CUDA(cudaMemcpyAsync(decision_out, e->decision.p, e->rows * sizeof(int32_t),
                               cudaMemcpyDeviceToHost, e->stream));
    step_finish(e, rep);
    if (expected_cost_out) *expected_cost_out = fetch_expected(e);
  });
}

int edx_engine_seed_entry(edx_engine* e, uint32_t id, int32_t worker, int latest, int owner) {
  return guard([&] {
    if (owner && !latest) edx::invalid("an owner's copy is always latest");
    if (worker < 0 || worker >= e->n) edx::invalid("worker out of range");
    if (!e->hashed && id >= e->id_space) edx::invalid("embedding id outside the engine's id_space");
    EDX_CUDA(cudaSetDevice(e->device));
    const uint32_t slot = host_slots(e, &id, 1, true)[0];
    auto& c = e->cache;
    int* status = reinterpret_cast<int*>(e->step.wscalars.p);
    k_seed_entry<<<1, 1, 0, e->stream>>>(slot, worker, latest, owner, static_cast<uint32_t>(e->clock),
                                         e->capacity, e->id_space, e->ol.p, e->res.p, c.slot_of.p,
                                         c.sid.p, c.smark.p, c.sfreq.p, c.slast.p, c.size.p,
                                         c.cur_mark.p, c.at_cur.p, status);
    EDX_LAUNCHED();
    int st = 0;
    EDX_CUDA(cudaMemcpyAsync(&st, status, sizeof st, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    if (st == 1) edx::logic("touch would insert into a full cache; evict first");
    ++e->state_version;
  });
}

int edx_engine_state_of(edx_engine* e, uint32_t id, uint64_t* owners, uint64_t* latest,
                        uint64_t* resident) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    const uint32_t slot = e->hashed ? host_slots(e, &id, 1, false)[0] : id;
    if (slot >= e->id_space) {  // unknown embeddings are {0,0,0} (sim.hpp:64-67)
      *owners = *latest = *resident = 0;
      return;
    }
    ulonglong2 st;
    unsigned long long r;
    EDX_CUDA(cudaMemcpyAsync(&st, e->ol.p + slot, sizeof st, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(&r, e->res.p + slot, sizeof r, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    *owners = st.x;
    *latest = st.y;
    *resident = r;
  });
}

int edx_engine_validate_consistency(edx_engine* e) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    DevBuf<int> status;
    status.ensure(8);
    DevBuf<unsigned long long> at;
    at.ensure(e->n);
    EDX_CUDA(cudaMemsetAsync(status.p, 0, 8 * sizeof(int), e->stream));
    EDX_CUDA(cudaMemsetAsync(at.p, 0, e->n * sizeof(unsigned long long), e->stream));
    auto& c = e->cache;
    const uint64_t cells = static_cast<uint64_t>(e->n) * e->capacity;
    k_validate_slots<<<grid_for(cells), kT, 0, e->stream>>>(e->n, e->capacity, e->id_space, c.size.p,
                                                           c.sid.p, e->res.p, c.slot_of.p, c.smark.p,
                                                           c.cur_mark.p, at.p, status.p);
    k_validate_ids<<<grid_for(e->id_space), kT, 0, e->stream>>>(
        e->n, e->id_space, e->ol.p, e->res.p, c.slot_of.p, e->hashed ? e->idt.slot2id.p : nullptr,
        status.p);
    EDX_LAUNCHED();
    int st[8];
    std::vector<unsigned long long> at_h(e->n), at_d(e->n);
    EDX_CUDA(cudaMemcpyAsync(st, status.p, sizeof st, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(at_h.data(), at.p, e->n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(at_d.data(), c.at_cur.p, e->n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    if (st[0]) edx::logic("cache entry missing from global resident set");
    if (st[1]) edx::logic("embedding state invariant violated for id " + std::to_string(static_cast<uint32_t>(st[3])));
    if (st[2]) edx::logic("global resident bit without a cache entry");
    for (int j = 0; j < e->n; ++j)
      if (at_h[j] != at_d[j]) edx::logic("at-current-mark count drifted on worker " + std::to_string(j));
  });
}

uint64_t edx_engine_clock(edx_engine* e) { return e->clock; }

uint64_t edx_engine_state_version(edx_engine* e) { return e->state_version; }

int edx_engine_synchronize(edx_engine* e) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    engine_sync_check(e);
  });
}

int edx_engine_expected_cost(edx_engine* e, double* out) {
  return guard([&] {
    if (!e->expected_ready) edx::invalid("no EcoMix dispatch decision to cost");
    EDX_CUDA(cudaSetDevice(e->device));
    *out = fetch_expected(e);
  });
}

int edx_nccl_unique_id(void* out, uint64_t len) {
  return guard([&] {
    if (len < 128) edx::invalid("nccl unique id buffer must hold 128 bytes");
    edx::nccl_unique_id(out);
  });
}

namespace {
// edx_transport behind the exchange steps (host buffers; a failing callback
// throws, and guard() turns it into the error code)
struct CallbackTransport final : edx::Transport {
  explicit CallbackTransport(const edx_transport* t) : t(t) {
    if (!t || !t->send || !t->recv || !t->broadcast) edx::invalid("incomplete edx_transport");
  }
  void send(const void* buf, uint64_t bytes, int peer) override {
    if (t->send(t->ctx, buf, bytes, peer) != 0) fail("send");
  }
  void recv(void* buf, uint64_t bytes, int peer) override {
    if (t->recv(t->ctx, buf, bytes, peer) != 0) fail("recv");
  }
  void broadcast(void* buf, uint64_t bytes, int root) override {
    if (t->broadcast(t->ctx, buf, bytes, root) != 0) fail("broadcast");
  }
  [[noreturn]] static void fail(const char* what) {
    throw edx::Error(EDX_RUNTIME_ERROR, std::string("transport ") + what + " failed");
  }
  const edx_transport* t;
};

void check_group(int32_t world, int32_t rank, int32_t root) {
  if (world < 1) edx::invalid("world_size must be >= 1");
  if (rank < 0 || rank >= world) edx::invalid("rank out of range");
  if (root < 0 || root >= world) edx::invalid("root out of range");
}
}  // namespace

int edx_shard_rows(uint64_t rows, int32_t world, uint64_t* lo, uint64_t* hi) {
  return guard([&] {
    if (world < 1) edx::invalid("world_size must be >= 1");
    if (!lo || !hi) edx::invalid("null shard bounds");
    edx::shard_rows(rows, world, lo, hi);
  });
}

int edx_exchange_gather_rows(const edx_transport* t, double* matrix, uint64_t rows, int32_t n,
                             int32_t world, int32_t rank, int32_t root) {
  return guard([&] {
    check_group(world, rank, root);
    if (n < 1) edx::invalid("n must be >= 1");
    if (rows && !matrix) edx::invalid("null matrix");
    CallbackTransport tr(t);
    std::vector<uint64_t> lo(world), hi(world);
    edx::shard_rows(rows, world, lo.data(), hi.data());
    edx::gather_rows(tr, matrix, lo.data(), hi.data(), world, rank, root, n);
  });
}

int edx_exchange_broadcast_decision(const edx_transport* t, int32_t* decision, uint64_t rows,
                                    int32_t root) {
  return guard([&] {
    if (root < 0) edx::invalid("root out of range");
    if (rows && !decision) edx::invalid("null decision");
    CallbackTransport tr(t);
    edx::broadcast_decision(tr, decision, rows, root);
  });
}

int edx_engine_stream(edx_engine* e, void** stream) {
  return guard([&] { *stream = static_cast<void*>(e->stream); });
}

int edx_engine_export_global(edx_engine* e, uint32_t* ids, uint64_t* owners, uint64_t* latest,
                             uint64_t* resident, uint64_t cap, uint64_t* count) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    DevBuf<unsigned long long> cnt;
    cnt.ensure(1);
    DevBuf<uint32_t> d_ids;
    DevBuf<unsigned long long> d_m;
    d_ids.ensure(cap);
    d_m.ensure(3 * cap);
    EDX_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), e->stream));
    k_export_global<<<grid_for(e->id_space), kT, 0, e->stream>>>(
        e->ol.p, e->res.p, e->id_space, e->hashed ? e->idt.slot2id.p : nullptr, d_ids.p, d_m.p, cap,
        cnt.p);
    EDX_LAUNCHED();
    unsigned long long total = 0;
    EDX_CUDA(cudaMemcpyAsync(&total, cnt.p, sizeof total, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    *count = total;
    if (cap == 0) return;
    const uint64_t got = std::min<uint64_t>(total, cap);
    std::vector<uint32_t> hid(got);
    std::vector<unsigned long long> hm(3 * got);
    EDX_CUDA(cudaMemcpy(hid.data(), d_ids.p, got * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    EDX_CUDA(cudaMemcpy(hm.data(), d_m.p, 3 * got * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    std::vector<uint64_t> perm(got);
    std::iota(perm.begin(), perm.end(), 0);
    std::sort(perm.begin(), perm.end(), [&](uint64_t a, uint64_t b) { return hid[a] < hid[b]; });
    for (uint64_t t = 0; t < got; ++t) {
      ids[t] = hid[perm[t]];
      owners[t] = hm[3 * perm[t]];
      latest[t] = hm[3 * perm[t] + 1];
      resident[t] = hm[3 * perm[t] + 2];
    }
  });
}

int edx_engine_cache_size(edx_engine* e, int32_t worker, uint64_t* size) {
  return guard([&] {
    if (worker < 0 || worker >= e->n) edx::invalid("worker out of range");
    EDX_CUDA(cudaSetDevice(e->device));
    uint32_t s = 0;
    EDX_CUDA(cudaMemcpyAsync(&s, e->cache.size.p + worker, sizeof s, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    *size = s;
  });
}

int edx_engine_export_cache(edx_engine* e, int32_t worker, uint32_t* ids, uint8_t* version,
                            uint32_t* mark, uint32_t* freq, uint64_t* last_access) {
  return guard([&] {
    if (worker < 0 || worker >= e->n) edx::invalid("worker out of range");
    EDX_CUDA(cudaSetDevice(e->device));
    auto& c = e->cache;
    uint32_t sz = 0;
    EDX_CUDA(cudaMemcpyAsync(&sz, c.size.p + worker, sizeof sz, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    if (sz == 0) return;
    const uint64_t g = static_cast<uint64_t>(worker) * e->capacity;
    std::vector<uint32_t> hid(sz), hm(sz), hf(sz), hl(sz);
    std::vector<uint8_t> hv(sz);
    DevBuf<uint8_t> dv;
    DevBuf<uint32_t> di;
    dv.ensure(sz);
    di.ensure(sz);
    k_export_cache<<<grid_for(sz), kT, 0, e->stream>>>(worker, e->capacity, sz, c.sid.p, e->ol.p,
                                                       e->hashed ? e->idt.slot2id.p : nullptr, dv.p,
                                                       di.p);
    EDX_LAUNCHED();
    EDX_CUDA(cudaMemcpyAsync(hid.data(), di.p, sz * 4, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(hm.data(), c.smark.p + g, sz * 4, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(hf.data(), c.sfreq.p + g, sz * 4, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(hl.data(), c.slast.p + g, sz * 4, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(hv.data(), dv.p, sz, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    std::vector<uint32_t> perm(sz);
    std::iota(perm.begin(), perm.end(), 0u);
    std::sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) { return hid[a] < hid[b]; });
    for (uint32_t t = 0; t < sz; ++t) {
      ids[t] = hid[perm[t]];
      version[t] = hv[perm[t]];
      mark[t] = hm[perm[t]];
      freq[t] = hf[perm[t]];
      last_access[t] = hl[perm[t]];
    }
  });
}

int edx_engine_cache_marks(edx_engine* e, int32_t worker, uint32_t* current_mark,
                           uint64_t* at_current_mark) {
  return guard([&] {
    if (worker < 0 || worker >= e->n) edx::invalid("worker out of range");
    EDX_CUDA(cudaSetDevice(e->device));
    unsigned long long at = 0;
    EDX_CUDA(cudaMemcpyAsync(current_mark, e->cache.cur_mark.p + worker, sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaMemcpyAsync(&at, e->cache.at_cur.p + worker, sizeof at, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    *at_current_mark = at;
  });
}

int edx_engine_import_snapshot(edx_engine* e, const uint32_t* ids, const uint64_t* owners,
                               const uint64_t* latest, const uint64_t* resident, uint64_t count) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    ++e->state_version;
    const std::vector<uint32_t> slots = host_slots(e, ids, count, true);
    ids = slots.data();
    EDX_CUDA(cudaMemsetAsync(e->ol.p, 0, e->id_space * sizeof(ulonglong2), e->stream));
    EDX_CUDA(cudaMemsetAsync(e->res.p, 0, e->id_space * sizeof(unsigned long long), e->stream));
    if (count) {
      DevBuf<uint32_t> d_ids;
      DevBuf<unsigned long long> a, b, c;
      d_ids.ensure(count);
      a.ensure(count);
      b.ensure(count);
      c.ensure(count);
      EDX_CUDA(cudaMemcpyAsync(d_ids.p, ids, count * 4, cudaMemcpyHostToDevice, e->stream));
      EDX_CUDA(cudaMemcpyAsync(a.p, owners, count * 8, cudaMemcpyHostToDevice, e->stream));
      EDX_CUDA(cudaMemcpyAsync(b.p, latest, count * 8, cudaMemcpyHostToDevice, e->stream));
      if (resident) EDX_CUDA(cudaMemcpyAsync(c.p, resident, count * 8, cudaMemcpyHostToDevice, e->stream));
      k_import<<<grid_for(count), kT, 0, e->stream>>>(d_ids.p, a.p, b.p, resident ? c.p : nullptr,
                                                     count, e->id_space, e->ol.p, e->res.p, e->flags.p);
      EDX_LAUNCHED();
      engine_sync_check(e);
    }
  });
}

int edx_engine_import_state(edx_engine* e, uint64_t clock, uint64_t g_count, const uint32_t* g_ids,
                            const uint64_t* g_owners, const uint64_t* g_latest,
                            const uint64_t* g_resident, const uint64_t* entry_off,
                            const uint32_t* e_ids, const uint8_t* e_version, const uint32_t* e_mark,
                            const uint32_t* e_freq, const uint64_t* e_last,
                            const uint32_t* current_mark, const uint64_t* at_current_mark) {
  const int rc = guard([&] {
    if (!e) edx::invalid("null engine");
    if (clock >= 0xFFFFFFFFull) edx::invalid("clock exceeds 2^32 iterations");
    const int n = e->n;
    if (entry_off[0] != 0) edx::invalid("entry offsets must start at 0");
    for (int j = 0; j < n; ++j) {
      if (entry_off[j + 1] < entry_off[j]) edx::invalid("entry offsets must be non-decreasing");
      if (entry_off[j + 1] - entry_off[j] > e->capacity)
        edx::invalid("imported cache exceeds its capacity");
    }
    EDX_CUDA(cudaSetDevice(e->device));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    edx::step_head_abandon(e);
    // ids -> slots (hashed mode) before any table is cleared: growth copies them
    const std::vector<uint32_t> gslots = host_slots(e, g_ids, g_count, true);
    const std::vector<uint32_t> eslots = host_slots(e, e_ids, entry_off[n], true);
    g_ids = gslots.data();
    e_ids = eslots.data();
    auto& c = e->cache;
    // the global table (SimState::global_): zero, then the imported rows
    EDX_CUDA(cudaMemsetAsync(e->ol.p, 0, e->id_space * sizeof(ulonglong2), e->stream));
    EDX_CUDA(cudaMemsetAsync(e->res.p, 0, e->id_space * sizeof(unsigned long long), e->stream));
    const uint64_t cells = static_cast<uint64_t>(n) * e->id_space;
    k_fill_slots<<<grid_for(cells), kT, 0, e->stream>>>(c.slot_of.p, cells);
    EDX_LAUNCHED();
    if (c.pin.p)  // pin stamps are iteration clocks: the imported clock may be lower
      EDX_CUDA(cudaMemsetAsync(c.pin.p, 0, c.pin.n * sizeof(uint32_t), e->stream));
    DevBuf<int> status;
    status.ensure(8);
    EDX_CUDA(cudaMemsetAsync(status.p, 0, 8 * sizeof(int), e->stream));
    if (g_count) {
      DevBuf<uint32_t> d_ids;
      DevBuf<unsigned long long> a, b, r;
      d_ids.ensure(g_count);
      a.ensure(g_count);
      b.ensure(g_count);
      r.ensure(g_count);
      EDX_CUDA(cudaMemcpyAsync(d_ids.p, g_ids, g_count * 4, cudaMemcpyHostToDevice, e->stream));
      EDX_CUDA(cudaMemcpyAsync(a.p, g_owners, g_count * 8, cudaMemcpyHostToDevice, e->stream));
      EDX_CUDA(cudaMemcpyAsync(b.p, g_latest, g_count * 8, cudaMemcpyHostToDevice, e->stream));
      EDX_CUDA(cudaMemcpyAsync(r.p, g_resident, g_count * 8, cudaMemcpyHostToDevice, e->stream));
      k_import<<<grid_for(g_count), kT, 0, e->stream>>>(d_ids.p, a.p, b.p, r.p, g_count,
                                                       e->id_space, e->ol.p, e->res.p, status.p);
      EDX_LAUNCHED();
      EDX_CUDA(cudaStreamSynchronize(e->stream));
    }
    // every worker's cache (WorkerCache::entries_, current_mark_, at_current_mark_)
    const uint64_t total = entry_off[n];
    std::vector<uint32_t> sizes(n);
    for (int j = 0; j < n; ++j) sizes[j] = static_cast<uint32_t>(entry_off[j + 1] - entry_off[j]);
    if (total) {
      DevBuf<uint32_t> di, dm, df;
      DevBuf<uint64_t> dl;
      DevBuf<uint8_t> dv;
      di.ensure(total);
      dm.ensure(total);
      df.ensure(total);
      dl.ensure(total);
      EDX_CUDA(cudaMemcpyAsync(di.p, e_ids, total * 4, cudaMemcpyHostToDevice, e->stream));
      EDX_CUDA(cudaMemcpyAsync(dm.p, e_mark, total * 4, cudaMemcpyHostToDevice, e->stream));
      EDX_CUDA(cudaMemcpyAsync(df.p, e_freq, total * 4, cudaMemcpyHostToDevice, e->stream));
      EDX_CUDA(cudaMemcpyAsync(dl.p, e_last, total * 8, cudaMemcpyHostToDevice, e->stream));
      if (e_version) {
        dv.ensure(total);
        EDX_CUDA(cudaMemcpyAsync(dv.p, e_version, total, cudaMemcpyHostToDevice, e->stream));
      }
      for (int j = 0; j < n; ++j) {
        const uint64_t a = entry_off[j], cnt = sizes[j];
        if (!cnt) continue;
        k_import_entries<<<grid_for(cnt), kT, 0, e->stream>>>(
            j, cnt, e->capacity, e->id_space, di.p + a, e_version ? dv.p + a : nullptr, dm.p + a,
            df.p + a, dl.p + a, e->ol.p, c.slot_of.p, c.sid.p, c.smark.p, c.sfreq.p, c.slast.p,
            status.p + 4);
        EDX_LAUNCHED();
      }
      EDX_CUDA(cudaStreamSynchronize(e->stream));
    }
    std::vector<unsigned long long> at(n);
    for (int j = 0; j < n; ++j) at[j] = at_current_mark[j];
    EDX_CUDA(cudaMemcpyAsync(c.size.p, sizes.data(), n * 4, cudaMemcpyHostToDevice, e->stream));
    EDX_CUDA(cudaMemcpyAsync(c.cur_mark.p, current_mark, n * 4, cudaMemcpyHostToDevice, e->stream));
    EDX_CUDA(cudaMemcpyAsync(c.at_cur.p, at.data(), n * 8, cudaMemcpyHostToDevice, e->stream));
    int st[8];
    EDX_CUDA(cudaMemcpyAsync(st, status.p, sizeof st, cudaMemcpyDeviceToHost, e->stream));
    EDX_CUDA(cudaStreamSynchronize(e->stream));
    if (st[edx::kFlagIdOutOfRange] || st[4])
      edx::invalid("embedding id outside the engine's id_space");
    if (st[5]) edx::invalid("last_access exceeds 2^32");
    if (st[6]) edx::logic("version flag diverged from global state");
    if (st[7]) edx::invalid("duplicate id in an imported cache");
    e->clock = clock;
    e->built = e->dispatched = e->expected_ready = false;
    ++e->state_version;
  });
  // the imported state must satisfy SimState::validate_consistency
  // (sim.hpp:222-248), at_current_mark included
  return rc != EDX_OK ? rc : edx_engine_validate_consistency(e);
}

int edx_engine_last_kernels(edx_engine* e, const char** build, const char** solver,
                            const char** greedy) {
  return guard([&] {
    if (build) *build = e->kname[edx::kKBuild];
    if (solver) *solver = e->kname[edx::kKSolver];
    if (greedy) *greedy = e->kname[edx::kKGreedy];
  });
}

int edx_engine_set_profiling(edx_engine* e, int on) {
  return guard([&] { e->profiling = on != 0; });
}

int edx_engine_phase_times(edx_engine* e, double* ms, uint64_t* counts, int reset) {
  return guard([&] {
    EDX_CUDA(cudaSetDevice(e->device));
    engine_sync_check(e);
    if (ms) std::copy(e->phase_ms, e->phase_ms + EDX_NUM_PHASES, ms);
    if (counts) {
      counts[0] = e->launches;
      counts[1] = edx::last_hungarian_steps(e->disp.hung, e->stream);
    }
    if (reset) {
      std::fill(e->phase_ms, e->phase_ms + EDX_NUM_PHASES, 0.0);
      e->launches = 0;
    }
  });
}

int edx_solver_stats(edx_engine* e, uint64_t* out) {
  return guard([&] {
    unsigned long long st[8];
    if (e) {
      EDX_CUDA(cudaSetDevice(e->device));
      edx::last_hungarian_stats(e->disp.hung, e->stream, st);
    } else {
      auto& c = dctx();
      std::lock_guard<std::mutex> lk(c.mu);
      c.init();
      edx::last_hungarian_stats(c.disp.hung, c.stream, st);
    }
    for (int i = 0; i < 8; ++i) out[i] = st[i];
  });
}

// ------------------------------------------------------ stateless matrix API

namespace {
void stateless_build(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                     const uint64_t* snap_owners, const uint64_t* snap_latest,
                     uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                     uint64_t R, double* out, const uint64_t* sizes = nullptr);
}  // namespace

int edx_build_matrix(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                     const uint64_t* snap_owners, const uint64_t* snap_latest,
                     const uint64_t* snap_resident, uint64_t snap_count, const uint32_t* ids,
                     const uint64_t* offsets, uint64_t R, double* out) {
  return guard([&] {
    if (!cfg || cfg->n < 1 || cfg->n > 64) edx::invalid(cfg && cfg->n > 64 ? "at most 64 workers supported" : "worker count must be >= 1");
    const uint64_t want = static_cast<uint64_t>(cfg->n) * static_cast<uint64_t>(cfg->m);
    if (R != want) edx::invalid("expected " + std::to_string(want) + " samples, got " + std::to_string(R));
    (void)snap_resident;  // residency never enters the cost (cost.hpp:81-100)
    stateless_build(cfg, snap_ids, snap_owners, snap_latest, snap_count, ids, offsets, R, out);
  });
}

int edx_hitgreedy(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                  const uint64_t* snap_owners, const uint64_t* snap_latest, uint64_t snap_count,
                  const uint32_t* ids, const uint64_t* offsets, uint64_t R, int32_t* decision) {
  return guard([&] {
    if (!cfg || cfg->n < 1 || cfg->n > 64) edx::invalid(cfg && cfg->n > 64 ? "at most 64 workers supported" : "worker count must be >= 1");
    if (R != static_cast<uint64_t>(cfg->n) * static_cast<uint64_t>(cfg->m))
      edx::invalid("sample count must be m*n");
    if (cfg->m >= (1 << 26)) edx::invalid("at most 2^26 samples per worker");
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    const uint64_t base = offsets[0], total = offsets[R] - base;
    uint64_t max_id = 0;
    for (uint64_t s = 0; s < snap_count; ++s) max_id = std::max<uint64_t>(max_id, snap_ids[s]);
    for (uint64_t t = 0; t < total; ++t) max_id = std::max<uint64_t>(max_id, ids[base + t]);
    const uint64_t space = max_id + 1;
    if (space > (1ULL << 28)) edx::invalid("ids too large for the stateless dense snapshot table (< 2^28)");
    std::vector<uint64_t> offs(offsets, offsets + R + 1);
    for (auto& o : offs) o -= base;
    c.ol.ensure(space);
    c.ids.ensure(total);
    c.offsets.ensure(R + 1);
    c.i32a.ensure(R);
    c.reset_flags();
    EDX_CUDA(cudaMemsetAsync(c.ol.p, 0, space * sizeof(ulonglong2), c.stream));
    if (total) EDX_CUDA(cudaMemcpyAsync(c.ids.p, ids + base, total * 4, cudaMemcpyHostToDevice, c.stream));
    EDX_CUDA(cudaMemcpyAsync(c.offsets.p, offs.data(), (R + 1) * 8, cudaMemcpyHostToDevice, c.stream));
    if (snap_count) {
      c.u32a.ensure(snap_count);
      c.snapA.ensure(snap_count);
      c.snapB.ensure(snap_count);
      EDX_CUDA(cudaMemcpyAsync(c.u32a.p, snap_ids, snap_count * 4, cudaMemcpyHostToDevice, c.stream));
      EDX_CUDA(cudaMemcpyAsync(c.snapA.p, snap_owners, snap_count * 8, cudaMemcpyHostToDevice, c.stream));
      EDX_CUDA(cudaMemcpyAsync(c.snapB.p, snap_latest, snap_count * 8, cudaMemcpyHostToDevice, c.stream));
      k_import<<<grid_for(snap_count), kT, 0, c.stream>>>(c.u32a.p, c.snapA.p, c.snapB.p, nullptr,
                                                         snap_count, space, c.ol.p, nullptr, c.flags.p);
      EDX_LAUNCHED();
    }
    edx::launch_hitgreedy(c.hit, c.ids.p, c.offsets.p, R, cfg->n, cfg->m, c.ol.p, space, c.i32a.p,
                          c.flags.p, c.stream);
    EDX_CUDA(cudaMemcpyAsync(decision, c.i32a.p, R * 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync_and_check();
  });
}

int edx_expected_costs(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                       const uint64_t* snap_owners, const uint64_t* snap_latest,
                       uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                       uint64_t num_samples, double* out) {
  return guard([&] {
    if (!cfg || cfg->n < 1 || cfg->n > 64) edx::invalid(cfg && cfg->n > 64 ? "at most 64 workers supported" : "worker count must be >= 1");
    if (cfg->n_bandwidths < cfg->n) edx::invalid("need one bandwidth per worker");
    if (num_samples == 0) return;
    stateless_build(cfg, snap_ids, snap_owners, snap_latest, snap_count, ids, offsets,
                    num_samples, out);
  });
}

int edx_build_matrix_sized(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                           const uint64_t* snap_owners, const uint64_t* snap_latest,
                           uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                           uint64_t R, const uint64_t* sizes, double* out) {
  return guard([&] {
    if (!cfg || cfg->n < 1 || cfg->n > 64) edx::invalid(cfg && cfg->n > 64 ? "at most 64 workers supported" : "worker count must be >= 1");
    const uint64_t want = static_cast<uint64_t>(cfg->n) * static_cast<uint64_t>(cfg->m);
    if (R != want) edx::invalid("expected " + std::to_string(want) + " samples, got " + std::to_string(R));
    if (cfg->n_bandwidths < cfg->n) edx::invalid("need one bandwidth per worker");
    stateless_build(cfg, snap_ids, snap_owners, snap_latest, snap_count, ids, offsets, R, out, sizes);
  });
}

int edx_expected_costs_sized(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                             const uint64_t* snap_owners, const uint64_t* snap_latest,
                             uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                             uint64_t num_samples, const uint64_t* sizes, double* out) {
  return guard([&] {
    if (!cfg || cfg->n < 1 || cfg->n > 64) edx::invalid(cfg && cfg->n > 64 ? "at most 64 workers supported" : "worker count must be >= 1");
    if (cfg->n_bandwidths < cfg->n) edx::invalid("need one bandwidth per worker");
    if (num_samples == 0) return;
    stateless_build(cfg, snap_ids, snap_owners, snap_latest, snap_count, ids, offsets,
                    num_samples, out, sizes);
  });
}

namespace {
void stateless_build(const edx_cluster_config* cfg, const uint32_t* snap_ids,
                     const uint64_t* snap_owners, const uint64_t* snap_latest,
                     uint64_t snap_count, const uint32_t* ids, const uint64_t* offsets,
                     uint64_t R, double* out, const uint64_t* sizes) {
  {
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    const uint64_t base = offsets[0], total = offsets[R] - base;
    uint64_t max_id = 0;
    for (uint64_t s = 0; s < snap_count; ++s) max_id = std::max<uint64_t>(max_id, snap_ids[s]);
    for (uint64_t t = 0; t < total; ++t) max_id = std::max<uint64_t>(max_id, ids[base + t]);
    const uint64_t space = max_id + 1;
    if (space > (1ULL << 28)) edx::invalid("ids too large for the stateless dense snapshot table (< 2^28)");
    const auto u = unit_costs(cfg);
    std::vector<uint64_t> offs(offsets, offsets + R + 1);
    for (auto& o : offs) o -= base;
    c.ol.ensure(space);
    c.ids.ensure(total);
    c.offsets.ensure(R + 1);
    c.ucost.ensure(cfg->n);
    c.values.ensure(R * cfg->n);
    c.reset_flags();
    EDX_CUDA(cudaMemsetAsync(c.ol.p, 0, space * sizeof(ulonglong2), c.stream));
    if (total) EDX_CUDA(cudaMemcpyAsync(c.ids.p, ids + base, total * 4, cudaMemcpyHostToDevice, c.stream));
    EDX_CUDA(cudaMemcpyAsync(c.offsets.p, offs.data(), (R + 1) * 8, cudaMemcpyHostToDevice, c.stream));
    EDX_CUDA(cudaMemcpyAsync(c.ucost.p, u.data(), cfg->n * 8, cudaMemcpyHostToDevice, c.stream));
    if (snap_count) {
      c.u32a.ensure(snap_count);
      c.snapA.ensure(snap_count);
      c.snapB.ensure(snap_count);
      EDX_CUDA(cudaMemcpyAsync(c.u32a.p, snap_ids, snap_count * 4, cudaMemcpyHostToDevice, c.stream));
      EDX_CUDA(cudaMemcpyAsync(c.snapA.p, snap_owners, snap_count * 8, cudaMemcpyHostToDevice, c.stream));
      EDX_CUDA(cudaMemcpyAsync(c.snapB.p, snap_latest, snap_count * 8, cudaMemcpyHostToDevice, c.stream));
      k_import<<<grid_for(snap_count), kT, 0, c.stream>>>(c.u32a.p, c.snapA.p, c.snapB.p, nullptr,
                                                         snap_count, space, c.ol.p, nullptr, c.flags.p);
      EDX_LAUNCHED();
    }
    const uint64_t* d_sizes = nullptr;
    if (sizes) {  // SizeLookupFn values, one per id position
      c.sizes.ensure(total);
      c.bw.ensure(cfg->n);
      if (total)
        EDX_CUDA(cudaMemcpyAsync(c.sizes.p, sizes + base, total * 8, cudaMemcpyHostToDevice, c.stream));
      EDX_CUDA(cudaMemcpyAsync(c.bw.p, cfg->bandwidths_bps, cfg->n * 8, cudaMemcpyHostToDevice, c.stream));
      d_sizes = c.sizes.p;
    }
    edx::launch_cost_build(c.ids.p, c.offsets.p, R, cfg->n, c.ol.p, space, c.ucost.p, c.values.p,
                           nullptr, nullptr, c.flags.p, c.stream, d_sizes, c.bw.p);
    EDX_CUDA(cudaMemcpyAsync(out, c.values.p, R * cfg->n * 8, cudaMemcpyDeviceToHost, c.stream));
    c.sync_and_check();
  }
}
}  // namespace

int edx_row_gap_key(uint64_t rows, uint64_t cols, const double* values, uint64_t row, double* out) {
  return guard([&] {
    if (cols == 0) edx::invalid("row is empty");
    if (row >= rows) edx::invalid("row index out of range");
    if (cols > 64) edx::invalid("at most 64 workers supported");
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    c.values.ensure(cols);
    c.u64a.ensure(1);
    c.u32a.ensure(1);
    EDX_CUDA(cudaMemcpyAsync(c.values.p, values + row * cols, cols * 8, cudaMemcpyHostToDevice, c.stream));
    edx::launch_gap_keys(c.values.p, 1, static_cast<int>(cols), c.u64a.p, c.u32a.p, c.stream);
    uint64_t key = 0;
    EDX_CUDA(cudaMemcpyAsync(&key, c.u64a.p, 8, cudaMemcpyDeviceToHost, c.stream));
    EDX_CUDA(cudaStreamSynchronize(c.stream));
    const uint64_t bits = ~key;
    std::memcpy(out, &bits, sizeof(double));
  });
}

int edx_rows_by_gap(uint64_t rows, uint64_t cols, const double* values, uint64_t* order) {
  return guard([&] {
    if (rows == 0) return;
    if (cols == 0) edx::invalid("row is empty");
    if (cols > 64) edx::invalid("at most 64 workers supported");
    if (rows >= (1ULL << 31)) edx::invalid("too many rows");
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    c.values.ensure(rows * cols);
    c.u64a.ensure(rows);
    c.u64b.ensure(rows);
    c.u32a.ensure(rows);
    c.u32b.ensure(rows);
    EDX_CUDA(cudaMemcpyAsync(c.values.p, values, rows * cols * 8, cudaMemcpyHostToDevice, c.stream));
    edx::launch_gap_keys(c.values.p, rows, static_cast<int>(cols), c.u64a.p, c.u32a.p, c.stream);
    edx::sort_rows_by_gap(c.disp.sort, c.u64a.p, c.u32a.p, c.u32b.p, rows, c.stream);
    k_u32_to_u64<<<grid_for(rows), kT, 0, c.stream>>>(c.u32b.p, rows, c.u64b.p);
    EDX_LAUNCHED();
    EDX_CUDA(cudaMemcpyAsync(order, c.u64b.p, rows * 8, cudaMemcpyDeviceToHost, c.stream));
    EDX_CUDA(cudaStreamSynchronize(c.stream));
  });
}

namespace {
void check_costs_host(const double* v, uint64_t count) {
  for (uint64_t i = 0; i < count; ++i)
    if (!std::isfinite(v[i]) || v[i] < 0.0) edx::invalid("costs must be finite and non-negative");
}
}  // namespace

int edx_hungarian(uint64_t k, const double* values, uint64_t* col_of_row, double* total) {
  return guard([&] {
    if (k < 1) edx::invalid("solver needs at least one row");
    if (k > 16384) edx::invalid("solver order above 16384 is not supported");
    check_costs_host(values, k * k);  // assign.hpp:86-90 rejects before solving
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    c.values.ensure(k * k);
    c.u64a.ensure(k);
    c.reset_flags();
    EDX_CUDA(cudaMemcpyAsync(c.values.p, values, k * k * 8, cudaMemcpyHostToDevice, c.stream));
    edx::launch_hungarian_dense(c.disp.hung, c.values.p, k, c.u64a.p, c.flags.p, c.stream, c.device);
    k_seq_gather_sum<<<1, 1, 0, c.stream>>>(c.values.p, k, c.u64a.p, c.scalar.p);
    EDX_LAUNCHED();
    double t = 0.0;
    EDX_CUDA(cudaMemcpyAsync(col_of_row, c.u64a.p, k * 8, cudaMemcpyDeviceToHost, c.stream));
    EDX_CUDA(cudaMemcpyAsync(&t, c.scalar.p, 8, cudaMemcpyDeviceToHost, c.stream));
    c.sync_and_check();
    if (total) *total = t;
  });
}

int edx_hungarian_blocks(uint64_t rows, uint64_t cols, const double* values,
                         const uint64_t* block_rows, int32_t mult, uint64_t* col_of_row,
                         double* total) {
  return guard([&] {
    if (mult < 1) edx::invalid("solver needs at least one row");
    if (cols < 1 || cols > 64) edx::invalid("at most 64 workers supported");
    const uint64_t k = cols * static_cast<uint64_t>(mult);
    for (uint64_t r = 0; r < k; ++r) {
      if (block_rows[r] >= rows) edx::invalid("row index out of range");
      check_costs_host(values + block_rows[r] * cols, cols);
    }
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    c.values.ensure(rows * cols);
    c.u64a.ensure(k);
    c.u64b.ensure(k);
    c.u32a.ensure(k);
    c.reset_flags();
    EDX_CUDA(cudaMemcpyAsync(c.values.p, values, rows * cols * 8, cudaMemcpyHostToDevice, c.stream));
    EDX_CUDA(cudaMemcpyAsync(c.u64b.p, block_rows, k * 8, cudaMemcpyHostToDevice, c.stream));
    k_u64_to_u32<<<grid_for(k), kT, 0, c.stream>>>(c.u64b.p, k, c.u32a.p);
    EDX_LAUNCHED();
    edx::launch_hungarian_blocks(c.disp.hung, c.values.p, static_cast<int>(cols), c.u32a.p, mult,
                                 nullptr, nullptr, c.u64a.p, c.flags.p, c.stream, c.device);
    k_seq_gather_sum_blocks<<<1, 1, 0, c.stream>>>(c.values.p, static_cast<int>(cols), c.u64b.p, k,
                                                   mult, c.u64a.p, c.scalar.p);
    EDX_LAUNCHED();
    double t = 0.0;
    EDX_CUDA(cudaMemcpyAsync(col_of_row, c.u64a.p, k * 8, cudaMemcpyDeviceToHost, c.stream));
    EDX_CUDA(cudaMemcpyAsync(&t, c.scalar.p, 8, cudaMemcpyDeviceToHost, c.stream));
    c.sync_and_check();
    if (total) *total = t;
  });
}

int edx_greedy_dispatch(uint64_t rows, uint64_t cols, const double* values, const uint64_t* order,
                        uint64_t n_order, const int32_t* capacity, uint64_t* out_rows,
                        int32_t* out_workers) {
  return guard([&] {
    if (cols < 1 || cols > 64) edx::invalid("need one capacity per worker");
    long total = 0;
    for (uint64_t j = 0; j < cols; ++j) total += capacity[j];
    if (total != static_cast<long>(n_order)) edx::invalid("capacities must sum to the number of rows");
    for (uint64_t t = 0; t < n_order; ++t)
      if (order[t] >= rows) edx::invalid("row index out of range");
    if (n_order == 0) return;
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    c.values.ensure(rows * cols);
    c.u64a.ensure(n_order);
    c.u32a.ensure(n_order);
    c.i32a.ensure(cols);
    c.i32b.ensure(n_order);
    c.reset_flags();
    EDX_CUDA(cudaMemcpyAsync(c.values.p, values, rows * cols * 8, cudaMemcpyHostToDevice, c.stream));
    EDX_CUDA(cudaMemcpyAsync(c.u64a.p, order, n_order * 8, cudaMemcpyHostToDevice, c.stream));
    EDX_CUDA(cudaMemcpyAsync(c.i32a.p, capacity, cols * 4, cudaMemcpyHostToDevice, c.stream));
    k_u64_to_u32<<<grid_for(n_order), kT, 0, c.stream>>>(c.u64a.p, n_order, c.u32a.p);
    EDX_LAUNCHED();
    edx::launch_greedy(c.values.p, rows, static_cast<int>(cols), c.u32a.p, n_order, c.i32a.p, 0,
                       nullptr, nullptr, c.i32b.p, c.flags.p, c.disp.greedy, c.stream);
    EDX_CUDA(cudaMemcpyAsync(out_workers, c.i32b.p, n_order * 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync_and_check();
    std::copy(order, order + n_order, out_rows);
  });
}

int edx_ecomix(const edx_cluster_config* cfg, uint64_t rows, uint64_t cols, const double* values,
               const uint64_t* row_ids, int32_t* decision) {
  return guard([&] {
    if (!cfg) edx::invalid("null cluster config");
    if (rows != static_cast<uint64_t>(cfg->n) * static_cast<uint64_t>(cfg->m) ||
        cols != static_cast<uint64_t>(cfg->n))
      edx::invalid("matrix shape does not match cluster config");
    if (cfg->n > 64) edx::invalid("at most 64 workers supported");
    const int mult = edx::exact_multiplicity(cfg->m, cfg->alpha);
    if (mult > 0) check_costs_host(values, rows * cols);
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    c.values.ensure(rows * cols);
    c.i32a.ensure(rows);
    c.reset_flags();
    EDX_CUDA(cudaMemcpyAsync(c.values.p, values, rows * cols * 8, cudaMemcpyHostToDevice, c.stream));
    EDX_CUDA(cudaMemsetAsync(c.i32a.p, 0xff, rows * 4, c.stream));
    edx::run_ecomix(c.disp, c.values.p, rows, cfg->n, cfg->m, cfg->alpha, false, c.i32a.p, c.flags.p,
                    c.stream, c.device, nullptr, nullptr);
    std::vector<int32_t> by_row(rows);
    EDX_CUDA(cudaMemcpyAsync(by_row.data(), c.i32a.p, rows * 4, cudaMemcpyDeviceToHost, c.stream));
    c.sync_and_check();
    // decision.worker_of_sample[sample_of_row(row)] (assign.hpp:260-262)
    std::fill(decision, decision + rows, -1);
    for (uint64_t r = 0; r < rows; ++r) {
      const uint64_t sidx = row_ids ? row_ids[r] : r;
      if (sidx >= rows) edx::invalid("worker id out of range");
      decision[sidx] = by_row[r];
    }
    validate_decision_host(decision, rows, cfg->n, cfg->m);
  });
}

int edx_decision_cost(uint64_t rows, uint64_t cols, const double* values, const int32_t* decision,
                      double* out) {
  return guard([&] {
    for (uint64_t i = 0; i < rows; ++i)
      if (decision[i] < 0 || static_cast<uint64_t>(decision[i]) >= cols) edx::invalid("worker id out of range");
    if (rows == 0) {
      *out = 0.0;
      return;
    }
    auto& c = dctx();
    std::lock_guard<std::mutex> lk(c.mu);
    c.init();
    c.values.ensure(rows * cols);
    c.i32a.ensure(rows);
    EDX_CUDA(cudaMemcpyAsync(c.values.p, values, rows * cols * 8, cudaMemcpyHostToDevice, c.stream));
    EDX_CUDA(cudaMemcpyAsync(c.i32a.p, decision, rows * 4, cudaMemcpyHostToDevice, c.stream));
    edx::launch_decision_cost(c.values.p, c.i32a.p, rows, static_cast<int>(cols), c.scalar.p, c.stream);
    EDX_CUDA(cudaMemcpyAsync(out, c.scalar.p, 8, cudaMemcpyDeviceToHost, c.stream));
    EDX_CUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"
