// Standalone WorkerCache (cache.hpp:73-240) on the device.
//
// SimState's caches are updated a whole batch at a time by K7 (step.cu).
// This is the reference's per-entry API for callers that drive one cache
// directly (tests/test_cache.cpp): touch / set_version / erase / find /
// select_victim / evict_for, under either victim policy:
//   kMarkVersion   least (version, mark, frequency, last_access, id)
//                  (VictimKey, cache.hpp:47-58; the std::set order_);
//   kPriorityRatio least ((version ? 2 : 1) * mark * frequency / footprint,
//                  last_access, id) (pick_victim, cache.hpp:203-230).
// Footprints are a host callback in the reference, consulted for every entry
// at selection time; they are evaluated once when an id is inserted and
// stored with the entry (the callback is a pure function of the id).
//
// Layout: entries are dense slots [0, size) (SoA: id, version, mark,
// frequency, last access, footprint) found through an open-addressing table
// of slot indices (linear probing, tombstones, rebuilt when they crowd it).
// Every mutation is one single-thread kernel; victim selection is one CTA
// reducing over the slots, erasing its pick and repeating while evict_for
// still needs room.  Each API call synchronises and reports the reference's
// exception through the error field.
#include <climits>
#include <memory>
#include <vector>

#include "edx_internal.cuh"

namespace edx {
namespace {

constexpr int kEmpty = -1, kTomb = -2;
constexpr int kSelT = 1024;

enum UcErr : int {
  kUcOk = 0,
  kUcTouchFull = 1,      // logic_error: touch would insert into a full cache
  kUcSetVersion = 2,     // invalid_argument: set_version on non-resident embedding
  kUcNoVictim = 3,       // logic_error: no evictable entry
  kUcAllPinned = 4,      // logic_error: every cache entry is pinned; cannot evict
};

struct UcHdr {
  unsigned long long size, at_cur, tombs, nvict;
  unsigned cur_mark;
  int err;
  // find() result
  int found;
  unsigned f_ver, f_mark, f_freq;
  unsigned long long f_last;
};

struct UcArrays {
  UcHdr* hdr;
  int32_t* table;
  uint64_t H;
  uint64_t cap;
  uint32_t* sid;
  uint8_t* sver;
  uint32_t* smark;
  uint32_t* sfreq;
  unsigned long long* slast;
  double* sfp;
  uint8_t* pin;
};

__device__ __forceinline__ uint64_t uc_hash(uint32_t id) {
  uint64_t x = id * 0x9E3779B97F4A7C15ULL;
  return x ^ (x >> 29);
}

// position of id's table entry, or -1
__device__ int64_t uc_lookup(const UcArrays& a, uint32_t id) {
  for (uint64_t h = uc_hash(id) & (a.H - 1), k = 0; k < a.H; h = (h + 1) & (a.H - 1), ++k) {
    const int32_t t = a.table[h];
    if (t == kEmpty) return -1;
    if (t >= 0 && a.sid[t] == id) return static_cast<int64_t>(h);
  }
  return -1;
}

__device__ void uc_insert_table(const UcArrays& a, uint32_t id, int32_t slot) {
  for (uint64_t h = uc_hash(id) & (a.H - 1);; h = (h + 1) & (a.H - 1)) {
    const int32_t t = a.table[h];
    if (t < 0) {
      if (t == kTomb) --a.hdr->tombs;
      a.table[h] = slot;
      return;
    }
  }
}

__device__ void uc_rebuild_if_crowded(const UcArrays& a) {
  if ((a.hdr->size + a.hdr->tombs) * 4 <= a.H * 3) return;
  for (uint64_t h = 0; h < a.H; ++h) a.table[h] = kEmpty;
  a.hdr->tombs = 0;
  for (uint64_t s = 0; s < a.hdr->size; ++s) uc_insert_table(a, a.sid[s], static_cast<int32_t>(s));
}

// erase (cache.hpp:174-180): the last slot moves into the hole
__device__ void uc_erase_at(const UcArrays& a, int64_t pos) {
  const int32_t slot = a.table[pos];
  if (a.smark[slot] == a.hdr->cur_mark) --a.hdr->at_cur;
  a.table[pos] = kTomb;
  ++a.hdr->tombs;
  const int32_t last = static_cast<int32_t>(a.hdr->size - 1);
  if (slot != last) {
    const int64_t lp = uc_lookup(a, a.sid[last]);
    a.table[lp] = slot;
    a.sid[slot] = a.sid[last];
    a.sver[slot] = a.sver[last];
    a.smark[slot] = a.smark[last];
    a.sfreq[slot] = a.sfreq[last];
    a.slast[slot] = a.slast[last];
    a.sfp[slot] = a.sfp[last];
    a.pin[slot] = a.pin[last];
  }
  a.pin[last] = 0;
  --a.hdr->size;
}

__global__ void k_uc_init(UcArrays a) {
  for (uint64_t h = blockIdx.x * blockDim.x + threadIdx.x; h < a.H; h += gridDim.x * blockDim.x)
    a.table[h] = kEmpty;
  for (uint64_t s = blockIdx.x * blockDim.x + threadIdx.x; s < a.cap; s += gridDim.x * blockDim.x)
    a.pin[s] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.hdr = UcHdr{};
    a.hdr->cur_mark = 1;
  }
}

// touch (cache.hpp:102-122)
__global__ void k_uc_touch(UcArrays a, uint32_t id, int latest, unsigned long long now, double fp) {
  UcHdr& h = *a.hdr;
  h.err = kUcOk;
  const int64_t pos = uc_lookup(a, id);
  if (pos < 0) {
    if (h.size == a.cap) {
      h.err = kUcTouchFull;
      return;
    }
    const int32_t s = static_cast<int32_t>(h.size++);
    a.sid[s] = id;
    a.sver[s] = latest ? 1 : 0;
    a.smark[s] = h.cur_mark;
    a.sfreq[s] = 1;
    a.slast[s] = now;
    a.sfp[s] = fp;
    a.pin[s] = 0;
    uc_insert_table(a, id, s);
    ++h.at_cur;
    uc_rebuild_if_crowded(a);
    return;
  }
  const int32_t s = a.table[pos];
  if (a.smark[s] != h.cur_mark) ++h.at_cur;
  a.smark[s] = h.cur_mark;
  a.sfreq[s] += 1;
  a.slast[s] = now;
  a.sver[s] = latest ? 1 : 0;
}

// set_version (cache.hpp:126-135)
__global__ void k_uc_set_version(UcArrays a, uint32_t id, int latest) {
  a.hdr->err = kUcOk;
  const int64_t pos = uc_lookup(a, id);
  if (pos < 0) {
    a.hdr->err = kUcSetVersion;
    return;
  }
  a.sver[a.table[pos]] = latest ? 1 : 0;
}

__global__ void k_uc_erase(UcArrays a, uint32_t id) {
  a.hdr->err = kUcOk;
  const int64_t pos = uc_lookup(a, id);
  if (pos >= 0) {
    uc_erase_at(a, pos);
    uc_rebuild_if_crowded(a);
  }
}

__global__ void k_uc_find(UcArrays a, uint32_t id) {
  UcHdr& h = *a.hdr;
  h.err = kUcOk;
  const int64_t pos = uc_lookup(a, id);
  h.found = pos >= 0;
  if (pos >= 0) {
    const int32_t s = a.table[pos];
    h.f_ver = a.sver[s];
    h.f_mark = a.smark[s];
    h.f_freq = a.sfreq[s];
    h.f_last = a.slast[s];
  }
}

// A candidate in victim order under the active policy.
struct Cand {
  double pri;  // priority ratio (policy 1)
  unsigned long long last;
  uint32_t ver, mark, freq, id;
  int slot;  // -1: none
};

__device__ __forceinline__ bool cand_less(const Cand& a, const Cand& b, int policy) {
  if (b.slot < 0) return a.slot >= 0;
  if (a.slot < 0) return false;
  if (policy == 0) {  // VictimKey (cache.hpp:47-58)
    if (a.ver != b.ver) return a.ver < b.ver;
    if (a.mark != b.mark) return a.mark < b.mark;
    if (a.freq != b.freq) return a.freq < b.freq;
    if (a.last != b.last) return a.last < b.last;
    return a.id < b.id;
  }
  // pick_victim (cache.hpp:213-224): strict '<' on priority, then recency, then id
  if (a.pri < b.pri) return true;
  if (!(a.pri == b.pri)) return false;
  if (a.last != b.last) return a.last < b.last;
  return a.id < b.id;
}

__device__ __forceinline__ Cand cand_shfl(const Cand& c, int src) {
  Cand o;
  o.pri = __shfl_sync(0xffffffffu, c.pri, src);
  o.last = __shfl_sync(0xffffffffu, c.last, src);
  o.ver = __shfl_sync(0xffffffffu, c.ver, src);
  o.mark = __shfl_sync(0xffffffffu, c.mark, src);
  o.freq = __shfl_sync(0xffffffffu, c.freq, src);
  o.id = __shfl_sync(0xffffffffu, c.id, src);
  o.slot = __shfl_sync(0xffffffffu, c.slot, src);
  return o;
}

// select_victim (needed == 0) or evict_for(needed, pinned) (cache.hpp:141-170):
// one CTA; pinned ids are flagged on their slots for the duration.
__global__ void __launch_bounds__(kSelT)
    k_uc_select(UcArrays a, int policy, unsigned long long needed, const uint32_t* __restrict__ pinned,
                uint64_t npinned, uint32_t* __restrict__ victims) {
  __shared__ Cand part[kSelT / 32];
  __shared__ int s_slot;
  UcHdr& h = *a.hdr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool select_only = needed == 0;
  if (tid == 0) {
    h.err = kUcOk;
    h.nvict = 0;
  }
  if (!select_only) {
    if (a.cap - h.size >= needed) return;  // evict_for: nothing to do
    __syncthreads();
    if (tid == 0 && h.size == a.cap && h.at_cur == h.size) {  // maybe_advance_mark (:187-192)
      ++h.cur_mark;
      h.at_cur = 0;
    }
    for (uint64_t q = tid; q < npinned; q += kSelT) {
      const int64_t pos = uc_lookup(a, pinned[q]);
      if (pos >= 0) a.pin[a.table[pos]] = 1;
    }
  }
  __syncthreads();
  for (;;) {
    if (!select_only && a.cap - h.size >= needed) break;
    Cand best;
    best.slot = -1;
    for (uint64_t s = tid; s < h.size; s += kSelT) {
      if (a.pin[s]) continue;
      Cand c;
      c.ver = a.sver[s];
      c.mark = a.smark[s];
      c.freq = a.sfreq[s];
      c.last = a.slast[s];
      c.id = a.sid[s];
      c.slot = static_cast<int>(s);
      c.pri = 0.0;
      if (policy == 1) {
        const double num = __dmul_rn(__dmul_rn(c.ver ? 2.0 : 1.0, static_cast<double>(c.mark)),
                                     static_cast<double>(c.freq));
        c.pri = __ddiv_rn(num, a.sfp[s]);
      }
      if (cand_less(c, best, policy)) best = c;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const Cand o = cand_shfl(best, (lane + off) & 31);
      if (cand_less(o, best, policy)) best = o;
    }
    if (lane == 0) part[warp] = best;
    __syncthreads();
    if (warp == 0) {
      best = part[lane];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const Cand o = cand_shfl(best, (lane + off) & 31);
        if (cand_less(o, best, policy)) best = o;
      }
      if (lane == 0) {
        s_slot = best.slot;
        if (best.slot < 0) {
          h.err = select_only ? kUcNoVictim : kUcAllPinned;
        } else {
          victims[h.nvict++] = best.id;
          if (!select_only) uc_erase_at(a, uc_lookup(a, best.id));
        }
      }
    }
    __syncthreads();
    if (select_only || s_slot < 0) break;
  }
  __syncthreads();
  for (uint64_t s = tid; s < a.cap; s += kSelT) a.pin[s] = 0;
  if (tid == 0 && !select_only) uc_rebuild_if_crowded(a);
}

}  // namespace
}  // namespace edx

struct edx_cache {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t cap = 0;
  int policy = 0;
  edx::DevBuf<edx::UcHdr> hdr;
  edx::DevBuf<int32_t> table;
  edx::DevBuf<uint32_t> sid, smark, sfreq, pinned, victims;
  edx::DevBuf<uint8_t> sver, pin;
  edx::DevBuf<unsigned long long> slast;
  edx::DevBuf<double> sfp;
  uint64_t H = 0;
  edx::UcHdr host{};

  edx::UcArrays arrays() {
    return edx::UcArrays{hdr.p, table.p, H, cap, sid.p, sver.p, smark.p, sfreq.p, slast.p, sfp.p,
                         pin.p};
  }
  // wait for the call, refresh the host copy of the header, raise its error
  void finish() {
    EDX_CUDA(cudaGetLastError());
    EDX_CUDA(cudaMemcpyAsync(&host, hdr.p, sizeof host, cudaMemcpyDeviceToHost, stream));
    EDX_CUDA(cudaStreamSynchronize(stream));
    switch (host.err) {
      case edx::kUcTouchFull:
        throw edx::Error(EDX_LOGIC_ERROR, "touch would insert into a full cache; evict first");
      case edx::kUcSetVersion:
        throw edx::Error(EDX_INVALID_ARGUMENT, "set_version on non-resident embedding");
      case edx::kUcNoVictim: throw edx::Error(EDX_LOGIC_ERROR, "no evictable entry");
      case edx::kUcAllPinned:
        throw edx::Error(EDX_LOGIC_ERROR, "every cache entry is pinned; cannot evict");
      default: break;
    }
  }
};

extern "C" {

int edx_cache_create(uint64_t capacity, int policy, int device, edx_cache** out) {
  return edx::guard([&] {
    if (capacity == 0) edx::invalid("cache capacity must be positive");
    if (capacity >= (1ULL << 30)) edx::invalid("cache capacity too large");
    if (policy != 0 && policy != 1) edx::invalid("unknown victim policy");
    auto c = std::make_unique<edx_cache>();
    c->device = device;
    EDX_CUDA(cudaSetDevice(device));
    EDX_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->cap = capacity;
    c->policy = policy;
    c->H = 16;
    while (c->H < 2 * capacity) c->H <<= 1;
    c->hdr.ensure(1);
    c->table.ensure(c->H);
    c->sid.ensure(capacity);
    c->smark.ensure(capacity);
    c->sfreq.ensure(capacity);
    c->victims.ensure(capacity);
    c->sver.ensure(capacity);
    c->pin.ensure(capacity);
    c->slast.ensure(capacity);
    c->sfp.ensure(capacity);
    edx::k_uc_init<<<64, 256, 0, c->stream>>>(c->arrays());
    c->finish();
    *out = c.release();
  });
}

void edx_cache_destroy(edx_cache* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int edx_cache_touch(edx_cache* c, uint32_t id, int latest, uint64_t now, double footprint) {
  return edx::guard([&] {
    EDX_CUDA(cudaSetDevice(c->device));
    edx::k_uc_touch<<<1, 1, 0, c->stream>>>(c->arrays(), id, latest, now, footprint);
    c->finish();
  });
}

int edx_cache_set_version(edx_cache* c, uint32_t id, int latest) {
  return edx::guard([&] {
    EDX_CUDA(cudaSetDevice(c->device));
    edx::k_uc_set_version<<<1, 1, 0, c->stream>>>(c->arrays(), id, latest);
    c->finish();
  });
}

int edx_cache_erase(edx_cache* c, uint32_t id) {
  return edx::guard([&] {
    EDX_CUDA(cudaSetDevice(c->device));
    edx::k_uc_erase<<<1, 1, 0, c->stream>>>(c->arrays(), id);
    c->finish();
  });
}

int edx_cache_find(edx_cache* c, uint32_t id, int* found, int* version_latest, uint32_t* mark,
                   uint32_t* frequency, uint64_t* last_access) {
  return edx::guard([&] {
    EDX_CUDA(cudaSetDevice(c->device));
    edx::k_uc_find<<<1, 1, 0, c->stream>>>(c->arrays(), id);
    c->finish();
    *found = c->host.found;
    if (c->host.found) {
      if (version_latest) *version_latest = static_cast<int>(c->host.f_ver);
      if (mark) *mark = c->host.f_mark;
      if (frequency) *frequency = c->host.f_freq;
      if (last_access) *last_access = c->host.f_last;
    }
  });
}

int edx_cache_select_victim(edx_cache* c, uint32_t* victim) {
  return edx::guard([&] {
    EDX_CUDA(cudaSetDevice(c->device));
    EDX_CUDA(cudaMemcpyAsync(&c->host, c->hdr.p, sizeof c->host, cudaMemcpyDeviceToHost, c->stream));
    EDX_CUDA(cudaStreamSynchronize(c->stream));
    if (c->host.size != c->cap) edx::logic("select_victim requires a full cache");
    edx::k_uc_select<<<1, edx::kSelT, 0, c->stream>>>(c->arrays(), c->policy, 0, nullptr, 0,
                                                      c->victims.p);
    c->finish();
    EDX_CUDA(cudaMemcpy(victim, c->victims.p, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  });
}

int edx_cache_evict_for(edx_cache* c, uint64_t needed, const uint32_t* pinned, uint64_t n_pinned,
                        uint32_t* victims, uint64_t* n_victims) {
  return edx::guard([&] {
    if (needed > c->cap) edx::invalid("cannot free more slots than the capacity");
    EDX_CUDA(cudaSetDevice(c->device));
    *n_victims = 0;
    if (needed == 0) return;
    if (n_pinned) {
      c->pinned.ensure(n_pinned);
      EDX_CUDA(cudaMemcpyAsync(c->pinned.p, pinned, n_pinned * 4, cudaMemcpyHostToDevice, c->stream));
    }
    edx::k_uc_select<<<1, edx::kSelT, 0, c->stream>>>(c->arrays(), c->policy, needed, c->pinned.p,
                                                      n_pinned, c->victims.p);
    try {
      c->finish();
    } catch (...) {
      // the reference reports the victims it erased before throwing only
      // through its state; the caller sees the state via export
      throw;
    }
    *n_victims = c->host.nvict;
    if (c->host.nvict)
      EDX_CUDA(cudaMemcpy(victims, c->victims.p, c->host.nvict * 4, cudaMemcpyDeviceToHost));
  });
}

int edx_cache_info(edx_cache* c, uint64_t* size, uint32_t* current_mark, uint64_t* at_current_mark) {
  return edx::guard([&] {
    EDX_CUDA(cudaSetDevice(c->device));
    EDX_CUDA(cudaMemcpyAsync(&c->host, c->hdr.p, sizeof c->host, cudaMemcpyDeviceToHost, c->stream));
    EDX_CUDA(cudaStreamSynchronize(c->stream));
    if (size) *size = c->host.size;
    if (current_mark) *current_mark = c->host.cur_mark;
    if (at_current_mark) *at_current_mark = c->host.at_cur;
  });
}

int edx_cache_export(edx_cache* c, uint32_t* ids, uint8_t* version, uint32_t* mark,
                     uint32_t* frequency, uint64_t* last_access, uint64_t cap_out, uint64_t* count) {
  return edx::guard([&] {
    EDX_CUDA(cudaSetDevice(c->device));
    EDX_CUDA(cudaMemcpyAsync(&c->host, c->hdr.p, sizeof c->host, cudaMemcpyDeviceToHost, c->stream));
    EDX_CUDA(cudaStreamSynchronize(c->stream));
    const uint64_t k = c->host.size;
    *count = k;
    if (ids == nullptr || k == 0) return;
    if (cap_out < k) edx::invalid("export buffer too small");
    EDX_CUDA(cudaMemcpy(ids, c->sid.p, k * 4, cudaMemcpyDeviceToHost));
    if (version) EDX_CUDA(cudaMemcpy(version, c->sver.p, k, cudaMemcpyDeviceToHost));
    if (mark) EDX_CUDA(cudaMemcpy(mark, c->smark.p, k * 4, cudaMemcpyDeviceToHost));
    if (frequency) EDX_CUDA(cudaMemcpy(frequency, c->sfreq.p, k * 4, cudaMemcpyDeviceToHost));
    if (last_access) EDX_CUDA(cudaMemcpy(last_access, c->slast.p, k * 8, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
