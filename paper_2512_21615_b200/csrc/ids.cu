// Arbitrary 32-bit embedding ids (SimState::global_ is an
// unordered_map<EmbeddingId, EmbeddingState>, sim.hpp:266; every WorkerCache
// is an unordered_map too, cache.hpp:238): the engine's device id table.
//
// The engine's per-embedding tables (global masks, per-worker cache index,
// step scratch) are dense arrays indexed by a *slot*.  With a known id bound
// (id_space > 0: Zipf and schema-flattened ids) the slot is the id itself.
// Otherwise every id of a batch is translated to its slot once, at the start
// of the iteration, through one GPU-resident open-addressing table shared by
// the global state and all n worker caches -- one probe per id occurrence,
// not one per (worker, id) -- and every kernel after it runs on the slot
// stream unchanged.  New ids take the next free slot; slots are never
// recycled, as the reference never erases global_ entries.
//
// Table: 2^k 64-bit entries (id << 32 | slot), linear probing, load <= 1/2,
// EMPTY = all ones (slot 0xFFFFFFFF never exists).  An insert claims its
// entry with a CAS that leaves slot = PENDING, allocates the slot, writes
// slot2id[slot] and publishes the entry; a prober that finds its own id still
// PENDING waits for that (already running) thread.  Lanes of a warp that hold
// the same id -- Zipf-hot ids repeat within a warp's 32 positions -- are
// grouped with __match_any_sync and probe once (warp-cooperative probing).
// Slot numbers depend on the order of concurrent inserts, but nothing
// observable depends on them: victim keys use the real id (slot2id), and the
// exports map slots back to ids.
#include <climits>

#include "ids.h"

namespace edx {
namespace {

constexpr unsigned long long kEmpty = ~0ULL;
constexpr uint32_t kPending = 0xFFFFFFFEu;
constexpr uint32_t kAbsent = 0xFFFFFFFFu;
constexpr int kT = 256;

__device__ __forceinline__ uint64_t id_hash(uint32_t id) {
  // murmur3 fmix32
  uint32_t h = id;
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ unsigned long long load_entry(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Slot of `id`, inserting it when `insert` (kAbsent when absent and not inserting).
__device__ uint32_t probe(uint32_t id, unsigned long long* tab, uint64_t mask, bool insert,
                          uint32_t* slot2id, unsigned long long* count, uint64_t cap,
                          int* flags) {
  uint64_t h = id_hash(id) & mask;
  for (uint64_t n = 0; n <= mask; ++n, h = (h + 1) & mask) {
    unsigned long long e = load_entry(tab + h);
    if (e == kEmpty) {
      if (!insert) return kAbsent;
      const unsigned long long claim = (static_cast<unsigned long long>(id) << 32) | kPending;
      const unsigned long long prev = atomicCAS(tab + h, kEmpty, claim);
      if (prev == kEmpty) {
        const unsigned long long s = atomicAdd(count, 1ULL);
        if (s >= cap) {  // the host sizes the slots before every batch: a bug
          atomicOr(flags + kFlagInternal, 1);
          atomicExch(tab + h, (static_cast<unsigned long long>(id) << 32) | 0u);
          return 0;
        }
        slot2id[s] = id;
        __threadfence();
        atomicExch(tab + h, (static_cast<unsigned long long>(id) << 32) | s);
        return static_cast<uint32_t>(s);
      }
      e = prev;
    }
    if (static_cast<uint32_t>(e >> 32) == id) {
      while (static_cast<uint32_t>(e) == kPending) {
        __nanosleep(20);
        e = load_entry(tab + h);
      }
      return static_cast<uint32_t>(e);
    }
  }
  atomicOr(flags + kFlagInternal, 1);  // table full: cannot happen at load <= 1/2
  return 0;
}

__global__ void __launch_bounds__(kT)
    k_translate(const uint32_t* __restrict__ ids, uint64_t T, unsigned long long* tab,
                uint64_t mask, int insert, uint32_t* slot2id, unsigned long long* count,
                uint64_t cap, uint32_t* __restrict__ out, int* flags) {
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const unsigned live = __ballot_sync(0xffffffffu, t < T);
  if (t >= T) return;
  const uint32_t id = ids[t];
  const unsigned grp = __match_any_sync(live, id);
  const int leader = __ffs(grp) - 1;
  uint32_t slot = 0;
  if ((threadIdx.x & 31) == leader)
    slot = probe(id, tab, mask, insert != 0, slot2id, count, cap, flags);
  out[t] = __shfl_sync(grp, slot, leader);
}

__global__ void k_fill_u64(unsigned long long* p, uint64_t n, unsigned long long v) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x < n) p[x] = v;
}

// Re-inserts every allocated slot (distinct ids) into a fresh table.
__global__ void k_rehash(const uint32_t* __restrict__ slot2id, uint64_t count,
                         unsigned long long* tab, uint64_t mask) {
  const uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (s >= count) return;
  const uint32_t id = slot2id[s];
  const unsigned long long v = (static_cast<unsigned long long>(id) << 32) | s;
  for (uint64_t h = id_hash(id) & mask;; h = (h + 1) & mask)
    if (atomicCAS(tab + h, kEmpty, v) == kEmpty) return;
}

unsigned grid(uint64_t n) { return static_cast<unsigned>(n ? (n + kT - 1) / kT : 1); }

uint64_t table_size_for(uint64_t slots) {
  uint64_t t = 1024;
  while (t < 2 * slots) t <<= 1;
  return t;
}

}  // namespace

void id_table_init(IdTable& t, uint64_t slot_cap, cudaStream_t s) {
  t.cap = slot_cap;
  t.tab_size = table_size_for(slot_cap);
  t.tab.ensure(t.tab_size);
  t.slot2id.ensure(slot_cap);
  t.count.ensure(1);
  k_fill_u64<<<grid(t.tab_size), kT, 0, s>>>(t.tab.p, t.tab_size, kEmpty);
  EDX_LAUNCHED();
  EDX_CUDA(cudaMemsetAsync(t.count.p, 0, sizeof(unsigned long long), s));
  t.used = 0;
}

void id_table_translate(IdTable& t, const uint32_t* ids, uint64_t T, uint32_t* slots, bool insert,
                        int* flags, cudaStream_t s) {
  if (T == 0) return;
  k_translate<<<grid(T), kT, 0, s>>>(ids, T, t.tab.p, t.tab_size - 1, insert ? 1 : 0, t.slot2id.p,
                                      t.count.p, t.cap, slots, flags);
  EDX_LAUNCHED();
}

void id_table_grow(IdTable& t, uint64_t slot_cap, cudaStream_t s) {
  // the slot -> id array keeps its prefix; the table is rebuilt from it
  DevBuf<uint32_t> old;
  std::swap(old.p, t.slot2id.p);
  std::swap(old.n, t.slot2id.n);
  t.slot2id.ensure(slot_cap);
  if (t.used)
    EDX_CUDA(cudaMemcpyAsync(t.slot2id.p, old.p, t.used * sizeof(uint32_t),
                             cudaMemcpyDeviceToDevice, s));
  t.cap = slot_cap;
  t.tab_size = table_size_for(slot_cap);
  t.tab.release();
  t.tab.ensure(t.tab_size);
  k_fill_u64<<<grid(t.tab_size), kT, 0, s>>>(t.tab.p, t.tab_size, kEmpty);
  EDX_LAUNCHED();
  if (t.used) {
    k_rehash<<<grid(t.used), kT, 0, s>>>(t.slot2id.p, t.used, t.tab.p, t.tab_size - 1);
    EDX_LAUNCHED();
  }
  EDX_CUDA(cudaStreamSynchronize(s));
}

}  // namespace edx
