// K7: SimState::step on device (sim.hpp:87-218) over WorkerCache semantics
// (cache.hpp:102-201).
//
// The reference walks the batch sample by sample, then each worker's needs
// one by one through a std::set of victim keys.  The device version rests on
// four properties of that code (re-derived in DESIGN.md §4):
//  1. Phases 1 and 3 mutate only the state of the id at hand (sim.hpp:123-153,
//     194-204): they are id-parallel and unordered_map order cannot matter.
//  2. Phase 2 of worker j flips only worker j's bits and cache (sim.hpp:157-190):
//     workers are independent.
//  3. Within worker j's phase 2, entries that are not needed this iteration
//     (not pinned) are never touched, so their VictimKeys are frozen after
//     phase 1; every eviction takes the least non-pinned key.  The victims are
//     therefore exactly the E_j least keys, E_j = max(0, inserts - free slots),
//     and the t-th evicting insert (in need order) removes the t-th least.
//  4. at_current_mark_ changes by +1 per touch of an entry whose mark is not
//     current, +1 per insert and -1 per eviction of a current-mark entry; the
//     epoch advance (cache.hpp:187-192) fires at the first evicting insert where
//     that counter equals the capacity.  A prefix scan over need order finds
//     it; it can fire at most once per step (a second firing means every entry
//     is pinned, which the reference reports as a logic_error).
// The rest is bookkeeping: need lists in first-occurrence order come from a
// stable sort of (worker, position) keys, counts are integer atomics
// (order-free), and the realised cost is summed on the host in worker order
// (sim.hpp:208-216).
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "engine.h"
#include "step.h"

namespace edx {

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("EDX_PDL");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  return on;
}

namespace {

constexpr int kT = 256;
inline unsigned grid_for(uint64_t n, int t = kT) {
  return static_cast<unsigned>(std::max<uint64_t>(1, (n + t - 1) / t));
}

// counters layout (unsigned long long)
//   [0,n) miss_pull_w  [n,2n) update_push_w  [2n,3n) evict_push_w  [3n] hits
//   [3n+1] unique ids U   [3n+2] need items N
// per-worker scalars (uint32, kWS per worker)
enum WS : int {
  kWsNeeds = 0,    // need items of the worker
  kWsInserts = 1,  // non-resident needs
  kWsFree = 2,     // free slots at phase-2 start
  kWsEvict = 3,    // evictions E_j
  kWsCand = 4,     // non-pinned candidates
  kWsAdvance = 5,  // need item (worker-local) of the epoch advance, UINT_MAX = none
  kWsSize0 = 6,
  kWsNeedOff = 7,  // start of the worker's need items
  kWsCandOff = 8,  // start of the worker's sorted candidates
  kWsInsBase = 9,  // exclusive insert-scan value at the worker's first item
  kWsConBase = 10, // exclusive contribution-scan value at the worker's first item
  kWsVa = 11,      // large caches: victims with version 0, mark != current
  kWsVb = 12,      //   version 0, mark == current
  kWsVc = 13,      //   version 1, mark != current (the rest: version 1, current)
  kWS = 14
};

// Head of the step: zero the counters and per-worker scalars, map each id
// position to its sample, and the first position of every id.
__global__ void k_step_begin(const uint64_t* __restrict__ offsets, uint64_t rows,
                             uint32_t* __restrict__ occ_sample, const uint32_t* __restrict__ ids,
                             uint64_t T, int32_t* __restrict__ first_pos,
                             unsigned long long* __restrict__ counters, uint32_t ncnt,
                             uint32_t* __restrict__ ws, uint32_t nws, uint32_t* __restrict__ epoch) {
  pdl_wait();
  pdl_trigger();
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i == 0) *epoch += 1;  // this step's need-cell tag (never 0; unique for 2^32 - 1 steps)
  if (i < ncnt) counters[i] = 0;
  if (i < nws) ws[i] = 0;
  if (i < rows)
    for (uint64_t p = offsets[i]; p < offsets[i + 1]; ++p) occ_sample[p] = static_cast<uint32_t>(i);
  if (i < T) {
    // Zipf-hot ids occur in thousands of samples: test before the atomic.  The
    // table only decreases, so a stale read is >= the true minimum -- skipping
    // when it is already <= p is exact -- and CTAs run roughly in position
    // order, so a hot id's minimum is in place after its first few occurrences.
    int32_t* slot = first_pos + ids[i];
    if (*slot > static_cast<int32_t>(i)) atomicMin(slot, static_cast<int32_t>(i));
  }
}

__global__ void k_unique_flag(const uint32_t* __restrict__ ids, uint64_t T,
                              const int32_t* __restrict__ first_pos, uint32_t* __restrict__ flag) {
  pdl_wait();
  pdl_trigger();
  const uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (p > T) return;
  flag[p] = (p < T && first_pos[ids[p]] == static_cast<int32_t>(p)) ? 1u : 0u;
}

__global__ void k_unique_scatter(const uint32_t* __restrict__ ids, uint64_t T,
                                 const int32_t* __restrict__ first_pos,
                                 const uint32_t* __restrict__ uidx, uint32_t* __restrict__ uniq,
                                 unsigned long long* counters, int n) {
  pdl_wait();
  pdl_trigger();
  const uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (p == T) counters[3 * n + 1] = uidx[T];
  if (p >= T) return;
  if (first_pos[ids[p]] == static_cast<int32_t>(p)) uniq[uidx[p]] = ids[p];
}

// The unique index of every occurrence's id, in the decision-independent head
// (which overlaps the dispatch): the step's passes read it by position.
__global__ void k_unique_of_pos(const uint32_t* __restrict__ ids, uint64_t T,
                                const int32_t* __restrict__ first_pos,
                                const uint32_t* __restrict__ uidx, uint32_t* __restrict__ upos) {
  pdl_wait();
  pdl_trigger();
  const uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (p < T) upos[p] = uidx[first_pos[ids[p]]];
}

// Need cells are tagged with the step's epoch (high 32 bits), so no pass
// resets them: a cell from an earlier step reads as empty.
//   first: epoch << 32 | ~position, kept by atomicMax (newest epoch, then
//          the least position);
//   count: epoch << 32 | occurrences; the first adder of a step installs
//          (epoch, 1) by CAS, every other occurrence adds 1.
__device__ __forceinline__ unsigned long long first_tag(uint32_t epoch, uint64_t p) {
  return (static_cast<unsigned long long>(epoch) << 32) | (0xFFFFFFFFu - static_cast<uint32_t>(p));
}

// needs (sim.hpp:103-117): per (worker, id) first position and count, and
// the trainer mask of every id.
__global__ void k_needs(uint64_t T, const uint32_t* __restrict__ occ_sample,
                        const int32_t* __restrict__ decision, const uint32_t* __restrict__ upos,
                        uint64_t ucap, unsigned long long* __restrict__ need_first,
                        unsigned long long* __restrict__ need_cnt,
                        unsigned long long* __restrict__ umask, const uint32_t* __restrict__ epoch_dev) {
  pdl_wait();
  pdl_trigger();
  const uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (p >= T) return;
  const uint32_t epoch = *epoch_dev;
  const int j = decision[occ_sample[p]];
  const uint32_t u = upos[p];
  const uint64_t x = static_cast<uint64_t>(j) * ucap + u;
  // test before the atomics: the cell only grows within a step
  const unsigned long long f = first_tag(epoch, p);
  if (need_first[x] < f) atomicMax(need_first + x, f);
  const unsigned long long tag = static_cast<unsigned long long>(epoch) << 32;
  unsigned long long cur = need_cnt[x];
  bool counted = false;
  while ((cur & 0xFFFFFFFF00000000ULL) != tag) {  // a stale cell: install (epoch, 1)
    const unsigned long long prev = atomicCAS(need_cnt + x, cur, tag | 1ULL);
    if (prev == cur) {
      counted = true;
      break;
    }
    cur = prev;
  }
  if (!counted) atomicAdd(need_cnt + x, 1ULL);
  if (!((umask[u] >> j) & 1ULL)) atomicOr(umask + u, 1ULL << j);
}

// first occurrence of (worker, id) -> sortable key (worker << 32 | position)
__global__ void k_need_keys(uint64_t T, const uint32_t* __restrict__ occ_sample,
                            const int32_t* __restrict__ decision, const uint32_t* __restrict__ upos,
                            uint64_t ucap, const unsigned long long* __restrict__ need_first,
                            uint64_t* __restrict__ keys, uint32_t* __restrict__ ws,
                            const uint32_t* __restrict__ epoch_dev) {
  pdl_wait();
  pdl_trigger();
  const uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (p >= T) return;
  const int j = decision[occ_sample[p]];
  const uint32_t u = upos[p];
  const bool first = need_first[static_cast<uint64_t>(j) * ucap + u] == first_tag(*epoch_dev, p);
  keys[p] = first ? ((static_cast<uint64_t>(j) << 32) | p) : ~0ULL;
  // per-worker need count: lanes of one sample share the worker, so one
  // atomic per (warp, worker) group
  const unsigned act = __activemask();
  const unsigned grp = __match_any_sync(act, first ? j : -1 - j);
  if (first && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(ws + j * kWS + kWsNeeds, __popc(grp));
}

// Phase 1: on-demand update push (sim.hpp:119-153).  set_version(false) on
// stale copies is the `latest` mask update itself (version == latest bit).
// Block 0 also lays out the per-worker need CSR (need items are sorted by
// worker, then position) and the phase-2 scalars.
__global__ void k_phase1(const uint32_t* __restrict__ uniq,
                         const unsigned long long* __restrict__ umask,
                         const unsigned long long* counters_ro, int n,
                         ulonglong2* __restrict__ ol, unsigned long long* counters,
                         uint32_t* __restrict__ ws, const uint32_t* __restrict__ size,
                         uint64_t capacity) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned int push[kMaxWorkers];
  if (threadIdx.x < kMaxWorkers) push[threadIdx.x] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t run = 0;
    for (int j = 0; j < n; ++j) {
      ws[j * kWS + kWsNeedOff] = run;
      run += ws[j * kWS + kWsNeeds];
      ws[j * kWS + kWsSize0] = size[j];
      ws[j * kWS + kWsFree] = static_cast<uint32_t>(capacity - size[j]);
      ws[j * kWS + kWsAdvance] = UINT_MAX;
    }
    counters[3 * n + 2] = run;
  }
  __syncthreads();
  const uint64_t U = counters_ro[3 * n + 1];
  const uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (u < U) {
    const uint32_t id = uniq[u];
    ulonglong2 st = ol[id];
    if (st.x != 0) {
      const unsigned long long need = umask[u];
      unsigned long long pushers = 0, own = st.x;
      while (own) {
        const int w = __ffsll(static_cast<long long>(own)) - 1;
        own &= own - 1;
        if (need & ~(1ULL << w)) pushers |= 1ULL << w;
      }
      if (pushers) {
        for (unsigned long long it = pushers; it; it &= it - 1)
          atomicAdd(&push[__ffsll(static_cast<long long>(it)) - 1], 1u);
        st.x &= ~pushers;
        if (st.x != 0) st.y = st.x;
        ol[id] = st;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < n && push[threadIdx.x])
    atomicAdd(counters + n + threadIdx.x, static_cast<unsigned long long>(push[threadIdx.x]));
}

__device__ __forceinline__ int item_worker(uint64_t key) { return static_cast<int>(key >> 32); }
__device__ __forceinline__ uint32_t item_pos(uint64_t key) { return static_cast<uint32_t>(key); }

// Phase 2 classification (sim.hpp:168-181): hit / refresh / insert, hit and
// miss-pull tallies, and the pre-advance at_current_mark contribution of
// touches of existing entries (cache.hpp:116).
__global__ void k_classify(const uint64_t* __restrict__ items,
                           const unsigned long long* counters_ro, int n,
                           const uint32_t* __restrict__ ids, const uint32_t* __restrict__ upos,
                           uint64_t ucap, const unsigned long long* __restrict__ need_cnt,
                           const ulonglong2* __restrict__ ol,
                           const unsigned long long* __restrict__ res, uint64_t id_space,
                           const int32_t* __restrict__ slot_of, uint64_t capacity,
                           const uint32_t* __restrict__ smark, const uint32_t* __restrict__ cur_mark,
                           uint8_t* __restrict__ type, uint32_t* __restrict__ ins_flag,
                           int32_t* __restrict__ contrib, unsigned long long* counters,
                           uint32_t* __restrict__ pin, const uint32_t* __restrict__ clock_dev,
                           int32_t* __restrict__ item_slot) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned int miss[kMaxWorkers];
  __shared__ unsigned long long hits;
  if (threadIdx.x < kMaxWorkers) miss[threadIdx.x] = 0;
  if (threadIdx.x == 0) hits = 0;
  __syncthreads();
  const uint64_t N = counters_ro[3 * n + 2];
  const uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (q < N) {
    const uint64_t key = items[q];
    const int j = item_worker(key);
    const uint32_t p = item_pos(key);
    const uint32_t id = ids[p];
    const unsigned long long bit = 1ULL << j;
    const ulonglong2 st = ol[id];
    uint8_t t;
    int32_t c = 1;
    if (st.y & bit) {
      t = 0;
      // (the cell carries this step's tag: its item exists)
      const uint64_t x = static_cast<uint64_t>(j) * ucap + upos[p];
      const uint32_t cnt = static_cast<uint32_t>(need_cnt[x]);
      atomicAdd(&hits, static_cast<unsigned long long>(cnt));
    } else {
      t = (res[id] & bit) ? 1 : 2;
      atomicAdd(&miss[j], 1u);
    }
    if (t != 2) {
      const int32_t s = slot_of[static_cast<uint64_t>(j) * id_space + id];
      item_slot[q] = s;  // k_apply's slot for this resident id
      c = smark[static_cast<uint64_t>(j) * capacity + s] != cur_mark[j] ? 1 : 0;
      // pinned for this iteration's victim selection (large caches)
      if (pin) pin[static_cast<uint64_t>(j) * capacity + s] = *clock_dev + 1u;
    }
    type[q] = t;
    ins_flag[q] = t == 2 ? 1u : 0u;
    contrib[q] = c;
  } else if (q == N) {
    ins_flag[q] = 0;
    contrib[q] = 0;
  }
  __syncthreads();
  if (threadIdx.x < n && miss[threadIdx.x])
    atomicAdd(counters + threadIdx.x, static_cast<unsigned long long>(miss[threadIdx.x]));
  if (threadIdx.x == 0 && hits) atomicAdd(counters + 3 * n, hits);
}

// inserts and evictions per worker (evict_for, cache.hpp:152-170)
__global__ void k_worker_inserts(int n, const uint32_t* __restrict__ ins_scan,
                                 uint32_t* __restrict__ ws, int* __restrict__ flags) {
  const int j = threadIdx.x;
  if (j >= n) return;
  uint32_t* w = ws + j * kWS;
  const uint32_t b = w[kWsNeedOff], e = b + w[kWsNeeds];
  const uint32_t ins = ins_scan[e] - ins_scan[b];
  w[kWsInserts] = ins;
  w[kWsInsBase] = ins_scan[b];
  w[kWsEvict] = ins > w[kWsFree] ? ins - w[kWsFree] : 0;
  w[kWsCand] = 0;
  (void)flags;
}

// --- victim selection for large caches (> kSelCap entries) ---------------
// One cooperative kernel (grid-wide syncs, no host round trip, capturable in
// the iteration's CUDA graph) selects, for every evicting worker j, its E_j
// least VictimKeys among the non-pinned entries (cache.hpp:47-58) -- an MSB
// radix select over the whole cache:
//  * ranges: per-worker min/max of mark, frequency, last access and id over
//    the candidates, so the key (version | mark | freq | last | id, each field
//    minus its minimum) packs into W <= 128 bits, MSB-aligned in a 128-bit word;
//  * level 0: a 4096-bin histogram of the key's top 12 bits (keys built from
//    the entry fields); the bin holding the E_j-th key is found with a block
//    scan; keys in lower bins are victims, keys in that bin stay undecided and
//    are compacted (key, slot) for the next level unless the whole bin is
//    needed; later levels run on the compacted keys only.
// Keys are unique (they end in the id), so the victims are exactly the keys
// <= the E_j-th.  They are written unsorted: the only order-dependent use,
// the epoch scan's "does the t-th victim carry the current mark", follows
// from four counts -- in key order the victims are [version 0, mark !=
// current][version 0, mark == current][version 1, mark != current][version 1,
// mark == current], since every mark is <= the current mark (a touch stamps
// the current one, which only grows) -- so k_evict_contrib derives it from
// kWsVa/kWsVb/kWsVc.  Pinned entries (needed by j this iteration) are the
// ones k_classify stamped with the iteration's stamp.
namespace big {
constexpr int kThreads = 512;
constexpr int kDigit = 12, kBins = 1 << kDigit;
constexpr uint32_t kChunk = 4096;  // entries per work unit
}  // namespace big

typedef unsigned __int128 u128;

// per-worker selection state (global)
struct BigState {
  uint32_t lo[4], hi[4];  // mark, frequency, last access, id over the candidates
  uint32_t cand, need, bin, take_all, active, level, nv, pinned_err;
  uint32_t vc[3];  // victims: version 0 non-current, version 0 current, version 1 non-current
  uint32_t nu[2];  // undecided keys per ping-pong buffer
  int w[5];        // field widths: version, mark, freq, last, id
  int W;
  uint32_t pad[2];
};

__device__ __forceinline__ uint32_t key_digit(u128 k, uint32_t level) {
  const int sh = 128 - big::kDigit * static_cast<int>(level + 1);
  return sh >= 0 ? static_cast<uint32_t>(k >> sh) & (big::kBins - 1)
                 : (static_cast<uint32_t>(k) << (-sh)) & (big::kBins - 1);
}

__device__ __forceinline__ u128 victim_key(const BigState& st, uint32_t ver, uint32_t mark,
                                           uint32_t freq, uint32_t last, uint32_t rid) {
  u128 k = ver;
  k = (k << st.w[1]) | (mark - st.lo[0]);
  k = (k << st.w[2]) | (freq - st.lo[1]);
  k = (k << st.w[3]) | (last - st.lo[2]);
  k = (k << st.w[4]) | (rid - st.lo[3]);
  return k << (128 - st.W);
}

// warp-aggregated append to a per-worker counter; every lane of `mask` calls it
__device__ __forceinline__ uint32_t warp_append(uint32_t* ctr, bool take, unsigned mask) {
  const unsigned bal = __ballot_sync(mask, take);
  const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
  uint32_t base = 0;
  if (lane == leader && bal) base = atomicAdd(ctr, static_cast<uint32_t>(__popc(bal)));
  base = __shfl_sync(mask, base, leader);
  return base + __popc(bal & ((1u << lane) - 1u));
}

struct BigArgs {
  int n;
  uint64_t capacity;
  uint32_t* ws;
  const uint32_t* sid;
  const uint32_t* smark;
  const uint32_t* sfreq;
  const uint32_t* slast;
  const uint32_t* pin;
  const ulonglong2* ol;
  const uint32_t* slot2id;
  const uint32_t* cur_mark;
  const uint32_t* clock_dev;
  BigState* st;
  uint32_t* hist;          // n * kBins
  u128* ukey[2];           // n * capacity each
  uint32_t* uslot[2];
  uint32_t* victims;       // n * capacity: worker j's victims from j * capacity
  uint8_t* eflag;          // n * capacity: candidate (bit 0) and version (bit 1) per entry,
                           // written by the ranges pass, read by the later passes
  int* flags;
};

// One candidate entry of worker j: its key (valid when the entry is a
// non-pinned resident entry), version and current-mark flag.
struct BigEntry {
  bool cand;
  uint32_t ver, mark, freq, last, rid;
};

// The first pass (`first`) derives candidacy and version from the pin stamp
// and the global masks (a random 16-byte gather per entry) and records them
// in one byte per entry; the later passes read that byte instead.
__device__ __forceinline__ BigEntry big_entry(const BigArgs& a, int j, uint32_t s, uint32_t size0,
                                              uint32_t stamp, bool first = false) {
  BigEntry e{};
  const uint64_t g = static_cast<uint64_t>(j) * a.capacity + s;
  uint32_t slot = 0;
  if (first) {
    e.cand = s < size0 && a.pin[g] != stamp;
    if (e.cand) {
      slot = a.sid[g];
      e.ver = static_cast<uint32_t>((a.ol[slot].y >> j) & 1ULL);
    }
    if (s < size0) a.eflag[g] = static_cast<uint8_t>((e.cand ? 1u : 0u) | (e.ver << 1));
  } else {
    const uint32_t f = s < size0 ? a.eflag[g] : 0u;
    e.cand = f & 1u;
    e.ver = (f >> 1) & 1u;
    if (e.cand) slot = a.sid[g];
  }
  if (e.cand) {
    e.mark = a.smark[g];
    e.freq = a.sfreq[g];
    e.last = a.slast[g];
    e.rid = a.slot2id ? a.slot2id[slot] : slot;
  }
  return e;
}

// One histogram increment per warp and digit: the lanes holding the same
// digit are grouped (a concentrated key distribution would otherwise
// serialise whole warps on one shared-memory word).  kNoBin: no increment.
constexpr uint32_t kNoBin = 0xFFFFFFFFu;
__device__ __forceinline__ void hist_add(uint32_t* hsh, uint32_t d) {
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, d);
  if (d != kNoBin && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hsh[d], __popc(peers));
}

// block-wide sum of two counters into shared memory
__device__ void big_block_hist_flush(uint32_t* sh, uint32_t* gh) {
  for (int b = threadIdx.x; b < big::kBins; b += blockDim.x) {
    const uint32_t v = sh[b];
    if (v) atomicAdd(gh + b, v);
    sh[b] = 0;
  }
}

// the bin holding the need-th key of worker j's histogram (block-wide)
__device__ void big_select(const BigArgs& a, int j, uint32_t* scan_sh) {
  BigState& st = a.st[j];
  uint32_t* h = a.hist + static_cast<uint64_t>(j) * big::kBins;
  constexpr int per = big::kBins / big::kThreads;  // 8 bins per thread
  uint32_t v[per], sum = 0;
#pragma unroll
  for (int q = 0; q < per; ++q) {
    v[q] = h[threadIdx.x * per + q];
    h[threadIdx.x * per + q] = 0;  // ready for the next level
    sum += v[q];
  }
  // block exclusive scan of the per-thread sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) scan_sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t x = lane < big::kThreads / 32 ? scan_sh[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane < big::kThreads / 32) scan_sh[32 + lane] = x - scan_sh[lane];
  }
  __syncthreads();
  const uint32_t need = st.need;
  uint32_t run = scan_sh[32 + warp] + inc - sum;  // exclusive prefix of this thread
  if (run < need && need <= run + sum) {
#pragma unroll
    for (int q = 0; q < per; ++q) {
      if (run + v[q] >= need) {
        st.bin = threadIdx.x * per + q;
        st.need = need - run;
        st.take_all = (need - run == v[q]) ? 1u : 0u;
        break;
      }
      run += v[q];
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(big::kThreads, 1)
    k_big_select(BigArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t hsh[big::kBins];
  __shared__ uint32_t red[big::kThreads / 32][9];
  __shared__ uint32_t scan_sh[64];
  const int n = a.n;
  const uint32_t stamp = *a.clock_dev + 1u;
  const uint32_t chunks = static_cast<uint32_t>((a.capacity + big::kChunk - 1) / big::kChunk);
  const uint64_t gtid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // no evicting worker (every step while the caches fill): nothing to select,
  // and no grid-wide sync -- every block sees the same E_j and returns
  {
    bool any = false;
    for (int j = 0; j < n; ++j) any |= a.ws[j * kWS + kWsEvict] > 0;
    if (!any) {
      if (gtid < static_cast<uint64_t>(n)) {
        uint32_t* w = a.ws + gtid * kWS;
        w[kWsCand] = 0;
        w[kWsCandOff] = static_cast<uint32_t>(gtid * a.capacity);
        w[kWsVa] = w[kWsVb] = w[kWsVc] = 0;
      }
      return;
    }
  }
  for (int b = threadIdx.x; b < big::kBins; b += blockDim.x) hsh[b] = 0;

  // ---- init
  if (gtid < static_cast<uint64_t>(n)) {
    BigState& st = a.st[gtid];
    const uint32_t* w = a.ws + gtid * kWS;
    for (int q = 0; q < 4; ++q) {
      st.lo[q] = UINT_MAX;
      st.hi[q] = 0;
    }
    st.cand = st.nv = st.level = st.bin = st.take_all = st.pinned_err = 0;
    st.pad[0] = UINT_MAX;  // level at which the worker's selection finished
    st.vc[0] = st.vc[1] = st.vc[2] = 0;
    st.nu[0] = st.nu[1] = 0;
    st.need = w[kWsEvict];
    st.active = w[kWsEvict] > 0 ? 1u : 0u;
  }
  for (uint64_t x = gtid; x < static_cast<uint64_t>(n) * big::kBins;
       x += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    a.hist[x] = 0;
  grid.sync();

  // ---- ranges of the candidates' fields
  for (uint32_t u = blockIdx.x; u < static_cast<uint32_t>(n) * chunks; u += gridDim.x) {
    const int j = static_cast<int>(u / chunks);
    if (!a.st[j].active) continue;
    const uint32_t size0 = a.ws[j * kWS + kWsSize0], base = (u % chunks) * big::kChunk;
    if (base >= size0) continue;
    uint32_t v[9] = {UINT_MAX, UINT_MAX, UINT_MAX, UINT_MAX, 0, 0, 0, 0, 0};
    for (uint32_t s = base + threadIdx.x; s < base + big::kChunk && s < size0; s += blockDim.x) {
      const BigEntry e = big_entry(a, j, s, size0, stamp, true);
      if (!e.cand) continue;
      const uint32_t f[4] = {e.mark, e.freq, e.last, e.rid};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[q] = min(v[q], f[q]);
        v[4 + q] = max(v[4 + q], f[q]);
      }
      ++v[8];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      v[q] = __reduce_min_sync(0xffffffffu, v[q]);
      v[4 + q] = __reduce_max_sync(0xffffffffu, v[4 + q]);
    }
    v[8] = __reduce_add_sync(0xffffffffu, v[8]);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 9; ++q) red[warp][q] = v[q];
    __syncthreads();
    if (threadIdx.x < 9) {
      const int q = threadIdx.x;
      uint32_t r = q < 4 ? UINT_MAX : 0u;
      for (int x = 0; x < big::kThreads / 32; ++x)
        r = q < 4 ? min(r, red[x][q]) : (q < 8 ? max(r, red[x][q]) : r + red[x][q]);
      BigState& st = a.st[j];
      if (q < 4) {
        if (r != UINT_MAX) atomicMin(&st.lo[q], r);
      } else if (q < 8) {
        if (r) atomicMax(&st.hi[q - 4], r);
      } else if (r) {
        atomicAdd(&st.cand, r);
      }
    }
    __syncthreads();
  }
  grid.sync();

  // ---- field widths (every block keeps its own copy in the state it reads)
  if (gtid < static_cast<uint64_t>(n)) {
    BigState& st = a.st[gtid];
    if (st.active) {
      st.w[0] = 1;
      int W = 1;
      for (int q = 0; q < 4; ++q) {
        const uint32_t span = st.hi[q] > st.lo[q] ? st.hi[q] - st.lo[q] : 0u;
        st.w[1 + q] = span ? 32 - __clz(span) : 0;
        W += st.w[1 + q];
      }
      st.W = W;
      if (st.cand < st.need) {  // every remaining entry is pinned (cache.hpp:164)
        st.pinned_err = 1;
        atomicOr(a.flags + kFlagPinned, 1);
        st.active = 0;
      } else if (W > 128) {  // only reachable at ~2^32 epochs
        atomicOr(a.flags + kFlagKeyRange, 1);
        st.active = 0;
      }
    }
  }
  grid.sync();

  // ---- radix select, level by level
  for (uint32_t level = 0;; ++level) {
    // any worker still selecting?  (uniform: every block reads the same state)
    bool any = false;
    for (int j = 0; j < n; ++j) any |= a.st[j].active != 0 && a.st[j].pad[0] == UINT_MAX;
    if (!any) break;
    const int in = (level + 1) & 1, out = level & 1;  // U buffers: level L reads in, writes out
    // histogram of this level's digit
    if (level == 0) {
      for (uint32_t u = blockIdx.x; u < static_cast<uint32_t>(n) * chunks; u += gridDim.x) {
        const int j = static_cast<int>(u / chunks);
        const BigState& st = a.st[j];
        if (!st.active || st.pad[0] != UINT_MAX) continue;
        const uint32_t size0 = a.ws[j * kWS + kWsSize0], base = (u % chunks) * big::kChunk;
        if (base >= size0) continue;
        for (uint32_t s = base + threadIdx.x; s < base + big::kChunk && s < size0; s += blockDim.x) {
          const BigEntry e = big_entry(a, j, s, size0, stamp);
          hist_add(hsh, e.cand ? key_digit(victim_key(st, e.ver, e.mark, e.freq, e.last, e.rid), 0)
                               : kNoBin);
        }
        __syncthreads();
        big_block_hist_flush(hsh, a.hist + static_cast<uint64_t>(j) * big::kBins);
        __syncthreads();
      }
    } else {
      for (int j = 0; j < n; ++j) {
        const BigState& st = a.st[j];
        if (!st.active || st.pad[0] != UINT_MAX) continue;
        const uint32_t cnt = st.nu[in];
        const uint32_t units = (cnt + big::kChunk - 1) / big::kChunk;
        const u128* K = a.ukey[in] + static_cast<uint64_t>(j) * a.capacity;
        for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
          const uint32_t base = u * big::kChunk;
          for (uint32_t t = base + threadIdx.x; t < base + big::kChunk && t < cnt; t += blockDim.x)
            hist_add(hsh, key_digit(K[t], level));
          __syncthreads();
          big_block_hist_flush(hsh, a.hist + static_cast<uint64_t>(j) * big::kBins);
          __syncthreads();
        }
      }
    }
    grid.sync();
    // the bin of each worker's need-th key
    for (int j = blockIdx.x; j < n; j += gridDim.x) {
      if (!a.st[j].active || a.st[j].pad[0] != UINT_MAX) continue;
      big_select(a, j, scan_sh);
      if (threadIdx.x == 0) {
        BigState& st = a.st[j];
        st.nu[out] = 0;
        if (!st.take_all && level >= (128 + big::kDigit - 1) / big::kDigit - 1) {
          atomicOr(a.flags + kFlagInternal, 1);  // unique keys: unreachable
          st.take_all = 1;
        }
        if (st.take_all) st.pad[0] = level;
      }
    }
    grid.sync();
    // compaction: lower bins are victims, the bin itself is undecided
    // (unless it is taken whole), higher bins drop out
    auto place = [&](const BigState& stc, BigState& st, int j, bool live, u128 key, uint32_t slot,
                     uint32_t ver, bool cur, unsigned mask) {
      const uint32_t d = live ? key_digit(key, level) : 0u;
      const bool victim = live && (d < stc.bin || (d == stc.bin && stc.take_all));
      const bool undecided = live && d == stc.bin && !stc.take_all;
      const uint32_t vi = warp_append(&st.nv, victim, mask);
      if (victim) a.victims[static_cast<uint64_t>(j) * a.capacity + vi] = slot;
      // class counts, one atomic per warp and class (a mass eviction puts
      // ~10^5 victims per worker on these three words)
      const int cls = victim ? (ver ? (cur ? 3 : 2) : (cur ? 1 : 0)) : 3;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const unsigned b = __ballot_sync(mask, cls == c);
        if (b && lane == __ffs(mask) - 1) atomicAdd(&st.vc[c], static_cast<uint32_t>(__popc(b)));
      }
      const uint32_t ui = warp_append(&st.nu[out], undecided, mask);
      if (undecided) {
        a.ukey[out][static_cast<uint64_t>(j) * a.capacity + ui] = key;
        a.uslot[out][static_cast<uint64_t>(j) * a.capacity + ui] = slot;
      }
    };
    if (level == 0) {
      for (uint32_t u = blockIdx.x; u < static_cast<uint32_t>(n) * chunks; u += gridDim.x) {
        const int j = static_cast<int>(u / chunks);
        BigState& st = a.st[j];
        if (!st.active || (st.pad[0] != UINT_MAX && st.pad[0] != level)) continue;
        const BigState stc = st;
        const uint32_t size0 = a.ws[j * kWS + kWsSize0], base = (u % chunks) * big::kChunk;
        if (base >= size0) continue;
        const uint32_t cm = a.cur_mark[j];
        for (uint32_t s0 = base; s0 < base + big::kChunk && s0 < size0; s0 += blockDim.x) {
          const uint32_t s = s0 + threadIdx.x;
          const bool in_range = s < base + big::kChunk && s < size0;
          const unsigned mask = __ballot_sync(0xffffffffu, in_range);
          if (!in_range) continue;
          const BigEntry e = big_entry(a, j, s, size0, stamp);
          const u128 key = e.cand ? victim_key(stc, e.ver, e.mark, e.freq, e.last, e.rid) : u128(0);
          place(stc, st, j, e.cand, key, s, e.ver, e.mark == cm, mask);
        }
      }
    } else {
      for (int j = 0; j < n; ++j) {
        BigState& st = a.st[j];
        if (!st.active || (st.pad[0] != UINT_MAX && st.pad[0] != level)) continue;
        const BigState stc = st;
        const uint32_t cnt = stc.nu[in];
        const uint32_t units = (cnt + big::kChunk - 1) / big::kChunk;
        const uint64_t gb = static_cast<uint64_t>(j) * a.capacity;
        const uint32_t cm = a.cur_mark[j];
        for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
          const uint32_t base = u * big::kChunk;
          for (uint32_t t0 = base; t0 < base + big::kChunk && t0 < cnt; t0 += blockDim.x) {
            const uint32_t t = t0 + threadIdx.x;
            const bool live = t < base + big::kChunk && t < cnt;
            const unsigned mask = __ballot_sync(0xffffffffu, live);
            if (!live) continue;
            const u128 key = a.ukey[in][gb + t];
            const uint32_t slot = a.uslot[in][gb + t];
            const uint32_t ver = static_cast<uint32_t>(key >> 127);
            const bool cur = a.smark[gb + slot] == cm;
            place(stc, st, j, true, key, slot, ver, cur, mask);
          }
        }
      }
    }
    grid.sync();
  }

  // ---- results in the per-worker scalars
  if (gtid < static_cast<uint64_t>(n)) {
    const BigState& st = a.st[gtid];
    uint32_t* w = a.ws + gtid * kWS;
    w[kWsCand] = w[kWsEvict] > 0 ? (st.pinned_err ? st.cand : w[kWsEvict]) : 0u;
    w[kWsCandOff] = static_cast<uint32_t>(gtid * a.capacity);
    w[kWsVa] = st.vc[0];
    w[kWsVb] = st.vc[1];
    w[kWsVc] = st.vc[2];
  }
}

__device__ __forceinline__ int width_of(uint32_t lo, uint32_t hi) {
  return hi > lo ? 32 - __clz(hi - lo) : 0;
}

// Victim selection for caches of up to kSelCap entries: one CTA per worker,
// every entry in registers (kSelItems per thread), no grid-wide sync.  The
// CTA classifies its entries (pinned = stamped by k_classify this
// iteration), reduces the candidates' field ranges, builds each VictimKey
// (cache.hpp:47-58) as a W <= 128-bit MSB-aligned integer (version | mark |
// freq | last | id, fields minus their minima) and radix-selects the E_j-th
// least key 8 bits at a time (keys are unique -- they end in the id); the
// victims are the keys at or below it, written unsorted with the class
// counts k_evict_contrib needs (see k_big_select).  Any key width works.
constexpr int kSelThreads = 1024, kSelItems = 12;
constexpr uint64_t kSelCap = static_cast<uint64_t>(kSelThreads) * kSelItems;

__device__ __forceinline__ uint32_t digit8(u128 k, int done) {
  return static_cast<uint32_t>(k >> (120 - done)) & 0xFFu;
}
__device__ __forceinline__ u128 top_bits(u128 k, int done) {
  return done == 0 ? u128(0) : (k >> (128 - done));
}

__global__ void __launch_bounds__(kSelThreads, 1)
    k_select_victims(uint64_t capacity, uint32_t* __restrict__ ws, const uint32_t* __restrict__ sid,
                     const uint32_t* __restrict__ smark, const uint32_t* __restrict__ sfreq,
                     const uint32_t* __restrict__ slast, const ulonglong2* __restrict__ ol,
                     const uint32_t* __restrict__ slot2id, const uint32_t* __restrict__ pin,
                     const uint32_t* __restrict__ clock_dev, const uint32_t* __restrict__ cur_mark,
                     const uint32_t* __restrict__ ins_scan, uint32_t* __restrict__ victims,
                     int* __restrict__ flags) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ u128 skey[];  // kSelItems * kSelThreads keys, item-major
  __shared__ uint32_t part[kSelThreads / 32][9];
  __shared__ uint32_t tot[9];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_bin, s_rank, s_take, s_nv, s_vc[3];
  const int j = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* w = ws + j * kWS;
  // inserts and evictions of worker j (evict_for, cache.hpp:152-170)
  const uint32_t nb0 = w[kWsNeedOff], ins0 = ins_scan[nb0];
  const uint32_t ins = ins_scan[nb0 + w[kWsNeeds]] - ins0, fr = w[kWsFree];
  const uint32_t E = ins > fr ? ins - fr : 0;
  const uint64_t gb = static_cast<uint64_t>(j) * capacity;
  if (tid == 0) {
    w[kWsInserts] = ins;
    w[kWsInsBase] = ins0;
    w[kWsEvict] = E;
    w[kWsCandOff] = static_cast<uint32_t>(gb);
    w[kWsVa] = w[kWsVb] = w[kWsVc] = 0;
  }
  if (E == 0) {
    if (tid == 0) w[kWsCand] = 0;
    return;
  }
  const uint32_t size0 = w[kWsSize0], stamp = *clock_dev + 1u, cm = cur_mark[j];
  unsigned cfm = 0;  // candidate items of this thread (bit k)
  // an item's (version, mark, freq, last, id); read twice -- for the ranges,
  // then for the keys -- rather than held in registers across the reduction
  auto fields = [&](int k, uint32_t (&fo)[5]) {
    const uint32_t sl = tid * kSelItems + k;
    const uint32_t slot = sid[gb + sl];
    fo[0] = static_cast<uint32_t>((ol[slot].y >> j) & 1ULL);
    fo[1] = smark[gb + sl];
    fo[2] = sfreq[gb + sl];
    fo[3] = slast[gb + sl];
    fo[4] = slot2id ? slot2id[slot] : slot;  // VictimKey's id: the embedding id
  };
  // v[0..3] = min of mark, freq, last, id; v[4..7] = max; v[8] = candidates
  uint32_t v[9] = {UINT_MAX, UINT_MAX, UINT_MAX, UINT_MAX, 0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < kSelItems; ++k) {
    const uint32_t sl = tid * kSelItems + k;
    if (sl < size0 && pin[gb + sl] != stamp) {
      cfm |= 1u << k;
      uint32_t fo[5];
      fields(k, fo);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        v[q] = min(v[q], fo[1 + q]);
        v[4 + q] = max(v[4 + q], fo[1 + q]);
      }
      ++v[8];
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[q] = __reduce_min_sync(0xffffffffu, v[q]);
    v[4 + q] = __reduce_max_sync(0xffffffffu, v[4 + q]);
  }
  v[8] = __reduce_add_sync(0xffffffffu, v[8]);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 9; ++q) part[warp][q] = v[q];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const uint32_t x = part[lane][q];
      tot[q] = q < 4 ? __reduce_min_sync(0xffffffffu, x)
                     : (q < 8 ? __reduce_max_sync(0xffffffffu, x) : __reduce_add_sync(0xffffffffu, x));
    }
  }
  __syncthreads();
  const uint32_t cnt = tot[8];
  if (cnt < E) {  // every remaining entry is pinned (cache.hpp:164)
    if (tid == 0) {
      w[kWsCand] = cnt;
      atomicOr(flags + kFlagPinned, 1);
    }
    return;
  }
  int wd[4], W = 1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    wd[q] = width_of(tot[q], tot[4 + q]);
    W += wd[q];
  }
  if (W > 128) {  // only reachable at ~2^32 epochs
    if (tid == 0) atomicOr(flags + kFlagKeyRange, 1);
    return;
  }
#pragma unroll 4
  for (int k = 0; k < kSelItems; ++k) {
    if (!((cfm >> k) & 1u)) continue;
    uint32_t fo[5];
    fields(k, fo);
    u128 x = fo[0];
#pragma unroll
    for (int q = 0; q < 4; ++q) x = (x << wd[q]) | (fo[1 + q] - tot[q]);
    skey[k * kSelThreads + tid] = x << (128 - W);
  }
  // MSB radix select of the E-th least key, 8 bits per level
  u128 prefix = 0;
  uint32_t rank = E;
  int done = 0;
  bool take_all = false;
  while (!take_all && done < W) {
    for (int x = tid; x < 256; x += kSelThreads) hist[x] = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSelItems; ++k) {
      const u128 key = skey[k * kSelThreads + tid];
      const bool in = ((cfm >> k) & 1u) && top_bits(key, done) == prefix;
      const int bin = in ? static_cast<int>(digit8(key, done)) : -1;
      const unsigned grp = __match_any_sync(0xffffffffu, bin);
      if (in && lane == __ffs(grp) - 1) atomicAdd(&hist[bin], static_cast<uint32_t>(__popc(grp)));
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t h[8], sum = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        h[q] = hist[8 * lane + q];
        sum += h[q];
      }
      uint32_t inc = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
      }
      uint32_t run = inc - sum;
      if (run < rank && rank <= inc) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (run + h[q] >= rank) {
            s_bin = 8 * lane + q;
            s_rank = rank - run;
            s_take = (rank - run == h[q]) ? 1u : 0u;
            break;
          }
          run += h[q];
        }
      }
    }
    __syncthreads();
    prefix = (prefix << 8) | s_bin;
    rank = s_rank;
    take_all = s_take != 0;
    done += 8;
    __syncthreads();
  }
  // victims: keys whose top `done` bits are at or below the prefix
  if (tid == 0) {
    s_nv = 0;
    s_vc[0] = s_vc[1] = s_vc[2] = 0;
  }
  __syncthreads();
  uint32_t vc[3] = {0, 0, 0};
  const int mshift = 128 - 1 - wd[0];  // the mark field's position in a key
#pragma unroll
  for (int k = 0; k < kSelItems; ++k) {
    const u128 key = skey[k * kSelThreads + tid];
    const bool sel = ((cfm >> k) & 1u) && top_bits(key, done) <= prefix;
    const unsigned bal = __ballot_sync(0xffffffffu, sel);
    uint32_t base = 0;
    if (lane == 0 && bal) base = atomicAdd(&s_nv, static_cast<uint32_t>(__popc(bal)));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (sel) {
      victims[gb + base + __popc(bal & ((1u << lane) - 1u))] = tid * kSelItems + k;
      const uint32_t vr = static_cast<uint32_t>(key >> 127);
      const uint32_t mk = wd[0] ? static_cast<uint32_t>(key >> mshift) & ((wd[0] == 32) ? 0xFFFFFFFFu : ((1u << wd[0]) - 1u)) : 0u;
      const bool cur = mk + tot[0] == cm;
      if (vr == 0) ++vc[cur ? 1 : 0];
      else if (!cur) ++vc[2];
    }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    vc[q] = __reduce_add_sync(0xffffffffu, vc[q]);
    if (lane == 0 && vc[q]) atomicAdd(&s_vc[q], vc[q]);
  }
  __syncthreads();
  if (tid == 0) {
    if (s_nv != E) atomicOr(flags + kFlagInternal, 1);  // unique keys: exactly E
    w[kWsCand] = E;
    w[kWsVa] = s_vc[0];
    w[kWsVb] = s_vc[1];
    w[kWsVc] = s_vc[2];
  }
}

// evicting insert contribution: +1 for the insert, -1 if its victim carries
// the current mark (cache.hpp:111,175), evaluated before any advance.
__global__ void k_evict_contrib(const uint64_t* __restrict__ items,
                                const unsigned long long* counters_ro, int n,
                                const uint8_t* __restrict__ type, const uint32_t* __restrict__ ins_scan,
                                const uint32_t* __restrict__ ws, int32_t* __restrict__ contrib) {
  pdl_wait();
  pdl_trigger();
  const uint64_t N = counters_ro[3 * n + 2];
  const uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (q >= N || type[q] != 2) return;
  const int j = item_worker(items[q]);
  const uint32_t* w = ws + j * kWS;
  const uint32_t e = ins_scan[q] - w[kWsInsBase];
  if (e < w[kWsFree]) return;
  const uint32_t t = e - w[kWsFree];
  if (t >= w[kWsCand]) return;  // reported through kFlagPinned
  // the t-th least victim's class (the victims themselves are unsorted)
  const uint32_t a = w[kWsVa], b = a + w[kWsVb], c = b + w[kWsVc];
  const bool cur = (t >= a && t < b) || t >= c;
  contrib[q] = cur ? 0 : 1;
}

// maybe_advance_mark (cache.hpp:187-192) at the first evicting insert whose
// running at_current_mark equals the capacity.
__device__ __forceinline__ void find_advance(uint64_t q, const uint64_t* __restrict__ items,
                                             const unsigned long long* counters_ro, int n,
                                             const uint8_t* __restrict__ type,
                                             const uint32_t* __restrict__ ins_scan,
                                             const int32_t* __restrict__ con_scan, uint32_t* ws,
                                             const unsigned long long* __restrict__ at_cur,
                                             uint64_t capacity) {
  const uint64_t N = counters_ro[3 * n + 2];
  if (q >= N || type[q] != 2) return;
  const int j = item_worker(items[q]);
  uint32_t* w = ws + j * kWS;
  const uint32_t e = ins_scan[q] - w[kWsInsBase];
  if (e < w[kWsFree]) return;
  const uint64_t before =
      at_cur[j] + static_cast<uint64_t>(con_scan[q] - con_scan[w[kWsNeedOff]]);
  if (before == capacity) atomicMin(w + kWsAdvance, static_cast<uint32_t>(q - w[kWsNeedOff]));
}

// evictions: clear the victim's bits of worker j (sim.hpp:177-184)
// (bx, jl) = (block within the worker, evicting worker), kEvictBlocks per worker
constexpr unsigned kEvictBlocks = 8;
__device__ __forceinline__ void evict_victims(unsigned bx, int jl, const int32_t* __restrict__ wlist,
                                              const uint32_t* ws,
                                              const uint32_t* __restrict__ cand_slot,
                                              const uint32_t* __restrict__ sid, uint64_t capacity,
                                              uint64_t id_space, ulonglong2* __restrict__ ol,
                                              unsigned long long* __restrict__ res,
                                              int32_t* __restrict__ slot_of,
                                              uint32_t* __restrict__ victim_id,
                                              unsigned long long* counters, int n) {
  const int j = wlist[jl];
  const uint32_t* w = ws + j * kWS;
  const uint32_t E = min(w[kWsEvict], w[kWsCand]);
  unsigned int pushes = 0;
  for (uint32_t t = bx * blockDim.x + threadIdx.x; t < E; t += kEvictBlocks * blockDim.x) {
    const uint32_t vs = cand_slot[w[kWsCandOff] + t];
    const uint64_t g = static_cast<uint64_t>(j) * capacity + vs;
    const uint32_t id = sid[g];
    victim_id[w[kWsCandOff] + t] = id;
    const unsigned long long bit = 1ULL << j;
    unsigned long long* olw = reinterpret_cast<unsigned long long*>(ol + id);
    const unsigned long long old_owners = atomicAnd(olw, ~bit);
    atomicAnd(olw + 1, ~bit);
    atomicAnd(res + id, ~bit);
    if (old_owners & bit) ++pushes;
    slot_of[static_cast<uint64_t>(j) * id_space + id] = -1;
  }
  for (int o = 16; o > 0; o >>= 1) pushes += __shfl_xor_sync(0xffffffffu, pushes, o);
  if ((threadIdx.x & 31) == 0 && pushes) atomicAdd(counters + 2 * n + j, static_cast<unsigned long long>(pushes));
}

// The epoch-advance search (blocks [0, ga)) and the evictions (kEvictBlocks
// blocks per evicting worker after them) are independent: one launch.
__global__ void k_advance_evict(uint32_t ga, const uint64_t* __restrict__ items,
                                const unsigned long long* counters_ro, int n,
                                const uint8_t* __restrict__ type,
                                const uint32_t* __restrict__ ins_scan,
                                const int32_t* __restrict__ con_scan, uint32_t* ws,
                                const unsigned long long* __restrict__ at_cur, uint64_t capacity,
                                const int32_t* __restrict__ wlist,
                                const uint32_t* __restrict__ cand_slot,
                                const uint32_t* __restrict__ sid, uint64_t id_space,
                                ulonglong2* __restrict__ ol, unsigned long long* __restrict__ res,
                                int32_t* __restrict__ slot_of, uint32_t* __restrict__ victim_id,
                                unsigned long long* counters) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x < ga) {
    find_advance(blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x, items, counters_ro, n,
                 type, ins_scan, con_scan, ws, at_cur, capacity);
  } else {
    const unsigned b = blockIdx.x - ga;
    evict_victims(b % kEvictBlocks, static_cast<int>(b / kEvictBlocks), wlist, ws, cand_slot, sid,
                  capacity, id_space, ol, res, slot_of, victim_id, counters, n);
  }
}

// touches and inserts (WorkerCache::touch, cache.hpp:102-122; sim.hpp:172,186-188)
__global__ void k_apply(const uint64_t* __restrict__ items,
                        const unsigned long long* counters_ro, int n,
                        const uint32_t* __restrict__ ids, const uint8_t* __restrict__ type,
                        const uint32_t* __restrict__ ins_scan, const uint32_t* __restrict__ ws,
                        const uint32_t* __restrict__ cand_slot, uint64_t capacity,
                        uint64_t id_space, const uint32_t* __restrict__ cur_mark,
                        const uint32_t* __restrict__ clock_dev,
                        ulonglong2* __restrict__ ol, unsigned long long* __restrict__ res,
                        int32_t* __restrict__ slot_of, uint32_t* __restrict__ sid,
                        uint32_t* __restrict__ smark, uint32_t* __restrict__ sfreq,
                        uint32_t* __restrict__ slast, const int32_t* __restrict__ item_slot) {
  pdl_wait();
  pdl_trigger();
  const uint32_t clock = *clock_dev;
  const uint64_t N = counters_ro[3 * n + 2];
  const uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (q >= N) return;
  const uint64_t key = items[q];
  const int j = item_worker(key);
  const uint32_t id = ids[item_pos(key)];
  const uint32_t* w = ws + j * kWS;
  const uint32_t local = static_cast<uint32_t>(q) - w[kWsNeedOff];
  const uint32_t mark = cur_mark[j] + (local >= w[kWsAdvance] ? 1u : 0u);
  const unsigned long long bit = 1ULL << j;
  const uint8_t t = type[q];
  if (t != 2) {
    const uint64_t g = static_cast<uint64_t>(j) * capacity + item_slot[q];
    smark[g] = mark;
    sfreq[g] += 1;
    slast[g] = clock;
    if (t == 1) atomicOr(reinterpret_cast<unsigned long long*>(ol + id) + 1, bit);
    return;
  }
  const uint32_t e = ins_scan[q] - w[kWsInsBase];
  uint32_t slot;
  if (e < w[kWsFree]) slot = w[kWsSize0] + e;
  else slot = cand_slot[w[kWsCandOff] + (e - w[kWsFree])];
  const uint64_t g = static_cast<uint64_t>(j) * capacity + slot;
  slot_of[static_cast<uint64_t>(j) * id_space + id] = static_cast<int32_t>(slot);
  sid[g] = id;
  smark[g] = mark;
  sfreq[g] = 1;
  slast[g] = clock;
  atomicOr(reinterpret_cast<unsigned long long*>(ol + id) + 1, bit);
  atomicOr(res + id, bit);
}

// Tail of the step: per-worker sizes and epoch state (block 0), phase 3
// ownership hand-over (sim.hpp:192-204), and the reset of the per-id tables
// for the next step.
__global__ void k_step_tail(int n, const uint32_t* __restrict__ ws,
                            const int32_t* __restrict__ con_scan, uint32_t* __restrict__ size,
                            uint32_t* __restrict__ cur_mark, unsigned long long* __restrict__ at_cur,
                            const uint32_t* __restrict__ uniq,
                            const unsigned long long* counters_ro, ulonglong2* __restrict__ ol,
                            int32_t* __restrict__ first_pos, unsigned long long* __restrict__ umask) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x < n) {
    const int j = threadIdx.x;
    const uint32_t* w = ws + j * kWS;
    const uint32_t E = min(w[kWsEvict], w[kWsCand]);
    size[j] = w[kWsSize0] + w[kWsInserts] - E;
    const uint32_t b = w[kWsNeedOff], cnt = w[kWsNeeds];
    if (w[kWsAdvance] != UINT_MAX) {
      cur_mark[j] += 1;
      at_cur[j] = cnt - w[kWsAdvance];
    } else {
      at_cur[j] += static_cast<unsigned long long>(con_scan[b + cnt] - con_scan[b]);
    }
  }
  const uint64_t U = counters_ro[3 * n + 1];
  const uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (u >= U) return;
  const unsigned long long m = umask[u];
  const uint32_t id = uniq[u];
  ol[id] = make_ulonglong2(m, m);
  first_pos[id] = INT_MAX;
  umask[u] = 0;
}

// Clears the per-id tables of a batch whose step head ran but whose step
// never did (the iteration failed in between).
__global__ void k_reset_unique(const uint32_t* __restrict__ uniq,
                               const unsigned long long* counters_ro, int n,
                               int32_t* __restrict__ first_pos) {
  const uint64_t U = counters_ro[3 * n + 1];
  const uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (u >= U) return;
  first_pos[uniq[u]] = INT_MAX;
}

__global__ void k_fill_i32(int32_t* p, uint64_t n, int32_t v) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x < n) p[x] = v;
}

// Caches of <= kSelCap entries select in one CTA per worker (k_select_victims);
// larger ones with the cooperative grid kernel (k_big_select).
bool use_cta_select(const edx_engine* e) { return e->capacity <= kSelCap; }

}  // namespace

void step_init_state(edx_engine* e) {
  const uint64_t n = static_cast<uint64_t>(e->n);
  auto& c = e->cache;
  c.slot_of.ensure(n * e->id_space);
  c.sid.ensure(n * e->capacity);
  c.smark.ensure(n * e->capacity);
  c.sfreq.ensure(n * e->capacity);
  c.slast.ensure(n * e->capacity);
  c.size.ensure(n);
  c.cur_mark.ensure(n);
  c.at_cur.ensure(n);
  const uint64_t cells = n * e->id_space;
  k_fill_i32<<<grid_for(cells), kT, 0, e->stream>>>(c.slot_of.p, cells, -1);
  EDX_LAUNCHED();
  EDX_CUDA(cudaMemsetAsync(c.size.p, 0, n * sizeof(uint32_t), e->stream));
  std::vector<uint32_t> ones(n, 1u);  // current_mark_ starts at 1 (cache.hpp:236)
  EDX_CUDA(cudaMemcpyAsync(c.cur_mark.p, ones.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                           e->stream));
  EDX_CUDA(cudaMemsetAsync(c.at_cur.p, 0, n * sizeof(unsigned long long), e->stream));

  auto& s = e->step;
  const uint64_t T = e->max_ids;
  s.occ_sample.ensure(T);
  s.first_pos.ensure(e->id_space);
  k_fill_i32<<<grid_for(e->id_space), kT, 0, e->stream>>>(s.first_pos.p, e->id_space, INT_MAX);
  EDX_LAUNCHED();
  s.uidx_of_pos.ensure(T + 1);
  s.upos.ensure(T);
  s.item_slot.ensure(T);
  s.uniq.ensure(T);
  s.umask.ensure(T);
  EDX_CUDA(cudaMemsetAsync(s.umask.p, 0, T * sizeof(unsigned long long), e->stream));
  // epoch-tagged need cells (k_needs): all-zero = no step
  s.need_first.ensure(n * T);
  EDX_CUDA(cudaMemsetAsync(s.need_first.p, 0, n * T * sizeof(unsigned long long), e->stream));
  s.need_cnt.ensure(n * T);
  EDX_CUDA(cudaMemsetAsync(s.need_cnt.p, 0, n * T * sizeof(unsigned long long), e->stream));
  s.epoch.ensure(1);
  EDX_CUDA(cudaMemsetAsync(s.epoch.p, 0, sizeof(uint32_t), e->stream));
  s.flag_scan.ensure(T + 1);
  s.need_key.ensure(T);
  s.need_key_sorted.ensure(T);
  s.need_type.ensure(T + 1);
  s.need_contrib.ensure(T + 1);
  s.ins_rank.ensure(T + 1);
  s.counters.ensure(3 * n + 4);
  s.wscalars.ensure(n * kWS);
  // victims of every worker (a worker with no evictions skips its share)
  const uint64_t cand = n * e->capacity;
  s.cand_slot_sorted.ensure(cand);
  s.cand_count.ensure(cand);  // the victim-id list
  // pin stamps per entry (k_classify marks this iteration's working set)
  c.pin.ensure(cand);
  EDX_CUDA(cudaMemsetAsync(c.pin.p, 0, cand * sizeof(uint32_t), e->stream));
  if (use_cta_select(e)) {
    EDX_CUDA(cudaFuncSetAttribute(k_select_victims, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSelItems * kSelThreads * sizeof(u128))));
  } else {  // the cooperative selection's scratch
    s.big_state.ensure(n * sizeof(BigState));
    s.big_hist.ensure(n * big::kBins);
    for (int b = 0; b < 2; ++b) {
      s.big_key[b].ensure(cand * sizeof(u128));
      s.big_slot[b].ensure(cand);
    }
    s.big_eflag.ensure(cand);
    int per_sm = 0, sms = 0;
    EDX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_big_select, big::kThreads, 0));
    EDX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, e->device));
    if (per_sm < 1) throw Error(EDX_CUDA_ERROR, "victim selection kernel cannot be resident");
    // enough CTAs for the work units, one per SM and two SMs' worth of room:
    // a cooperative grid starts only when all its CTAs are resident, and the
    // step runs beside decision_cost (a 1024-thread CTA on the side stream)
    const uint64_t units = n * ((e->capacity + big::kChunk - 1) / big::kChunk);
    s.big_grid = std::max<uint64_t>(1, std::min<uint64_t>(units, sms > 2 ? sms - 2 : 1));
  }
  s.cand_off.ensure(128);  // [0,64): workers 0..n-1; [64,128): evicting workers (large caches)
  std::vector<int32_t> wl(n);
  for (uint64_t j = 0; j < n; ++j) wl[j] = static_cast<int32_t>(j);
  EDX_CUDA(cudaMemcpyAsync(s.cand_off.p, wl.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice,
                           e->stream));
  EDX_CUDA(cudaStreamSynchronize(e->stream));
}

namespace {

template <class F>
void cub_call(edx_engine* e, F&& f) {
  size_t bytes = 0;
  EDX_CUDA(f(static_cast<void*>(nullptr), bytes));
  e->step.temp.ensure(bytes);
  bytes = e->step.temp.n;
  EDX_CUDA(f(static_cast<void*>(e->step.temp.p), bytes));
}

}  // namespace

bool step_device_only(const edx_engine*) { return true; }

namespace {

// The decision-independent head of the step on stream `st`: the iteration
// clock, zeroed counters, the sample of every id position, and the unique ids
// of the batch in first-occurrence order.  Returns the kernels launched.
int launch_step_head(edx_engine* e, cudaStream_t st) {
  auto& s = e->step;
  const int n = e->n;
  const uint64_t T = e->total_ids, R = e->rows;
  // the clock goes through pinned memory so a captured graph reads each
  // iteration's value at replay time
  *e->h_clock = static_cast<uint32_t>(e->clock);
  EDX_CUDA(cudaMemcpyAsync(e->d_clock.p, e->h_clock, sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  const uint32_t ncnt = static_cast<uint32_t>(3 * n + 4), nws = static_cast<uint32_t>(n * kWS);
  const uint64_t span = std::max<uint64_t>(std::max<uint64_t>(R, T), nws);
  k_step_begin<<<grid_for(span), kT, 0, st>>>(e->cur_offsets, R, s.occ_sample.p, e->cur_ids, T,
                                              s.first_pos.p, s.counters.p, ncnt, s.wscalars.p, nws,
                                              s.epoch.p);
  launch_pdl(k_unique_flag, grid_for(T + 1), kT, 0, st, e->cur_ids, T, s.first_pos.p, s.flag_scan.p);
  EDX_LAUNCHED();
  cub_call(e, [&](void* tmp, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(tmp, b, s.flag_scan.p, s.uidx_of_pos.p,
                                         static_cast<int>(T + 1), st);
  });
  launch_pdl(k_unique_scatter, grid_for(T + 1), kT, 0, st, e->cur_ids, T, s.first_pos.p, s.uidx_of_pos.p,
                                                   s.uniq.p, s.counters.p, n);
  launch_pdl(k_unique_of_pos, grid_for(T), kT, 0, st, e->cur_ids, T, s.first_pos.p,
             s.uidx_of_pos.p, s.upos.p);
  EDX_LAUNCHED();
  return 6;
}

}  // namespace

void step_head(edx_engine* e) {
  if (e->head_pending) return;
  EDX_CUDA(cudaEventRecord(e->head_fork, e->stream));
  EDX_CUDA(cudaStreamWaitEvent(e->step_side, e->head_fork, 0));
  e->launches += launch_step_head(e, e->step_side);
  EDX_CUDA(cudaEventRecord(e->head_done, e->step_side));
  e->head_pending = true;
}

void step_head_abandon(edx_engine* e) {
  if (!e->head_pending) return;
  e->head_pending = false;
  if (e->capturing) return;  // the captured head never ran
  EDX_CUDA(cudaStreamWaitEvent(e->stream, e->head_done, 0));
  k_reset_unique<<<grid_for(e->total_ids), kT, 0, e->stream>>>(e->step.uniq.p, e->step.counters.p,
                                                               e->n, e->step.first_pos.p);
  EDX_LAUNCHED();
}

void step_run(edx_engine* e, const int32_t* d_decision, StepResult* out) {
  cudaStream_t st = e->stream;
  auto& s = e->step;
  auto& c = e->cache;
  const int n = e->n;
  const uint64_t T = e->total_ids, ucap = e->max_ids;
  int launches = 0;
  if (e->head_pending) {  // launched by the fused iteration, overlapping the dispatch
    EDX_CUDA(cudaStreamWaitEvent(st, e->head_done, 0));
    e->head_pending = false;
  } else {
    launches += launch_step_head(e, st);
  }
  k_needs<<<grid_for(T), kT, 0, st>>>(T, s.occ_sample.p, d_decision, s.upos.p, ucap,
                                      s.need_first.p, s.need_cnt.p, s.umask.p, s.epoch.p);
  launch_pdl(k_need_keys, grid_for(T), kT, 0, st, T, s.occ_sample.p, d_decision, s.upos.p, ucap,
             s.need_first.p, s.need_key.p, s.wscalars.p, s.epoch.p);
  EDX_LAUNCHED();
  launches += 2;
  int wbits = 1;
  while ((1 << wbits) < n) ++wbits;
  cub_call(e, [&](void* tmp, size_t& b) {
    // items arrive in position order and the sort is stable: sorting on the
    // worker field alone leaves each worker's items in first-occurrence order
    return cub::DeviceRadixSort::SortKeys(tmp, b, s.need_key.p, s.need_key_sorted.p,
                                          static_cast<int>(T), 32, 32 + wbits + 1, st);
  });
  launches += 3;
  launch_pdl(k_phase1, grid_for(T), kT, 0, st, s.uniq.p, s.umask.p, s.counters.p, n, e->ol.p, s.counters.p,
                                       s.wscalars.p, c.size.p, e->capacity);
  launch_pdl(k_classify, grid_for(T + 1), kT, 0, st, 
      s.need_key_sorted.p, s.counters.p, n, e->cur_ids, s.upos.p, ucap,
      s.need_cnt.p, e->ol.p, e->res.p, e->id_space, c.slot_of.p, e->capacity, c.smark.p,
      c.cur_mark.p, s.need_type.p, s.flag_scan.p, s.need_contrib.p, s.counters.p,
      c.pin.p, e->d_clock.p, s.item_slot.p);
  EDX_LAUNCHED();
  launches += 2;
  // insert ordinals: exclusive scan over the (worker-grouped) need items
  cub_call(e, [&](void* tmp, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(tmp, b, s.flag_scan.p, s.ins_rank.p,
                                         static_cast<int>(T + 1), st);
  });
  launches += 2;
  if (!use_cta_select(e)) {
    k_worker_inserts<<<1, 64, 0, st>>>(n, s.ins_rank.p, s.wscalars.p, e->flags.p);
    EDX_LAUNCHED();
    launches += 1;
  }

  // Victim selection (evict_for, cache.hpp:152-170), every worker at once;
  // workers without evictions drop out on the device.
  const int32_t* d_wlist = reinterpret_cast<const int32_t*>(s.cand_off.p);
  int nw = n;  // workers the victim kernels visit
  if (use_cta_select(e)) {
    launch_pdl(k_select_victims, n, kSelThreads, kSelItems * kSelThreads * sizeof(u128), st,
               e->capacity, s.wscalars.p, c.sid.p,
               c.smark.p, c.sfreq.p, c.slast.p, e->ol.p, e->hashed ? e->idt.slot2id.p : nullptr,
               c.pin.p, e->d_clock.p, c.cur_mark.p, s.ins_rank.p, s.cand_slot_sorted.p,
               e->flags.p);
    EDX_LAUNCHED();
    launches += 1;
  } else {
    // One cooperative kernel selects every evicting worker's victims on the
    // device (k_big_select); no host round trip, any key width.
    BigArgs ba;
    ba.n = n;
    ba.capacity = e->capacity;
    ba.ws = s.wscalars.p;
    ba.sid = c.sid.p;
    ba.smark = c.smark.p;
    ba.sfreq = c.sfreq.p;
    ba.slast = c.slast.p;
    ba.pin = c.pin.p;
    ba.ol = e->ol.p;
    ba.slot2id = e->hashed ? e->idt.slot2id.p : nullptr;
    ba.cur_mark = c.cur_mark.p;
    ba.clock_dev = e->d_clock.p;
    ba.st = reinterpret_cast<BigState*>(s.big_state.p);
    ba.hist = s.big_hist.p;
    ba.ukey[0] = reinterpret_cast<u128*>(s.big_key[0].p);
    ba.ukey[1] = reinterpret_cast<u128*>(s.big_key[1].p);
    ba.uslot[0] = s.big_slot[0].p;
    ba.uslot[1] = s.big_slot[1].p;
    ba.victims = s.cand_slot_sorted.p;
    ba.eflag = s.big_eflag.p;
    ba.flags = e->flags.p;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(s.big_grid));
    cfg.blockDim = dim3(big::kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    EDX_CUDA(cudaLaunchKernelEx(&cfg, k_big_select, ba));
    launches += 1;
  }
  launch_pdl(k_evict_contrib, grid_for(T), kT, 0, st, s.need_key_sorted.p, s.counters.p, n,
             s.need_type.p, s.ins_rank.p, s.wscalars.p, s.need_contrib.p);
  EDX_LAUNCHED();
  cub_call(e, [&](void* tmp, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(tmp, b, s.need_contrib.p,
                                         reinterpret_cast<int32_t*>(s.flag_scan.p),
                                         static_cast<int>(T + 1), st);
  });
  const int32_t* con_scan = reinterpret_cast<const int32_t*>(s.flag_scan.p);
  {
    const unsigned ga = grid_for(T);
    const int32_t* wlv = d_wlist;
    launch_pdl(k_advance_evict, ga + kEvictBlocks * static_cast<unsigned>(nw), kT, 0, st, 
        ga, s.need_key_sorted.p, s.counters.p, n, s.need_type.p, s.ins_rank.p, con_scan,
        s.wscalars.p, c.at_cur.p, e->capacity, wlv, s.cand_slot_sorted.p, c.sid.p, e->id_space,
        e->ol.p, e->res.p, c.slot_of.p, s.cand_count.p, s.counters.p);
  }
  EDX_LAUNCHED();
  launches += 3;  // contribution, scan (2), advance + evict
  launch_pdl(k_apply, grid_for(T), kT, 0, st, s.need_key_sorted.p, s.counters.p, n, e->cur_ids,
                                      s.need_type.p, s.ins_rank.p, s.wscalars.p,
                                      s.cand_slot_sorted.p, e->capacity, e->id_space, c.cur_mark.p,
                                      e->d_clock.p, e->ol.p, e->res.p, c.slot_of.p, c.sid.p,
                                      c.smark.p, c.sfreq.p, c.slast.p, s.item_slot.p);
  launch_pdl(k_step_tail, grid_for(T), kT, 0, st, n, s.wscalars.p, con_scan, c.size.p, c.cur_mark.p,
                                          c.at_cur.p, s.uniq.p, s.counters.p, e->ol.p,
                                          s.first_pos.p, s.umask.p);
  EDX_LAUNCHED();
  launches += 2;
  EDX_CUDA(cudaMemcpyAsync(e->h_counters, s.counters.p, (3 * n + 4) * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
  out->launches = launches;
  out->evicting_workers = -1;  // decided on the device
}

}  // namespace edx
