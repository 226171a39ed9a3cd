// K3 row ordering, K4 capacity-bounded greedy, decision checks, and the
// EcoMix orchestration (assign.hpp:162-298).
#include <cub/device/device_merge_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "edx_internal.cuh"

namespace edx {

// ------------------------------------------------------------------ K3 sort
// rows_by_gap (assign.hpp:197-207) orders rows by (gap desc, index asc).  The
// gap keys are ~bits(gap) (cost.cu), so an ascending *stable* sort of
// (key, row) pairs with rows fed in index order reproduces std::sort with the
// reference's total order exactly.  A stable merge sort: the 64-bit keys cost
// a radix sort eight onesweep passes (C3: 0.100 -> 0.049 ms, C5 0.119 -> 0.095).
namespace {
struct KeyLess {
  __device__ bool operator()(uint64_t a, uint64_t b) const { return a < b; }
};
}  // namespace

void sort_rows_by_gap(SortScratch& sc, const uint64_t* keys_in, const uint32_t* idx_in,
                      uint32_t* idx_out, uint64_t rows, cudaStream_t s) {
  sc.keys_out.ensure(rows);
  EDX_CUDA(cudaMemcpyAsync(sc.keys_out.p, keys_in, rows * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                           s));
  EDX_CUDA(cudaMemcpyAsync(idx_out, idx_in, rows * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  size_t bytes = 0;
  EDX_CUDA(cub::DeviceMergeSort::StableSortPairs(nullptr, bytes, sc.keys_out.p, idx_out,
                                                 static_cast<int64_t>(rows), KeyLess{}, s));
  sc.temp.ensure(bytes);
  EDX_CUDA(cub::DeviceMergeSort::StableSortPairs(sc.temp.p, bytes, sc.keys_out.p, idx_out,
                                                 static_cast<int64_t>(rows), KeyLess{}, s));
}

// ---------------------------------------------------------------- K4 greedy
// greedy_dispatch (assign.hpp:162-192) is sequential: each row, in order,
// takes its cheapest worker with capacity left (strict '<', lowest index on
// ties).  The open set only changes when a worker is exhausted, so the
// sequential result equals rounds of "every pending row takes its argmin over
// the current open set": positions before the first row whose choice exceeds
// that worker's remaining capacity are final, then the exhausted workers
// close and the next round starts at that row.  Rows after an exhaustion that
// did not pick the exhausted worker keep their argmin (removing a worker that
// is not the minimum does not move the minimum), so the first over-capacity
// row is the first divergence.  Each cut closes >= 1 worker: <= n cut rounds
// plus one round per 1024 rows.  (A grid-wide version -- one cooperative CTA
// per tile of 1024 rows, one grid-wide sync per round -- measured slower at
// every config: C5 greedy 0.60 -> 1.03 ms, ~15 us per grid-wide round.)
namespace {


// Each position's whole preference list: its initially open workers in
// (cost, index) order -- the order in which the reference's scan
// (assign.hpp:177-184: ascending j, strict '<') would pick them as workers
// close -- one byte each, 0xFF past the last.  One warp per position, a
// 64-element bitonic sort in registers (two elements per lane).  The greedy
// then takes the first still-open entry: no rescan of the row's costs.
constexpr int kListBytes = 64;

__device__ __forceinline__ bool pref_less(double ca, int ia, double cb, int ib) {
  return ca < cb || (!(cb < ca) && ia < ib);
}

__global__ void k_greedy_prefs(const double* __restrict__ matrix, int n,
                               const uint32_t* __restrict__ order, uint64_t n_order,
                               const int32_t* __restrict__ capacity_dev, int cap_uniform,
                               const uint32_t* __restrict__ row_ids, uint8_t* __restrict__ prefs,
                               uint32_t* __restrict__ dest) {
  const uint64_t t = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n_order) return;  // warp-uniform
  const uint32_t row = order[t];
  if (lane == 0) dest[t] = row_ids ? row_ids[row] : row;
  const double* r = matrix + static_cast<uint64_t>(row) * n;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double c[2];
  int id[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int w = h * 32 + lane;
    const bool open = w < n && (capacity_dev ? capacity_dev[w] : cap_uniform) > 0;
    c[h] = open ? r[w] : inf;
    id[h] = open ? w : 0xFF;
  }
  // bitonic sort of element e = h * 32 + lane, ascending by (cost, index)
#pragma unroll
  for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
    for (int d = size >> 1; d > 0; d >>= 1) {
      if (d == 32) {
        const bool asc = (lane & size) == 0;  // size == 64: always ascending
        const bool gt = pref_less(c[1], id[1], c[0], id[0]);
        if (gt == asc) {
          const double tc = c[0];
          const int ti = id[0];
          c[0] = c[1];
          id[0] = id[1];
          c[1] = tc;
          id[1] = ti;
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double oc = __shfl_xor_sync(0xffffffffu, c[h], d);
          const int oi = __shfl_xor_sync(0xffffffffu, id[h], d);
          const bool asc = ((h * 32 + lane) & size) == 0;
          const bool lower = (lane & d) == 0;
          const bool other_less = pref_less(oc, oi, c[h], id[h]);
          if ((lower == asc) ? other_less : !other_less) {
            c[h] = oc;
            id[h] = oi;
          }
        }
      }
    }
  }
  uint8_t* out = prefs + t * kListBytes;
  out[lane] = static_cast<uint8_t>(id[0]);
  out[32 + lane] = static_cast<uint8_t>(id[1]);
}

constexpr int kGreedyThreads = 1024;
constexpr int kGreedyWarps = kGreedyThreads / 32;
constexpr int kGreedySlots = 3;  // staged chunks of kGreedyThreads positions
constexpr size_t kGreedySmem = static_cast<size_t>(kGreedySlots) * kGreedyThreads * kListBytes;

// One CTA walks the positions in windows of 1024 (one thread per position),
// each window in rounds of three barriers until all of it is committed.  Per
// window and worker, lanes[warp][w] holds which lanes of the warp chose w and
// total[w] how many pending positions did; positions below q0 are committed.
//  A  the window's first round: every position takes the first open worker
//     of its preference list; the lanes of a warp that chose the same worker
//     (six ballots over its bits) are recorded by their leader.  Later
//     rounds: only a pending position whose worker closed takes its next open
//     worker (closing a worker that is not a position's minimum does not move
//     it) and moves its bit between the two workers' masks.
//  B  a worker whose pending total reaches its remaining capacity r cuts the
//     round at its r-th pending occurrence (0-based): one warp scans the
//     per-warp pending counts, the crossing warp's mask gives the lane (fns);
//     the earliest cut wins;
//  C  pending positions before the cut commit; each worker takes their count
//     (a warp reduction over the masks) off its capacity and closes at zero;
//     a round without a cut ends the window.
// Windows' preference lists are staged in shared memory by 1D bulk copies
// (TMA) three deep, so a round reads no global memory; choices are written in
// position order (coalesced) and scattered to the decision by k_greedy_scatter.
__device__ __forceinline__ unsigned lanes_from(int lo) {  // lanes >= lo of a warp
  return lo <= 0 ? 0xffffffffu : (lo >= 32 ? 0u : (0xffffffffu << lo));
}

__global__ void __launch_bounds__(kGreedyThreads)
    k_greedy(int n, uint64_t n_order, const int32_t* __restrict__ capacity_dev, int cap_uniform,
             int32_t* __restrict__ pair_worker, int* __restrict__ flags,
             const uint8_t* __restrict__ prefs, unsigned long long* __restrict__ stats) {
  extern __shared__ __align__(128) uint8_t gsm[];
  uint8_t* const plist = gsm;  // [slot][position][kListBytes]
  __shared__ int remaining[kMaxWorkers];
  __shared__ int total[kMaxWorkers];
  __shared__ unsigned lanes[kGreedyWarps][kMaxWorkers + 1];
  __shared__ unsigned long long open_mask;
  __shared__ int qmin[2];
  __shared__ __align__(8) uint64_t bars[kGreedySlots];
  // stats (EDX_GREEDY_STATS=1), kept by thread 0: [0] rounds [1] top barrier
  // [2] A until thread 0's scan is done [3] A barrier [4] B [5] C (thread 0)
  // [6] total [7] last lap
  __shared__ unsigned long long st[8];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t nch = (n_order + kGreedyThreads - 1) / kGreedyThreads;
  auto stage = [&](uint64_t c) {  // thread 0: window c -> slot c % kGreedySlots
    const int sl = static_cast<int>(c % kGreedySlots);
    const uint64_t p0 = c * kGreedyThreads;
    const uint64_t cntp = n_order - p0 < kGreedyThreads ? n_order - p0 : kGreedyThreads;
    const unsigned lb = static_cast<unsigned>(cntp * kListBytes);
    mbar_expect_tx(&bars[sl], lb);
    bulk_g2s(plist + static_cast<size_t>(sl) * kGreedyThreads * kListBytes, prefs + p0 * kListBytes,
             lb, &bars[sl]);
  };
  if (tid < n) {
    remaining[tid] = capacity_dev ? capacity_dev[tid] : cap_uniform;
    total[tid] = 0;
  }
  for (int x = tid; x < kGreedyWarps * (kMaxWorkers + 1); x += kGreedyThreads) (&lanes[0][0])[x] = 0;
  if (tid == 0) {
    qmin[0] = qmin[1] = kGreedyThreads;
    for (int q = 0; q < kGreedySlots; ++q) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint64_t c = 0; c < nch && c < kGreedySlots; ++c) stage(c);
    if (stats) {
      for (int q = 0; q < 7; ++q) st[q] = 0;
      st[7] = clock64();
      st[6] = st[7];
    }
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long om = 0;
    for (int w = 0; w < n; ++w)
      if (remaining[w] > 0) om |= 1ULL << w;
    open_mask = om;
  }
  auto lap = [&](int slot) {
    if (stats && tid == 0) {
      const unsigned long long now = clock64();
      st[slot] += now - st[7];
      st[7] = now;
    }
  };

  unsigned round = 0;
  for (uint64_t c = 0; c < nch; ++c) {
    const int sl = static_cast<int>(c % kGreedySlots);
    const uint64_t t = c * kGreedyThreads + tid;
    const bool valid = t < n_order;
    mbar_wait(&bars[sl], static_cast<unsigned>((c / kGreedySlots) & 1));
    const size_t off = static_cast<size_t>(sl) * kGreedyThreads + tid;
    const uint4* lst = reinterpret_cast<const uint4*>(plist + off * kListBytes);
    int choice = -1;
    int q0 = 0;  // positions of the window before q0 are committed
    for (bool first = true;; first = false, ++round) {
      __syncthreads();  // open_mask, totals and masks are current; qmin reads are done
      if (tid == 0) qmin[(round + 1) & 1] = kGreedyThreads;  // the next round's cut
      lap(1);
      // ---- A
      const bool pending = valid && tid >= q0;
      const unsigned long long om = open_mask;
      const int old = choice;
      // (a position left without a worker -- the error case -- stays so)
      if (pending && (first || (choice >= 0 && !((om >> choice) & 1ULL)))) {
        // the first still-open worker of the position's preference list is
        // its argmin over the open set: every worker ranked before it is closed
        choice = -1;
        const int nv = (n + 15) >> 4;
        for (int q = 0; q < nv; ++q) {
          const uint4 v4 = lst[q];
          const uint32_t wd[4] = {v4.x, v4.y, v4.z, v4.w};
          bool stop = false;
#pragma unroll
          for (int b = 0; b < 16; ++b) {
            const int w = static_cast<int>((wd[b >> 2] >> (8 * (b & 3))) & 0xFFu);
            if (w == 0xFF) {  // past the last initially open worker
              stop = true;
              break;
            }
            if ((om >> w) & 1ULL) {
              choice = w;
              stop = true;
              break;
            }
          }
          if (stop) break;
        }
        if (choice < 0) atomicOr(flags + kFlagUnbalanced, 1);  // "capacities exhausted"
        if (!first) {  // move this lane's bit to its new worker
          if (stats) atomicAdd(stats + 8, 1ULL);
          atomicAnd(&lanes[warp][old], ~(1u << lane));
          atomicSub(&total[old], 1);
          if (choice >= 0) {
            atomicOr(&lanes[warp][choice], 1u << lane);
            atomicAdd(&total[choice], 1);
          }
        }
      }
      lap(2);
      if (first) {
        const int key = valid ? choice : -1;
        // lanes with the same worker: six ballots over its bits
        unsigned peers = __ballot_sync(0xffffffffu, key >= 0);
#pragma unroll
        for (int bit = 0; bit < 6; ++bit) {
          const unsigned bm = __ballot_sync(0xffffffffu, (key >> bit) & 1);
          peers &= ((key >> bit) & 1) ? bm : ~bm;
        }
        if (key >= 0 && lane == __ffs(peers) - 1) {
          lanes[warp][key] = peers;
          atomicAdd(&total[key], __popc(peers));
        }
      }
      __syncthreads();
      lap(3);
      if (stats && tid == 0) ++st[0];

      // ---- B: cuts of the workers the round would overfill (pending lanes:
      // positions >= q0 of the window)
      const int qw = q0 >> 5, ql = q0 & 31;
      const unsigned pend = lane < qw ? 0u : (lane == qw ? lanes_from(ql) : 0xffffffffu);
#pragma unroll
      for (int h = 0; h < kMaxWorkers / kGreedyWarps; ++h) {
        const int w = warp + h * kGreedyWarps;
        if (w < n && total[w] > 0 && total[w] >= remaining[w]) {  // warp-uniform
          const int k = remaining[w];  // >= 1: only open workers are chosen
          const unsigned m = lanes[lane][w] & pend;
          const int v = __popc(m);
          int inc = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
          }
          const unsigned cross = __ballot_sync(0xffffffffu, inc - v <= k && k < inc);
          if (lane == __ffs(cross) - 1)  // the (k - excl)-th (0-based) pending lane of this warp
            atomicMin(&qmin[round & 1], lane * 32 + static_cast<int>(__fns(m, 0, k - (inc - v) + 1)));
        }
      }
      __syncthreads();
      lap(4);

      // ---- C
      const int limit = qmin[round & 1];
      // in position order (coalesced); the scatter to rows is a separate grid
      if (pending && choice >= 0 && tid < limit) pair_worker[t] = choice;
      // capacities: a worker's pending positions before the cut
      const int lw = limit >> 5, ll = limit & 31;
      const unsigned upto = lane < lw ? 0xffffffffu : (lane == lw ? ~lanes_from(ll) : 0u);
#pragma unroll
      for (int h = 0; h < kMaxWorkers / kGreedyWarps; ++h) {
        const int w = warp + h * kGreedyWarps;
        if (w < n && total[w] > 0) {  // warp-uniform
          int used = total[w];
          if (limit < kGreedyThreads)
            used = static_cast<int>(
                __reduce_add_sync(0xffffffffu, static_cast<unsigned>(__popc(lanes[lane][w] & pend & upto))));
          if (lane == 0 && used > 0) {
            total[w] -= used;
            const int rem = remaining[w] - used;
            remaining[w] = rem;
            if (rem <= 0) atomicAnd(&open_mask, ~(1ULL << w));
          }
        }
      }
      lap(5);
      if (limit >= kGreedyThreads) {  // uniform: the window is committed
        if (valid && choice < 0) pair_worker[t] = -1;  // left without a worker (flagged)
        break;
      }
      q0 = limit;
    }
    ++round;
    // the window's masks are spent: clear them for the next (every read of
    // them precedes this barrier); every read of this window's slot precedes
    // it too, so the slot takes the window kGreedySlots further on
    __syncthreads();
    for (int x = tid; x < kGreedyWarps * (kMaxWorkers + 1); x += kGreedyThreads) (&lanes[0][0])[x] = 0;
    if (tid == 0 && c + kGreedySlots < nch) {
      fence_proxy_async_smem();
      stage(c + kGreedySlots);
    }
  }
  if (stats && tid == 0) {
    st[6] = clock64() - st[6];
    for (int q = 0; q < 7; ++q) atomicAdd(stats + q, st[q]);
  }
}

// decision[dest[t]] = pair_worker[t]: the greedy's choices, from position
// order to rows (a position left without a worker raised kFlagUnbalanced).
__global__ void k_greedy_scatter(const int32_t* __restrict__ pw, const uint32_t* __restrict__ dest,
                                 uint64_t n_order, int32_t* __restrict__ decision) {
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (t < n_order && pw[t] >= 0) decision[dest[t]] = pw[t];
}

// DispatchDecision::validate on the device (assign.hpp:41-57): per block a
// shared histogram, added to the global counts; the last block to finish
// compares them with m and clears them for the next call.
constexpr int kBalanceThreads = 256, kBalanceRows = 2048;
__global__ void __launch_bounds__(kBalanceThreads)
    k_check_balance(const int32_t* __restrict__ decision, uint64_t rows, int n, int m,
                    int* __restrict__ flags, int* __restrict__ counts) {
  __shared__ int load[kMaxWorkers];
  __shared__ bool last;
  if (threadIdx.x < kMaxWorkers) load[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kBalanceRows;
  for (uint64_t i = b0 + threadIdx.x; i < rows && i < b0 + kBalanceRows; i += kBalanceThreads) {
    const int w = decision[i];
    if (w < 0 || w >= n) atomicOr(flags + kFlagUnbalanced, 1);
    else atomicAdd(&load[w], 1);
  }
  __syncthreads();
  if (threadIdx.x < n && load[threadIdx.x]) atomicAdd(&counts[threadIdx.x], load[threadIdx.x]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&counts[kMaxWorkers], 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < n) {
    if (atomicExch(&counts[threadIdx.x], 0) != m) atomicOr(flags + kFlagUnbalanced, 1);
  }
  if (threadIdx.x == 0) counts[kMaxWorkers] = 0;
}

// decision_cost (assign.hpp:288-298): a left-to-right fp64 sum in sample
// order.  The order is part of the result, so one thread adds (a chain of
// dependent DADDs, ~8 cycles each); the other warps gather the next chunk of
// C[i, w_i] into the second buffer meanwhile.
constexpr int kCostThreads = 1024, kCostChunk = 2048;

__global__ void __launch_bounds__(kCostThreads)
    k_decision_cost(const double* __restrict__ matrix, const int32_t* __restrict__ decision,
                    uint64_t rows, int n, double* __restrict__ out) {
  __shared__ __align__(16) double vals[2][kCostChunk];
  const int tid = threadIdx.x;
  auto gather = [&](uint64_t base, double* dst, int first, int stride) {
    const int cnt = rows - base < kCostChunk ? static_cast<int>(rows - base) : kCostChunk;
    for (int t = first; t < cnt; t += stride) {
      const uint64_t i = base + t;
      dst[t] = matrix[i * n + decision[i]];
    }
  };
  double total = 0.0;
  if (rows > 0) gather(0, vals[0], tid, kCostThreads);
  __syncthreads();
  int par = 0;
  for (uint64_t base = 0; base < rows; base += kCostChunk, par ^= 1) {
    if (tid >= 32) {
      if (base + kCostChunk < rows) gather(base + kCostChunk, vals[par ^ 1], tid - 32, kCostThreads - 32);
    } else if (tid == 0) {
      const int cnt = rows - base < kCostChunk ? static_cast<int>(rows - base) : kCostChunk;
      const double2* v2 = reinterpret_cast<const double2*>(vals[par]);
      int t = 0;
      for (; t + 8 <= cnt; t += 8) {
        const double2 a = v2[t / 2], b = v2[t / 2 + 1], c = v2[t / 2 + 2], d = v2[t / 2 + 3];
        total = __dadd_rn(total, a.x);
        total = __dadd_rn(total, a.y);
        total = __dadd_rn(total, b.x);
        total = __dadd_rn(total, b.y);
        total = __dadd_rn(total, c.x);
        total = __dadd_rn(total, c.y);
        total = __dadd_rn(total, d.x);
        total = __dadd_rn(total, d.y);
      }
      for (; t < cnt; ++t) total = __dadd_rn(total, vals[par][t]);
    }
    __syncthreads();
  }
  if (tid == 0) *out = total;
}

}  // namespace

void launch_greedy(const double* matrix, uint64_t rows, int n, const uint32_t* order,
                   uint64_t n_order, const int32_t* capacity_dev, int cap_uniform,
                   int32_t* decision, const uint32_t* row_ids, int32_t* pair_worker,
                   int* flags, GreedyScratch& g, cudaStream_t s) {
  (void)rows;
  if (n_order == 0) return;
  g.prefs.ensure(n_order * kListBytes);
  g.dest.ensure(n_order);
  int32_t* pw = pair_worker;
  if (!pw) {
    g.pw.ensure(n_order);
    pw = g.pw.p;
  }
  k_greedy_prefs<<<static_cast<unsigned>((n_order * 32 + 255) / 256), 256, 0, s>>>(
      matrix, n, order, n_order, capacity_dev, cap_uniform, row_ids, g.prefs.p, g.dest.p);
  g_kernel_name[kKGreedy] = "k_greedy";
  static bool attr = [] {
    EDX_CUDA(cudaFuncSetAttribute(k_greedy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kGreedySmem)));
    return true;
  }();
  (void)attr;
  static const bool want_stats = [] {  // EDX_GREEDY_STATS=1: round counters on stderr (tools)
    const char* e = std::getenv("EDX_GREEDY_STATS");
    return e && std::strcmp(e, "1") == 0;
  }();
  if (want_stats) {
    g.stats.ensure(9);
    EDX_CUDA(cudaMemsetAsync(g.stats.p, 0, 9 * sizeof(unsigned long long), s));
  }
  k_greedy<<<1, kGreedyThreads, kGreedySmem, s>>>(n, n_order, capacity_dev, cap_uniform, pw, flags,
                                                  g.prefs.p, want_stats ? g.stats.p : nullptr);
  if (decision)
    k_greedy_scatter<<<static_cast<unsigned>((n_order + 255) / 256), 256, 0, s>>>(pw, g.dest.p,
                                                                                 n_order, decision);
  if (want_stats) {
    unsigned long long h[9];
    EDX_CUDA(cudaMemcpyAsync(h, g.stats.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    EDX_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr,
                 "{\"greedy_stats\": {\"positions\": %llu, \"rounds\": %llu, \"top\": %llu, "
                 "\"A_scan0\": %llu, \"A_bar\": %llu, \"B\": %llu, \"C0\": %llu, \"total\": %llu, "
                 "\"rescans\": %llu}}\n",
                 static_cast<unsigned long long>(n_order), h[0], h[1], h[2], h[3], h[4], h[5], h[6],
                 h[8]);
  }
  EDX_LAUNCHED();
}

void launch_check_balance(const int32_t* decision, uint64_t rows, int n, int m, int* flags,
                          DevBuf<int>& counts, cudaStream_t s) {
  if (counts.n < kMaxWorkers + 1) {  // zeroed once; every call leaves them zero
    counts.ensure(kMaxWorkers + 1);
    EDX_CUDA(cudaMemsetAsync(counts.p, 0, (kMaxWorkers + 1) * sizeof(int), s));
  }
  const unsigned blocks = static_cast<unsigned>(rows ? (rows + kBalanceRows - 1) / kBalanceRows : 1);
  k_check_balance<<<blocks, kBalanceThreads, 0, s>>>(decision, rows, n, m, flags, counts.p);
  EDX_LAUNCHED();
}

void launch_decision_cost(const double* matrix, const int32_t* decision, uint64_t rows, int n,
                          double* out, cudaStream_t s) {
  k_decision_cost<<<1, kCostThreads, 0, s>>>(matrix, decision, rows, n, out);
  EDX_LAUNCHED();
}

// ------------------------------------------------------------------ EcoMix
// detail::exact_multiplicity (assign.hpp:213-216), evaluated on the host in
// the same double arithmetic.
int exact_multiplicity(int m, double alpha) {
  int mult = static_cast<int>(std::floor(m * alpha + 1e-9));
  if (mult < 0) mult = 0;
  if (mult > m) mult = m;
  return mult;
}

DispatchScratch::~DispatchScratch() {
  if (fork) cudaEventDestroy(fork);
  if (join) cudaEventDestroy(join);
  if (side) cudaStreamDestroy(side);
}

void DispatchScratch::init(int device) {
  (void)device;
  if (side) return;
  EDX_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  EDX_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  EDX_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
}

// ecomix (assign.hpp:247-285): rows ordered by gap; the top n*mult rows go to
// the exact solver on the column-expanded block, the rest to the greedy with
// capacity m - mult per worker.  The two parts are independent (the greedy
// capacities do not depend on the exact block's answer), so the greedy runs
// on a side stream concurrently with the latency-bound Hungarian.
void run_ecomix(DispatchScratch& sc, const double* matrix, uint64_t rows, int n, int m,
                double alpha, bool gap_ready, int32_t* decision, int* flags, cudaStream_t s,
                int device, const PhaseEvents* ev, int* launches) {
  sc.init(device);
  const int mult = exact_multiplicity(m, alpha);
  const uint64_t k = static_cast<uint64_t>(n) * static_cast<uint64_t>(mult);
  sc.gap_keys.ensure(rows);
  sc.row_index.ensure(rows);
  sc.order.ensure(rows);
  if (ev && ev->sort0) EDX_CUDA(cudaEventRecord(ev->sort0, s));
  if (!gap_ready) {
    launch_gap_keys(matrix, rows, n, sc.gap_keys.p, sc.row_index.p, s);
    if (launches) ++*launches;
  }
  sort_rows_by_gap(sc.sort, sc.gap_keys.p, sc.row_index.p, sc.order.p, rows, s);
  if (launches) {  // CUB merge sort: one block sort of 2048-key tiles, then a partition and a
                   // merge kernel per pass (as in the launch lists: 5 at 8,192 rows, 11 at 65,536)
    int passes = 0;
    for (uint64_t tiles = (rows + 2047) / 2048; tiles > 1; tiles = (tiles + 1) / 2) ++passes;
    *launches += 1 + 2 * passes;
  }
  if (ev && ev->sort1) EDX_CUDA(cudaEventRecord(ev->sort1, s));
  const bool greedy = k < rows;
  if (greedy) {
    EDX_CUDA(cudaEventRecord(sc.fork, s));
    EDX_CUDA(cudaStreamWaitEvent(sc.side, sc.fork, 0));
    if (ev && ev->greedy0) EDX_CUDA(cudaEventRecord(ev->greedy0, sc.side));
    const NvtxRange nv("edx.greedy (K4 assign.hpp:162-192)");
    launch_greedy(matrix, rows, n, sc.order.p + k, rows - k, nullptr, m - mult, decision,
                  nullptr, nullptr, flags, sc.greedy, sc.side);
    if (launches) ++*launches;
    if (ev && ev->greedy1) EDX_CUDA(cudaEventRecord(ev->greedy1, sc.side));
    EDX_CUDA(cudaEventRecord(sc.join, sc.side));
  }
  if (ev && ev->exact0) EDX_CUDA(cudaEventRecord(ev->exact0, s));
  if (mult > 0) {
    const NvtxRange nv("edx.exact_solve (K6 assign.hpp:80-157)");
    launch_hungarian_blocks(sc.hung, matrix, n, sc.order.p, mult, decision, nullptr, nullptr,
                            flags, s, device);
    if (launches) ++*launches;
  }
  if (ev && ev->exact1) EDX_CUDA(cudaEventRecord(ev->exact1, s));
  if (greedy) EDX_CUDA(cudaStreamWaitEvent(s, sc.join, 0));
  launch_check_balance(decision, rows, n, m, flags, sc.balance, s);
  if (launches) ++*launches;
}

}  // namespace edx
