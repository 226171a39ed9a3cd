// K3 row ordering, K4 capacity-bounded greedy, decision checks, and the
// EcoMix orchestration (assign.hpp:162-298).
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>

#include "edx_internal.cuh"

namespace edx {

// ------------------------------------------------------------------ K3 sort
// rows_by_gap (assign.hpp:197-207) orders rows by (gap desc, index asc).  The
// gap keys are ~bits(gap) (cost.cu), so an ascending *stable* radix sort of
// (key, row) pairs with rows fed in index order reproduces std::sort with the
// reference's total order exactly.
void sort_rows_by_gap(SortScratch& sc, const uint64_t* keys_in, const uint32_t* idx_in,
                      uint32_t* idx_out, uint64_t rows, cudaStream_t s) {
  sc.keys_out.ensure(rows);
  size_t bytes = 0;
  EDX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys_in, sc.keys_out.p, idx_in,
                                           idx_out, static_cast<int>(rows), 0, 64, s));
  sc.temp.ensure(bytes);
  EDX_CUDA(cub::DeviceRadixSort::SortPairs(sc.temp.p, bytes, keys_in, sc.keys_out.p, idx_in,
                                           idx_out, static_cast<int>(rows), 0, 64, s));
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
// row is the first divergence.  Each round closes >= 1 worker: <= n rounds.
namespace {


// Each position's eight best workers among the initially open ones, in
// (cost, index) order -- strict '<' over ascending j, as the reference's scan
// (assign.hpp:177-184) -- packed 8 bits each (0xFF = none).  One thread per
// position, grid-wide: the matrix is read once.
constexpr int kPrefs = 8;

__global__ void k_greedy_prefs(const double* __restrict__ matrix, int n,
                               const uint32_t* __restrict__ order, uint64_t n_order,
                               const int32_t* __restrict__ capacity_dev, int cap_uniform,
                               uint64_t* __restrict__ prefs) {
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (t >= n_order) return;
  const double* r = matrix + static_cast<uint64_t>(order[t]) * n;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double cb[kPrefs];
  int wb[kPrefs];
#pragma unroll
  for (int q = 0; q < kPrefs; ++q) {
    cb[q] = inf;
    wb[q] = 0xFF;
  }
  for (int w = 0; w < n; ++w) {
    if ((capacity_dev ? capacity_dev[w] : cap_uniform) <= 0) continue;
    const double c = r[w];
    if (!(c < cb[kPrefs - 1])) continue;
    // insertion keeps equal costs in index order (strict '<')
    bool placed = false;
#pragma unroll
    for (int q = kPrefs - 1; q > 0; --q) {
      if (!placed) {
        if (c < cb[q - 1]) {
          cb[q] = cb[q - 1];
          wb[q] = wb[q - 1];
        } else {
          cb[q] = c;
          wb[q] = w;
          placed = true;
        }
      }
    }
    if (!placed) {
      cb[0] = c;
      wb[0] = w;
    }
  }
  uint64_t pk = 0;
#pragma unroll
  for (int q = 0; q < kPrefs; ++q) pk |= static_cast<uint64_t>(wb[q]) << (8 * q);
  prefs[t] = pk;
}

// The rounds on the whole GPU: one cooperative kernel, tile b of positions
// owned by CTA b.  A round (one grid-wide sync) is
//  A: every position >= q0 whose stored choice is unset or now closed takes
//     its argmin over the open set (first open of its eight preferences, else
//     a rescan); each CTA publishes its per-worker counts of positions >= q0;
//  B: every CTA, redundantly and identically, scans those counts over the
//     tiles to find for each worker w the tile holding its (remaining_w+1)-th
//     pick -- the earliest such tile holds the round's first over-capacity
//     position qm, found exactly from that tile's stored choices -- then
//     finalises its own positions in [q0, qm), subtracts every worker's picks
//     in [q0, qm) from its remaining capacity, closes exhausted workers and
//     moves q0 to qm.
// Positions before qm never change again, so a CTA still in phase B of round
// r reads only settled choices while others already rewrite choices >= qm in
// round r+1; the counts are double-buffered by round parity.  Rows whose
// choice stays open keep it across rounds (closing a worker that is not a
// row's minimum does not move that minimum).
constexpr int kGGThreads = 1024;

struct GreedyGridArgs {
  const double* matrix;
  int n;
  const uint32_t* order;
  uint64_t n_order;
  const int32_t* capacity_dev;
  int cap_uniform;
  int32_t* decision;
  const uint32_t* row_ids;
  int32_t* pair_worker;
  int* flags;
  const uint64_t* prefs;
  int32_t* choice;  // n_order
  uint32_t* cnt;    // 2 * gridDim.x * kMaxWorkers
  int ppt;          // positions per thread
};

// argmin over the open workers (assign.hpp:177-184: ascending j, strict '<')
__device__ __forceinline__ int greedy_pick(const GreedyGridArgs& a, uint64_t t,
                                           unsigned long long om) {
  const uint64_t pf = a.prefs[t];
#pragma unroll
  for (int q = 0; q < kPrefs; ++q) {
    const int w = static_cast<int>((pf >> (8 * q)) & 0xFFu);
    if (w != 0xFF && ((om >> w) & 1ULL)) return w;
  }
  const double* r = a.matrix + static_cast<uint64_t>(a.order[t]) * a.n;
  double best = __longlong_as_double(0x7ff0000000000000LL);
  int choice = -1;
  for (int base = 0; base < a.n; base += 16) {
    double c[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int w = base + k;
      c[k] = (w < a.n && ((om >> w) & 1ULL)) ? r[w] : best;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (c[k] < best) {
        best = c[k];
        choice = base + k;
      }
  }
  return choice;
}

__global__ void __launch_bounds__(kGGThreads)
    k_greedy_grid(GreedyGridArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ int rem[kMaxWorkers];
  __shared__ uint32_t cntL[kMaxWorkers];
  __shared__ int cw[kMaxWorkers];        // tile of each worker's over-capacity pick
  __shared__ uint32_t kw[kMaxWorkers];   // its rank inside that tile
  __shared__ uint32_t used[kMaxWorkers];
  __shared__ uint32_t wsum[kGGThreads / 32];
  __shared__ unsigned long long open_s;
  __shared__ int cstar_s;
  __shared__ uint32_t chunk_hits;
  __shared__ unsigned long long qm_s;
  const int n = a.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const uint64_t tile = static_cast<uint64_t>(kGGThreads) * a.ppt;
  const uint64_t tb = blockIdx.x * tile;
  const uint64_t te = min(a.n_order, tb + tile);
  if (tid < kMaxWorkers) rem[tid] = tid < n ? (a.capacity_dev ? a.capacity_dev[tid] : a.cap_uniform) : 0;
  __syncthreads();
  if (tid == 0) {
    unsigned long long om = 0;
    for (int w = 0; w < n; ++w)
      if (rem[w] > 0) om |= 1ULL << w;
    open_s = om;
  }
  __syncthreads();
  uint64_t q0 = 0;
  int par = 0;
  bool first = true;
  for (;;) {
    // ---- A: choices of the unsettled positions, per-CTA counts
    if (tid < kMaxWorkers) cntL[tid] = 0;
    __syncthreads();
    const unsigned long long om = open_s;
    for (int j = 0; j < a.ppt; ++j) {
      const uint64_t t = tb + tid + static_cast<uint64_t>(j) * kGGThreads;
      const bool live = t < te && t >= q0;
      int c = -1;
      if (live) {
        c = first ? -1 : a.choice[t];
        if (c < 0 || !((om >> c) & 1ULL)) {
          c = greedy_pick(a, t, om);
          if (c < 0) atomicOr(a.flags + kFlagUnbalanced, 1);  // capacities exhausted
          a.choice[t] = c;
        }
      }
      const unsigned grp = __match_any_sync(0xffffffffu, c);
      if (c >= 0 && lane == __ffs(grp) - 1) atomicAdd(&cntL[c], static_cast<uint32_t>(__popc(grp)));
    }
    __syncthreads();
    uint32_t* cnt = a.cnt + static_cast<uint64_t>(par) * G * kMaxWorkers;
    if (tid < n) cnt[blockIdx.x * kMaxWorkers + tid] = cntL[tid];
    grid.sync();
    // ---- B: the first over-capacity position, identically in every CTA
    const int c0 = static_cast<int>(q0 / tile);
    for (int w = warp; w < n; w += kGGThreads / 32) {
      uint32_t carry = 0;
      int found = G;
      uint32_t kk = 0;
      for (int cb = c0; cb < G && found == G; cb += 32) {
        const int c = cb + lane;
        const uint32_t v = c < G ? cnt[c * kMaxWorkers + w] : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        const uint32_t cum = carry + inc;
        const unsigned over = __ballot_sync(0xffffffffu, c < G && cum > static_cast<uint32_t>(rem[w]));
        if (over) {
          const int l = __ffs(over) - 1;
          found = cb + l;
          kk = static_cast<uint32_t>(rem[w]) - (__shfl_sync(0xffffffffu, cum, l) -
                                                __shfl_sync(0xffffffffu, v, l)) + 1u;
        }
        carry = __shfl_sync(0xffffffffu, cum, 31);
      }
      if (lane == 0) {
        cw[w] = found;
        kw[w] = kk;
      }
    }
    __syncthreads();
    if (warp == 0) {
      int m = G;
      for (int w = lane; w < n; w += 32) m = min(m, cw[w]);
      m = __reduce_min_sync(0xffffffffu, m);
      if (lane == 0) {
        cstar_s = m;
        qm_s = a.n_order;
      }
    }
    __syncthreads();
    const int cstar = cstar_s;
    if (cstar < G) {
      // exact position of each over-capacity pick in tile cstar (usually one worker)
      const uint64_t sb = cstar * tile, se = min(a.n_order, sb + tile);
      for (int w = 0; w < n; ++w) {
        if (cw[w] != cstar) continue;  // uniform
        uint32_t need = kw[w];  // rank of the pick among tile cstar's picks of w at >= q0
        for (int j = 0; j < a.ppt && need > 0; ++j) {  // `need` is block-uniform
          const uint64_t t = sb + tid + static_cast<uint64_t>(j) * kGGThreads;
          const bool hit = t < se && t >= q0 && a.choice[t] == w;
          const unsigned bal = __ballot_sync(0xffffffffu, hit);
          if (lane == 0) wsum[warp] = __popc(bal);
          __syncthreads();
          if (warp == 0) {
            const uint32_t x = wsum[lane];
            uint32_t inc = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
              if (lane >= o) inc += y;
            }
            wsum[lane] = inc - x;  // exclusive over warps
            if (lane == 31) chunk_hits = inc;
          }
          __syncthreads();
          const uint32_t before = wsum[warp] + __popc(bal & ((1u << lane) - 1u));
          if (hit && before + 1 == need) atomicMin(&qm_s, static_cast<unsigned long long>(t));
          need = need > chunk_hits ? need - chunk_hits : 0u;
          __syncthreads();
        }
      }
    }
    __syncthreads();
    const uint64_t qm = qm_s;
    // picks per worker in [q0, qm): whole tiles before cstar from the counts,
    // the part of tile cstar from its choices
    if (tid < kMaxWorkers) used[tid] = 0;
    __syncthreads();
    const int cend = cstar < G ? cstar : G;
    for (int w = warp; w < n; w += kGGThreads / 32) {
      uint32_t sum = 0;
      for (int c = c0 + lane; c < cend; c += 32) sum += cnt[c * kMaxWorkers + w];
      sum = __reduce_add_sync(0xffffffffu, sum);
      if (lane == 0) used[w] = sum;
    }
    __syncthreads();
    if (cstar < G) {
      const uint64_t sb = cstar * tile;
      for (int j = 0; j < a.ppt; ++j) {
        const uint64_t t = sb + tid + static_cast<uint64_t>(j) * kGGThreads;
        const int c = (t >= q0 && t < qm) ? a.choice[t] : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, c);
        if (c >= 0 && lane == __ffs(grp) - 1) atomicAdd(&used[c], static_cast<uint32_t>(__popc(grp)));
      }
    }
    // this CTA's settled positions
    for (int j = 0; j < a.ppt; ++j) {
      const uint64_t t = tb + tid + static_cast<uint64_t>(j) * kGGThreads;
      if (t < te && t >= q0 && t < qm) {
        const int c = a.choice[t];
        if (a.decision) {
          const uint32_t row = a.order[t];
          a.decision[a.row_ids ? a.row_ids[row] : row] = c;
        }
        if (a.pair_worker) a.pair_worker[t] = c;
      }
    }
    __syncthreads();
    if (qm >= a.n_order) break;
    if (tid < n) rem[tid] -= static_cast<int>(used[tid]);
    __syncthreads();
    if (tid == 0) {
      unsigned long long o = 0;
      for (int w = 0; w < n; ++w)
        if (rem[w] > 0) o |= 1ULL << w;
      open_s = o;
    }
    __syncthreads();
    q0 = qm;
    par ^= 1;
    first = false;
  }
}

__global__ void k_check_balance(const int32_t* __restrict__ decision, uint64_t rows, int n,
                                int m, int* __restrict__ flags) {
  __shared__ int load[kMaxWorkers];
  if (threadIdx.x < kMaxWorkers) load[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const int w = decision[i];
    if (w < 0 || w >= n) atomicOr(flags + kFlagUnbalanced, 1);
    else atomicAdd(&load[w], 1);
  }
  __syncthreads();
  if (threadIdx.x < n && load[threadIdx.x] != m) atomicOr(flags + kFlagUnbalanced, 1);
}

// decision_cost (assign.hpp:288-298): a left-to-right fp64 sum in sample
// order.  The order is part of the result, so one thread adds; the gather of
// C[i, w_i] (the latency) is done by the whole block into shared memory
// first, chunk by chunk.
constexpr int kCostThreads = 1024, kCostChunk = 4096;

__global__ void __launch_bounds__(kCostThreads)
    k_decision_cost(const double* __restrict__ matrix, const int32_t* __restrict__ decision,
                    uint64_t rows, int n, double* __restrict__ out) {
  __shared__ double vals[kCostChunk];
  double total = 0.0;
  for (uint64_t base = 0; base < rows; base += kCostChunk) {
    const int cnt = rows - base < kCostChunk ? static_cast<int>(rows - base) : kCostChunk;
    for (int t = threadIdx.x; t < cnt; t += kCostThreads) {
      const uint64_t i = base + t;
      vals[t] = matrix[i * n + decision[i]];
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int t = 0; t < cnt; ++t) total = __dadd_rn(total, vals[t]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = total;
}

}  // namespace

void launch_greedy(const double* matrix, uint64_t rows, int n, const uint32_t* order,
                   uint64_t n_order, const int32_t* capacity_dev, int cap_uniform,
                   int32_t* decision, const uint32_t* row_ids, int32_t* pair_worker,
                   int* flags, GreedyScratch& g, cudaStream_t s) {
  (void)rows;
  if (n_order == 0) return;
  if (g.sms == 0) {
    int dev = 0;
    EDX_CUDA(cudaGetDevice(&dev));
    EDX_CUDA(cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // one tile of >= 1024 positions per CTA, at most one CTA per SM but one (the
  // exact solver, running concurrently on its own SM, holds a whole SM)
  const uint64_t want = (n_order + kGGThreads - 1) / kGGThreads;
  const int G = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(want, g.sms > 1 ? g.sms - 1 : 1)));
  const int ppt = static_cast<int>((n_order + static_cast<uint64_t>(G) * kGGThreads - 1) /
                                   (static_cast<uint64_t>(G) * kGGThreads));
  g.prefs.ensure(n_order);
  g.choice.ensure(n_order);
  g.cnt.ensure(2 * static_cast<size_t>(G) * kMaxWorkers);
  k_greedy_prefs<<<static_cast<unsigned>((n_order + 255) / 256), 256, 0, s>>>(
      matrix, n, order, n_order, capacity_dev, cap_uniform, g.prefs.p);
  EDX_LAUNCHED();
  GreedyGridArgs a{matrix, n, order, n_order, capacity_dev, cap_uniform, decision, row_ids,
                   pair_worker, flags, g.prefs.p, g.choice.p, g.cnt.p, ppt};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(G));
  cfg.blockDim = dim3(kGGThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  EDX_CUDA(cudaLaunchKernelEx(&cfg, k_greedy_grid, a));
  g_kernel_name[kKGreedy] = "k_greedy_grid";
}

void launch_check_balance(const int32_t* decision, uint64_t rows, int n, int m, int* flags,
                          cudaStream_t s) {
  k_check_balance<<<1, 1024, 0, s>>>(decision, rows, n, m, flags);
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
  if (launches) *launches += 4;  // CUB onesweep: histogram + 3..4 passes (approx.)
  if (ev && ev->sort1) EDX_CUDA(cudaEventRecord(ev->sort1, s));
  const bool greedy = k < rows;
  if (greedy) {
    EDX_CUDA(cudaEventRecord(sc.fork, s));
    EDX_CUDA(cudaStreamWaitEvent(sc.side, sc.fork, 0));
    if (ev && ev->greedy0) EDX_CUDA(cudaEventRecord(ev->greedy0, sc.side));
    launch_greedy(matrix, rows, n, sc.order.p + k, rows - k, nullptr, m - mult, decision,
                  nullptr, nullptr, flags, sc.greedy, sc.side);
    if (launches) ++*launches;
    if (ev && ev->greedy1) EDX_CUDA(cudaEventRecord(ev->greedy1, sc.side));
    EDX_CUDA(cudaEventRecord(sc.join, sc.side));
  }
  if (ev && ev->exact0) EDX_CUDA(cudaEventRecord(ev->exact0, s));
  if (mult > 0) {
    launch_hungarian_blocks(sc.hung, matrix, n, sc.order.p, mult, decision, nullptr, nullptr,
                            flags, s, device);
    if (launches) ++*launches;
  }
  if (ev && ev->exact1) EDX_CUDA(cudaEventRecord(ev->exact1, s));
  if (greedy) EDX_CUDA(cudaStreamWaitEvent(s, sc.join, 0));
  launch_check_balance(decision, rows, n, m, flags, s);
  if (launches) ++*launches;
}

}  // namespace edx
