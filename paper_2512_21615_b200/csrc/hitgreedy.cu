// K8: baseline_hitgreedy on device (assign.hpp:346-392) -- the paper's
// relevance-score (LAIA proxy) baseline, SURVEY §8(f) item 1.
//
// Reference: a sample scores worker j by how many of its ids have their latest
// copy on j; samples commit in order of best score (desc), index (asc); each
// takes its best-scoring worker with workload left, ties to the larger
// remaining workload, then the lower index (strict comparisons, ascending j).
//
// Device version:
//  * scores: one thread per (sample, worker) cell, integer counts from the
//    dense {owners, latest} table; a row's best score by shared atomicMax.
//  * order: stable radix sort of (~best, index) -- equal bests keep index order.
//  * assignment: the remaining workloads make it sequential, so one warp walks
//    the order with lane j holding worker j's (and j+32's) workload: the choice
//    is the max of the packed key (score << 32 | remaining << 6 | 63 - j) --
//    higher score, then larger remaining, then lower index -- over the open
//    workers, two redux.sync.max.  The other warps of the CTA gather the next
//    256 rows' scores into a shared double buffer meanwhile.
#include <cub/device/device_radix_sort.cuh>

#include "edx_internal.cuh"

namespace edx {

namespace {

constexpr int kScoreThreads = 256;
constexpr int kAssignThreads = 256;
constexpr int kAssignRows = 256;  // rows per gathered batch

__global__ void __launch_bounds__(kScoreThreads)
    k_hit_scores(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ offsets,
                 uint64_t rows, int n, int rows_per_block, const ulonglong2* __restrict__ ol,
                 uint64_t id_space, int32_t* __restrict__ scores, uint32_t* __restrict__ keys,
                 uint32_t* __restrict__ index, int* __restrict__ flags) {
  __shared__ int best[kScoreThreads];
  const int local_row = threadIdx.x / n;
  const int j = threadIdx.x - local_row * n;
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * rows_per_block + local_row;
  const bool active = local_row < rows_per_block && i < rows;
  if (threadIdx.x < rows_per_block) best[threadIdx.x] = 0;
  __syncthreads();
  if (active) {
    int s = 0;
    bool bad = false;
    for (uint64_t t = offsets[i]; t < offsets[i + 1]; ++t) {
      const uint32_t id = __ldg(ids + t);
      if (id < id_space) s += static_cast<int>((__ldg(&ol[id].y) >> j) & 1ULL);
      else bad = true;
    }
    if (bad) atomicOr(flags + kFlagIdOutOfRange, 1);
    scores[i * n + j] = s;
    atomicMax(&best[local_row], s);
  }
  __syncthreads();
  if (threadIdx.x < rows_per_block) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * rows_per_block + threadIdx.x;
    if (r < rows) {
      keys[r] = ~static_cast<uint32_t>(best[threadIdx.x]);  // best score descending
      index[r] = static_cast<uint32_t>(r);
    }
  }
}

__global__ void __launch_bounds__(kAssignThreads, 1)
    k_hit_assign(const int32_t* __restrict__ scores, const uint32_t* __restrict__ order,
                 uint64_t rows, int n, int m, int32_t* __restrict__ decision) {
  extern __shared__ __align__(16) int32_t sh[];
  int32_t* sc[2] = {sh, sh + kAssignRows * n};
  uint32_t* rid[2] = {reinterpret_cast<uint32_t*>(sh + 2 * kAssignRows * n),
                      reinterpret_cast<uint32_t*>(sh + 2 * kAssignRows * n) + kAssignRows};
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t nb = (rows + kAssignRows - 1) / kAssignRows;
  auto gather = [&](uint64_t b, int buf, int t0, int stride) {
    const uint64_t r0 = b * kAssignRows;
    const int cnt = static_cast<int>(rows - r0 < kAssignRows ? rows - r0 : kAssignRows);
    for (int r = t0; r < cnt; r += stride) rid[buf][r] = order[r0 + r];
    // four gathers in flight per thread (the loads are independent)
    for (int e0 = t0; e0 < cnt * n; e0 += 4 * stride) {
      int32_t v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = e0 + q * stride;
        v[q] = 0;
        if (e < cnt * n) {
          const int r = e / n, j = e - r * n;
          v[q] = __ldg(scores + static_cast<uint64_t>(__ldg(order + r0 + r)) * n + j);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (e0 + q * stride < cnt * n) sc[buf][e0 + q * stride] = v[q];
    }
  };
  gather(0, 0, tid, kAssignThreads);
  __syncthreads();
  // lane j holds workers j and j + 32 (n <= 64)
  const int j0 = lane, j1 = lane + 32;
  uint32_t rem0 = j0 < n ? static_cast<uint32_t>(m) : 0u;
  uint32_t rem1 = j1 < n ? static_cast<uint32_t>(m) : 0u;
  for (uint64_t b = 0; b < nb; ++b) {
    const int buf = static_cast<int>(b & 1);
    if (warp != 0) {
      if (b + 1 < nb) gather(b + 1, buf ^ 1, tid - 32, kAssignThreads - 32);
    } else {
      const int cnt = static_cast<int>(rows - b * kAssignRows < kAssignRows ? rows - b * kAssignRows : kAssignRows);
      // the next row's scores are loaded one row ahead, off the REDUX chain
      uint32_t s0 = j0 < n ? static_cast<uint32_t>(sc[buf][j0]) : 0u;
      uint32_t s1 = j1 < n ? static_cast<uint32_t>(sc[buf][j1]) : 0u;
      for (int r = 0; r < cnt; ++r) {
        const int32_t* nrow = sc[buf] + (r + 1 < cnt ? r + 1 : r) * n;
        const uint32_t ns0 = j0 < n ? static_cast<uint32_t>(nrow[j0]) : 0u;
        const uint32_t ns1 = j1 < n ? static_cast<uint32_t>(nrow[j1]) : 0u;
        const uint64_t k0 = rem0 ? (static_cast<uint64_t>(s0) << 32) |
                                       (static_cast<uint64_t>(rem0) << 6) | static_cast<uint64_t>(63 - j0)
                                 : 0ULL;
        const uint64_t k1 = rem1 ? (static_cast<uint64_t>(s1) << 32) |
                                       (static_cast<uint64_t>(rem1) << 6) | static_cast<uint64_t>(63 - j1)
                                 : 0ULL;
        s0 = ns0;
        s1 = ns1;
        const uint64_t k = k0 > k1 ? k0 : k1;
        const unsigned hi = static_cast<unsigned>(k >> 32), lo = static_cast<unsigned>(k);
        const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
        const int w = 63 - static_cast<int>(ml & 63u);
        if (w == j0) --rem0;
        if (w == j1) --rem1;
        if (lane == 0) decision[rid[buf][r]] = w;
      }
    }
    __syncthreads();
  }
}

}  // namespace

void launch_hitgreedy(HitScratch& sc, const uint32_t* ids, const uint64_t* offsets, uint64_t rows,
                      int n, int m, const ulonglong2* ol, uint64_t id_space, int32_t* decision,
                      int* flags, cudaStream_t s) {
  if (rows == 0) return;
  sc.scores.ensure(rows * n);
  sc.keys.ensure(rows);
  sc.keys_sorted.ensure(rows);
  sc.index.ensure(rows);
  sc.index_sorted.ensure(rows);
  const int rows_per_block = kScoreThreads / n;
  const unsigned blocks = static_cast<unsigned>((rows + rows_per_block - 1) / rows_per_block);
  k_hit_scores<<<blocks, rows_per_block * n, 0, s>>>(ids, offsets, rows, n, rows_per_block, ol,
                                                     id_space, sc.scores.p, sc.keys.p, sc.index.p,
                                                     flags);
  EDX_LAUNCHED();
  size_t bytes = 0;
  EDX_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, sc.keys.p, sc.keys_sorted.p, sc.index.p,
                                           sc.index_sorted.p, static_cast<int>(rows), 0, 32, s));
  sc.temp.ensure(bytes);
  bytes = sc.temp.n;
  EDX_CUDA(cub::DeviceRadixSort::SortPairs(sc.temp.p, bytes, sc.keys.p, sc.keys_sorted.p, sc.index.p,
                                           sc.index_sorted.p, static_cast<int>(rows), 0, 32, s));
  const size_t smem = (2 * static_cast<size_t>(kAssignRows) * n + 2 * kAssignRows) * sizeof(int32_t);
  if (smem > 48 * 1024)
    EDX_CUDA(cudaFuncSetAttribute(k_hit_assign, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  k_hit_assign<<<1, kAssignThreads, smem, s>>>(sc.scores.p, sc.index_sorted.p, rows, n, m, decision);
  EDX_LAUNCHED();
}

}  // namespace edx
