// K1 cost build + K2 row gap keys.
//
// Reference: expected_cost / build_matrix (cost.hpp:81-125) and row_gap_key
// (cost.hpp:130-146).  Each cell (i, j) is a strictly left-to-right fp64
// chain over sample i's ids: for an id whose latest copy is not on j, add
// u_j, then u_o for every other owner o in ascending worker order.  Ties are
// pervasive in real matrices, so cells must be bit-identical to
// the reference: one thread owns one cell's whole chain, every add is an
// explicit __dadd_rn, and nothing is ever re-associated.
//
// Layout: one thread per cell, a block holds whole rows (rows_per_block * n
// threads), so the R x n row-major matrix is written fully coalesced and the
// gap epilogue reads its rows from shared memory.  The per-id state masks
// {owners, latest} are one 16-byte gather per id from the dense state table;
// threads of one row hit the same address (a broadcast), so each id costs
// one L1/L2 transaction per row.  Loads are batched 4 ids ahead of the add
// chain to keep memory-level parallelism despite the serial adds.
#include <type_traits>

#include "edx_internal.cuh"

namespace edx {

namespace {

constexpr int kBlockCells = 256;
constexpr int kPrefetch = 4;

__device__ __forceinline__ uint64_t gap_sort_key(double gap) {
  // gap = second - smallest >= +0.0 and finite, so its bit pattern is
  // order-preserving; ~bits sorts descending (rows_by_gap, assign.hpp:202-205).
  return ~static_cast<uint64_t>(__double_as_longlong(gap));
}

// row_gap_key (cost.hpp:130-146): same selection loop, column order.
__device__ __forceinline__ double row_gap(const double* row, int n) {
  if (n == 1) return 0.0;
  double smallest = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  double second = smallest;
  for (int c = 0; c < n; ++c) {
    const double v = row[c];
    if (v < smallest) {
      second = smallest;
      smallest = v;
    } else if (v < second) {
      second = v;
    }
  }
  return __dsub_rn(second, smallest);
}

__global__ void __launch_bounds__(kBlockCells)
    k_cost_build(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ offsets,
                 uint64_t rows, int n, int rows_per_block, const ulonglong2* __restrict__ ol,
                 uint64_t id_space, const double* __restrict__ ucost,
                 const uint64_t* __restrict__ sizes, const double* __restrict__ bw,
                 double* __restrict__ matrix, uint64_t* __restrict__ gap_keys,
                 uint32_t* __restrict__ row_index, int* __restrict__ flags) {
  __shared__ double u_s[kMaxWorkers];
  __shared__ double tile[kBlockCells];
  // sizes == nullptr: u_s = unit costs; else u_s = bandwidths and every add is
  // transfer_seconds (cost.hpp:68-73) of the id's own size: bytes * 8.0 / bw
  if (threadIdx.x < n) u_s[threadIdx.x] = sizes ? bw[threadIdx.x] : ucost[threadIdx.x];
  __syncthreads();

  const int local_row = threadIdx.x / n;
  const int j = threadIdx.x - local_row * n;
  const uint64_t row0 = static_cast<uint64_t>(blockIdx.x) * rows_per_block;
  const uint64_t i = row0 + local_row;
  const bool active = local_row < rows_per_block && i < rows;

  double c = 0.0;
  if (active) {
    const uint64_t jbit = 1ULL << j;
    const double uj = u_s[j];
    const uint64_t beg = offsets[i], end = offsets[i + 1];
    bool bad = false;
    for (uint64_t t = beg; sizes && t < end; ++t) {  // SizeLookupFn path (cost.hpp:64-73)
      const uint32_t id = __ldg(ids + t);
      ulonglong2 st = make_ulonglong2(0, 0);
      if (id < id_space) st = __ldg(ol + id);
      else bad = true;
      if (st.y & jbit) continue;
      const double bytes8 = __dmul_rn(__ull2double_rn(sizes[t]), 8.0);
      c = __dadd_rn(c, __ddiv_rn(bytes8, u_s[j]));
      uint64_t others = st.x & ~jbit;
      while (others) {
        const int o = __ffsll(static_cast<long long>(others)) - 1;
        others &= others - 1;
        c = __dadd_rn(c, __ddiv_rn(bytes8, u_s[o]));
      }
    }
    for (uint64_t t = beg; !sizes && t < end; t += kPrefetch) {
      ulonglong2 st[kPrefetch];
#pragma unroll
      for (int q = 0; q < kPrefetch; ++q) {
        st[q] = make_ulonglong2(0, 0);
        if (t + q < end) {
          const uint32_t id = __ldg(ids + t + q);
          if (id < id_space) st[q] = __ldg(ol + id);
          else bad = true;
        }
      }
#pragma unroll
      for (int q = 0; q < kPrefetch; ++q) {
        if (t + q >= end) break;
        if (st[q].y & jbit) continue;  // latest copy already on j: free
        c = __dadd_rn(c, uj);          // miss pull over j's link
        uint64_t others = st[q].x & ~jbit;
        while (others) {                // one push per other owner, ascending
          const int o = __ffsll(static_cast<long long>(others)) - 1;
          others &= others - 1;
          c = __dadd_rn(c, u_s[o]);
        }
      }
    }
    if (bad) atomicOr(flags + kFlagIdOutOfRange, 1);
    matrix[i * n + j] = c;
  }
  if (gap_keys == nullptr) return;
  if (local_row < rows_per_block) tile[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x < rows_per_block) {
    const uint64_t r = row0 + threadIdx.x;
    if (r < rows) {
      gap_keys[r] = gap_sort_key(row_gap(tile + threadIdx.x * n, n));
      row_index[r] = static_cast<uint32_t>(r);
    }
  }
}

// ------------------------------------------------ K1, 2 <= n <= 8 (warp rows)
// A warp holds 32 / NP rows, one group of NP >= n lanes per row (lane j of a
// group = worker j).  Each lane loads up to 4 of its row's ids and their
// {owners, latest} masks up front, so every gather of the row is in flight at
// once.  Ids are then taken 8 at a time: for each, the group expands the
// id's owner list into shared memory -- owner o's unit cost at position
// popc(owners below o), -0.0 after the last owner -- and afterwards every
// lane runs its chains for the 8 ids back to back: += u_j, then += u_o for
// the owners in ascending order, two per 16-byte broadcast load, entering a
// fully unrolled run of pairs at the right offset (no loop, no predicate).
// A lane whose worker holds the latest copy reads an all -0.0 list instead:
// x + -0.0 == x for every x these chains produce, so padding and inactive
// lanes are exact no-ops and each cell's add sequence is the reference's.
// The row gap (two smallest of the row, with multiplicity) is a shuffle
// reduction, order-independent, then one __dsub_rn.
constexpr int kWarpRowsThreads = 128;

__device__ __forceinline__ int popc_mask(unsigned x) { return __popc(x); }
__device__ __forceinline__ int popc_mask(unsigned long long x) { return __popcll(x); }
constexpr int kIdsPerLane = 4;

template <int NP>
__global__ void __launch_bounds__(kWarpRowsThreads)
    k_cost_build_warp(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ offsets,
                      uint64_t rows, int n, const ulonglong2* __restrict__ ol, uint64_t id_space,
                      const double* __restrict__ ucost, double* __restrict__ matrix,
                      uint64_t* __restrict__ gap_keys, uint32_t* __restrict__ row_index,
                      int* __restrict__ flags) {
  constexpr int RPW = 32 / NP;
  constexpr int NW = kWarpRowsThreads / 32;
  static_assert(NP <= 8, "wide rows use k_cost_build_wide");
  constexpr int kSub = NP;  // ids per sub-batch: one whole load slot
  // [warp][buffer][id of the sub-batch][32 lanes' list entries]
  __shared__ __align__(16) double lists[NW][2][kSub][32];
  __shared__ __align__(16) double zeros[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 32) zeros[threadIdx.x] = -0.0;
  __syncthreads();
  const int g = lane / NP, j = lane - g * NP;
  const uint64_t i = (static_cast<uint64_t>(blockIdx.x) * NW + warp) * RPW + g;
  const bool rowok = i < rows;
  const bool cell = rowok && j < n;
  const double uj = j < n ? ucost[j] : 0.0;
  uint64_t beg = 0, end = 0;
  if (rowok) {
    beg = offsets[i];
    end = offsets[i + 1];
  }
  const int len = static_cast<int>(end - beg);
  const int maxlen = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(len));
  const unsigned below_j = (1u << j) - 1u;
  double c = 0.0;
  bool bad = false;
  int sb = 0;  // sub-batch parity
  for (int t0 = 0; t0 < maxlen; t0 += kIdsPerLane * NP) {
    unsigned own[kIdsPerLane], lat[kIdsPerLane];
    uint32_t idv[kIdsPerLane];
#pragma unroll
    for (int s = 0; s < kIdsPerLane; ++s) {
      const int idx = t0 + s * NP + j;
      idv[s] = idx < len ? __ldg(ids + beg + idx) : 0xffffffffu;
    }
#pragma unroll
    for (int s = 0; s < kIdsPerLane; ++s) {
      const int idx = t0 + s * NP + j;
      own[s] = 0u;
      lat[s] = 0xffffffffu;  // past the row's end: no lane adds
      if (idx < len) {
        if (idv[s] < id_space) {
          const ulonglong2 m = __ldg(ol + idv[s]);
          own[s] = static_cast<unsigned>(m.x);
          lat[s] = static_cast<unsigned>(m.y);
        } else {
          bad = true;
        }
      }
    }
    // Ids of slot s are t0 + s * NP + tt, held by lane tt of each group; a
    // lane past its row's end holds (owners 0, latest all-ones), so ids beyond
    // a row need no masking -- nobody adds for them.
#pragma unroll
    for (int s = 0; s < kIdsPerLane; ++s) {
      if (t0 + s * NP >= maxlen) break;
      for (int u0 = 0; u0 < NP; u0 += kSub) {
        if (t0 + s * NP + u0 >= maxlen) break;
        double (*buf)[32] = lists[warp][sb];
        unsigned pm[kSub];
        bool act[kSub];
#pragma unroll
        for (int q = 0; q < kSub; ++q) {
          const unsigned O = __shfl_sync(0xffffffffu, own[s], u0 + q, NP);
          const unsigned Lm = __shfl_sync(0xffffffffu, lat[s], u0 + q, NP);
          const int p = __popc(O);
          pm[q] = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(p));
          const bool has = (O >> j) & 1u;
          const int below = __popc(O & below_j);
          buf[q][g * NP + (has ? below : p + (j - below))] = has ? uj : -0.0;
          act[q] = cell && !((Lm >> j) & 1u);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kSub; ++q) {
          c = __dadd_rn(c, act[q] ? uj : -0.0);  // miss pull over j's link
          // pushes, owners ascending, in blocks of 4 pairs: positions past the
          // last owner hold -0.0, so whole blocks are exact
          const double* lp = act[q] ? &buf[q][g * NP] : zeros;
          const int nblk = (static_cast<int>(pm[q]) + 7) >> 3;
#pragma unroll
          for (int bk = 0; bk < (NP + 7) / 8; ++bk) {
            if (bk >= nblk) break;
            double2 v2[4];
#pragma unroll
            for (int h = 0; h < 4; ++h)
              v2[h] = (8 * bk + 2 * h < NP) ? *reinterpret_cast<const double2*>(lp + 8 * bk + 2 * h)
                                            : make_double2(-0.0, -0.0);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              if (8 * bk + 2 * h < NP) {
                c = __dadd_rn(c, v2[h].x);
                c = __dadd_rn(c, v2[h].y);
              }
            }
          }
        }
        sb ^= 1;
      }
    }
  }
  if (bad) atomicOr(flags + kFlagIdOutOfRange, 1);
  if (cell) matrix[i * n + j] = c;
  if (gap_keys == nullptr) return;
  // two smallest of the row with multiplicity (row_gap_key, cost.hpp:130-146)
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double s1 = cell ? c : inf, s2 = inf;
#pragma unroll
  for (int off = NP / 2; off > 0; off >>= 1) {
    const double b1 = __shfl_xor_sync(0xffffffffu, s1, off, NP);
    const double b2 = __shfl_xor_sync(0xffffffffu, s2, off, NP);
    const double lo = s1 < b1 ? s1 : b1, hi = s1 < b1 ? b1 : s1;
    const double m2 = s2 < b2 ? s2 : b2;
    s1 = lo;
    s2 = hi < m2 ? hi : m2;
  }
  if (rowok && j == 0) {
    gap_keys[i] = gap_sort_key(__dsub_rn(s2, s1));
    row_index[i] = static_cast<uint32_t>(i);
  }
}

// K1 for 16 workers (NP = 16, two rows per warp): the
// same row layout, loads and list expansion, one id at a time -- list, one
// __syncwarp, then the chain with every lane reading the same list (a
// single broadcast per load) and the adds taken only by the lanes whose
// worker does not hold the latest copy.  A compact loop body keeps the
// instruction stream in cache.
template <int NP>
__global__ void __launch_bounds__(kWarpRowsThreads)
    k_cost_build_wide(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ offsets,
                      uint64_t rows, int n, const ulonglong2* __restrict__ ol, uint64_t id_space,
                      const double* __restrict__ ucost, double* __restrict__ matrix,
                      uint64_t* __restrict__ gap_keys, uint32_t* __restrict__ row_index,
                      int* __restrict__ flags) {
  constexpr int RPW = 32 / NP;
  __shared__ __align__(16) double lists[kWarpRowsThreads / 32][2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / NP, j = lane - g * NP;
  const uint64_t i = (static_cast<uint64_t>(blockIdx.x) * (kWarpRowsThreads / 32) + warp) * RPW + g;
  const bool rowok = i < rows;
  const bool cell = rowok && j < n;
  const double uj = j < n ? ucost[j] : 0.0;
  uint64_t beg = 0, end = 0;
  if (rowok) {
    beg = offsets[i];
    end = offsets[i + 1];
  }
  const int len = static_cast<int>(end - beg);
  const int maxlen = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(len));
  const unsigned below_j = (1u << j) - 1u;
  double* const mylist = &lists[warp][0][g * NP];
  double c = 0.0;
  bool bad = false;
  int t = 0;
  for (int t0 = 0; t0 < maxlen; t0 += kIdsPerLane * NP) {
    unsigned own[kIdsPerLane], lat[kIdsPerLane];
    uint32_t idv[kIdsPerLane];
#pragma unroll
    for (int s = 0; s < kIdsPerLane; ++s) {
      const int idx = t0 + s * NP + j;
      idv[s] = idx < len ? __ldg(ids + beg + idx) : 0xffffffffu;
    }
#pragma unroll
    for (int s = 0; s < kIdsPerLane; ++s) {
      const int idx = t0 + s * NP + j;
      own[s] = 0u;
      lat[s] = 0xffffffffu;  // past the row's end: no lane adds
      if (idx < len) {
        if (idv[s] < id_space) {
          const ulonglong2 m = __ldg(ol + idv[s]);
          own[s] = static_cast<unsigned>(m.x);
          lat[s] = static_cast<unsigned>(m.y);
        } else {
          bad = true;
        }
      }
    }
#pragma unroll
    for (int s = 0; s < kIdsPerLane; ++s) {
      for (int tt = 0; tt < NP; ++tt, ++t) {
        if (t >= maxlen) break;
        const unsigned O = __shfl_sync(0xffffffffu, own[s], tt, NP);
        const unsigned Lm = __shfl_sync(0xffffffffu, lat[s], tt, NP);
        const int p = __popc(O);
        const int pmax = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(p)));
        const bool has = (O >> j) & 1u;
        const int below = __popc(O & below_j);
        double* buf = mylist + (t & 1) * 32;
        buf[has ? below : p + (j - below)] = has ? uj : -0.0;
        __syncwarp();
        const bool active = cell && !((Lm >> j) & 1u);
        if (active) c = __dadd_rn(c, uj);  // miss pull over j's link
        for (int q = 0; q < pmax; q += 2) {  // one push per other owner, ascending
          const double2 v2 = *reinterpret_cast<const double2*>(buf + q);
          if (active) {
            c = __dadd_rn(c, v2.x);
            c = __dadd_rn(c, v2.y);
          }
        }
      }
    }
  }
  if (bad) atomicOr(flags + kFlagIdOutOfRange, 1);
  if (cell) matrix[i * n + j] = c;
  if (gap_keys == nullptr) return;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double s1 = cell ? c : inf, s2 = inf;
#pragma unroll
  for (int off = NP / 2; off > 0; off >>= 1) {
    const double b1 = __shfl_xor_sync(0xffffffffu, s1, off, NP);
    const double b2 = __shfl_xor_sync(0xffffffffu, s2, off, NP);
    const double lo = s1 < b1 ? s1 : b1, hi = s1 < b1 ? b1 : s1;
    const double m2 = s2 < b2 ? s2 : b2;
    s1 = lo;
    s2 = hi < m2 ? hi : m2;
  }
  if (rowok && j == 0) {
    gap_keys[i] = gap_sort_key(__dsub_rn(s2, s1));
    row_index[i] = static_cast<uint32_t>(i);
  }
}

// The pushes of one id, owners ascending: every lane of a group reads the
// same list (one broadcast 16-byte load feeds two adds of each of its cells)
// and a cell holding the latest copy skips the add; entries past the last
// owner hold -0.0.  A cell slot none of whose
// lanes lacks the latest copy (ids with many owners have few such cells) is
// skipped as a whole (ON0/ON1: warp-uniform).
template <int NC, bool ON0, bool ON1>
__device__ __forceinline__ void push_list(double (&c)[NC], const double* buf, int pmax,
                                          const bool (&act)[NC]) {
  constexpr bool kOn[2] = {ON0, ON1};
  // an unrolled ladder of 32 pairs entered at pair 32 - ceil(pmax / 2) (one
  // indirect branch per id, no loop counter); pairs past pmax hold -0.0
  const int skip = 32 - ((pmax + 1) >> 1);
  const double2* base = reinterpret_cast<const double2*>(buf) - skip;
#define EDX_PUSH_PAIR(k)                                  \
  case k: {                                               \
    const double2 v2 = base[k];                           \
    _Pragma("unroll") for (int h = 0; h < NC; ++h)        \
      if (kOn[h] && act[h]) {                             \
        c[h] = __dadd_rn(c[h], v2.x);                     \
        c[h] = __dadd_rn(c[h], v2.y);                     \
      }                                                   \
  }                                                       \
    [[fallthrough]];
  switch (skip) {
    EDX_PUSH_PAIR(0) EDX_PUSH_PAIR(1) EDX_PUSH_PAIR(2) EDX_PUSH_PAIR(3)
    EDX_PUSH_PAIR(4) EDX_PUSH_PAIR(5) EDX_PUSH_PAIR(6) EDX_PUSH_PAIR(7)
    EDX_PUSH_PAIR(8) EDX_PUSH_PAIR(9) EDX_PUSH_PAIR(10) EDX_PUSH_PAIR(11)
    EDX_PUSH_PAIR(12) EDX_PUSH_PAIR(13) EDX_PUSH_PAIR(14) EDX_PUSH_PAIR(15)
    EDX_PUSH_PAIR(16) EDX_PUSH_PAIR(17) EDX_PUSH_PAIR(18) EDX_PUSH_PAIR(19)
    EDX_PUSH_PAIR(20) EDX_PUSH_PAIR(21) EDX_PUSH_PAIR(22) EDX_PUSH_PAIR(23)
    EDX_PUSH_PAIR(24) EDX_PUSH_PAIR(25) EDX_PUSH_PAIR(26) EDX_PUSH_PAIR(27)
    EDX_PUSH_PAIR(28) EDX_PUSH_PAIR(29) EDX_PUSH_PAIR(30) EDX_PUSH_PAIR(31)
    default:
      break;
  }
#undef EDX_PUSH_PAIR
}

// K1 for 16 < n <= 64 (NP = 32: one row per warp; NP = 64: one row per warp,
// two cells per lane -- workers j and j + 32, two independent chains over the
// same lists).  A group of G = min(NP, 32) lanes
// loads G consecutive ids of its row (one per lane) and their masks; a ballot
// then drops every id whose latest copy is on all n workers (no cell adds
// anything: at steady state the hot ids -- 43% of occurrences at C4) and the
// group walks the remaining ids in row order.  An id without owners costs
// each non-latest cell one pull and needs no list; otherwise the group
// expands the id's owner-cost list into shared memory (owner o's u_o at
// position popc(owners below o), -0.0 at every other position), one
// __syncwarp, and the chains run over it in fully unrolled blocks of 8
// entries (one 16-byte broadcast load per 2 adds).  x + (-0.0) == x for every
// value these chains produce, so padding and the lanes holding the latest
// copy are exact no-ops: every cell's add sequence is the reference's.
template <int NP>
__global__ void __launch_bounds__(kWarpRowsThreads)
    k_cost_build_wide64(const uint32_t* __restrict__ ids, const uint64_t* __restrict__ offsets,
                      uint64_t rows, int n, const ulonglong2* __restrict__ ol, uint64_t id_space,
                      const double* __restrict__ ucost, double* __restrict__ matrix,
                      uint64_t* __restrict__ gap_keys, uint32_t* __restrict__ row_index,
                      int* __restrict__ flags) {
  constexpr int G = NP < 32 ? NP : 32;  // lanes per row
  constexpr int RPW = 32 / G;           // rows per warp
  constexpr int NC = NP / G;            // cells per lane (1 or 2)
  constexpr int NW = kWarpRowsThreads / 32;
  using M = typename std::conditional<(NP > 32), unsigned long long, unsigned>::type;
  // [warp][buffer][RPW groups x NP list entries]
  __shared__ __align__(16) double lists[NW][2][RPW * NP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / G, jl = lane - g * G;
  const uint64_t i = (static_cast<uint64_t>(blockIdx.x) * NW + warp) * RPW + g;
  const bool rowok = i < rows;
  int jw[NC];
  bool cell[NC];
  double uj[NC], c[NC];
  M jbit[NC], below_mask[NC];
#pragma unroll
  for (int h = 0; h < NC; ++h) {
    jw[h] = jl + 32 * h;
    cell[h] = rowok && jw[h] < n;
    uj[h] = jw[h] < n ? ucost[jw[h]] : 0.0;
    c[h] = 0.0;
    jbit[h] = M(1) << jw[h];
    below_mask[h] = jbit[h] - 1;
  }
  const M full = n >= static_cast<int>(8 * sizeof(M)) ? ~M(0) : ((M(1) << n) - 1);
  uint64_t beg = 0, end = 0;
  if (rowok) {
    beg = offsets[i];
    end = offsets[i + 1];
  }
  const int len = static_cast<int>(end - beg);
  const int maxlen = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(len));
  double* const mylist = &lists[warp][0][g * NP];
  const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
  bool bad = false;
  int par = 0;
  // software pipeline: ids two batches ahead, masks one batch ahead
  auto load_id = [&](int t0) -> uint32_t {
    const int idx = t0 + jl;
    return idx < len ? __ldg(ids + beg + idx) : 0xffffffffu;
  };
  auto load_masks = [&](int t0, uint32_t id, M& own, M& lat) {
    own = 0;
    lat = ~M(0);  // past the row's end: every worker "holds" it, nobody adds
    if (t0 + jl < len) {
      if (id < id_space) {
        const ulonglong2 m = __ldg(ol + id);
        own = static_cast<M>(m.x);
        lat = static_cast<M>(m.y);
      } else {
        bad = true;
      }
    }
  };
  uint32_t id_next = load_id(G);
  M own_n, lat_n;
  load_masks(0, load_id(0), own_n, lat_n);
  for (int t0 = 0; t0 < maxlen; t0 += G) {
    const M own = own_n, lat = lat_n;
    if (t0 + G < maxlen) {
      const uint32_t id1 = id_next;
      id_next = load_id(t0 + 2 * G);
      load_masks(t0 + G, id1, own_n, lat_n);
    }
    // ids some worker of its row lacks, slot-aligned over the warp's groups
    unsigned todo = __ballot_sync(0xffffffffu, (lat & full) != full);
    unsigned owned = __ballot_sync(0xffffffffu, own != 0);  // ids with a push list
    if constexpr (RPW == 2) {
      todo = (todo | (todo >> 16)) & gmask;
      owned = (owned | (owned >> 16)) & gmask;
    }
    while (todo) {
      const int s = __ffs(todo) - 1;
      todo &= todo - 1;
      const M Lm = __shfl_sync(0xffffffffu, lat, s, G);
      bool act[NC];
#pragma unroll
      for (int h = 0; h < NC; ++h) act[h] = cell[h] && !(Lm & jbit[h]);
      if (!((owned >> s) & 1u)) {  // no owners: one pull per non-latest cell
#pragma unroll
        for (int h = 0; h < NC; ++h)
          if (act[h]) c[h] = __dadd_rn(c[h], uj[h]);
        continue;
      }
      const M O = __shfl_sync(0xffffffffu, own, s, G);
      const int p = popc_mask(O);
      const int pmax = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(p)));
      double* buf = mylist + par * (RPW * NP);
      par ^= 1;
#pragma unroll
      for (int h = 0; h < NC; ++h) {
        const bool has = (O & jbit[h]) != 0;
        const int below = popc_mask(O & below_mask[h]);
        buf[has ? below : p + (jw[h] - below)] = has ? uj[h] : -0.0;
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < NC; ++h)
        if (act[h]) c[h] = __dadd_rn(c[h], uj[h]);  // miss pull
      if constexpr (NC == 2) {
        const bool a0 = __any_sync(0xffffffffu, act[0]), a1 = __any_sync(0xffffffffu, act[1]);
        if (a0 && a1) push_list<NC, true, true>(c, buf, pmax, act);
        else if (a0) push_list<NC, true, false>(c, buf, pmax, act);
        else push_list<NC, false, true>(c, buf, pmax, act);
      } else {
        push_list<NC, true, false>(c, buf, pmax, act);
      }
    }
  }
  if (bad) atomicOr(flags + kFlagIdOutOfRange, 1);
#pragma unroll
  for (int h = 0; h < NC; ++h)
    if (cell[h]) matrix[i * n + jw[h]] = c[h];
  if (gap_keys == nullptr) return;
  // two smallest of the row with multiplicity (row_gap_key, cost.hpp:130-146)
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double s1 = cell[0] ? c[0] : inf, s2 = inf;
  if constexpr (NC == 2) {
    const double b = cell[1] ? c[1] : inf;
    const double lo = s1 < b ? s1 : b, hi = s1 < b ? b : s1;
    s1 = lo;
    s2 = hi;
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    const double b1 = __shfl_xor_sync(0xffffffffu, s1, off, G);
    const double b2 = __shfl_xor_sync(0xffffffffu, s2, off, G);
    const double lo = s1 < b1 ? s1 : b1, hi = s1 < b1 ? b1 : s1;
    const double m2 = s2 < b2 ? s2 : b2;
    s1 = lo;
    s2 = hi < m2 ? hi : m2;
  }
  if (rowok && jl == 0) {
    gap_keys[i] = gap_sort_key(__dsub_rn(s2, s1));
    row_index[i] = static_cast<uint32_t>(i);
  }
}

__global__ void k_gap_keys(const double* __restrict__ matrix, uint64_t rows, int n,
                           uint64_t* __restrict__ gap_keys, uint32_t* __restrict__ row_index) {
  const uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  gap_keys[r] = gap_sort_key(row_gap(matrix + r * n, n));
  row_index[r] = static_cast<uint32_t>(r);
}

}  // namespace

void launch_cost_build(const uint32_t* ids, const uint64_t* offsets, uint64_t rows, int n,
                       const ulonglong2* ol, uint64_t id_space, const double* ucost,
                       double* matrix, uint64_t* gap_keys, uint32_t* row_index, int* flags,
                       cudaStream_t s, const uint64_t* sizes, const double* bw) {
  if (rows == 0) return;
  if (n >= 2 && sizes == nullptr) {
    const int np = n <= 2 ? 2 : n <= 4 ? 4 : n <= 8 ? 8 : n <= 16 ? 16 : n <= 32 ? 32 : 64;
    const uint64_t rows_per_block = static_cast<uint64_t>(kWarpRowsThreads / 32) * (np >= 32 ? 1 : 32 / np);
    const unsigned blocks = static_cast<unsigned>((rows + rows_per_block - 1) / rows_per_block);
    auto go = [&](auto kern) {
      kern<<<blocks, kWarpRowsThreads, 0, s>>>(ids, offsets, rows, n, ol, id_space, ucost, matrix,
                                               gap_keys, row_index, flags);
    };
    switch (np) {
      case 2: go(k_cost_build_warp<2>); g_kernel_name[kKBuild] = "k_cost_build_warp<2>"; break;
      case 4: go(k_cost_build_warp<4>); g_kernel_name[kKBuild] = "k_cost_build_warp<4>"; break;
      case 8: go(k_cost_build_warp<8>); g_kernel_name[kKBuild] = "k_cost_build_warp<8>"; break;
      // 16 workers: lockstep over every id (C3: 1.7 us faster than the skip
      // kernel at 8,192 rows); above: all-latest ids skipped by ballot
      case 16: go(k_cost_build_wide<16>); g_kernel_name[kKBuild] = "k_cost_build_wide<16>"; break;
      case 32: go(k_cost_build_wide64<32>); g_kernel_name[kKBuild] = "k_cost_build_wide64<32>"; break;
      default: go(k_cost_build_wide64<64>); g_kernel_name[kKBuild] = "k_cost_build_wide64<64>"; break;
    }
    EDX_LAUNCHED();
    return;
  }
  // n == 1 or per-id sizes: one thread per cell
  const int rows_per_block = n >= kBlockCells ? 1 : kBlockCells / n;
  const int threads = rows_per_block * n;
  const uint64_t blocks = (rows + rows_per_block - 1) / rows_per_block;
  k_cost_build<<<static_cast<unsigned>(blocks), threads, 0, s>>>(
      ids, offsets, rows, n, rows_per_block, ol, id_space, ucost, sizes, bw, matrix, gap_keys,
      row_index, flags);
  EDX_LAUNCHED();
  g_kernel_name[kKBuild] = "k_cost_build";
}

void launch_gap_keys(const double* matrix, uint64_t rows, int n, uint64_t* gap_keys,
                     uint32_t* row_index, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((rows + 255) / 256);
  k_gap_keys<<<blocks, 256, 0, s>>>(matrix, rows, n, gap_keys, row_index);
  EDX_LAUNCHED();
}

}  // namespace edx
