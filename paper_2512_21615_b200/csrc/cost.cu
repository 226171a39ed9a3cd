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
                 double* __restrict__ matrix, uint64_t* __restrict__ gap_keys,
                 uint32_t* __restrict__ row_index, int* __restrict__ flags) {
  __shared__ double u_s[kMaxWorkers];
  __shared__ double tile[kBlockCells];
  if (threadIdx.x < n) u_s[threadIdx.x] = ucost[threadIdx.x];
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
    for (uint64_t t = beg; t < end; t += kPrefetch) {
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
                       cudaStream_t s) {
  const int rows_per_block = n >= kBlockCells ? 1 : kBlockCells / n;
  const int threads = rows_per_block * n;
  const uint64_t blocks = (rows + rows_per_block - 1) / rows_per_block;
  k_cost_build<<<static_cast<unsigned>(blocks), threads, 0, s>>>(
      ids, offsets, rows, n, rows_per_block, ol, id_space, ucost, matrix, gap_keys, row_index,
      flags);
  EDX_LAUNCHED();
}

void launch_gap_keys(const double* matrix, uint64_t rows, int n, uint64_t* gap_keys,
                     uint32_t* row_index, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((rows + 255) / 256);
  k_gap_keys<<<blocks, 256, 0, s>>>(matrix, rows, n, gap_keys, row_index);
  EDX_LAUNCHED();
}

}  // namespace edx
