// K6 block-collapsed e-maxx Hungarian (EcoMix exact block) and K5 dense
// e-maxx Hungarian (the general hungarian() API).
//
// Reference: hungarian (assign.hpp:80-157).  Costs are scaled to int64 by
// llround(v * 1e12) and capped at INT64_MAX / (8 (k+1)); rows are inserted
// 1..k in order; each Dijkstra step relaxes the unused columns from the row
// just reached (strict '<' keeps the earliest way) and picks the unused
// column of least minv (strict '<' over ascending j: lowest index on ties);
// potentials then move by delta.  An equal-cost re-solve moves rows
// (SURVEY §0 hazard 3), so both kernels execute this exact algorithm, step
// for step, in int64.
//
// K6 exploits the structure ecomix feeds the solver (expand_columns,
// assign.hpp:223-241): columns [w*mult, (w+1)*mult) repeat worker w's cost.
// Within one row's search v[j] of an unused column never changes (only used
// columns' potentials move), and every unused column of block w is relaxed
// by the same a[i0][w] - u[i0].  Writing Δ for the running sum of the
// step's deltas, every unused j in block w therefore has
//     minv[j] = D_w - Δ - v[j],   D_w = min over reached rows (a[r][w] - u[r] + Δ_r)
// with one shared way_w.  The block's least-minv column is its unused column
// of largest v (lowest index on ties), blocks are index-ordered, so the global
// argmin is a per-block candidate argmin, and the per-step cost is O(n)
// instead of O(k).  The potential moves of used columns are applied lazily at
// the end of the row from Δ at the time each column was reached, which is
// exact in int64.  Each block keeps its columns sorted by (v desc, j asc);
// within a row the chosen columns are a prefix of that order (a cursor), and
// at row end only that prefix changes key and is merged back.
//
// K6 runs on ONE warp of one SM: lane w owns block w (n <= 64, two blocks per
// lane above 32).  It is latency-bound by construction (one dependent
// Dijkstra step after another); state lives in shared memory when it fits.
#include <algorithm>
#include <climits>
#include <cmath>

#include "edx_internal.cuh"

#include <cstdlib>
#include <cstring>

namespace edx {

namespace {

constexpr int64_t kInf = LLONG_MAX;

// std::llround(x * 1e12) then std::min(., cap) as compiled for x86-64/glibc
// (assign.hpp:96-100): round half away from zero; out-of-range -> INT64_MIN.
__device__ __forceinline__ int64_t scale_cost(double x, int64_t cap) {
  const double y = __dmul_rn(x, 1e12);
  int64_t s;
  if (!(y < 9223372036854775808.0)) {
    s = LLONG_MIN;
  } else {
    const long long t = __double2ll_rz(y);
    const double f = __dsub_rn(y, __ll2double_rn(t));
    s = t + (f >= 0.5 ? 1 : 0);
  }
  return s < cap ? s : cap;
}

__device__ __forceinline__ bool bad_cost(double x) { return !isfinite(x) || x < 0.0; }

__device__ __forceinline__ size_t dynamic_smem_bytes() {
  unsigned v;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}

// S[r][w] = scaled cost of block row r (matrix row order[r]) for worker w.
__global__ void k_scale_block(const double* __restrict__ matrix, int n,
                              const uint32_t* __restrict__ order, uint64_t k, int64_t cap,
                              int64_t* __restrict__ S, int* __restrict__ flags,
                              unsigned long long* __restrict__ max_scaled) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  unsigned long long sv = 0;
  if (x < k * n) {
    const uint64_t r = x / n, w = x - r * n;
    const double v = matrix[static_cast<uint64_t>(order[r]) * n + w];
    if (bad_cost(v)) atomicOr(flags + kFlagBadCost, 1);
    const int64_t sc = scale_cost(v, cap);
    S[x] = sc;
    sv = sc < 0 ? ~0ULL : static_cast<unsigned long long>(sc);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ov = __shfl_xor_sync(0xffffffffu, sv, o);
    sv = ov > sv ? ov : sv;
  }
  if ((threadIdx.x & 31) == 0 && sv) atomicMax(max_scaled, sv);
}

struct BlockArrays {
  const int64_t* S;  // k x n
  int64_t *u, *v, *dlt;
  int32_t *p, *way, *ulist, *ord, *tmp;
};

// (v desc, j asc): does column a come before column b in its block's order?
__device__ __forceinline__ bool before(const int64_t* v, int a, int b) {
  const int64_t va = v[a], vb = v[b];
  return va > vb || (va == vb && a < b);
}

template <int NB>
__device__ bool hungarian_blocks_warp(const BlockArrays A, int n, int mult, int k,
                                      unsigned long long* steps_out, int* flags) {
  const int lane = threadIdx.x & 31;
  const int64_t* __restrict__ S = A.S;
  int64_t* __restrict__ u = A.u;
  int64_t* __restrict__ v = A.v;
  int64_t* __restrict__ dlt = A.dlt;
  int32_t* __restrict__ p = A.p;
  int32_t* __restrict__ way = A.way;
  int32_t* __restrict__ ulist = A.ulist;
  int32_t* __restrict__ ord = A.ord;
  int32_t* __restrict__ tmp = A.tmp;

  for (int x = lane; x <= k; x += 32) {
    u[x] = 0;
    v[x] = 0;
    p[x] = 0;
    way[x] = 0;
  }
  for (int x = lane; x < k; x += 32) ord[x] = x + 1;  // v all 0: index order
  __syncwarp();

  unsigned long long steps = 0;
  long long c_step = 0, c_pot = 0, c_aug = 0, c_rekey = 0, hops = 0, prefix = 0;
  const long long c_start = clock64();
  int64_t D[NB], bestv[NB];
  int wy[NB], cur[NB], bestc[NB];

  for (int i = 1; i <= k; ++i) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int w = lane + 32 * b;
      D[b] = kInf;
      wy[b] = 0;
      cur[b] = 0;
      if (w < n) {
        bestc[b] = ord[w * mult];
        bestv[b] = v[bestc[b]];
      } else {
        bestc[b] = 0;
        bestv[b] = 0;
      }
    }
    if (lane == 0) {
      p[0] = i;
      ulist[0] = 0;
      dlt[0] = 0;
    }
    int nused = 1;
    int j0 = 0, r = i, j1;
    int64_t Dl = 0;  // Δ: running sum of this row's deltas
    __syncwarp();
    long long t0 = clock64();
    for (;;) {
      ++steps;
      const int64_t ur = u[r];
      const int64_t* __restrict__ Srow = S + static_cast<int64_t>(r - 1) * n;
      int64_t bv = kInf;
      int bw = INT_MAX;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int w = lane + 32 * b;
        if (w < n && cur[b] < mult) {
          const int64_t c = Srow[w] - ur + Dl;  // = cur + v[j] + Δ for every unused j of w
          if (c < D[b]) {
            D[b] = c;
            wy[b] = j0;
          }
          const int64_t val = D[b] - Dl - bestv[b];  // minv of the block's best column
          if (val < bv) {
            bv = val;
            bw = w;
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const int64_t ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int ow = __shfl_xor_sync(0xffffffffu, bw, off);
        if (ov < bv || (ov == bv && ow < bw)) {
          bv = ov;
          bw = ow;
        }
      }
      if (bw == INT_MAX) {  // no unused column: only reachable on corrupt input
        if (lane == 0) atomicOr(flags + kFlagBadCost, 1);
        return false;
      }
      const int owner = bw & 31, ob = bw >> 5;
      int mine = bestc[0];
#pragma unroll
      for (int b = 1; b < NB; ++b)
        if (ob == b) mine = bestc[b];
      j1 = __shfl_sync(0xffffffffu, mine, owner);
      Dl += bv;
      if (lane == owner) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          if (b != ob) continue;
          way[j1] = wy[b];
          dlt[j1] = Dl;
          ++cur[b];
          if (cur[b] < mult) {
            bestc[b] = ord[bw * mult + cur[b]];
            bestv[b] = v[bestc[b]];
          }
        }
      }
      if (lane == 0) ulist[nused] = j1;
      ++nused;
      __syncwarp();
      const int pj = p[j1];
      if (pj == 0) break;
      j0 = j1;
      r = pj;
    }
    long long t1 = clock64();
    c_step += t1 - t0;
    // lazy potential moves (assign.hpp:131-138 applied per reached column)
    for (int t = lane; t < nused; t += 32) {
      const int j = ulist[t];
      const int64_t d = Dl - dlt[j];
      u[p[j]] += d;
      v[j] -= d;
    }
    __syncwarp();
    long long t2 = clock64();
    c_pot += t2 - t1;
    if (lane == 0) {  // augment along way[] (assign.hpp:141-145)
      int jj = j1;
      do {
        const int jp = way[jj];
        p[jj] = p[jp];
        jj = jp;
        ++hops;
      } while (jj != 0);
    }
    __syncwarp();
    long long t3 = clock64();
    c_aug += t3 - t2;
    // re-key the consumed prefix of every touched block
    const long long t4 = clock64();
    for (int w = 0; w < n; ++w) {
      int P = 0;
#pragma unroll
      for (int b = 0; b < NB; ++b)
        if ((w >> 5) == b) P = __shfl_sync(0xffffffffu, cur[b], w & 31);
      if (P == 0) continue;
      prefix += P;
      int32_t* base = ord + w * mult;
      int32_t* sorted = tmp;         // P entries
      int32_t* merged = tmp + mult;  // mult entries
      __syncwarp();
      for (int t = lane; t < P; t += 32) {
        const int a = base[t];
        int rank = 0;
        for (int s2 = 0; s2 < P; ++s2) rank += before(v, base[s2], a) ? 1 : 0;
        sorted[rank] = a;
      }
      __syncwarp();
      const int Q = mult - P;
      const int32_t* suf = base + P;
      for (int t = lane; t < P; t += 32) {
        const int a = sorted[t];
        int lo = 0, hi = Q;  // # suffix entries before a
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (before(v, suf[mid], a)) lo = mid + 1;
          else hi = mid;
        }
        merged[t + lo] = a;
      }
      for (int t = lane; t < Q; t += 32) {
        const int b2 = suf[t];
        int lo = 0, hi = P;  // # prefix entries before b2
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (before(v, sorted[mid], b2)) lo = mid + 1;
          else hi = mid;
        }
        merged[t + lo] = b2;
      }
      __syncwarp();
      for (int t = lane; t < mult; t += 32) base[t] = merged[t];
      __syncwarp();
    }
    c_rekey += clock64() - t4;
  }
  if (lane == 0 && steps_out) {
    steps_out[0] = steps;
    steps_out[1] = c_step;
    steps_out[2] = c_pot;
    steps_out[3] = c_aug;
    steps_out[4] = c_rekey;
    steps_out[5] = hops;
    steps_out[6] = prefix;
    steps_out[7] = clock64() - c_start;
  }
  return true;
}

template <int NB>
__global__ void __launch_bounds__(32)
    k_hungarian_blocks_wide(const int64_t* __restrict__ S_global, int n, int mult, int k,
                       int s_in_smem, uint8_t* __restrict__ arena,
                       const uint32_t* __restrict__ order, int32_t* __restrict__ decision,
                       const uint32_t* __restrict__ row_ids, uint64_t* __restrict__ col_of_row,
                       unsigned long long* steps_out, int* flags) {
  extern __shared__ __align__(16) uint8_t smem[];
  const size_t K1 = static_cast<size_t>(k) + 1;
  const size_t s_bytes = (static_cast<size_t>(k) * n * sizeof(int64_t) + 15) & ~size_t(15);
  // [S | arrays] in shared memory, or S in global with the arrays in shared
  // memory, or both in global memory (L2) when even the arrays do not fit.
  uint8_t* abase = arena ? arena : smem + (s_in_smem ? s_bytes : 0);
  int64_t* S_s = reinterpret_cast<int64_t*>(smem);
  size_t off = 0;
  BlockArrays A;
  auto take = [&](size_t bytes) {
    uint8_t* q = abase + off;
    off += (bytes + 15) & ~size_t(15);
    return q;
  };
  A.u = reinterpret_cast<int64_t*>(take(K1 * 8));
  A.v = reinterpret_cast<int64_t*>(take(K1 * 8));
  A.dlt = reinterpret_cast<int64_t*>(take(K1 * 8));
  A.p = reinterpret_cast<int32_t*>(take(K1 * 4));
  A.way = reinterpret_cast<int32_t*>(take(K1 * 4));
  A.ulist = reinterpret_cast<int32_t*>(take(K1 * 4));
  A.ord = reinterpret_cast<int32_t*>(take(static_cast<size_t>(k) * 4));
  A.tmp = reinterpret_cast<int32_t*>(take(static_cast<size_t>(2 * mult) * 4));
  if (s_in_smem) {
    const int4* src = reinterpret_cast<const int4*>(S_global);
    int4* dst = reinterpret_cast<int4*>(S_s);
    const size_t n16 = static_cast<size_t>(k) * n / 2;  // k*n int64 = k*n/2 int4
    for (size_t x = threadIdx.x; x < n16; x += 32) dst[x] = src[x];
    if ((static_cast<size_t>(k) * n) & 1) {
      if (threadIdx.x == 0) S_s[static_cast<size_t>(k) * n - 1] = S_global[static_cast<size_t>(k) * n - 1];
    }
    __syncwarp();
    A.S = S_s;
  } else {
    A.S = S_global;
  }
  if (!hungarian_blocks_warp<NB>(A, n, mult, k, steps_out, flags)) return;
  __syncwarp();
  // p[j] = block row matched to column j (1-based); column j -> worker (j-1)/mult
  for (int j = threadIdx.x + 1; j <= k; j += 32) {
    const int r = A.p[j] - 1;
    if (col_of_row) col_of_row[r] = static_cast<uint64_t>(j - 1);
    if (decision) {
      const uint32_t row = order[r];
      decision[row_ids ? row_ids[row] : row] = (j - 1) / mult;
    }
  }
}

// ------------------------------------------------------ K6 fast (packed keys)
// Same algorithm as k_hungarian_blocks_wide, organised for the latency of one
// Dijkstra step on a B200 SM (measured: LDS 29 cycles, SHFL 26, REDUX 22):
//  * every array is addressed through __shared__ (LDS/STS, no generic loads);
//  * a block's minv key is packed as (minv << 6 | w) and the warp argmin is
//    two redux.sync.min.u32 (high word, then low word among the minima); the
//    block index in the low bits makes the lowest block win ties, i.e. the
//    lowest column (blocks are index-ordered);
//  * E_w = D_w - Δ is kept pre-shifted, so a step's relax is
//    E_w = min(E_w - delta, A_w(r)) with A_w(r) = (S[r][w] - u[r]) << 6
//    staged in shared memory for every block's current candidate row;
//    the only load on the step's critical path is the winner's A;
//  * `way` is recorded as the index (in the row's list of reached columns)
//    of the column whose row last improved the block, so no shuffle is
//    needed to broadcast it;
//  * at the end of a row, potentials and the (v desc, j asc) re-keying of
//    every touched block run on all warps (one block per warp) while one
//    thread augments.
// Packing needs 0 <= minv < 2^57; the launcher checks the cost range and
// falls back to the wide kernel otherwise.
constexpr int kFastMaxWarps = 16;

template <int NB, int MODE>  // MODE 0: S + arrays shared; 1: S global; 2: S + arrays global
__global__ void __launch_bounds__(kFastMaxWarps * 32, 1)
    k_hungarian_blocks_fast(const int64_t* __restrict__ S_global, int n, int mult, int k,
                            uint8_t* __restrict__ arena, const uint32_t* __restrict__ order,
                            int32_t* __restrict__ decision, const uint32_t* __restrict__ row_ids,
                            uint64_t* __restrict__ col_of_row, unsigned long long* stats,
                            int* flags, const unsigned long long* __restrict__ max_scaled) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  constexpr int W = 32 * NB;
  // Packed keys need minv < 2^57; reduced costs stay below (k+1) * max cost
  // (the reference's own overflow budget, assign.hpp:93-94).
  const unsigned long long mx = *max_scaled;
  const bool packable = mx < (1ULL << 57) / (8ULL * static_cast<unsigned long long>(k + 1));  // row stride of the A staging
  const size_t K1 = static_cast<size_t>(k) + 1;
  size_t so = 0, go = 0;
  auto stake = [&](size_t bytes) {
    uint8_t* q = smem + so;
    so += (bytes + 15) & ~size_t(15);
    return q;
  };
  auto gtake = [&](size_t bytes) {
    uint8_t* q = arena + go;
    go += (bytes + 15) & ~size_t(15);
    return q;
  };
  const int64_t* S;
  int64_t *u, *v, *dlt;
  int32_t *p, *way, *ulist, *ord;
  if constexpr (MODE == 0) {
    int64_t* Ss = reinterpret_cast<int64_t*>(stake(static_cast<size_t>(k) * n * 8));
    const size_t total = static_cast<size_t>(k) * n;
    for (size_t x = tid; x < total; x += blockDim.x) Ss[x] = S_global[x];
    S = Ss;
  } else {
    S = S_global;
  }
  if constexpr (MODE <= 1) {
    u = reinterpret_cast<int64_t*>(stake(K1 * 8));
    v = reinterpret_cast<int64_t*>(stake(K1 * 8));
    dlt = reinterpret_cast<int64_t*>(stake(K1 * 8));
    p = reinterpret_cast<int32_t*>(stake(K1 * 4));
    way = reinterpret_cast<int32_t*>(stake(K1 * 4));
    ulist = reinterpret_cast<int32_t*>(stake(K1 * 4));
    ord = reinterpret_cast<int32_t*>(stake(static_cast<size_t>(k) * 4));
  } else {
    u = reinterpret_cast<int64_t*>(gtake(K1 * 8));
    v = reinterpret_cast<int64_t*>(gtake(K1 * 8));
    dlt = reinterpret_cast<int64_t*>(gtake(K1 * 8));
    p = reinterpret_cast<int32_t*>(gtake(K1 * 4));
    way = reinterpret_cast<int32_t*>(gtake(K1 * 4));
    ulist = reinterpret_cast<int32_t*>(gtake(K1 * 4));
    ord = reinterpret_cast<int32_t*>(gtake(static_cast<size_t>(k) * 4));
  }
  int64_t* A6 = reinterpret_cast<int64_t*>(stake(static_cast<size_t>(n) * W * 8));
  int32_t* cand_r = reinterpret_cast<int32_t*>(stake(64 * 4));
  int32_t* cur_s = reinterpret_cast<int32_t*>(stake(64 * 4));
  int64_t* scal = reinterpret_cast<int64_t*>(stake(4 * 8));  // Dl, nused, abort
  int64_t* rk_v = reinterpret_cast<int64_t*>(stake(static_cast<size_t>(nw) * mult * 8));
  int32_t* rk_i = reinterpret_cast<int32_t*>(stake(static_cast<size_t>(nw) * 2 * mult * 4));
  if (so > dynamic_smem_bytes()) {  // host/device layout mismatch: fail loudly, touch nothing
    if (tid == 0) atomicOr(flags + kFlagInternal, 1);
    return;
  }

  for (size_t x = tid; x < K1; x += blockDim.x) {
    u[x] = 0;
    v[x] = 0;
    p[x] = 0;
    way[x] = 0;
  }
  for (int x = tid; x < k; x += blockDim.x) ord[x] = x + 1;  // all v = 0: index order
  if (tid == 0) scal[2] = 0;
  __syncthreads();

  if (!packable) {  // wide-range path: the 64-bit (value, index) shuffle argmin
    if (warp == 0) {
      BlockArrays A{S, u, v, dlt, p, way, ulist, ord, rk_i};
      if (!hungarian_blocks_warp<NB>(A, n, mult, k, stats, flags)) return;
      __syncwarp();
      for (int j = lane + 1; j <= k; j += 32) {
        const int r = p[j] - 1;
        if (col_of_row) col_of_row[r] = static_cast<uint64_t>(j - 1);
        if (decision) {
          const uint32_t row = order[r];
          decision[row_ids ? row_ids[row] : row] = (j - 1) / mult;
        }
      }
    }
    return;
  }

  unsigned long long steps = 0;
  long long c_step = 0, c_end = 0, rekeyed = 0;
  const long long c_start = clock64();
  for (int i = 1; i <= k; ++i) {
    const long long t0 = clock64();
    if (warp == 0) {
      int64_t E6[NB], B[NB];
      int wyi[NB], cur[NB], bestc[NB];
      const int64_t ui = u[i];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int w = lane + 32 * b;
        cur[b] = 0;
        wyi[b] = 0;
        E6[b] = 0;
        B[b] = 0;
        bestc[b] = 0;
        if (w < n) {
          const int c = ord[w * mult];
          bestc[b] = c;
          B[b] = static_cast<int64_t>(w) - (v[c] << 6);
          cand_r[w] = p[c];
          // relax from row i (reached through the virtual column 0, Δ = 0)
          E6[b] = (S[static_cast<size_t>(i - 1) * n + w] - ui) << 6;
        }
      }
      if (lane == 0) {
        p[0] = i;
        ulist[0] = 0;
        dlt[0] = 0;
      }
      __syncwarp();
      for (int x = 0; x < n; ++x) {  // stage every block's candidate row
        const int r = cand_r[x];
        if (r > 0) {
          const int64_t ur = u[r];
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const int w = lane + 32 * b;
            if (w < n) A6[x * W + w] = (S[static_cast<size_t>(r - 1) * n + w] - ur) << 6;
          }
        }
      }
      int nused = 1, pw = -1;
      int64_t Dl = 0;
      bool abort = false;
      for (;;) {
        ++steps;
        if (pw >= 0) {  // the previous winner block moved to a new candidate: restage it
          const int r = cand_r[pw];
          if (r > 0) {
            const int64_t ur = u[r];
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              const int w = lane + 32 * b;
              if (w < n) A6[pw * W + w] = (S[static_cast<size_t>(r - 1) * n + w] - ur) << 6;
            }
          }
        }
        uint64_t key = ~0ULL;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int w = lane + 32 * b;
          if (w < n && cur[b] < mult) {
            const uint64_t kb = static_cast<uint64_t>(E6[b] + B[b]);
            key = kb < key ? kb : key;
          }
        }
        const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
        const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
        const uint64_t kmin = (static_cast<uint64_t>(mh) << 32) | ml;
        if (kmin == ~0ULL) {  // no unused column: only reachable on corrupt input
          abort = true;
          break;
        }
        const int ws = static_cast<int>(ml & 63u);
        const int64_t delta6 = static_cast<int64_t>(kmin & ~63ULL);
        Dl += delta6 >> 6;
        const int r = cand_r[ws];
        int64_t a[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) a[b] = A6[ws * W + lane + 32 * b];
        __syncwarp();  // cand_r[ws] read by all lanes before its owner moves on
        const int owner = ws & 31, ob = ws >> 5;
        if (lane == owner) {
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if (b != ob) continue;
            const int j1 = bestc[b];
            way[j1] = ulist[wyi[b]];
            dlt[j1] = Dl;
            ulist[nused] = j1;
            if (++cur[b] < mult) {
              const int c = ord[ws * mult + cur[b]];
              bestc[b] = c;
              B[b] = static_cast<int64_t>(ws) - (v[c] << 6);
              cand_r[ws] = p[c];
            }
          }
        }
        const int s_cur = nused++;
        if (r == 0) break;  // a free column: the augmenting path ends here
#pragma unroll
        for (int b = 0; b < NB; ++b) {  // relax from row r (assign.hpp:119-125)
          const int64_t t = E6[b] - delta6;
          if (a[b] < t) {
            E6[b] = a[b];
            wyi[b] = s_cur;
          } else {
            E6[b] = t;
          }
        }
        __syncwarp();
        pw = ws;
      }
      if (lane == 0) {
        scal[0] = Dl;
        scal[1] = nused;
        if (abort) scal[2] = 1;
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int w = lane + 32 * b;
        if (w < n) cur_s[w] = cur[b];
      }
    }
    __syncthreads();
    const long long t1 = clock64();
    c_step += t1 - t0;
    if (scal[2]) {
      if (tid == 0) atomicOr(flags + kFlagBadCost, 1);
      return;
    }
    const int64_t Dl = scal[0];
    const int nu = static_cast<int>(scal[1]);
    for (int t = tid; t < nu; t += blockDim.x) {  // potentials (assign.hpp:131-138), lazily
      const int j = ulist[t];
      const int64_t d = Dl - dlt[j];
      u[p[j]] += d;
      v[j] -= d;
    }
    __syncthreads();
    if (tid == 0) {  // augment (assign.hpp:141-145)
      int jj = ulist[nu - 1];
      do {
        const int jp = way[jj];
        p[jj] = p[jp];
        jj = jp;
      } while (jj != 0);
    }
    // re-key each touched block's consumed prefix (v changed), one block per warp
    for (int w = warp; w < n; w += nw) {
      const int P = cur_s[w];
      if (P == 0) continue;
      if (lane == 0) rekeyed += P;
      int32_t* base = ord + w * mult;
      int64_t* pv = rk_v + static_cast<size_t>(warp) * mult;
      int32_t* sorted = rk_i + static_cast<size_t>(warp) * 2 * mult;
      int32_t* merged = sorted + mult;
      for (int t = lane; t < P; t += 32) pv[t] = v[base[t]];
      __syncwarp();
      for (int t = lane; t < P; t += 32) {
        const int a = base[t];
        const int64_t va = pv[t];
        int rank = 0;
        for (int s2 = 0; s2 < P; ++s2) {
          const int64_t vb = pv[s2];
          rank += (vb > va || (vb == va && base[s2] < a)) ? 1 : 0;
        }
        sorted[rank] = a;
      }
      __syncwarp();
      const int Q = mult - P;
      const int32_t* suf = base + P;
      for (int t = lane; t < P; t += 32) {
        const int a = sorted[t];
        const int64_t va = v[a];
        int lo2 = 0, hi2 = Q;  // suffix entries ordered before a
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          const int b2 = suf[mid];
          const int64_t vb = v[b2];
          if (vb > va || (vb == va && b2 < a)) lo2 = mid + 1;
          else hi2 = mid;
        }
        merged[t + lo2] = a;
      }
      for (int t = lane; t < Q; t += 32) {
        const int b2 = suf[t];
        const int64_t vb = v[b2];
        int lo2 = 0, hi2 = P;  // prefix entries ordered before b2
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          const int a = sorted[mid];
          const int64_t va = v[a];
          if (va > vb || (va == vb && a < b2)) lo2 = mid + 1;
          else hi2 = mid;
        }
        merged[t + lo2] = b2;
      }
      __syncwarp();
      for (int t = lane; t < mult; t += 32) base[t] = merged[t];
      __syncwarp();
    }
    __syncthreads();
    c_end += clock64() - t1;
  }
  for (int j = tid + 1; j <= k; j += blockDim.x) {
    const int r = p[j] - 1;
    if (col_of_row) col_of_row[r] = static_cast<uint64_t>(j - 1);
    if (decision) {
      const uint32_t row = order[r];
      decision[row_ids ? row_ids[row] : row] = (j - 1) / mult;
    }
  }
  if (tid == 0 && stats) {
    stats[0] = steps;
    stats[1] = c_step;
    stats[2] = c_end;
    stats[3] = 0;
    stats[4] = 0;
    stats[5] = 0;
    stats[6] = rekeyed;
    stats[7] = clock64() - c_start;
  }
}

// Warp-wide bitonic sort of 32*E (hi, lo) keys held in registers, element
// index i = e*32 + lane, ascending by (hi, lo).  Used to re-sort a block's
// columns by (v desc, j asc) = ascending (-v, j) at the end of a row.
template <int E>
__device__ __forceinline__ void warp_bitonic_sort(int64_t (&hi)[E], int32_t (&lo)[E], int lane) {
  constexpr int M = 32 * E;
#pragma unroll
  for (int size = 2; size <= M; size <<= 1) {
#pragma unroll
    for (int d = size >> 1; d > 0; d >>= 1) {
      if (d >= 32) {
        const int de = d >> 5;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int pe = e ^ de;
          if (pe > e) {
            const bool asc = ((e * 32 + lane) & size) == 0;
            const bool gt = hi[e] > hi[pe] || (hi[e] == hi[pe] && lo[e] > lo[pe]);
            if (gt == asc) {
              const int64_t th = hi[e];
              const int32_t tl = lo[e];
              hi[e] = hi[pe];
              lo[e] = lo[pe];
              hi[pe] = th;
              lo[pe] = tl;
            }
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int64_t oh = __shfl_xor_sync(0xffffffffu, hi[e], d);
          const int32_t ol = __shfl_xor_sync(0xffffffffu, lo[e], d);
          const bool asc = ((e * 32 + lane) & size) == 0;
          const bool lower = (lane & d) == 0;
          const bool other_less = oh < hi[e] || (oh == hi[e] && ol < lo[e]);
          if ((lower == asc) ? other_less : !other_less) {
            hi[e] = oh;
            lo[e] = ol;
          }
        }
      }
    }
  }
}

// Re-sorts ord[base .. base+mult) by (v desc, j asc) with one warp.
template <int E>
__device__ __forceinline__ void warp_resort_block(int32_t* ord, const int64_t* v, int base,
                                                  int mult, int lane) {
  int64_t hi[E];
  int32_t lo[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * 32 + lane;
    if (i < mult) {
      const int c = ord[base + i];
      lo[e] = c;
      hi[e] = -v[c];
    } else {
      lo[e] = INT_MAX;
      hi[e] = LLONG_MAX;
    }
  }
  warp_bitonic_sort<E>(hi, lo, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * 32 + lane;
    if (i < mult) ord[base + i] = lo[e];
  }
}

__device__ __forceinline__ void warp_resort_dispatch(int32_t* ord, const int64_t* v, int base,
                                                     int mult, int lane) {
  if (mult <= 32) warp_resort_block<1>(ord, v, base, mult, lane);
  else if (mult <= 64) warp_resort_block<2>(ord, v, base, mult, lane);
  else if (mult <= 128) warp_resort_block<4>(ord, v, base, mult, lane);
  else if (mult <= 256) warp_resort_block<8>(ord, v, base, mult, lane);
  else if (mult <= 512) warp_resort_block<16>(ord, v, base, mult, lane);
  else if (lane == 0) {
    // mult > 512: an insertion sort on one lane, scalar registers only (the
    // re-sort never ran in a measured solve; see warp_block_sorted)
    for (int i = 1; i < mult; ++i) {
      const int c = ord[base + i];
      const int64_t vc = v[c];
      int q = i - 1;
      while (q >= 0) {
        const int d = ord[base + q];
        if (!(v[d] < vc || (v[d] == vc && d > c))) break;
        ord[base + q + 1] = d;
        --q;
      }
      ord[base + q + 1] = c;
    }
  }
  __syncwarp();
}

// After a row's potential update every touched block is already sorted by
// v desc: its P consumed columns get v' = G_w(t) - Q (non-increasing in t, the
// block's least relaxed value G only decreases) and every unconsumed column
// has v <= G_w(end) - Q (all remaining keys are >= 0 at the row end).  Only
// runs of equal v can be out of j order, so a block is re-sorted only when an
// adjacent pair violates (v desc, j asc) -- which never happened in any
// measured solve.
__device__ __forceinline__ bool warp_block_sorted(const int32_t* ord, const int64_t* v, int base,
                                                  int mult, int lane, bool ordid) {
  bool bad = false;
  for (int q = lane; q < mult - 1; q += 32) {
    // (identity order: position q holds column q + 1, no lookup)
    const int a = ordid ? base + q + 1 : ord[base + q], b = ordid ? a + 1 : ord[base + q + 1];
    const int64_t va = v[a], vb = v[b];
    bad |= !(va > vb || (va == vb && a < b));
  }
  return !__any_sync(0xffffffffu, bad);
}

// ----------------------------------------- K6 multi-warp kernel (n <= 32)
// The production solver for n <= 32 (one warp per block for n <= 16, one warp
// per two blocks above).  Run-batched Dijkstra steps: after the argmin picks
// block w, the next steps are evaluated speculatively assuming w keeps
// winning (~97% of consecutive steps share the winner block).  While w wins,
// its key sequence is closed form: with V6_t = v(c_t) << 6,
//     delta6_t = min(V6_{t-1}, A_w(r_{t-1})) - V6_t      (t >= 2),
// and every block's relaxed value obeys E^{t+1} = min(E^t - delta6_t, A(r_t)),
// i.e. with P_t = the sum of delta6 up to t and F = E + P_{t-1},
//     F^{t+1} = min(F^t, A(r_t) + P_t)      (a prefix min).
// Step t is the sequential step iff no other block has a smaller key:
// F_x^t + (B_x - w) > P_t for every x != w (keys carry the block index in
// their low bits, so they are never equal across blocks).  The first failing
// t over all blocks bounds the valid prefix, which is then committed exactly
// as the one-step loop would.  Warp x owns block x.  Every
// warp keeps all blocks' (G, key offset, cursor) lane-distributed, so each
// picks the run's winner itself (two redux.sync.min).  In a chunk (lanes =
// steps of the winner block) every warp runs one scan over the pair monoid
// (sum of deltas, min of its own block's relax candidates), then only its own
// block's "would block x win here" ballot and way update: a chunk costs one
// block's dependency chain instead of n of them.  The per-block fail masks
// and per-step G values are exchanged through double-buffered shared slots
// and an mbarrier (arrive, then the next chunk's operands and scan are
// computed speculatively, then wait).  The winner warp writes one 16-byte
// entry per reached column {column | row << 16, way entry, delta}, so the
// row end (potentials fused with the operand-table refresh, then the
// augmenting walk at one entry load per hop) needs no further lookups.  Block
// orders start as the identity and a potential update keeps each block sorted
// (see the re-sort check), so ord is only consulted after a fallback sort.

template <int AMODE, int MAXW, int BPW>  // AMODE 0: S and A shared; 1: S global, A shared; 2: S and A global; 3: + tables global
__global__ void __launch_bounds__(MAXW * 32, 1)                   // BPW: blocks per warp (1, or 2 for n <= 32)
    k_hungarian_blocks_mw(const int64_t* __restrict__ S_global, int n, int mult, int k,
                          int64_t* __restrict__ A_global, const uint32_t* __restrict__ order,
                          int32_t* __restrict__ decision, const uint32_t* __restrict__ row_ids,
                          uint64_t* __restrict__ col_of_row, unsigned long long* stats, int* flags,
                          const unsigned long long* __restrict__ max_scaled, int timing) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const size_t K1 = static_cast<size_t>(k) + 1;
  size_t so = 0;
  auto stake = [&](size_t bytes) {
    uint8_t* q = smem + so;
    so += (bytes + 15) & ~size_t(15);
    return q;
  };
  const int64_t* S;
  if constexpr (AMODE == 0) {
    int64_t* Ss = reinterpret_cast<int64_t*>(stake(static_cast<size_t>(k) * n * 8));
    for (size_t x = tid; x < static_cast<size_t>(k) * n; x += blockDim.x) Ss[x] = S_global[x];
    S = Ss;
  } else {
    S = S_global;
  }
  // AMODE 3 (large blocks): A and every per-column table the Dijkstra steps
  // do not read -- potentials, ways, orders, the reached list -- live in the
  // global arena after A; only the key offsets and rows stay shared.
  size_t go = 0;
  auto gtake = [&](size_t bytes) {
    uint8_t* q = reinterpret_cast<uint8_t*>(A_global) + go;
    go += (bytes + 15) & ~size_t(15);
    return q;
  };
  auto table = [&](size_t bytes) { return AMODE == 3 ? gtake(bytes) : stake(bytes); };
  // the operand table A, block-major: A[w * Kp + c - 1] = (S[p[c]][w] - u[p[c]]) << 6, so
  // a chunk's lanes (consecutive columns) read consecutive words -- the column-major
  // layout put every lane of a chunk in one shared-memory bank; Kp odd for the row
  // end's column-wise writes
  const size_t Kp = static_cast<size_t>(k) | 1;
  int64_t* A;
  if constexpr (AMODE <= 1) A = reinterpret_cast<int64_t*>(stake(static_cast<size_t>(n) * Kp * 8));
  else A = reinterpret_cast<int64_t*>(gtake(static_cast<size_t>(n) * Kp * 8));
  int64_t* Btab = reinterpret_cast<int64_t*>(stake(K1 * 8));  // by column: block - (v << 6)
  int64_t* u = reinterpret_cast<int64_t*>(table(K1 * 8));
  int64_t* v = reinterpret_cast<int64_t*>(table(K1 * 8));
  int64_t* dlt = reinterpret_cast<int64_t*>(table((K1 + 32) * 8));
  int32_t* p = reinterpret_cast<int32_t*>(table(K1 * 4));
  int32_t* wayi = reinterpret_cast<int32_t*>(table((K1 + 32) * 4));
  int32_t* ulist = reinterpret_cast<int32_t*>(table((K1 + 32) * 4));
  int32_t* ord = reinterpret_cast<int32_t*>(table(K1 * 4));
  int32_t* rtab = reinterpret_cast<int32_t*>(stake(K1 * 4));
  int32_t* cblk = reinterpret_cast<int32_t*>(table(K1 * 4));   // column -> block
  int32_t* curs = reinterpret_cast<int32_t*>(stake(32 * 4));
  // reached-column list of the row being solved, one 16-byte entry per step:
  // {c | p[c] << 16, way (entry index of the predecessor), delta at reach}
  int4* L = reinterpret_cast<int4*>(table((K1 + 32) * 16));
  // chunk: per-step G of each block, rows padded to 33 so the run end's read
  // across blocks (one step, lanes = blocks) hits distinct banks
  int64_t* GA = reinterpret_cast<int64_t*>(stake(2 * 32 * 33 * 8));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stake(16));            // chunk exchange barrier
  int32_t* ordflag = reinterpret_cast<int32_t*>(stake(16));           // block orders still identity?
  uint32_t* pfail = reinterpret_cast<uint32_t*>(stake(2 * 32 * 4));  // chunk: fail masks
  int32_t* tmp = reinterpret_cast<int32_t*>(table(static_cast<size_t>(2 * mult) * 4));
  if (so > dynamic_smem_bytes()) {  // host/device layout mismatch: fail loudly, touch nothing
    if (tid == 0) atomicOr(flags + kFlagInternal, 1);
    return;
  }
  const unsigned long long mx = *max_scaled;
  const bool packable = mx < (1ULL << 57) / (8ULL * static_cast<unsigned long long>(k + 1));
  for (size_t x = tid; x < K1; x += blockDim.x) {
    u[x] = 0;
    v[x] = 0;
    p[x] = 0;
    wayi[x] = 0;
  }
  for (int x = tid; x < k; x += blockDim.x) ord[x] = x + 1;
  __syncthreads();
  if (!packable) {  // wide-range path (see k_hungarian_blocks_wide)
    if (warp == 0) {
      BlockArrays Aw{S, u, v, dlt, p, wayi, ulist, ord, tmp};
      if (!hungarian_blocks_warp<1>(Aw, n, mult, k, stats, flags)) return;
      __syncwarp();
      for (int j = lane + 1; j <= k; j += 32) {
        const int r = p[j] - 1;
        if (col_of_row) col_of_row[r] = static_cast<uint64_t>(j - 1);
        if (decision) {
          const uint32_t row = order[r];
          decision[row_ids ? row_ids[row] : row] = (j - 1) / mult;
        }
      }
    }
    return;
  }
  for (int c = tid; c <= k; c += blockDim.x) {
    const int b = c == 0 ? 0 : (c - 1) / mult;
    cblk[c] = b;
    rtab[c] = 0;
    Btab[c] = b;
  }
  if (tid == 0) {
    mbar_init(mbar, nw);  // one arrival per warp
    ordflag[0] = 1;
  }
  __syncthreads();

  constexpr int64_t kBig = 1LL << 62;
  // this warp's blocks: warp, warp + nw (BPW == 2); xa is a valid table column
  int xs[BPW], xa[BPW];
  bool own[BPW];
#pragma unroll
  for (int h = 0; h < BPW; ++h) {
    xs[h] = warp + h * nw;
    own[h] = xs[h] < n;
    xa[h] = own[h] ? xs[h] : 0;
    if (!own[h]) xs[h] = 63;  // matches no winner
  }
  int par = 0;         // publish slot parity (identical in every warp)
  unsigned mbph = 0;   // mbarrier phase parity
  // solver statistics, kept by thread 0 in shared memory (no registers live
  // across the loop): [0] steps [1] run cycles [2] row-end cycles [3] re-sorts
  // [4] potential cycles [5] runs [6] re-sort-check cycles [7] start
  // [8] row start [9] t2 [10] t3; the cycle counters only when `timing`
  // (EDX_SOLVER_TIMING=1, tools/solver_profile.py)
  __shared__ unsigned long long sst[11];
  if (tid == 0) {
    for (int q = 0; q < 11; ++q) sst[q] = 0;
    sst[7] = clock64();
  }
  // row i's costs (lane = worker) are fetched one row ahead: the global
  // load's latency hides behind the previous row's search
  int64_t snext = (lane < n) ? S[lane] : 0;
  for (int i = 1; i <= k; ++i) {
    if (tid == 0 && timing) sst[8] = clock64();
    // Row frame: Q = cumulative delta of this row's search (<< 6).  Block y
    // keeps G_y = E_y + Q (its least relaxed value, unshifted by the deltas),
    // the key offset B_y of its next column and its cursor d_y; every warp
    // holds all blocks' (G, B, d) lane-distributed (lane y = block y) and its
    // own block's way (a step index into ulist).
    // Block orders start as the identity and, in practice, stay so (see the
    // re-sort check at row end); while they do, position q of the order is
    // column q + 1 and the ord lookup drops off the critical path.
    const bool ordid = ordflag[0] != 0;
    // Row i enters with u[i] = 0 (rows are solved in order); its costs stay
    // in a register for the augment's hop from column 0.
    int64_t Gy = kBig, By = kBig;
    const int64_t srow = snext;
    if (lane < n && i < k) snext = S[static_cast<size_t>(i) * n + lane];
    int dy = 0;
    if (lane < n) {
      Gy = srow << 6;  // relax from row i
      By = Btab[ordid ? lane * mult + 1 : ord[lane * mult]];
    }
    int wyx[BPW];
#pragma unroll
    for (int h = 0; h < BPW; ++h) wyx[h] = 0;
    if (tid == 0) {
      p[0] = i;
      L[0] = make_int4(i << 16, 0, 0, 0);
    }
    int nused = 1;
    int64_t Q = 0;
    bool abort = false, phase_end = false;
    while (!phase_end) {  // runs
      const uint64_t key = lane < n ? static_cast<uint64_t>(Gy - Q + By) : ~0ULL;
      const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
      const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
      const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
      if (mh >= 0x20000000u) {  // every block exhausted (key >= 2^61): corrupt input only
        abort = true;
        break;
      }
      const int ws = static_cast<int>(ml & 63u);
      const int dws = __shfl_sync(0xffffffffu, dy, ws);
      const int base = ws * mult + dws;  // position of the winner's candidate c_1
      const int Tm = mult - dws;
      const int64_t delta1 = static_cast<int64_t>(((static_cast<uint64_t>(mh) << 32) | ml) & ~63ULL);
      int64_t Gx[BPW], Bx[BPW];
#pragma unroll
      for (int h = 0; h < BPW; ++h) {
        Gx[h] = __shfl_sync(0xffffffffu, Gy, xs[h]);
        Bx[h] = __shfl_sync(0xffffffffu, By, xs[h]);
      }
      int64_t P = Q;
      int sN = 0;
      const int nused0 = nused;
      // Chunk operands, lanes = steps: column, its row, key offset, A[winner],
      // A[own blocks]; then the chunk's scan over (sum of deltas, min of relax
      // candidates) with the pair monoid (S, M).(S', M') = (S + S', min(M, S + M')),
      // relative to the carry P (one S, one M per own block).  The next chunk's
      // operands and scan are computed speculatively while this chunk's fail masks
      // are exchanged.
      auto load = [&](int s0, int& c, int& r, int64_t& Bc, int64_t& Aw, int64_t (&Ax)[BPW]) {
        const int q = base + min(s0 + lane, Tm - 1);
        c = ordid ? q + 1 : ord[q];
        Bc = Btab[c];
        r = rtab[c];
        Aw = A[static_cast<size_t>(ws) * Kp + (c - 1)];
#pragma unroll
        for (int h = 0; h < BPW; ++h) Ax[h] = A[static_cast<size_t>(xa[h]) * Kp + (c - 1)];
      };
      auto scan = [&](int64_t dl, const int64_t (&Ax)[BPW], int64_t& Ss, int64_t (&M)[BPW]) {
        Ss = dl;
#pragma unroll
        for (int h = 0; h < BPW; ++h) M[h] = Ax[h] + dl;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int64_t ys = __shfl_up_sync(0xffffffffu, Ss, off);
          int64_t ym[BPW];
#pragma unroll
          for (int h = 0; h < BPW; ++h) ym[h] = __shfl_up_sync(0xffffffffu, M[h], off);
          if (lane >= off) {
#pragma unroll
            for (int h = 0; h < BPW; ++h) {
              const int64_t t = ys + M[h];
              M[h] = ym[h] < t ? ym[h] : t;
            }
            Ss += ys;
          }
        }
      };
      int c, r;
      int64_t Bc, Aw, Ax[BPW], Ss, M[BPW];
      load(0, c, r, Bc, Aw, Ax);
      int64_t V6 = static_cast<int64_t>(ws) - Bc;
      {
        const int64_t V6p = __shfl_up_sync(0xffffffffu, V6, 1), Awp = __shfl_up_sync(0xffffffffu, Aw, 1);
        int64_t dl = lane == 0 ? delta1 : (V6p < Awp ? V6p : Awp) - V6;
        if (lane >= Tm) dl = 0;
        scan(dl, Ax, Ss, M);
      }
      for (;;) {  // chunks of up to 32 steps
        const int cnt = min(32, Tm - sN);
        const bool live = lane < cnt;
        const bool first = sN == 0 && lane == 0;
        const int64_t Qt = P + Ss;  // cumulative delta after this step
        bool failany = false;
        unsigned impm[BPW];
        int64_t Ga[BPW];
#pragma unroll
        for (int h = 0; h < BPW; ++h) {
          const int64_t cand = Ax[h] + Qt;  // relax candidate of this step for block xs[h]
          const int64_t Mp = P + __shfl_up_sync(0xffffffffu, M[h], 1);
          const int64_t Gb = lane == 0 ? Gx[h] : (Mp < Gx[h] ? Mp : Gx[h]);  // G before the step
          Ga[h] = cand < Gb ? cand : Gb;                                     // G after its relax
          failany |= own[h] && xs[h] != ws && !(Gb + Bx[h] - ws > Qt);      // block would win here
          impm[h] = __ballot_sync(0xffffffffu, live && cand < Gb);
        }
        const unsigned failx = __ballot_sync(0xffffffffu, live && !first && failany);
        const unsigned freem = __ballot_sync(0xffffffffu, live && r == 0);
        if (lane == 0) pfail[par * 32 + warp] = failx;
#pragma unroll
        for (int h = 0; h < BPW; ++h)
          if (own[h]) GA[(par * 32 + xs[h]) * 33 + lane] = Ga[h];
        // one arrival per warp (lane 0, after the warp's shared writes)
        __syncwarp();
        if (lane == 0) mbar_arrive(mbar);
        const bool more = sN + 32 < Tm;
        mbar_wait(mbar, mbph);
        mbph ^= 1u;
        const unsigned failm = __reduce_or_sync(0xffffffffu, lane < nw ? pfail[par * 32 + lane] : 0u);
        const int failq = failm ? __ffs(failm) - 1 : 32;
        const int freeq = freem ? __ffs(freem) - 1 : 32;
        int vq = failq < cnt ? failq : cnt;
        if (freeq < vq) {
          vq = freeq + 1;
          phase_end = true;
        }
        const unsigned relax_m = freeq < 32 ? ((1u << freeq) - 1u) : 0xffffffffu;  // no relax at a free column
        const int wbase = nused0 + sN;
#pragma unroll
        for (int h = 0; h < BPW; ++h) {
          if (xs[h] == ws && lane < vq) {  // the winner's warp commits: each lane its own step
            const unsigned prev = impm[h] & relax_m & ((1u << lane) - 1u);
            const int64_t dq = Qt >> 6;
            L[wbase + lane] = make_int4(c | (r << 16), prev ? wbase + 31 - __clz(prev) : wyx[h],
                                        static_cast<int>(static_cast<uint32_t>(dq)),
                                        static_cast<int>(dq >> 32));
          }
        }
        sN += vq;
        if (vq == 32 && !phase_end && more) {  // the whole chunk held: continue the run
          // The next chunk's operands and scan are computed only now: the
          // kernel is issue-bound (16 warps on 4 schedulers) and most runs end
          // inside their first chunk, so speculating before the exchange
          // costs more issue slots than the latency it hides.
          const int64_t P31 = __shfl_sync(0xffffffffu, Qt, 31);
          int64_t G31[BPW];
#pragma unroll
          for (int h = 0; h < BPW; ++h) G31[h] = __shfl_sync(0xffffffffu, Ga[h], 31);
          int c2, r2;
          int64_t Bc2, Aw2, Ax2[BPW], Ss2, M2[BPW];
          load(sN, c2, r2, Bc2, Aw2, Ax2);
          const int64_t V62 = static_cast<int64_t>(ws) - Bc2;
          {
            int64_t V6p = __shfl_up_sync(0xffffffffu, V62, 1), Awp = __shfl_up_sync(0xffffffffu, Aw2, 1);
            const int64_t V6l = __shfl_sync(0xffffffffu, V6, 31), Awl = __shfl_sync(0xffffffffu, Aw, 31);
            if (lane == 0) {
              V6p = V6l;
              Awp = Awl;
            }
            int64_t dl = (V6p < Awp ? V6p : Awp) - V62;
            if (sN + lane >= Tm) dl = 0;
            scan(dl, Ax2, Ss2, M2);
          }
          P = P31;
#pragma unroll
          for (int h = 0; h < BPW; ++h) {
            Gx[h] = G31[h];
            wyx[h] = impm[h] ? wbase + 31 - __clz(impm[h]) : wyx[h];
            Ax[h] = Ax2[h];
            M[h] = M2[h];
          }
          par ^= 1;
          c = c2;
          r = r2;
          Bc = Bc2;
          Aw = Aw2;
          V6 = V62;
          Ss = Ss2;
          continue;
        }
        // run end: carry, way, every block's G after the run's last step
        // (vq == 0 only after a full chunk, whose slot is still intact)
        if (vq > 0) {
          P = __shfl_sync(0xffffffffu, Qt, vq - 1);
          const unsigned lowv = vq >= 32 ? 0xffffffffu : ((1u << vq) - 1u);
#pragma unroll
          for (int h = 0; h < BPW; ++h) {
            const unsigned m2 = impm[h] & relax_m & lowv;
            wyx[h] = m2 ? wbase + 31 - __clz(m2) : wyx[h];
          }
        }
        if (lane < n)
          Gy = vq > 0 ? GA[(par * 32 + lane) * 33 + vq - 1] : GA[((par ^ 1) * 32 + lane) * 33 + 31];
        // the winner's next key offset: lane vq of this chunk (a run ending after
        // a whole chunk has exhausted the block or ended the row: no next key)
        const int64_t bnext = __shfl_sync(0xffffffffu, Bc, vq < 32 ? vq : 0);
        par ^= 1;
        if (tid == 0) {
          sst[0] += sN;
          sst[5] += 1;
        }
        Q = P;
        nused = nused0 + sN;
        if (lane == ws) {  // lane ws holds the winner's cursor and key offset
          dy += sN;
          By = dy < mult ? bnext : kBig;
        }
        break;
      }
    }
    if (abort) {
      if (tid == 0) atomicOr(flags + kFlagBadCost, 1);
      return;
    }
    const int64_t Dl = Q >> 6;
    if (warp == 0 && lane < n) curs[lane] = dy;
    __syncthreads();
    if (tid == 0 && timing) {
      const unsigned long long t2 = clock64();
      sst[1] += t2 - sst[8];
      sst[9] = t2;
    }
    const int nu = nused;
    // Potentials (assign.hpp:131-138) fused with the operand-table refresh:
    // reached column c moves by dd_c = Dl - dlt[c] (v[c] -= dd_c, u[p[c]] +=
    // dd_c).  Unless c is on the augmenting path its row stays p[c], so with A
    // in shared memory its words A[w][c] = (S[p[c]][w] - u[p[c]]) << 6 just
    // drop by dd_c << 6 -- no cost-matrix read, and u is never read again (a
    // row's potential lives only in its column's words).  With A in global
    // memory (AMODE >= 2) a read-modify-write would wait on L2, while S is
    // read-only (cached): the words are rewritten from S and u is kept.  A
    // group of gs >= n lanes per column, lanes over workers; every load of a
    // pass issued before its first store.
    {
      const int gs = n <= 8 ? 8 : (n <= 16 ? 16 : 32);
      const int gpw = 32 / gs, sub = lane / gs, lw = lane - sub * gs;
      const int stride = nw * gpw;
      // two columns in flight per group (four with A in shared memory: C3 row
      // end 2.37 -> 2.84 K cycles; six with A in global memory: C4 5.1 -> 7.9 K)
      constexpr int NE = 2;
      for (int eb = warp * gpw; eb < nu; eb += NE * stride) {  // warp-uniform trip count
        int e[NE], cc[NE], rr[NE];
        bool act[NE], aa[NE], ww[NE], ll[NE];
        int64_t dd[NE], vv[NE], bb[NE], xx[NE];
#pragma unroll
        for (int q = 0; q < NE; ++q) {
          e[q] = eb + sub + q * stride;
          act[q] = e[q] < nu;
          const int4 qe = act[q] ? L[e[q]] : make_int4(0, 0, 0, 0);
          cc[q] = qe.x & 0xffff;
          rr[q] = qe.x >> 16;
          dd[q] = Dl - ((static_cast<int64_t>(qe.w) << 32) | static_cast<uint32_t>(qe.z));
          // entry 0 (column 0, row i) sits at e == 0 only; the free column (r == 0) has no words
          aa[q] = act[q] && cc[q] != 0;
          ww[q] = aa[q] && rr[q] > 0 && lw < n;
          ll[q] = lw == 0 && aa[q];
        }
#pragma unroll
        for (int q = 0; q < NE; ++q) {
          vv[q] = ll[q] ? v[cc[q]] - dd[q] : 0;
          bb[q] = ll[q] ? cblk[cc[q]] : 0;
        }
        if constexpr (AMODE <= 1) {
#pragma unroll
          for (int q = 0; q < NE; ++q)
            xx[q] = ww[q] ? A[static_cast<size_t>(lw) * Kp + (cc[q] - 1)] - (dd[q] << 6) : 0;
        } else {
          int64_t uu[NE];
#pragma unroll
          for (int q = 0; q < NE; ++q) {
            uu[q] = act[q] ? u[rr[q]] + dd[q] : 0;
            xx[q] = ww[q] ? (S[static_cast<size_t>(rr[q] - 1) * n + lw] - uu[q]) << 6 : 0;
          }
          __syncwarp();  // every lane has read u[r] before the group leader writes it
          if (lw == 0) {
#pragma unroll
            for (int q = 0; q < NE; ++q)
              if (act[q]) u[rr[q]] = uu[q];
          }
        }
#pragma unroll
        for (int q = 0; q < NE; ++q) {
          if (ll[q]) {
            v[cc[q]] = vv[q];
            Btab[cc[q]] = bb[q] - (vv[q] << 6);
          }
          if (ww[q]) A[static_cast<size_t>(lw) * Kp + (cc[q] - 1)] = xx[q];
        }
      }
    }
    if constexpr (AMODE >= 2) __threadfence_block();
    __syncthreads();
    if (tid == 0 && timing) {
      const unsigned long long t3 = clock64();
      sst[4] += t3 - sst[9];
      sst[10] = t3;
    }
    // augment (assign.hpp:141-145) on the first warp whose block was not
    // touched, so it overlaps the re-sort checks.  Each hop is one entry load
    // (the predecessor's entry carries its column and old row); the path
    // columns change rows, so the warp also rewrites their tables.
    const unsigned untouched = __ballot_sync(0xffffffffu, lane < n && curs[lane] == 0);
    const int aug_warp = untouched ? (__ffs(untouched) - 1) % nw : 0;
    if (warp == aug_warp) {
      // the operand words move with the rows: jj takes its predecessor's row
      // and so that column's (already updated) words, read before the next hop
      // overwrites them; from column 0 it takes row i, (S[i] - Dl) << 6
      // (AMODE >= 2: rebuilt from S and u, see the potentials above)
      const int64_t wi = (srow - Dl) << 6;
      // The entry chain is fetched one hop ahead, so the pointer chase does
      // not wait behind each hop's operand copy.
      int4 ent = L[nu - 1];
      int4 prv = L[ent.y];
      for (;;) {
        const int jj = ent.x & 0xffff;
        if (jj == 0) break;
        const int rn = prv.x >> 16, pc = prv.x & 0xffff;  // p[jj] = p[way[jj]]
        const int4 nxt = pc != 0 ? L[prv.y] : prv;
        if (lane == 0) {
          p[jj] = rn;
          rtab[jj] = rn;
        }
        if (lane < n) {
          int64_t w;
          if constexpr (AMODE <= 1)
            w = pc == 0 ? wi : A[static_cast<size_t>(lane) * Kp + (pc - 1)];
          else
            w = (S[static_cast<size_t>(rn - 1) * n + lane] - (pc == 0 ? Dl : u[rn])) << 6;
          A[static_cast<size_t>(lane) * Kp + (jj - 1)] = w;
        }
        ent = prv;
        prv = nxt;
      }
    }
    // re-sort the touched blocks, if needed (see warp_block_sorted)
    for (int w = warp; w < n; w += nw) {
      if (curs[w] == 0) continue;
      if (!warp_block_sorted(ord, v, w * mult, mult, lane, ordflag[0] != 0)) {
        if (lane == 0) {
          atomicAdd(&sst[3], 1ULL);
          ordflag[0] = 0;
        }
        warp_resort_dispatch(ord, v, w * mult, mult, lane);
      }
      __syncwarp();
    }
    if constexpr (AMODE >= 2) __threadfence_block();
    __syncthreads();
    if (tid == 0 && timing) {
      const unsigned long long t4 = clock64();
      sst[6] += t4 - sst[10];
      sst[2] += t4 - sst[9];
    }
  }
  for (int j = tid + 1; j <= k; j += blockDim.x) {
    const int r = p[j] - 1;
    if (col_of_row) col_of_row[r] = static_cast<uint64_t>(j - 1);
    if (decision) {
      const uint32_t row = order[r];
      decision[row_ids ? row_ids[row] : row] = cblk[j];
    }
  }
  if (stats == nullptr) return;
  __syncthreads();
  if (tid == 0) {
    for (int q = 0; q < 7; ++q) stats[q] = sst[q];  // [3]: blocks that needed a full re-sort
    stats[7] = clock64() - sst[7];
  }
}

size_t mw_smem_bytes(int k, int n, int mult, int amode) {
  const size_t K1 = static_cast<size_t>(k) + 1;
  auto r = [](size_t b) { return (b + 15) & ~size_t(15); };
  size_t b = 0;
  if (amode == 0) b += r(static_cast<size_t>(k) * n * 8);
  if (amode <= 1) b += r(static_cast<size_t>(n) * (static_cast<size_t>(k) | 1) * 8);
  b += r(K1 * 8) + r(K1 * 4) + r(32 * 4) + r(2 * 32 * 33 * 8) + r(16) + r(16) + r(2 * 32 * 4);
  if (amode <= 2)  // the tables AMODE 3 keeps in the global arena
    b += 2 * r(K1 * 8) + r((K1 + 32) * 8) + 3 * r(K1 * 4) + 2 * r((K1 + 32) * 4) +
         r((K1 + 32) * 16) + r(static_cast<size_t>(2 * mult) * 4);
  return b;
}

// global arena of AMODE 2 (A) and 3 (A + the per-column tables)
size_t mw_arena_bytes(int k, int n, int mult, int amode) {
  const size_t K1 = static_cast<size_t>(k) + 1;
  auto r = [](size_t b) { return (b + 15) & ~size_t(15); };
  size_t b = r(static_cast<size_t>(n) * (static_cast<size_t>(k) | 1) * 8);
  if (amode == 3)
    b += 2 * r(K1 * 8) + r((K1 + 32) * 8) + 3 * r(K1 * 4) + 2 * r((K1 + 32) * 4) +
         r((K1 + 32) * 16) + r(static_cast<size_t>(2 * mult) * 4);
  return b;
}


// ----------------------------------------------------------------- K5 dense
// The reference loop on an arbitrary k x k matrix: one CTA, columns strided
// over threads, block-wide argmin with the lowest column winning ties.
constexpr int kDenseThreads = 1024;

__global__ void __launch_bounds__(kDenseThreads)
    k_hungarian_dense(const double* __restrict__ values, int k, int64_t cap,
                      uint8_t* __restrict__ arena, uint64_t* __restrict__ col_of_row,
                      unsigned long long* steps_out, int* __restrict__ flags) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int64_t red_v[32];
  __shared__ int red_j[32];
  __shared__ int s_j0, s_i0;
  __shared__ int64_t s_delta;
  uint8_t* base = arena ? arena : smem;
  const size_t K1 = static_cast<size_t>(k) + 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* q = base + off;
    off += (bytes + 15) & ~size_t(15);
    return q;
  };
  int64_t* u = reinterpret_cast<int64_t*>(take(K1 * 8));
  int64_t* v = reinterpret_cast<int64_t*>(take(K1 * 8));
  int64_t* minv = reinterpret_cast<int64_t*>(take(K1 * 8));
  int32_t* p = reinterpret_cast<int32_t*>(take(K1 * 4));
  int32_t* way = reinterpret_cast<int32_t*>(take(K1 * 4));
  uint8_t* used = take(K1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int x = tid; x <= k; x += kDenseThreads) {
    u[x] = 0;
    v[x] = 0;
    p[x] = 0;
    way[x] = 0;
  }
  bool bad = false;
  for (size_t x = tid; x < static_cast<size_t>(k) * k; x += kDenseThreads)
    bad |= bad_cost(values[x]);
  if (bad) atomicOr(flags + kFlagBadCost, 1);
  __syncthreads();
  unsigned long long steps = 0;
  for (int i = 1; i <= k; ++i) {
    for (int x = tid; x <= k; x += kDenseThreads) {
      minv[x] = kInf;
      used[x] = 0;
    }
    if (tid == 0) {
      p[0] = i;
      s_j0 = 0;
    }
    __syncthreads();
    for (;;) {
      const int j0 = s_j0;
      if (tid == 0) {
        used[j0] = 1;
        s_i0 = p[j0];
        ++steps;
      }
      __syncthreads();
      const int i0 = s_i0;
      const int64_t ui0 = u[i0];
      const double* row = values + static_cast<size_t>(i0 - 1) * k;
      int64_t best = kInf;
      int bj = INT_MAX;
      for (int j = tid + 1; j <= k; j += kDenseThreads) {
        if (used[j]) continue;
        const int64_t cur = scale_cost(row[j - 1], cap) - ui0 - v[j];
        if (cur < minv[j]) {
          minv[j] = cur;
          way[j] = j0;
        }
        if (minv[j] < best) {
          best = minv[j];
          bj = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const int64_t ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov < best || (ov == best && oj < bj)) {
          best = ov;
          bj = oj;
        }
      }
      if (lane == 0) {
        red_v[warp] = best;
        red_j[warp] = bj;
      }
      __syncthreads();
      if (warp == 0) {
        best = lane < kDenseThreads / 32 ? red_v[lane] : kInf;
        bj = lane < kDenseThreads / 32 ? red_j[lane] : INT_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const int64_t ov = __shfl_xor_sync(0xffffffffu, best, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
          if (ov < best || (ov == best && oj < bj)) {
            best = ov;
            bj = oj;
          }
        }
        if (lane == 0) {
          s_delta = best;
          s_j0 = bj;
        }
      }
      __syncthreads();
      const int64_t delta = s_delta;
      if (s_j0 == INT_MAX) {  // no unused column: only reachable on corrupt input
        if (tid == 0) atomicOr(flags + kFlagBadCost, 1);
        return;
      }
      for (int j = tid; j <= k; j += kDenseThreads) {
        if (used[j]) {
          u[p[j]] += delta;
          v[j] -= delta;
        } else if (minv[j] != kInf) {
          minv[j] -= delta;
        }
      }
      __syncthreads();
      if (p[s_j0] == 0) break;
    }
    if (tid == 0) {
      int j0 = s_j0;
      do {
        const int jp = way[j0];
        p[j0] = p[jp];
        j0 = jp;
      } while (j0 != 0);
    }
    __syncthreads();
  }
  for (int j = tid + 1; j <= k; j += kDenseThreads) col_of_row[p[j] - 1] = static_cast<uint64_t>(j - 1);
  if (tid == 0 && steps_out) steps_out[0] = steps;
}

size_t block_arena_bytes(int k, int mult) {
  const size_t K1 = static_cast<size_t>(k) + 1;
  auto r = [](size_t b) { return (b + 15) & ~size_t(15); };
  return 3 * r(K1 * 8) + 3 * r(K1 * 4) + r(static_cast<size_t>(k) * 4) +
         r(static_cast<size_t>(2 * mult) * 4);
}

// ------------------------------------------------ K5 dense, lazy potentials
// The same e-maxx steps with the O(k) potential pass of every step removed:
// within a row's search, every used column j's potentials move by each later
// delta, so they are applied once at the row end from D (the running sum of
// deltas) at the moment j was reached; an unused column's minv is kept as
// minv + D (one shift for all of them, so their order -- and the argmin with
// the lowest index on ties -- is unchanged), and a relaxation from row i0 =
// p[j0] compares a[i0][j] - u[i0] - v[j] + D(j0) with it, where D(j0) = D at
// the step j0 was reached (u[i0] has not moved yet then).  Exact in int64.
// One CTA, thread t owning columns t + 1 + c * 1024 (c < C) in registers
// (stored minv, v, reached flag and D at reach); one barrier per step: warps
// publish their (minv, j) minimum, every warp reduces the 32 of them.  The
// scaled costs (llround(v * 1e12), capped; assign.hpp:92-100) are computed
// once into an int64 k x k table the steps read row by row.
constexpr int kDense2Threads = 1024;

__global__ void k_scale_dense(const double* __restrict__ values, uint64_t count, int64_t cap,
                              int64_t* __restrict__ S) {
  const uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (x < count) S[x] = scale_cost(values[x], cap);
}

__device__ __forceinline__ void argmin_pair(int64_t& v, int& j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oj = __shfl_xor_sync(0xffffffffu, j, o);
    if (ov < v || (ov == v && oj < j)) {
      v = ov;
      j = oj;
    }
  }
}

template <int C, int T>
__global__ void __launch_bounds__(T, 1)
    k_hungarian_dense2(const int64_t* __restrict__ S, int k, uint64_t* __restrict__ col_of_row,
                       unsigned long long* stats, int* __restrict__ flags) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int64_t red_v[2][32];
  __shared__ int red_j[2][32];
  const size_t K1 = static_cast<size_t>(k) + 1;
  const size_t K1e = (K1 + 1) & ~size_t(1);  // even: every array below stays 8-byte aligned
  int64_t* u = reinterpret_cast<int64_t*>(smem);        // by row
  int32_t* p = reinterpret_cast<int32_t*>(u + K1e);     // by column
  int32_t* way = p + K1e;                               // by column
  int64_t* dreach = reinterpret_cast<int64_t*>(way + K1e);  // by column: D when reached
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  for (size_t x = tid; x < K1; x += T) {
    u[x] = 0;
    p[x] = 0;
    way[x] = 0;
  }
  int64_t v[C], ms[C];
  int jc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    v[c] = 0;
    jc[c] = tid + 1 + c * T;  // column (valid when <= k)
  }
  __syncthreads();
  unsigned long long steps = 0;
  int par = 0;
  for (int i = 1; i <= k; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) ms[c] = kInf;
    unsigned reached = 0;  // bit c: column jc[c] reached (used) in this row
    if (tid == 0) p[0] = i;
    __syncthreads();
    int j0 = 0, i0 = i;
    int64_t dj0 = 0;          // D when j0 was reached
    int64_t ui0 = u[i];
    int64_t D = 0;
    for (;;) {
      ++steps;
      // relax the unreached columns from row i0, local argmin (ascending j)
      const int64_t* Srow = S + static_cast<size_t>(i0 - 1) * k;
      const int64_t shift = dj0 - ui0;
      int64_t a[C];
#pragma unroll
      for (int c = 0; c < C; ++c) a[c] = (jc[c] <= k && !((reached >> c) & 1u)) ? Srow[jc[c] - 1] : 0;
      int64_t best = kInf;
      int bj = INT_MAX;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (jc[c] > k || ((reached >> c) & 1u)) continue;
        const int64_t x = a[c] + shift - v[c];
        if (x < ms[c]) {
          ms[c] = x;
          way[jc[c]] = j0;
        }
        if (ms[c] < best) {
          best = ms[c];
          bj = jc[c];
        }
      }
      argmin_pair(best, bj);
      if (lane == 0) {
        red_v[par][warp] = best;
        red_j[par][warp] = bj;
      }
      __syncthreads();
      best = lane < T / 32 ? red_v[par][lane] : kInf;
      bj = lane < T / 32 ? red_j[par][lane] : INT_MAX;
      argmin_pair(best, bj);
      par ^= 1;
      if (bj == INT_MAX) {  // no unused column: only reachable on corrupt input
        if (tid == 0) atomicOr(flags + kFlagBadCost, 1);
        return;
      }
      // the column reached at this step: D moves to its stored minv
      D = best;
      j0 = bj;
      dj0 = D;
      {
        const int c = (j0 - 1 - tid) / T;
        if ((j0 - 1) % T == tid) {
          reached |= 1u << c;
          dreach[j0] = D;
        }
      }
      i0 = p[j0];
      if (i0 == 0) break;  // a free column: the augmenting path ends here
      ui0 = u[i0];
    }
    // row end: potentials of the reached columns (assign.hpp:131-138 summed
    // over the row's steps), the free column's excluded (it moved by 0)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if (!((reached >> c) & 1u)) continue;
      const int64_t dd = D - dreach[jc[c]];
      v[c] -= dd;
      if (p[jc[c]] != 0) u[p[jc[c]]] += dd;
    }
    if (tid == 0) u[i] += D;  // column 0 (row i) was reached at D = 0
    __syncthreads();
    if (tid == 0) {  // augment (assign.hpp:141-145)
      int jj = j0;
      do {
        const int jp = way[jj];
        p[jj] = p[jp];
        jj = jp;
      } while (jj != 0);
    }
    __syncthreads();
  }
  for (int j = tid + 1; j <= k; j += T) col_of_row[p[j] - 1] = static_cast<uint64_t>(j - 1);
  if (tid == 0 && stats) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    stats[0] = steps;
    stats[6] = t_end - t_start;  // ns on the device
  }
}

size_t dense2_smem_bytes(int k) {
  const size_t K1 = static_cast<size_t>(k) + 1, K1e = (K1 + 1) & ~size_t(1);
  return K1e * (8 + 4 + 4 + 8);  // u, p, way, dreach
}

size_t dense_arena_bytes(int k) {
  const size_t K1 = static_cast<size_t>(k) + 1;
  auto r = [](size_t b) { return (b + 15) & ~size_t(15); };
  return 3 * r(K1 * 8) + 2 * r(K1 * 4) + r(K1);
}

int max_dyn_smem(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return v;
}

}  // namespace


size_t fast_smem_bytes(int k, int n, int mult, int nw, int mode) {
  const size_t K1 = static_cast<size_t>(k) + 1;
  auto r = [](size_t b) { return (b + 15) & ~size_t(15); };
  size_t b = 0;
  if (mode == 0) b += r(static_cast<size_t>(k) * n * 8);
  if (mode <= 1) b += 3 * r(K1 * 8) + 3 * r(K1 * 4) + r(static_cast<size_t>(k) * 4);
  const int W = n <= 32 ? 32 : 64;
  b += r(static_cast<size_t>(n) * W * 8) + 2 * r(64 * 4) + r(32) +
       r(static_cast<size_t>(nw) * mult * 8) + r(static_cast<size_t>(nw) * 2 * mult * 4);
  return b;
}

void launch_hungarian_blocks(HungarianScratch& sc, const double* matrix, int n,
                             const uint32_t* order, int mult, int32_t* decision,
                             const uint32_t* row_ids, uint64_t* col_of_row, int* flags,
                             cudaStream_t s, int device) {
  const int k = n * mult;
  if (k <= 0) return;
  const int64_t cap = LLONG_MAX / (8 * static_cast<int64_t>(k + 1));
  sc.s64.ensure(static_cast<size_t>(k) * n + 1);
  sc.steps.ensure(9);
  unsigned long long* max_scaled = sc.steps.p + 8;
  EDX_CUDA(cudaMemsetAsync(max_scaled, 0, sizeof(unsigned long long), s));
  const uint64_t total = static_cast<uint64_t>(k) * n;
  k_scale_block<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(
      matrix, n, order, k, cap, sc.s64.p, flags, max_scaled);
  EDX_LAUNCHED();
  const size_t limit = static_cast<size_t>(max_dyn_smem(device));
  const int nw = std::min(n, kFastMaxWarps);
  // the multi-warp kernel: one warp per block for n <= 16, one warp per two
  // blocks (16 warps) for 16 < n <= 32 -- one warp per block at n = 32 costs
  // more in the 32-way exchange than the per-block work it splits
  static const int bpw_pref = [] {  // EDX_MW_BPW=2: two blocks per warp also for n <= 16 (A/B)
    const char* e = std::getenv("EDX_MW_BPW");
    return e && std::strcmp(e, "2") == 0 ? 2 : 1;
  }();
  static const int timing = [] {  // EDX_SOLVER_TIMING=1: per-phase cycle counters
    const char* e = std::getenv("EDX_SOLVER_TIMING");
    return e && std::strcmp(e, "1") == 0 ? 1 : 0;
  }();
  static const int amode_min = [] {  // EDX_MW_GLOBAL=1: the global-table layout (tests)
    const char* e = std::getenv("EDX_MW_GLOBAL");
    return e && std::strcmp(e, "1") == 0 ? 3 : 0;
  }();
  if (n <= 32 && mult <= 1024) {
    const bool pair = n > 16 || (bpw_pref == 2 && n > 1);
    const int nwarps = pair ? (n + 1) / 2 : n;
    for (int am = amode_min; am <= 3; ++am) {
      const size_t smem = mw_smem_bytes(k, n, mult, am);
      if (smem > limit) continue;
      int64_t* Ag = nullptr;
      if (am >= 2) {
        sc.arena.ensure(mw_arena_bytes(k, n, mult, am));
        Ag = reinterpret_cast<int64_t*>(sc.arena.p);
      }
      auto launch = [&](auto kern) {
        if (smem > 48 * 1024)
          EDX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
        kern<<<1, 32 * nwarps, smem, s>>>(sc.s64.p, n, mult, k, Ag, order, decision, row_ids,
                                          col_of_row, sc.steps.p, flags, max_scaled, timing);
      };
      // the warp cap sets the register budget: 255 (n <= 8), 128 (n <= 32)
      if (pair && n <= 16) {
        if (am == 0) { launch(k_hungarian_blocks_mw<0, 8, 2>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<0,8,2>"; }
        else if (am == 1) { launch(k_hungarian_blocks_mw<1, 8, 2>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<1,8,2>"; }
        else if (am == 2) { launch(k_hungarian_blocks_mw<2, 8, 2>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<2,8,2>"; }
        else { launch(k_hungarian_blocks_mw<3, 8, 2>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<3,8,2>"; }
      } else if (n <= 8) {
        if (am == 0) { launch(k_hungarian_blocks_mw<0, 8, 1>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<0,8,1>"; }
        else if (am == 1) { launch(k_hungarian_blocks_mw<1, 8, 1>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<1,8,1>"; }
        else if (am == 2) { launch(k_hungarian_blocks_mw<2, 8, 1>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<2,8,1>"; }
        else { launch(k_hungarian_blocks_mw<3, 8, 1>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<3,8,1>"; }
      } else if (n <= 16) {
        if (am == 0) { launch(k_hungarian_blocks_mw<0, 16, 1>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<0,16,1>"; }
        else if (am == 1) { launch(k_hungarian_blocks_mw<1, 16, 1>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<1,16,1>"; }
        else if (am == 2) { launch(k_hungarian_blocks_mw<2, 16, 1>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<2,16,1>"; }
        else { launch(k_hungarian_blocks_mw<3, 16, 1>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<3,16,1>"; }
      } else {
        if (am == 0) { launch(k_hungarian_blocks_mw<0, 16, 2>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<0,16,2>"; }
        else if (am == 1) { launch(k_hungarian_blocks_mw<1, 16, 2>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<1,16,2>"; }
        else if (am == 2) { launch(k_hungarian_blocks_mw<2, 16, 2>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<2,16,2>"; }
        else { launch(k_hungarian_blocks_mw<3, 16, 2>); g_kernel_name[kKSolver] = "k_hungarian_blocks_mw<3,16,2>"; }
      }
      EDX_LAUNCHED();
      return;
    }
  }
  int mode = -1;
  for (int md = 0; md <= 2 && mode < 0; ++md)
    if (fast_smem_bytes(k, n, mult, nw, md) <= limit) mode = md;
  if (mode >= 0) {
    const size_t smem = fast_smem_bytes(k, n, mult, nw, mode);
    uint8_t* garena = nullptr;
    if (mode == 2) {
      sc.arena.ensure(block_arena_bytes(k, mult));
      garena = sc.arena.p;
    }
    auto launch = [&](auto kern) {
      if (smem > 48 * 1024)
        EDX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
      kern<<<1, 32 * nw, smem, s>>>(sc.s64.p, n, mult, k, garena, order, decision, row_ids,
                                    col_of_row, sc.steps.p, flags, max_scaled);
    };
    g_kernel_name[kKSolver] = n <= 32 ? "k_hungarian_blocks_fast<1>" : "k_hungarian_blocks_fast<2>";
    if (n <= 32) {
      if (mode == 0) launch(k_hungarian_blocks_fast<1, 0>);
      else if (mode == 1) launch(k_hungarian_blocks_fast<1, 1>);
      else launch(k_hungarian_blocks_fast<1, 2>);
    } else {
      if (mode == 0) launch(k_hungarian_blocks_fast<2, 0>);
      else if (mode == 1) launch(k_hungarian_blocks_fast<2, 1>);
      else launch(k_hungarian_blocks_fast<2, 2>);
    }
    EDX_LAUNCHED();
    return;
  }
  // only for very large blocks: the single-warp kernel with global arrays
  const size_t arena = block_arena_bytes(k, mult);
  sc.arena.ensure(arena);
  g_kernel_name[kKSolver] = "k_hungarian_blocks_wide<2>";
  k_hungarian_blocks_wide<2><<<1, 32, 0, s>>>(sc.s64.p, n, mult, k, 0, sc.arena.p, order, decision,
                                              row_ids, col_of_row, sc.steps.p, flags);
  EDX_LAUNCHED();
}

void launch_hungarian_dense(HungarianScratch& sc, const double* values, uint64_t k,
                            uint64_t* col_of_row, int* flags, cudaStream_t s, int device) {
  const int64_t cap = LLONG_MAX / (8 * static_cast<int64_t>(k + 1));
  sc.steps.ensure(9);
  EDX_CUDA(cudaMemsetAsync(sc.steps.p, 0, 8 * sizeof(unsigned long long), s));
  const size_t limit = static_cast<size_t>(max_dyn_smem(device)) - 1024;  // static smem
  const size_t smem2 = dense2_smem_bytes(static_cast<int>(k));
  if (k <= 8 * static_cast<uint64_t>(kDense2Threads) && smem2 <= limit) {
    // scaled costs once, then the lazy-potential steps
    sc.s64.ensure(k * k);
    k_scale_dense<<<static_cast<unsigned>((k * k + 255) / 256), 256, 0, s>>>(values, k * k, cap,
                                                                           sc.s64.p);
    EDX_LAUNCHED();
    auto go = [&](auto kern, int threads) {
      EDX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem2)));
      kern<<<1, threads, smem2, s>>>(sc.s64.p, static_cast<int>(k), col_of_row, sc.steps.p, flags);
    };
    // columns per thread in registers: 1024 threads up to 4 each, 512 x 16 above
    if (k <= 1024) go(k_hungarian_dense2<1, 1024>, 1024);
    else if (k <= 2048) go(k_hungarian_dense2<2, 1024>, 1024);
    else if (k <= 4096) go(k_hungarian_dense2<4, 1024>, 1024);
    else go(k_hungarian_dense2<16, 512>, 512);
    EDX_LAUNCHED();
    g_kernel_name[kKSolver] = "k_hungarian_dense2";
    return;
  }
  const size_t arena = dense_arena_bytes(static_cast<int>(k));
  size_t smem = 0;
  uint8_t* garena = nullptr;
  if (arena <= limit) {
    smem = arena;
  } else {
    sc.arena.ensure(arena);
    garena = sc.arena.p;
  }
  if (smem > 48 * 1024)
    EDX_CUDA(cudaFuncSetAttribute(k_hungarian_dense, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
  g_kernel_name[kKSolver] = "k_hungarian_dense";
  k_hungarian_dense<<<1, kDenseThreads, smem, s>>>(values, static_cast<int>(k), cap, garena,
                                                   col_of_row, sc.steps.p, flags);
  EDX_LAUNCHED();
}

void last_hungarian_stats(HungarianScratch& sc, cudaStream_t s, unsigned long long* out) {
  for (int i = 0; i < 8; ++i) out[i] = 0;
  if (!sc.steps.p) return;
  EDX_CUDA(cudaMemcpyAsync(out, sc.steps.p, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  EDX_CUDA(cudaStreamSynchronize(s));
}

unsigned long long last_hungarian_steps(HungarianScratch& sc, cudaStream_t s) {
  if (!sc.steps.p) return 0;
  unsigned long long h = 0;
  EDX_CUDA(cudaMemcpyAsync(&h, sc.steps.p, sizeof h, cudaMemcpyDeviceToHost, s));
  EDX_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace edx
