// Block-wide bitonic sort of (key, value) pairs in shared memory, ascending
// by (key, value): the victims of one worker (step.cu, k_select_victims).
// (Measured as a single-CTA replacement for the 1,024-row gap sort it lost to
// CUB's single-tile radix sort: 25 vs 19 us per sort, so it is not used there.)
//
// Thread t owns elements [4t, 4t+4) for the register part: strides 1 and 2
// are in-thread, strides 4..64 are warp shuffles (the partner sits in lane ^
// stride/4, same register slot), strides >= 128 go through shared memory.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace edx {

__device__ __forceinline__ bool kv_less(uint64_t ak, uint32_t av, uint64_t bk, uint32_t bv) {
  return ak < bk || (ak == bk && av < bv);
}

template <int S>
__device__ __forceinline__ void bitonic_in_thread(uint32_t base, uint32_t size, uint64_t (&rk)[4],
                                                  uint32_t (&rv)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q & S) continue;
    const uint32_t i = base + q;
    if (kv_less(rk[q + S], rv[q + S], rk[q], rv[q]) == ((i & size) == 0)) {
      const uint64_t tk = rk[q];
      rk[q] = rk[q + S];
      rk[q + S] = tk;
      const uint32_t tv = rv[q];
      rv[q] = rv[q + S];
      rv[q + S] = tv;
    }
  }
}

// stages (size, stride), (size, stride/2), ..., (size, 1) for stride <= 64
__device__ __forceinline__ void bitonic_reg_stages(uint32_t base, uint32_t size, uint32_t stride,
                                                   uint64_t (&rk)[4], uint32_t (&rv)[4]) {
  for (; stride >= 4; stride >>= 1) {
    const int lx = static_cast<int>(stride >> 2);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t i = base + q;
      const uint64_t ok = __shfl_xor_sync(0xffffffffu, rk[q], lx);
      const uint32_t ov = __shfl_xor_sync(0xffffffffu, rv[q], lx);
      const bool asc = (i & size) == 0, lower = (i & stride) == 0;
      if (lower == asc ? kv_less(ok, ov, rk[q], rv[q]) : kv_less(rk[q], rv[q], ok, ov)) {
        rk[q] = ok;
        rv[q] = ov;
      }
    }
  }
  if (stride >= 2) bitonic_in_thread<2>(base, size, rk, rv);
  bitonic_in_thread<1>(base, size, rk, rv);
}

// Sorts sk[0, P), sv[0, P) ascending by (key, value).  P is a power of two
// with 128 <= P <= 4 * blockDim.x.  Every thread of the block calls it, after
// the arrays are filled and a __syncthreads(); it ends with one.
__device__ __forceinline__ void block_bitonic_sort(uint64_t* sk, uint32_t* sv, uint32_t P) {
  const uint32_t tid = threadIdx.x, base = 4 * tid;
  const bool owner = base < P;  // warp-uniform since P % 128 == 0
  uint64_t rk[4];
  uint32_t rv[4];
  auto load4 = [&] {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      rk[q] = sk[base + q];
      rv[q] = sv[base + q];
    }
  };
  auto store4 = [&] {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      sk[base + q] = rk[q];
      sv[base + q] = rv[q];
    }
  };
  if (owner) {
    load4();
    for (uint32_t size = 2; size <= 128; size <<= 1) bitonic_reg_stages(base, size, size >> 1, rk, rv);
    store4();
  }
  __syncthreads();
  for (uint32_t size = 256; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride >= 128; stride >>= 1) {
      for (uint32_t t = tid; t < P / 2; t += blockDim.x) {
        const uint32_t lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const uint64_t a = sk[lo], b = sk[hi];
        const uint32_t av = sv[lo], bv = sv[hi];
        if (kv_less(b, bv, a, av) == ((lo & size) == 0)) {
          sk[lo] = b;
          sk[hi] = a;
          sv[lo] = bv;
          sv[hi] = av;
        }
      }
      __syncthreads();
    }
    if (owner) {
      load4();
      bitonic_reg_stages(base, size, 64, rk, rv);
      store4();
    }
    __syncthreads();
  }
}

}  // namespace edx
