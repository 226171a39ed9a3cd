// NCCL plumbing of the multi-GPU engine; see nccl_comm.cpp.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>

#include "edx_internal.cuh"

namespace edx {

void nccl_unique_id(void* out128);
void* nccl_comm_create(const void* id128, int world, int rank);
void nccl_comm_destroy(void* comm);
void nccl_gather_rows(void* comm, double* matrix, const uint64_t* lo, const uint64_t* hi,
                      int world, int rank, int root, int n, cudaStream_t s);
void nccl_broadcast_i32(void* comm, int32_t* buf, uint64_t count, int root, cudaStream_t s);

// Contiguous, balanced row shards: rank r builds rows [lo_r, hi_r).
inline void shard_rows(uint64_t rows, int world, uint64_t* lo, uint64_t* hi) {
  for (int r = 0; r < world; ++r) {
    lo[r] = rows * static_cast<uint64_t>(r) / static_cast<uint64_t>(world);
    hi[r] = rows * static_cast<uint64_t>(r + 1) / static_cast<uint64_t>(world);
  }
}

}  // namespace edx
