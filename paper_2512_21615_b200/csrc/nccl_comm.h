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

// The byte-moving primitives the exchange steps below are written against:
// NcclTransport (device buffers, enqueued on a stream, grouped) in the
// engine; CallbackTransport (host buffers, the caller's functions) behind
// edx_exchange_* -- the same bookkeeping either way.
struct Transport {
  virtual ~Transport() = default;
  virtual void group_start() {}
  virtual void group_end() {}
  virtual void send(const void* buf, uint64_t bytes, int peer) = 0;
  virtual void recv(void* buf, uint64_t bytes, int peer) = 0;
  virtual void broadcast(void* buf, uint64_t bytes, int root) = 0;
};

struct NcclTransport final : Transport {
  NcclTransport(void* comm, cudaStream_t s) : comm(comm), stream(s) {}
  void group_start() override;
  void group_end() override;
  void send(const void* buf, uint64_t bytes, int peer) override;
  void recv(void* buf, uint64_t bytes, int peer) override;
  void broadcast(void* buf, uint64_t bytes, int root) override;
  void* comm;
  cudaStream_t stream;
};

// Rows [lo_r, hi_r) of every rank -> the root's full row-major matrix
// (n doubles per row): each non-root rank sends its shard once, the root
// receives every other shard in place; one group.
void gather_rows(Transport& t, double* matrix, const uint64_t* lo, const uint64_t* hi, int world,
                 int rank, int root, int n);
// The root's decision (one int32 per sample) to every rank.
void broadcast_decision(Transport& t, int32_t* decision, uint64_t rows, int root);
// The root's expected cost (one double) to every rank.
void broadcast_cost(Transport& t, double* cost, int root);

// Contiguous, balanced row shards: rank r builds rows [lo_r, hi_r).
inline void shard_rows(uint64_t rows, int world, uint64_t* lo, uint64_t* hi) {
  for (int r = 0; r < world; ++r) {
    lo[r] = rows * static_cast<uint64_t>(r) / static_cast<uint64_t>(world);
    hi[r] = rows * static_cast<uint64_t>(r + 1) / static_cast<uint64_t>(world);
  }
}

}  // namespace edx
