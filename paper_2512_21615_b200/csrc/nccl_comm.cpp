// NCCL plumbing of the multi-GPU engine: the cost-matrix rows
// are sharded by sample across the ranks of one box, gathered to the solver
// rank over NVLink, and the decision is broadcast back.  libnccl is resolved
// at run time (dlopen, reusing the copy torch already loaded when present) so
// libedx.so has no link-time NCCL dependency and single-GPU use never loads it.
#include "nccl_comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <stdexcept>
#include <string>

namespace edx {

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

NcclApi* api() {
  static NcclApi a;
  static std::once_flag once;
  static std::string failure;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      failure = std::string("cannot load libnccl: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p) failure = std::string("libnccl lacks ") + n;
      return p;
    };
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
    a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(sym("ncclBroadcast"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(sym("ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(sym("ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
  });
  if (!failure.empty()) throw Error(EDX_RUNTIME_ERROR, failure);
  return &a;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(EDX_RUNTIME_ERROR, std::string(what) + ": " + api()->error_string(r));
}

}  // namespace

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  check(api()->get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof id);
}

void* nccl_comm_create(const void* id128, int world, int rank) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t comm = nullptr;
  check(api()->comm_init_rank(&comm, world, id, rank), "ncclCommInitRank");
  return comm;
}

void nccl_comm_destroy(void* comm) {
  if (comm) api()->comm_destroy(static_cast<ncclComm_t>(comm));
}

// Rows [lo_r, hi_r) of every rank -> the root's full matrix (grouped send/recv;
// NCCL 2.27 has no Gather).
void nccl_gather_rows(void* comm, double* matrix, const uint64_t* lo, const uint64_t* hi,
                      int world, int rank, int root, int n, cudaStream_t s) {
  auto* c = static_cast<ncclComm_t>(comm);
  check(api()->group_start(), "ncclGroupStart");
  if (rank == root) {
    for (int r = 0; r < world; ++r) {
      if (r == root || hi[r] == lo[r]) continue;
      check(api()->recv(matrix + lo[r] * n, (hi[r] - lo[r]) * n, ncclFloat64, r, c, s), "ncclRecv");
    }
  } else if (hi[rank] > lo[rank]) {
    check(api()->send(matrix + lo[rank] * n, (hi[rank] - lo[rank]) * n, ncclFloat64, root, c, s),
          "ncclSend");
  }
  check(api()->group_end(), "ncclGroupEnd");
}

void nccl_broadcast_i32(void* comm, int32_t* buf, uint64_t count, int root, cudaStream_t s) {
  check(api()->broadcast(buf, buf, count, ncclInt32, root, static_cast<ncclComm_t>(comm), s),
        "ncclBroadcast");
}

}  // namespace edx
