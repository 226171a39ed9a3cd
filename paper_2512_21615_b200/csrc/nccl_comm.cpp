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

void NcclTransport::group_start() { check(api()->group_start(), "ncclGroupStart"); }
void NcclTransport::group_end() { check(api()->group_end(), "ncclGroupEnd"); }
void NcclTransport::send(const void* buf, uint64_t bytes, int peer) {
  check(api()->send(buf, bytes, ncclInt8, peer, static_cast<ncclComm_t>(comm), stream), "ncclSend");
}
void NcclTransport::recv(void* buf, uint64_t bytes, int peer) {
  check(api()->recv(buf, bytes, ncclInt8, peer, static_cast<ncclComm_t>(comm), stream), "ncclRecv");
}
void NcclTransport::broadcast(void* buf, uint64_t bytes, int root) {
  check(api()->broadcast(buf, buf, bytes, ncclInt8, root, static_cast<ncclComm_t>(comm), stream),
        "ncclBroadcast");
}

// (NCCL 2.27 has no Gather: grouped point-to-point.)
void gather_rows(Transport& t, double* matrix, const uint64_t* lo, const uint64_t* hi, int world,
                 int rank, int root, int n) {
  const uint64_t row_bytes = static_cast<uint64_t>(n) * sizeof(double);
  t.group_start();
  if (rank == root) {
    for (int r = 0; r < world; ++r) {
      if (r == root || hi[r] == lo[r]) continue;
      t.recv(matrix + lo[r] * n, (hi[r] - lo[r]) * row_bytes, r);
    }
  } else if (hi[rank] > lo[rank]) {
    t.send(matrix + lo[rank] * n, (hi[rank] - lo[rank]) * row_bytes, root);
  }
  t.group_end();
}

void broadcast_decision(Transport& t, int32_t* decision, uint64_t rows, int root) {
  if (rows) t.broadcast(decision, rows * sizeof(int32_t), root);
}

void broadcast_cost(Transport& t, double* cost, int root) { t.broadcast(cost, sizeof(double), root); }

}  // namespace edx
