// Internal declarations shared by the libedx translation units.
// Everything here is sm_100a device code or host orchestration around it;
// the public surface is include/edx.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "edx.h"

namespace edx {

// ---- shared-memory mbarriers and 1D bulk (TMA) copies, CTA scope
#ifdef __CUDACC__
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// Arms `bar` for `bytes` of bulk-copy traffic (one arrival of its count).
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
// Global -> shared bulk copy completing on `bar` (16-byte aligned, size % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
// Orders this thread's earlier generic shared-memory accesses before later async-proxy (bulk copy) writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
#endif

// NVTX range for the host-side enqueue of one phase (build, gap sort, exact
// solve, greedy, step): header-only NVTX v3, a no-op unless a tool (ncu
// --nvtx, Nsight Systems) is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- errors
// Host-side exceptions carry an edx_status; the C ABI boundary converts them.
struct Error : std::runtime_error {
  edx_status code;
  Error(edx_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw Error(EDX_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file +
                                  ":" + std::to_string(line) + ")");
}

#define EDX_CUDA(x)                                                   \
  do {                                                                \
    cudaError_t _e = (x);                                             \
    if (_e != cudaSuccess) ::edx::throw_cuda(_e, #x, __FILE__, __LINE__); \
  } while (0)

#define EDX_LAUNCHED()                                                        \
  do {                                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) ::edx::throw_cuda(_e, "kernel launch", __FILE__, __LINE__); \
  } while (0)

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while its stream predecessor drains; it must call pdl_wait()
// before touching memory (the wait returns once the predecessor grid has
// completed and its writes are visible).  pdl_trigger() lets the successor's
// CTAs be scheduled early.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// EDX_PDL=0 turns the attribute off (A/B switch)
bool pdl_enabled();

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  EDX_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

inline void invalid(const std::string& m) { throw Error(EDX_INVALID_ARGUMENT, m); }
inline void logic(const std::string& m) { throw Error(EDX_LOGIC_ERROR, m); }

// Name of the kernel each phase launched last on this thread (the bench's
// labels; edx_engine_last_kernels): [0] cost build, [1] exact solver, [2] greedy.
enum KernelSlot { kKBuild = 0, kKSolver = 1, kKGreedy = 2 };
inline thread_local const char* g_kernel_name[3] = {"", "", ""};

// edx_last_error() storage (engine.cu)
void set_last_error(const char* m);

// C-ABI wrapper: exceptions -> edx_status + edx_last_error()
template <class F>
int guard(F&& f) {
  try {
    f();
    return EDX_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return EDX_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return EDX_RUNTIME_ERROR;
  }
}

// Device-side error flags (set by kernels, checked by the host after a sync).
enum DevFlag : int {
  kFlagIdOutOfRange = 0,   // an id >= id_space reached a dense-table kernel
  kFlagBadCost = 1,        // a solver input was negative or non-finite
  kFlagPinned = 2,         // every cache entry pinned (cache.hpp:164)
  kFlagUnbalanced = 3,     // a dispatch decision broke the m-per-worker balance
  kFlagKeyRange = 4,       // victim-key fields exceed the 57-bit packing
  kFlagInternal = 5,       // internal launch-configuration error (bug)
  kFlagBadBatch = 6,       // a device batch's offsets disagree with its declared id count
  kFlagCount = 8
};

constexpr int kMaxWorkers = 64;  // WorkerMask is one uint64 (types.hpp:89,124)

// --------------------------------------------------------- device buffers
// Bumped on every device (re)allocation: a captured CUDA graph bakes buffer
// addresses in, so it is only replayed while this is unchanged.
inline std::atomic<unsigned long long> g_alloc_epoch{0};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void ensure(size_t count) {
    if (count <= n && p) return;
    release();
    size_t c = count ? count : 1;
    EDX_CUDA(cudaMalloc(&p, c * sizeof(T)));
    n = c;
    g_alloc_epoch.fetch_add(1, std::memory_order_relaxed);
  }
  void swap(DevBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    g_alloc_epoch.fetch_add(1, std::memory_order_relaxed);
  }
};

// ------------------------------------------------------ kernel launchers
// cost.cu — K1 build + K2 gap keys (cost.hpp:81-146)
void launch_cost_build(const uint32_t* ids, const uint64_t* offsets, uint64_t rows, int n,
                       const ulonglong2* ol, uint64_t id_space, const double* ucost,
                       double* matrix, uint64_t* gap_keys, uint32_t* row_index, int* flags,
                       cudaStream_t s, const uint64_t* sizes = nullptr, const double* bw = nullptr);
// gap keys only, for an externally supplied matrix (rows_by_gap on a host matrix)
void launch_gap_keys(const double* matrix, uint64_t rows, int n, uint64_t* gap_keys,
                     uint32_t* row_index, cudaStream_t s);

// dispatch.cu — K3 sort, K4 greedy, decision scatter/validation/cost
struct SortScratch {
  DevBuf<uint8_t> temp;
  DevBuf<uint64_t> keys_out;
  size_t temp_bytes = 0;
};
void sort_rows_by_gap(SortScratch& sc, const uint64_t* keys_in, const uint32_t* idx_in,
                      uint32_t* idx_out, uint64_t rows, cudaStream_t s);
// K4 scratch: each position's preference list (64 bytes)
struct GreedyScratch {
  DevBuf<uint8_t> prefs;
  DevBuf<uint32_t> dest;  // per position: its decision index (row_ids[order[t]])
  DevBuf<int32_t> pw;     // per position: its worker (when the caller wants rows only)
  DevBuf<unsigned long long> stats;  // EDX_GREEDY_STATS=1 only
};
void launch_greedy(const double* matrix, uint64_t rows, int n, const uint32_t* order,
                   uint64_t n_order, const int32_t* capacity_dev, int cap_uniform,
                   int32_t* decision, const uint32_t* row_ids, int32_t* pair_worker,
                   int* flags, GreedyScratch& g, cudaStream_t s);
void launch_check_balance(const int32_t* decision, uint64_t rows, int n, int m, int* flags,
                          DevBuf<int>& counts, cudaStream_t s);
void launch_decision_cost(const double* matrix, const int32_t* decision, uint64_t rows, int n,
                          double* out, cudaStream_t s);

// hungarian.cu — K6 block-collapsed e-maxx and K5 dense e-maxx (assign.hpp:80-157)
struct HungarianScratch {
  DevBuf<int64_t> s64;   // global fallback for the scaled cost rows
  DevBuf<uint8_t> arena; // global fallback for the solver arrays
  DevBuf<unsigned long long> steps;
};
// Collapsed solver on the column-expanded block of `k = n*mult` rows
// order[0..k) of matrix; writes decision[row_ids? row_ids[row]: row] = worker
// (or col_of_row[r] when col_of_row != nullptr).
void launch_hungarian_blocks(HungarianScratch& sc, const double* matrix, int n,
                             const uint32_t* order, int mult, int32_t* decision,
                             const uint32_t* row_ids, uint64_t* col_of_row, int* flags,
                             cudaStream_t s, int device);
void launch_hungarian_dense(HungarianScratch& sc, const double* values, uint64_t k,
                            uint64_t* col_of_row, int* flags, cudaStream_t s, int device);
unsigned long long last_hungarian_steps(HungarianScratch& sc, cudaStream_t s);
// [0] steps [1] step-loop cycles [2] potential cycles [3] augment cycles
// [4] re-key cycles [5] augment hops [6] consumed prefixes [7] total cycles
void last_hungarian_stats(HungarianScratch& sc, cudaStream_t s, unsigned long long* out);

// The EcoMix pipeline on a device matrix (assign.hpp:247-285).
struct DispatchScratch {
  SortScratch sort;
  DevBuf<int> balance;  // k_check_balance: per-worker counts + finished blocks
  HungarianScratch hung;
  DevBuf<uint64_t> gap_keys;
  DevBuf<uint32_t> row_index, order;
  GreedyScratch greedy;
  DevBuf<double> cost;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  ~DispatchScratch();
  void init(int device);
};
// Phase events (may be null) bracket gap/sort, exact solve, greedy.
struct PhaseEvents {
  cudaEvent_t sort0 = nullptr, sort1 = nullptr, exact0 = nullptr, exact1 = nullptr,
              greedy0 = nullptr, greedy1 = nullptr;
};
int exact_multiplicity(int m, double alpha);
// `gap_ready` = gap keys/row index already produced by the build epilogue.
void run_ecomix(DispatchScratch& sc, const double* matrix, uint64_t rows, int n, int m,
                double alpha, bool gap_ready, int32_t* decision, int* flags, cudaStream_t s,
                int device, const PhaseEvents* ev, int* launches);

// hitgreedy.cu — K8 baseline_hitgreedy (assign.hpp:346-392)
struct HitScratch {
  DevBuf<int32_t> scores;
  DevBuf<uint32_t> keys, keys_sorted, index, index_sorted;
  DevBuf<uint8_t> temp;
};
void launch_hitgreedy(HitScratch& sc, const uint32_t* ids, const uint64_t* offsets, uint64_t rows,
                      int n, int m, const ulonglong2* ol, uint64_t id_space, int32_t* decision,
                      int* flags, cudaStream_t s);

}  // namespace edx
