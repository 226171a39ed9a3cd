// The edx_engine object: one SimState (sim.hpp:54-268) resident on one GPU.
#pragma once

#include <memory>
#include <vector>

#include "edx_internal.cuh"
#include "ids.h"

namespace edx {

// Device-resident per-worker caches (WorkerCache, cache.hpp:73-240).  Entry
// metadata lives in per-worker slot arrays (capacity entries each); a slot is
// located by slot_of[j * id_space + id].  The version flag is not stored: the
// reference keeps CacheEntry::version_latest equal to the worker's bit of the
// global `latest` mask at all times (validate_consistency, sim.hpp:229-231),
// so the step reads it from the mask.
struct CacheState {
  DevBuf<int32_t> slot_of;   // n * id_space, -1 = not resident
  DevBuf<uint32_t> sid;      // n * capacity : id in slot
  DevBuf<uint32_t> smark;    // mark (cache.hpp:39)
  DevBuf<uint32_t> sfreq;    // frequency (cache.hpp:40)
  DevBuf<uint32_t> slast;    // last_access (cache.hpp:41), < 2^32 enforced
  DevBuf<uint32_t> size;     // n
  DevBuf<uint32_t> cur_mark; // n (current_mark_, cache.hpp:236)
  DevBuf<unsigned long long> at_cur;  // n (at_current_mark_, cache.hpp:237)
  DevBuf<uint32_t> pin;      // n * capacity, large caches: iteration stamp of pinned entries
};

// Scratch of one SimState::step (sim.hpp:87-218).
struct StepScratch {
  DevBuf<uint32_t> occ_sample;   // occurrence -> sample
  DevBuf<int32_t> first_pos;     // id_space: first occurrence of the id in the batch (or INT_MAX)
  DevBuf<uint32_t> uidx_of_pos;  // occurrence -> unique index (valid at first occurrences)
  DevBuf<uint32_t> upos;         // occurrence -> unique index of its id (every occurrence)
  DevBuf<int32_t> item_slot;     // need item -> cache slot of a resident id (k_classify)
  DevBuf<uint32_t> uniq;         // unique ids in first-appearance order
  DevBuf<unsigned long long> umask;  // trainers mask per unique id
  DevBuf<unsigned long long> need_first;  // n * U : epoch << 32 | ~first position of (j, id)
  DevBuf<unsigned long long> need_cnt;    // n * U : epoch << 32 | occurrences of (j, id)
  DevBuf<uint32_t> epoch;                 // step counter tagging the need cells
  DevBuf<uint8_t> flag;          // per occurrence: 1 = first occurrence of (worker, id)
  DevBuf<uint32_t> flag_scan;    // scratch
  DevBuf<uint64_t> need_key;     // (worker << 32 | pos) of first occurrences
  DevBuf<uint64_t> need_key_sorted;
  DevBuf<uint32_t> need_off;     // n + 1 : CSR of the need lists
  DevBuf<uint8_t> need_type;     // 0 hit, 1 refresh, 2 insert
  DevBuf<int32_t> need_contrib;  // epoch-scan contribution
  DevBuf<uint32_t> ins_rank;     // insert ordinal within the worker
  DevBuf<unsigned long long> counters;  // per-worker counters + totals
  DevBuf<uint32_t> cand_slot_sorted;  // victims per worker (sorted for small caches)
  DevBuf<uint32_t> cand_count;   // victim ids
  DevBuf<uint32_t> cand_off;     // worker list
  DevBuf<uint32_t> wscalars;     // per-worker scalars of the step
  // large caches: the cooperative victim selection (k_big_select)
  DevBuf<uint8_t> big_state;     // n BigState
  DevBuf<uint32_t> big_hist;     // n * 4096
  DevBuf<uint8_t> big_key[2];    // n * capacity 128-bit keys (undecided, ping-pong)
  DevBuf<uint32_t> big_slot[2];  // n * capacity
  DevBuf<uint8_t> big_eflag;     // n * capacity: candidate / version bits of each entry
  uint64_t big_grid = 0;
  DevBuf<uint8_t> temp;          // CUB temp storage
  DevBuf<uint32_t> ucount;       // number of unique ids
};

}  // namespace edx

struct edx_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  int n = 0, m = 0;
  double alpha = 1.0;
  uint64_t capacity = 0, d_tran = 0;
  std::vector<double> bw, ucost_h;
  // id_space = the slot count of the dense per-embedding tables.  Dense mode
  // (created with id_space > 0): slot = id, ids must be < id_space.  Hashed
  // mode (created with id_space 0): any uint32 id, mapped to a slot by the
  // device id table (ids.cu) at the start of each iteration; the tables grow.
  uint64_t id_space = 0, max_ids = 0;
  bool hashed = false;
  edx::IdTable idt;
  edx::DevBuf<uint32_t> kslots;        // the current batch as slots (hashed mode)
  const uint32_t* cur_raw = nullptr;   // the current batch's ids as loaded
  bool translated = true;
  uint64_t used_bound = 0;             // >= slots in use (exact after each sync)
  unsigned long long* h_used = nullptr;  // pinned copy of idt.count
  int rank = 0, world = 1;
  void* comm = nullptr;  // ncclComm_t when world > 1; rank 0 is the solver rank
  uint64_t clock = 0;
  // bumped by every state mutation (step, seed_entry, imports): a Snapshot
  // view of the device state is current while this is unchanged
  uint64_t state_version = 0;

  // global per-embedding state (SimState::global_, sim.hpp:266), dense by id
  edx::DevBuf<ulonglong2> ol;             // {owners, latest}
  edx::DevBuf<unsigned long long> res;    // resident
  edx::DevBuf<double> ucost;
  edx::CacheState cache;
  edx::StepScratch step;

  // current batch
  edx::DevBuf<uint32_t> ids;
  edx::DevBuf<uint64_t> offsets;
  const uint32_t* cur_ids = nullptr;
  const uint64_t* cur_offsets = nullptr;
  uint64_t rows = 0, total_ids = 0;
  std::vector<uint64_t> h_offsets;  // host copy of the current offsets

  // per-iteration products
  edx::DevBuf<double> matrix;
  edx::DevBuf<int32_t> decision;
  edx::DevBuf<double> expected;
  edx::DispatchScratch disp;
  edx::HitScratch hit;
  bool built = false, gap_ready = false, dispatched = false;
  bool expected_ready = false;  // the last EcoMix dispatch's decision_cost is enqueued

  edx::DevBuf<int> flags;
  int* h_flags = nullptr;            // pinned
  unsigned long long* h_counters = nullptr;  // pinned
  double* h_expected = nullptr;      // pinned
  uint32_t* h_clock = nullptr;       // pinned: the iteration clock, copied to d_clock in-stream
  edx::DevBuf<uint32_t> d_clock;
  // the decision-independent head of the step runs on its own stream during
  // a fused iteration's build and dispatch (step_head / step_run)
  cudaStream_t step_side = nullptr;
  // input prefetch (edx_engine_prefetch): two device slots filled on copy_stream
  struct Prefetch {
    edx::DevBuf<uint32_t> ids;
    edx::DevBuf<uint64_t> offsets;
    uint64_t* h_offsets = nullptr;  // pinned, base-adjusted offsets
    uint64_t h_cap = 0;
    cudaEvent_t ready = nullptr, free = nullptr;
    bool valid = false, used = false;
    const void* host_ids = nullptr;
    const void* host_offsets = nullptr;
    uint64_t rows = 0, total = 0;
  } pf[2];
  int pf_next = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t head_fork = nullptr, head_done = nullptr;
  bool head_pending = false;

  // CUDA graph of one fused iteration (build -> dispatch -> step), replayed
  // while the shape is unchanged; eligible on one GPU, with device-decided
  // victims (caches <= kSelCap) and profiling off
  int graph_mode = -1;               // -1: undecided (env EDX_GRAPH, default on); 0 off; 1 on
  cudaGraphExec_t gexec = nullptr;
  uint64_t g_rows = 0, g_total = 0;
  double g_alpha = -1.0;
  uint64_t g_launches = 0;
  unsigned long long g_epoch = 0;  // edx::g_alloc_epoch at capture
  bool capturing = false;

  // the kernels the last build / exact solve / greedy launched (bench labels)
  const char* kname[3] = {"", "", ""};

  // profiling
  bool profiling = false;
  cudaEvent_t ev[12] = {};
  cudaEvent_t cost_done = nullptr;  // decision_cost finished (side stream)
  double phase_ms[EDX_NUM_PHASES] = {};
  uint64_t launches = 0;
  uint64_t solver_steps = 0;
  bool pending_build = false, pending_dispatch = false, pending_step = false,
       pending_greedy = false;
};
