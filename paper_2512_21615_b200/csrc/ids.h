// The engine's device id table (ids.cu): uint32 embedding id -> dense slot.
#pragma once

#include "edx_internal.cuh"

namespace edx {

struct IdTable {
  DevBuf<unsigned long long> tab;    // tab_size entries (id << 32 | slot), EMPTY = ~0
  DevBuf<uint32_t> slot2id;          // cap entries
  DevBuf<unsigned long long> count;  // slots allocated (device)
  uint64_t tab_size = 0, cap = 0;
  uint64_t used = 0;                 // host copy of `count` as of the last sync
};

// An empty table for slot_cap slots.
void id_table_init(IdTable& t, uint64_t slot_cap, cudaStream_t s);
// slots[t] = slot of ids[t] for t < T; new ids are inserted when `insert`
// (the caller guarantees used + T <= cap), else absent ids give 0xFFFFFFFF.
void id_table_translate(IdTable& t, const uint32_t* ids, uint64_t T, uint32_t* slots, bool insert,
                        int* flags, cudaStream_t s);
// Grows to slot_cap slots (t.used must be current): slot2id keeps its
// prefix, the table is rebuilt.  Synchronises the stream.
void id_table_grow(IdTable& t, uint64_t slot_cap, cudaStream_t s);

}  // namespace edx
