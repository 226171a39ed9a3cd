// Drop-in for the reference's cache.hpp data types.  The caches themselves
// live on the device (libedx step.cu implements WorkerCache::touch /
// set_version / evict_for for the whole batch at once); SimState::cache(j)
// returns a read-only host view of one worker's cache built from the device
// tables, with the reference's accessors.
#pragma once

#include <cstdint>
#include <tuple>
#include <unordered_map>

#include "embdispatch/types.hpp"

namespace embdispatch {

// cache.hpp:36-42.
struct CacheEntry {
  EmbeddingId id = 0;
  bool version_latest = true;
  std::uint32_t mark = 1;
  std::uint32_t frequency = 1;
  std::uint64_t last_access = 0;
};

// cache.hpp:47-58: eviction order, ascending.
struct VictimKey {
  bool version_latest;
  std::uint32_t mark;
  std::uint32_t frequency;
  std::uint64_t last_access;
  EmbeddingId id;
  friend bool operator<(const VictimKey& a, const VictimKey& b) {
    return std::tie(a.version_latest, a.mark, a.frequency, a.last_access, a.id) <
           std::tie(b.version_latest, b.mark, b.frequency, b.last_access, b.id);
  }
};

inline VictimKey victim_key(const CacheEntry& e) {
  return VictimKey{e.version_latest, e.mark, e.frequency, e.last_access, e.id};
}

enum class VictimPolicy { kMarkVersion, kPriorityRatio };

// Read-only view of one device-resident WorkerCache (cache.hpp:73-240).
class WorkerCache {
 public:
  WorkerCache() = default;
  WorkerCache(std::size_t capacity, std::uint32_t current_mark,
              std::unordered_map<EmbeddingId, CacheEntry> entries)
      : capacity_(capacity), current_mark_(current_mark), entries_(std::move(entries)) {}
  std::size_t capacity() const { return capacity_; }
  std::size_t size() const { return entries_.size(); }
  bool full() const { return entries_.size() == capacity_; }
  std::size_t free_slots() const { return capacity_ - entries_.size(); }
  std::uint32_t current_mark() const { return current_mark_; }
  bool resident(EmbeddingId id) const { return entries_.count(id) != 0; }
  const CacheEntry* find(EmbeddingId id) const {
    auto it = entries_.find(id);
    return it == entries_.end() ? nullptr : &it->second;
  }
  const std::unordered_map<EmbeddingId, CacheEntry>& entries() const { return entries_; }

 private:
  std::size_t capacity_ = 0;
  std::uint32_t current_mark_ = 1;
  std::unordered_map<EmbeddingId, CacheEntry> entries_;
};

}  // namespace embdispatch
