// Drop-in for the reference's cache.hpp.  A WorkerCache built by the
// reference's constructor (capacity, policy, footprint) is a device-resident
// cache driven entry by entry through libedx (workercache.cu): touch,
// set_version, erase, select_victim and evict_for under either victim
// policy.  SimState's own caches are updated a batch at a time on the device
// (step.cu); SimState::cache(j) returns a read-only host view of one of them
// with the same accessors.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <tuple>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

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

// cache.hpp:73-240.
class WorkerCache {
 public:
  using FootprintFn = std::function<double(EmbeddingId)>;
  using NeedsPushFn = std::function<bool(EmbeddingId)>;
  using PinnedSet = std::unordered_set<EmbeddingId>;

  WorkerCache() = default;
  // cache.hpp:79-84: a standalone cache on the current device.
  explicit WorkerCache(std::size_t capacity, VictimPolicy policy = VictimPolicy::kMarkVersion,
                       FootprintFn footprint = nullptr)
      : capacity_(capacity), footprint_(std::move(footprint)) {
    int dev = 0;
    edx_cache* h = nullptr;
    edxc::check(edx_cache_create(capacity, policy == VictimPolicy::kPriorityRatio ? 1 : 0, dev, &h));
    dev_ = std::shared_ptr<edx_cache>(h, edx_cache_destroy);
  }
  // Read-only view of a SimState cache (SimState::cache(j)).
  WorkerCache(std::size_t capacity, std::uint32_t current_mark,
              std::unordered_map<EmbeddingId, CacheEntry> entries)
      : capacity_(capacity), current_mark_(current_mark), entries_(std::move(entries)) {}

  std::size_t capacity() const { return capacity_; }
  std::size_t size() const {
    if (!dev_) return entries_.size();
    uint64_t n = 0;
    edxc::check(edx_cache_info(dev_.get(), &n, nullptr, nullptr));
    return static_cast<std::size_t>(n);
  }
  bool full() const { return size() == capacity_; }
  std::size_t free_slots() const { return capacity_ - size(); }
  std::uint32_t current_mark() const {
    if (!dev_) return current_mark_;
    uint32_t m = 0;
    edxc::check(edx_cache_info(dev_.get(), nullptr, &m, nullptr));
    return m;
  }
  bool resident(EmbeddingId id) const { return find(id) != nullptr; }
  const CacheEntry* find(EmbeddingId id) const {
    if (!dev_) {
      auto it = entries_.find(id);
      return it == entries_.end() ? nullptr : &it->second;
    }
    int found = 0, ver = 0;
    uint32_t mark = 0, freq = 0;
    uint64_t last = 0;
    edxc::check(edx_cache_find(dev_.get(), id, &found, &ver, &mark, &freq, &last));
    if (!found) return nullptr;
    // per-id storage: a pointer from an earlier find() of another id stays
    // valid and unchanged (it shows that id's entry as of its own find())
    CacheEntry& slot = found_[id];
    slot = CacheEntry{id, ver != 0, mark, freq, last};
    return &slot;
  }
  // cache.hpp:102-122
  void touch(EmbeddingId id, bool latest, std::uint64_t now) {
    edxc::check(edx_cache_touch(device(), id, latest ? 1 : 0, now, footprint_ ? footprint_(id) : 1.0));
  }
  // cache.hpp:126-135
  void set_version(EmbeddingId id, bool latest) {
    edxc::check(edx_cache_set_version(device(), id, latest ? 1 : 0));
  }
  // cache.hpp:141-148
  EmbeddingId select_victim() const {
    uint32_t v = 0;
    edxc::check(edx_cache_select_victim(device(), &v));
    return v;
  }
  // cache.hpp:152-170
  std::vector<std::pair<EmbeddingId, bool>> evict_for(std::size_t needed,
                                                      const NeedsPushFn& needs_push,
                                                      const PinnedSet* pinned = nullptr) {
    std::vector<uint32_t> pins;
    if (pinned) pins.assign(pinned->begin(), pinned->end());
    std::vector<uint32_t> out(capacity_ + 1);
    uint64_t n = 0;
    edxc::check(edx_cache_evict_for(device(), needed, pins.data(), pins.size(), out.data(), &n));
    std::vector<std::pair<EmbeddingId, bool>> evicted;
    for (uint64_t t = 0; t < n; ++t)
      evicted.emplace_back(out[t], needs_push ? needs_push(out[t]) : false);
    return evicted;
  }
  // cache.hpp:172-178
  void erase(EmbeddingId id) { edxc::check(edx_cache_erase(device(), id)); }
  const std::unordered_map<EmbeddingId, CacheEntry>& entries() const {
    if (!dev_) return entries_;
    uint64_t n = 0;
    edxc::check(edx_cache_export(dev_.get(), nullptr, nullptr, nullptr, nullptr, nullptr, 0, &n));
    std::vector<uint32_t> ids(n), mark(n), freq(n);
    std::vector<uint8_t> ver(n);
    std::vector<uint64_t> last(n);
    edxc::check(edx_cache_export(dev_.get(), ids.data(), ver.data(), mark.data(), freq.data(),
                                 last.data(), n, &n));
    entries_.clear();
    for (uint64_t t = 0; t < n; ++t)
      entries_[ids[t]] = CacheEntry{ids[t], ver[t] != 0, mark[t], freq[t], last[t]};
    return entries_;
  }

 private:
  edx_cache* device() const {
    if (!dev_) throw std::logic_error("read-only view of a SimState cache");
    return dev_.get();
  }

  std::size_t capacity_ = 0;
  std::uint32_t current_mark_ = 1;
  FootprintFn footprint_;
  std::shared_ptr<edx_cache> dev_;
  mutable std::unordered_map<EmbeddingId, CacheEntry> found_;
  mutable std::unordered_map<EmbeddingId, CacheEntry> entries_;
};

}  // namespace embdispatch
