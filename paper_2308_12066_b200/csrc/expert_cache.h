// expert_cache.h — HBM expert cache with the reference's LIFO / LFU / LRU
// victim rules (cache.py:49-103), keyed by (block, expert).  Entries are
// whole expert records, so the byte capacity is a record count.  The policy
// is a pure function of the access sequence (the property the reference's
// replay oracle checks); the runtime maps each entry to a slot of an HBM
// region and orders slot reuse with CUDA events.
#pragma once
#include <cstdint>
#include <map>
#include <utility>
#include <vector>

namespace pgmoe {

enum CachePolicy { kCacheNone = 0, kCacheLifo = 1, kCacheLfu = 2, kCacheLru = 3 };

struct CacheOutcome {
    bool hit = false, inserted = false;
    int slot = -1;               // HBM slot holding the entry (hit or inserted)
    std::vector<int64_t> evicted;  // keys
};

class ExpertCacheIndex {
  public:
    ExpertCacheIndex(int capacity_records, int policy) : cap_(capacity_records), policy_(policy) {
        for (int s = capacity_records - 1; s >= 0; --s) free_.push_back(s);
    }
    static int64_t key(int block, int expert) { return ((int64_t)block << 32) | (uint32_t)expert; }

    // cache.py:80-103 — hits update freq / last_use; a miss evicts per policy
    // until the entry fits (entries larger than the cache bypass it).
    CacheOutcome access(int64_t k, int64_t now) {
        CacheOutcome out;
        auto it = entries_.find(k);
        if (it != entries_.end()) {
            it->second.freq += 1;
            it->second.last_use = now;
            ++hits_;
            out.hit = true;
            out.slot = it->second.slot;
            return out;
        }
        ++misses_;
        if (cap_ < 1) return out;  // bypass
        while ((int)entries_.size() + 1 > cap_) {
            auto v = victim();
            free_.push_back(v->second.slot);
            out.evicted.push_back(v->first);
            entries_.erase(v);
        }
        Entry e;
        e.insert_seq = seq_++;
        e.freq = 1;
        e.last_use = now;
        e.slot = free_.back();
        free_.pop_back();
        entries_[k] = e;
        out.inserted = true;
        out.slot = e.slot;
        return out;
    }
    int64_t hits() const { return hits_; }
    int64_t misses() const { return misses_; }
    int capacity() const { return cap_; }

  private:
    struct Entry {
        int64_t insert_seq = 0, freq = 0, last_use = 0;
        int slot = -1;
    };
    // cache.py:70-78
    std::map<int64_t, Entry>::iterator victim() {
        auto best = entries_.begin();
        for (auto it = entries_.begin(); it != entries_.end(); ++it) {
            const Entry &a = it->second, &b = best->second;
            bool better = false;
            if (policy_ == kCacheLifo) better = a.insert_seq > b.insert_seq;
            else if (policy_ == kCacheLfu) better = a.freq < b.freq || (a.freq == b.freq && a.insert_seq < b.insert_seq);
            else better = a.last_use < b.last_use || (a.last_use == b.last_use && a.insert_seq < b.insert_seq);
            if (better) best = it;
        }
        return best;
    }
    int cap_, policy_;
    int64_t seq_ = 0, hits_ = 0, misses_ = 0;
    std::map<int64_t, Entry> entries_;
    std::vector<int> free_;
};

}  // namespace pgmoe
