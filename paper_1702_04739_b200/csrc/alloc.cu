// Stream-ordered device scratch with a host-side block cache.
//
// Every pipeline run allocates the same scratch sizes (sigma's wave slots,
// omega's subtree slots, the MST handle, the tree, the sweeps).  Served by
// cudaMallocAsync each time, those calls occasionally stall the host for
// 30-300 ms on the B200 boxes (measured: an 8 MB cudaMallocAsync taking
// 59 ms inside the MST phase, with the pool's reserved size unchanged), so a
// freed block is kept here, keyed by (device, stream, size), and handed to
// the next request of the same size on the same stream: in stream order the
// free precedes every later use on that stream, so the reuse is safe without
// any synchronisation.  Requests of other sizes or streams go to the pool.
// The cache is bounded (kCacheMax) and is flushed back to the pool when an
// allocation fails, before retrying; evictions use cudaFree, which waits for
// the device, so a block still in use on its stream is never released early.
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/isoclust_b200.h"
#include "common.cuh"

namespace isoc {

namespace {

constexpr size_t kCacheMax = (size_t)96 << 30;

struct Live {
    size_t bytes;
    int dev;
};
using Key = std::tuple<int, cudaStream_t, size_t>;

struct Cache {
    std::mutex mu;
    std::unordered_map<void*, Live> live;
    std::map<Key, std::vector<void*>> free_blocks;
    std::vector<std::pair<Key, void*>> order;   // cached blocks, oldest first (eviction)
    size_t cached = 0;
};

Cache& cache() {
    static Cache* c = new Cache();   // never destroyed: frees at exit would race the context teardown
    return *c;
}

// Return `bytes` or more of the oldest cached blocks of device `dev` to the
// pool (all of them when bytes == SIZE_MAX).  Caller holds the lock.
void evict_locked(Cache& c, int dev, size_t bytes) {
    size_t freed = 0;
    std::vector<std::pair<Key, void*>> keep;
    keep.reserve(c.order.size());
    for (auto& kv : c.order) {
        const Key& k = kv.first;
        if (freed >= bytes || std::get<0>(k) != dev) {
            keep.push_back(kv);
            continue;
        }
        auto it = c.free_blocks.find(k);
        if (it == c.free_blocks.end()) continue;
        auto& v = it->second;
        bool found = false;
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i] == kv.second) {
                v.erase(v.begin() + (long)i);
                found = true;
                break;
            }
        if (!found) continue;
        if (v.empty()) c.free_blocks.erase(it);
        cudaFree(kv.second);
        c.cached -= std::get<2>(k);
        freed += std::get<2>(k);
    }
    c.order.swap(keep);
}

}  // namespace

cudaError_t isoc_malloc_async(void** p, size_t bytes, cudaStream_t st) {
    if (bytes == 0) bytes = 1;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    Cache& c = cache();
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto it = c.free_blocks.find(Key{dev, st, bytes});
        if (it != c.free_blocks.end() && !it->second.empty()) {
            void* q = it->second.back();
            it->second.pop_back();
            if (it->second.empty()) c.free_blocks.erase(it);
            for (size_t i = c.order.size(); i-- > 0;)
                if (c.order[i].second == q) {
                    c.order.erase(c.order.begin() + (long)i);
                    break;
                }
            c.cached -= bytes;
            c.live[q] = Live{bytes, dev};
            *p = q;
            return cudaSuccess;
        }
    }
    e = cudaMallocAsync(p, bytes, st);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();   // clear the sticky-free allocation error
        {
            std::lock_guard<std::mutex> g(c.mu);
            evict_locked(c, dev, SIZE_MAX);
        }
        e = cudaMallocAsync(p, bytes, st);
    }
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(c.mu);
    c.live[*p] = Live{bytes, dev};
    return cudaSuccess;
}

cudaError_t isoc_free_async(void* p, cudaStream_t st) {
    if (p == nullptr) return cudaSuccess;
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return cudaFreeAsync(p, st);   // not ours
    const Live l = it->second;
    c.live.erase(it);
    const Key k{l.dev, st, l.bytes};
    c.free_blocks[k].push_back(p);
    c.order.emplace_back(k, p);
    c.cached += l.bytes;
    if (c.cached > kCacheMax) evict_locked(c, l.dev, c.cached - kCacheMax);
    return cudaSuccess;
}

}  // namespace isoc

extern "C" int isoc_release_cached_memory(unsigned long long* released_bytes_host) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return ISOC_ECUDA;
    isoc::Cache& c = isoc::cache();
    std::lock_guard<std::mutex> g(c.mu);
    const size_t before = c.cached;
    isoc::evict_locked(c, dev, SIZE_MAX);
    if (released_bytes_host) *released_bytes_host = (unsigned long long)(before - c.cached);
    return ISOC_OK;
}
