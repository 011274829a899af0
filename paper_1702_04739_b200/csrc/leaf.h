// Constant-time successor of a pairwise-sum leaf (host + device).
//
// numpy's pairwise_sum splits a run of n elements at floor(n/2) rounded down
// to a multiple of 8.  In octets (M = total >> 3 full octets; the r0 =
// total & 7 extra elements always stay in the rightmost node) a node of x
// octets splits into floor(x/2) and ceil(x/2), so the node reached by path
// bits b_1..b_t (b = 1: right) holds floor((M + sum_k b_k 2^(k-1)) / 2^t)
// octets, i.e. count(t, i) = floor((M + rev_t(i)) >> t) for index i at depth
// t.  Every node above depth T = t_a + 1 (t_a: last depth whose smallest
// count is >= 17 octets) splits, and a depth-T node is either a leaf or
// splits once more into two leaves.  Walking the depth-T nodes left to right
// therefore enumerates the leaves in flat order with O(1) work per leaf.
#pragma once
#include <cstdint>

#ifndef ISOC_HD
#ifdef __CUDACC__
#define ISOC_HD __host__ __device__ __forceinline__
#else
#define ISOC_HD inline
#endif
#endif

namespace isoc {

ISOC_HD uint64_t rev_bits(uint64_t i, int t) {
    if (t == 0) return 0;
#ifdef __CUDA_ARCH__
    return __brevll(i) >> (64 - t);
#else
    uint64_t r = 0;
    for (int k = 0; k < t; ++k) r |= ((i >> k) & 1ull) << (t - 1 - k);
    return r;
#endif
}

// elements of node (t, i)
ISOC_HD int64_t node_len(uint64_t M, int r0, int t, uint64_t i) {
    const int64_t oct = (int64_t)((M + rev_bits(i, t)) >> t);
    return 8 * oct + ((i + 1 == (1ull << t)) ? r0 : 0);
}

ISOC_HD int leaf_base_depth(int64_t total) {
    const uint64_t M = (uint64_t)total >> 3;
    int t = 0;
    if (M >= 17) {
        while ((M >> (t + 1)) >= 17) ++t;
        ++t;
    }
    return t;
}

// Iterator over leaves: the current leaf and its place among depth-T nodes.
struct LeafIter {
    int64_t start;
    int64_t len;
    uint64_t i;   // depth-T node index
    int sub;      // 0: the depth-T node is the leaf, 1: its left child, 2: its right child
    int T;
    ISOC_HD uint64_t hid() const {
        return sub == 0 ? ((1ull << T) | i) : ((1ull << (T + 1)) | (2 * i + (sub == 2 ? 1 : 0)));
    }
};

// Position an iterator on a leaf given by (start, len, heap id).
ISOC_HD LeafIter leaf_iter_from(int64_t total, int64_t start, int64_t len, uint64_t hid) {
    LeafIter it;
    it.start = start;
    it.len = len;
    it.T = leaf_base_depth(total);
    int depth = 63;
    while (depth > 0 && !((hid >> depth) & 1ull)) --depth;
    const uint64_t idx = hid - (1ull << depth);
    if (depth == it.T) {
        it.i = idx;
        it.sub = 0;
    } else {  // depth T + 1
        it.i = idx >> 1;
        it.sub = (idx & 1ull) ? 2 : 1;
    }
    return it;
}

// Advance to the next leaf (caller checks start + len < total).
ISOC_HD void leaf_next(LeafIter& it, int64_t total) {
    const uint64_t M = (uint64_t)total >> 3;
    const int r0 = (int)(total & 7);
    const int64_t nstart = it.start + it.len;
    if (it.sub == 1) {
        it.sub = 2;
        it.start = nstart;
        it.len = node_len(M, r0, it.T + 1, 2 * it.i + 1);
        return;
    }
    it.i += 1;
    it.start = nstart;
    const int64_t L = node_len(M, r0, it.T, it.i);
    if (L <= 128) {
        it.sub = 0;
        it.len = L;
    } else {
        it.sub = 1;
        it.len = node_len(M, r0, it.T + 1, 2 * it.i);
    }
}

}  // namespace isoc
