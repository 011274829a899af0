// Tree construction on the device.
//
//  * MST rooting (replaces the parent/depth/child_id bookkeeping of prim_mst
//    and _bfs_root_first, /root/reference/pkg/src/isoclust/mst.py:46-65,
//    128-181): adjacency lists sorted by (d, neighbour) -- Prim's sibling rank
//    equals the rank of (d(parent,u), u) among siblings -- then a
//    level-synchronous BFS in one cooperative kernel that assigns BFS
//    positions, parents, depths and child ranks.
//  * tree_from_parent_list (mst.py:78-125): children grouped by parent in
//    ascending vertex order via a stable radix sort, then the same BFS.
//  * parent flows exp(-d/sigma) (mst.py:168-170) and bracket extrema
//    (affinity.py:260-279) with the reference's pow2 zero-padded fold.
#include <cstdint>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace isoc {

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__global__ void degree_kernel(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                              int64_t m, int32_t* __restrict__ deg) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    atomicAdd(&deg[eu[e]], 1);
    atomicAdd(&deg[ev[e]], 1);
}

__global__ void fill_adj_kernel(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev,
                                const double* __restrict__ ed, int64_t m,
                                int32_t* __restrict__ cursor, int32_t* __restrict__ adj,
                                double* __restrict__ adjd) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    int32_t s = atomicAdd(&cursor[eu[e]], 1);
    adj[s] = ev[e];
    adjd[s] = ed[e];
    s = atomicAdd(&cursor[ev[e]], 1);
    adj[s] = eu[e];
    adjd[s] = ed[e];
}

// insertion sort of each adjacency list by (d, neighbour)
__global__ void sort_adj_kernel(const int32_t* __restrict__ off, int64_t n, int32_t* __restrict__ adj,
                                double* __restrict__ adjd) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int32_t a = off[v], b = off[v + 1];
    for (int32_t i = a + 1; i < b; ++i) {
        const int32_t w = adj[i];
        const double dw = adjd[i];
        int32_t j = i - 1;
        while (j >= a && (adjd[j] > dw || (adjd[j] == dw && adj[j] > w))) {
            adj[j + 1] = adj[j];
            adjd[j + 1] = adjd[j];
            --j;
        }
        adj[j + 1] = w;
        adjd[j + 1] = dw;
    }
}

struct BfsArgs {
    int64_t n;
    int64_t root;
    int undirected;              // skip the parent entry in adjacency lists
    const int32_t* off;          // n+1
    const int32_t* adj;
    const double* adjd;          // may be null (tree_from_parent_list)
    int32_t* bfs;                // position -> vertex
    int32_t* pos_of;             // vertex -> position
    int32_t* parent_v;           // vertex -> parent vertex (-1 at root)
    int32_t* depth_v;            // vertex -> depth
    int32_t* child_id_v;         // vertex -> sibling rank (written when undirected)
    double* parent_d;            // vertex -> parent edge weight (undirected only)
    int32_t* pos_parent;         // position -> parent position
    int32_t* child_lo;           // position -> first child position
    int32_t* child_cnt;          // position -> number of children
    int64_t* level_off;          // level boundaries (capacity n+2)
    int32_t* scratch_cnt;        // per-position child counts / offsets (n)
    int32_t* chunk_sum;          // gridDim.x
    int64_t* out_levels;         // number of levels
    unsigned int* bar;
};

__device__ __forceinline__ int32_t child_count(const BfsArgs& A, int32_t v) {
    int32_t c = A.off[v + 1] - A.off[v];
    if (A.undirected && v != A.root) c -= 1;
    return c;
}

__global__ void __launch_bounds__(512) bfs_kernel(BfsArgs A) {
    __shared__ int32_t warp_tot[16];
    __shared__ int64_t s_base, s_total;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    if (b == 0 && tid == 0) {
        A.bfs[0] = (int32_t)A.root;
        A.pos_of[A.root] = 0;
        A.parent_v[A.root] = -1;
        A.depth_v[A.root] = 0;
        A.pos_parent[0] = -1;
        if (A.undirected) { A.child_id_v[A.root] = 0; A.parent_d[A.root] = 0.0; }
        A.level_off[0] = 0;
        A.level_off[1] = 1;
    }
    grid_barrier(A.bar);
    int64_t lo = 0, hi = 1;
    int level = 0;
    while (true) {
        const int64_t W = hi - lo;
        const int64_t cb = lo + W * b / G, ce = lo + W * (b + 1) / G;
        // phase 1: per-position child counts, chunk-local exclusive scan
        int64_t carry = 0;
        for (int64_t base = cb; base < ce; base += blockDim.x) {
            const int64_t p = base + tid;
            int32_t c = 0;
            if (p < ce) c = child_count(A, A.bfs[p]);
            int32_t x = c;
            for (int o = 1; o < 32; o <<= 1) {
                int32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) warp_tot[wid] = x;
            __syncthreads();
            if (wid == 0) {
                int32_t t = lane < nw ? warp_tot[lane] : 0;
                for (int o = 1; o < 32; o <<= 1) {
                    int32_t y = __shfl_up_sync(0xffffffffu, t, o);
                    if (lane >= o) t += y;
                }
                if (lane < nw) warp_tot[lane] = t;
            }
            __syncthreads();
            const int32_t wpre = wid > 0 ? warp_tot[wid - 1] : 0;
            if (p < ce) A.scratch_cnt[p] = (int32_t)(carry + wpre + x - c);
            carry += warp_tot[nw - 1];
            __syncthreads();
        }
        if (tid == 0) A.chunk_sum[b] = (int32_t)carry;
        grid_barrier(A.bar);
        // chunk base and level total
        if (tid == 0) {
            int64_t pre = 0, tot = 0;
            for (int q = 0; q < G; ++q) {
                const int64_t s = A.chunk_sum[q];
                if (q < b) pre += s;
                tot += s;
            }
            s_base = pre;
            s_total = tot;
            if (b == 0) A.level_off[level + 2] = hi + tot;
        }
        __syncthreads();
        const int64_t base_off = s_base;
        const int64_t total = s_total;
        // phase 2: write children
        for (int64_t p = cb + tid; p < ce; p += blockDim.x) {
            const int32_t v = A.bfs[p];
            const int64_t first = hi + base_off + A.scratch_cnt[p];
            const int32_t pv = A.parent_v[v];
            int32_t rank = 0;
            for (int32_t e = A.off[v]; e < A.off[v + 1]; ++e) {
                const int32_t w = A.adj[e];
                if (A.undirected && w == pv) continue;
                const int64_t q = first + rank;
                A.bfs[q] = w;
                A.pos_of[w] = (int32_t)q;
                A.parent_v[w] = v;
                A.depth_v[w] = level + 1;
                A.pos_parent[q] = (int32_t)p;
                if (A.undirected) {
                    A.child_id_v[w] = rank;
                    A.parent_d[w] = A.adjd[e];
                }
                ++rank;
            }
            A.child_lo[p] = (int32_t)first;
            A.child_cnt[p] = rank;
        }
        grid_barrier(A.bar);
        if (total == 0) {
            if (b == 0 && tid == 0) *A.out_levels = level + 1;
            break;
        }
        lo = hi;
        hi = hi + total;
        ++level;
        if (hi > A.n) {  // not a tree (cycle); stop
            if (b == 0 && tid == 0) *A.out_levels = -1;
            break;
        }
    }
}

__global__ void flows_kernel(const double* __restrict__ parent_d, const int32_t* __restrict__ parent_v,
                             int64_t n, double sigma, double* __restrict__ flow) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    flow[v] = parent_v[v] < 0 ? 0.0 : isoc_flow(parent_d[v], sigma);
}

// position-space copies used by the decision sweep
__global__ void gather_pos_kernel(const int32_t* __restrict__ bfs, int64_t n,
                                  const double* __restrict__ flow_v, const double* __restrict__ omega_v,
                                  const double* __restrict__ p_v, double* __restrict__ f_pos,
                                  double* __restrict__ om_pos, double* __restrict__ p_pos) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int32_t v = bfs[q];
    f_pos[q] = flow_v[v];
    om_pos[q] = omega_v[v];
    p_pos[q] = p_v[v];
}

// ---------------------------------------------------- parent-list input
__global__ void parent_check_kernel(const int64_t* __restrict__ parent,
                                    const int64_t* __restrict__ child_id, int64_t n, int64_t root,
                                    unsigned long long* __restrict__ keys, int32_t* __restrict__ vals,
                                    int32_t* __restrict__ pkeys, int32_t* __restrict__ bad,
                                    int32_t* __restrict__ nroots, int32_t* __restrict__ found) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int64_t p = parent[u];
    if (p == ISOC_NO_VERTEX) {
        atomicAdd(nroots, 1);
        if (root >= 0 && u != root) atomicOr(bad, 1);
        if (found) atomicMax(found, (int32_t)u);   // root < 0: the (unique) sentinel
    } else if (p < 0 || p >= n) {
        atomicOr(bad, 2);
    }
    const uint64_t pk = (p == ISOC_NO_VERTEX || p < 0 || p >= n) ? (uint64_t)n : (uint64_t)p;
    // sibling order: given ranks (RootedTree.child_id) or ascending vertex
    // index (tree_from_parent_list, mst.py:104-111)
    const uint64_t rank = child_id ? (uint64_t)child_id[u] : (uint64_t)u;
    keys[u] = (pk << 32) | (rank & 0xffffffffull);
    pkeys[u] = (int32_t)pk;
    vals[u] = (int32_t)u;
}

__global__ void child_ids_kernel(const unsigned long long* __restrict__ sorted_keys,
                                 const int32_t* __restrict__ sorted_vals, const int32_t* __restrict__ off,
                                 int64_t n, int32_t* __restrict__ child_id_v) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int64_t p = (int64_t)(sorted_keys[s] >> 32);
    const int32_t u = sorted_vals[s];
    child_id_v[u] = (p >= n) ? 0 : (int32_t)(s - off[p]);
}

__global__ void count_children_kernel(const int32_t* __restrict__ keys, int64_t n,
                                      int32_t* __restrict__ deg) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    if (keys[u] < n) atomicAdd(&deg[keys[u]], 1);
}

// -------------------------------------------------------------- extrema
// pow2 zero-padded adjacent-pair fold (_primitives.py:95-124) of a mapped
// array; blocks of 2048 are complete subtrees, block sums are folded again.
template <int MODE>
__device__ __forceinline__ double ext_get(const double* v, int64_t m, int64_t root, int64_t i) {
    if (i >= m) return 0.0;
    if (MODE == 1) return v[i < root ? i : i + 1];  // non-root parent flows
    return v[i];
}

template <int MODE>
__global__ void fold_blocks_kernel(const double* __restrict__ v, int64_t m, int64_t root,
                                   int64_t width, double* __restrict__ out) {
    __shared__ double s[2][2048];
    const int64_t base = (int64_t)blockIdx.x * width;
    for (int i = threadIdx.x; i < width; i += blockDim.x) s[0][i] = ext_get<MODE>(v, m, root, base + i);
    __syncthreads();
    int cur = 0;
    for (int64_t w = width; w > 1; w >>= 1) {
        for (int i = threadIdx.x; i < w / 2; i += blockDim.x)
            s[cur ^ 1][i] = __dadd_rn(s[cur][2 * i], s[cur][2 * i + 1]);
        cur ^= 1;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = s[cur][0];
}

template <int MODE>
__global__ void min_kernel(const double* __restrict__ v, int64_t m, int64_t root,
                           unsigned long long* __restrict__ out) {
    // values are >= 0 here except potentials (>= 0 too); order via bits
    double best = INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        best = fmin(best, ext_get<MODE>(v, m, root, i));
    for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0) {
        long long b = __double_as_longlong(best);
        // map to an order-preserving unsigned key (handles negatives)
        unsigned long long k = (b < 0) ? ~(unsigned long long)b : ((unsigned long long)b | (1ull << 63));
        atomicMin(out, k);
    }
}

__global__ void key_to_double_kernel(const unsigned long long* __restrict__ key, double* __restrict__ out) {
    const unsigned long long k = *key;
    const unsigned long long b = (k & (1ull << 63)) ? (k & ~(1ull << 63)) : ~k;
    *out = __longlong_as_double((long long)b);
}

template <int MODE>
static cudaError_t pow2_sum(const double* v, int64_t m, int64_t root, double* out, double* tmp,
                            cudaStream_t st) {
    int64_t P = 1;
    while (P < m) P <<= 1;
    if (P <= 2048) {
        fold_blocks_kernel<MODE><<<1, 256, 0, st>>>(v, m, root, P, out);
        return cudaGetLastError();
    }
    const int64_t nb = P / 2048;
    fold_blocks_kernel<MODE><<<(unsigned)nb, 256, 0, st>>>(v, m, root, 2048, tmp);
    // fold block sums (a perfect binary tree of nb leaves)
    double* a = tmp;
    double* b = tmp + nb;
    int64_t cur = nb;
    while (cur > 2048) {
        fold_blocks_kernel<0><<<(unsigned)(cur / 2048), 256, 0, st>>>(a, cur, 0, 2048, b);
        cur /= 2048;
        double* t = a; a = b; b = t;
    }
    fold_blocks_kernel<0><<<1, 256, 0, st>>>(a, cur, 0, cur, out);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t min_value(const double* v, int64_t m, int64_t root, double* out,
                             unsigned long long* key, cudaStream_t st) {
    cudaMemsetAsync(key, 0xff, 8, st);
    min_kernel<MODE><<<296, 256, 0, st>>>(v, m, root, key);
    key_to_double_kernel<<<1, 1, 0, st>>>(key, out);
    return cudaGetLastError();
}

// plain pow2 zero-padded fold / minimum of a device vector (the stage API's
// sum_reduce / min_reduce, _primitives.py:69-124)
cudaError_t launch_pow2_sum(const double* v, int64_t m, double* out, double* tmp, cudaStream_t st) {
    return pow2_sum<0>(v, m, 0, out, tmp, st);
}
cudaError_t launch_min_value(const double* v, int64_t m, double* out, unsigned long long* key, cudaStream_t st) {
    return min_value<0>(v, m, 0, out, key, st);
}

// ------------------------------------------------------------- launchers
cudaError_t launch_build_adjacency(const int32_t* eu, const int32_t* ev, const double* ed,
                                   int64_t n, int32_t* off, int32_t* adj, double* adjd,
                                   int32_t* work, cudaStream_t st) {
    const int64_t m = n - 1;
    int32_t* deg = work;  // n+1
    cudaMemsetAsync(deg, 0, (size_t)(n + 1) * sizeof(int32_t), st);
    if (m > 0) degree_kernel<<<nblk(m, 256), 256, 0, st>>>(eu, ev, m, deg);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, off, (int)(n + 1), st);
    void* tmp = nullptr;
    cudaError_t e = isoc_malloc_async(&tmp, tb, st);
    if (e != cudaSuccess) return e;
    cub::DeviceScan::ExclusiveSum(tmp, tb, deg, off, (int)(n + 1), st);
    isoc_free_async(tmp, st);
    cudaMemcpyAsync(deg, off, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
    if (m > 0) fill_adj_kernel<<<nblk(m, 256), 256, 0, st>>>(eu, ev, ed, m, deg, adj, adjd);
    sort_adj_kernel<<<nblk(n, 256), 256, 0, st>>>(off, n, adj, adjd);
    note_launch(3);
    return cudaGetLastError();
}

cudaError_t launch_children_from_parent(const int64_t* parent, const int64_t* child_id, int64_t n,
                                        int64_t root, int32_t* off, int32_t* adj, int32_t* child_id_v,
                                        int32_t* flags, int32_t* nroots, int32_t* found_root,
                                        cudaStream_t st) {
    unsigned long long *keys = nullptr, *skeys = nullptr;
    int32_t *vals = nullptr, *pkeys = nullptr, *deg = nullptr;
    cudaError_t e;
#define ACK(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
    ACK(isoc_malloc_async((void**)&keys, (size_t)n * 8, st));
    ACK(isoc_malloc_async((void**)&skeys, (size_t)n * 8, st));
    ACK(isoc_malloc_async((void**)&vals, (size_t)n * 4, st));
    ACK(isoc_malloc_async((void**)&pkeys, (size_t)n * 4, st));
    ACK(isoc_malloc_async((void**)&deg, (size_t)(n + 1) * 4, st));
    cudaMemsetAsync(nroots, 0, sizeof(int32_t), st);
    parent_check_kernel<<<nblk(n, 256), 256, 0, st>>>(parent, child_id, n, root, keys, vals, pkeys,
                                                       flags, nroots, found_root);
    int bits = 32;
    while ((int64_t(1) << (bits - 32)) <= n) ++bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, skeys, vals, adj, (int)n, 0, bits, st);
    void* tmp = nullptr;
    ACK(isoc_malloc_async(&tmp, tb, st));
    cub::DeviceRadixSort::SortPairs(tmp, tb, keys, skeys, vals, adj, (int)n, 0, bits, st);
    isoc_free_async(tmp, st);
    cudaMemsetAsync(deg, 0, (size_t)(n + 1) * sizeof(int32_t), st);
    count_children_kernel<<<nblk(n, 256), 256, 0, st>>>(pkeys, n, deg);
    tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, off, (int)(n + 1), st);
    ACK(isoc_malloc_async(&tmp, tb, st));
    cub::DeviceScan::ExclusiveSum(tmp, tb, deg, off, (int)(n + 1), st);
    isoc_free_async(tmp, st);
    child_ids_kernel<<<nblk(n, 256), 256, 0, st>>>(skeys, adj, off, n, child_id_v);
    note_launch(3);
    isoc_free_async(keys, st); isoc_free_async(skeys, st); isoc_free_async(vals, st);
    isoc_free_async(pkeys, st); isoc_free_async(deg, st);
#undef ACK
    return cudaGetLastError();
}

// Small trees (n <= BFS_SMALL_N, e.g. C1's 228-level MST): one warp walks the
// levels with the adjacency, BFS order and parents in shared memory, so a
// level costs shuffles and shared-memory latencies instead of two grid
// barriers over global memory.  Same outputs and order as bfs_kernel
// (children in adjacency order, i.e. Prim's (d, id) rank for the MST).
constexpr int64_t BFS_SMALL_N = 8192;

__global__ void __launch_bounds__(512, 1) bfs_small_kernel(BfsArgs A) {
    // all 512 threads stage the adjacency (overlapping the global loads),
    // then warp 0 alone walks the levels
    extern __shared__ __align__(16) unsigned char bs_raw[];
    const int lane = threadIdx.x;
    const int nst = blockDim.x;
    const int64_t n = A.n;
    int32_t* off = reinterpret_cast<int32_t*>(bs_raw);
    const int64_t m = A.off[n];
    int32_t* adj = off + n + 1;
    int32_t* bfs = adj + m;
    int32_t* par = bfs + n;
    for (int64_t q = lane; q <= n; q += nst) off[q] = A.off[q];
    for (int64_t q = lane; q < m; q += nst) adj[q] = A.adj[q];
    __syncthreads();
    if (lane >= 32) return;
    if (lane == 0) {
        bfs[0] = (int32_t)A.root;
        par[A.root] = -1;
        A.bfs[0] = (int32_t)A.root;
        A.pos_of[A.root] = 0;
        A.parent_v[A.root] = -1;
        A.depth_v[A.root] = 0;
        A.pos_parent[0] = -1;
        if (A.undirected) { A.child_id_v[A.root] = 0; A.parent_d[A.root] = 0.0; }
        A.level_off[0] = 0;
        A.level_off[1] = 1;
    }
    __syncwarp();
    int64_t lo = 0, hi = 1;
    int level = 0;
    while (true) {
        int64_t carry = 0;
        for (int64_t base = lo; base < hi; base += 32) {
            const int64_t p = base + lane;
            int32_t v = 0, c = 0;
            if (p < hi) {
                v = bfs[p];
                c = off[v + 1] - off[v];
                if (A.undirected && v != A.root) c -= 1;
            }
            int32_t x = c;
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (p < hi) {
                const int64_t first = hi + carry + x - c;
                const int32_t pv = par[v];
                int32_t rank = 0;
                for (int32_t e = off[v]; e < off[v + 1]; ++e) {
                    const int32_t w = adj[e];
                    if (A.undirected && w == pv) continue;
                    const int64_t q = first + rank;
                    if (q < n) {
                        bfs[q] = w;
                        par[w] = v;
                        A.bfs[q] = w;
                        A.pos_of[w] = (int32_t)q;
                        A.parent_v[w] = v;
                        A.depth_v[w] = level + 1;
                        A.pos_parent[q] = (int32_t)p;
                        if (A.undirected) {
                            A.child_id_v[w] = rank;
                            A.parent_d[w] = A.adjd[e];
                        }
                    }
                    ++rank;
                }
                A.child_lo[p] = (int32_t)first;
                A.child_cnt[p] = rank;
            }
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
        __syncwarp();
        if (lane == 0) A.level_off[level + 2] = hi + carry;
        if (carry == 0) {
            if (lane == 0) *A.out_levels = level + 1;
            break;
        }
        lo = hi;
        hi = hi + carry;
        ++level;
        if (hi > n) {  // not a tree (cycle); stop
            if (lane == 0) *A.out_levels = -1;
            break;
        }
    }
}

int bfs_grid_size(int64_t n) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_kernel, 512, 0);
    int64_t want = (n + 16383) / 16384;  // ~16k positions per CTA per wide level
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    if (want < 1) want = 1;
    return (int)(want < cap ? want : cap);
}

cudaError_t launch_bfs(int64_t n, int64_t root, int undirected, const int32_t* off,
                       const int32_t* adj, const double* adjd, int32_t* bfs, int32_t* pos_of,
                       int32_t* parent_v, int32_t* depth_v, int32_t* child_id_v, double* parent_d,
                       int32_t* pos_parent, int32_t* child_lo, int32_t* child_cnt,
                       int64_t* level_off, int32_t* scratch, int64_t* out_levels, cudaStream_t st) {
    const bool small = n <= BFS_SMALL_N;
    const int G = small ? 1 : bfs_grid_size(n);
    BfsArgs A;
    A.n = n; A.root = root; A.undirected = undirected; A.off = off; A.adj = adj; A.adjd = adjd;
    A.bfs = bfs; A.pos_of = pos_of; A.parent_v = parent_v; A.depth_v = depth_v;
    A.child_id_v = child_id_v; A.parent_d = parent_d; A.pos_parent = pos_parent;
    A.child_lo = child_lo; A.child_cnt = child_cnt; A.level_off = level_off;
    A.scratch_cnt = scratch;                // n
    A.chunk_sum = scratch + n;              // G
    A.bar = reinterpret_cast<unsigned int*>(scratch + n + G + 2);
    A.out_levels = out_levels;
    cudaMemsetAsync(A.bar, 0, 2 * sizeof(unsigned int), st);
    if (small) {
        // off (n+1) + adj (<= 2n) + bfs (n) + parents (n), int32: the adjacency
        // length is read on the device, so size for the undirected maximum
        const size_t smem = (size_t)(n + 1 + 2 * n + 2 * n) * sizeof(int32_t);
        cudaError_t e = ensure_max_dyn_smem((const void*)bfs_small_kernel, smem);
        if (e != cudaSuccess) return e;
        const int pid = prof_begin(PK_BFS, st);
        bfs_small_kernel<<<1, 512, smem, st>>>(A);
        prof_end(pid, st);
        note_launch();
        return cudaGetLastError();
    }
    void* args[] = {&A};
    const int pid = prof_begin(PK_BFS, st);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)bfs_kernel, dim3(G), dim3(512), args, 0, st);
    prof_end(pid, st);
    note_launch();
    return e;
}

cudaError_t launch_flows(const double* parent_d, const int32_t* parent_v, int64_t n, double sigma,
                         double* flow, cudaStream_t st) {
    flows_kernel<<<nblk(n, 256), 256, 0, st>>>(parent_d, parent_v, n, sigma, flow);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_gather_pos(const int32_t* bfs, int64_t n, const double* flow_v,
                              const double* omega_v, const double* p_v, double* f_pos,
                              double* om_pos, double* p_pos, cudaStream_t st) {
    gather_pos_kernel<<<nblk(n, 256), 256, 0, st>>>(bfs, n, flow_v, omega_v, p_v, f_pos, om_pos,
                                                     p_pos);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_extrema(const double* flow_v, int64_t root, const double* omega, const double* p,
                           int64_t n, double* out6, double* tmp, unsigned long long* key,
                           cudaStream_t st) {
    // tmp: >= 2 * (next_pow2(n) / 2048 + 1) doubles
    note_launch(12);
    pow2_sum<1>(flow_v, n - 1, root, out6 + 0, tmp, st);
    min_value<1>(flow_v, n - 1, root, out6 + 1, key, st);
    pow2_sum<0>(omega, n, 0, out6 + 2, tmp, st);
    min_value<0>(omega, n, 0, out6 + 3, key + 1, st);
    pow2_sum<0>(p, n, 0, out6 + 4, tmp, st);
    min_value<0>(p, n, 0, out6 + 5, key + 2, st);
    return cudaGetLastError();
}

}  // namespace isoc
