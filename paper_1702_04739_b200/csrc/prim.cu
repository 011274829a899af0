// Exact Prim on the device: the tie-rule fallback of the MST stage.
//
// The lexicographic (d, min, max) Boruvka MST equals the reference's Prim
// tree whenever the component minima are unique. When
// a round reports an exact distance tie, the edge set can differ (the
// reference keeps its own rule: frontier minimum with ties to the smallest
// vertex id, strict `<` relaxation so the earliest-inserted attach vertex
// wins; mst.py:144-166, _primitives.py:69-92). This kernel replays that rule
// step for step, one cooperative launch with one grid barrier per step:
//   step s: each thread relaxes its columns j (static grid-stride ownership)
//           against the vertex u chosen at step s-1 (exact scipy-order
//           distance), then the CTA forms its lexicographic (key, j) minimum
//           over the frontier; partials are double-buffered by step parity,
//           so after one barrier every CTA reduces them to the same winner.
// Work: n-1 steps x n exact distances (3d fp64 ops each) -- one extra
// distance pass plus n grid barriers; it only runs when ties were seen (or
// ISOC_MST=prim).
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/isoclust_b200.h"
#include "common.cuh"

namespace isoc {
int set_error(int code, const char* fmt, ...);
}

namespace {

using isoc::exact_dist;
using isoc::grid_barrier;

constexpr int PRIM_THREADS = 512;

__device__ __forceinline__ bool lex_less(double av, int64_t ai, double bv, int64_t bi) {
    if (bi < 0) return ai >= 0;
    if (ai < 0) return false;
    return av < bv || (av == bv && ai < bi);
}

__device__ __forceinline__ void warp_min(double& v, int64_t& i) {
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, v, o);
        int64_t oi = __shfl_down_sync(0xffffffffu, i, o);
        if (lex_less(ov, oi, v, i)) { v = ov; i = oi; }
    }
}

// DENSE: X is the (n, n) distance matrix (the dense stage API, prim_mst(dist));
// row u is read coalesced as D[u*n + j].  Otherwise X is (n, d) points and the
// distance is recomputed exactly in scipy order.
template <bool DENSE>
__device__ __forceinline__ double prim_dist(const double* __restrict__ X, int64_t n, int d, int64_t u,
                                            int64_t j) {
    if (DENSE) return X[u * n + j];
    return exact_dist(X + u * d, X + j * d, d);
}

template <bool DENSE>
__global__ void __launch_bounds__(PRIM_THREADS) prim_kernel(
    const double* __restrict__ X, int64_t n, int d, int64_t root, double* key, int32_t* from,
    uint8_t* done, double* pv, int64_t* pi, int32_t* eu, int32_t* ev, double* ew, unsigned int* bar) {
    __shared__ double sv[PRIM_THREADS / 32];
    __shared__ int64_t si[PRIM_THREADS / 32];
    __shared__ int64_t s_u;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int G = gridDim.x;
    int64_t u = root;
    for (int64_t step = 0; step < n - 1; ++step) {
        double bv = 0.0;
        int64_t bi = -1;
        for (int64_t j = tid; j < n; j += stride) {
            if (step == 0) {
                // best = d[root], best_from = root (mst.py:144-147)
                done[j] = (j == root);
                from[j] = (int32_t)root;
                key[j] = prim_dist<DENSE>(X, n, d, root, j);
                if (j == root) continue;
            } else {
                if (done[j]) continue;
                if (j == u) {           // the vertex the last step inserted
                    done[j] = 1;
                    continue;
                }
                const double r = prim_dist<DENSE>(X, n, d, u, j);
                if (r < key[j]) {       // strict: ties keep the earlier attach vertex
                    key[j] = r;
                    from[j] = (int32_t)u;
                }
            }
            if (bi < 0 || key[j] < bv) { bv = key[j]; bi = j; }   // j ascending per thread
        }
        warp_min(bv, bi);
        if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
        __syncthreads();
        if (wid == 0) {
            bv = lane < PRIM_THREADS / 32 ? sv[lane] : 0.0;
            bi = lane < PRIM_THREADS / 32 ? si[lane] : -1;
            warp_min(bv, bi);
            if (lane == 0) {
                const int64_t slot = (step & 1) * G + blockIdx.x;
                pv[slot] = bv;
                pi[slot] = bi;
            }
        }
        grid_barrier(bar);
        if (wid == 0) {
            bv = 0.0;
            bi = -1;
            for (int c = lane; c < G; c += 32) {
                const int64_t slot = (step & 1) * G + c;
                const double cv = __ldcg(pv + slot);
                const int64_t ci = __ldcg(pi + slot);
                if (lex_less(cv, ci, bv, bi)) { bv = cv; bi = ci; }
            }
            warp_min(bv, bi);
            if (lane == 0) {
                s_u = bi;
                if (blockIdx.x == 0) {
                    eu[step] = __ldcg(from + bi);
                    ev[step] = (int32_t)bi;
                    ew[step] = __ldcg(key + bi);
                }
            }
        }
        __syncthreads();
        u = s_u;
    }
}

}  // namespace

static int prim_launch(bool dense, const double* X, int64_t n, int32_t d, int64_t root, int32_t* u,
                       int32_t* v, double* w, void* stream) {
    if (n < 2) return isoc::set_error(ISOC_EINVAL, "need at least 2 vertices");
    if (n > INT32_MAX) return isoc::set_error(ISOC_EINVAL, "n too large for int32 edge ids");
    if (root < 0 || root >= n)
        return isoc::set_error(ISOC_EINVAL, "root must be in [0, %lld), got %lld", (long long)n,
                               (long long)root);
    cudaStream_t st = (cudaStream_t)stream;
    const void* kern = dense ? (const void*)prim_kernel<true> : (const void*)prim_kernel<false>;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PRIM_THREADS, 0);
    if (per_sm < 1) return isoc::set_error(ISOC_ECUDA, "prim_kernel cannot be resident");
    int G = sms;  // one CTA per SM: the step is barrier-latency bound
    const int64_t need = (G + 31) / 32 * 32;
    if ((int64_t)G * PRIM_THREADS > n) G = (int)((n + PRIM_THREADS - 1) / PRIM_THREADS);
    char* scratch = nullptr;
    const size_t bytes = (size_t)n * (8 + 4 + 1) + 2 * need * 16 + 64 + 16;
    cudaError_t e = isoc::isoc_malloc_async((void**)&scratch, bytes, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return isoc::set_error(e == cudaErrorMemoryAllocation ? ISOC_ENOMEM : ISOC_ECUDA,
                               "prim scratch: %s", cudaGetErrorString(e));
    }
    double* key = (double*)scratch;
    double* pv = key + n;
    int64_t* pi = (int64_t*)(pv + 2 * need);
    int32_t* from = (int32_t*)(pi + 2 * need);
    unsigned int* bar = (unsigned int*)(from + n + (n & 1));
    uint8_t* done = (uint8_t*)(bar + 16);
    cudaMemsetAsync(bar, 0, 64, st);
    int dd = d;
    void* args[] = {(void*)&X, &n, &dd, &root, &key, &from, &done, &pv, &pi, &u, &v, &w, &bar};
    e = cudaLaunchCooperativeKernel(kern, dim3(G), dim3(PRIM_THREADS), args, 0, st);
    isoc::isoc_free_async(scratch, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return isoc::set_error(ISOC_ECUDA, "prim_kernel launch: %s", cudaGetErrorString(e));
    }
    return ISOC_OK;
}

extern "C" int isoc_prim_edges(const double* X, int64_t n, int32_t d, int64_t root, int32_t* u,
                               int32_t* v, double* w, void* stream) {
    return prim_launch(false, X, n, d, root, u, v, w, stream);
}

extern "C" int isoc_prim_edges_dense(const double* D, int64_t n, int64_t root, int32_t* u, int32_t* v,
                                     double* w, void* stream) {
    return prim_launch(true, D, n, 1, root, u, v, w, stream);
}
