// Dense-input stage functions of the reference's public API
// (/root/reference/pkg/src/isoclust/__init__.py:71-122), on the device:
//   distance_matrix          affinity.py:124-158 (scipy order, exact)
//   flow                     affinity.py:161-172 (exp((-d)/sigma), glibc exp)
//   vertex_weights           affinity.py:175-201 (pow2 row folds, diagonal 0)
//   potentials               affinity.py:204-230 (alpha * pow2 row fold)
//   auto_sigma               affinity.py:233-241 (numpy pairwise d.sum())
//   validate_distance_matrix affinity.py:101-121
//   prim_mst on a matrix     mst.py:128-181 (lexicographic Boruvka: the same
//                            edge set as Prim for distinct distances)
//   sum_reduce / min_reduce / exclusive_scan  _primitives.py:62-159
//   extract_labels           isoperim.py:164-181
//   brute_force_miso         isoperim.py:324-390 (exhaustive labelling search)
// The matrix-free pipeline never builds these n^2 arrays; these entry points
// serve callers of the stage API that hold a distance matrix (the reference
// caps those at n <= 46,340).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "../../include/isoclust_b200.h"
#include "common.cuh"
#include "scratch.h"
#include "kernels.h"
#include "leaf.h"
#include "prof.h"

namespace isoc {
int set_error(int code, const char* fmt, ...);

namespace {

__global__ void dist_dense_kernel(const double* __restrict__ XT, int64_t np, int d, int64_t n,
                                  double* __restrict__ D) {
    const int64_t i = blockIdx.y;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double s = 0.0;
    for (int k = 0; k < d; ++k) s = exact_sq_step(s, XT[(int64_t)k * np + i], XT[(int64_t)k * np + j]);
    D[i * n + j] = __dsqrt_rn(s);
}

__global__ void flow_kernel(const double* __restrict__ d, int64_t m, double sigma, double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = isoc_exp(__ddiv_rn(-d[i], sigma));
}

// One CTA per row: pow2 zero-padded adjacent-pair fold over the row
// (pairwise_row_sums, _primitives.py:162-175) in 2048-wide complete
// subtrees combined by a binary counter.  MODE 0: flows with the diagonal
// zeroed (vertex_weights); MODE 1: alpha * fold of d (potentials).
template <int MODE>
__global__ void __launch_bounds__(256) row_fold_kernel(const double* __restrict__ D, int64_t n, double param,
                                                       double* __restrict__ out) {
    __shared__ double s[2][2048];
    __shared__ double slots[40];
    const int64_t r = blockIdx.x;
    int64_t P = 1;
    while (P < n) P <<= 1;
    const int64_t W = P < 2048 ? P : 2048;
    const double* row = D + r * n;
    for (int64_t c = 0; c < P / W; ++c) {
        for (int i = threadIdx.x; i < W; i += blockDim.x) {
            const int64_t j = c * W + i;
            double v = 0.0;
            if (j < n) {
                v = row[j];
                if (MODE == 0) v = (j == r) ? 0.0 : isoc_exp(__ddiv_rn(-v, param));
            }
            s[0][i] = v;
        }
        __syncthreads();
        int cur = 0;
        for (int64_t w = W; w > 1; w >>= 1) {
            for (int i = threadIdx.x; i < w / 2; i += blockDim.x)
                s[cur ^ 1][i] = __dadd_rn(s[cur][2 * i], s[cur][2 * i + 1]);
            cur ^= 1;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            double v = s[cur][0];
            int lvl = 0;
            for (int64_t t = c; t & 1; t >>= 1, ++lvl) v = __dadd_rn(slots[lvl], v);
            slots[lvl] = v;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int top = 0;
        while (((int64_t)1 << top) < P / W) ++top;
        const double f = slots[top];
        out[r] = MODE == 0 ? f : __dmul_rn(param, f);
    }
}

// numpy pairwise_sum over a flat device array: thread t sums the leaves
// starting in [t*S, (t+1)*S) and pushes them (heap ids) onto its fold stack;
// the stacks of consecutive ranges then concatenate in order.
constexpr int64_t kSumSpan = 8192;
__global__ void pairwise_chunks_kernel(const double* __restrict__ v, int64_t m, int64_t nchunks,
                                       FoldStack* __restrict__ out, int32_t* __restrict__ flags) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nchunks) return;
    FoldStack& S = out[t];
    int cnt = 0, ovf = 0;
    const int64_t lo = t * kSumSpan, hi = (lo + kSumSpan < m) ? lo + kSumSpan : m;
    const Leaf L0 = find_leaf(m, lo);
    LeafIter it = leaf_iter_from(m, L0.start, L0.len, L0.hid);
    if (it.start < lo) {
        if (it.start + it.len >= m) { S.count = 0; S.overflow = 0; return; }
        leaf_next(it, m);
    }
    while (it.start < hi) {
        const int64_t st = it.start;
        const double x = np_leaf_sum([&](int64_t q) { return v[st + q]; }, it.len);
        stack_push(S.value, S.id, cnt, kStackCap, ovf, x, it.hid());
        if (it.start + it.len >= m) break;
        leaf_next(it, m);
    }
    S.count = cnt;
    S.overflow = ovf;
    if (ovf) atomicOr(flags, 1);
}

__global__ void validate_kernel(const double* __restrict__ D, int64_t n, int32_t* __restrict__ flags) {
    const int64_t i = blockIdx.y;
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double a = D[i * n + j];
    int f = 0;
    if (!isfinite(a)) f |= 1;
    else if (a < 0.0) f |= 2;
    if (j > i && !(a == D[j * n + i])) f |= 4;
    if (j == i && a != 0.0) f |= 8;
    if (f) atomicOr(flags, f);
}

// Boruvka on a dense matrix: per row the lexicographic (d, j) minimum over
// columns in other components (one warp per row).
__global__ void dense_row_min_kernel(const double* __restrict__ D, int64_t n, const int32_t* __restrict__ comp,
                                     double* __restrict__ cand_d, int32_t* __restrict__ cand_j,
                                     int8_t* __restrict__ cand_state, int8_t* __restrict__ cand_tie) {
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int32_t ci = comp[i];
    double m1 = INFINITY, m2 = INFINITY;
    int32_t j1 = INT32_MAX;
    for (int64_t j = lane; j < n; j += 32) {
        if (comp[j] == ci) continue;
        const double v = D[i * n + j];
        if (v < m1) { m2 = m1; m1 = v; j1 = (int32_t)j; }
        else if (v < m2) m2 = v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double om1 = __shfl_xor_sync(0xffffffffu, m1, o), om2 = __shfl_xor_sync(0xffffffffu, m2, o);
        const int32_t oj = __shfl_xor_sync(0xffffffffu, j1, o);
        const bool other = om1 < m1 || (om1 == m1 && oj < j1);
        const double lose = other ? m1 : om1;
        m2 = fmin(fmin(m2, om2), lose);
        if (other) { m1 = om1; j1 = oj; }
    }
    if (lane == 0) {
        cand_d[i] = m1;
        cand_j[i] = j1 == INT32_MAX ? -1 : j1;
        cand_state[i] = j1 != INT32_MAX;
        cand_tie[i] = (m1 == m2) && j1 != INT32_MAX;
    }
}

__global__ void iota32_kernel(int32_t* v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (int32_t)i;
}

__global__ void labels_from_cut_kernel(const int64_t* __restrict__ scan, const int64_t* __restrict__ eta,
                                       int64_t n, int64_t* __restrict__ labels, int32_t* __restrict__ flags) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t e = eta[i];
    if (e == ISOC_NO_VERTEX) { labels[i] = 0; return; }
    if (e < 0 || e >= n) { atomicOr(flags, 1); labels[i] = 0; return; }
    labels[i] = 1 + scan[e];
}

__global__ void cut_to_i64_kernel(const int8_t* __restrict__ cut, int64_t n, int64_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = cut[i] ? 1 : 0;
}

__global__ void argmin_index_kernel(const double* __restrict__ v, int64_t m, const double* __restrict__ mval,
                                    unsigned long long* __restrict__ idx) {
    const double target = *mval;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        if (v[i] == target) atomicMin(idx, (unsigned long long)i);
}

__global__ void finite_kernel(const double* __restrict__ v, int64_t m, int32_t* __restrict__ flags) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(v[i])) atomicOr(flags, 1);
}

// brute_force_miso (isoperim.py:324-390): labelling code c in [0, (k+1)^n)
// puts vertex v in cluster digit_v(c) (base k+1, vertex 0 least
// significant).  Per cluster, mass and potential accumulate in ascending
// vertex order and the boundary in ascending child order (the sequential
// order of the reference's 0/1-indicator dot products; a product by 0 or 1
// is exact).  worst = max(0, max_c sparsity_c); a code leaving a cluster
// empty is infeasible (+inf).  PASS 0 takes the minimum worst as its bit
// pattern (nonnegative doubles order as unsigned integers); PASS 1 the
// smallest code attaining it (np.argmin keeps the first, isoperim.py:380).
constexpr int BF_MAXN = 12;

template <int PASS>
__global__ void __launch_bounds__(256) brute_force_kernel(const int32_t* __restrict__ parent,
                                                          const double* __restrict__ flow,
                                                          const double* __restrict__ omega,
                                                          const double* __restrict__ pot, int n, int k,
                                                          uint32_t total, unsigned long long* best_bits,
                                                          unsigned long long* best_code) {
    __shared__ int32_t s_par[BF_MAXN];
    __shared__ double s_flow[BF_MAXN], s_om[BF_MAXN], s_p[BF_MAXN];
    if (threadIdx.x < n) {
        s_par[threadIdx.x] = parent[threadIdx.x];
        s_flow[threadIdx.x] = flow[threadIdx.x];
        s_om[threadIdx.x] = omega[threadIdx.x];
        s_p[threadIdx.x] = pot[threadIdx.x];
    }
    __syncthreads();
    const uint32_t base = (uint32_t)k + 1;
    const unsigned long long target = PASS ? *best_bits : 0ull;
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t rounds = (total + stride - 1) / stride;
    for (uint32_t r = 0; r < rounds; ++r) {
        const uint32_t code = r * stride + blockIdx.x * blockDim.x + threadIdx.x;
        unsigned long long bits = ~0ull;
        if (code < total) {
            int dig[BF_MAXN];
            uint32_t c = code;
#pragma unroll
            for (int v = 0; v < BF_MAXN; ++v) {
                dig[v] = (int)(c % base);
                c /= base;
            }
            double mass[BF_MAXN + 1], bnd[BF_MAXN + 1], pp[BF_MAXN + 1];
            int cnt[BF_MAXN + 1];
            for (int q = 0; q <= k; ++q) mass[q] = bnd[q] = pp[q] = 0.0, cnt[q] = 0;
            for (int v = 0; v < n; ++v) {
                const int a = dig[v];
                mass[a] = __dadd_rn(mass[a], s_om[v]);
                pp[a] = __dadd_rn(pp[a], s_p[v]);
                cnt[a] += 1;
                const int w = s_par[v];
                if (w >= 0) {
                    const int b = dig[w];
                    if (a != b) {
                        bnd[a] = __dadd_rn(bnd[a], s_flow[v]);
                        bnd[b] = __dadd_rn(bnd[b], s_flow[v]);
                    }
                }
            }
            double worst = 0.0;
            bool feasible = true;
            for (int q = 1; q <= k; ++q) {
                feasible &= cnt[q] > 0;
                const double sp = __ddiv_rn(__dadd_rn(bnd[q], pp[q]), mass[q]);
                worst = sp > worst ? sp : worst;
            }
            if (!feasible) worst = __longlong_as_double(0x7ff0000000000000ll);
            bits = (unsigned long long)__double_as_longlong(worst);
        }
        if (PASS == 0) {
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
                bits = other < bits ? other : bits;
            }
            if ((threadIdx.x & 31) == 0 && bits != ~0ull) atomicMin(best_bits, bits);
        } else if (code < total && bits == target) {
            atomicMin(best_code, (unsigned long long)code);
        }
    }
}

inline unsigned nb(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace
}  // namespace isoc

using namespace isoc;

#define SCK(expr)                                                                                  \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess) {                                                                   \
            cudaGetLastError();                                                                    \
            return isoc::set_error(_e == cudaErrorMemoryAllocation ? ISOC_ENOMEM : ISOC_ECUDA, "%s: %s", \
                                   #expr, cudaGetErrorString(_e));                                 \
        }                                                                                          \
    } while (0)

extern "C" {

int isoc_distance_matrix(const double* X, int64_t n, int32_t d, double* D, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (n < 1 || d < 1) return set_error(ISOC_EINVAL, "need n >= 1 and d >= 1");
    if (n > 65535) return set_error(ISOC_EINVAL, "dense distance matrix limited to 65535 rows");
    const int64_t np = (n + 1023) / 1024 * 1024;
    double* XT = nullptr;
    SCK(S.alloc(&XT, (size_t)np * d));
    SCK(launch_transpose_pad(X, n, d, np, d, XT, st));
    dist_dense_kernel<<<dim3(nb(n, 256), (unsigned)n), 256, 0, st>>>(XT, np, d, n, D);
    note_launch(1);
    SCK(cudaGetLastError());
    return ISOC_OK;
}

int isoc_flow(const double* dist, int64_t m, double sigma, double* out, void* stream) {
    if (!(sigma > 0.0)) return set_error(ISOC_EINVAL, "sigma must be > 0, got %g", sigma);
    if (m <= 0) return ISOC_OK;
    flow_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(dist, m, sigma, out);
    note_launch(1);
    SCK(cudaGetLastError());
    return ISOC_OK;
}

int isoc_vertex_weights_dense(const double* D, int64_t n, double sigma, double* omega, void* stream) {
    if (!(sigma > 0.0)) return set_error(ISOC_EINVAL, "sigma must be > 0, got %g", sigma);
    if (n < 1) return set_error(ISOC_EINVAL, "empty matrix");
    row_fold_kernel<0><<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(D, n, sigma, omega);
    note_launch(1);
    SCK(cudaGetLastError());
    return ISOC_OK;
}

int isoc_potentials_dense(const double* D, int64_t n, double alpha, double* p, void* stream) {
    if (!(alpha >= 0.0)) return set_error(ISOC_EINVAL, "alpha must be >= 0, got %g", alpha);
    if (n < 1) return set_error(ISOC_EINVAL, "empty matrix");
    cudaStream_t st = (cudaStream_t)stream;
    if (alpha == 0.0) {
        SCK(cudaMemsetAsync(p, 0, (size_t)n * 8, st));
        return ISOC_OK;
    }
    row_fold_kernel<1><<<(unsigned)n, 256, 0, st>>>(D, n, alpha, p);
    note_launch(1);
    SCK(cudaGetLastError());
    return ISOC_OK;
}

int isoc_pairwise_sum(const double* v, int64_t m, double* total_host, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (m < 1) return set_error(ISOC_EINVAL, "pairwise sum of an empty array");
    const int64_t nch = (m + kSumSpan - 1) / kSumSpan;
    FoldStack *stacks = nullptr, *out = nullptr;
    int32_t* flags = nullptr;
    SCK(S.alloc(&stacks, (size_t)nch));
    SCK(S.alloc(&out, 1));
    SCK(S.alloc(&flags, 1));
    SCK(cudaMemsetAsync(flags, 0, 4, st));
    pairwise_chunks_kernel<<<nb(nch, 128), 128, 0, st>>>(v, m, nch, stacks, flags);
    note_launch(1);
    // merge the stacks in order, 64 at a time
    FoldStack* a = stacks;
    int64_t cur = nch;
    FoldStack* tmp = nullptr;
    if (cur > 1) SCK(S.alloc(&tmp, (size_t)((cur + 63) / 64) * 2));
    FoldStack* b = tmp;
    FoldStack* c2 = tmp ? tmp + (cur + 63) / 64 : nullptr;
    while (cur > 1) {
        SCK(launch_stack_merge(a, cur, 64, b, flags, st));
        cur = (cur + 63) / 64;
        a = b;
        b = (b == tmp) ? c2 : tmp;
    }
    FoldStack h;
    SCK(cudaMemcpyAsync(&h, a, sizeof(FoldStack), cudaMemcpyDeviceToHost, st));
    int32_t hf = 0;
    SCK(cudaMemcpyAsync(&hf, flags, 4, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    if (hf || h.overflow) return set_error(ISOC_ECUDA, "pairwise fold stack overflow");
    if (h.count != 1 || h.id[0] != 1) return set_error(ISOC_ECUDA, "pairwise fold did not close (%d)", h.count);
    *total_host = h.value[0];
    return ISOC_OK;
}

int isoc_validate_distance_matrix(const double* D, int64_t n, int32_t* flags_host, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (n < 1) return set_error(ISOC_EINVAL, "empty matrix");
    int32_t* flags = nullptr;
    SCK(S.alloc(&flags, 1));
    SCK(cudaMemsetAsync(flags, 0, 4, st));
    validate_kernel<<<dim3(nb(n, 256), (unsigned)n), 256, 0, st>>>(D, n, flags);
    note_launch(1);
    SCK(cudaMemcpyAsync(flags_host, flags, 4, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    return ISOC_OK;
}

int isoc_mst_dense(const double* D, int64_t n, int32_t* eu, int32_t* ev, double* ed, int64_t* ties_host,
                   void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (n < 2) return set_error(ISOC_EINVAL, "need at least 2 points");
    int32_t *comp = nullptr, *cand_j = nullptr, *succ = nullptr, *succ2 = nullptr, *cnt = nullptr;
    double* cand_d = nullptr;
    int8_t *cand_state = nullptr, *cand_tie = nullptr;
    unsigned long long *compD = nullptr, *compE = nullptr;
    SCK(S.alloc(&comp, n));
    SCK(S.alloc(&cand_j, n));
    SCK(S.alloc(&succ, n));
    SCK(S.alloc(&succ2, n));
    SCK(S.alloc(&cnt, 8));
    SCK(S.alloc(&cand_d, n));
    SCK(S.alloc(&cand_state, n));
    SCK(S.alloc(&cand_tie, n));
    SCK(S.alloc(&compD, n));
    SCK(S.alloc(&compE, n));
    SCK(cudaMemsetAsync(cnt, 0, 8 * 4, st));
    iota32_kernel<<<nb(n, 256), 256, 0, st>>>(comp, n);
    int64_t comps = n, rounds = 0;
    int32_t c[8] = {0};
    while (comps > 1) {
        dense_row_min_kernel<<<nb(n, 8), 256, 0, st>>>(D, n, comp, cand_d, cand_j, cand_state, cand_tie);
        SCK(launch_comp_exact_min(cand_d, cand_state, comp, n, 0, n, compD, st));
        SCK(launch_comp_edge(cand_d, cand_j, cand_state, comp, n, 0, n, compD, compE, st));
        SCK(launch_comp_ties(cand_d, cand_j, cand_state, cand_tie, comp, 0, n, compD, compE, cnt + 1, st));
        SCK(launch_hook_contract(comp, n, compD, compE, succ, succ2, eu, ev, ed, cnt + 2, cnt + 3, cnt + 4, st));
        note_launch(1);
        SCK(cudaMemcpyAsync(c, cnt, sizeof c, cudaMemcpyDeviceToHost, st));
        SCK(cudaStreamSynchronize(st));
        if (c[4] >= comps) return set_error(ISOC_ECUDA, "Boruvka made no progress (%d components)", c[4]);
        comps = c[4];
        if (++rounds > 64) return set_error(ISOC_ECUDA, "Boruvka did not converge");
    }
    SCK(cudaStreamSynchronize(st));
    if (c[2] != n - 1) return set_error(ISOC_ECUDA, "MST has %d edges, expected %lld", c[2], (long long)(n - 1));
    if (ties_host) *ties_host = c[1];
    return ISOC_OK;
}

int isoc_sum_reduce(const double* v, int64_t m, double* out_host, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (m < 1) return set_error(ISOC_EINVAL, "sum_reduce of an empty array");
    double* out = nullptr;
    double* tmp = nullptr;
    int32_t* flags = nullptr;
    SCK(S.alloc(&out, 1));
    SCK(S.alloc(&tmp, (size_t)(m / 1024 + 8) * 2));
    SCK(S.alloc(&flags, 1));
    SCK(cudaMemsetAsync(flags, 0, 4, st));
    finite_kernel<<<148 * 4, 256, 0, st>>>(v, m, flags);
    SCK(launch_pow2_sum(v, m, out, tmp, st));
    int32_t hf = 0;
    SCK(cudaMemcpyAsync(out_host, out, 8, cudaMemcpyDeviceToHost, st));
    SCK(cudaMemcpyAsync(&hf, flags, 4, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    if (hf) return set_error(ISOC_EINVAL, "sum_reduce requires finite values");
    return ISOC_OK;
}

int isoc_min_reduce(const double* v, int64_t m, double* val_host, int64_t* idx_host, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (m < 1) return set_error(ISOC_EINVAL, "min_reduce of an empty array");
    double* out = nullptr;
    unsigned long long *key = nullptr, *idx = nullptr;
    int32_t* flags = nullptr;
    SCK(S.alloc(&out, 1));
    SCK(S.alloc(&key, 1));
    SCK(S.alloc(&idx, 1));
    SCK(S.alloc(&flags, 1));
    SCK(cudaMemsetAsync(flags, 0, 4, st));
    SCK(cudaMemsetAsync(idx, 0xff, 8, st));
    finite_kernel<<<148 * 4, 256, 0, st>>>(v, m, flags);
    SCK(launch_min_value(v, m, out, key, st));
    argmin_index_kernel<<<148 * 4, 256, 0, st>>>(v, m, out, idx);
    note_launch(2);
    unsigned long long hi = 0;
    int32_t hf = 0;
    SCK(cudaMemcpyAsync(val_host, out, 8, cudaMemcpyDeviceToHost, st));
    SCK(cudaMemcpyAsync(&hi, idx, 8, cudaMemcpyDeviceToHost, st));
    SCK(cudaMemcpyAsync(&hf, flags, 4, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    if (hf) return set_error(ISOC_EINVAL, "min_reduce requires finite values");
    *idx_host = (int64_t)hi;
    return ISOC_OK;
}

int isoc_exclusive_scan(const int64_t* v, int64_t m, int64_t* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (m < 1) return ISOC_OK;
    size_t tb = 0;
    SCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, v, out, (int)m, st));
    void* tmp = nullptr;
    SCK(S.alloc(reinterpret_cast<uint8_t**>(&tmp), tb));
    SCK(cub::DeviceScan::ExclusiveSum(tmp, tb, v, out, (int)m, st));
    note_launch(1);
    SCK(cudaGetLastError());
    return ISOC_OK;
}

int isoc_brute_force_miso(const int32_t* parent, const double* flow, const double* omega, const double* p,
                          int32_t n, int32_t k, int64_t* code_host, double* worst_host, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (n < 1 || n > BF_MAXN) return set_error(ISOC_EINVAL, "brute force supports 1 <= n <= %d, got %d", BF_MAXN, n);
    if (k < 1) return set_error(ISOC_EINVAL, "k must be >= 1, got %d", k);
    if (k > n)
        return set_error(ISOC_EINFEASIBLE, "no feasible labeling: k=%d clusters require k <= n=%d vertices", k, n);
    double total = 1.0;
    for (int v = 0; v < n; ++v) total *= (double)(k + 1);
    if (total > (double)(1 << 26))
        return set_error(ISOC_EINVAL, "enumeration of %.0f labelings exceeds the supported size", total);
    unsigned long long *bits = nullptr, *code = nullptr;
    SCK(S.alloc(&bits, 1));
    SCK(S.alloc(&code, 1));
    SCK(cudaMemsetAsync(bits, 0xff, 8, st));
    SCK(cudaMemsetAsync(code, 0xff, 8, st));
    const uint32_t tot = (uint32_t)total;
    const unsigned grid = (unsigned)std::min<int64_t>(148 * 8, ((int64_t)tot + 255) / 256);
    brute_force_kernel<0><<<grid, 256, 0, st>>>(parent, flow, omega, p, n, k, tot, bits, code);
    brute_force_kernel<1><<<grid, 256, 0, st>>>(parent, flow, omega, p, n, k, tot, bits, code);
    note_launch(2);
    SCK(cudaGetLastError());
    unsigned long long hb = 0, hc = 0;
    SCK(cudaMemcpyAsync(&hb, bits, 8, cudaMemcpyDeviceToHost, st));
    SCK(cudaMemcpyAsync(&hc, code, 8, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    double w;
    memcpy(&w, &hb, 8);
    *worst_host = w;
    *code_host = (hc == ~0ull || !(w < __builtin_inf())) ? -1 : (int64_t)hc;
    return ISOC_OK;
}

int isoc_extract_labels(const int8_t* cut, const int64_t* eta, int64_t n, int64_t* labels, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    Scratch S(st);
    if (n < 1) return ISOC_OK;
    int64_t *c64 = nullptr, *scan = nullptr;
    int32_t* flags = nullptr;
    SCK(S.alloc(&c64, n));
    SCK(S.alloc(&scan, n));
    SCK(S.alloc(&flags, 1));
    SCK(cudaMemsetAsync(flags, 0, 4, st));
    cut_to_i64_kernel<<<nb(n, 256), 256, 0, st>>>(cut, n, c64);
    int rc = isoc_exclusive_scan(c64, n, scan, stream);
    if (rc) return rc;
    labels_from_cut_kernel<<<nb(n, 256), 256, 0, st>>>(scan, eta, n, labels, flags);
    note_launch(2);
    int32_t hf = 0;
    SCK(cudaMemcpyAsync(&hf, flags, 4, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    if (hf) return set_error(ISOC_EINVAL, "eta holds an out-of-range vertex");
    return ISOC_OK;
}

}  // extern "C"
