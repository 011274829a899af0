// Exact fp64 passes over all n^2 ordered pairs, never materialising the
// distance matrix.
//
//  K1 sigma_pass: distances bit-identical to scipy cdist (affinity.py:124-158),
//     folded into numpy's pairwise_sum over the flat row-major n*n buffer
//     (auto_sigma, affinity.py:233-241).  Each CTA owns a block of rows and
//     streams 128-column tiles through a 256-column shared-memory ring; each
//     recursion leaf (<=128 flat elements) that lies inside one row is summed
//     from the ring with numpy's 8-accumulator kernel and pushed onto a per-row
//     stack of maximal complete recursion nodes.  Leaves that cross a row
//     boundary are summed by sigma_straddle_kernel; sigma_merge_kernel
//     concatenates the row stacks in flat order, which folds them into the
//     exact recursion tree.  The same pass also yields the exact nearest
//     neighbour of every row (Boruvka round 1) and, when alpha > 0, the
//     pow2 row folds of d for the potentials (affinity.py:204-230).
//  K2 omega_pass: omega_i = pow2 fold over j of exp(-d_ij/sigma), diagonal
//     zeroed (affinity.py:175-201, _primitives.py:162-175).  128-column tiles
//     are complete subtrees of the pow2 fold; a per-row binary counter folds
//     the tile sums.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace isoc {

constexpr int XM = 32;        // rows per CTA
constexpr int XN = 128;       // columns per tile
constexpr int XK = 16;        // k chunk
constexpr int XT = 256;       // threads
constexpr int RING = 256;     // ring columns (two tiles)
constexpr int ROW_CAP = 40;   // per-row stack capacity (<= 2 log2(n/64) + 2 used)
constexpr int PC_LEVELS = 32; // binary-counter levels for pow2 row folds

struct TileSmem {
    double As[XK][XM];
    double Bs[XK][XN + 1];
};

// Accumulate the exact squared distances of rows [r0, r0+XM) x cols
// [c0, c0+XN) into acc (thread owns rows ty+8i, cols tx+32j).
__device__ __forceinline__ void exact_tile(const double* __restrict__ X, int64_t n, int d,
                                           int64_t r0, int64_t c0, TileSmem& sm,
                                           double acc[4][4]) {
    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < d; k0 += XK) {
        __syncthreads();
        // rows: 32 x 16
        for (int e = tid; e < XM * XK; e += XT) {
            int r = e / XK, kk = e % XK;
            int64_t row = r0 + r;
            int k = k0 + kk;
            sm.As[kk][r] = (row < n && k < d) ? X[row * d + k] : 0.0;
        }
        for (int e = tid; e < XN * XK; e += XT) {
            int c = e / XK, kk = e % XK;
            int64_t col = c0 + c;
            int k = k0 + kk;
            sm.Bs[kk][c] = (col < n && k < d) ? X[col * d + k] : 0.0;
        }
        __syncthreads();
        const int kmax = (d - k0) < XK ? (d - k0) : XK;
        for (int kk = 0; kk < kmax; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sm.As[kk][ty + 8 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sm.Bs[kk][tx + 32 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = exact_sq_step(acc[i][j], a[i], b[j]);
        }
    }
}

// Binary-counter push for a pow2 fold whose leaves arrive in order.
__device__ __forceinline__ void counter_push(double* slots, int64_t block_index, double v) {
    int lvl = 0;
    int64_t t = block_index;
    while (t & 1) {
        v = __dadd_rn(slots[lvl], v);
        t >>= 1;
        ++lvl;
    }
    slots[lvl] = v;
}

// Fold the pending left siblings of a counter that received `blocks` leaves;
// missing right subtrees are zero padding (x + 0 == x).
__device__ __forceinline__ double counter_flush(const double* slots, int64_t blocks) {
    double acc = 0.0;
    bool have = false;
    for (int lvl = 0; lvl < PC_LEVELS && (blocks >> lvl) != 0; ++lvl) {
        if ((blocks >> lvl) & 1) {
            acc = have ? __dadd_rn(slots[lvl], acc) : slots[lvl];
            have = true;
        }
    }
    return acc;
}

// Warp-cooperative pow2 fold of the 128 values v(col), col in [0,128):
// returns the subtree sum in lane 0.
template <typename Get>
__device__ __forceinline__ double warp_fold128(Get get) {
    const int lane = threadIdx.x & 31;
    double s = __dadd_rn(__dadd_rn(get(4 * lane), get(4 * lane + 1)),
                         __dadd_rn(get(4 * lane + 2), get(4 * lane + 3)));
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        double o = __shfl_down_sync(0xffffffffu, s, off);
        if ((lane & (2 * off - 1)) == 0) s = __dadd_rn(s, o);
    }
    return s;
}

struct NNState {
    double m1, m2;
    int64_t j1;
};

__device__ __forceinline__ NNState nn_combine(NNState a, NNState b) {
    bool a_first = (a.m1 < b.m1) || (a.m1 == b.m1 && a.j1 < b.j1);
    NNState f = a_first ? a : b;
    NNState s = a_first ? b : a;
    f.m2 = fmin(f.m2, s.m1);
    return f;
}

// --------------------------------------------------------------- K1
struct SigmaSmem {
    TileSmem tile;
    double ring[XM][RING];
    double st_val[XM][ROW_CAP];
    uint64_t st_id[XM][ROW_CAP];
    double pc[XM][PC_LEVELS];
    int64_t lf_start[XM];
    int32_t lf_len[XM];
    uint64_t lf_id[XM];
    int32_t lf_done[XM];
    int32_t st_cnt[XM];
    int32_t st_ovf[XM];
};

__global__ void __launch_bounds__(XT, 2)
sigma_pass_kernel(const double* __restrict__ X, int64_t n, int d, int64_t row_lo, int64_t row_hi,
                  int want_p, double* __restrict__ row_vals, uint64_t* __restrict__ row_ids,
                  int32_t* __restrict__ row_cnt, int32_t* __restrict__ flags,
                  int32_t* __restrict__ nn_j, double* __restrict__ nn_d, int8_t* __restrict__ nn_tie,
                  double* __restrict__ pfold) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SigmaSmem& sm = *reinterpret_cast<SigmaSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t r0 = row_lo + (int64_t)blockIdx.x * XM;
    const int64_t total = n * n;

    if (tid < XM) {
        int64_t row = r0 + tid;
        sm.st_cnt[tid] = 0;
        sm.st_ovf[tid] = 0;
        int done = 1;
        if (row < row_hi) {
            int64_t rs = row * n, re = rs + n;
            Leaf L = find_leaf(total, rs);
            if (L.start < rs) L = (L.start + L.len < re) ? find_leaf(total, L.start + L.len) : Leaf{re, 0, 0};
            if (L.len > 0 && L.start + L.len <= re) {
                done = 0;
                sm.lf_start[tid] = L.start;
                sm.lf_len[tid] = (int32_t)L.len;
                sm.lf_id[tid] = L.hid;
            }
        }
        sm.lf_done[tid] = done;
    }
    NNState nn[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) nn[q] = NNState{INFINITY, INFINITY, -1};

    const int64_t ntiles = (n + XN - 1) / XN;
    for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t c0 = t * XN;
        double acc[4][4];
        exact_tile(X, n, d, r0, c0, sm.tile, acc);
        const int tx = tid & 31, ty = tid >> 5;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                int64_t col = c0 + tx + 32 * j;
                sm.ring[ty + 8 * i][(col) & (RING - 1)] = col < n ? __dsqrt_rn(acc[i][j]) : 0.0;
            }
        __syncthreads();

        // nearest neighbour (exact, ties -> smaller column) for 4 rows per warp
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = warp + 8 * q;
            const int64_t row = r0 + r;
            NNState s{INFINITY, INFINITY, -1};
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                int64_t col = c0 + lane + 32 * m;
                if (col < n && col != row) {
                    double v = sm.ring[r][col & (RING - 1)];
                    s = nn_combine(s, NNState{v, INFINITY, col});
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                NNState o;
                o.m1 = __shfl_xor_sync(0xffffffffu, s.m1, off);
                o.m2 = __shfl_xor_sync(0xffffffffu, s.m2, off);
                o.j1 = __shfl_xor_sync(0xffffffffu, s.j1, off);
                s = nn_combine(s, o);
            }
            nn[q] = nn_combine(nn[q], s);
        }

        // pow2 row folds of d for potentials
        if (want_p) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = warp + 8 * q;
                double s = warp_fold128([&](int c) { return sm.ring[r][(c0 + c) & (RING - 1)]; });
                if (lane == 0) counter_push(sm.pc[r], t, s);
            }
        }

        // sigma leaves ending inside this tile: 8 lanes per row, 4 rows per warp
        {
            const int g = lane >> 3, j8 = lane & 7;
            const int r = warp + 8 * g;
            const int64_t row = r0 + r;
            const int64_t rs = row * n, re = rs + n;
            const unsigned gmask = 0xffu << (8 * g);
            while (true) {
                int active = !sm.lf_done[r] &&
                             (sm.lf_start[r] + sm.lf_len[r] - rs) <= c0 + XN;
                if (!__any_sync(0xffffffffu, active)) break;
                double res = 0.0;
                if (active) {
                    const int64_t ls = sm.lf_start[r] - rs;  // row-relative start
                    const int len = sm.lf_len[r];
                    const int main_end = len - (len % 8);
                    double acc8 = 0.0;
                    if (len >= 8) {
                        acc8 = sm.ring[r][(ls + j8) & (RING - 1)];
                        for (int i = 8; i < main_end; i += 8)
                            acc8 = __dadd_rn(acc8, sm.ring[r][(ls + i + j8) & (RING - 1)]);
                    }
                    double o = __shfl_down_sync(gmask, acc8, 1);
                    if ((j8 & 1) == 0) acc8 = __dadd_rn(acc8, o);
                    o = __shfl_down_sync(gmask, acc8, 2);
                    if ((j8 & 3) == 0) acc8 = __dadd_rn(acc8, o);
                    o = __shfl_down_sync(gmask, acc8, 4);
                    if (j8 == 0) {
                        if (len >= 8) {
                            res = __dadd_rn(acc8, o);
                            for (int i = main_end; i < len; ++i)
                                res = __dadd_rn(res, sm.ring[r][(ls + i) & (RING - 1)]);
                        } else {
                            res = 0.0;
                            for (int i = 0; i < len; ++i)
                                res = __dadd_rn(res, sm.ring[r][(ls + i) & (RING - 1)]);
                        }
                        int cnt = sm.st_cnt[r], ovf = sm.st_ovf[r];
                        stack_push(sm.st_val[r], sm.st_id[r], cnt, ROW_CAP, ovf, res, sm.lf_id[r]);
                        sm.st_cnt[r] = cnt;
                        sm.st_ovf[r] = ovf;
                        int64_t end = sm.lf_start[r] + sm.lf_len[r];
                        if (end >= re) {
                            sm.lf_done[r] = 1;
                        } else {
                            Leaf L = find_leaf(total, end);
                            if (L.start + L.len > re) {
                                sm.lf_done[r] = 1;
                            } else {
                                sm.lf_start[r] = L.start;
                                sm.lf_len[r] = (int32_t)L.len;
                                sm.lf_id[r] = L.hid;
                            }
                        }
                    }
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }

    // outputs
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = warp + 8 * q;
            const int64_t row = r0 + r;
            if (row < row_hi) {
                int64_t li = row - row_lo;
                nn_j[li] = (int32_t)nn[q].j1;
                nn_d[li] = nn[q].m1;
                nn_tie[li] = (int8_t)(nn[q].m2 == nn[q].m1);
                if (want_p) pfold[li] = counter_flush(sm.pc[r], ntiles);
            }
        }
    }
    for (int e = tid; e < XM * ROW_CAP; e += XT) {
        int r = e / ROW_CAP, s = e % ROW_CAP;
        int64_t row = r0 + r;
        if (row < row_hi && s < sm.st_cnt[r]) {
            int64_t li = row - row_lo;
            row_vals[li * ROW_CAP + s] = sm.st_val[r][s];
            row_ids[li * ROW_CAP + s] = sm.st_id[r][s];
        }
    }
    if (tid < XM) {
        int64_t row = r0 + tid;
        if (row < row_hi) {
            row_cnt[row - row_lo] = sm.st_cnt[tid];
            if (sm.st_ovf[tid]) atomicOr(flags, 1);
        }
    }
}

// Leaves of the flat recursion that cross a row boundary.  Boundary b (row
// b starts at flat b*n) owns the leaf containing flat b*n when that leaf
// starts inside row b-1.  One warp per boundary.
__global__ void sigma_straddle_kernel(const double* __restrict__ X, int64_t n, int d,
                                      int64_t b_lo, int64_t b_hi, double* __restrict__ sval,
                                      uint64_t* __restrict__ sid, int8_t* __restrict__ sown) {
    const int lane = threadIdx.x & 31;
    const int64_t b = b_lo + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    if (b >= b_hi) return;
    const int64_t total = n * n;
    Leaf L = find_leaf(total, b * n);
    const bool own = (L.start < b * n) && (L.start / n == b - 1);
    if (!own) {
        if (lane == 0) sown[b - b_lo] = 0;
        return;
    }
    // distances of the leaf elements: lane handles elements lane + 32m
    double v[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        int64_t e = lane + 32 * m;
        v[m] = 0.0;
        if (e < L.len) {
            int64_t f = L.start + e;
            int64_t i = f / n, j = f % n;
            v[m] = exact_dist(X + i * d, X + j * d, d);
        }
    }
    auto get = [&](int64_t e) -> double {
        int src = (int)(e & 31), m = (int)(e >> 5);
        double r = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double t = __shfl_sync(0xffffffffu, v[q], src);
            if (q == m) r = t;
        }
        return r;
    };
    // all lanes walk the same sequential leaf kernel (uniform control flow)
    double res = np_leaf_sum(get, L.len);
    if (lane == 0) {
        sval[b - b_lo] = res;
        sid[b - b_lo] = L.hid;
        sown[b - b_lo] = 1;
    }
}

// Merge level 1: rows [lo, hi) in groups of G rows -> one FoldStack each.
// Sequence per row i: straddle(i) if i > lo and owned, then row stack(i);
// the last group also appends straddle(hi) (hi < n).
__global__ void sigma_merge_rows_kernel(int64_t n, int64_t lo, int64_t hi, int G,
                                        const double* __restrict__ row_vals,
                                        const uint64_t* __restrict__ row_ids,
                                        const int32_t* __restrict__ row_cnt,
                                        const double* __restrict__ sval,
                                        const uint64_t* __restrict__ sid,
                                        const int8_t* __restrict__ sown,
                                        FoldStack* __restrict__ out, int32_t* __restrict__ flags) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ngroups = (hi - lo + G - 1) / G;
    if (g >= ngroups) return;
    FoldStack& S = out[g];
    int cnt = 0, ovf = 0;
    const int64_t a = lo + g * G, b = (a + G < hi) ? a + G : hi;
    for (int64_t i = a; i < b; ++i) {
        if (i > lo && sown[i - lo - 1])
            stack_push(S.value, S.id, cnt, kStackCap, ovf, sval[i - lo - 1], sid[i - lo - 1]);
        const int64_t li = i - lo;
        const int c = row_cnt[li];
        for (int s = 0; s < c; ++s)
            stack_push(S.value, S.id, cnt, kStackCap, ovf, row_vals[li * ROW_CAP + s],
                       row_ids[li * ROW_CAP + s]);
    }
    if (b == hi && hi < n && sown[hi - lo - 1])
        stack_push(S.value, S.id, cnt, kStackCap, ovf, sval[hi - lo - 1], sid[hi - lo - 1]);
    S.count = cnt;
    S.overflow = ovf;
    if (ovf) atomicOr(flags, 2);
}

// Merge groups of G consecutive stacks into one.
__global__ void stack_merge_kernel(const FoldStack* __restrict__ in, int64_t nin, int G,
                                   FoldStack* __restrict__ out, int32_t* __restrict__ flags) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nout = (nin + G - 1) / G;
    if (g >= nout) return;
    FoldStack& S = out[g];
    int cnt = 0, ovf = 0;
    for (int64_t q = g * G; q < nin && q < (g + 1) * G; ++q) {
        const FoldStack& I = in[q];
        ovf |= I.overflow;
        for (int s = 0; s < I.count; ++s)
            stack_push(S.value, S.id, cnt, kStackCap, ovf, I.value[s], I.id[s]);
    }
    S.count = cnt;
    S.overflow = ovf;
    if (ovf) atomicOr(flags, 2);
}

// --------------------------------------------------------------- K2
struct OmegaSmem {
    TileSmem tile;
    double D[XM][XN];
    double pc[XM][PC_LEVELS];
};

__global__ void __launch_bounds__(XT, 2)
omega_pass_kernel(const double* __restrict__ X, int64_t n, int d, int64_t row_lo,
                  int64_t row_hi, double sigma, double* __restrict__ omega) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    OmegaSmem& sm = *reinterpret_cast<OmegaSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tid & 31, ty = tid >> 5;
    const int64_t r0 = row_lo + (int64_t)blockIdx.x * XM;
    const int64_t ntiles = (n + XN - 1) / XN;
    for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t c0 = t * XN;
        double acc[4][4];
        exact_tile(X, n, d, r0, c0, sm.tile, acc);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t row = r0 + ty + 8 * i;
                const int64_t col = c0 + tx + 32 * j;
                double f = 0.0;
                if (col < n && col != row) f = isoc_flow(__dsqrt_rn(acc[i][j]), sigma);
                sm.D[ty + 8 * i][tx + 32 * j] = f;
            }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = warp + 8 * q;
            double s = warp_fold128([&](int c) { return sm.D[r][c]; });
            if (lane == 0) counter_push(sm.pc[r], t, s);
        }
    }
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = warp + 8 * q;
            const int64_t row = r0 + r;
            if (row < row_hi) omega[row - row_lo] = counter_flush(sm.pc[r], ntiles);
        }
    }
}

// ----------------------------------------------------------- launchers
size_t sigma_rowstack_entries(int64_t rows) { return (size_t)rows * ROW_CAP; }

cudaError_t launch_sigma_pass(const double* X, int64_t n, int d, int64_t lo, int64_t hi,
                              int want_p, double* row_vals, uint64_t* row_ids, int32_t* row_cnt,
                              int32_t* flags, int32_t* nn_j, double* nn_d, int8_t* nn_tie,
                              double* pfold, cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return cudaSuccess;
    const size_t smem = sizeof(SigmaSmem);
    cudaError_t e = cudaFuncSetAttribute(sigma_pass_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((rows + XM - 1) / XM);
    sigma_pass_kernel<<<grid, XT, smem, st>>>(X, n, d, lo, hi, want_p, row_vals, row_ids, row_cnt,
                                              flags, nn_j, nn_d, nn_tie, pfold);
    return cudaGetLastError();
}

cudaError_t launch_sigma_straddle(const double* X, int64_t n, int d, int64_t b_lo, int64_t b_hi,
                                  double* sval, uint64_t* sid, int8_t* sown, cudaStream_t st) {
    const int64_t nb = b_hi - b_lo;
    if (nb <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((nb * 32 + 255) / 256);
    sigma_straddle_kernel<<<grid, 256, 0, st>>>(X, n, d, b_lo, b_hi, sval, sid, sown);
    return cudaGetLastError();
}

cudaError_t launch_sigma_merge_rows(int64_t n, int64_t lo, int64_t hi, int G,
                                    const double* row_vals, const uint64_t* row_ids,
                                    const int32_t* row_cnt, const double* sval,
                                    const uint64_t* sid, const int8_t* sown, FoldStack* out,
                                    int32_t* flags, cudaStream_t st) {
    const int64_t ng = (hi - lo + G - 1) / G;
    const unsigned grid = (unsigned)((ng + 127) / 128);
    sigma_merge_rows_kernel<<<grid, 128, 0, st>>>(n, lo, hi, G, row_vals, row_ids, row_cnt, sval,
                                                  sid, sown, out, flags);
    return cudaGetLastError();
}

cudaError_t launch_stack_merge(const FoldStack* in, int64_t nin, int G, FoldStack* out,
                               int32_t* flags, cudaStream_t st) {
    const int64_t nout = (nin + G - 1) / G;
    const unsigned grid = (unsigned)((nout + 127) / 128);
    stack_merge_kernel<<<grid, 128, 0, st>>>(in, nin, G, out, flags);
    return cudaGetLastError();
}

cudaError_t launch_omega_pass(const double* X, int64_t n, int d, int64_t lo, int64_t hi,
                              double sigma, double* omega, cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return cudaSuccess;
    const size_t smem = sizeof(OmegaSmem);
    cudaError_t e = cudaFuncSetAttribute(omega_pass_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((rows + XM - 1) / XM);
    omega_pass_kernel<<<grid, XT, smem, st>>>(X, n, d, lo, hi, sigma, omega);
    return cudaGetLastError();
}

}  // namespace isoc
