// Exact fp64 passes over all n^2 ordered pairs, never materialising the
// distance matrix.
//
//  K1 sigma_pass: distances bit-identical to scipy cdist (affinity.py:124-158),
//     folded into numpy's pairwise_sum over the flat row-major n*n buffer
//     (auto_sigma, affinity.py:233-241).  Each CTA owns 32 rows and streams
//     128-column tiles of the transposed points through a cp.async double
//     buffer.  Recursion leaves start at multiples of 8 and (except the very
//     last leaf) have lengths that are multiples of 8, so numpy's 8-way leaf
//     kernel is an "octet" stream: lane j of an 8-lane group accumulates the
//     flat elements = j (mod 8) of its row; at a leaf end the group combines
//     ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and pushes the value onto the row's
//     stack of complete recursion nodes.  A 7-element carry bridges octets
//     split across tiles.  Leaves crossing a row boundary are summed by
//     sigma_straddle_kernel; merge kernels push the row stacks in flat order,
//     which folds the exact recursion tree.  The same pass yields the exact
//     nearest neighbour of every row (Boruvka round 1) and, when alpha > 0,
//     the pow2 row folds of d (potentials, affinity.py:204-230).
//  K2 omega_pass: omega_i = pow2 fold over j of exp(-d_ij/sigma), diagonal
//     zeroed (affinity.py:175-201, _primitives.py:162-175).  128-column tiles
//     are complete subtrees of the pow2 fold; a per-row binary counter folds
//     the tile sums.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "leaf.h"
#include "kernels.h"
#include "prof.h"

namespace isoc {

constexpr int XM = 32;        // rows per CTA
constexpr int XN = 128;       // columns per tile
constexpr int XK = 16;        // k chunk
constexpr int XTH = 256;      // threads
constexpr int ROW_CAP = kRowCap;  // per-row stack capacity (<= 2 log2(n/64) + 2 used)
constexpr int PC_LEVELS = 32; // binary-counter levels for pow2 row folds

// Transposed, zero-padded copy of the points: XT[k * np + i] = X[i, k] for
// k < dpad (multiple of XK), i < np (multiple of XN).
__global__ void transpose_pad_kernel(const double* __restrict__ X, int64_t n, int d, int64_t np,
                                     int dpad, double* __restrict__ XT) {
    __shared__ double t[32][33];
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int k0 = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int64_t i = i0 + y;
        const int k = k0 + threadIdx.x;
        t[y][threadIdx.x] = (i < n && k < d) ? X[i * d + k] : 0.0;
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int k = k0 + y;
        const int64_t i = i0 + threadIdx.x;
        if (k < dpad && i < np) XT[(int64_t)k * np + i] = t[threadIdx.x][y];
    }
}

struct Stage {
    double A[XK][XM];
    double B[XK][XN];
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Issue the cp.async copies of k-chunk kc for rows [r0, r0+32) and columns
// [c0, c0+128) from XT (row stride np).
__device__ __forceinline__ void load_stage(Stage& s, const double* __restrict__ XT, int64_t np,
                                           int64_t r0, int64_t c0, int kc) {
    const int tid = threadIdx.x;
    // rows: 8-byte copies (a shard's first row may be odd)
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        const int q = tid + XTH * m;
        const int kk = q >> 5, r = q & 31;
        cp_async8(&s.A[kk][r], XT + (int64_t)(kc * XK + kk) * np + r0 + r);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int q = tid + XTH * m;
        const int kk = q >> 6, part = q & 63;
        cp_async16(&s.B[kk][part * 2], XT + (int64_t)(kc * XK + kk) * np + c0 + part * 2);
    }
}

__device__ __forceinline__ void compute_stage(const Stage& s, double acc[4][4]) {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
    for (int kk = 0; kk < XK; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = s.A[kk][ty + 8 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = s.B[kk][tx + 32 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = exact_sq_step(acc[i][j], a[i], b[j]);
    }
}

// Software pipeline over (tile, k-chunk): the epilogue of tile t runs while
// the first chunk of tile t+1 is in flight.  `epi(t, acc)` must end with all
// threads done reading shared state it shares with the next epilogue.
template <typename Epi>
__device__ __forceinline__ void exact_tiles(const double* __restrict__ XT, int64_t np, int dpad,
                                            int64_t r0, int64_t ntiles, Stage* st, Epi epi) {
    const int nk = dpad / XK;
    double acc[4][4];
    int buf = 0;
    load_stage(st[0], XT, np, r0, 0, 0);
    cp_commit();
    for (int64_t t = 0; t < ntiles; ++t) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
        for (int kc = 0; kc < nk; ++kc) {
            // prefetch the next (tile, chunk) while this one is consumed
            if (kc + 1 < nk) load_stage(st[buf ^ 1], XT, np, r0, t * XN, kc + 1);
            else if (t + 1 < ntiles) load_stage(st[buf ^ 1], XT, np, r0, (t + 1) * XN, 0);
            cp_commit();
            cp_wait<1>();
            __syncthreads();
            compute_stage(st[buf], acc);
            __syncthreads();
            buf ^= 1;
        }
        epi(t, acc);
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

// per-thread running (m1, j1, m2) with columns visited in increasing order
__device__ __forceinline__ void nn_update(NNState& s, double v, int64_t j) {
    const bool lt = v < s.m1;
    s.m2 = fmin(s.m2, lt ? s.m1 : v);
    s.m1 = lt ? v : s.m1;
    s.j1 = lt ? j : s.j1;
}

// --------------------------------------------------------------- K1
struct SigmaSmem {
    Stage st[2];
    double D[XM][XN + 1];
    double st_val[XM][ROW_CAP];
    uint64_t st_id[XM][ROW_CAP];
    double carry[XM][8];
    double pc[XM][PC_LEVELS];
    int32_t st_cnt[XM];
    int32_t st_ovf[XM];
};

__global__ void __launch_bounds__(XTH, 2)
sigma_pass_kernel(const double* __restrict__ XT, int64_t np, int dpad, int64_t n, int64_t row_lo,
                  int64_t row_hi, int want_p, double* __restrict__ row_vals,
                  uint64_t* __restrict__ row_ids, int32_t* __restrict__ row_cnt,
                  int32_t* __restrict__ flags, int32_t* __restrict__ nn_j, double* __restrict__ nn_d,
                  int8_t* __restrict__ nn_tie, double* __restrict__ pfold) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SigmaSmem& sm = *reinterpret_cast<SigmaSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = lane, ty = warp;
    const int64_t r0 = row_lo + (int64_t)blockIdx.x * XM;
    const int64_t total = n * n;

    // octet-stream state: group g of warp w owns row w + 8g; lane j8 owns
    // accumulator j8.  [s_first, e_last) = internal (non-straddling) leaves.
    const int g = lane >> 3, j8 = lane & 7;
    const int orow = warp + 8 * g;
    const int64_t grow = r0 + orow;
    const int64_t rs = grow * n, re = rs + n;
    int64_t s_first = re, e_last = re;
    LeafIter lit;
    lit.start = 0; lit.len = 0; lit.i = 0; lit.sub = 0; lit.T = 0;
    if (grow < row_hi) {
        Leaf L = find_leaf(total, rs);
        if (L.start < rs) L = (L.start + L.len < re) ? find_leaf(total, L.start + L.len) : Leaf{re, 0, 0};
        if (L.len > 0 && L.start + L.len <= re) {
            s_first = L.start;
            lit = leaf_iter_from(total, L.start, L.len, L.hid);
            // the octet stream covers leaves inside the row whose length is a
            // multiple of 8: the row's last leaf is excluded when it straddles
            // into the next row or is the global final leaf with a tail
            // (total % 8 != 0); the straddle kernel sums those.
            Leaf E = find_leaf(total, re - 1);
            const bool final_tail = (E.start + E.len == total) && (total % 8 != 0);
            e_last = (E.start + E.len <= re && !final_tail) ? re : E.start;
        }
    }
    double acc8 = 0.0;
    if (tid < XM) {
        sm.st_cnt[tid] = 0;
        sm.st_ovf[tid] = 0;
    }

    NNState nn[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) nn[i] = NNState{INFINITY, INFINITY, -1};

    const int64_t ntiles = (n + XN - 1) / XN;
    exact_tiles(XT, np, dpad, r0, ntiles, sm.st, [&](int64_t t, double (&acc)[4][4]) {
        const int64_t c0 = t * XN;
        if (c0 + XN <= n && (c0 >= r0 + XM || c0 + XN <= r0)) {
            // interior tile: no padding columns, no diagonal
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double v = __dsqrt_rn(acc[i][j]);
                    sm.D[ty + 8 * i][tx + 32 * j] = v;
                    nn_update(nn[i], v, c0 + tx + 32 * j);
                }
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t row = r0 + ty + 8 * i;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t col = c0 + tx + 32 * j;
                    const double v = __dsqrt_rn(acc[i][j]);
                    sm.D[ty + 8 * i][tx + 32 * j] = col < n ? v : 0.0;
                    if (col < n && col != row) nn_update(nn[i], v, col);
                }
            }
        }
        __syncthreads();
        if (want_p) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = warp + 8 * q;
                double s = warp_fold128([&](int c) { return sm.D[r][c]; });
                if (lane == 0) counter_push(sm.pc[r], t, s);
            }
        }
        // octets of row `orow` that complete inside this tile; offsets are
        // relative to the tile's first flat index tf0 (32-bit)
        const int64_t tf0 = rs + c0;
        const int tlen = (int)((c0 + XN < n) ? XN : (n - c0));
        const int64_t oabs0 = ((tf0 >> 3) > (s_first >> 3)) ? (tf0 >> 3) : (s_first >> 3);
        const int64_t lim = (tf0 + tlen < e_last) ? tf0 + tlen : e_last;
        const int nq = (grow < row_hi) ? max(0, (int)((lim >> 3) - oabs0)) : 0;
        const int base = (int)(oabs0 * 8 - tf0);
        // Leaves hold >= 8 octets, so at most two leaf ends fall among the
        // <= 16 octets of a tile: ea / eb = octet count at which they close.
        int ea = 0, eb = 0;
        LeafIter lit2 = lit;
        if (nq > 0) {
            const int64_t rel = lit.start + lit.len - (tf0 + base);
            if (rel <= 8 * (int64_t)nq) {
                ea = (int)(rel >> 3);
                if (lit.start + lit.len < e_last) {
                    leaf_next(lit2, total);
                    const int64_t rel2 = lit2.start + lit2.len - (tf0 + base);
                    if (rel2 <= 8 * (int64_t)nq) eb = (int)(rel2 >> 3);
                }
            }
        }
        int nq_max = nq;
#pragma unroll
        for (int off = 8; off < 32; off <<= 1) nq_max = max(nq_max, __shfl_xor_sync(0xffffffffu, nq_max, off));
        double pa = 0.0, pb = 0.0;
        if (nq_max > 0) {
            // rows with no octets here read in-bounds garbage that is discarded
            const double* drow = &sm.D[orow][0];
            const int fb = nq > 0 ? base : 0;
            {
                const int f = fb + j8;
                const double x = f < 0 ? sm.carry[orow][j8] : drow[f];
                if (nq > 0) acc8 = __dadd_rn(acc8, x);
                if (ea == 1) { pa = acc8; acc8 = 0.0; }
            }
#pragma unroll
            for (int q = 1; q < 16; ++q) {
                if (q < nq_max) {
                    const double x = drow[fb + 8 * q + j8];
                    if (q < nq) acc8 = __dadd_rn(acc8, x);
                    if (ea == q + 1) { pa = acc8; acc8 = 0.0; }
                    if (eb == q + 1) { pb = acc8; acc8 = 0.0; }
                }
            }
        }
        // close the (at most two) finished leaves: group-combine the eight
        // lane accumulators, push onto the row's stack, advance the iterator
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const bool ending = (e == 0) ? ea > 0 : eb > 0;
            if (__any_sync(0xffffffffu, ending)) {
                double x = (e == 0) ? pa : pb;
                double y = __shfl_down_sync(0xffffffffu, x, 1);
                if ((j8 & 1) == 0) x = __dadd_rn(x, y);
                y = __shfl_down_sync(0xffffffffu, x, 2);
                if ((j8 & 3) == 0) x = __dadd_rn(x, y);
                y = __shfl_down_sync(0xffffffffu, x, 4);
                if (ending && j8 == 0) {
                    x = __dadd_rn(x, y);
                    int cnt = sm.st_cnt[orow], ovf = sm.st_ovf[orow];
                    stack_push(sm.st_val[orow], sm.st_id[orow], cnt, ROW_CAP, ovf, x, lit.hid());
                    sm.st_cnt[orow] = cnt;
                    sm.st_ovf[orow] = ovf;
                }
            }
            if (ending) {
                if (e == 0) {
                    if (lit.start + lit.len < e_last) lit = lit2;
                } else if (lit.start + lit.len < e_last) {
                    leaf_next(lit, total);
                }
            }
        }
        // carry the partial octet at the tile end
        {
            const int64_t tf1 = tf0 + tlen;
            const int64_t f = (tf1 & ~int64_t(7)) + j8;
            if (grow < row_hi && f < tf1 && f >= tf0) sm.carry[orow][j8] = sm.D[orow][f - tf0];
        }
        __syncthreads();
    });

    // nearest neighbours: reduce the 32 column lanes of each row
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        NNState s = nn[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            NNState o;
            o.m1 = __shfl_xor_sync(0xffffffffu, s.m1, off);
            o.m2 = __shfl_xor_sync(0xffffffffu, s.m2, off);
            o.j1 = __shfl_xor_sync(0xffffffffu, s.j1, off);
            s = nn_combine(s, o);
        }
        const int64_t row = r0 + ty + 8 * i;
        if (lane == 0 && row < row_hi) {
            const int64_t li = row - row_lo;
            nn_j[li] = (int32_t)s.j1;
            nn_d[li] = s.m1;
            nn_tie[li] = (int8_t)(s.m2 == s.m1);
            if (want_p) pfold[li] = counter_flush(sm.pc[ty + 8 * i], ntiles);
        }
    }
    __syncthreads();
    for (int e = tid; e < XM * ROW_CAP; e += XTH) {
        const int r = e / ROW_CAP, s = e % ROW_CAP;
        const int64_t row = r0 + r;
        if (row < row_hi && s < sm.st_cnt[r]) {
            const int64_t li = row - row_lo;
            row_vals[li * ROW_CAP + s] = sm.st_val[r][s];
            row_ids[li * ROW_CAP + s] = sm.st_id[r][s];
        }
    }
    if (tid < XM) {
        const int64_t row = r0 + tid;
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
    Leaf L;
    bool own;
    if (b < n) {
        L = find_leaf(total, b * n);
        own = (L.start < b * n) && (L.start / n == b - 1);
    } else {
        // boundary n: the final leaf, when it has a tail (total % 8 != 0) and
        // lies inside the last row (otherwise an earlier boundary owns it)
        L = find_leaf(total, total - 1);
        own = (total % 8 != 0) && (L.start >= (n - 1) * n);
    }
    if (!own) {
        if (lane == 0) sown[b - b_lo] = 0;
        return;
    }
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
    double res = np_leaf_sum(get, L.len);
    if (lane == 0) {
        sval[b - b_lo] = res;
        sid[b - b_lo] = L.hid;
        sown[b - b_lo] = 1;
    }
}

// Merge level 1: rows [lo, hi) in groups of G rows -> one FoldStack each.
// Sequence per row i: straddle(i) if i > lo and owned, then row stack(i);
// the last group also appends straddle(hi) (boundary n = the final leaf).
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
    if (b == hi && sown[hi - lo - 1])
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
    Stage st[2];
    double D[XM][XN];
    double pc[XM][PC_LEVELS];
    uint64_t exp_tab[256];
};

__global__ void __launch_bounds__(XTH, 2)
omega_pass_kernel(const double* __restrict__ XT, int64_t np, int dpad, int64_t n, int64_t row_lo,
                  int64_t row_hi, double sigma, double rs, const int32_t* __restrict__ comp,
                  double* __restrict__ omega, int32_t* __restrict__ nn_j, double* __restrict__ nn_d,
                  int8_t* __restrict__ nn_tie) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    OmegaSmem& sm = *reinterpret_cast<OmegaSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = lane, ty = warp;
    const int64_t r0 = row_lo + (int64_t)blockIdx.x * XM;
    const int64_t ntiles = (n + XN - 1) / XN;
    for (int e2 = tid; e2 < 256; e2 += XTH) sm.exp_tab[e2] = ISOC_EXP_TAB[e2];
    NNState nn[4];
    int32_t crow[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        nn[i] = NNState{INFINITY, INFINITY, -1};
        const int64_t row = r0 + ty + 8 * i;
        crow[i] = (comp && row < n) ? comp[row] : -1;
    }
    exact_tiles(XT, np, dpad, r0, ntiles, sm.st, [&](int64_t t, double (&acc)[4][4]) {
        const int64_t c0 = t * XN;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t col = c0 + tx + 32 * j;
            const int32_t cc = (comp && col < n) ? comp[col] : -2;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int64_t row = r0 + ty + 8 * i;
                double f = 0.0;
                if (col < n && col != row) {
                    const double dd = __dsqrt_rn(acc[i][j]);
                    f = isoc_flow_fast(dd, sigma, rs, sm.exp_tab);
                    if (comp && cc != crow[i]) nn_update(nn[i], dd, col);
                }
                sm.D[ty + 8 * i][tx + 32 * j] = f;
            }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = warp + 8 * q;
            double s = warp_fold128([&](int c) { return sm.D[r][c]; });
            if (lane == 0) counter_push(sm.pc[r], t, s);
        }
        __syncthreads();
    });
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = warp + 8 * q;
            const int64_t row = r0 + r;
            if (row < row_hi) omega[row - row_lo] = counter_flush(sm.pc[r], ntiles);
        }
    }
    if (comp) {
        // columns were visited in increasing order per lane: reduce the lanes
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            NNState s = nn[i];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                NNState o;
                o.m1 = __shfl_xor_sync(0xffffffffu, s.m1, off);
                o.m2 = __shfl_xor_sync(0xffffffffu, s.m2, off);
                o.j1 = __shfl_xor_sync(0xffffffffu, s.j1, off);
                s = nn_combine(s, o);
            }
            const int64_t row = r0 + ty + 8 * i;
            if (lane == 0 && row < row_hi) {
                nn_j[row - row_lo] = (int32_t)s.j1;
                nn_d[row - row_lo] = s.m1;
                nn_tie[row - row_lo] = (int8_t)(s.m2 == s.m1);
            }
        }
    }
}

// ----------------------------------------------------------- launchers
size_t sigma_rowstack_entries(int64_t rows) { return (size_t)rows * ROW_CAP; }

cudaError_t launch_transpose_pad(const double* X, int64_t n, int d, int64_t np, int dpad, double* XT,
                                 cudaStream_t st) {
    dim3 grid((unsigned)((np + 31) / 32), (unsigned)((dpad + 31) / 32));
    transpose_pad_kernel<<<grid, dim3(32, 8), 0, st>>>(X, n, d, np, dpad, XT);
    note_launch();
    return cudaGetLastError();
}

static cudaError_t make_xt(const double* X, int64_t n, int d, double** XT, int64_t* np, int* dpad,
                           cudaStream_t st) {
    *np = (n + XN - 1) / XN * XN + XN;
    *dpad = (d + XK - 1) / XK * XK;
    cudaError_t e = isoc_malloc_async((void**)XT, (size_t)(*np) * (*dpad) * sizeof(double), st);
    if (e != cudaSuccess) return e;
    return launch_transpose_pad(X, n, d, *np, *dpad, *XT, st);
}

cudaError_t launch_sigma_pass(const double* X, int64_t n, int d, int64_t lo, int64_t hi,
                              int want_p, double* row_vals, uint64_t* row_ids, int32_t* row_cnt,
                              int32_t* flags, int32_t* nn_j, double* nn_d, int8_t* nn_tie,
                              double* pfold, cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return cudaSuccess;
    double* XT = nullptr;
    int64_t np = 0;
    int dpad = 0;
    cudaError_t e = make_xt(X, n, d, &XT, &np, &dpad, st);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(SigmaSmem);
    e = ensure_max_dyn_smem((const void*)sigma_pass_kernel, (size_t)((int)smem));
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((rows + XM - 1) / XM);
    const int pid = prof_begin(PK_SIGMA, st);
    sigma_pass_kernel<<<grid, XTH, smem, st>>>(XT, np, dpad, n, lo, hi, want_p, row_vals, row_ids,
                                              row_cnt, flags, nn_j, nn_d, nn_tie, pfold);
    prof_end(pid, st);
    note_launch();
    isoc_free_async(XT, st);
    return cudaGetLastError();
}

cudaError_t launch_sigma_straddle(const double* X, int64_t n, int d, int64_t b_lo, int64_t b_hi,
                                  double* sval, uint64_t* sid, int8_t* sown, cudaStream_t st) {
    const int64_t nb = b_hi - b_lo;
    if (nb <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((nb * 32 + 255) / 256);
    sigma_straddle_kernel<<<grid, 256, 0, st>>>(X, n, d, b_lo, b_hi, sval, sid, sown);
    note_launch();
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
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_stack_merge(const FoldStack* in, int64_t nin, int G, FoldStack* out,
                               int32_t* flags, cudaStream_t st) {
    const int64_t nout = (nin + G - 1) / G;
    const unsigned grid = (unsigned)((nout + 127) / 128);
    stack_merge_kernel<<<grid, 128, 0, st>>>(in, nin, G, out, flags);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_omega_pass(const double* X, int64_t n, int d, int64_t lo, int64_t hi,
                              double sigma, const int32_t* comp, double* omega, int32_t* nn_j,
                              double* nn_d, int8_t* nn_tie, cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return cudaSuccess;
    double* XT = nullptr;
    int64_t np = 0;
    int dpad = 0;
    cudaError_t e = make_xt(X, n, d, &XT, &np, &dpad, st);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(OmegaSmem);
    e = ensure_max_dyn_smem((const void*)omega_pass_kernel, (size_t)((int)smem));
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((rows + XM - 1) / XM);
    const int pid = prof_begin(PK_OMEGA, st);
    omega_pass_kernel<<<grid, XTH, smem, st>>>(XT, np, dpad, n, lo, hi, sigma, 1.0 / sigma, comp, omega,
                                               nn_j, nn_d, nn_tie);
    prof_end(pid, st);
    note_launch();
    isoc_free_async(XT, st);
    return cudaGetLastError();
}

}  // namespace isoc
