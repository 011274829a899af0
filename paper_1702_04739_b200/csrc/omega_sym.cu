// K2s: symmetric omega pass with Boruvka round 2 fused (single GPU).
//
// Each unordered pair is computed once: CTA (I, J), I <= J, owns the
// 1024 x 1024 super-tile of super-blocks I (rows) and J (columns) and walks
// its 8 x 8 tiles of 128 x 128.  From every tile of flows
// f_ij = exp(-d_ij/sigma) (diagonal zeroed, vertex_weights,
// /root/reference/pkg/src/isoclust/affinity.py:175-201) it folds
//   rows i in I over the tile's columns  -> pow2 subtree sums, level 7, and
//   columns j in J over the tile's rows  -> the transposed sums (d_ji == d_ij
//                                           bitwise: scipy squares u-v)
// and pushes them through per-row / per-column binary counters into complete
// 1024-wide subtrees PS[J][i] and PS[I][j].  omega_finish folds PS[.][i] over
// the super-blocks (the top of the same pow2 tree, _primitives.py:162-175).
// With comp != NULL the same tiles give each row's exact minimum
// (d, j) over columns in other components: Boruvka round 2 for free.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace isoc {

constexpr int SB = 1024;      // super-block
constexpr int TBK = 128;      // tile
constexpr int SK = 16;        // k chunk
constexpr int STH = 512;      // threads

struct SymStage {
    double A[SK][TBK];
    double B[SK][TBK];
};

struct SymSmem {
    SymStage st[2];
    double rc[TBK][4];         // row counters (3 levels used)
    double cc[SB][4];          // column counters over row tiles
    double xrow[2][TBK];       // row partials of the two column-half warps
    double xcol[8][TBK];       // column partials of the eight row warps
    double xrm[2][TBK];        // row-min exchange
    int32_t xrj[2][TBK];
    double xcm[8][TBK];        // column-min exchange
    int32_t xcj[8][TBK];
    double rmin[TBK];
    int32_t rminj[TBK];
    double cmin[SB];
    int32_t cminj[SB];
    int32_t comp_r[TBK];       // component ids of the tile's rows / columns
    int32_t comp_c[TBK];
    uint64_t exp_tab[256];     // exp table in shared memory (lane-divergent lookups)
};

__device__ __forceinline__ void sym_cp16(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}

__device__ __forceinline__ void sym_load(SymStage& s, const double* __restrict__ XT, int64_t np,
                                         int64_t r0, int64_t c0, int kc) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        const int q = tid + STH * m;            // 0..1023 chunks of 16 B
        const int kk = q >> 6, part = q & 63;
        const int64_t krow = (int64_t)(kc * SK + kk) * np;
        sym_cp16(&s.A[kk][part * 2], XT + krow + r0 + part * 2);
        sym_cp16(&s.B[kk][part * 2], XT + krow + c0 + part * 2);
    }
}

__device__ __forceinline__ bool lex_less(double a, int32_t ja, double b, int32_t jb) {
    return a < b || (a == b && ja < jb);
}

__device__ __forceinline__ double csum_push(double* slots, int idx, double v) {
    // binary counter over 8 tiles (3 levels); returns v unchanged
    int lvl = 0;
    int t = idx;
    while (t & 1) {
        v = __dadd_rn(slots[lvl], v);
        t >>= 1;
        ++lvl;
    }
    slots[lvl] = v;
    return v;
}

__global__ void __launch_bounds__(STH, 1)
omega_sym_kernel(const double* __restrict__ XT, int64_t np, int dpad, int64_t n, int64_t nbs,
                 double sigma, double rs, const int32_t* __restrict__ comp, double* __restrict__ PS,
                 double* __restrict__ PSm, int32_t* __restrict__ PSj) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SymSmem& sm = *reinterpret_cast<SymSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int wr = w >> 1, wc = w & 1;
    const int rg = wr * 4 + (lane >> 3), cl = lane & 7;
    // thread columns (within the tile): wc*64 + 2*cl + 16*q + h, q < 4, h < 2
    // -> the 8 lanes of a row group read 8 consecutive 16-byte chunks (no
    //    bank conflicts); pairs (2p, 2p+1) are this thread's, p = cl + 8q
    // triangular decode of blockIdx -> (I, J), I <= J
    const int64_t b = blockIdx.x;
    int64_t J = (int64_t)((sqrt(8.0 * (double)b + 1.0) - 1.0) / 2.0);
    while ((J + 1) * (J + 2) / 2 <= b) ++J;
    while (J * (J + 1) / 2 > b) --J;
    const int64_t I = b - J * (J + 1) / 2;
    const bool diag = (I == J);
    const int64_t R0 = I * SB, C0 = J * SB;
    const int nk = dpad / SK;
    const bool want_min = comp != nullptr;

    for (int e = tid; e < SB; e += STH) {
        sm.cmin[e] = INFINITY;
        sm.cminj[e] = INT32_MAX;
    }
    for (int e = tid; e < 256; e += STH) sm.exp_tab[e] = ISOC_EXP_TAB[e];
    double acc[4][8];
    // linear pipeline over (ti, tj, kc)
    const int total = 64 * nk;
    sym_load(sm.st[0], XT, np, R0, C0, 0);
    asm volatile("cp.async.commit_group;\n" ::);
    for (int it = 0; it < total; ++it) {
        const int tile = it / nk, kc = it % nk;
        const int ti = tile >> 3, tj = tile & 7;
        if (kc == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
            if (tj == 0 && tid < TBK) {
                sm.rmin[tid] = INFINITY;
                sm.rminj[tid] = INT32_MAX;
            }
        }
        if (kc == 0 && want_min && tid < 2 * TBK) {
            const int64_t g = (tid < TBK) ? R0 + ti * TBK + tid : C0 + tj * TBK + (tid - TBK);
            const int32_t v = g < n ? comp[g] : (tid < TBK ? -1 : -2);
            if (tid < TBK) sm.comp_r[tid] = v; else sm.comp_c[tid - TBK] = v;
        }
        if (it + 1 < total) {
            const int t1 = (it + 1) / nk, k1 = (it + 1) % nk;
            sym_load(sm.st[(it + 1) & 1], XT, np, R0 + (t1 >> 3) * TBK, C0 + (t1 & 7) * TBK, k1);
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 1;\n" ::);
        __syncthreads();
        {
            const SymStage& s = sm.st[it & 1];
#pragma unroll 4
            for (int kk = 0; kk < SK; ++kk) {
                const double2 a01 = *reinterpret_cast<const double2*>(&s.A[kk][rg * 4]);
                const double2 a23 = *reinterpret_cast<const double2*>(&s.A[kk][rg * 4 + 2]);
                const double a[4] = {a01.x, a01.y, a23.x, a23.y};
                double bv[8];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double2 t = *reinterpret_cast<const double2*>(&s.B[kk][wc * 64 + 2 * cl + 16 * q]);
                    bv[2 * q] = t.x;
                    bv[2 * q + 1] = t.y;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = exact_sq_step(acc[i][j], a[i], bv[j]);
            }
        }
        __syncthreads();
        if (kc != nk - 1) continue;

        // ------------------------------------------------ tile epilogue
        const int64_t gr0 = R0 + ti * TBK + rg * 4;   // first global row of this thread
        const int64_t gcb = C0 + tj * TBK;             // first global col of the tile
#define LCOL(j) (wc * 64 + 2 * cl + 16 * ((j) >> 1) + ((j) & 1))
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = __dsqrt_rn(acc[i][j]);
        if (want_min) {
            // row minima (columns ascend within the thread; ties -> smaller column)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int32_t cr = sm.comp_r[rg * 4 + i];
                double m = INFINITY;
                int32_t mj = INT32_MAX;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int64_t gi = gr0 + i, gj = gcb + LCOL(j);
                    const bool ok = gi < n && gj < n && sm.comp_c[LCOL(j)] != cr;
                    if (ok && lex_less(acc[i][j], (int32_t)gj, m, mj)) { m = acc[i][j]; mj = (int32_t)gj; }
                }
#pragma unroll
                for (int off = 1; off < 8; off <<= 1) {
                    const double om = __shfl_xor_sync(0xffffffffu, m, off);
                    const int32_t oj = __shfl_xor_sync(0xffffffffu, mj, off);
                    if (lex_less(om, oj, m, mj)) { m = om; mj = oj; }
                }
                if ((lane & 7) == 0) { sm.xrm[wc][rg * 4 + i] = m; sm.xrj[wc][rg * 4 + i] = mj; }
            }
            // column minima (rows ascend within the thread)
            if (!diag) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int32_t cc = sm.comp_c[LCOL(j)];
                    double m = INFINITY;
                    int32_t mj = INT32_MAX;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int64_t gi = gr0 + i, gj = gcb + LCOL(j);
                        const bool ok = gi < n && gj < n && sm.comp_r[rg * 4 + i] != cc;
                        if (ok && acc[i][j] < m) { m = acc[i][j]; mj = (int32_t)gi; }
                    }
#pragma unroll
                    for (int off = 8; off < 32; off <<= 1) {
                        const double om = __shfl_xor_sync(0xffffffffu, m, off);
                        const int32_t oj = __shfl_xor_sync(0xffffffffu, mj, off);
                        if (lex_less(om, oj, m, mj)) { m = om; mj = oj; }
                    }
                    if ((lane >> 3) == 0) { sm.xcm[wr][LCOL(j)] = m; sm.xcj[wr][LCOL(j)] = mj; }
                }
            }
        }
        // flows in place (diagonal and padding -> 0)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int64_t gi = gr0 + i, gj = gcb + LCOL(j);
                const bool valid = gi < n && gj < n && gi != gj;
                acc[i][j] = valid ? isoc_flow_fast(acc[i][j], sigma, rs, sm.exp_tab) : 0.0;
            }
        // row folds (pow2 tree over the tile's 128 columns): own pairs (level
        // 1), lanes cl^1, cl^2, cl^4 (levels 2-4, one 16-column block per q),
        // own q pairs (levels 5-6), then the two column halves (level 7)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                double x = __dadd_rn(acc[i][2 * q], acc[i][2 * q + 1]);
                double y = __shfl_down_sync(0xffffffffu, x, 1);
                if ((cl & 1) == 0) x = __dadd_rn(x, y);
                y = __shfl_down_sync(0xffffffffu, x, 2);
                if ((cl & 3) == 0) x = __dadd_rn(x, y);
                y = __shfl_down_sync(0xffffffffu, x, 4);
                v[q] = __dadd_rn(x, y);
            }
            if (cl == 0)
                sm.xrow[wc][rg * 4 + i] = __dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3]));
        }
        // column folds: 4 own rows, then the 4 row groups of the warp
        if (!diag) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                double x = __dadd_rn(__dadd_rn(acc[0][j], acc[1][j]), __dadd_rn(acc[2][j], acc[3][j]));
                double y = __shfl_down_sync(0xffffffffu, x, 8);
                if (((lane >> 3) & 1) == 0) x = __dadd_rn(x, y);
                y = __shfl_down_sync(0xffffffffu, x, 16);
                if ((lane >> 3) == 0) sm.xcol[wr][LCOL(j)] = __dadd_rn(x, y);
            }
        }
        __syncthreads();
        if (tid < TBK) {
            const int r = tid;
            const double full = csum_push(sm.rc[r], tj, __dadd_rn(sm.xrow[0][r], sm.xrow[1][r]));
            if (want_min) {
                double m = sm.rmin[r];
                int32_t mj = sm.rminj[r];
                for (int h = 0; h < 2; ++h)
                    if (lex_less(sm.xrm[h][r], sm.xrj[h][r], m, mj)) { m = sm.xrm[h][r]; mj = sm.xrj[h][r]; }
                sm.rmin[r] = m;
                sm.rminj[r] = mj;
            }
            if (tj == 7) {
                const int64_t gi = R0 + ti * TBK + r;
                if (gi < n) {
                    PS[J * n + gi] = full;   // 8 tiles = one complete 1024-wide subtree
                    if (want_min) { PSm[J * n + gi] = sm.rmin[r]; PSj[J * n + gi] = sm.rminj[r]; }
                }
            }
        } else if (!diag && tid < 2 * TBK) {
            const int c = tid - TBK;
            const double x01 = __dadd_rn(sm.xcol[0][c], sm.xcol[1][c]);
            const double x23 = __dadd_rn(sm.xcol[2][c], sm.xcol[3][c]);
            const double x45 = __dadd_rn(sm.xcol[4][c], sm.xcol[5][c]);
            const double x67 = __dadd_rn(sm.xcol[6][c], sm.xcol[7][c]);
            const int col = tj * TBK + c;
            csum_push(sm.cc[col], ti, __dadd_rn(__dadd_rn(x01, x23), __dadd_rn(x45, x67)));
            if (want_min) {
                double m = sm.cmin[col];
                int32_t mj = sm.cminj[col];
                for (int h = 0; h < 8; ++h)
                    if (lex_less(sm.xcm[h][c], sm.xcj[h][c], m, mj)) { m = sm.xcm[h][c]; mj = sm.xcj[h][c]; }
                sm.cmin[col] = m;
                sm.cminj[col] = mj;
            }
        }
        __syncthreads();
    }
    if (!diag) {
        for (int c = tid; c < SB; c += STH) {
            const int64_t gj = C0 + c;
            if (gj < n) {
                PS[I * n + gj] = sm.cc[c][3];   // counter slot of the 8th row tile
                if (want_min) { PSm[I * n + gj] = sm.cmin[c]; PSj[I * n + gj] = sm.cminj[c]; }
            }
        }
    }
}

// omega[i] = pow2 fold of PS[0..nbs)[i] (complete 1024-wide subtrees, zero
// padded); round-2 minimum over the blocks (ties -> smaller column).
__global__ void omega_finish_kernel(const double* __restrict__ PS, const double* __restrict__ PSm,
                                    const int32_t* __restrict__ PSj, int64_t n, int64_t nbs,
                                    double* __restrict__ omega, int32_t* __restrict__ nn_j,
                                    double* __restrict__ nn_d, int8_t* __restrict__ nn_tie) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double slots[40];
    double m = INFINITY;
    int32_t mj = INT32_MAX;
    for (int64_t b = 0; b < nbs; ++b) {
        double v = PS[b * n + i];
        int lvl = 0;
        int64_t t = b;
        while (t & 1) {
            v = __dadd_rn(slots[lvl], v);
            t >>= 1;
            ++lvl;
        }
        slots[lvl] = v;
        if (PSm) {
            const double x = PSm[b * n + i];
            const int32_t xj = PSj[b * n + i];
            if (lex_less(x, xj, m, mj)) { m = x; mj = xj; }
        }
    }
    double acc = 0.0;
    bool have = false;
    for (int lvl = 0; lvl < 40 && (nbs >> lvl) != 0; ++lvl)
        if ((nbs >> lvl) & 1) {
            acc = have ? __dadd_rn(slots[lvl], acc) : slots[lvl];
            have = true;
        }
    omega[i] = acc;
    if (PSm) {
        nn_j[i] = mj == INT32_MAX ? -1 : mj;
        nn_d[i] = m;
        nn_tie[i] = 0;
    }
}

size_t omega_sym_smem() { return sizeof(SymSmem); }

cudaError_t launch_omega_sym(const double* X, int64_t n, int d, double sigma, const int32_t* comp,
                             double* omega, int32_t* nn_j, double* nn_d, int8_t* nn_tie,
                             cudaStream_t st) {
    const int64_t nbs = (n + SB - 1) / SB;
    const int64_t np = nbs * SB;
    const int dpad = (d + SK - 1) / SK * SK;
    double *XT = nullptr, *PS = nullptr, *PSm = nullptr;
    int32_t* PSj = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&XT, (size_t)np * dpad * 8, st);
    if (e != cudaSuccess) return e;
    e = cudaMallocAsync((void**)&PS, (size_t)nbs * n * 8, st);
    if (e != cudaSuccess) return e;
    if (comp) {
        e = cudaMallocAsync((void**)&PSm, (size_t)nbs * n * 8, st);
        if (e != cudaSuccess) return e;
        e = cudaMallocAsync((void**)&PSj, (size_t)nbs * n * 4, st);
        if (e != cudaSuccess) return e;
    }
    e = launch_transpose_pad(X, n, d, np, dpad, XT, st);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(SymSmem);
    e = cudaFuncSetAttribute(omega_sym_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t ctas = nbs * (nbs + 1) / 2;
    const int pid = prof_begin(PK_OMEGA, st);
    omega_sym_kernel<<<(unsigned)ctas, STH, smem, st>>>(XT, np, dpad, n, nbs, sigma, 1.0 / sigma, comp, PS,
                                                        PSm, PSj);
    prof_end(pid, st);
    omega_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(PS, PSm, PSj, n, nbs, omega, nn_j,
                                                                     nn_d, nn_tie);
    note_launch(2);
    cudaFreeAsync(XT, st);
    cudaFreeAsync(PS, st);
    if (PSm) cudaFreeAsync(PSm, st);
    if (PSj) cudaFreeAsync(PSj, st);
    return cudaGetLastError();
}

}  // namespace isoc
