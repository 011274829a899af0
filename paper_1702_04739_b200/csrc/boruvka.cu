// Boruvka MST rounds on the complete Euclidean graph (replaces prim_mst,
// /root/reference/pkg/src/isoclust/mst.py:128-181).
//
// Edge order is the lexicographic key (d_exact, min(u,v), max(u,v)); with
// distinct exact distances the resulting edge set is the unique MST that Prim
// returns.  Per round:
//   1. boruvka_filter_kernel: FP32 Gram-form FFMA tiles (centred data) with
//      a fused per-row arg-min epilogue over columns in other components:
//      best approximate value a1 (column j1) and second best a2.
//   2. certified selection: |a - d_exact^2| <= E_i (rigorous FP32 bound, see
//      DESIGN.md); rows that cannot hold their component's minimum are
//      dropped, rows with a unique candidate get one exact fp64 distance,
//      ambiguous rows are rescanned exactly.
//   3. per-component exact minimum (two 64-bit atomicMin phases: weight bits,
//      then packed endpoints), hooking with mutual-pair resolution, pointer
//      jumping.  The 64-bit keys are what the multi-GPU path all-reduces.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace isoc {

constexpr int FM = 128, FN = 128, FK = 8, FT = 256;
// "no edge" sentinel: INT64_MAX, so keys also order correctly as signed
// int64 (NCCL/torch MIN all-reduce); weight bits of positive doubles and
// packed endpoint pairs are all below 2^63.
constexpr unsigned long long kNoKey = 0x7fffffffffffffffull;

__global__ void fill_u64_kernel(unsigned long long* v, int64_t m, unsigned long long x) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) v[i] = x;
}

constexpr int FSTAGES = 3;
constexpr int FKC = 16;   // k per stage

struct FilterStage {
    float A[FKC][FM];
    float B[FKC][FN];
};

struct FilterSmem {
    FilterStage st[FSTAGES];
    int32_t ccomp[4][FN];   // tile metadata ring: prefetch runs up to 2 chunks (tiles) ahead
    float cnorm[4][FN];
    float red_a1[16][FM];
    float red_a2[16][FM];
    int32_t red_j1[16][FM];
};

__device__ __forceinline__ void approx_update(float a, int32_t j, float& a1, int32_t& j1, float& a2) {
    const bool lt = a < a1;
    a2 = fminf(a2, fmaxf(a, a1));
    j1 = lt ? j : j1;
    a1 = fminf(a1, a);
}

__device__ __forceinline__ void fcp16(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}

// YT: dp x npad fp32 (transposed, zero padded), ny: |y|^2, comp: component ids
// (both padded to npad with comp = -3 beyond n).
__global__ void __launch_bounds__(FT, 1)
boruvka_filter_kernel(const float* __restrict__ YT, const float* __restrict__ ny,
                      const int32_t* __restrict__ comp, int64_t n, int64_t npad, int dp,
                      int64_t row_lo, int64_t row_hi, float* __restrict__ out_a1,
                      int32_t* __restrict__ out_j1, float* __restrict__ out_a2) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FilterSmem& sm = *reinterpret_cast<FilterSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t r0 = row_lo + (int64_t)blockIdx.x * FM;

    int32_t rc[8];
    float rn[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = r0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        const bool ok = row < row_hi;
        rc[i] = ok ? comp[row] : -2;
        rn[i] = ok ? ny[row] : 0.f;
    }
    float a1[8], a2[8];
    int32_t j1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a1[i] = INFINITY; a2[i] = INFINITY; j1[i] = -1; }

    const int nk = dp / FKC;
    const int64_t ntiles = (n + FN - 1) / FN;
    // linear (tile, chunk) stream through a 3-stage cp.async ring; the column
    // metadata (comp, |y|^2) of a tile rides with its first chunk
    int64_t lt = 0;
    int lk = 0, ls = 0;
    auto issue = [&]() {
        if (lt < ntiles) {
            FilterStage& S = sm.st[ls];
            const int kk = tid >> 4, part = tid & 15;    // 16 k-rows x 32 chunks of 16 B
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const int p = part + 16 * m;
                const int64_t krow = (int64_t)(lk * FKC + kk) * npad;
                fcp16(&S.A[kk][p * 4], YT + krow + r0 + p * 4);
                fcp16(&S.B[kk][p * 4], YT + krow + lt * FN + p * 4);
            }
            if (lk == 0 && tid < 64) {
                const int half = tid >> 5, q = tid & 31;
                if (half == 0) fcp16(&sm.ccomp[lt & 3][q * 4], comp + lt * FN + q * 4);
                else fcp16(&sm.cnorm[lt & 3][q * 4], ny + lt * FN + q * 4);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
        ls = (ls + 1 == FSTAGES) ? 0 : ls + 1;
        if (++lk == nk) { lk = 0; ++lt; }
    };
    issue();
    issue();
    int cs = 0;
    for (int64_t t = 0; t < ntiles; ++t) {
        const int64_t c0 = t * FN;
        float acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        for (int kc = 0; kc < nk; ++kc) {
            issue();
            asm volatile("cp.async.wait_group 2;\n" ::);
            __syncthreads();
            const FilterStage& S = sm.st[cs];
#pragma unroll
            for (int kk = 0; kk < FKC; ++kk) {
                const float4 a_lo = *reinterpret_cast<const float4*>(&S.A[kk][ty * 4]);
                const float4 a_hi = *reinterpret_cast<const float4*>(&S.A[kk][64 + ty * 4]);
                const float4 b_lo = *reinterpret_cast<const float4*>(&S.B[kk][tx * 4]);
                const float4 b_hi = *reinterpret_cast<const float4*>(&S.B[kk][64 + tx * 4]);
                const float av[8] = {a_lo.x, a_lo.y, a_lo.z, a_lo.w, a_hi.x, a_hi.y, a_hi.z, a_hi.w};
                const float bv[8] = {b_lo.x, b_lo.y, b_lo.z, b_lo.w, b_hi.x, b_hi.y, b_hi.z, b_hi.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            __syncthreads();
            cs = (cs + 1 == FSTAGES) ? 0 : cs + 1;
        }
        // epilogue: approximate squared distance, other-component arg-min
        const int mb = (int)(t & 3);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int lc = (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            const int32_t cc = sm.ccomp[mb][lc];
            const float cn = sm.cnorm[mb][lc];
            const int32_t col = (int32_t)(c0 + lc);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float a = fmaf(-2.f, acc[i][j], rn[i] + cn);
                a = (cc != rc[i]) ? a : INFINITY;
                approx_update(a, col, a1[i], j1[i], a2[i]);
            }
        }
    }
    // reduce across the 16 column groups
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int lr = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
        sm.red_a1[tx][lr] = a1[i];
        sm.red_a2[tx][lr] = a2[i];
        sm.red_j1[tx][lr] = j1[i];
    }
    __syncthreads();
    if (tid < FM) {
        const int64_t row = r0 + tid;
        float b1 = INFINITY, b2 = INFINITY;
        int32_t bj = -1;
        for (int g = 0; g < 16; ++g) {
            const float x1 = sm.red_a1[g][tid], x2 = sm.red_a2[g][tid];
            const int32_t xj = sm.red_j1[g][tid];
            const bool first = (x1 < b1) || (x1 == b1 && xj >= 0 && (bj < 0 || xj < bj));
            if (first) {
                b2 = fminf(x2, b1);
                b1 = x1;
                bj = xj;
            } else {
                b2 = fminf(b2, x1);
            }
        }
        if (row < row_hi) {
            out_a1[row - row_lo] = b1;
            out_j1[row - row_lo] = bj;
            out_a2[row - row_lo] = b2;
        }
    }
}

// Centre, round to fp32 and store transposed (YT[k * npad + i], zero padded
// to dp x npad); norms in the same FFMA order as the dot products; R_i = |y_i|
// rounded up, for the error bound.
__global__ void prep_fp32_kernel(const double* __restrict__ X, const double* __restrict__ centre,
                                 int64_t n, int d, int dp, int64_t npad, float* __restrict__ YT,
                                 float* __restrict__ ny, float* __restrict__ rad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npad) return;
    float s = 0.f;
    double r2 = 0.0;
    for (int k = 0; k < dp; ++k) {
        float y = 0.f;
        if (k < d && i < n) y = (float)(X[i * d + k] - centre[k]);
        YT[(int64_t)k * npad + i] = y;
        s = fmaf(y, y, s);
        r2 += (double)y * (double)y;
    }
    ny[i] = i < n ? s : INFINITY;   // padding columns can never be candidates
    if (i < n) rad[i] = __double2float_ru(sqrt(r2) * (1.0 + 1e-12));
}

__global__ void column_mean_kernel(const double* __restrict__ X, int64_t n, int d,
                                   double* __restrict__ centre) {
    // one block per dimension; any deterministic mean works (it only
    // conditions the fp32 filter, the bound covers its rounding)
    const int k = blockIdx.x;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += X[i * d + k];
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int off = blockDim.x / 2; off > 0; off >>= 1) {
        if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) centre[k] = red[0] / (double)n;
}

__global__ void max_float_kernel(const float* __restrict__ v, int64_t n, uint32_t* __restrict__ out) {
    float m = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = fmaxf(m, v[i]);
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// ------------------------------------------------------------ selection
__device__ __forceinline__ float row_bound(float Ri, float Rmax, float cd, float cabs) {
    const float s = __fadd_ru(Ri, Rmax);
    return __fadd_ru(__fmul_ru(cd, __fmul_ru(s, s)), __fmul_ru(cabs, s));
}

__global__ void comp_bound_kernel(const float* __restrict__ a1, const float* __restrict__ rad,
                                  const int32_t* __restrict__ comp, int64_t lo, int64_t hi,
                                  const uint32_t* __restrict__ rmax_bits, float cd, float cabs,
                                  uint32_t* __restrict__ compB) {
    const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    const float v = a1[i - lo];
    if (!(v < INFINITY)) return;
    const float E = row_bound(rad[i], __uint_as_float(*rmax_bits), cd, cabs);
    atomicMin(&compB[comp[i]], float_to_ordered(__fadd_ru(v, E)));
}

// Rows that may hold their component's minimum: certified rows get one exact
// distance; ambiguous rows are queued for an exact rescan.
__global__ void candidate_kernel(const double* __restrict__ X, int d, const float* __restrict__ a1,
                                 const int32_t* __restrict__ j1, const float* __restrict__ a2,
                                 const float* __restrict__ rad, const int32_t* __restrict__ comp,
                                 int64_t lo, int64_t hi, const uint32_t* __restrict__ rmax_bits,
                                 float cd, float cabs, const uint32_t* __restrict__ compB,
                                 double* __restrict__ cand_d, int32_t* __restrict__ cand_j,
                                 int8_t* __restrict__ cand_state, int32_t* __restrict__ rescan_list,
                                 int32_t* __restrict__ rescan_count) {
    const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    const int64_t li = i - lo;
    cand_state[li] = 0;
    const float v = a1[li];
    if (!(v < INFINITY)) return;
    const float E = row_bound(rad[i], __uint_as_float(*rmax_bits), cd, cabs);
    const float B = ordered_to_float(compB[comp[i]]);
    if (__fsub_rd(v, E) > B) return;
    if (__fsub_rd(a2[li], E) > __fadd_ru(v, E)) {
        const int32_t j = j1[li];
        cand_d[li] = exact_dist(X + i * d, X + (int64_t)j * d, d);
        cand_j[li] = j;
        cand_state[li] = 1;
    } else {
        cand_state[li] = 2;
        const int32_t slot = atomicAdd(rescan_count, 1);
        rescan_list[slot] = (int32_t)i;
    }
}

// ------------------------------------------------ candidate lists (tc filter)
// A row's list holds its FILTER_LIST_K best (a, j) over the columns that were
// in other components when the filter last ran for its block, plus lb <= a of
// every unlisted column.  Components only merge, so a listed column that is
// still in another component is still a valid candidate, and every column
// not listed has a >= lb.  Per row: a1/j1 = the first still-external entry,
// a2 = min(next still-external entry, lb) -- the (a1, j1, a2) contract of
// the filter kernels, consumed unchanged by comp_bound / candidate_kernel.
// No still-external entry: a1 = inf and the row's lower bound lbo = lb.
__global__ void list_select_kernel(const float* __restrict__ la, const int32_t* __restrict__ lj,
                                   const float* __restrict__ lb, const int32_t* __restrict__ comp,
                                   int64_t lo, int64_t hi, float* __restrict__ a1, int32_t* __restrict__ j1,
                                   float* __restrict__ a2, float* __restrict__ lbo) {
    const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    const int64_t li = i - lo;
    const int32_t c = comp[i];
    float f1 = INFINITY, f2 = INFINITY;
    int32_t g1 = -1;
    int found = 0;
#pragma unroll
    for (int p = 0; p < FILTER_LIST_K; ++p) {
        const int32_t j = lj[li * FILTER_LIST_K + p];
        if (j < 0 || found == 2) continue;
        if (comp[j] == c) continue;
        const float v = la[li * FILTER_LIST_K + p];
        if (found == 0) { f1 = v; g1 = j; } else { f2 = v; }
        ++found;
    }
    const float b = lb[li];
    a1[li] = f1;
    j1[li] = g1;
    a2[li] = fminf(f2, b);
    lbo[li] = found ? INFINITY : b;
}

// Rows whose list has no external entry but whose lower bound does not rule
// them out of their component's minimum (lb - E <= B, or no bound yet) flag
// their 256-row filter block for a refresh.
__global__ void list_refresh_kernel(const float* __restrict__ lbo, const float* __restrict__ rad,
                                    const int32_t* __restrict__ comp, int64_t lo, int64_t hi,
                                    const uint32_t* __restrict__ rmax_bits, float cd, float cabs,
                                    const uint32_t* __restrict__ compB, int32_t* __restrict__ blk_flag,
                                    int32_t* __restrict__ nflag, int32_t* __restrict__ rows_list) {
    const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    const float b = lbo[i - lo];
    if (!(b < INFINITY)) return;
    const float E = row_bound(rad[i], __uint_as_float(*rmax_bits), cd, cabs);
    const float B = ordered_to_float(compB[comp[i]]);
    if (__fsub_rd(b, E) > B) return;   // (false when B is NaN: no bound yet)
    const int64_t blk = (i / 128 - lo / 128) / 2;
    rows_list[atomicAdd(nflag + 1, 1)] = (int32_t)i;           // rows (any order: each row's
                                                               // list is computed on its own)
    if (blk_flag[blk] == 0 && atomicExch(&blk_flag[blk], 1) == 0) atomicAdd(nflag, 1);   // blocks
}

// Exact rescan of one row per CTA: min (d, j) over other-component columns,
// plus whether the minimum is attained twice.  Each thread keeps four
// independent distance chains in flight (columns j, j+T, j+2T, j+3T).
__device__ __forceinline__ void rescan_take(double v, int64_t j, double& m1, double& m2, int64_t& bj) {
    if (v < m1 || (v == m1 && j < bj)) {
        m2 = m1;
        m1 = v;
        bj = j;
    } else {
        m2 = fmin(m2, v);
    }
}

__global__ void rescan_kernel(const double* __restrict__ X, int64_t n, int d,
                              const int32_t* __restrict__ comp, int64_t lo,
                              const int32_t* __restrict__ rescan_list,
                              const int32_t* __restrict__ rescan_count, double* __restrict__ cand_d,
                              int32_t* __restrict__ cand_j, int8_t* __restrict__ cand_tie) {
    const int32_t cnt = *rescan_count;
    __shared__ double xi[512];
    for (int32_t q = blockIdx.x; q < cnt; q += gridDim.x) {
        const int64_t i = rescan_list[q];
        const int32_t ci = comp[i];
        const bool cached = d <= 512;
        __syncthreads();
        if (cached)
            for (int k = threadIdx.x; k < d; k += blockDim.x) xi[k] = X[i * d + k];
        __syncthreads();
        const double* xr = cached ? xi : X + i * d;
        double m1 = INFINITY, m2 = INFINITY;
        int64_t bj = -1;
        const int64_t T = blockDim.x;
        // Each thread walks its columns j = tid, tid+T, ... skipping its own
        // component, and computes four distances at a time.
        int64_t j = threadIdx.x;
        while (true) {
            int64_t jj[4];
            int got = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                while (j < n && comp[j] == ci) j += T;
                jj[u] = j < n ? j : -1;
                got += j < n;
                if (j < n) j += T;
            }
            if (got == 0) break;
            double s[4] = {0.0, 0.0, 0.0, 0.0};
            const double* xj[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) xj[u] = X + (jj[u] >= 0 ? jj[u] : 0) * d;
            for (int k = 0; k < d; ++k) {
                const double a = xr[k];
#pragma unroll
                for (int u = 0; u < 4; ++u) s[u] = exact_sq_step(s[u], a, xj[u][k]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (jj[u] >= 0) rescan_take(__dsqrt_rn(s[u]), jj[u], m1, m2, bj);
        }
        __shared__ double s1[256], s2[256];
        __shared__ int64_t sj[256];
        s1[threadIdx.x] = m1; s2[threadIdx.x] = m2; sj[threadIdx.x] = bj;
        __syncthreads();
        for (int off = blockDim.x / 2; off > 0; off >>= 1) {
            if ((int)threadIdx.x < off) {
                const int o = threadIdx.x + off;
                const bool first = (s1[o] < s1[threadIdx.x]) ||
                                   (s1[o] == s1[threadIdx.x] && sj[o] >= 0 &&
                                    (sj[threadIdx.x] < 0 || sj[o] < sj[threadIdx.x]));
                if (first) {
                    s2[threadIdx.x] = fmin(s2[o], s1[threadIdx.x]);
                    s1[threadIdx.x] = s1[o];
                    sj[threadIdx.x] = sj[o];
                } else {
                    s2[threadIdx.x] = fmin(s2[threadIdx.x], s1[o]);
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            cand_d[i - lo] = s1[0];
            cand_j[i - lo] = (int32_t)sj[0];
            cand_tie[i - lo] = (int8_t)(s2[0] == s1[0]);
        }
        __syncthreads();
    }
}

// Tiled exact rescan: work item (group of RR rescan rows, chunk of RCW
// columns); each column tile of RT points is read once for all RR rows.
// Global -> shared through a cp.async double buffer (8-byte copies transpose
// row-major X into k-major tiles; out-of-range rows, columns and k zero-fill,
// and a zero pair adds an exact (0-0)^2 = 0).  Thread (ty, tx) owns rows
// 4ty..4ty+3 (two broadcast LDS.128) and columns 2tx + 64j + {0,1} (four
// LDS.128): 6 shared loads per 96 fp64 ops.  Per (row, chunk) the
// lexicographic (d, j) minimum over other-component columns and the
// second-smallest value (tie flag) go to scratch; the reduce kernel folds the
// chunks in column order.
constexpr int RR = 32;
constexpr int RT = 256;
constexpr int RCW = 32768;
constexpr int RKC = 16;
constexpr int RBS = RT + 2;   // B row stride (doubles): 16-byte aligned rows
struct RescanStage {
    double A[RKC][RR];
    double B[RKC][RBS];
};
constexpr size_t RESCAN_SMEM = 2 * sizeof(RescanStage);

// Column chunking from the device-side row count: at least the RCW-wide
// chunks, narrower (down to one RT tile) when few row groups would leave SMs
// idle -- (row group, chunk) items fill the SMs about eight times over.
// Partials live at q * nchunks + c; cnt * nchunks <= rescan_capacity(rows).
struct RescanChunks {
    int64_t cw, nchunks;
};
__host__ __device__ __forceinline__ RescanChunks rescan_chunks(int64_t cnt, int64_t n, int sms) {
    const int64_t ngroups = (cnt + RR - 1) / RR;
    const int64_t nc0 = (n + RCW - 1) / RCW, ncmax = (n + RT - 1) / RT;
    int64_t want = ngroups > 0 ? (8 * (int64_t)sms + ngroups - 1) / ngroups : 1;
    if (want > ncmax) want = ncmax;
    const int64_t nch = want > nc0 ? want : nc0;
    int64_t cw = (n + nch - 1) / nch;
    cw = (cw + RT - 1) / RT * RT;
    if (cw < RT) cw = RT;
    return {cw, (n + cw - 1) / cw};
}
static int64_t rescan_capacity(int64_t rows, int64_t n, int sms) {
    return rows * ((n + RCW - 1) / RCW + 1) + (int64_t)RR * (8 * (int64_t)sms + 1);
}

__device__ __forceinline__ void rcp8(void* dst, const void* src, bool ok) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(ok ? 8 : 0));
}

__global__ void __launch_bounds__(256, 1)
rescan_tile_kernel(const double* __restrict__ X, int64_t n, int d, const int32_t* __restrict__ comp,
                   const int32_t* __restrict__ rescan_list, const int32_t* __restrict__ rescan_count,
                   int sms, double* __restrict__ pm1, double* __restrict__ pm2,
                   int32_t* __restrict__ pj) {
    extern __shared__ __align__(16) unsigned char rsm[];
    RescanStage* stg = reinterpret_cast<RescanStage*>(rsm);
    __shared__ int32_t crow[RR];
    __shared__ int32_t grow[RR];
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int64_t cnt = *rescan_count;
    const int64_t ngroups = (cnt + RR - 1) / RR;
    const RescanChunks ch = rescan_chunks(cnt, n, sms);
    const int64_t cw = ch.cw, nchunks = ch.nchunks;
    const int64_t items = ngroups * nchunks;
    const int nkc = (d + RKC - 1) / RKC;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t g = item / nchunks, c = item % nchunks;
        __syncthreads();
        if (tid < RR) {
            const int64_t q = g * RR + tid;
            const int32_t r = q < cnt ? rescan_list[q] : -1;
            grow[tid] = r;
            crow[tid] = r >= 0 ? comp[r] : INT32_MIN;
        }
        __syncthreads();
        double m1[4], m2[4];
        int32_t j1[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { m1[i] = INFINITY; m2[i] = INFINITY; j1[i] = INT32_MAX; }
        const int64_t cend = ((c + 1) * cw < n) ? (c + 1) * cw : n;
        for (int64_t t0 = c * cw; t0 < cend; t0 += RT) {
            double acc[4][8];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
            auto issue = [&](int kc, RescanStage& S) {
                const int k0 = kc * RKC;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int idx = tid + 256 * e;
                    const int r = idx / RKC, kk = idx % RKC;
                    const int32_t gr = grow[r];
                    const bool ok = gr >= 0 && k0 + kk < d;
                    rcp8(&S.A[kk][r], ok ? X + (int64_t)gr * d + k0 + kk : X, ok);
                }
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const int idx = tid + 256 * e;
                    const int j = idx / RKC, kk = idx % RKC;
                    const int64_t col = t0 + j;
                    const bool ok = col < n && k0 + kk < d;
                    rcp8(&S.B[kk][j], ok ? X + col * d + k0 + kk : X, ok);
                }
                asm volatile("cp.async.commit_group;\n" ::);
            };
            issue(0, stg[0]);
            for (int kc = 0; kc < nkc; ++kc) {
                if (kc + 1 < nkc) {
                    issue(kc + 1, stg[(kc + 1) & 1]);
                    asm volatile("cp.async.wait_group 1;\n" ::);
                } else {
                    asm volatile("cp.async.wait_group 0;\n" ::);
                }
                __syncthreads();
                const RescanStage& S = stg[kc & 1];
#pragma unroll
                for (int kk = 0; kk < RKC; ++kk) {
                    const double2 a01 = *reinterpret_cast<const double2*>(&S.A[kk][4 * ty]);
                    const double2 a23 = *reinterpret_cast<const double2*>(&S.A[kk][4 * ty + 2]);
                    const double a[4] = {a01.x, a01.y, a23.x, a23.y};
                    double bb[8];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double2 v = *reinterpret_cast<const double2*>(&S.B[kk][2 * tx + 64 * j]);
                        bb[2 * j] = v.x;
                        bb[2 * j + 1] = v.y;
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[i][j] = exact_sq_step(acc[i][j], a[i], bb[j]);
                }
                __syncthreads();
            }
            // columns in increasing order per thread: a strict < keeps the
            // smallest column among equal values
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int64_t col = t0 + 2 * tx + 64 * (j >> 1) + (j & 1);
                if (col >= n) continue;
                const int32_t cc = comp[col];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (cc == crow[4 * ty + i]) continue;
                    const double v = __dsqrt_rn(acc[i][j]);
                    const bool lt = v < m1[i];
                    const double cand = lt ? m1[i] : v;
                    m2[i] = cand < m2[i] ? cand : m2[i];
                    m1[i] = lt ? v : m1[i];
                    j1[i] = lt ? (int32_t)col : j1[i];
                }
            }
        }
        // reduce the 32 column lanes of each row
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double om1 = __shfl_xor_sync(0xffffffffu, m1[i], off);
                const double om2 = __shfl_xor_sync(0xffffffffu, m2[i], off);
                const int32_t oj = __shfl_xor_sync(0xffffffffu, j1[i], off);
                const bool other_first = om1 < m1[i] || (om1 == m1[i] && oj < j1[i]);
                const double s1 = other_first ? m1[i] : om1;
                const double s2 = other_first ? om2 : m2[i];
                m2[i] = s1 < s2 ? s1 : s2;
                m1[i] = other_first ? om1 : m1[i];
                j1[i] = other_first ? oj : j1[i];
            }
            const int64_t q = g * RR + 4 * ty + i;
            if (tx == 0 && q < cnt) {
                pm1[q * nchunks + c] = m1[i];
                pm2[q * nchunks + c] = m2[i];
                pj[q * nchunks + c] = j1[i];
            }
        }
    }
}

__global__ void rescan_reduce_kernel(const int32_t* __restrict__ rescan_list,
                                     const int32_t* __restrict__ rescan_count, int64_t lo,
                                     int64_t n, int sms, const double* __restrict__ pm1,
                                     const double* __restrict__ pm2, const int32_t* __restrict__ pj,
                                     double* __restrict__ cand_d, int32_t* __restrict__ cand_j,
                                     int8_t* __restrict__ cand_tie) {
    const int64_t cnt = *rescan_count;
    const int64_t nchunks = rescan_chunks(cnt, n, sms).nchunks;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt;
         q += (int64_t)gridDim.x * blockDim.x) {
        double m1 = INFINITY, m2 = INFINITY;
        int32_t j1 = INT32_MAX;
        for (int64_t c = 0; c < nchunks; ++c) {
            const double om1 = pm1[q * nchunks + c], om2 = pm2[q * nchunks + c];
            const int32_t oj = pj[q * nchunks + c];
            const bool other_first = om1 < m1 || (om1 == m1 && oj < j1);
            const double s1 = other_first ? m1 : om1;
            const double s2 = other_first ? om2 : m2;
            m2 = s1 < s2 ? s1 : s2;
            m1 = other_first ? om1 : m1;
            j1 = other_first ? oj : j1;
        }
        const int64_t i = rescan_list[q];
        cand_d[i - lo] = m1;
        cand_j[i - lo] = j1 == INT32_MAX ? -1 : j1;
        cand_tie[i - lo] = (int8_t)(m2 == m1);
    }
}

// Exact rescans of the rows in rescan_list (count on the device): tiles ->
// per-chunk partials -> fold, into cand_* (indexed by row - lo).
static cudaError_t launch_rescan(const double* X, int64_t n, int d, const int32_t* comp, int64_t lo,
                                 int64_t rows, const int32_t* rescan_list, const int32_t* rescan_count,
                                 double* cand_d, int32_t* cand_j, int8_t* cand_tie, cudaStream_t st) {
    const int sms = device_sm_count();
    cudaError_t e = ensure_max_dyn_smem((const void*)rescan_tile_kernel, RESCAN_SMEM);
    if (e != cudaSuccess) return e;
    const size_t cap = (size_t)rescan_capacity(rows, n, sms);
    double *pm1 = nullptr, *pm2 = nullptr;
    int32_t* pj = nullptr;
    e = isoc_malloc_async((void**)&pm1, cap * 8, st);
    if (e != cudaSuccess) return e;
    e = isoc_malloc_async((void**)&pm2, cap * 8, st);
    if (e != cudaSuccess) { isoc_free_async(pm1, st); return e; }
    e = isoc_malloc_async((void**)&pj, cap * 4, st);
    if (e != cudaSuccess) { isoc_free_async(pm1, st); isoc_free_async(pm2, st); return e; }
    const int pid = prof_begin(PK_RESCAN, st);
    rescan_tile_kernel<<<sms, 256, RESCAN_SMEM, st>>>(X, n, d, comp, rescan_list, rescan_count, sms, pm1, pm2,
                                                      pj);
    rescan_reduce_kernel<<<sms, 256, 0, st>>>(rescan_list, rescan_count, lo, n, sms, pm1, pm2, pj, cand_d,
                                              cand_j, cand_tie);
    prof_end(pid, st);
    isoc_free_async(pm1, st);
    isoc_free_async(pm2, st);
    isoc_free_async(pj, st);
    return cudaGetLastError();
}

// Round 1 from the fused exact nearest neighbours: every row is a candidate.
__global__ void nn_candidates_kernel(const int32_t* __restrict__ nn_j, const double* __restrict__ nn_d,
                                     const int8_t* __restrict__ nn_tie, int64_t rows,
                                     double* __restrict__ cand_d, int32_t* __restrict__ cand_j,
                                     int8_t* __restrict__ cand_state, int8_t* __restrict__ cand_tie) {
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= rows) return;
    cand_d[li] = nn_d[li];
    cand_j[li] = nn_j[li];
    cand_state[li] = 1;
    cand_tie[li] = nn_tie[li];
}

__global__ void comp_exact_min_kernel(const double* __restrict__ cand_d,
                                      const int8_t* __restrict__ cand_state,
                                      const int32_t* __restrict__ comp, int64_t lo, int64_t hi,
                                      unsigned long long* __restrict__ compD) {
    const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    if (!cand_state[i - lo]) return;
    atomicMin(&compD[comp[i]], (unsigned long long)__double_as_longlong(cand_d[i - lo]));
}

__device__ __forceinline__ unsigned long long pack_edge(int64_t a, int64_t b) {
    const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
    return (unsigned long long)((lo << 32) | hi);
}

__global__ void comp_edge_kernel(const double* __restrict__ cand_d, const int32_t* __restrict__ cand_j,
                                 const int8_t* __restrict__ cand_state,
                                 const int32_t* __restrict__ comp, int64_t lo, int64_t hi,
                                 const unsigned long long* __restrict__ compD,
                                 unsigned long long* __restrict__ compE) {
    const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    const int64_t li = i - lo;
    if (!cand_state[li]) return;
    const int32_t c = comp[i];
    if ((unsigned long long)__double_as_longlong(cand_d[li]) != compD[c]) return;
    atomicMin(&compE[c], pack_edge(i, cand_j[li]));
}

// Exact ties at a component's minimum weight (a different edge, or a row
// whose own minimum is attained twice) make the MST possibly non-unique.
__global__ void comp_tie_kernel(const double* __restrict__ cand_d, const int32_t* __restrict__ cand_j,
                                const int8_t* __restrict__ cand_state, const int8_t* __restrict__ cand_tie,
                                const int32_t* __restrict__ comp, int64_t lo, int64_t hi,
                                const unsigned long long* __restrict__ compD,
                                const unsigned long long* __restrict__ compE,
                                int32_t* __restrict__ ties) {
    const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    const int64_t li = i - lo;
    if (!cand_state[li]) return;
    const int32_t c = comp[i];
    if ((unsigned long long)__double_as_longlong(cand_d[li]) != compD[c]) return;
    if (pack_edge(i, cand_j[li]) != compE[c] || cand_tie[li]) atomicAdd(ties, 1);
}

// succ[c] = component on the other side of c's minimum edge (reps only).
__global__ void hook_kernel(const int32_t* __restrict__ comp, int64_t n,
                            const unsigned long long* __restrict__ compE, int32_t* __restrict__ succ) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    if (comp[c] != c) return;  // not a representative
    const unsigned long long e = compE[c];
    if (e == kNoKey) { succ[c] = (int32_t)c; return; }
    const int64_t a = (int64_t)(e >> 32), b = (int64_t)(e & 0xffffffffull);
    const int32_t ca = comp[a], cb = comp[b];
    succ[c] = (ca == c) ? cb : ca;
}

// Mutual pairs: the smaller representative becomes the root; every other
// hooked representative contributes its edge once.
__global__ void resolve_emit_kernel(const int32_t* __restrict__ comp, int64_t n,
                                    const unsigned long long* __restrict__ compE,
                                    const unsigned long long* __restrict__ compD,
                                    int32_t* __restrict__ succ, int32_t* __restrict__ succ2,
                                    int32_t* __restrict__ eu, int32_t* __restrict__ ev,
                                    double* __restrict__ ed, int32_t* __restrict__ ecount) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    if (comp[c] != c) return;
    int32_t s = succ[c];
    if (s != c && succ[s] == c && c < s) s = (int32_t)c;
    succ2[c] = s;
    if (s != c) {
        const unsigned long long e = compE[c];
        const int32_t slot = atomicAdd(ecount, 1);
        eu[slot] = (int32_t)(e >> 32);
        ev[slot] = (int32_t)(e & 0xffffffffull);
        ed[slot] = __longlong_as_double((long long)compD[c]);
    }
}

__global__ void jump_kernel(const int32_t* __restrict__ comp, int64_t n, int32_t* __restrict__ succ,
                            int32_t* __restrict__ changed) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    if (comp[c] != c) return;
    const int32_t s = succ[c], ss = succ[s];
    if (s != ss) {
        succ[c] = ss;
        *changed = 1;
    }
}

__global__ void relabel_kernel(int32_t* __restrict__ comp, int64_t n, const int32_t* __restrict__ succ,
                               int32_t* __restrict__ nroots) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t c = comp[i];
    const int32_t r = succ[c];
    comp[i] = r;
    if (i == r) atomicAdd(nroots, 1);
}

__global__ void absmax_kernel(const float* __restrict__ v, int64_t m, uint32_t* __restrict__ out) {
    float x = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        x = fmaxf(x, fabsf(v[i]));
    for (int off = 16; off > 0; off >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(x));
}

cudaError_t launch_absmax(const float* v, int64_t m, uint32_t* out, cudaStream_t st) {
    cudaMemsetAsync(out, 0, sizeof(uint32_t), st);
    absmax_kernel<<<296, 256, 0, st>>>(v, m, out);
    note_launch();
    return cudaGetLastError();
}

// ------------------------------------------------------------ launchers
static inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

cudaError_t launch_prep_fp32(const double* X, int64_t n, int d, int dp, int64_t npad, double* centre,
                             float* Y, float* ny, float* rad, uint32_t* rmax_bits, cudaStream_t st) {
    column_mean_kernel<<<d, 256, 0, st>>>(X, n, d, centre);
    prep_fp32_kernel<<<blocks_for(npad, 256), 256, 0, st>>>(X, centre, n, d, dp, npad, Y, ny, rad);
    cudaMemsetAsync(rmax_bits, 0, sizeof(uint32_t), st);
    max_float_kernel<<<296, 256, 0, st>>>(rad, n, rmax_bits);
    note_launch(3);
    return cudaGetLastError();
}

cudaError_t launch_boruvka_filter(const float* Y, const float* ny, const int32_t* comp, int64_t n,
                                  int64_t npad, int dp, int64_t lo, int64_t hi, float* a1, int32_t* j1,
                                  float* a2, cudaStream_t st) {
    if (hi <= lo) return cudaSuccess;
    const size_t smem = sizeof(FilterSmem);
    cudaError_t e = ensure_max_dyn_smem((const void*)boruvka_filter_kernel, (size_t)((int)smem));
    if (e != cudaSuccess) return e;
    const int pid = prof_begin(PK_FILTER, st);
    boruvka_filter_kernel<<<blocks_for(hi - lo, FM), FT, smem, st>>>(Y, ny, comp, n, npad, dp, lo, hi,
                                                                       a1, j1, a2);
    prof_end(pid, st);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_boruvka_select(const double* X, int64_t n, int d, const float* a1,
                                  const int32_t* j1, const float* a2, const float* rad,
                                  const uint32_t* rmax_bits, float cd, float cabs, const int32_t* comp,
                                  int64_t lo, int64_t hi, uint32_t* compB, double* cand_d,
                                  int32_t* cand_j, int8_t* cand_state, int8_t* cand_tie,
                                  int32_t* rescan_list, int32_t* rescan_count, cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return cudaSuccess;
    cudaMemsetAsync(compB, 0xff, (size_t)n * sizeof(uint32_t), st);
    cudaMemsetAsync(rescan_count, 0, sizeof(int32_t), st);
    cudaMemsetAsync(cand_tie, 0, (size_t)rows, st);
    comp_bound_kernel<<<blocks_for(rows, 256), 256, 0, st>>>(a1, rad, comp, lo, hi, rmax_bits, cd,
                                                              cabs, compB);
    candidate_kernel<<<blocks_for(rows, 256), 256, 0, st>>>(X, d, a1, j1, a2, rad, comp, lo, hi,
                                                             rmax_bits, cd, cabs, compB, cand_d, cand_j,
                                                             cand_state, rescan_list, rescan_count);
    cudaError_t e = launch_rescan(X, n, d, comp, lo, rows, rescan_list, rescan_count, cand_d, cand_j, cand_tie, st);
    note_launch(4);
    return e;
}

cudaError_t launch_list_select(const float* la, const int32_t* lj, const float* lb, const int32_t* comp,
                               int64_t lo, int64_t hi, float* a1, int32_t* j1, float* a2, float* lbo,
                               cudaStream_t st) {
    if (hi <= lo) return cudaSuccess;
    list_select_kernel<<<blocks_for(hi - lo, 256), 256, 0, st>>>(la, lj, lb, comp, lo, hi, a1, j1, a2, lbo);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_list_refresh(const float* a1, const float* lbo, const float* rad, const int32_t* comp,
                                int64_t n, int64_t lo, int64_t hi, const uint32_t* rmax_bits, float cd,
                                float cabs, uint32_t* compB, int32_t* blk_flag, int64_t nblk, int32_t* nflag,
                                int32_t* rows_list, cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return cudaSuccess;
    cudaMemsetAsync(compB, 0xff, (size_t)n * sizeof(uint32_t), st);
    cudaMemsetAsync(blk_flag, 0, (size_t)nblk * sizeof(int32_t), st);
    cudaMemsetAsync(nflag, 0, 2 * sizeof(int32_t), st);
    comp_bound_kernel<<<blocks_for(rows, 256), 256, 0, st>>>(a1, rad, comp, lo, hi, rmax_bits, cd, cabs, compB);
    list_refresh_kernel<<<blocks_for(rows, 256), 256, 0, st>>>(lbo, rad, comp, lo, hi, rmax_bits, cd, cabs,
                                                                compB, blk_flag, nflag, rows_list);
    note_launch(2);
    return cudaGetLastError();
}

// Tiny problems (n^2 d small, e.g. C1): every row is rescanned exactly --
// the tiled exact rescan over all rows costs less than a filter launch, its
// list bookkeeping and the host round trip of a refresh.
__global__ void all_rows_rescan_kernel(int64_t lo, int64_t hi, int8_t* __restrict__ cand_state,
                                       int32_t* __restrict__ rescan_list, int32_t* __restrict__ rescan_count) {
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li == 0) *rescan_count = (int32_t)(hi - lo);
    if (li >= hi - lo) return;
    cand_state[li] = 2;
    rescan_list[li] = (int32_t)(lo + li);
}

cudaError_t launch_boruvka_exact_all(const double* X, int64_t n, int d, const int32_t* comp, int64_t lo,
                                     int64_t hi, double* cand_d, int32_t* cand_j, int8_t* cand_state,
                                     int8_t* cand_tie, int32_t* rescan_list, int32_t* rescan_count,
                                     cudaStream_t st) {
    const int64_t rows = hi - lo;
    if (rows <= 0) return cudaSuccess;
    cudaMemsetAsync(cand_tie, 0, (size_t)rows, st);
    all_rows_rescan_kernel<<<blocks_for(rows, 256), 256, 0, st>>>(lo, hi, cand_state, rescan_list, rescan_count);
    cudaError_t e = launch_rescan(X, n, d, comp, lo, rows, rescan_list, rescan_count, cand_d, cand_j, cand_tie, st);
    note_launch(3);
    return e;
}

cudaError_t launch_nn_candidates(const int32_t* nn_j, const double* nn_d, const int8_t* nn_tie,
                                 int64_t rows, double* cand_d, int32_t* cand_j, int8_t* cand_state,
                                 int8_t* cand_tie, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    nn_candidates_kernel<<<blocks_for(rows, 256), 256, 0, st>>>(nn_j, nn_d, nn_tie, rows, cand_d,
                                                                 cand_j, cand_state, cand_tie);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_comp_exact_min(const double* cand_d, const int8_t* cand_state,
                                  const int32_t* comp, int64_t n, int64_t lo, int64_t hi,
                                  unsigned long long* compD, cudaStream_t st) {
    fill_u64_kernel<<<blocks_for(n, 256), 256, 0, st>>>(compD, n, kNoKey);
    if (hi > lo)
        comp_exact_min_kernel<<<blocks_for(hi - lo, 256), 256, 0, st>>>(cand_d, cand_state, comp, lo,
                                                                         hi, compD);
    note_launch(2);
    return cudaGetLastError();
}

cudaError_t launch_comp_edge(const double* cand_d, const int32_t* cand_j, const int8_t* cand_state,
                             const int32_t* comp, int64_t n, int64_t lo, int64_t hi,
                             const unsigned long long* compD, unsigned long long* compE,
                             cudaStream_t st) {
    fill_u64_kernel<<<blocks_for(n, 256), 256, 0, st>>>(compE, n, kNoKey);
    if (hi > lo)
        comp_edge_kernel<<<blocks_for(hi - lo, 256), 256, 0, st>>>(cand_d, cand_j, cand_state, comp,
                                                                    lo, hi, compD, compE);
    note_launch(2);
    return cudaGetLastError();
}

cudaError_t launch_comp_ties(const double* cand_d, const int32_t* cand_j, const int8_t* cand_state,
                             const int8_t* cand_tie, const int32_t* comp, int64_t lo, int64_t hi,
                             const unsigned long long* compD, const unsigned long long* compE,
                             int32_t* ties, cudaStream_t st) {
    if (hi > lo)
        comp_tie_kernel<<<blocks_for(hi - lo, 256), 256, 0, st>>>(cand_d, cand_j, cand_state,
                                                                   cand_tie, comp, lo, hi, compD,
                                                                   compE, ties);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_hook_contract(int32_t* comp, int64_t n, const unsigned long long* compD,
                                 const unsigned long long* compE, int32_t* succ, int32_t* succ2,
                                 int32_t* eu, int32_t* ev, double* ed, int32_t* ecount,
                                 int32_t* changed, int32_t* nroots, cudaStream_t st) {
    const unsigned g = blocks_for(n, 256);
    hook_kernel<<<g, 256, 0, st>>>(comp, n, compE, succ);
    resolve_emit_kernel<<<g, 256, 0, st>>>(comp, n, compE, compD, succ, succ2, eu, ev, ed, ecount);
    // pointer jumping until every representative points at a root; a fixed
    // number of passes (log2 n) avoids a host round trip per pass
    int passes = 1;
    while ((int64_t(1) << passes) < n) ++passes;
    for (int p = 0; p < passes + 1; ++p) jump_kernel<<<g, 256, 0, st>>>(comp, n, succ2, changed);
    cudaMemsetAsync(nroots, 0, sizeof(int32_t), st);
    relabel_kernel<<<g, 256, 0, st>>>(comp, n, succ2, nroots);
    note_launch(passes + 4);
    return cudaGetLastError();
}

}  // namespace isoc
