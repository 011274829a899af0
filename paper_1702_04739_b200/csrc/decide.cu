// Tree phase on the device: the level-synchronous decision sweep, witness
// labels and the exact subpartition cost.
//
//  decide_kernel restates par_decide (/root/reference/pkg/src/isoclust/
//  parengine.py:116-209), itself field-for-field equal to decide
//  (isoperim.py:82-144).  Vertices live in BFS-position space, so a level is
//  a contiguous position range and the canonical (reverse-BFS) order inside
//  a level is descending position.  Per level:
//    A  branch conditions on frozen state, cut counts per CTA chunk
//    B  exclusive cut prefix in canonical order; a vertex is committed iff
//       fewer than (k - j) cuts precede it (stop at the k-th cut); committed
//       cuts record their sparsity at slot j + prefix (cut order)
//    C  one thread per parent folds its committed children in descending
//       child rank (the reference's serial same-parent commit order)
//  One cooperative launch covers all levels (software grid barrier).
//
//  labels: extract_labels (isoperim.py:164-181) + _resolve_groups (:147-161)
//  cost:   subpartition_cost (isoperim.py:184-219) with numpy's pairwise
//          np.sum on the stably compacted per-cluster arrays.
#include <cstdint>
#include <cstdlib>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"
#include "prof.h"

namespace isoc {

static inline unsigned nb(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

struct DecideArgs {
    int64_t n;
    int64_t levels;
    const int64_t* level_off;
    const double* f_pos;
    const double* om0;
    const double* p0;
    const int32_t* child_lo;
    const int32_t* child_cnt;
    double thr;
    int64_t k;
    double* om;
    double* p;
    int8_t* code;       // 0 uncommitted, 1 cut, 2 join, 3 discard
    int32_t* excl;      // per-position chunk-local exclusive cut count
    double* spars;      // k
    int32_t* chunk_cnt; // gridDim.x
    int64_t* j_out;
    unsigned int* bar;
};

constexpr int DK_MAXG = 1024;  // chunk counts live in scratch[0, 1024)
#ifndef DK_UA
#define DK_UA 2   // phase A: consecutive elements per thread per pass
#endif
#ifndef DK_UF
#define DK_UF 2   // fold: parents per thread per pass
#endif
#ifndef DK_FOLD_COND
#define DK_FOLD_COND 0  // 1: load a child's f / omega / p only where its condition uses them
#endif
#ifndef DK_MINB
#define DK_MINB 2 // resident CTAs per SM the register budget is sized for
#endif

// Exclusive prefix of the G chunk cut counts into s_pre[0..G] (s_pre[G] =
// level total), computed by every CTA.
__device__ __forceinline__ void chunk_prefix(const int32_t* __restrict__ cnt, int G, int32_t* s_pre,
                                             int32_t* warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int per = (G + blockDim.x - 1) / blockDim.x;   // <= 2 for G <= 1024
    int32_t v[2] = {0, 0};
    int32_t sum = 0;
    for (int i = 0; i < per; ++i) {
        const int q = tid * per + i;
        v[i] = q < G ? ((volatile const int32_t*)cnt)[q] : 0;
        sum += v[i];
    }
    int32_t x = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int32_t t = lane < nw ? warp_tot[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) warp_tot[lane] = t;
    }
    __syncthreads();
    int32_t e = (wid > 0 ? warp_tot[wid - 1] : 0) + x - sum;
    for (int i = 0; i < per; ++i) {
        const int q = tid * per + i;
        if (q <= G) s_pre[q] = e;
        e += v[i];
    }
    if (tid == blockDim.x - 1 && tid * per + per <= G) s_pre[G] = e;
    __syncthreads();
}

__global__ void __launch_bounds__(512, DK_MINB) decide_kernel(DecideArgs A) {
    __shared__ int32_t warp_tot[16];
    __shared__ int32_t s_pre[DK_MAXG + 1];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int bd = blockDim.x;
    const int G = gridDim.x, b = blockIdx.x;
    // Inputs are never mutated.  Instead of copying (om, p) to working
    // arrays per sweep, the deepest level reads om0 / p0 directly and every
    // fold writes its parents' working values (om0 / p0 plus the children's
    // contributions), which the next level up reads; code is written for
    // every decided position and cleared above the level where the sweep
    // stops.  Per level two grid barriers: A (conditions + chunk-local cut
    // ranks) | prefix of the chunk counts in every CTA, then the parents'
    // fold, which also commits each child (the reference's stop at the k-th
    // cut: committed iff fewer than k - j cuts precede it in canonical
    // order) | next level.
    int64_t j = 0;
    const double thr = A.thr;
    int64_t stop_lo = 0;   // positions [0, stop_lo) were never decided
    for (int64_t lv = A.levels - 1; lv >= 0; --lv) {
        const int64_t lo = A.level_off[lv], hi = A.level_off[lv + 1];
        const bool deepest = lv == A.levels - 1;
        const double* pv = deepest ? A.p0 : A.p;
        const double* ov = deepest ? A.om0 : A.om;
        const uint32_t W = (uint32_t)(hi - lo);
        // canonical index c in [0, W) <-> position hi-1-c; chunk b = [b*CH, (b+1)*CH)
        const uint32_t CH = (W + G - 1) / G;
        const uint32_t cb = min(W, (uint32_t)b * CH), ce = min(W, cb + CH);
        int32_t carry = 0;
        for (uint32_t base = cb; base < ce; base += DK_UA * bd) {
            const uint32_t c0 = base + DK_UA * tid;
            double f[DK_UA], pw[DK_UA], ow[DK_UA];
#pragma unroll
            for (int i = 0; i < DK_UA; ++i)
                if (c0 + i < ce) {
                    const int64_t pos = hi - 1 - (c0 + i);
                    f[i] = A.f_pos[pos];
                    pw[i] = pv[pos];
                    ow[i] = ov[pos];
                }
            int32_t cuts = 0;
            uint32_t cutmask = 0;
#pragma unroll
            for (int i = 0; i < DK_UA; ++i)
                if (c0 + i < ce) {
                    const double rhs = __dmul_rn(thr, ow[i]);
                    int8_t cond;
                    if (__dadd_rn(f[i], pw[i]) <= rhs) cond = 1;
                    else if (__dsub_rn(pw[i], f[i]) < rhs) cond = 2;
                    else cond = 3;
                    A.code[hi - 1 - (c0 + i)] = cond;  // provisional; the fold clears it if not committed
                    if (cond == 1) { cutmask |= 1u << i; ++cuts; }
                }
            int32_t x = cuts;
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) warp_tot[wid] = x;
            __syncthreads();
            if (wid == 0) {
                int32_t t = lane < nw ? warp_tot[lane] : 0;
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
                    if (lane >= o) t += y;
                }
                if (lane < nw) warp_tot[lane] = t;
            }
            __syncthreads();
            int32_t e = carry + (wid > 0 ? warp_tot[wid - 1] : 0) + x - cuts;
#pragma unroll
            for (int i = 0; i < DK_UA; ++i)
                if (c0 + i < ce) {
                    A.excl[hi - 1 - (c0 + i)] = e;
                    e += (cutmask >> i) & 1;
                }
            carry += warp_tot[nw - 1];
            __syncthreads();
        }
        if (tid == 0) A.chunk_cnt[b] = carry;
        grid_barrier(A.bar);
        chunk_prefix(A.chunk_cnt, G, s_pre, warp_tot);
        const int64_t need = A.k - j;
        const int64_t tot = s_pre[G];
        if (lv > 0) {
            // parents [plo, lo): fold committed children in descending child
            // rank (the reference's serial same-parent commit order), DK_UF
            // parents per thread with their child loads issued together
            const int64_t plo = A.level_off[lv - 1];
            const int64_t PW = lo - plo;
            const int64_t ub = plo + (PW * b) / G, ue = plo + (PW * (b + 1)) / G;
            for (int64_t u0 = ub + tid; u0 < ue; u0 += (int64_t)DK_UF * bd) {
                int32_t clo[DK_UF], cnt[DK_UF];
                double pu[DK_UF], ou[DK_UF];
                int32_t mx = 0;
#pragma unroll
                for (int i = 0; i < DK_UF; ++i) {
                    const int64_t u = u0 + (int64_t)i * bd;
                    cnt[i] = 0;
                    if (u < ue) {
                        clo[i] = A.child_lo[u];
                        cnt[i] = A.child_cnt[u];
                        pu[i] = A.p0[u];
                        ou[i] = A.om0[u];
                    }
                    mx = max(mx, cnt[i]);
                }
                for (int32_t r = 0; r < mx; ++r) {
                    int8_t cd[DK_UF];
                    int32_t ex[DK_UF];
                    double fq[DK_UF], oq[DK_UF], pq[DK_UF];
#pragma unroll
                    for (int i = 0; i < DK_UF; ++i)
                        if (r < cnt[i]) {
                            const int64_t q = clo[i] + cnt[i] - 1 - r;
                            cd[i] = A.code[q];
                            ex[i] = A.excl[q];
#if DK_FOLD_COND
                        }
#pragma unroll
                    for (int i = 0; i < DK_UF; ++i)
                        if (r < cnt[i]) {
                            const int64_t q = clo[i] + cnt[i] - 1 - r;
                            // only the values this child's condition uses
                            fq[i] = cd[i] == 1 || cd[i] == 3 ? A.f_pos[q] : 0.0;
                            oq[i] = cd[i] == 2 || cd[i] == 1 ? ov[q] : 0.0;
                            pq[i] = cd[i] == 1 || cd[i] == 2 ? pv[q] : 0.0;
#else
                            fq[i] = A.f_pos[q];
                            oq[i] = ov[q];
                            pq[i] = pv[q];
#endif
                        }
#pragma unroll
                    for (int i = 0; i < DK_UF; ++i)
                        if (r < cnt[i]) {
                            const int64_t q = clo[i] + cnt[i] - 1 - r;
                            const uint32_t c = (uint32_t)(hi - 1 - q);
                            const int64_t e = (int64_t)s_pre[c / CH] + ex[i];
                            int8_t d = cd[i];
                            if (e < need) {
                                if (d == 1) A.spars[j + e] = __ddiv_rn(__dadd_rn(fq[i], pq[i]), oq[i]);
                            } else {
                                A.code[q] = 0;
                                d = 0;
                            }
                            if (d == 1 || d == 3) {
                                pu[i] = __dadd_rn(pu[i], fq[i]);
                            } else if (d == 2) {
                                ou[i] = __dadd_rn(ou[i], oq[i]);
                                pu[i] = __dadd_rn(pu[i], pq[i]);
                            }
                        }
                }
#pragma unroll
                for (int i = 0; i < DK_UF; ++i) {
                    const int64_t u = u0 + (int64_t)i * bd;
                    if (u < ue) {
                        A.p[u] = pu[i];
                        A.om[u] = ou[i];
                    }
                }
            }
        } else {
            // the root level has no parent fold: commit in place
            for (uint32_t c = cb + tid; c < ce; c += bd) {
                const int64_t pos = hi - 1 - c;
                const int64_t e = (int64_t)s_pre[b] + A.excl[pos];
                if (e < need) {
                    if (A.code[pos] == 1) A.spars[j + e] = __ddiv_rn(__dadd_rn(A.f_pos[pos], pv[pos]), ov[pos]);
                } else {
                    A.code[pos] = 0;
                }
            }
        }
        j += (tot < need) ? tot : need;
        grid_barrier(A.bar);
        if (j >= A.k) { stop_lo = lo; break; }
    }
    for (int64_t q = (int64_t)b * blockDim.x + tid; q < stop_lo; q += (int64_t)G * blockDim.x) A.code[q] = 0;
    if (b == 0 && tid == 0) *A.j_out = j;
}

// Batched decision sweeps: K thresholds share one level-synchronous pass
// (the speculative bisection of SURVEY 8f: the 2^m - 1 thresholds the next m
// bisection steps could visit).  Same per-instance arithmetic as
// decide_kernel; only the feasibility count j per threshold is returned (the
// witness of the chosen threshold is re-derived by one decide_kernel sweep).
constexpr int DB_MAX = 16;

struct DecideBatchArgs {
    int64_t n;
    int64_t levels;
    const int64_t* level_off;
    const double* f_pos;
    const double* om0;
    const double* p0;
    const int32_t* child_lo;
    const int32_t* child_cnt;
    const double* thr;   // K thresholds (device)
    int K;
    int64_t k;
    double* om;          // [K][n]
    double* p;           // [K][n]
    int8_t* code;        // [K][n]
    int32_t* excl;       // [K][n]
    int32_t* chunk_cnt;  // [K][gridDim.x]
    int64_t* j_out;      // [K]
    unsigned int* bar;
};

__global__ void __launch_bounds__(512) decide_batch_kernel(DecideBatchArgs A) {
    // instance kk = blockIdx.x / Gi runs on its own Gi CTAs (local index bi);
    // all CTAs share the grid barriers
    __shared__ int32_t warp_tot[16];
    __shared__ int64_t s_off, s_tot;
    __shared__ int s_all_done;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const int K = A.K;
    const int Gi = gridDim.x / K;
    const int kk = blockIdx.x / Gi, bi = blockIdx.x % Gi;
    // one CTA per instance: the instances are independent, so CTA barriers
    // replace the grid barriers and each CTA stops at its own k-th cut
    const bool solo = Gi == 1;
    const int64_t n = A.n;
    const double thr = A.thr[kk];
    double* om = A.om + kk * n;
    double* pp = A.p + kk * n;
    int8_t* code = A.code + kk * n;
    int32_t* excl = A.excl + kk * n;
    int32_t* chunk_cnt = A.chunk_cnt + kk * Gi;
    // no working copies: the deepest level reads om0 / p0, every fold writes
    // its parents' working values (as decide_kernel)
    int64_t j = 0;
    for (int64_t lv = A.levels - 1; lv >= 0; --lv) {
        const int64_t lo = A.level_off[lv], hi = A.level_off[lv + 1];
        const bool deepest = lv == A.levels - 1;
        const double* pv = deepest ? A.p0 : pp;
        const double* ov = deepest ? A.om0 : om;
        const int64_t W = hi - lo;
        const int64_t cb = W * bi / Gi, ce = W * (bi + 1) / Gi;
        const bool active = j < A.k;
        int64_t carry = 0;
        if (active) {
            for (int64_t base = cb; base < ce; base += blockDim.x) {
                const int64_t c = base + tid;
                int32_t is_cut = 0;
                if (c < ce) {
                    const int64_t pos = hi - 1 - c;
                    const double f = A.f_pos[pos], pw = pv[pos], ow = ov[pos];
                    const double rhs = __dmul_rn(thr, ow);
                    int8_t cond;
                    if (__dadd_rn(f, pw) <= rhs) cond = 1;
                    else if (__dsub_rn(pw, f) < rhs) cond = 2;
                    else cond = 3;
                    is_cut = cond == 1;
                    code[pos] = cond;
                }
                int32_t x = is_cut;
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
                if (c < ce) excl[hi - 1 - c] = (int32_t)(carry + wpre + x - is_cut);
                carry += warp_tot[nw - 1];
                __syncthreads();
            }
        }
        if (tid == 0) chunk_cnt[bi] = (int32_t)carry;
        if (solo) __syncthreads(); else grid_barrier(A.bar);
        if (tid == 0) {
            int64_t pre = 0, tot = 0;
            for (int q = 0; q < Gi; ++q) {
                const int64_t s = chunk_cnt[q];
                if (q < bi) pre += s;
                tot += s;
            }
            s_off = pre;
            s_tot = tot;
        }
        __syncthreads();
        const int64_t need = A.k - j;
        const int64_t off = s_off, tot = s_tot;
        if (active)
            for (int64_t c = cb + tid; c < ce; c += blockDim.x) {
                const int64_t pos = hi - 1 - c;
                if (off + excl[pos] >= need) code[pos] = 0;
            }
        if (solo) __syncthreads(); else grid_barrier(A.bar);
        if (lv > 0 && active) {
            const int64_t plo = A.level_off[lv - 1], phi = lo;
            const int64_t PW = phi - plo;
            for (int64_t u = plo + (PW * bi) / Gi + tid; u < plo + (PW * (bi + 1)) / Gi; u += blockDim.x) {
                const int32_t clo = A.child_lo[u], cnt = A.child_cnt[u];
                double pu = A.p0[u], ou = A.om0[u];
                for (int32_t q = clo + cnt - 1; q >= clo; --q) {
                    const int8_t cd = code[q];
                    if (cd == 1 || cd == 3) {
                        pu = __dadd_rn(pu, A.f_pos[q]);
                    } else if (cd == 2) {
                        ou = __dadd_rn(ou, ov[q]);
                        pu = __dadd_rn(pu, pv[q]);
                    }
                }
                {
                    pp[u] = pu;
                    om[u] = ou;
                }
            }
        }
        if (active) j += (tot < need) ? tot : need;
        // instances publish whether they are done; stop when all are
        if (solo) {
            __syncthreads();
            if (j >= A.k) break;
            continue;
        }
        if (bi == 0 && tid == 0) A.j_out[kk] = j;
        grid_barrier(A.bar);
        if (tid == 0) {
            int done = 1;
            for (int q = 0; q < K; ++q) done &= (((volatile int64_t*)A.j_out)[q] >= A.k);
            s_all_done = done;
        }
        __syncthreads();
        if (s_all_done) break;
    }
    if (bi == 0 && tid == 0) A.j_out[kk] = j;
}

// ---------------------------------------------------- small trees (C1)
// A tree whose per-vertex state fits in one CTA's shared memory (n of a few
// thousand, e.g. the MST of config C1 with 228 levels) is swept by ONE CTA per
// threshold with every array staged in shared memory: a level costs a few
// __syncthreads and shared-memory latencies instead of two grid barriers and
// dependent global loads.  Same arithmetic, canonical order, k-th-cut stop
// and fold order as decide_kernel (which is this with G = 1).
constexpr int DS_THREADS = 512;   // staging threads; warp 0 sweeps

size_t decide_small_smem(int64_t n, int64_t levels) {
    // f, om0, p0, om, p (8 B) + child_lo, child_cnt, excl (4 B) + code (1 B) + level_off
    return (size_t)n * (5 * 8 + 3 * 4 + 1) + (size_t)(levels + 1) * 8 + 64;
}

struct DecideSmallArgs {
    int64_t n;
    int64_t levels;
    const int64_t* level_off;
    const double* f_pos;
    const double* om0;
    const double* p0;
    const int32_t* child_lo;
    const int32_t* child_cnt;
    const double* thr;   // K thresholds (device) -- one CTA each
    int64_t k;
    int8_t* code;        // witness (K == 1): per-position codes, else nullptr
    double* spars;       // witness: k sparsities in cut order, else nullptr
    int64_t* j_out;      // [K]
};

__global__ void __launch_bounds__(DS_THREADS, 1) decide_small_kernel(DecideSmallArgs A) {
    // one warp per threshold: MST levels are narrow (median width 6-71 at
    // C1), so a level is a few shuffles and __syncwarp()s.  The CTA has
    // DS_STAGE threads: all of them stage the tree into shared memory (the
    // global loads overlap), then warp 0 alone sweeps.
    extern __shared__ __align__(16) unsigned char ds_raw[];
    const int lane = threadIdx.x;
    const int nst = blockDim.x;
    const int64_t n = A.n, L = A.levels;
    double* f = reinterpret_cast<double*>(ds_raw);
    double* om0 = f + n;
    double* p0 = om0 + n;
    double* om = p0 + n;
    double* pp = om + n;
    int64_t* loff = reinterpret_cast<int64_t*>(pp + n);
    int32_t* clo = reinterpret_cast<int32_t*>(loff + L + 1);
    int32_t* ccnt = clo + n;
    int32_t* excl = ccnt + n;
    int8_t* code = reinterpret_cast<int8_t*>(excl + n);
    for (int64_t q = lane; q < n; q += nst) {
        f[q] = A.f_pos[q];
        om0[q] = A.om0[q];
        p0[q] = A.p0[q];
        clo[q] = A.child_lo[q];
        ccnt[q] = A.child_cnt[q];
        code[q] = 0;
    }
    for (int64_t q = lane; q <= L; q += nst) loff[q] = A.level_off[q];
    __syncthreads();
    if (lane >= 32) return;
    const double thr = A.thr[blockIdx.x];
    const bool witness = A.code != nullptr;
    int64_t j = 0, stop_lo = 0;
    for (int64_t lv = L - 1; lv >= 0; --lv) {
        const int64_t lo = loff[lv], hi = loff[lv + 1];
        const bool deepest = lv == L - 1;
        const double* pv = deepest ? p0 : pp;
        const double* ov = deepest ? om0 : om;
        const int64_t W = hi - lo;
        // conditions and the exclusive cut prefix in canonical (descending
        // position) order over the whole level
        int32_t carry = 0;
        for (int64_t base = 0; base < W; base += 32) {
            const int64_t c = base + lane;
            int32_t is_cut = 0;
            if (c < W) {
                const int64_t pos = hi - 1 - c;
                const double rhs = __dmul_rn(thr, ov[pos]);
                int8_t cond;
                if (__dadd_rn(f[pos], pv[pos]) <= rhs) cond = 1;
                else if (__dsub_rn(pv[pos], f[pos]) < rhs) cond = 2;
                else cond = 3;
                code[pos] = cond;
                is_cut = cond == 1;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, is_cut);
            if (c < W) excl[hi - 1 - c] = carry + __popc(bal & ((1u << lane) - 1u));
            carry += __popc(bal);
        }
        __syncwarp();
        const int64_t need = A.k - j;
        const int64_t tot = carry;
        if (lv > 0) {
            // one lane per parent folds its children in descending child
            // rank, committing each (fewer than need cuts precede it)
            const int64_t plo = loff[lv - 1];
            for (int64_t u = plo + lane; u < lo; u += 32) {
                const int32_t c0 = clo[u], cn = ccnt[u];
                double pu = p0[u], ou = om0[u];
                for (int32_t q = c0 + cn - 1; q >= c0; --q) {
                    int8_t d = code[q];
                    const int64_t e = excl[q];
                    if (e < need) {
                        if (d == 1 && witness) A.spars[j + e] = __ddiv_rn(__dadd_rn(f[q], pv[q]), ov[q]);
                    } else {
                        code[q] = 0;
                        d = 0;
                    }
                    if (d == 1 || d == 3) {
                        pu = __dadd_rn(pu, f[q]);
                    } else if (d == 2) {
                        ou = __dadd_rn(ou, ov[q]);
                        pu = __dadd_rn(pu, pv[q]);
                    }
                }
                pp[u] = pu;
                om[u] = ou;
            }
        } else {
            for (int64_t c = lane; c < W; c += 32) {
                const int64_t pos = hi - 1 - c;
                const int64_t e = excl[pos];
                if (e < need) {
                    if (code[pos] == 1 && witness) A.spars[j + e] = __ddiv_rn(__dadd_rn(f[pos], pv[pos]), ov[pos]);
                } else {
                    code[pos] = 0;
                }
            }
        }
        j += (tot < need) ? tot : need;
        __syncwarp();
        if (j >= A.k) { stop_lo = lo; break; }
    }
    if (witness) {
        for (int64_t q = lane; q < n; q += 32) A.code[q] = q < stop_lo ? 0 : code[q];
    }
    if (lane == 0) A.j_out[blockIdx.x] = j;
}

bool decide_small_fits(int64_t n, int64_t levels, size_t* smem) {
    *smem = decide_small_smem(n, levels);
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return *smem <= (size_t)optin;
}

// Resident 512-thread CTAs per SM of the cooperative sweep kernels, queried
// once per device (slot 0: decide_kernel, 1: decide_batch_kernel).
static int resident_per_sm(const void* kern, int slot) {
    static int cache[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev][slot] == 0) {
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 512, 0);
        cache[dev][slot] = per_sm > 0 ? per_sm : 1;
    }
    return cache[dev][slot];
}

static cudaError_t launch_decide_small(int64_t n, int64_t levels, const int64_t* level_off, const double* f_pos,
                                       const double* om0, const double* p0, const int32_t* child_lo,
                                       const int32_t* child_cnt, const double* thr, int K, int64_t k,
                                       int8_t* code, double* spars, int64_t* j_out, size_t smem,
                                       cudaStream_t st) {
    cudaError_t e = ensure_max_dyn_smem((const void*)decide_small_kernel, (size_t)((int)smem));
    if (e != cudaSuccess) return e;
    DecideSmallArgs A;
    A.n = n; A.levels = levels; A.level_off = level_off; A.f_pos = f_pos; A.om0 = om0; A.p0 = p0;
    A.child_lo = child_lo; A.child_cnt = child_cnt; A.thr = thr; A.k = k; A.code = code; A.spars = spars;
    A.j_out = j_out;
    const int pid = prof_begin(PK_DECIDE, st);
    decide_small_kernel<<<K, DS_THREADS, smem, st>>>(A);
    prof_end(pid, st);
    note_launch();
    return cudaGetLastError();
}

int decide_grid_size(int64_t max_width);

cudaError_t launch_decide_batch(int64_t n, int64_t levels, const int64_t* level_off, int64_t max_width,
                                const double* f_pos, const double* om0, const double* p0,
                                const int32_t* child_lo, const int32_t* child_cnt, const double* thr,
                                int K, int64_t k, double* om, double* p, int8_t* code, int32_t* excl,
                                int32_t* scratch, int64_t* j_out, cudaStream_t st) {
    size_t smem = 0;
    if (decide_small_fits(n, levels, &smem))
        return launch_decide_small(n, levels, level_off, f_pos, om0, p0, child_lo, child_cnt, thr, K, k,
                                   nullptr, nullptr, j_out, smem, st);
    const int64_t cap = (int64_t)device_sm_count() * resident_per_sm((const void*)decide_batch_kernel, 1);
    int64_t gi = (max_width + 8191) / 8192;
    if (gi < 1) gi = 1;
    if (gi * K > cap) gi = cap / K > 0 ? cap / K : 1;
    const int G = (int)(gi * K);
    DecideBatchArgs A;
    A.n = n; A.levels = levels; A.level_off = level_off; A.f_pos = f_pos; A.om0 = om0; A.p0 = p0;
    A.child_lo = child_lo; A.child_cnt = child_cnt; A.thr = thr; A.K = K; A.k = k; A.om = om; A.p = p;
    A.code = code; A.excl = excl; A.chunk_cnt = scratch; A.j_out = j_out;
    A.bar = reinterpret_cast<unsigned int*>(scratch + DB_MAX * 1024);
    cudaMemsetAsync(A.bar, 0, 2 * sizeof(unsigned int), st);
    cudaMemsetAsync(j_out, 0, (size_t)K * sizeof(int64_t), st);
    void* args[] = {&A};
    const int pid = prof_begin(PK_DECIDE, st);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)decide_batch_kernel, dim3(G), dim3(512), args, 0, st);
    prof_end(pid, st);
    note_launch();
    return e;
}

int decide_grid_size(int64_t max_width) {
    int64_t want = (max_width + 8191) / 8192;
    int64_t cap = (int64_t)device_sm_count() * resident_per_sm((const void*)decide_kernel, 0);
    if (cap > DK_MAXG) cap = DK_MAXG;
    if (want < 1) want = 1;
    return (int)(want < cap ? want : cap);
}

cudaError_t launch_decide(int64_t n, int64_t levels, const int64_t* level_off, int64_t max_width,
                          const double* f_pos, const double* om0, const double* p0,
                          const int32_t* child_lo, const int32_t* child_cnt, double thr, int64_t k,
                          double* om, double* p, int8_t* code, int32_t* excl, double* spars,
                          int32_t* scratch, int64_t* j_out, cudaStream_t st) {
    size_t smem = 0;
    if (decide_small_fits(n, levels, &smem)) {
        // the threshold goes to the device through the scratch tail
        double* dthr = reinterpret_cast<double*>(scratch + 1024 + 16);
        cudaMemcpyAsync(dthr, &thr, sizeof(double), cudaMemcpyHostToDevice, st);
        return launch_decide_small(n, levels, level_off, f_pos, om0, p0, child_lo, child_cnt, dthr, 1, k, code,
                                   spars, j_out, smem, st);
    }
    const int G = decide_grid_size(max_width);
    DecideArgs A;
    A.n = n; A.levels = levels; A.level_off = level_off; A.f_pos = f_pos; A.om0 = om0; A.p0 = p0;
    A.child_lo = child_lo; A.child_cnt = child_cnt; A.thr = thr; A.k = k; A.om = om; A.p = p;
    A.code = code; A.excl = excl; A.spars = spars; A.chunk_cnt = scratch; A.j_out = j_out;
    A.bar = reinterpret_cast<unsigned int*>(scratch + 1024);
    cudaMemsetAsync(A.bar, 0, 2 * sizeof(unsigned int), st);
    void* args[] = {&A};
    const int pid = prof_begin(PK_DECIDE, st);
    cudaError_t e = cudaLaunchCooperativeKernel((void*)decide_kernel, dim3(G), dim3(512), args, 0, st);
    prof_end(pid, st);
    note_launch();
    return e;
}

// ----------------------------------------------------------------- labels
__global__ void rep_init_kernel(const int8_t* __restrict__ code, const int32_t* __restrict__ pos_parent,
                                int64_t n, int32_t* __restrict__ rep) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    rep[q] = code[q] == 2 ? pos_parent[q] : (int32_t)q;
}

__global__ void rep_jump_kernel(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    out[q] = in[in[q]];
}

__global__ void cut_vertex_kernel(const int8_t* __restrict__ code, const int32_t* __restrict__ bfs,
                                  int64_t n, int8_t* __restrict__ cut_v, int32_t* __restrict__ cut_i) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int32_t v = bfs[q];
    const int8_t c = code[q] == 1;
    cut_v[v] = c;
    cut_i[v] = c;
}

__global__ void labels_kernel(const int32_t* __restrict__ rep, const int8_t* __restrict__ code,
                              const int32_t* __restrict__ bfs, const int32_t* __restrict__ scan,
                              int64_t n, int64_t* __restrict__ eta, int64_t* __restrict__ labels,
                              int32_t* __restrict__ lab32) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int32_t v = bfs[q];
    const int32_t r = rep[q];
    if (code[r] == 1) {
        const int32_t rv = bfs[r];
        eta[v] = rv;
        labels[v] = 1 + scan[rv];
        lab32[v] = 1 + scan[rv];
    } else {
        eta[v] = ISOC_NO_VERTEX;
        labels[v] = 0;
        lab32[v] = 0;
    }
}

cudaError_t launch_labels(const int8_t* code, const int32_t* pos_parent, const int32_t* bfs,
                          int64_t n, int64_t levels, int8_t* cut_v, int64_t* eta, int64_t* labels,
                          int32_t* lab32, int32_t* work, cudaStream_t st) {
    // work: rep[n], rep2[n], cut_i[n], scan[n]
    int32_t* rep = work;
    int32_t* rep2 = work + n;
    int32_t* cut_i = work + 2 * n;
    int32_t* scan = work + 3 * n;
    rep_init_kernel<<<nb(n, 256), 256, 0, st>>>(code, pos_parent, n, rep);
    int passes = 0;
    while ((int64_t(1) << passes) < levels + 1) ++passes;
    for (int i = 0; i < passes; ++i) {
        rep_jump_kernel<<<nb(n, 256), 256, 0, st>>>(rep, n, rep2);
        int32_t* t = rep; rep = rep2; rep2 = t;
    }
    cut_vertex_kernel<<<nb(n, 256), 256, 0, st>>>(code, bfs, n, cut_v, cut_i);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cut_i, scan, (int)n, st);
    void* tmp = nullptr;
    cudaError_t e = isoc_malloc_async(&tmp, tb, st);
    if (e != cudaSuccess) return e;
    cub::DeviceScan::ExclusiveSum(tmp, tb, cut_i, scan, (int)n, st);
    isoc_free_async(tmp, st);
    labels_kernel<<<nb(n, 256), 256, 0, st>>>(rep, code, bfs, scan, n, eta, labels, lab32);
    note_launch(passes + 3);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- cost
// keys (cluster << 32 | index) for member and crossing-edge entries;
// cluster k+1 marks "no entry".
__global__ void cost_keys_kernel(const int32_t* __restrict__ lab, const int32_t* __restrict__ parent_v,
                                 const double* __restrict__ flow, const double* __restrict__ omega,
                                 const double* __restrict__ p, int64_t n, int64_t k,
                                 unsigned long long* __restrict__ mkeys, int32_t* __restrict__ mvals,
                                 unsigned long long* __restrict__ bkeys, double* __restrict__ bvals) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const uint64_t none = (uint64_t)(k + 1) << 32;
    const int32_t lu = lab[u];
    mkeys[u] = lu >= 1 ? (((uint64_t)lu << 32) | (uint64_t)u) : (none | (uint64_t)u);
    mvals[u] = (int32_t)u;
    const int32_t pu = parent_v[u];
    uint64_t ka = none | (uint64_t)u, kb = none | (uint64_t)u;
    if (pu >= 0) {
        const int32_t lp = lab[pu];
        if (lu != lp) {
            if (lu >= 1) ka = ((uint64_t)lu << 32) | (uint64_t)u;
            if (lp >= 1) kb = ((uint64_t)lp << 32) | (uint64_t)u;
        }
    }
    bkeys[u] = ka;
    bkeys[n + u] = kb;
    const double f = pu >= 0 ? flow[u] : 0.0;
    bvals[u] = f;
    bvals[n + u] = f;
}

// first sorted index of each cluster c in [1, k+1]
__global__ void segment_bounds_kernel(const unsigned long long* __restrict__ keys, int64_t m,
                                      int64_t k, int64_t* __restrict__ seg) {
    const int64_t c = 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c > k + 1) return;
    const unsigned long long target = (unsigned long long)c << 32;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    seg[c - 1] = lo;
}

// slot s of a segment's depth-T grid: the pairwise-recursion node reached by
// the T path bits of s; a leaf met earlier is owned by the slot whose
// remaining bits are zero, others are empty.
template <typename Get>
__device__ double slot_value(Get get, int64_t m, int T, int64_t s, bool& empty) {
    int64_t start = 0, len = m;
    for (int t = 0; t < T; ++t) {
        if (len <= 128) {
            const int64_t rest = s & ((int64_t(1) << (T - t)) - 1);
            if (rest != 0) { empty = true; return 0.0; }
            break;
        }
        const int64_t n2 = np_split(len);
        if ((s >> (T - 1 - t)) & 1) { start += n2; len -= n2; } else { len = n2; }
    }
    empty = false;
    if (len > 128) return np_pairwise_small([&](int64_t i) { return get(start + i); }, len);
    return np_leaf_sum([&](int64_t i) { return get(start + i); }, len);
}

__host__ __device__ __forceinline__ int seg_depth(int64_t m) {
    int T = 0;
    while ((m >> T) > 64) ++T;
    return T;
}


// Per (cluster, quantity) segment: 0 = boundary flows, 1 = potentials,
// 2 = masses.  A segment of m values is the numpy pairwise recursion cut at
// depth T (seg_depth): S = 2^T slots (slot_value), folded pairwise back up.
// The slots are split into aligned blocks of SEG_B (one CTA each, so a
// cluster holding most of the tree no longer runs on one CTA); each block
// folds to the value of its subtree node, and one CTA per segment folds the
// block values.  Same binary tree, same additions: bitwise the single-CTA
// fold.
constexpr int SEG_B = 2048;

// slot blocks over all segments: 2^T <= max(1, 2m/64) slots per segment,
// segment lengths total at most 2n (boundary) + n + n (members twice), one
// block per SEG_B slots or per nonempty segment
static inline int64_t cost_block_bound(int64_t n, int64_t k) { return (4 * n / 32) / SEG_B + 3 * k + 1; }

// seg_blocks: per segment the number of slot blocks (0 for an empty one);
// blk_off: their exclusive prefix, blk_off[3k] = total.
__global__ void slot_offsets_kernel(const int64_t* __restrict__ bseg, const int64_t* __restrict__ mseg,
                                    int64_t k, int64_t* __restrict__ blk_off) {
    int64_t acc = 0;
    for (int64_t q = 0; q < 3 * k; ++q) {
        const int64_t c = q / 3;
        const int64_t* seg = (q % 3) == 0 ? bseg : mseg;
        const int64_t m = seg[c + 1] - seg[c];
        blk_off[q] = acc;
        if (m > 0) {
            const int64_t S = int64_t(1) << seg_depth(m);
            acc += S > SEG_B ? S / SEG_B : 1;
        }
    }
    blk_off[3 * k] = acc;
}

// In-shared-memory pairwise fold of w (a power of two) slot values; an
// empty right child passes the left value through (the leaf above it IS the
// node); a node is empty iff its left child is.  Returns the root.
__device__ double fold_slots(double* v0, double* v1, uint8_t* e0, uint8_t* e1, int w, bool& empty) {
    for (; w > 1; w >>= 1) {
        for (int i = threadIdx.x; i < w / 2; i += blockDim.x) {
            const double l = v0[2 * i], r = v0[2 * i + 1];
            v1[i] = e0[2 * i + 1] ? l : __dadd_rn(l, r);
            e1[i] = e0[2 * i];
        }
        __syncthreads();
        double* tv = v0; v0 = v1; v1 = tv;
        uint8_t* te = e0; e0 = e1; e1 = te;
    }
    empty = e0[0];
    const double r = v0[0];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(256) segment_part_kernel(const double* __restrict__ bvals_sorted,
                                                           const int32_t* __restrict__ mvals_sorted,
                                                           const double* __restrict__ omega,
                                                           const double* __restrict__ p,
                                                           const int64_t* __restrict__ bseg,
                                                           const int64_t* __restrict__ mseg, int64_t k,
                                                           const int64_t* __restrict__ blk_off,
                                                           double* __restrict__ part, uint8_t* __restrict__ pempty) {
    __shared__ double v[2][SEG_B];
    __shared__ uint8_t e[2][SEG_B];
    const int64_t g = blockIdx.x;
    const int64_t nseg = 3 * k;
    if (g >= blk_off[nseg]) return;
    int64_t lo = 0, hi = nseg;   // last q with blk_off[q] <= g (empty segments own no block)
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (blk_off[mid] <= g) lo = mid; else hi = mid;
    }
    const int64_t q = lo, c = q / 3;
    const int what = (int)(q % 3);
    const int64_t* seg = what == 0 ? bseg : mseg;
    const int64_t a = seg[c], m = seg[c + 1] - seg[c];
    const int T = seg_depth(m);
    const int64_t S = int64_t(1) << T;
    const int B = S > SEG_B ? SEG_B : (int)S;
    const int64_t s0 = (g - blk_off[q]) * B;
    auto get = [&](int64_t i) -> double {
        if (what == 0) return bvals_sorted[a + i];
        const int32_t x = mvals_sorted[a + i];
        return what == 1 ? p[x] : omega[x];
    };
    for (int s = threadIdx.x; s < B; s += blockDim.x) {
        bool em = false;
        v[0][s] = slot_value(get, m, T, s0 + s, em);
        e[0][s] = em;
    }
    __syncthreads();
    bool em;
    const double r = fold_slots(v[0], v[1], e[0], e[1], B, em);
    if (threadIdx.x == 0) {
        part[g] = r;
        pempty[g] = em;
    }
}

__global__ void __launch_bounds__(256) segment_sum_kernel(const int64_t* __restrict__ blk_off,
                                                          const double* __restrict__ part,
                                                          const uint8_t* __restrict__ pempty,
                                                          double* __restrict__ sums) {
    __shared__ double v[2][SEG_B];
    __shared__ uint8_t e[2][SEG_B];
    __shared__ double cv[2][64];
    __shared__ uint8_t ce[2][64];
    const int64_t q = blockIdx.x;
    const int64_t b0 = blk_off[q], nb = blk_off[q + 1] - b0;   // a power of two (or 0)
    if (nb == 0) {
        if (threadIdx.x == 0) sums[q] = 0.0;
        return;
    }
    const int C = nb > SEG_B ? SEG_B : (int)nb;
    const int chunks = (int)(nb / C);   // <= 64 for n < 2^32 (m < 2^33, S <= 2^28)
    for (int ch = 0; ch < chunks; ++ch) {
        for (int s = threadIdx.x; s < C; s += blockDim.x) {
            v[0][s] = part[b0 + (int64_t)ch * C + s];
            e[0][s] = pempty[b0 + (int64_t)ch * C + s];
        }
        __syncthreads();
        bool em;
        const double r = fold_slots(v[0], v[1], e[0], e[1], C, em);
        if (threadIdx.x == 0) {
            cv[0][ch] = r;
            ce[0][ch] = em;
        }
    }
    __syncthreads();
    bool em;
    const double r = fold_slots(cv[0], cv[1], ce[0], ce[1], chunks, em);
    if (threadIdx.x == 0) sums[q] = __dadd_rn(0.0, r);
}

__global__ void miso_kernel(const double* __restrict__ sums, int64_t k, double* __restrict__ out) {
    double worst = -INFINITY;
    for (int64_t c = 0; c < k; ++c) {
        const double s = __ddiv_rn(__dadd_rn(sums[3 * c + 0], sums[3 * c + 1]), sums[3 * c + 2]);
        worst = fmax(worst, s);
    }
    *out = worst;
}

cudaError_t launch_cost(const int32_t* lab32, const int32_t* parent_v, const double* flow,
                        const double* omega, const double* p, int64_t n, int64_t k,
                        void* work, size_t work_bytes, double* sums, double* miso, cudaStream_t st) {
    // work layout
    char* w = reinterpret_cast<char*>(work);
    auto take = [&](size_t bytes) { char* r = w; w += (bytes + 255) & ~size_t(255); return r; };
    unsigned long long* mkeys = (unsigned long long*)take(8 * n);
    unsigned long long* mkeys_s = (unsigned long long*)take(8 * n);
    int32_t* mvals = (int32_t*)take(4 * n);
    int32_t* mvals_s = (int32_t*)take(4 * n);
    unsigned long long* bkeys = (unsigned long long*)take(16 * n);
    unsigned long long* bkeys_s = (unsigned long long*)take(16 * n);
    double* bvals = (double*)take(16 * n);
    double* bvals_s = (double*)take(16 * n);
    int64_t* mseg = (int64_t*)take(8 * (k + 2));
    int64_t* bseg = (int64_t*)take(8 * (k + 2));
    int64_t* blk_off = (int64_t*)take(8 * (3 * k + 1));
    const int64_t nblk = cost_block_bound(n, k);
    double* part = (double*)take(8 * nblk);
    uint8_t* pempty = (uint8_t*)take(nblk);
    if ((size_t)(w - reinterpret_cast<char*>(work)) > work_bytes) return cudaErrorInvalidValue;

    cost_keys_kernel<<<nb(n, 256), 256, 0, st>>>(lab32, parent_v, flow, omega, p, n, k, mkeys, mvals,
                                                  bkeys, bvals);
    int bits = 32;
    while ((int64_t(1) << (bits - 32)) <= k + 1) ++bits;
    size_t tb1 = 0, tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb1, mkeys, mkeys_s, mvals, mvals_s, (int)n, 0, bits, st);
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, bkeys, bkeys_s, bvals, bvals_s, (int)(2 * n), 0, bits,
                                    st);
    void* tmp = nullptr;
    cudaError_t e = isoc_malloc_async(&tmp, tb1 > tb2 ? tb1 : tb2, st);
    if (e != cudaSuccess) return e;
    cub::DeviceRadixSort::SortPairs(tmp, tb1, mkeys, mkeys_s, mvals, mvals_s, (int)n, 0, bits, st);
    cub::DeviceRadixSort::SortPairs(tmp, tb2, bkeys, bkeys_s, bvals, bvals_s, (int)(2 * n), 0, bits, st);
    isoc_free_async(tmp, st);
    segment_bounds_kernel<<<nb(k + 1, 128), 128, 0, st>>>(mkeys_s, n, k, mseg);
    segment_bounds_kernel<<<nb(k + 1, 128), 128, 0, st>>>(bkeys_s, 2 * n, k, bseg);
    slot_offsets_kernel<<<1, 1, 0, st>>>(bseg, mseg, k, blk_off);
    segment_part_kernel<<<(unsigned)nblk, 256, 0, st>>>(bvals_s, mvals_s, omega, p, bseg, mseg, k, blk_off,
                                                        part, pempty);
    segment_sum_kernel<<<(unsigned)(3 * k), 256, 0, st>>>(blk_off, part, pempty, sums);
    miso_kernel<<<1, 1, 0, st>>>(sums, k, miso);
    note_launch(7);
    return cudaGetLastError();
}

size_t cost_work_bytes(int64_t n, int64_t k) {
    const int64_t nblk = cost_block_bound(n, k);
    size_t b = 0;
    auto add = [&](size_t bytes) { b += (bytes + 255) & ~size_t(255); };
    add(8 * n); add(8 * n); add(4 * n); add(4 * n); add(16 * n); add(16 * n); add(16 * n); add(16 * n);
    add(8 * (k + 2)); add(8 * (k + 2)); add(8 * (3 * k + 1)); add(8 * nblk); add(nblk);
    return b;
}

}  // namespace isoc
