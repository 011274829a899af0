// K2s: symmetric omega pass with Boruvka round 2 fused (single GPU).
//
// Each unordered pair is computed once: CTA (I, J), I <= J, owns the
// 1024 x 1024 super-tile of super-blocks I (rows) and J (columns).  Two
// ping-pong teams of 256 threads each take 512 of the columns and walk their
// 8 x 8 tiles of 128 x 64; their tile epilogues strictly alternate (named
// barriers), so one team's FP64 loop always covers the other's epilogue.  From every tile of flows
// f_ij = exp(-d_ij/sigma) (diagonal zeroed, vertex_weights,
// /root/reference/pkg/src/isoclust/affinity.py:175-201) it folds
//   rows i in I over the tile's columns  -> pow2 subtree sums, level 6, and
//   columns j in J over the tile's rows  -> the transposed sums (d_ji == d_ij
//                                           bitwise: scipy squares u-v)
// and pushes them through per-row / per-column binary counters into complete
// 1024-wide subtrees PS[J][i] and PS[I][j].  omega_finish folds PS[.][i] over
// the super-blocks (the top of the same pow2 tree, _primitives.py:162-175).
// With comp != NULL the same tiles give each row's exact minimum
// (d, j) over columns in other components: Boruvka round 2 for free.
#include <cstdint>
#include <type_traits>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#include "common.cuh"
#include "scratch.h"
#include "kernels.h"
#include "prof.h"

namespace isoc {

constexpr int SB = 1024;      // super-block
constexpr int TBM = 128;      // tile rows
constexpr int TBN = 64;       // tile columns
constexpr int SK = 16;        // k chunk
constexpr int TEAM = 256;     // threads per team
constexpr int STH = 2 * TEAM; // two ping-pong teams
constexpr int HALF = SB / 2;  // columns per team

struct SymStage {
    double A[SK][TBM];
    double B[SK][TBN];
};

struct TeamSmem {
    SymStage st[2];
    double rc[TBM][4];         // row counters over the team's 8 column tiles
    double cc[HALF][4];        // column counters over the 8 row tiles
    double xcol[8][TBN];       // column partials of the team's eight warps
    double xcm[8][TBN];        // column-min exchange
    int32_t xcj[8][TBN];
    double rmin[TBM];
    int32_t rminj[TBM];
    uint64_t trm[4][TEAM];     // per-thread running row minima over the column tiles
    int32_t trj[4][TEAM];
    double cmin[HALF];
    int32_t cminj[HALF];
    int32_t comp_r[TBM];       // component ids of the tile's rows / columns
    int32_t comp_c[TBN];
};

struct SymSmem {
    TeamSmem t[2];
    double rowv[TBM];          // team 0's 512-column row subtrees / minima of the row tile
    double rowm[TBM];
    int32_t rowj[TBM];
    uint64_t exp_tab[256];     // exp table in shared memory (lane-divergent lookups)
};

__device__ __forceinline__ void sym_cp16(void* dst, const void* src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}

__device__ __forceinline__ void sym_load(SymStage& s, const double* __restrict__ XT, int64_t np,
                                         int64_t r0, int64_t c0, int kc, int ttid) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int q = ttid + TEAM * m;           // 0..1023 chunks of 16 B (A)
        const int kk = q >> 6, part = q & 63;
        sym_cp16(&s.A[kk][part * 2], XT + (int64_t)(kc * SK + kk) * np + r0 + part * 2);
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        const int q = ttid + TEAM * m;           // 0..511 chunks of 16 B (B)
        const int kk = q >> 5, part = q & 31;
        sym_cp16(&s.B[kk][part * 2], XT + (int64_t)(kc * SK + kk) * np + c0 + part * 2);
    }
}

// Slot of the 1024-wide subtree of row i over super-block b.
//
// One GPU: [b][i].
//
// Sharded (G ranks; rank r owns rows [n*r/G, n*(r+1)/G) and evaluates the
// super-tiles (I, J), I <= J, J in its block range [jlo_r, jhi_r)): the
// producer of slot (b, i) is the rank whose range holds max(b, B_i), B_i =
// i / SB.  For a row in block B, rank s produces the contiguous block range
//   b in [jlo_s, jhi_s)   when B <  jlo_s   (row role of its tiles)
//   b in [0, jhi_s)       when B in [jlo_s, jhi_s) (column role below, row role from B)
//   nothing               when B >= jhi_s.
// The message s -> g holds exactly those slots for g's rows, row by row, so
// every rank sends only what it produced (n * nbs slots over the whole job,
// ~n * nbs / G per rank) -- an all-to-all with per-peer split sizes.  The
// plan (host-built, uploaded per call) holds, for every (s, g), the offset
// of the first row of g in block B within the message, and the send /
// receive displacements:
//   P[0, G) jlo, P[G, 2G) jhi, T[(s*G + g)*(nbs+1) + B], MC[s*G + g] (slots),
//   SD[s*G + g] (send displacement of s's message to g),
//   RD[g*G + s] (receive displacement of s's message at g).
struct OmegaPlanView {
    const int64_t* P;
    int G;
    int64_t n, nbs;
    __host__ __device__ const int64_t* T() const { return P + 2 * G; }
    __host__ __device__ const int64_t* MC() const { return P + 2 * G + (int64_t)G * G * (nbs + 1); }
    __host__ __device__ const int64_t* SD() const { return MC() + G * G; }
    __host__ __device__ const int64_t* RD() const { return SD() + G * G; }
    // offset of slot (b, i) within the message s -> g (s produces it)
    __host__ __device__ int64_t msg_off(int s, int g, int64_t i, int64_t b) const {
        const int64_t B = i / SB, jlo = P[s], jhi = P[G + s];
        const int64_t cnt = B < jlo ? jhi - jlo : (B < jhi ? jhi : 0);
        const int64_t bst = B < jlo ? jlo : 0;
        const int64_t lo_g = n * g / G;
        const int64_t r0 = lo_g > B * SB ? lo_g : B * SB;
        return T()[((int64_t)s * G + g) * (nbs + 1) + B] + (i - r0) * cnt + (b - bst);
    }
    __host__ __device__ int owner(int64_t i) const {
        int64_t r = i * G / n;
        while (n * (r + 1) / G <= i) ++r;
        while (n * r / G > i) --r;
        return (int)r;
    }
    __host__ __device__ int producer(int64_t b, int64_t B) const {
        const int64_t m = b > B ? b : B;
        for (int s = 0; s < G; ++s)
            if (m >= P[s] && m < P[G + s]) return s;
        return -1;
    }
};

__device__ __forceinline__ int64_t ps_slot(int64_t b, int64_t i, int64_t n, const OmegaPlanView& pv, int rank) {
    if (pv.P == nullptr) return b * n + i;
    const int g = pv.owner(i);
    return pv.SD()[rank * pv.G + g] + pv.msg_off(rank, g, i, b);
}

// Round-2 minima carry an exact-tie flag in the sign bit of the column
// index: (m, jt) with jt = j | TIEBIT when the minimum value m was attained
// by two different columns (each (row, column) pair is evaluated exactly once
// over the pass, so two equal candidates are two edges).  Boruvka's
// comp_tie_kernel turns the flag into an exact_ties count, which makes the
// pipeline replay Prim's tie rule (mst.py:153-166, _primitives.py:69-92).
constexpr int32_t TIEBIT = (int32_t)0x80000000u;
__device__ __forceinline__ int32_t jof(int32_t jt) { return jt & 0x7fffffff; }

__device__ __forceinline__ void tie_merge(double& m, int32_t& mjt, double x, int32_t xjt) {
    if (x < m) {
        m = x;
        mjt = xjt;
    } else if (x == m && x < INFINITY) {
        mjt = min(jof(mjt), jof(xjt)) | TIEBIT;
    }
}
// the same on the distance bit patterns (d >= 0 orders like its bits)
__device__ __forceinline__ void tie_merge_bits(uint64_t& m, int32_t& mjt, uint64_t x, int32_t xjt) {
    if (x < m) {
        m = x;
        mjt = xjt;
    } else if (x == m && x < 0x7ff0000000000000ull) {
        mjt = min(jof(mjt), jof(xjt)) | TIEBIT;
    }
}

__device__ __forceinline__ double csum_push(double* slots, int idx, double v) {
    // binary counter over the tiles; returns the value stored (the full
    // subtree after the last push)
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

__device__ __forceinline__ void team_sync(int team) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + team), "n"(TEAM) : "memory");
}
// epilogue tokens: team 0 waits on barrier 3, team 1 on barrier 4
__device__ __forceinline__ void token_wait(int team) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(3 + team), "n"(STH) : "memory");
}
__device__ __forceinline__ void token_pass(int team) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(4 - team), "n"(STH) : "memory");
}

__global__ void __launch_bounds__(STH, 1)
omega_sym_kernel(const double* __restrict__ XT, int64_t np, int dpad, int64_t n, int64_t nbs,
                 double sigma, double rs, const int32_t* __restrict__ comp, double* __restrict__ PS,
                 double* __restrict__ PSm, int32_t* __restrict__ PSj, int64_t b0, OmegaPlanView pv, int rank) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SymSmem& sm = *reinterpret_cast<SymSmem*>(smem_raw);
    const int tid = threadIdx.x;
    const int team = tid >> 8, ttid = tid & (TEAM - 1);
    TeamSmem& ts = sm.t[team];
    const int lane = tid & 31, w = ttid >> 5;
    const int rg = ttid >> 3, cl = lane & 7;
    // thread columns (within the tile): 2*cl + 16*q + h, q < 4, h < 2 -> the 8
    // lanes of a row group read 8 consecutive 16-byte chunks (no bank
    // conflicts); thread rows: 4*rg + i, i < 4
    // triangular decode of blockIdx -> (I, J), I <= J
    const int64_t b = b0 + blockIdx.x;
    int64_t J = (int64_t)((sqrt(8.0 * (double)b + 1.0) - 1.0) / 2.0);
    while ((J + 1) * (J + 2) / 2 <= b) ++J;
    while (J * (J + 1) / 2 > b) --J;
    const int64_t I = b - J * (J + 1) / 2;
    const bool diag = (I == J);
    const int64_t R0 = I * SB, C0 = J * SB + team * HALF;   // this team's columns
    const int nk = dpad / SK;
    const bool want_min = comp != nullptr;
    constexpr int TI = SB / TBM, TJ = HALF / TBN;   // 8 x 8 tiles per team

    for (int e = ttid; e < HALF; e += TEAM) {
        ts.cmin[e] = INFINITY;
        ts.cminj[e] = INT32_MAX;
    }
    for (int e = tid; e < 256; e += STH) sm.exp_tab[e] = ISOC_EXP_TAB[e];
    __syncthreads();
    if (team == 1) token_pass(team);     // team 0 takes the first epilogue
    double acc[4][8];
    int32_t compv = 0;
    // linear pipeline over (ti, tj, kc)
    const int total = TI * TJ * nk;
    sym_load(ts.st[0], XT, np, R0, C0, 0, ttid);
    asm volatile("cp.async.commit_group;\n" ::);
    int kc = 0, tile = 0;
    for (int it = 0; it < total; ++it) {
        const int ti = tile / TJ, tj = tile % TJ;
        if (kc == 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
            if (want_min && ttid < TBM + TBN) {
                const int64_t g = (ttid < TBM) ? R0 + ti * TBM + ttid : C0 + tj * TBN + (ttid - TBM);
                compv = g < n ? comp[g] : (ttid < TBM ? -1 : -2);
            }
        }
        // chunk it's copies (the only group in flight) land; after the team
        // barrier every thread has also left chunk it-1, so its buffer takes
        // chunk it+1's copies while chunk it computes (one barrier per chunk)
        asm volatile("cp.async.wait_group 0;\n" ::);
        team_sync(team);
        if (it + 1 < total) {
            const int k1 = (kc + 1 == nk) ? 0 : kc + 1;
            const int t1 = (kc + 1 == nk) ? tile + 1 : tile;
            sym_load(ts.st[(it + 1) & 1], XT, np, R0 + (t1 / TJ) * TBM, C0 + (t1 % TJ) * TBN, k1, ttid);
        }
        asm volatile("cp.async.commit_group;\n" ::);
        // the tile's component ids go to shared memory only now: every thread
        // of the team has left the previous tile's epilogue (which reads them;
        // a diagonal tile's epilogue ends without a team barrier)
        if (kc == 0 && want_min && ttid < TBM + TBN) {
            if (ttid < TBM) ts.comp_r[ttid] = compv; else ts.comp_c[ttid - TBM] = compv;
        }
        {
            const SymStage& s = ts.st[it & 1];
#pragma unroll 16
            for (int kk = 0; kk < SK; ++kk) {
                const double2 a01 = *reinterpret_cast<const double2*>(&s.A[kk][rg * 4]);
                const double2 a23 = *reinterpret_cast<const double2*>(&s.A[kk][rg * 4 + 2]);
                const double a[4] = {a01.x, a01.y, a23.x, a23.y};
                double bv[8];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double2 t = *reinterpret_cast<const double2*>(&s.B[kk][2 * cl + 16 * q]);
                    bv[2 * q] = t.x;
                    bv[2 * q + 1] = t.y;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = exact_sq_step(acc[i][j], a[i], bv[j]);
            }
        }
        if (++kc != nk) continue;
        kc = 0;
        ++tile;

        // ------------------------------------------------ tile epilogue
        // (the two teams' epilogues alternate; the other team's FP64 loop
        // runs meanwhile)
        token_wait(team);
        const int64_t gr0 = R0 + ti * TBM + rg * 4;    // first global row of this thread
        const int64_t gcb = C0 + tj * TBN;              // first global col of the tile
#define LCOL(j) (2 * cl + 16 * ((j) >> 1) + ((j) & 1))
        // validity with 32-bit compares: thread rows i < rlim, tile columns
        // LCOL(j) < clim, off the diagonal (dd + i != LCOL(j))
        const int rlim = (int)(n - gr0 < 0 ? 0 : (n - gr0 > 4 ? 4 : n - gr0));
        const int clim = (int)(n - gcb < 0 ? 0 : (n - gcb > TBN ? TBN : n - gcb));
        const int64_t dd64 = gr0 - gcb;
        const int dd = (int)(dd64 < -TBN - 8 ? -TBN - 8 : (dd64 > TBN + 8 ? TBN + 8 : dd64));
        {
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) ok = ok && sqrt_fast_ok(acc[i][j]);
            if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = isoc_sqrt_fast(acc[i][j]);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = __dsqrt_rn(acc[i][j]);
            }
        }
        // Inner patches (warp-uniform): every element is a real off-diagonal
        // pair, so the minima and flows below skip the per-element masks.
        const bool inner = __all_sync(0xffffffffu, rlim == 4 && clim == TBN && (dd64 <= -4 || dd64 >= TBN));
        auto mins_flows = [&](auto chk) {
            constexpr bool CHK = decltype(chk)::value;
            if (want_min) {
                // row minima over the tile's 64 columns (ascending within the
                // thread, so a strict compare keeps the smaller column); d >= 0,
                // so the bit patterns order like the values
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int32_t cr = ts.comp_r[rg * 4 + i];
                    uint64_t m = 0x7ff0000000000000ull;
                    int32_t mj = INT32_MAX;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const bool ok = (!CHK || (i < rlim && LCOL(j) < clim)) && ts.comp_c[LCOL(j)] != cr;
                        const uint64_t bv = (uint64_t)__double_as_longlong(acc[i][j]);
                        // columns ascend within the thread: an equal value is a tie
                        // with the (smaller) column already held
                        if (ok && bv < m) { m = bv; mj = (int32_t)(gcb + LCOL(j)); }
                        else if (ok && bv == m) mj |= TIEBIT;
                    }
                    // the thread's running minimum over the team's column tiles;
                    // one merge across the row's 8 lanes after the last tile
                    // (the merge is associative: min value, min column, tie
                    // flag iff the minimum occurs twice)
                    if (tj > 0) tie_merge_bits(m, mj, ts.trm[i][ttid], ts.trj[i][ttid]);
                    if (tj + 1 < TJ) {
                        ts.trm[i][ttid] = m;
                        ts.trj[i][ttid] = mj;
                    } else {
#pragma unroll
                        for (int off = 1; off < 8; off <<= 1) {
                            const uint64_t om = (uint64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off);
                            const int32_t oj = __shfl_xor_sync(0xffffffffu, mj, off);
                            tie_merge_bits(m, mj, om, oj);
                        }
                        if (cl == 0) {
                            const int r = rg * 4 + i;
                            ts.rmin[r] = __longlong_as_double((long long)m);
                            ts.rminj[r] = mj;
                        }
                    }
                }
                // column minima over the thread's rows (ascending), then the warp
                if (!diag) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int32_t cc = ts.comp_c[LCOL(j)];
                        uint64_t m = 0x7ff0000000000000ull;
                        int32_t mj = INT32_MAX;
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const bool ok = (!CHK || (i < rlim && LCOL(j) < clim)) && ts.comp_r[rg * 4 + i] != cc;
                            const uint64_t bv = (uint64_t)__double_as_longlong(acc[i][j]);
                            if (ok && bv < m) { m = bv; mj = (int32_t)(gr0 + i); }
                            else if (ok && bv == m) mj |= TIEBIT;
                        }
#pragma unroll
                        for (int off = 8; off < 32; off <<= 1) {
                            const uint64_t om = (uint64_t)__shfl_xor_sync(0xffffffffu, (long long)m, off);
                            const int32_t oj = __shfl_xor_sync(0xffffffffu, mj, off);
                            tie_merge_bits(m, mj, om, oj);
                        }
                        if ((lane >> 3) == 0) {
                            ts.xcm[w][LCOL(j)] = __longlong_as_double((long long)m);
                            ts.xcj[w][LCOL(j)] = mj;
                        }
                    }
                }
            }
            // flows in place (diagonal and padding -> 0): x = (-d)/sigma for the
            // batch, one vote, then the branch-free exp or the table exp
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double x = isoc_div_rs(-acc[i][j], sigma, rs);
                    const bool valid = !CHK || (i < rlim && LCOL(j) < clim && dd + i != LCOL(j));
                    ok = ok && (!valid || exp_fast_ok(x));
                    acc[i][j] = valid ? x : 0.0;
                }
            if (__all_sync(0xffffffffu, ok)) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const double f = isoc_exp_fast(acc[i][j], sm.exp_tab);
                        if (CHK) {
                            const bool valid = i < rlim && LCOL(j) < clim && dd + i != LCOL(j);
                            acc[i][j] = valid ? f : 0.0;
                        } else {
                            acc[i][j] = f;
                        }
                    }
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const bool valid = !CHK || (i < rlim && LCOL(j) < clim && dd + i != LCOL(j));
                        acc[i][j] = valid ? isoc_exp(acc[i][j], sm.exp_tab) : 0.0;
                    }
            }
        };
        if (inner) mins_flows(std::false_type{});
        else mins_flows(std::true_type{});
        // row folds (pow2 tree over the tile's 64 columns): own pairs (level
        // 1), lanes cl^1, cl^2, cl^4 (levels 2-4, one 16-column block per q),
        // own q pairs (levels 5-6); 8 tiles -> the team's 512-column subtree;
        // team 1 adds team 0's (left) subtree: the row's 1024-wide subtree
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
            if (cl == 0) {
                const int r = rg * 4 + i;
                const double half = csum_push(ts.rc[r], tj, __dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3])));
                if (tj == TJ - 1) {
                    if (team == 0) {
                        sm.rowv[r] = half;
                        if (want_min) { sm.rowm[r] = ts.rmin[r]; sm.rowj[r] = ts.rminj[r]; }
                    } else {
                        const int64_t gi = R0 + ti * TBM + r;
                        if (gi < n) {
                            const int64_t o = ps_slot(J, gi, n, pv, rank);
                            PS[o] = __dadd_rn(sm.rowv[r], half);
                            if (want_min) {
                                double m = sm.rowm[r];
                                int32_t mj = sm.rowj[r];
                                tie_merge(m, mj, ts.rmin[r], ts.rminj[r]);
                                PSm[o] = m;
                                PSj[o] = mj;
                            }
                        }
                    }
                }
            }
        }
        // column folds: 4 own rows, then the 4 row groups of the warp, then
        // the team's 8 warps through shared memory
        if (!diag) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                double x = __dadd_rn(__dadd_rn(acc[0][j], acc[1][j]), __dadd_rn(acc[2][j], acc[3][j]));
                double y = __shfl_down_sync(0xffffffffu, x, 8);
                if (((lane >> 3) & 1) == 0) x = __dadd_rn(x, y);
                y = __shfl_down_sync(0xffffffffu, x, 16);
                if ((lane >> 3) == 0) ts.xcol[w][LCOL(j)] = __dadd_rn(x, y);
            }
            team_sync(team);
            if (ttid < TBN) {
                const int c = ttid;
                const double x01 = __dadd_rn(ts.xcol[0][c], ts.xcol[1][c]);
                const double x23 = __dadd_rn(ts.xcol[2][c], ts.xcol[3][c]);
                const double x45 = __dadd_rn(ts.xcol[4][c], ts.xcol[5][c]);
                const double x67 = __dadd_rn(ts.xcol[6][c], ts.xcol[7][c]);
                const int col = tj * TBN + c;
                csum_push(ts.cc[col], ti, __dadd_rn(__dadd_rn(x01, x23), __dadd_rn(x45, x67)));
                if (want_min) {
                    double m = ts.cmin[col];
                    int32_t mj = ts.cminj[col];
                    for (int h = 0; h < 8; ++h) tie_merge(m, mj, ts.xcm[h][c], ts.xcj[h][c]);
                    ts.cmin[col] = m;
                    ts.cminj[col] = mj;
                }
            }
            team_sync(team);
        }
        token_pass(team);
#undef LCOL
    }
    if (team == 0) token_wait(team);     // consume team 1's final hand-over
    if (!diag) {
        for (int c = ttid; c < HALF; c += TEAM) {
            const int64_t gj = C0 + c;
            if (gj < n) {
                const int64_t o = ps_slot(I, gj, n, pv, rank);
                PS[o] = ts.cc[c][3];   // counter slot of the 8th row tile
                if (want_min) { PSm[o] = ts.cmin[c]; PSj[o] = ts.cminj[c]; }
            }
        }
    }
}

// omega[i] = pow2 fold of the row's complete 1024-wide subtrees over the
// super-blocks (zero padded); round-2 minimum over the blocks (ties ->
// smaller column, flagged).  One GPU (pv.P == nullptr): slot (b, i) at
// b * n + i.  Sharded: this owner's rows [row_lo, row_lo + rows), slot (b, i)
// read from its producer's message in the received buffer.
__global__ void omega_finish_kernel(const double* __restrict__ PS, const double* __restrict__ PSm,
                                    const int32_t* __restrict__ PSj, int64_t row_lo, int64_t rows, int64_t n,
                                    int64_t nbs, OmegaPlanView pv, int rank, double* __restrict__ omega,
                                    int32_t* __restrict__ nn_j, double* __restrict__ nn_d,
                                    int8_t* __restrict__ nn_tie) {
    const int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= rows) return;
    const int64_t i = row_lo + li;
    const int64_t B = i / SB;
    double slots[40];
    double m = INFINITY;
    int32_t mj = INT32_MAX;
    for (int64_t b = 0; b < nbs; ++b) {
        int64_t o;
        if (pv.P == nullptr) {
            o = b * n + i;
        } else {
            const int s = pv.producer(b, B);
            o = pv.RD()[rank * pv.G + s] + pv.msg_off(s, rank, i, b);
        }
        double v = PS[o];
        int lvl = 0;
        int64_t t = b;
        while (t & 1) {
            v = __dadd_rn(slots[lvl], v);
            t >>= 1;
            ++lvl;
        }
        slots[lvl] = v;
        if (PSm) tie_merge(m, mj, PSm[o], PSj[o]);
    }
    double acc = 0.0;
    bool have = false;
    for (int lvl = 0; lvl < 40 && (nbs >> lvl) != 0; ++lvl)
        if ((nbs >> lvl) & 1) {
            acc = have ? __dadd_rn(slots[lvl], acc) : slots[lvl];
            have = true;
        }
    omega[li] = acc;
    if (PSm) {
        nn_j[li] = jof(mj) == INT32_MAX ? -1 : jof(mj);
        nn_d[li] = m;
        nn_tie[li] = (int8_t)((mj & TIEBIT) != 0);
    }
}

size_t omega_sym_smem() { return sizeof(SymSmem); }

// Host-built plan of the sharded pass (layout: OmegaPlanView).
void omega_plan_build(int64_t n, int G, std::vector<int64_t>& P) {
    const int64_t nbs = (n + SB - 1) / SB;
    const int64_t nT = (int64_t)G * G * (nbs + 1);
    P.assign((size_t)(2 * G + nT + 3 * G * G), 0);
    for (int s = 0; s < G; ++s) sym_block_range(n, s, G, &P[s], &P[G + s], SB);
    int64_t* T = P.data() + 2 * G;
    int64_t* MC = T + nT;
    int64_t* SD = MC + G * G;
    int64_t* RD = SD + G * G;
    for (int s = 0; s < G; ++s) {
        const int64_t jlo = P[s], jhi = P[G + s];
        for (int g = 0; g < G; ++g) {
            const int64_t lo_g = n * g / G, hi_g = n * (g + 1) / G;
            int64_t acc = 0;
            for (int64_t B = 0; B <= nbs; ++B) {
                T[((int64_t)s * G + g) * (nbs + 1) + B] = acc;
                if (B == nbs) break;
                const int64_t a = std::max(lo_g, B * SB), e = std::min(hi_g, (B + 1) * SB);
                const int64_t rows = e > a ? e - a : 0;
                const int64_t cnt = B < jlo ? jhi - jlo : (B < jhi ? jhi : 0);
                acc += rows * cnt;
            }
            MC[s * G + g] = acc;
        }
    }
    for (int s = 0; s < G; ++s) {
        int64_t a = 0;
        for (int g = 0; g < G; ++g) { SD[s * G + g] = a; a += MC[s * G + g]; }
    }
    for (int g = 0; g < G; ++g) {
        int64_t a = 0;
        for (int s = 0; s < G; ++s) { RD[g * G + s] = a; a += MC[s * G + g]; }
    }
}

void omega_shard_counts(int64_t n, int G, int rank, int64_t* send, int64_t* recv) {
    std::vector<int64_t> P;
    omega_plan_build(n, G, P);
    const int64_t nbs = (n + SB - 1) / SB;
    const int64_t* MC = P.data() + 2 * G + (int64_t)G * G * (nbs + 1);
    for (int g = 0; g < G; ++g) {
        send[g] = MC[rank * G + g];
        recv[g] = MC[g * G + rank];
    }
}

static cudaError_t upload_plan(int64_t n, int G, Scratch& sc, OmegaPlanView* pv, cudaStream_t st) {
    std::vector<int64_t> P;
    omega_plan_build(n, G, P);
    int64_t* dP = nullptr;
    cudaError_t e = sc.alloc(&dP, P.size());
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(dP, P.data(), P.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    pv->P = dP;
    pv->G = G;
    pv->n = n;
    pv->nbs = (n + SB - 1) / SB;
    // the host vector must outlive the copy
    return cudaStreamSynchronize(st);
}

// Super-tiles (I, J), I <= J, J in [jlo, jhi) into the slot buffers (layout
// of ps_slot).
static cudaError_t omega_sym_tiles(const double* X, int64_t n, int d, double sigma, const int32_t* comp,
                                   int64_t jlo, int64_t jhi, const OmegaPlanView& pv, int rank, double* PS,
                                   double* PSm, int32_t* PSj, cudaStream_t st) {
    const int64_t nbs = (n + SB - 1) / SB;
    const int64_t np = nbs * SB;
    const int dpad = (d + SK - 1) / SK * SK;
    Scratch sc(st);
    double* XT = nullptr;
    cudaError_t e = sc.alloc(&XT, (size_t)np * dpad);
    if (e != cudaSuccess) return e;
    e = launch_transpose_pad(X, n, d, np, dpad, XT, st);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(SymSmem);
    e = ensure_max_dyn_smem((const void*)omega_sym_kernel, (size_t)((int)smem));
    if (e != cudaSuccess) return e;
    const int64_t b0 = jlo * (jlo + 1) / 2;
    const int64_t ctas = jhi * (jhi + 1) / 2 - b0;
    if (ctas > 0) {
        const int pid = prof_begin(PK_OMEGA, st);
        omega_sym_kernel<<<(unsigned)ctas, STH, smem, st>>>(XT, np, dpad, n, nbs, sigma, 1.0 / sigma, comp,
                                                            PS, PSm, PSj, b0, pv, rank);
        prof_end(pid, st);
        note_launch(1);
    }
    return cudaGetLastError();
}

cudaError_t launch_omega_sym(const double* X, int64_t n, int d, double sigma, const int32_t* comp,
                             double* omega, int32_t* nn_j, double* nn_d, int8_t* nn_tie,
                             cudaStream_t st) {
    const int64_t nbs = (n + SB - 1) / SB;
    Scratch sc(st);   // PS / PSm / PSj freed on every return path
    double *PS = nullptr, *PSm = nullptr;
    int32_t* PSj = nullptr;
    cudaError_t e = sc.alloc(&PS, (size_t)nbs * n);
    if (e != cudaSuccess) return e;
    if (comp) {
        e = sc.alloc(&PSm, (size_t)nbs * n);
        if (e != cudaSuccess) return e;
        e = sc.alloc(&PSj, (size_t)nbs * n);
        if (e != cudaSuccess) return e;
    }
    const OmegaPlanView one{nullptr, 1, n, nbs};
    e = omega_sym_tiles(X, n, d, sigma, comp, 0, nbs, one, 0, PS, PSm, PSj, st);
    if (e != cudaSuccess) return e;
    omega_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(PS, PSm, PSj, 0, n, n, nbs, one, 0, omega,
                                                                     nn_j, nn_d, nn_tie);
    note_launch(1);
    return cudaGetLastError();
}

cudaError_t launch_omega_sym_range(const double* X, int64_t n, int d, double sigma, const int32_t* comp,
                                   int rank, int G, double* PS, double* PSm, int32_t* PSj, cudaStream_t st) {
    Scratch sc(st);
    OmegaPlanView pv;
    cudaError_t e = upload_plan(n, G, sc, &pv, st);
    if (e != cudaSuccess) return e;
    int64_t jlo, jhi;
    sym_block_range(n, rank, G, &jlo, &jhi, SB);
    return omega_sym_tiles(X, n, d, sigma, comp, jlo, jhi, pv, rank, PS, comp ? PSm : nullptr,
                           comp ? PSj : nullptr, st);
}

cudaError_t launch_omega_rank_merge(int64_t n, int rank, int G, const double* PS, const double* PSm,
                                    const int32_t* PSj, double* omega, int32_t* nn_j, double* nn_d,
                                    int8_t* nn_tie, cudaStream_t st) {
    Scratch sc(st);
    OmegaPlanView pv;
    cudaError_t e = upload_plan(n, G, sc, &pv, st);
    if (e != cudaSuccess) return e;
    const int64_t lo = n * rank / G, hi = n * (rank + 1) / G;
    const int64_t rows = hi - lo;
    if (rows <= 0) return cudaSuccess;
    omega_finish_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(PS, PSm, PSj, lo, rows, n, pv.nbs, pv,
                                                                        rank, omega, nn_j, nn_d, nn_tie);
    note_launch(1);
    return cudaGetLastError();
}

}  // namespace isoc
