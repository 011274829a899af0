/*
 * isoc_fast.c -- full-size CPU oracle kernels (N up to ~1M points).
 *
 * TEST INFRASTRUCTURE ONLY (same rules as isoc_oracle.c): nothing in the
 * product package links, loads or calls this file.
 *
 * The scalar oracle (isoc_oracle.c) restates the reference pair by pair; at
 * C3 (N = 1e6, d = 64) its Prim alone would stream X once per step (~256 TB).
 * This file computes the same numbers with the same per-pair operation order,
 * vectorised ACROSS pairs (each SIMD lane is one pair; inside a lane the
 * d-term sum is the scipy order s = s + t*t, separately rounded:
 * -ffp-contract=off):
 *
 *   ocf_flat_distance_sum  float(dist.sum())  affinity.py:237, numpy
 *       pairwise recursion over the flat n*n buffer.  The
 *       recursion is split into OpenMP tasks; a task whose range is <= TASK
 *       elements materialises that range (row-blocked, cache-tiled) and runs
 *       the same recursion on it, so the combination tree is unchanged.
 *   ocf_omega_knn  vertex_weights  affinity.py:175-201 (+ pairwise_row_sums
 *       _primitives.py:162-175): per row, the zero-padded pow2 adjacent fold
 *       of exp((-d)/sigma) with the diagonal 0.  The fold is an aligned binary
 *       tree, so 256-column block subtrees fold while the block is in cache.
 *       Also keeps each row's K lexicographically smallest (d, j), j != i.
 *   ocf_boruvka  the MST edge set of prim_mst (mst.py:128-181) through a
 *       uniqueness certificate: in every Boruvka round each component's
 *       minimum outgoing edge is found EXACTLY (kNN lists where they decide
 *       it, an exact rescan of the row otherwise) and checked to be the only
 *       outgoing edge of that weight.  A strictly lightest edge across a cut
 *       lies in every MST, so if every round certifies, the MST is unique
 *       and equals Prim's tree edge for edge, whatever Prim's tie rules.  If
 *       any component minimum is tied the call reports it (no certificate)
 *       and the caller must fall back to the scalar Prim (oc_prim).
 *   Rooting (parent, child_id = rank of (d(p,u), u) among p's children,
 *       SURVEY A.5, BFS order) is done by ocf_root_tree.
 *
 * Compiled twice (x86-64-v4 and x86-64-v3) by oracle/Makefile; the exported
 * entry points dispatch on __builtin_cpu_supports at run time.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#include "exp_table.h"

#ifndef OCF_SUFFIX
#define OCF_SUFFIX _generic
#endif
#define OCF_CAT2(a, b) a##b
#define OCF_CAT(a, b) OCF_CAT2(a, b)
#define OCF(name) OCF_CAT(name, OCF_SUFFIX)

typedef double v8d __attribute__((vector_size(64), aligned(8)));

#define CB 256        /* column block (XT block 256 x d doubles stays in L2) */
#define RB 64         /* rows sharing one XT block */
#define TASK (1LL << 26) /* flat elements materialised per sigma task */

double oc_exp(double x); /* scalar restatement (isoc_oracle.c), used for special lanes */

/* ------------------------------------------------------------ distances */
/* out[c] = d(xi, column j0+c) for c in [0, CB).  XT holds X block-transposed:
 * column block b (columns [b*CB, (b+1)*CB), zero padded past n) is one
 * contiguous d x CB panel, so a block's 2 KB-per-k rows never alias in the
 * caches the way a d x n transpose with a power-of-two stride does. */
static inline void dist_block(const double *xi, const double *XT, int64_t ld, int64_t j0, int d,
                              double *out)
{
    (void)ld;
    const double *panel = XT + j0 * (int64_t)d; /* = (j0/CB) * d * CB */
    for (int c = 0; c < CB; c += 32) {
        v8d s0 = {0}, s1 = {0}, s2 = {0}, s3 = {0};
        const double *p = panel + c;
        for (int k = 0; k < d; k++, p += CB) {
            const double a = xi[k];
            v8d t0 = a - *(const v8d *)(p + 0);
            v8d t1 = a - *(const v8d *)(p + 8);
            v8d t2 = a - *(const v8d *)(p + 16);
            v8d t3 = a - *(const v8d *)(p + 24);
            s0 = s0 + t0 * t0;
            s1 = s1 + t1 * t1;
            s2 = s2 + t2 * t2;
            s3 = s3 + t3 * t3;
        }
        *(v8d *)(out + c + 0) = s0;
        *(v8d *)(out + c + 8) = s1;
        *(v8d *)(out + c + 16) = s2;
        *(v8d *)(out + c + 24) = s3;
    }
    for (int c = 0; c < CB; c++) out[c] = __builtin_sqrt(out[c]);
}

/* ------------------------------------------------- numpy pairwise sum */
static double pw_leaf(const double *a, int64_t n)
{
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    }
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
}

static double pw_rec(const double *a, int64_t n)
{
    if (n <= 128) return pw_leaf(a, n);
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pw_rec(a, n2) + pw_rec(a + n2, n - n2);
}

typedef struct {
    const double *X, *XT;
    int64_t n, ld;
    int d;
    double **bufs; /* one TASK-sized buffer per thread */
} flat_ctx;

/* materialise flat range [s, s+len) of the row-major distance matrix */
static void fill_range(const flat_ctx *c, int64_t s, int64_t len, double *buf)
{
    const int64_t n = c->n;
    const int64_t r0 = s / n, r1 = (s + len - 1) / n;
    double tile[CB] __attribute__((aligned(64)));
    for (int64_t rb = r0; rb <= r1; rb += RB) {
        const int64_t re = rb + RB - 1 < r1 ? rb + RB - 1 : r1;
        for (int64_t j0 = 0; j0 < n; j0 += CB) {
            for (int64_t r = rb; r <= re; r++) {
                int64_t lo = r * n + j0, hi = lo + CB;
                if (hi > (r + 1) * n) hi = (r + 1) * n;
                if (lo < s) lo = s;
                if (hi > s + len) hi = s + len;
                if (lo >= hi) continue;
                dist_block(c->X + r * c->d, c->XT, c->ld, j0, c->d, tile);
                memcpy(buf + (lo - s), tile + (lo - r * n - j0), (size_t)(hi - lo) * sizeof(double));
            }
        }
    }
}

static double flat_rec(const flat_ctx *c, int64_t start, int64_t len)
{
    if (len <= TASK) {
        double *buf = c->bufs[omp_get_thread_num()];
        fill_range(c, start, len, buf);
        return pw_rec(buf, len);
    }
    /* len > TASK > 128: the split is pw_rec's */
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    double a, b;
#pragma omp task shared(a) firstprivate(c, start, n2)
    a = flat_rec(c, start, n2);
#pragma omp task shared(b) firstprivate(c, start, n2, len)
    b = flat_rec(c, start + n2, len - n2);
#pragma omp taskwait
    return a + b;
}

static double *make_xt(const double *X, int64_t n, int d, int64_t *ld_out)
{
    int64_t ld = (n + CB - 1) / CB * CB;
    double *XT = (double *)aligned_alloc(64, (size_t)(ld * d) * sizeof(double));
    if (!XT) return NULL;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < ld / CB; b++)
        for (int k = 0; k < d; k++)
            for (int c = 0; c < CB; c++) {
                const int64_t j = b * CB + c;
                XT[(b * d + k) * CB + c] = j < n ? X[j * d + k] : 0.0;
            }
    *ld_out = ld;
    return XT;
}

/* float(d.sum()) over the implicit n x n distance matrix; NAN on OOM */
double OCF(ocf_flat_distance_sum)(const double *X, int64_t n, int d)
{
    int64_t ld;
    double *XT = make_xt(X, n, d, &ld);
    if (!XT) return NAN;
    int nt = omp_get_max_threads();
    double **bufs = (double **)calloc((size_t)nt, sizeof(double *));
    int64_t blen = n * n < TASK ? n * n : TASK;
    int ok = 1;
    for (int t = 0; t < nt; t++) {
        bufs[t] = (double *)malloc((size_t)blen * sizeof(double));
        if (!bufs[t]) ok = 0;
    }
    double out = NAN;
    if (ok) {
        flat_ctx c = {X, XT, n, ld, d, bufs};
#pragma omp parallel
#pragma omp single
        out = flat_rec(&c, 0, n * n);
        out = 0.0 + out;
    }
    for (int t = 0; t < nt; t++) free(bufs[t]);
    free(bufs);
    free(XT);
    return out;
}

/* ------------------------------------------------------------------ exp */
/* Vector form of oc_exp's main path (glibc 2.39 exp, FMA variant; see
 * isoc_oracle.c); lanes outside the main-path range are recomputed by the
 * scalar oc_exp, so every lane equals oc_exp bitwise. */
static const double E_INVLN2N = 0x1.71547652b82fep0 * 128.0;
static const double E_SHIFT = 0x1.8p52;
static const double E_NEGLN2HIN = -0x1.62e42fefa0000p-8;
static const double E_NEGLN2LON = -0x1.cf79abc9e3b3ap-47;
static const double E_C2 = 0x1.ffffffffffdbdp-2;
static const double E_C3 = 0x1.555555555543cp-3;
static const double E_C4 = 0x1.55555cf172b91p-5;
static const double E_C5 = 0x1.1111167a4d017p-7;

static void flows_block(const double *dist, double *out, int len, double sigma)
{
    int special = 0;
    for (int l = 0; l < len; l++) {
        double x = (-dist[l]) / sigma;
        uint64_t xb;
        memcpy(&xb, &x, 8);
        uint32_t abstop = (uint32_t)(xb >> 52) & 0x7ff;
        special |= (abstop - 0x3c9u >= 0x408u - 0x3c9u);
        double kd = fma(x, E_INVLN2N, E_SHIFT);
        uint64_t ki;
        memcpy(&ki, &kd, 8);
        kd -= E_SHIFT;
        double r = fma(kd, E_NEGLN2LON, fma(kd, E_NEGLN2HIN, x));
        uint64_t idx = 2 * (ki % 128);
        uint64_t top = ki << 45;
        double tail;
        memcpy(&tail, &ISOC_EXP_TAB[idx], 8);
        uint64_t sbits = ISOC_EXP_TAB[idx + 1] + top;
        double r2 = r * r;
        double tmp = fma(r2 * r2, fma(r, E_C5, E_C4), fma(fma(r, E_C3, E_C2), r2, tail + r));
        double scale;
        memcpy(&scale, &sbits, 8);
        out[l] = fma(scale, tmp, scale);
    }
    if (special) {
        for (int l = 0; l < len; l++) {
            double x = (-dist[l]) / sigma;
            uint64_t xb;
            memcpy(&xb, &x, 8);
            uint32_t abstop = (uint32_t)(xb >> 52) & 0x7ff;
            if (abstop - 0x3c9u >= 0x408u - 0x3c9u) out[l] = oc_exp(x);
        }
    }
}

/* -------------------------------------------------- omega + kNN pass */
static inline void knn_insert(double *kd, int64_t *kj, int K, double v, int64_t j)
{
    /* list sorted by (d, j); j arrives in increasing order, so an equal d
       never displaces an earlier entry */
    int p = K - 1;
    if (!(v < kd[p])) return;
    while (p > 0 && v < kd[p - 1]) {
        kd[p] = kd[p - 1];
        kj[p] = kj[p - 1];
        p--;
    }
    kd[p] = v;
    kj[p] = j;
}

/* omega[i] for i in [lo, hi) (vertex_weights, affinity.py:175-201, diagonal
 * zero before the fold) and the K nearest (d, j != i) of every row.
 * knn_d/knn_j: (hi-lo) x K, unused slots (n-1 < K) hold +inf / -1. */
int OCF(ocf_omega_knn)(const double *X, int64_t n, int d, double sigma, int64_t lo, int64_t hi,
                       int K, double *omega, double *knn_d, int64_t *knn_j)
{
    int64_t ld;
    double *XT = make_xt(X, n, d, &ld);
    if (!XT) return 4;
    int64_t size = 1;
    while (size < n) size <<= 1;
    const int64_t nblk = (size + CB - 1) / CB; /* CB-wide aligned subtrees */
    int err = 0;
#pragma omp parallel
    {
        double *bsum = (double *)malloc((size_t)(RB * (nblk > 1 ? nblk : 1)) * sizeof(double));
        double tile[CB] __attribute__((aligned(64)));
        double fl[CB] __attribute__((aligned(64)));
        if (!bsum) {
#pragma omp atomic write
            err = 4;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t rb = lo; rb < hi; rb += RB) {
            if (err) continue;
            const int64_t re = rb + RB < hi ? rb + RB : hi;
            for (int64_t r = rb; r < re; r++)
                for (int q = 0; q < K; q++) {
                    knn_d[(r - lo) * K + q] = INFINITY;
                    knn_j[(r - lo) * K + q] = -1;
                }
            for (int64_t b = 0; b < nblk; b++) {
                const int64_t j0 = b * CB;
                for (int64_t r = rb; r < re; r++) {
                    double *bs = bsum + (r - rb) * nblk;
                    if (j0 >= n) { bs[b] = 0.0; continue; }
                    dist_block(X + r * d, XT, ld, j0, d, tile);
                    int cnt = n - j0 < CB ? (int)(n - j0) : CB;
                    flows_block(tile, fl, cnt, sigma);
                    for (int c = cnt; c < CB; c++) fl[c] = 0.0;
                    if (r >= j0 && r < j0 + cnt) fl[r - j0] = 0.0;
                    /* kNN: vector-friendly threshold test, scalar insert */
                    double *kd = knn_d + (r - lo) * K;
                    int64_t *kj = knn_j + (r - lo) * K;
                    double thr = kd[K - 1];
                    double mn = tile[0];
                    for (int c = 1; c < cnt; c++) mn = tile[c] < mn ? tile[c] : mn;
                    for (int c = 0; c < cnt && mn < thr; c++) {
                        if (tile[c] < thr && j0 + c != r) {
                            knn_insert(kd, kj, K, tile[c], j0 + c);
                            thr = kd[K - 1];
                        }
                    }
                    /* aligned pow2 fold of the block (a subtree of the row fold) */
                    for (int w = CB; w > 1; w >>= 1)
                        for (int c = 0; c < w / 2; c++) fl[c] = fl[2 * c] + fl[2 * c + 1];
                    bs[b] = fl[0];
                }
            }
            for (int64_t r = rb; r < re; r++) {
                double *bs = bsum + (r - rb) * nblk;
                int64_t w = nblk;
                if (size < CB) {
                    /* n < CB: the block fold above already folded size..CB zeros;
                       the zero padding beyond size adds exact zeros */
                    omega[r - lo] = bs[0];
                    continue;
                }
                while (w > 1) {
                    for (int64_t c = 0; c < w / 2; c++) bs[c] = bs[2 * c] + bs[2 * c + 1];
                    w >>= 1;
                }
                omega[r - lo] = bs[0];
            }
        }
        free(bsum);
    }
    free(XT);
    return err;
}

/* --------------------------------------------- exact external rescan */
/* For each listed row r (component comp[r]): its K lexicographically smallest
 * (d, j) over j with comp[j] != comp[r], written over the row's kNN slots
 * (rows[q]'s list at knn_d/knn_j + q*K).  Unused slots: +inf / -1. */
int OCF(ocf_rescan_rows)(const double *X, int64_t n, int d, const int64_t *rows, int64_t nrows,
                         const int32_t *comp, int K, double *knn_d, int64_t *knn_j)
{
    int64_t ld;
    double *XT = make_xt(X, n, d, &ld);
    if (!XT) return 4;
#pragma omp parallel
    {
        double tile[CB] __attribute__((aligned(64)));
#pragma omp for schedule(dynamic, 1)
        for (int64_t q0 = 0; q0 < nrows; q0 += RB) {
            const int64_t q1 = q0 + RB < nrows ? q0 + RB : nrows;
            for (int64_t q = q0; q < q1; q++)
                for (int t = 0; t < K; t++) { knn_d[q * K + t] = INFINITY; knn_j[q * K + t] = -1; }
            for (int64_t j0 = 0; j0 < n; j0 += CB) {
                const int cnt = n - j0 < CB ? (int)(n - j0) : CB;
                for (int64_t q = q0; q < q1; q++) {
                    const int64_t r = rows[q];
                    const int32_t cr = comp[r];
                    double *kd = knn_d + q * K;
                    int64_t *kj = knn_j + q * K;
                    double thr = kd[K - 1];
                    dist_block(X + r * d, XT, ld, j0, d, tile);
                    double mn = tile[0];
                    for (int c = 1; c < cnt; c++) mn = tile[c] < mn ? tile[c] : mn;
                    if (!(mn < thr)) continue;
                    for (int c = 0; c < cnt; c++) {
                        if (tile[c] < thr && comp[j0 + c] != cr) {
                            knn_insert(kd, kj, K, tile[c], j0 + c);
                            thr = kd[K - 1];
                        }
                    }
                }
            }
        }
    }
    free(XT);
    return 0;
}
