/*
 * isoc_oracle.c -- CPU restatement of the reference clustering path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs do, and only as the checker or as the
 * timed CPU baseline.
 *
 * Every function restates one reference function (paths relative to
 * /root/reference/pkg/src/isoclust/) with the same floating-point operation
 * order, so results are bitwise comparable:
 *   distances      affinity.py:124-158 via scipy 1.18.1 cdist/pdist
 *                  (s = 0; s = s + t*t sequentially, t = u-v; sqrt(s))
 *   flat d.sum()   affinity.py:233-241 -> numpy pairwise_sum over the n*n
 *                  row-major buffer (leaves <= 128, 8 accumulators)
 *   row folds      affinity.py:175-230 + _primitives.py:162-175 (pow2 fold)
 *   exp            numpy exp in pinned mode == glibc 2.39 exp (FMA variant),
 *                  restated from the published table-driven algorithm
 *   prim           mst.py:128-181 (+ min_reduce _primitives.py:69-92)
 *   bfs / tree     mst.py:46-125
 *   extrema        affinity.py:260-279 (+ sum_reduce/min_reduce)
 *   decide         isoperim.py:82-144, _resolve_groups :147-161
 *   cost           isoperim.py:184-219 (np.sum == pairwise_sum on the
 *                  compacted arrays)
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#include "exp_table.h"

#define NO_VERTEX (-1)

/* ------------------------------------------------------------------ exp */
/* glibc 2.39 exp, FMA ifunc variant (the one selected on x86-64 hosts with
 * FMA/AVX2; numpy's pinned-mode np.exp resolves to it).  Operation order
 * follows the compiled FMA variant: kd = fma(x, InvLn2N, Shift), r via two
 * fmas, tmp = fma(r2*r2, fma(r,C5,C4), fma(fma(r,C3,C2), r2, tail + r)),
 * result = fma(scale, tmp, scale). */
static const double OC_INVLN2N = 0x1.71547652b82fep0 * 128.0;
static const double OC_SHIFT = 0x1.8p52;
static const double OC_NEGLN2HIN = -0x1.62e42fefa0000p-8;
static const double OC_NEGLN2LON = -0x1.cf79abc9e3b3ap-47;
static const double OC_C2 = 0x1.ffffffffffdbdp-2;
static const double OC_C3 = 0x1.555555555543cp-3;
static const double OC_C4 = 0x1.55555cf172b91p-5;
static const double OC_C5 = 0x1.1111167a4d017p-7;

static inline uint64_t asu64(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double asf64(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

static double oc_exp_special(double tmp, uint64_t sbits, uint64_t ki)
{
    double scale, y;
    if ((ki & 0x80000000ull) == 0) {
        sbits -= 1009ull << 52;
        scale = asf64(sbits);
        return 0x1p1009 * fma(scale, tmp, scale);
    }
    /* k < 0 (subnormal range); the compiled variant rounds scale*tmp once
       and reuses it (no fma on this branch) */
    sbits += 1022ull << 52;
    scale = asf64(sbits);
    double st = scale * tmp;
    y = scale + st;
    if (y < 1.0) {
        double hi, lo;
        lo = (scale - y) + st;
        hi = 1.0 + y;
        lo = ((1.0 - hi) + y) + lo;
        y = (hi + lo) - 1.0;
        if (y == 0.0) y = 0.0;
    }
    return 0x1p-1022 * y;
}

double oc_exp(double x)
{
    uint32_t abstop = (uint32_t)(asu64(x) >> 52) & 0x7ff;
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;
        if (abstop >= 0x409u) {
            if (asu64(x) == asu64(-INFINITY)) return 0.0;
            if (abstop >= 0x7ffu) return 1.0 + x;
            return (asu64(x) >> 63) ? 0.0 : INFINITY;
        }
        abstop = 0;
    }
    double kd = fma(x, OC_INVLN2N, OC_SHIFT);
    uint64_t ki = asu64(kd);
    kd -= OC_SHIFT;
    double r = fma(kd, OC_NEGLN2LON, fma(kd, OC_NEGLN2HIN, x));
    uint64_t idx = 2 * (ki % 128);
    uint64_t top = ki << 45;
    double tail = asf64(ISOC_EXP_TAB[idx]);
    uint64_t sbits = ISOC_EXP_TAB[idx + 1] + top;
    double r2 = r * r;
    double tmp = fma(r2 * r2, fma(r, OC_C5, OC_C4), fma(fma(r, OC_C3, OC_C2), r2, tail + r));
    if (abstop == 0) return oc_exp_special(tmp, sbits, ki);
    double scale = asf64(sbits);
    return fma(scale, tmp, scale);
}

void oc_exp_array(const double *x, double *y, int64_t n)
{
    for (int64_t i = 0; i < n; i++) y[i] = oc_exp(x[i]);
}

/* flow(d, sigma) = exp(-d / sigma)  (affinity.py:161-172) */
static inline double oc_flow(double d, double sigma) { return oc_exp((-d) / sigma); }

/* ------------------------------------------------------------ distances */
static inline double oc_dist(const double *a, const double *b, int64_t d)
{
    double s = 0.0;
    for (int64_t k = 0; k < d; k++) {
        double t = a[k] - b[k];
        double t2 = t * t;
        s = s + t2;
    }
    return sqrt(s);
}

double oc_pair_distance(const double *X, int64_t d, int64_t i, int64_t j)
{
    return oc_dist(X + i * d, X + j * d, d);
}

void oc_distance_rows(const double *X, int64_t n, int64_t d, int64_t lo, int64_t hi, double *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = lo; i < hi; i++)
        for (int64_t j = 0; j < n; j++)
            out[(i - lo) * n + j] = oc_dist(X + i * d, X + j * d, d);
}

/* ------------------------------------------------ numpy pairwise_sum */
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

/* np.sum of a contiguous 1-d float64 array */
double oc_pairwise_sum(const double *a, int64_t n) { return 0.0 + pw_rec(a, n); }

/* d.sum() over the implicit n*n distance buffer; leaves computed on the fly */
typedef struct { const double *X; int64_t n, d; } flat_ctx;

static double flat_leaf(const flat_ctx *c, int64_t start, int64_t len)
{
    double buf[128];
    for (int64_t e = 0; e < len; e++) {
        int64_t f = start + e, i = f / c->n, j = f % c->n;
        buf[e] = oc_dist(c->X + i * c->d, c->X + j * c->d, c->d);
    }
    return pw_leaf(buf, len);
}

static double flat_rec(const flat_ctx *c, int64_t start, int64_t len, int depth)
{
    if (len <= 128) return flat_leaf(c, start, len);
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    double a, b;
    if (depth < 10) {
#pragma omp task shared(a) firstprivate(c, start, n2, depth)
        a = flat_rec(c, start, n2, depth + 1);
#pragma omp task shared(b) firstprivate(c, start, n2, len, depth)
        b = flat_rec(c, start + n2, len - n2, depth + 1);
#pragma omp taskwait
    } else {
        a = flat_rec(c, start, n2, depth + 1);
        b = flat_rec(c, start + n2, len - n2, depth + 1);
    }
    return a + b;
}

/* float(d.sum()) for d = distance_matrix(X)  (affinity.py:237) */
double oc_flat_distance_sum(const double *X, int64_t n, int64_t d)
{
    flat_ctx c = {X, n, d};
    double out = 0.0;
#pragma omp parallel
#pragma omp single
    out = flat_rec(&c, 0, n * n, 0);
    return 0.0 + out;
}

/* auto_sigma (affinity.py:233-241); returns <= 0 when all points coincide */
double oc_auto_sigma(const double *X, int64_t n, int64_t d)
{
    double total = oc_flat_distance_sum(X, n, d);
    return total / (double)(n * (n - 1));
}

/* ----------------------------------------------------- pow2 row folds */
static double pow2_fold(double *v, int64_t size)
{
    while (size > 1) {
        for (int64_t i = 0; i < size / 2; i++) v[i] = v[2 * i] + v[2 * i + 1];
        size /= 2;
    }
    return v[0];
}

static int64_t next_pow2(int64_t n)
{
    int64_t s = 1;
    while (s < n) s <<= 1;
    return s;
}

/* vertex_weights (affinity.py:175-201) and potentials (:204-230).
 * omega[i] = fold_j exp(-d_ij/sigma) with the diagonal zeroed;
 * p[i] = alpha * fold_j d_ij (exact zeros when alpha == 0). */
void oc_row_folds(const double *X, int64_t n, int64_t d, double sigma, double alpha,
                  int64_t lo, int64_t hi, double *omega, double *p)
{
    int64_t size = next_pow2(n);
#pragma omp parallel
    {
        double *fb = (double *)calloc((size_t)size, sizeof(double));
        double *db = (double *)calloc((size_t)size, sizeof(double));
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = lo; i < hi; i++) {
            for (int64_t j = 0; j < n; j++) {
                double dij = oc_dist(X + i * d, X + j * d, d);
                fb[j] = (j == i) ? 0.0 : oc_flow(dij, sigma);
                db[j] = dij;
            }
            for (int64_t j = n; j < size; j++) { fb[j] = 0.0; db[j] = 0.0; }
            omega[i - lo] = pow2_fold(fb, size);
            if (alpha == 0.0) p[i - lo] = 0.0;
            else p[i - lo] = alpha * pow2_fold(db, size);
        }
        free(fb);
        free(db);
    }
}

/* sum_reduce (_primitives.py:102-124): zero-padded pow2 adjacent fold */
double oc_sum_reduce(const double *a, int64_t n)
{
    int64_t size = next_pow2(n);
    double *v = (double *)calloc((size_t)size, sizeof(double));
    memcpy(v, a, (size_t)n * sizeof(double));
    double r = pow2_fold(v, size);
    free(v);
    return r;
}

/* min_reduce value and index (_primitives.py:69-92): ties -> lower index */
double oc_min_reduce(const double *a, int64_t n, int64_t *idx)
{
    double best = a[0];
    int64_t bi = 0;
    for (int64_t i = 1; i < n; i++)
        if (a[i] < best) { best = a[i]; bi = i; }
    if (idx) *idx = bi;
    return best;
}

/* ------------------------------------------------------------ BFS order */
/* _bfs_root_first (mst.py:46-65): children visited by child_id.
 * out receives the root-first order; returns number of vertices reached. */
static int64_t bfs_root_first(const int64_t *parent, const int64_t *child_id, int64_t n,
                              int64_t root, int64_t *out)
{
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *kids = (int64_t *)malloc((size_t)(n > 1 ? n : 1) * sizeof(int64_t));
    for (int64_t u = 0; u < n; u++)
        if (parent[u] != NO_VERTEX) cnt[parent[u] + 1]++;
    for (int64_t u = 0; u < n; u++) cnt[u + 1] += cnt[u];
    /* place each child at offset(parent) + child_id when ids are a
       permutation of 0..deg-1 (true for both constructors) */
    for (int64_t u = 0; u < n; u++) {
        int64_t p = parent[u];
        if (p != NO_VERTEX) kids[cnt[p] + child_id[u]] = u;
    }
    int64_t head = 0, tail = 0;
    out[tail++] = root;
    while (head < tail) {
        int64_t u = out[head++];
        for (int64_t e = cnt[u]; e < cnt[u + 1]; e++) {
            if (tail >= n) { tail = n + 1; break; }
            out[tail++] = kids[e];
        }
        if (tail > n) break;
    }
    free(cnt);
    free(kids);
    return tail > n ? -1 : tail;
}

/* ------------------------------------------------------------------ Prim */
/* prim_mst (mst.py:128-181) on the implicit distance matrix.
 * parent_dist[u] = d(u, parent[u]) (0 at the root), kept for tree weight. */
int oc_prim(const double *X, int64_t n, int64_t d, int64_t root, double sigma,
            int64_t *parent, double *parent_flow, int64_t *depth, int64_t *child_id,
            int64_t *bfs_order, double *parent_dist)
{
    double *best = (double *)malloc((size_t)n * sizeof(double));
    int64_t *best_from = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *child_count = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    char *in_tree = (char *)calloc((size_t)n, 1);
    int nthreads = omp_get_max_threads();
    double *tv = (double *)malloc((size_t)nthreads * 8 * sizeof(double));
    int64_t *ti = (int64_t *)malloc((size_t)nthreads * 8 * sizeof(int64_t));
    for (int64_t u = 0; u < n; u++) {
        parent[u] = NO_VERTEX; depth[u] = 0; child_id[u] = 0;
        best_from[u] = root;
        best[u] = oc_dist(X + root * d, X + u * d, d);
    }
    in_tree[root] = 1;
    int64_t u = -1;
#pragma omp parallel
    {
        int t = omp_get_thread_num(), nt = omp_get_num_threads();
        int64_t lo = n * t / nt, hi = n * (t + 1) / nt;
        for (int64_t step = 0; step < n - 1; step++) {
            /* frontier min: smallest value, ties -> smallest vertex index */
            double bv = INFINITY; int64_t bi = -1;
            for (int64_t j = lo; j < hi; j++)
                if (!in_tree[j] && (bi < 0 || best[j] < bv)) { bv = best[j]; bi = j; }
            tv[t * 8] = bv; ti[t * 8] = bi;
#pragma omp barrier
#pragma omp single
            {
                double gv = INFINITY; int64_t gi = -1;
                for (int s = 0; s < nt; s++) {
                    int64_t ci = ti[s * 8];
                    if (ci < 0) continue;
                    if (gi < 0 || tv[s * 8] < gv) { gv = tv[s * 8]; gi = ci; }
                }
                u = gi;
                int64_t pu = best_from[u];
                parent[u] = pu;
                depth[u] = depth[pu] + 1;
                child_id[u] = child_count[pu]++;
                in_tree[u] = 1;
            }
            const double *xu = X + u * d;
            for (int64_t j = lo; j < hi; j++) {
                if (in_tree[j]) continue;
                double r = oc_dist(xu, X + j * d, d);
                if (r < best[j]) { best[j] = r; best_from[j] = u; }
            }
#pragma omp barrier
        }
    }
    for (int64_t v = 0; v < n; v++) {
        if (parent[v] == NO_VERTEX) { parent_flow[v] = 0.0; parent_dist[v] = 0.0; continue; }
        double dv = oc_dist(X + v * d, X + parent[v] * d, d);
        parent_dist[v] = dv;
        parent_flow[v] = oc_flow(dv, sigma);
    }
    int64_t *order = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t got = bfs_root_first(parent, child_id, n, root, order);
    for (int64_t i = 0; i < n; i++) bfs_order[i] = order[n - 1 - i];
    free(order); free(best); free(best_from); free(child_count); free(in_tree); free(tv); free(ti);
    return got == n ? 0 : 1;
}

/* tree_from_parent_list (mst.py:78-125): child ids by ascending vertex
 * index, depth by BFS; returns 1 if not one connected tree. */
int oc_tree_from_parent(const int64_t *parent, int64_t n, int64_t root,
                        int64_t *depth, int64_t *child_id, int64_t *bfs_order)
{
    int64_t *cc = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    for (int64_t u = 0; u < n; u++) {
        child_id[u] = 0;
        if (parent[u] != NO_VERTEX) child_id[u] = cc[parent[u]]++;
    }
    free(cc);
    int64_t *order = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t got = bfs_root_first(parent, child_id, n, root, order);
    if (got != n) { free(order); return 1; }
    depth[root] = 0;
    for (int64_t i = 1; i < n; i++) depth[order[i]] = depth[parent[order[i]]] + 1;
    for (int64_t i = 0; i < n; i++) bfs_order[i] = order[n - 1 - i];
    free(order);
    return 0;
}

/* ---------------------------------------------------------------- decide */
/* decide (isoperim.py:82-144) + _resolve_groups (:147-161).
 * Returns clusters_found j; cut/eta/sparsities filled (sparsities in cut order). */
int64_t oc_decide(int64_t n, int64_t root, const int64_t *parent, const double *flows,
                  const int64_t *bfs_order, const double *omega0, const double *p0,
                  int64_t k, double N, int8_t *cut, int64_t *eta, double *sparsities)
{
    double *om = (double *)malloc((size_t)n * sizeof(double));
    double *p = (double *)malloc((size_t)n * sizeof(double));
    int64_t *merged = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    memcpy(om, omega0, (size_t)n * sizeof(double));
    memcpy(p, p0, (size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; i++) { merged[i] = i; cut[i] = 0; }
    int64_t j = 0;
    for (int64_t t = 0; t < n; t++) {
        if (j >= k) break;
        int64_t x = bfs_order[t], u;
        double f;
        if (x == root) { u = NO_VERTEX; f = 0.0; }
        else { u = parent[x]; f = flows[x]; }
        double px = p[x], ox = om[x];
        double rhs = N * ox;
        if (f + px <= rhs) {
            sparsities[j] = (f + px) / ox;
            j += 1;
            cut[x] = 1;
            if (u != NO_VERTEX) p[u] = p[u] + f;
        } else if (px - f < rhs) {
            merged[x] = u;
            om[u] = om[u] + ox;
            p[u] = p[u] + px;
        } else {
            if (u != NO_VERTEX) p[u] = p[u] + f;
        }
    }
    int64_t *rep = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    for (int64_t t = n - 1; t >= 0; t--) {
        int64_t x = bfs_order[t];
        int64_t m = merged[x];
        rep[x] = (m == x) ? x : rep[m];
    }
    for (int64_t i = 0; i < n; i++) eta[i] = cut[rep[i]] ? rep[i] : NO_VERTEX;
    free(rep); free(om); free(p); free(merged);
    return j;
}

/* extract_labels (isoperim.py:164-181) */
void oc_extract_labels(const int8_t *cut, const int64_t *eta, int64_t n, int64_t *labels)
{
    int64_t *scan = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t acc = 0;
    for (int64_t i = 0; i < n; i++) { scan[i] = acc; acc += cut[i]; }
    for (int64_t i = 0; i < n; i++) labels[i] = eta[i] != NO_VERTEX ? 1 + scan[eta[i]] : 0;
    free(scan);
}

/* subpartition_cost (isoperim.py:184-219); returns NaN on invalid labels */
double oc_subpartition_cost(const int64_t *labels, int64_t n, const int64_t *parent,
                            const double *flows, const double *omega, const double *p)
{
    int64_t k = 0;
    for (int64_t i = 0; i < n; i++) if (labels[i] > k) k = labels[i];
    if (k < 1) return NAN;
    double *buf = (double *)malloc((size_t)n * sizeof(double));
    double worst = -INFINITY;
    for (int64_t c = 1; c <= k; c++) {
        int64_t m = 0;
        for (int64_t u = 0; u < n; u++) {
            int64_t pu = parent[u];
            if (pu == NO_VERTEX) continue;
            if ((labels[u] == c) != (labels[pu] == c)) buf[m++] = flows[u];
        }
        double boundary = oc_pairwise_sum(buf, m);
        m = 0;
        for (int64_t u = 0; u < n; u++) if (labels[u] == c) buf[m++] = p[u];
        if (m == 0) { free(buf); return NAN; }
        double potential = oc_pairwise_sum(buf, m);
        m = 0;
        for (int64_t u = 0; u < n; u++) if (labels[u] == c) buf[m++] = omega[u];
        double mass = oc_pairwise_sum(buf, m);
        double s = (boundary + potential) / mass;
        if (s > worst) worst = s;
    }
    free(buf);
    return worst;
}

int oc_num_threads(void) { return omp_get_max_threads(); }
void oc_set_threads(int t) { omp_set_num_threads(t); }
