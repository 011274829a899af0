/* Run-time dispatch for isoc_fast.c (TEST INFRASTRUCTURE ONLY): the x86-64-v4
 * (AVX-512) build where the host has it, else the x86-64-v3 (AVX2+FMA) build.
 * Both builds compute identical bits: the arithmetic is per lane with
 * contraction off, and the exp's fmas are explicit. */
#include <stdint.h>

#define DECL(sfx)                                                                          \
    double ocf_flat_distance_sum##sfx(const double *, int64_t, int);                        \
    int ocf_omega_knn##sfx(const double *, int64_t, int, double, int64_t, int64_t, int,     \
                           double *, double *, int64_t *);                                  \
    int ocf_rescan_rows##sfx(const double *, int64_t, int, const int64_t *, int64_t,        \
                             const int32_t *, int, double *, int64_t *);
DECL(_v4)
DECL(_v3)

static int use_v4(void)
{
    static int v = -1;
    if (v < 0) {
        __builtin_cpu_init();
        v = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512dq") &&
            __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512bw");
    }
    return v;
}

int ocf_isa(void) { return use_v4() ? 4 : 3; }

double ocf_flat_distance_sum(const double *X, int64_t n, int d)
{
    return use_v4() ? ocf_flat_distance_sum_v4(X, n, d) : ocf_flat_distance_sum_v3(X, n, d);
}

int ocf_omega_knn(const double *X, int64_t n, int d, double sigma, int64_t lo, int64_t hi, int K,
                  double *omega, double *knn_d, int64_t *knn_j)
{
    return use_v4() ? ocf_omega_knn_v4(X, n, d, sigma, lo, hi, K, omega, knn_d, knn_j)
                    : ocf_omega_knn_v3(X, n, d, sigma, lo, hi, K, omega, knn_d, knn_j);
}

int ocf_rescan_rows(const double *X, int64_t n, int d, const int64_t *rows, int64_t nrows,
                    const int32_t *comp, int K, double *knn_d, int64_t *knn_j)
{
    return use_v4() ? ocf_rescan_rows_v4(X, n, d, rows, nrows, comp, K, knn_d, knn_j)
                    : ocf_rescan_rows_v3(X, n, d, rows, nrows, comp, K, knn_d, knn_j);
}
