/* Plain-C host of the one-call boundary: read n x d fp64 points from a raw
 * file, run isoc_run on GPU 0, print sigma, miso, iterations and labels.
 * Built and run by tests/test_gpu_parity.py::test_plain_c_host. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "isoclust_b200.h"

int main(int argc, char **argv) {
    if (argc != 5) {
        fprintf(stderr, "usage: %s points.f64 n d k\n", argv[0]);
        return 2;
    }
    const int64_t n = atoll(argv[2]);
    const int32_t d = atoi(argv[3]);
    const int64_t k = atoll(argv[4]);
    double *pts = malloc((size_t)n * d * sizeof(double));
    FILE *f = fopen(argv[1], "rb");
    if (!f || fread(pts, sizeof(double), (size_t)n * d, f) != (size_t)n * d) return 2;
    fclose(f);
    int64_t *labels = malloc((size_t)n * sizeof(int64_t));
    isoc_run_out out = {0};
    out.labels = labels;
    int s = isoc_run(pts, n, d, k, 0.0, 0.0, 0, NULL, &out);
    if (s != ISOC_OK) {
        fprintf(stderr, "isoc_run failed (%d): %s\n", s, isoc_last_error());
        return 1;
    }
    printf("%.17g %.17g %lld\n", out.sigma, out.miso, (long long)out.iterations);
    for (int64_t i = 0; i < n; ++i) printf("%lld\n", (long long)labels[i]);
    free(labels);
    free(pts);
    return 0;
}
