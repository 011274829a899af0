// Microbenchmark: throughput of the exact-distance op pattern
// (t = a-b; s = s + t*t, separately rounded) vs ILP and occupancy.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void chain(double* out, int iters, double seed) {
    double s[C], a[C];
#pragma unroll
    for (int c = 0; c < C; ++c) { s[c] = 0.0; a[c] = seed + c + threadIdx.x; }
    double b = seed * 0.5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double t = __dsub_rn(a[c], b);
            s[c] = __dadd_rn(s[c], __dmul_rn(t, t));
        }
        b = b + 1e-9;
    }
    double r = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) r += s[c];
    if (r == -1.0) out[0] = r;
}
template <int C>
void run(int threads, int blocks_per_sm, int sms) {
    double* out; cudaMalloc(&out, 8);
    int iters = 2048;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    chain<C><<<sms * blocks_per_sm, threads>>>(out, 16, 1.0);
    cudaEventRecord(a);
    chain<C><<<sms * blocks_per_sm, threads>>>(out, iters, 1.0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = 3.0 * C * iters * (double)threads * sms * blocks_per_sm;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("C=%2d threads=%4d blk/sm=%d: %.2f Tops/s = %.1f ops/clk/SM\n", C, threads, blocks_per_sm,
           ops / ms / 1e9, ops / (ms * 1e-3) / (clk * 1e3) / sms);
    cudaFree(out);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int tb : {1, 2, 4}) {
        run<4>(256, tb, sms); run<8>(256, tb, sms); run<16>(256, tb, sms); run<32>(256, tb, sms);
    }
    run<16>(512, 1, sms); run<16>(1024, 1, sms); run<32>(512, 1, sms);
    return 0;
}
