// extern "C" entry points of libisoclust_b200.so (see include/isoclust_b200.h).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/isoclust_b200.h"
#include "common.cuh"
#include "kernels.h"
#include "scratch.h"

using namespace isoc;

static_assert(sizeof(FoldStack) == ISOC_FOLD_STACK_BYTES, "fold stack layout");

namespace {
thread_local std::string g_err;

// Keep freed stream-ordered allocations cached in the device's default pool
// (the default release threshold of 0 unmaps them at every synchronize, and
// re-mapping GBs of per-pass scratch costs hundreds of ms per pipeline run).
void ensure_pool() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

}  // namespace

namespace isoc {
// error reporting for the host-side modules (run.cu)
int set_error(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
}  // namespace isoc

namespace {

#define CK(expr)                                                                              \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess) {                                                              \
            cudaGetLastError();                                                               \
            return fail(_e == cudaErrorMemoryAllocation ? ISOC_ENOMEM : ISOC_ECUDA,           \
                        "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__,      \
                        __LINE__);                                                            \
        }                                                                                     \
    } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t count, cudaStream_t st) {
    ensure_pool();
    return isoc_malloc_async(reinterpret_cast<void**>(p), (count ? count : 1) * sizeof(T), st);
}

template <typename T>
cudaError_t aalloc(T** p, size_t count, cudaStream_t st) {
    ensure_pool();
    return isoc_malloc_async(reinterpret_cast<void**>(p), (count ? count : 1) * sizeof(T), st);
}

// Per-thread scratch arena for the partition phase (batched sweeps, the
// witness): its buffers outlive the tree handles, so repeated pipeline runs
// allocate nothing there (a pool allocation inside the bisection loop was
// seen to stall the host for up to ~0.3 s).  Growth frees the old buffer in
// stream order; every user synchronizes its stream before returning, so a
// buffer is idle whenever another handle picks it up.
enum ArenaSlot { AR_BOM, AR_BP, AR_BCODE, AR_BEXCL, AR_BSCRATCH, AR_BTHR, AR_BJ, AR_CUT, AR_ETA, AR_LAB,
                 AR_LAB32, AR_WORK, AR_SUMS, AR_MISO, AR_CWORK, AR_COUNT };
template <typename T>
cudaError_t arena(ArenaSlot slot, T** p, size_t count, cudaStream_t st) {
    struct Buf { void* p = nullptr; size_t bytes = 0; int dev = -1; };
    static thread_local Buf bufs[AR_COUNT];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const size_t bytes = (count ? count : 1) * sizeof(T);
    Buf& b = bufs[slot];
    if (b.dev != dev || b.bytes < bytes) {
        if (b.p && b.dev == dev) isoc_free_async(b.p, st);
        b.p = nullptr;
        b.bytes = 0;
        ensure_pool();
        e = isoc_malloc_async(&b.p, bytes, st);
        if (e != cudaSuccess) return e;
        b.bytes = bytes;
        b.dev = dev;
    }
    *p = static_cast<T*>(b.p);
    return cudaSuccess;
}

static size_t device_total_memory() {
    static size_t cache[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev] == 0) {
        cudaDeviceProp prop;
        cache[dev] = cudaGetDeviceProperties(&prop, dev) == cudaSuccess ? prop.totalGlobalMem : ((size_t)80 << 30);
    }
    return cache[dev];
}

// Per-thread page-locked staging (4 KB) for the small read-backs of the MST
// rounds and the sweeps (each use copies, synchronizes and reads within one
// call), and the witness's side stream: created once per thread and device,
// not per handle -- cudaMallocHost / cudaFreeHost / stream creation on every
// pipeline run were part of the same random host stalls as the allocations.
static void* host_stage() {
    struct Pin { void* p = nullptr; };
    static thread_local Pin pin;
    if (!pin.p && cudaMallocHost(&pin.p, 4096) != cudaSuccess) pin.p = nullptr;
    return pin.p;
}

struct SideStream {
    int dev = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t ready = nullptr, copied = nullptr;
};
static cudaError_t side_stream(SideStream** out) {
    static thread_local SideStream side;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (side.dev != dev) {   // first use on this device (a previous device's stream is left to the context)
        e = cudaStreamCreateWithFlags(&side.s, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&side.ready, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&side.copied, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
        side.dev = dev;
    }
    *out = &side;
    return cudaSuccess;
}

__global__ void scale_kernel(double* v, int64_t m, double a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) v[i] = __dmul_rn(a, v[i]);
}

__global__ void iota_kernel(int32_t* v, int64_t m) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) v[i] = (int32_t)i;
}

// component ids 0..n-1; padding columns get -3 (never equal to a row's id)
__global__ void iota_pad_kernel(int32_t* v, int64_t n, int64_t npad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < npad) v[i] = i < n ? (int32_t)i : -3;
}

__global__ void exp_kernel(const double* x, double* y, int64_t m) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) y[i] = isoc_exp(x[i]);
}

__global__ void root_flow_kernel(double* flow, int64_t root) { flow[root] = 0.0; }

inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Merge `count` stacks in place (ping-pong) until one remains; result in *out.
cudaError_t fold_stacks(const FoldStack* in, int64_t count, FoldStack* out, int32_t* flags,
                        cudaStream_t st) {
    if (count == 1) return cudaMemcpyAsync(out, in, sizeof(FoldStack), cudaMemcpyDeviceToDevice, st);
    FoldStack *a = nullptr, *b = nullptr;
    const int64_t n1 = (count + 63) / 64;
    cudaError_t e = aalloc(&a, n1, st);
    if (e != cudaSuccess) return e;
    e = aalloc(&b, n1, st);
    if (e != cudaSuccess) return e;
    launch_stack_merge(in, count, 64, a, flags, st);
    int64_t cur = n1;
    while (cur > 1) {
        launch_stack_merge(a, cur, 64, b, flags, st);
        cur = (cur + 63) / 64;
        FoldStack* t = a; a = b; b = t;
    }
    cudaMemcpyAsync(out, a, sizeof(FoldStack), cudaMemcpyDeviceToDevice, st);
    isoc_free_async(a, st);
    isoc_free_async(b, st);
    return cudaGetLastError();
}
}  // namespace

extern "C" {

int isoc_version(void) { return 1; }

const char* isoc_last_error(void) { return g_err.c_str(); }

int isoc_exp_dev(const double* x, double* y, int64_t m, void* stream) {
    if (m <= 0) return ISOC_OK;
    exp_kernel<<<blocks(m, 256), 256, 0, (cudaStream_t)stream>>>(x, y, m);
    CK(cudaGetLastError());
    return ISOC_OK;
}

// ------------------------------------------------------------------ sigma
int isoc_sigma_partial(const double* X, int64_t n, int32_t d, int64_t lo, int64_t hi, double alpha,
                       void* stack_dev, int32_t* nn_j, double* nn_d, int8_t* nn_tie, double* p_dev,
                       void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 2 || d < 1) return fail(ISOC_EINVAL, "need n >= 2 and d >= 1 (n=%lld, d=%d)", (long long)n, d);
    if (lo < 0 || hi > n || lo >= hi) return fail(ISOC_EINVAL, "bad row range [%lld, %lld)", (long long)lo, (long long)hi);
    if (n > (int64_t)INT32_MAX) return fail(ISOC_EINVAL, "n too large");
    const int64_t rows = hi - lo;
    const int want_p = alpha > 0.0;
    double* row_vals = nullptr;
    int32_t *row_cnt = nullptr, *flags = nullptr;
    uint64_t *row_ids = nullptr, *sid = nullptr;
    double* sval = nullptr;
    int8_t* sown = nullptr;
    FoldStack* groups = nullptr;
    CK(aalloc(&row_vals, sigma_rowstack_entries(rows), st));
    CK(aalloc(&row_ids, sigma_rowstack_entries(rows), st));
    CK(aalloc(&row_cnt, rows, st));
    CK(aalloc(&flags, 1, st));
    CK(aalloc(&sval, rows, st));
    CK(aalloc(&sid, rows, st));
    CK(aalloc(&sown, rows, st));
    const int64_t ng = (rows + 63) / 64;
    CK(aalloc(&groups, ng, st));
    CK(cudaMemsetAsync(flags, 0, sizeof(int32_t), st));
    CK(cudaMemsetAsync(sown, 0, rows, st));
    if (sigma_sym_applicable(n, lo, hi, want_p))
        CK(launch_sigma_sym(X, n, d, row_vals, row_ids, row_cnt, flags, nn_j, nn_d, nn_tie, st));
    else {
        // the row pass always evaluates the nearest neighbours; give it scratch
        // when the caller does not want them
        int32_t* tj = nn_j;
        double* td = nn_d;
        int8_t* tt = nn_tie;
        if (!nn_j) {
            CK(aalloc(&tj, rows, st));
            CK(aalloc(&td, rows, st));
            CK(aalloc(&tt, rows, st));
        }
        CK(launch_sigma_pass(X, n, d, lo, hi, want_p, row_vals, row_ids, row_cnt, flags, tj, td, tt,
                             want_p ? p_dev : nullptr, st));
        if (!nn_j) {
            isoc_free_async(tj, st);
            isoc_free_async(td, st);
            isoc_free_async(tt, st);
        }
    }
    const int64_t b_hi = hi + 1;  // boundaries lo+1 .. hi (boundary n = the final leaf)
    CK(launch_sigma_straddle(X, n, d, lo + 1, b_hi, sval, sid, sown, st));
    CK(launch_sigma_merge_rows(n, lo, hi, 64, row_vals, row_ids, row_cnt, sval, sid, sown, groups,
                               flags, st));
    CK(fold_stacks(groups, ng, reinterpret_cast<FoldStack*>(stack_dev), flags, st));
    if (want_p) {
        scale_kernel<<<blocks(rows, 256), 256, 0, st>>>(p_dev, rows, alpha);
        CK(cudaGetLastError());
    } else if (p_dev) {
        CK(cudaMemsetAsync(p_dev, 0, (size_t)rows * sizeof(double), st));
    }
    int32_t hflags = 0;
    CK(cudaMemcpyAsync(&hflags, flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    isoc_free_async(row_vals, st); isoc_free_async(row_ids, st); isoc_free_async(row_cnt, st);
    isoc_free_async(sval, st); isoc_free_async(sid, st); isoc_free_async(sown, st);
    isoc_free_async(groups, st); isoc_free_async(flags, st);
    CK(cudaStreamSynchronize(st));
    if (hflags) return fail(ISOC_ECUDA, "pairwise fold stack overflow (flags=%d)", hflags);
    return ISOC_OK;
}

int isoc_sym_block_range(int64_t n, int32_t rank, int32_t world, int64_t* jlo, int64_t* jhi) {
    if (n < 1 || world < 1 || rank < 0 || rank >= world) return fail(ISOC_EINVAL, "bad rank/world");
    sym_block_range(n, rank, world, jlo, jhi, sigma_sym_block());
    return ISOC_OK;
}

int isoc_omega_block_range(int64_t n, int32_t rank, int32_t world, int64_t* jlo, int64_t* jhi) {
    if (n < 1 || world < 1 || rank < 0 || rank >= world) return fail(ISOC_EINVAL, "bad rank/world");
    sym_block_range(n, rank, world, jlo, jhi, 1024);
    return ISOC_OK;
}

int isoc_sigma_sym_range(const double* X, int64_t n, int32_t d, int64_t jlo, int64_t jhi, double* vals,
                         uint64_t* ids, int32_t* cnt, double* m1, double* m2, int32_t* j1, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 2 || d < 1) return fail(ISOC_EINVAL, "need n >= 2 and d >= 1");
    if (n > (int64_t)INT32_MAX) return fail(ISOC_EINVAL, "n too large");
    const int64_t nbs = (n + sigma_sym_block() - 1) / sigma_sym_block();
    if (jlo < 0 || jhi > nbs || jlo > jhi) return fail(ISOC_EINVAL, "bad block range [%lld, %lld)", (long long)jlo, (long long)jhi);
    ensure_pool();
    int32_t* flags = nullptr;
    CK(aalloc(&flags, 1, st));
    CK(cudaMemsetAsync(flags, 0, sizeof(int32_t), st));
    CK(launch_sigma_sym_range(X, n, d, jlo, jhi, 1, vals, ids, cnt, flags, m1 ? j1 : nullptr, m1, nullptr, m2, st));
    int32_t hflags = 0;
    CK(cudaMemcpyAsync(&hflags, flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    isoc_free_async(flags, st);
    CK(cudaStreamSynchronize(st));
    if (hflags) return fail(ISOC_ECUDA, "pairwise fold stack overflow (flags=%d)", hflags);
    return ISOC_OK;
}

int isoc_sigma_rank_merge(const double* X, int64_t n, int32_t d, int64_t lo, int64_t hi, int32_t G,
                          const double* vals, const uint64_t* ids, const int32_t* cnt, const double* m1,
                          const double* m2, const int32_t* j1, void* stack_dev, int32_t* nn_j, double* nn_d,
                          int8_t* nn_tie, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (n < 2 || d < 1) return fail(ISOC_EINVAL, "need n >= 2 and d >= 1");
    if (lo < 0 || hi > n || lo >= hi) return fail(ISOC_EINVAL, "bad row range");
    if (G < 1) return fail(ISOC_EINVAL, "need at least one rank");
    ensure_pool();
    const int64_t rows = hi - lo;
    double* row_vals = nullptr;
    int32_t *row_cnt = nullptr, *flags = nullptr;
    uint64_t *row_ids = nullptr, *sid = nullptr;
    double* sval = nullptr;
    int8_t* sown = nullptr;
    FoldStack* groups = nullptr;
    CK(aalloc(&row_vals, sigma_rowstack_entries(rows), st));
    CK(aalloc(&row_ids, sigma_rowstack_entries(rows), st));
    CK(aalloc(&row_cnt, rows, st));
    CK(aalloc(&flags, 1, st));
    CK(aalloc(&sval, rows, st));
    CK(aalloc(&sid, rows, st));
    CK(aalloc(&sown, rows, st));
    const int64_t ng = (rows + 63) / 64;
    CK(aalloc(&groups, ng, st));
    CK(cudaMemsetAsync(flags, 0, sizeof(int32_t), st));
    CK(cudaMemsetAsync(sown, 0, rows, st));
    CK(launch_sigma_rank_merge(rows, G, vals, ids, cnt, m1, m2, j1, row_vals, row_ids, row_cnt, flags,
                               (m1 && nn_j) ? nn_j : nullptr, nn_d, nn_tie, st));
    CK(launch_sigma_straddle(X, n, d, lo + 1, hi + 1, sval, sid, sown, st));
    CK(launch_sigma_merge_rows(n, lo, hi, 64, row_vals, row_ids, row_cnt, sval, sid, sown, groups, flags, st));
    CK(fold_stacks(groups, ng, reinterpret_cast<FoldStack*>(stack_dev), flags, st));
    int32_t hflags = 0;
    CK(cudaMemcpyAsync(&hflags, flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    isoc_free_async(row_vals, st); isoc_free_async(row_ids, st); isoc_free_async(row_cnt, st);
    isoc_free_async(sval, st); isoc_free_async(sid, st); isoc_free_async(sown, st);
    isoc_free_async(groups, st); isoc_free_async(flags, st);
    CK(cudaStreamSynchronize(st));
    if (hflags) return fail(ISOC_ECUDA, "pairwise fold stack overflow (flags=%d)", hflags);
    return ISOC_OK;
}

int isoc_sigma_finish(const void* stacks_dev, int64_t nseg, double* total_host, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (nseg < 1) return fail(ISOC_EINVAL, "no fold stacks");
    FoldStack* out = nullptr;
    int32_t* flags = nullptr;
    CK(aalloc(&out, 1, st));
    CK(aalloc(&flags, 1, st));
    CK(cudaMemsetAsync(flags, 0, sizeof(int32_t), st));
    CK(fold_stacks(reinterpret_cast<const FoldStack*>(stacks_dev), nseg, out, flags, st));
    FoldStack h;
    CK(cudaMemcpyAsync(&h, out, sizeof(FoldStack), cudaMemcpyDeviceToHost, st));
    isoc_free_async(out, st);
    isoc_free_async(flags, st);
    CK(cudaStreamSynchronize(st));
    if (h.count != 1 || h.id[0] != 1 || h.overflow)
        return fail(ISOC_EINVAL, "fold stacks do not close to one root (count=%d id=%llu)", h.count,
                    h.count > 0 ? (unsigned long long)h.id[0] : 0ull);
    *total_host = 0.0 + h.value[0];
    return ISOC_OK;
}

// -------------------------------------------------------------------- MST
struct isoc_mst {
    const double* X;
    int64_t n, lo, hi, rows, npad;
    int32_t d, dp;
    cudaStream_t st;
    float cd, cabs;
    int use_tc, filter_forced;
    float kscale;
    uint8_t* img;
    float *Y, *ny, *rad;
    double* centre;
    uint32_t* rmax;
    int32_t* comp;
    float *a1, *a2;
    int32_t* j1;
    uint32_t* compB;
    double* cand_d;
    int32_t* cand_j;
    int8_t *cand_state, *cand_tie;
    int32_t *rescan_list, *counters;  // counters: rescan, ties, ecount, changed, nroots
    int32_t *succ, *succ2;
    int32_t *eu, *ev;
    double* ed;
    // tc filter candidate lists (FILTER_LIST_K per row) and block refresh flags
    float *la, *lb, *lbo;
    int32_t* lj;
    int32_t *blk_flag, *refresh_rows;
    uint8_t* imgA;
    int64_t nblk;
    int lists_valid;
    int64_t filter_blocks_run, filter_blocks_total, filter_rows_refreshed;
    int32_t* pin;   // page-locked copy of the counters (one per-round read-back)
};

static void mst_free(isoc_mst* h) {
    if (!h) return;
    void* ptrs[] = {h->img, h->Y, h->ny, h->rad, h->centre, h->rmax, h->comp, h->a1, h->a2, h->j1,
                    h->compB, h->cand_d, h->cand_j, h->cand_state, h->cand_tie, h->rescan_list,
                    h->counters, h->succ, h->succ2, h->eu, h->ev, h->ed, h->la, h->lb, h->lbo, h->lj,
                    h->blk_flag, h->refresh_rows, h->imgA};
    for (void* p : ptrs)
        if (p) isoc_free_async(p, h->st);
    delete h;
}

int isoc_mst_create(const double* X, int64_t n, int32_t d, int64_t lo, int64_t hi, void* stream,
                    isoc_mst** out) {
    *out = nullptr;
    if (n < 2 || d < 1) return fail(ISOC_EINVAL, "need n >= 2 and d >= 1");
    if (lo < 0 || hi > n || lo >= hi) return fail(ISOC_EINVAL, "bad row range");
    if (n > (int64_t)INT32_MAX) return fail(ISOC_EINVAL, "n too large");
    isoc_mst* h = new isoc_mst();
    memset(h, 0, sizeof(*h));
    h->X = X; h->n = n; h->d = d; h->lo = lo; h->hi = hi; h->rows = hi - lo;
    h->dp = (d + 15) / 16 * 16;
    h->npad = (n + 127) / 128 * 128 + 128;
    h->st = (cudaStream_t)stream;
    // rigorous FP32 Gram error coefficient, inflated ("filter bound")
    h->cd = (float)((((double)h->dp + 9.0) * 0x1p-24 + 0x1p-30) * 1.0625);
#define MCK(expr)                                              \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) {                               \
            mst_free(h);                                       \
            cudaGetLastError();                                \
            return fail(_e == cudaErrorMemoryAllocation ? ISOC_ENOMEM : ISOC_ECUDA, \
                        "%s: %s", #expr, cudaGetErrorString(_e)); \
        }                                                      \
    } while (0)
    MCK(dalloc(&h->Y, (size_t)h->npad * h->dp, h->st));
    MCK(dalloc(&h->ny, h->npad, h->st));
    MCK(dalloc(&h->rad, n, h->st));
    MCK(dalloc(&h->centre, d, h->st));
    MCK(dalloc(&h->rmax, 1, h->st));
    MCK(dalloc(&h->comp, h->npad, h->st));
    MCK(dalloc(&h->a1, h->rows, h->st));
    MCK(dalloc(&h->a2, h->rows, h->st));
    MCK(dalloc(&h->j1, h->rows, h->st));
    MCK(dalloc(&h->compB, n, h->st));
    MCK(dalloc(&h->cand_d, h->rows, h->st));
    MCK(dalloc(&h->cand_j, h->rows, h->st));
    MCK(dalloc(&h->cand_state, h->rows, h->st));
    MCK(dalloc(&h->cand_tie, h->rows, h->st));
    MCK(dalloc(&h->rescan_list, h->rows, h->st));
    MCK(dalloc(&h->counters, 8, h->st));
    MCK(dalloc(&h->succ, n, h->st));
    MCK(dalloc(&h->succ2, n, h->st));
    MCK(dalloc(&h->eu, n, h->st));
    MCK(dalloc(&h->ev, n, h->st));
    MCK(dalloc(&h->ed, n, h->st));
    MCK(cudaMemsetAsync(h->counters, 0, 8 * sizeof(int32_t), h->st));
    iota_pad_kernel<<<blocks(h->npad, 256), 256, 0, h->st>>>(h->comp, n, h->npad);
    MCK(cudaGetLastError());
    MCK(launch_prep_fp32(X, n, d, h->dp, h->npad, h->centre, h->Y, h->ny, h->rad, h->rmax, h->st));
    // tensor-core filter (tcgen05, 3-term FP16 split) for d <= 64 unless ISOC_FILTER=ffma
    const char* fenv = getenv("ISOC_FILTER");
    h->use_tc = (d <= 512) && !(fenv && strcmp(fenv, "ffma") == 0);
    h->filter_forced = fenv != nullptr;
    if (h->use_tc) {
        uint32_t* am = nullptr;
        MCK(dalloc(&am, 1, h->st));
        MCK(launch_absmax(h->Y, (int64_t)h->npad * h->dp, am, h->st));
        uint32_t amb = 0;
        MCK(cudaMemcpyAsync(&amb, am, 4, cudaMemcpyDeviceToHost, h->st));
        MCK(cudaStreamSynchronize(h->st));
        isoc_free_async(am, h->st);
        float amax = 0.f;
        memcpy(&amax, &amb, 4);
        int s = 0;  // y * 2^s stays below 2^14 in FP16
        if (amax > 0.f) s = 14 - (int)ceil(log2((double)amax));
        if (s > 40) s = 40;
        if (s < -14) s = -14;
        const float scale = (float)ldexp(1.0, s);
        h->kscale = (float)-ldexp(1.0, 1 - 2 * s);
        // split + tensor-core accumulation bound ("filter bound")
        // (linear in the padded depth, as the FFMA bound; 64 per K atom)
        const double kd = (double)((d + 63) / 64 * 64);
        h->cd = (float)(((13.0 * kd + 40.0) * 0x1p-24 + 0x1p-30) * 1.25);
        h->cabs = (float)(ldexp(1.0, -22 - s) * 8.0 * 2.0 * (kd / 64.0));
        MCK(dalloc(&h->img, tc_image_bytes(n, d), h->st));
        MCK(launch_tc_image(h->Y, h->npad, d, scale, n, h->img, h->st));
        MCK(dalloc(&h->la, h->rows * FILTER_LIST_K, h->st));
        MCK(dalloc(&h->lj, h->rows * FILTER_LIST_K, h->st));
        MCK(dalloc(&h->lb, h->rows, h->st));
        MCK(dalloc(&h->lbo, h->rows, h->st));
        h->nblk = filter_tc_blocks(lo, hi);
        MCK(dalloc(&h->blk_flag, h->nblk, h->st));
        MCK(dalloc(&h->refresh_rows, h->rows, h->st));
        MCK(dalloc(&h->imgA, tc_image_bytes((h->rows + 255) / 256 * 256, d), h->st));
    } else {
        h->cabs = 0.f;
    }
#undef MCK
    *out = h;
    return ISOC_OK;
}

int isoc_mst_round_local(isoc_mst* h, int use_nn, const int32_t* nn_j, const double* nn_d,
                         const int8_t* nn_tie, uint64_t* comp_min) {
    cudaStream_t st = h->st;
    if (use_nn) {
        CK(launch_nn_candidates(nn_j, nn_d, nn_tie, h->rows, h->cand_d, h->cand_j, h->cand_state,
                                h->cand_tie, st));
    } else if ((double)h->n * (double)h->n * (double)h->d <= 2.0e8 && !h->filter_forced) {
        // tiny problem: exact rescans of every row beat the filter's launches
        // (ISOC_FILTER=tc|ffma forces a filter: tests)
        CK(launch_boruvka_exact_all(h->X, h->n, h->d, h->comp, h->lo, h->hi, h->cand_d, h->cand_j,
                                    h->cand_state, h->cand_tie, h->rescan_list, h->counters + 0, st));
    } else {
        if (h->use_tc) {
            // candidate lists: the first filter round scans every block; later
            // rounds read each row's minimum from its list and re-run the
            // filter only for blocks holding a row whose list ran out while it
            // may still hold its component's minimum
            if (!h->lists_valid) {
                CK(launch_filter_tc(h->img, h->ny, h->comp, h->n, h->d, h->lo, h->hi, h->kscale, h->la, h->lj,
                                    h->lb, nullptr, nullptr, 0, nullptr, st));
                h->lists_valid = 1;
                h->filter_blocks_run += h->nblk;
                h->filter_blocks_total += h->nblk;
                CK(launch_list_select(h->la, h->lj, h->lb, h->comp, h->lo, h->hi, h->a1, h->j1, h->a2, h->lbo,
                                      st));
            } else {
                CK(launch_list_select(h->la, h->lj, h->lb, h->comp, h->lo, h->hi, h->a1, h->j1, h->a2, h->lbo,
                                      st));
                CK(launch_list_refresh(h->a1, h->lbo, h->rad, h->comp, h->n, h->lo, h->hi, h->rmax, h->cd,
                                       h->cabs, h->compB, h->blk_flag, h->nblk, h->counters + 5,
                                       h->refresh_rows, st));
                h->pin = static_cast<int32_t*>(host_stage());
                if (!h->pin) return fail(ISOC_ECUDA, "page-locked staging unavailable");
                CK(cudaMemcpyAsync(h->pin + 8, h->counters + 5, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                const int32_t nf[2] = {h->pin[8], h->pin[9]};   // flagged blocks, rows
                h->filter_blocks_total += h->nblk;
                h->filter_rows_refreshed += nf[1];
                if (nf[1] > 0) {
                    // the rows whose list ran out, gathered (row granularity)
                    h->filter_blocks_run += (nf[1] + 255) / 256;
                    CK(launch_filter_tc(h->img, h->ny, h->comp, h->n, h->d, h->lo, h->hi, h->kscale, h->la,
                                        h->lj, h->lb, h->refresh_rows, h->counters + 6, nf[1], h->imgA, st));
                    CK(launch_list_select(h->la, h->lj, h->lb, h->comp, h->lo, h->hi, h->a1, h->j1, h->a2,
                                          h->lbo, st));
                }
            }
        } else
            CK(launch_boruvka_filter(h->Y, h->ny, h->comp, h->n, h->npad, h->dp, h->lo, h->hi, h->a1,
                                     h->j1, h->a2, st));
        CK(launch_boruvka_select(h->X, h->n, h->d, h->a1, h->j1, h->a2, h->rad, h->rmax, h->cd, h->cabs,
                                 h->comp,
                                 h->lo, h->hi, h->compB, h->cand_d, h->cand_j, h->cand_state,
                                 h->cand_tie, h->rescan_list, h->counters + 0, st));
    }
    CK(launch_comp_exact_min(h->cand_d, h->cand_state, h->comp, h->n, h->lo, h->hi,
                             reinterpret_cast<unsigned long long*>(comp_min), st));
    return ISOC_OK;
}

int isoc_mst_round_edges(isoc_mst* h, const uint64_t* comp_min, uint64_t* comp_edge) {
    CK(launch_comp_edge(h->cand_d, h->cand_j, h->cand_state, h->comp, h->n, h->lo, h->hi,
                        reinterpret_cast<const unsigned long long*>(comp_min),
                        reinterpret_cast<unsigned long long*>(comp_edge), h->st));
    return ISOC_OK;
}

int isoc_mst_round_finish(isoc_mst* h, const uint64_t* comp_min, const uint64_t* comp_edge,
                          int64_t* components, int64_t* ties, int64_t* rescans) {
    cudaStream_t st = h->st;
    const auto* cm = reinterpret_cast<const unsigned long long*>(comp_min);
    const auto* ce = reinterpret_cast<const unsigned long long*>(comp_edge);
    CK(launch_comp_ties(h->cand_d, h->cand_j, h->cand_state, h->cand_tie, h->comp, h->lo, h->hi, cm,
                        ce, h->counters + 1, st));
    CK(launch_hook_contract(h->comp, h->n, cm, ce, h->succ, h->succ2, h->eu, h->ev, h->ed,
                            h->counters + 2, h->counters + 3, h->counters + 4, st));
    h->pin = static_cast<int32_t*>(host_stage());
    if (!h->pin) return fail(ISOC_ECUDA, "page-locked staging unavailable");
    CK(cudaMemcpyAsync(h->pin, h->counters, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int32_t c[8];
    memcpy(c, h->pin, sizeof c);
    if (components) *components = c[4];
    if (ties) *ties = c[1];
    if (rescans) *rescans = c[0];
    if (c[2] > h->n - 1) return fail(ISOC_ECUDA, "MST edge overflow (%d edges)", c[2]);
    return ISOC_OK;
}

int isoc_mst_edges(isoc_mst* h, int32_t* u, int32_t* v, double* w) {
    int32_t cnt = 0;
    CK(cudaMemcpyAsync(&cnt, h->counters + 2, sizeof cnt, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (cnt != h->n - 1) return fail(ISOC_ECUDA, "MST has %d edges, expected %lld", cnt, (long long)(h->n - 1));
    if (u) CK(cudaMemcpyAsync(u, h->eu, (size_t)cnt * 4, cudaMemcpyDeviceToDevice, h->st));
    if (v) CK(cudaMemcpyAsync(v, h->ev, (size_t)cnt * 4, cudaMemcpyDeviceToDevice, h->st));
    if (w) CK(cudaMemcpyAsync(w, h->ed, (size_t)cnt * 8, cudaMemcpyDeviceToDevice, h->st));
    return ISOC_OK;
}

int isoc_mst_filter_stats(isoc_mst* h, int64_t* blocks_run, int64_t* blocks_total, int64_t* rows_refreshed) {
    if (!h) return fail(ISOC_EINVAL, "null MST handle");
    if (blocks_run) *blocks_run = h->filter_blocks_run;
    if (blocks_total) *blocks_total = h->filter_blocks_total;
    if (rows_refreshed) *rows_refreshed = h->filter_rows_refreshed;
    return ISOC_OK;
}

void isoc_mst_destroy(isoc_mst* h) {
    if (h) cudaStreamSynchronize(h->st);
    mst_free(h);
}

// ------------------------------------------------------------------ omega
int isoc_omega(const double* X, int64_t n, int32_t d, int64_t lo, int64_t hi, double sigma,
               double* omega, void* stream) {
    if (n < 2 || d < 1) return fail(ISOC_EINVAL, "need n >= 2 and d >= 1");
    if (!(sigma > 0.0)) return fail(ISOC_EINVAL, "sigma must be > 0, got %g", sigma);
    if (lo < 0 || hi > n || lo >= hi) return fail(ISOC_EINVAL, "bad row range");
    return isoc_omega_mst(X, n, d, lo, hi, sigma, nullptr, omega, nullptr, nullptr, nullptr, stream);
}

int isoc_omega_mst(const double* X, int64_t n, int32_t d, int64_t lo, int64_t hi, double sigma,
                   isoc_mst* h, double* omega, int32_t* nn_j, double* nn_d, int8_t* nn_tie,
                   void* stream) {
    if (n < 2 || d < 1) return fail(ISOC_EINVAL, "need n >= 2 and d >= 1");
    if (!(sigma > 0.0)) return fail(ISOC_EINVAL, "sigma must be > 0, got %g", sigma);
    if (lo < 0 || hi > n || lo >= hi) return fail(ISOC_EINVAL, "bad row range");
    ensure_pool();
    const int32_t* comp = h ? h->comp : nullptr;
    if (h && (h->lo != lo || h->hi != hi)) return fail(ISOC_EINVAL, "MST handle rows differ");
    // the symmetric pass keeps one 1024-wide subtree (+ round-2 minimum) per
    // (block, row): 20 B x n^2 / 1024 -- use it while that fits comfortably,
    // and once its I <= J super-tiles fill the SMs (n >~ 17k); below that the
    // row pass finishes sooner (bitwise identical)
    const int64_t nbs = (n + 1023) / 1024;
    const int mode = passes_mode();
    const bool sym_wide = mode == 1 || (mode == 0 && nbs * (nbs + 1) / 2 >= device_sm_count());
    bool sym = lo == 0 && hi == n && sym_wide;
    if (sym) {   // against the device's capacity (queried once: no driver query per call)
        const double ps_bytes = (double)nbs * (double)n * (comp ? 20.0 : 8.0);
        sym = ps_bytes < 0.35 * (double)device_total_memory();
    }
    if (sym) {
        const cudaError_t e = launch_omega_sym(X, n, d, sigma, comp, omega, nn_j, nn_d, nn_tie, (cudaStream_t)stream);
        if (e == cudaErrorMemoryAllocation) {   // the slot buffers did not fit after all: row pass
            cudaGetLastError();
            sym = false;
        } else {
            CK(e);
        }
    }
    if (!sym) {
        CK(launch_omega_pass(X, n, d, lo, hi, sigma, comp, omega, nn_j, nn_d, nn_tie,
                             (cudaStream_t)stream));
    }
    return ISOC_OK;
}

int isoc_omega_shard_counts(int64_t n, int32_t G, int32_t rank, int64_t* send_counts, int64_t* recv_counts) {
    if (n < 2 || G < 1 || rank < 0 || rank >= G) return fail(ISOC_EINVAL, "need n >= 2 and 0 <= rank < G");
    if (!send_counts || !recv_counts) return fail(ISOC_EINVAL, "missing count arrays");
    omega_shard_counts(n, G, rank, send_counts, recv_counts);
    return ISOC_OK;
}

int isoc_omega_sym_range(const double* X, int64_t n, int32_t d, int32_t rank, int32_t G, double sigma,
                         isoc_mst* h, double* ps, double* psm, int32_t* psj, void* stream) {
    if (n < 2 || d < 1) return fail(ISOC_EINVAL, "need n >= 2 and d >= 1");
    if (n > (int64_t)INT32_MAX) return fail(ISOC_EINVAL, "n too large");
    if (!(sigma > 0.0)) return fail(ISOC_EINVAL, "sigma must be > 0, got %g", sigma);
    if (G < 1 || rank < 0 || rank >= G) return fail(ISOC_EINVAL, "need 0 <= rank < G");
    if (!ps || (h && (!psm || !psj))) return fail(ISOC_EINVAL, "missing slot buffers");
    ensure_pool();
    CK(launch_omega_sym_range(X, n, d, sigma, h ? h->comp : nullptr, rank, G, ps, psm, psj,
                              (cudaStream_t)stream));
    return ISOC_OK;
}

int isoc_omega_rank_merge(int64_t n, int32_t rank, int32_t G, const double* ps, const double* psm,
                          const int32_t* psj, double* omega, int32_t* nn_j, double* nn_d, int8_t* nn_tie,
                          void* stream) {
    if (n < 2 || G < 1 || rank < 0 || rank >= G) return fail(ISOC_EINVAL, "need n >= 2 and 0 <= rank < G");
    if (psm && (!psj || !nn_j || !nn_d || !nn_tie)) return fail(ISOC_EINVAL, "missing neighbour buffers");
    CK(launch_omega_rank_merge(n, rank, G, ps, psm, psj, omega, nn_j, nn_d, nn_tie, (cudaStream_t)stream));
    return ISOC_OK;
}

// ------------------------------------------------------------------- tree
struct isoc_tree {
    int64_t n, root, levels, max_width;
    cudaStream_t st;
    std::vector<int64_t> level_off_h;
    int32_t *bfs, *pos_of, *parent_v, *depth_v, *child_id_v, *pos_parent, *child_lo, *child_cnt;
    double *parent_d, *flow_v;
    int64_t* level_off;
    double *omega_v, *p_v, *f_pos, *om_pos, *p_pos;
    double *om_w, *p_w;
    int8_t* code[2];
    double* spars[2];
    int64_t spars_cap[2];
    int32_t *excl, *scratch;
    int64_t* j_out;
    // batched speculative sweeps (isoc_decide_batch), allocated on first use
    void* pin;   // page-locked staging for the per-sweep thresholds / counts (no blocking pageable copies)
    double *bom, *bp, *bthr;
    int8_t* bcode;
    int32_t *bexcl, *bscratch;
    int64_t* bj;
};

static void tree_free(isoc_tree* t) {
    if (!t) return;
    void* ptrs[] = {t->bfs, t->pos_of, t->parent_v, t->depth_v, t->child_id_v, t->pos_parent,
                    t->child_lo, t->child_cnt, t->parent_d, t->flow_v, t->level_off, t->omega_v,
                    t->p_v, t->f_pos, t->om_pos, t->p_pos, t->om_w, t->p_w, t->code[0], t->code[1],
                    t->spars[0], t->spars[1], t->excl, t->scratch, t->j_out};
    for (void* p : ptrs)
        if (p) isoc_free_async(p, t->st);
    delete t;
}

static int tree_alloc(isoc_tree* t, int64_t n) {
    CK(dalloc(&t->bfs, n, t->st));
    CK(dalloc(&t->pos_of, n, t->st));
    CK(dalloc(&t->parent_v, n, t->st));
    CK(dalloc(&t->depth_v, n, t->st));
    CK(dalloc(&t->child_id_v, n, t->st));
    CK(dalloc(&t->pos_parent, n, t->st));
    CK(dalloc(&t->child_lo, n, t->st));
    CK(dalloc(&t->child_cnt, n, t->st));
    CK(dalloc(&t->parent_d, n, t->st));
    CK(dalloc(&t->flow_v, n, t->st));
    CK(dalloc(&t->level_off, n + 2, t->st));
    CK(dalloc(&t->scratch, n + 4096, t->st));
    CK(dalloc(&t->j_out, 4, t->st));
    return ISOC_OK;
}

static int tree_finish_layout(isoc_tree* t, int64_t levels_dev_value) {
    if (levels_dev_value <= 0) return fail(ISOC_EINVAL, "parent array does not describe one connected tree");
    t->levels = levels_dev_value;
    t->level_off_h.resize(t->levels + 1);
    CK(cudaMemcpyAsync(t->level_off_h.data(), t->level_off, (t->levels + 1) * sizeof(int64_t),
                       cudaMemcpyDeviceToHost, t->st));
    CK(cudaStreamSynchronize(t->st));
    if (t->level_off_h[t->levels] != t->n)
        return fail(ISOC_EINVAL, "parent array does not describe one connected tree");
    t->max_width = 0;
    for (int64_t l = 0; l < t->levels; ++l)
        t->max_width = std::max(t->max_width, t->level_off_h[l + 1] - t->level_off_h[l]);
    return ISOC_OK;
}

int isoc_tree_from_edges(const int32_t* u, const int32_t* v, const double* w, int64_t n, int64_t root,
                         double sigma, void* stream, isoc_tree** out) {
    *out = nullptr;
    if (n < 2) return fail(ISOC_EINVAL, "need at least 2 vertices");
    if (root < 0 || root >= n) return fail(ISOC_EINVAL, "root must be in [0, %lld), got %lld", (long long)n, (long long)root);
    if (!(sigma > 0.0)) return fail(ISOC_EINVAL, "sigma must be > 0, got %g", sigma);
    isoc_tree* t = new isoc_tree();
    t->n = n; t->root = root; t->st = (cudaStream_t)stream;
    int rc = tree_alloc(t, n);
    if (rc) { tree_free(t); return rc; }
    int32_t *off = nullptr, *adj = nullptr, *work = nullptr;
    double* adjd = nullptr;
    int64_t* lv = nullptr;
    int64_t levels = 0;
    cudaStream_t st = t->st;
#define TCK(expr) do { cudaError_t _e = (expr); if (_e != cudaSuccess) { cudaGetLastError(); tree_free(t); \
    return fail(_e == cudaErrorMemoryAllocation ? ISOC_ENOMEM : ISOC_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e)); } } while (0)
    {
    Scratch sc(st);   // off / adj / adjd / work / lv freed on every return path
    TCK(sc.alloc(&off, n + 1));
    TCK(sc.alloc(&adj, 2 * n));
    TCK(sc.alloc(&adjd, 2 * n));
    TCK(sc.alloc(&work, n + 2));
    TCK(sc.alloc(&lv, 1));
    TCK(launch_build_adjacency(u, v, w, n, off, adj, adjd, work, st));
    TCK(launch_bfs(n, root, 1, off, adj, adjd, t->bfs, t->pos_of, t->parent_v, t->depth_v,
                   t->child_id_v, t->parent_d, t->pos_parent, t->child_lo, t->child_cnt, t->level_off,
                   t->scratch, lv, st));
    TCK(launch_flows(t->parent_d, t->parent_v, n, sigma, t->flow_v, st));
    TCK(cudaMemcpyAsync(&levels, lv, sizeof levels, cudaMemcpyDeviceToHost, st));
    TCK(cudaStreamSynchronize(st));
    }
    rc = tree_finish_layout(t, levels);
    if (rc) { tree_free(t); return rc; }
    *out = t;
    return ISOC_OK;
}

int isoc_tree_from_parent(const int64_t* parent, const double* flow, const int64_t* child_id,
                          int64_t n, int64_t root, void* stream, isoc_tree** out) {
    *out = nullptr;
    if (n < 1) return fail(ISOC_EINVAL, "empty parent array");
    if (n > (int64_t)INT32_MAX - 1) return fail(ISOC_EINVAL, "n too large");
    if (root >= n) return fail(ISOC_EINVAL, "root does not match the parent array's sentinel");
    isoc_tree* t = new isoc_tree();
    t->n = n; t->root = root; t->st = (cudaStream_t)stream;
    int rc = tree_alloc(t, n);
    if (rc) { tree_free(t); return rc; }
    cudaStream_t st = t->st;
    int32_t *off = nullptr, *adj = nullptr, *flags = nullptr;
    int64_t* lv = nullptr;
    int64_t levels = 0;
    {
    Scratch sc(st);   // off / adj / flags / lv freed on every return path
    TCK(sc.alloc(&off, n + 1));
    TCK(sc.alloc(&adj, n));
    TCK(sc.alloc(&flags, 3));
    TCK(sc.alloc(&lv, 1));
    TCK(cudaMemsetAsync(flags, 0, 2 * sizeof(int32_t), st));
    TCK(cudaMemsetAsync(flags + 2, 0xff, sizeof(int32_t), st));   // found root: -1
    TCK(launch_children_from_parent(parent, child_id, n, root, off, adj, t->child_id_v, flags,
                                    flags + 1, root < 0 ? flags + 2 : nullptr, st));
    int32_t hf[3] = {0, 0, -1};
    TCK(cudaMemcpyAsync(hf, flags, 12, cudaMemcpyDeviceToHost, st));
    TCK(cudaStreamSynchronize(st));
    const int32_t hflags = hf[0], nroots = hf[1];
    // mst.py:95-103: exactly one sentinel (the given root, when one is given)
    if (nroots != 1) {
        tree_free(t);
        return fail(ISOC_EINVAL, "expected exactly one root sentinel, found %d", nroots);
    }
    if (hflags & 1) { tree_free(t); return fail(ISOC_EINVAL, "root does not match the parent array's sentinel"); }
    if (hflags & 2) { tree_free(t); return fail(ISOC_EINVAL, "parent indices out of range"); }
    if (root < 0) root = hf[2];
    t->root = root;
    TCK(launch_bfs(n, root, 0, off, adj, nullptr, t->bfs, t->pos_of, t->parent_v, t->depth_v,
                   t->child_id_v, t->parent_d, t->pos_parent, t->child_lo, t->child_cnt, t->level_off,
                   t->scratch, lv, st));
    TCK(cudaMemcpyAsync(t->flow_v, flow, (size_t)n * 8, cudaMemcpyDeviceToDevice, st));
    root_flow_kernel<<<1, 1, 0, st>>>(t->flow_v, root);
    TCK(cudaMemcpyAsync(&levels, lv, sizeof levels, cudaMemcpyDeviceToHost, st));
    TCK(cudaStreamSynchronize(st));
    }
    rc = tree_finish_layout(t, levels);
    if (rc) { tree_free(t); return rc; }
    *out = t;
    return ISOC_OK;
}

int isoc_tree_export(isoc_tree* t, int64_t* parent, double* parent_flow, int64_t* depth,
                     int64_t* child_id, int64_t* bfs_order, int64_t* max_depth, double* parent_dist) {
    const int64_t n = t->n;
    std::vector<int32_t> tmp(n);
    auto pull32 = [&](const int32_t* src, int64_t* dst) -> int {
        CK(cudaMemcpyAsync(tmp.data(), src, n * 4, cudaMemcpyDeviceToHost, t->st));
        CK(cudaStreamSynchronize(t->st));
        for (int64_t i = 0; i < n; ++i) dst[i] = tmp[i];
        return ISOC_OK;
    };
    int rc;
    if (parent && (rc = pull32(t->parent_v, parent))) return rc;
    if (depth && (rc = pull32(t->depth_v, depth))) return rc;
    if (child_id && (rc = pull32(t->child_id_v, child_id))) return rc;
    if (bfs_order) {
        CK(cudaMemcpyAsync(tmp.data(), t->bfs, n * 4, cudaMemcpyDeviceToHost, t->st));
        CK(cudaStreamSynchronize(t->st));
        for (int64_t i = 0; i < n; ++i) bfs_order[i] = tmp[n - 1 - i];
    }
    if (parent_flow) CK(cudaMemcpyAsync(parent_flow, t->flow_v, n * 8, cudaMemcpyDeviceToHost, t->st));
    if (parent_dist) CK(cudaMemcpyAsync(parent_dist, t->parent_d, n * 8, cudaMemcpyDeviceToHost, t->st));
    CK(cudaStreamSynchronize(t->st));
    if (max_depth) *max_depth = t->levels - 1;
    return ISOC_OK;
}

int isoc_tree_root(const isoc_tree* t, int64_t* root) {
    if (!t || !root) return fail(ISOC_EINVAL, "null tree");
    *root = t->root;
    return ISOC_OK;
}

int isoc_tree_set_weights(isoc_tree* t, const double* omega, const double* p, double* extrema) {
    const int64_t n = t->n;
    cudaStream_t st = t->st;
    if (!t->omega_v) {
        CK(dalloc(&t->omega_v, n, t->st)); CK(dalloc(&t->p_v, n, t->st));
        CK(dalloc(&t->f_pos, n, t->st)); CK(dalloc(&t->om_pos, n, t->st)); CK(dalloc(&t->p_pos, n, t->st));
        CK(dalloc(&t->om_w, n, t->st)); CK(dalloc(&t->p_w, n, t->st));
        CK(dalloc(&t->code[0], n, t->st)); CK(dalloc(&t->code[1], n, t->st));
        CK(dalloc(&t->excl, n, t->st));
    }
    CK(cudaMemcpyAsync(t->omega_v, omega, n * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(t->p_v, p, n * 8, cudaMemcpyDeviceToDevice, st));
    CK(launch_gather_pos(t->bfs, n, t->flow_v, t->omega_v, t->p_v, t->f_pos, t->om_pos, t->p_pos, st));
    if (extrema) {
        double* out6 = nullptr;
        double* tmp = nullptr;
        unsigned long long* key = nullptr;
        int64_t P = 1;
        while (P < n) P <<= 1;
        CK(aalloc(&out6, 6, st));
        CK(aalloc(&tmp, 2 * (P / 2048 + 2), st));
        CK(aalloc(&key, 3, st));
        CK(launch_extrema(t->flow_v, t->root, t->omega_v, t->p_v, n, out6, tmp, key, st));
        CK(cudaMemcpyAsync(extrema, out6, 6 * 8, cudaMemcpyDeviceToHost, st));
        isoc_free_async(out6, st); isoc_free_async(tmp, st); isoc_free_async(key, st);
        CK(cudaStreamSynchronize(st));
    }
    return ISOC_OK;
}

int isoc_decide(isoc_tree* t, double N, int64_t k, int32_t slot, int64_t* j_host) {
    if (!t->omega_v) return fail(ISOC_EINVAL, "weights not attached");
    if (k < 1) return fail(ISOC_EINVAL, "k must be >= 1, got %lld", (long long)k);
    if (!std::isfinite(N)) return fail(ISOC_EINVAL, "threshold must be finite, got %g", N);
    if (slot < 0 || slot > 1) return fail(ISOC_EINVAL, "slot must be 0 or 1");
    cudaStream_t st = t->st;
    if (t->spars_cap[slot] < k) {
        if (t->spars[slot]) isoc_free_async(t->spars[slot], t->st);
        t->spars[slot] = nullptr;
        CK(dalloc(&t->spars[slot], k, t->st));
        t->spars_cap[slot] = k;
    }
    t->pin = host_stage();
    if (!t->pin) return fail(ISOC_ECUDA, "page-locked staging unavailable");
    CK(launch_decide(t->n, t->levels, t->level_off, t->max_width, t->f_pos, t->om_pos, t->p_pos,
                     t->child_lo, t->child_cnt, N, k, t->om_w, t->p_w, t->code[slot], t->excl,
                     t->spars[slot], t->scratch, t->j_out, st));
    int64_t* pj = static_cast<int64_t*>(t->pin);
    CK(cudaMemcpyAsync(pj, t->j_out, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *j_host = *pj;
    return ISOC_OK;
}

int isoc_tree_shape(isoc_tree* t, int64_t* levels, int64_t* max_width) {
    if (!t) return fail(ISOC_EINVAL, "tree is NULL");
    if (levels) *levels = t->levels;
    if (max_width) *max_width = t->max_width;
    return ISOC_OK;
}

int isoc_decide_batch_capacity(isoc_tree* t, int32_t* cap) {
    if (!t || !cap) return fail(ISOC_EINVAL, "null argument");
    size_t smem = 0;
    *cap = decide_small_fits(t->n, t->levels, &smem) ? DECIDE_SMALL_MAX_BATCH : 16;
    return ISOC_OK;
}

int isoc_decide_batch(isoc_tree* t, const double* thresholds, int32_t count, int64_t k, int64_t* j_host) {
    if (!t->omega_v) return fail(ISOC_EINVAL, "weights not attached");
    if (k < 1) return fail(ISOC_EINVAL, "k must be >= 1, got %lld", (long long)k);
    int32_t cap = 16;
    isoc_decide_batch_capacity(t, &cap);
    if (count < 1 || count > cap) return fail(ISOC_EINVAL, "batch of %d thresholds (1..%d)", count, cap);
    size_t smem_small = 0;
    if (decide_small_fits(t->n, t->levels, &smem_small)) {
        // one warp per threshold in shared memory: only thresholds and counts on the device
        cudaStream_t st = t->st;
        CK(arena(AR_BTHR, &t->bthr, DECIDE_SMALL_MAX_BATCH, st));
        CK(arena(AR_BJ, &t->bj, DECIDE_SMALL_MAX_BATCH, st));
        t->pin = host_stage();
        if (!t->pin) return fail(ISOC_ECUDA, "page-locked staging unavailable");
        double* pthr = static_cast<double*>(t->pin);
        int64_t* pj = reinterpret_cast<int64_t*>(pthr + 64);
        memcpy(pthr, thresholds, (size_t)count * 8);
        CK(cudaMemcpyAsync(t->bthr, pthr, (size_t)count * 8, cudaMemcpyHostToDevice, st));
        CK(launch_decide_batch(t->n, t->levels, t->level_off, t->max_width, t->f_pos, t->om_pos, t->p_pos,
                               t->child_lo, t->child_cnt, t->bthr, count, k, nullptr, nullptr, nullptr,
                               nullptr, nullptr, t->bj, st));
        CK(cudaMemcpyAsync(pj, t->bj, (size_t)count * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        memcpy(j_host, pj, (size_t)count * 8);
        return ISOC_OK;
    }
    for (int i = 0; i < count; ++i)
        if (!std::isfinite(thresholds[i])) return fail(ISOC_EINVAL, "threshold must be finite, got %g", thresholds[i]);
    cudaStream_t st = t->st;
    const int64_t n = t->n;
    CK(arena(AR_BOM, &t->bom, (size_t)count * n, st));
    CK(arena(AR_BP, &t->bp, (size_t)count * n, st));
    CK(arena(AR_BCODE, &t->bcode, (size_t)count * n, st));
    CK(arena(AR_BEXCL, &t->bexcl, (size_t)count * n, st));
    CK(arena(AR_BSCRATCH, &t->bscratch, 16 * 1024 + 8, st));
    CK(arena(AR_BTHR, &t->bthr, DECIDE_SMALL_MAX_BATCH, st));
    CK(arena(AR_BJ, &t->bj, DECIDE_SMALL_MAX_BATCH, st));
    CK(cudaMemcpyAsync(t->bthr, thresholds, (size_t)count * 8, cudaMemcpyHostToDevice, st));
    CK(launch_decide_batch(n, t->levels, t->level_off, t->max_width, t->f_pos, t->om_pos, t->p_pos,
                           t->child_lo, t->child_cnt, t->bthr, count, k, t->bom, t->bp, t->bcode,
                           t->bexcl, t->bscratch, t->bj, st));
    CK(cudaMemcpyAsync(j_host, t->bj, (size_t)count * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return ISOC_OK;
}

int isoc_witness(isoc_tree* t, int32_t slot, int64_t k, int64_t* labels, int8_t* cut, int64_t* eta,
                 double* sparsities, double* miso) {
    const int64_t n = t->n;
    cudaStream_t st = t->st;
    if (slot < 0 || slot > 1 || !t->code[slot]) return fail(ISOC_EINVAL, "no witness in slot %d", slot);
    int8_t* cut_v = nullptr;
    int64_t *eta_v = nullptr, *lab_v = nullptr;
    int32_t *lab32 = nullptr, *work = nullptr;
    double *sums = nullptr, *miso_d = nullptr;
    void* cwork = nullptr;
    const size_t cbytes = cost_work_bytes(n, k);
    CK(arena(AR_CUT, &cut_v, n, st));
    CK(arena(AR_ETA, &eta_v, n, st));
    CK(arena(AR_LAB, &lab_v, n, st));
    CK(arena(AR_LAB32, &lab32, n, st));
    CK(arena(AR_WORK, &work, 4 * n, st));
    CK(arena(AR_SUMS, &sums, 3 * k, st));
    CK(arena(AR_MISO, &miso_d, 1, st));
    CK(arena(AR_CWORK, reinterpret_cast<unsigned char**>(&cwork), cbytes, st));
    CK(launch_labels(t->code[slot], t->pos_parent, t->bfs, n, t->levels, cut_v, eta_v, lab_v, lab32,
                     work, st));
    // the label / cut / eta read-back (copy engine) overlaps the cost kernels
    // (SMs): a side stream waits for the labels, the main stream goes on
    SideStream* ss = nullptr;
    CK(side_stream(&ss));
    cudaStream_t side = ss->s;
    cudaEvent_t ready = ss->ready, copied = ss->copied;
    CK(cudaEventRecord(ready, st));
    CK(cudaStreamWaitEvent(side, ready, 0));
    if (labels) CK(cudaMemcpyAsync(labels, lab_v, n * 8, cudaMemcpyDeviceToHost, side));
    if (cut) CK(cudaMemcpyAsync(cut, cut_v, n, cudaMemcpyDeviceToHost, side));
    if (eta) CK(cudaMemcpyAsync(eta, eta_v, n * 8, cudaMemcpyDeviceToHost, side));
    CK(cudaEventRecord(copied, side));
    CK(launch_cost(lab32, t->parent_v, t->flow_v, t->omega_v, t->p_v, n, k, cwork, cbytes, sums,
                   miso_d, st));
    if (sparsities && t->spars[slot])
        CK(cudaMemcpyAsync(sparsities, t->spars[slot], k * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(miso, miso_d, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamWaitEvent(st, copied, 0));   // the arena buffers are idle once the copies are done
    CK(cudaStreamSynchronize(st));
    return ISOC_OK;
}

__global__ void labels_to_i32_kernel(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int32_t)in[i];
}

int isoc_tree_cost(isoc_tree* t, const int64_t* labels, int64_t k, double* miso) {
    if (!t || !t->omega_v) return fail(ISOC_EINVAL, "weights not attached");
    if (k < 1) return fail(ISOC_EINVAL, "no clusters: labels contain no value >= 1");
    const int64_t n = t->n;
    cudaStream_t st = t->st;
    int32_t* lab32 = nullptr;
    double *sums = nullptr, *miso_d = nullptr;
    void* cwork = nullptr;
    const size_t cbytes = cost_work_bytes(n, k);
    CK(aalloc(&lab32, n, st));
    CK(aalloc(&sums, 3 * k, st));
    CK(aalloc(&miso_d, 1, st));
    CK(isoc_malloc_async(&cwork, cbytes, st));
    labels_to_i32_kernel<<<blocks(n, 256), 256, 0, st>>>(labels, n, lab32);
    CK(launch_cost(lab32, t->parent_v, t->flow_v, t->omega_v, t->p_v, n, k, cwork, cbytes, sums, miso_d, st));
    CK(cudaMemcpyAsync(miso, miso_d, 8, cudaMemcpyDeviceToHost, st));
    isoc_free_async(lab32, st); isoc_free_async(sums, st); isoc_free_async(miso_d, st); isoc_free_async(cwork, st);
    CK(cudaStreamSynchronize(st));
    return ISOC_OK;
}

void isoc_tree_destroy(isoc_tree* t) {
    if (t) cudaStreamSynchronize(t->st);
    tree_free(t);
}

}  // extern "C"
