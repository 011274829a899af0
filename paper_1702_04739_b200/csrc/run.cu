// isoc_run: the whole run_pipeline (/root/reference/pkg/src/isoclust/pipeline.py:41-104)
// behind one C call, for hosts that bind the library without Python.
//
// Same stage order as paper_1702_04739_b200/pipeline.py (the Python host):
// sigma pass (+ exact nearest neighbours) -> Boruvka round 1 -> symmetric
// omega pass (+ round 2) -> filter rounds -> rooting -> extrema -> the
// bisection of run_bisection (isoperim.py:222-308) -> witness labels and the
// exact cost.  One GPU (row range [0, n)); multi-GPU runs go through the
// Python host, which adds the all-reduces between the same calls.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/isoclust_b200.h"
#include "common.cuh"
#include "prof.h"

namespace isoc {
int set_error(int code, const char* fmt, ...);
}

namespace {

__global__ void nonfinite_kernel(const double* X, int64_t m, int32_t* flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(X[i])) *flag = 1;
}

struct DevBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    ~DevBuf() {
        if (p) isoc::isoc_free_async(p, st);
    }
    template <typename T>
    T* get() const { return static_cast<T*>(p); }
};

inline double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

#define RCK(x)                                   \
    do {                                         \
        const int _s = (x);                      \
        if (_s != ISOC_OK) return _s;            \
    } while (0)
#define RCU(x)                                                                                   \
    do {                                                                                         \
        const cudaError_t _e = (x);                                                              \
        if (_e != cudaSuccess) return isoc::set_error(ISOC_ECUDA, "%s", cudaGetErrorString(_e)); \
    } while (0)

int alloc(DevBuf& b, size_t bytes, cudaStream_t st) {
    b.st = st;
    const cudaError_t e = isoc::isoc_malloc_async(&b.p, bytes ? bytes : 1, st);
    if (e != cudaSuccess)
        return isoc::set_error(e == cudaErrorMemoryAllocation ? ISOC_ENOMEM : ISOC_ECUDA, "%s",
                               cudaGetErrorString(e));
    return ISOC_OK;
}

// One Boruvka round on one GPU (the all-reduces of pipeline._boruvka are
// identities): returns the component count.
int one_round(isoc_mst* h, int64_t n, int use_nn, const int32_t* nn_j, const double* nn_d,
              const int8_t* nn_tie, uint64_t* cmin, uint64_t* cedge, int64_t* comps, int64_t* rounds,
              int64_t* ties, int64_t* rescans) {
    RCK(isoc_mst_round_local(h, use_nn, nn_j, nn_d, nn_tie, cmin));
    RCK(isoc_mst_round_edges(h, cmin, cedge));
    int64_t c = 0, t = 0, r = 0;
    RCK(isoc_mst_round_finish(h, cmin, cedge, &c, &t, &r));
    *rounds += 1;
    *ties += t;
    *rescans += r;
    if (c >= *comps)
        return isoc::set_error(ISOC_ECUDA, "Boruvka round %lld made no progress (%lld components)",
                               (long long)*rounds, (long long)c);
    *comps = c;
    (void)n;
    return ISOC_OK;
}

int run_impl(const double* points, int64_t n, int32_t d, int64_t k, double sigma, double alpha,
             int64_t root, cudaStream_t st, isoc_run_out* out) {
    if (!out) return isoc::set_error(ISOC_EINVAL, "out is NULL");
    if (n < 2) return isoc::set_error(ISOC_EINVAL, "need at least 2 points, got %lld", (long long)n);
    if (d < 1) return isoc::set_error(ISOC_EINVAL, "points must have at least one coordinate");
    if (k < 1) return isoc::set_error(ISOC_EINVAL, "k must be >= 1, got %lld", (long long)k);
    if (!(alpha >= 0.0)) return isoc::set_error(ISOC_EINVAL, "alpha must be >= 0, got %g", alpha);
    if (std::isnan(sigma)) return isoc::set_error(ISOC_EINVAL, "sigma must be > 0, got nan");
    const double t_start = now_ms();
    double t0 = t_start;

    // points: a device pointer is used in place, a host pointer is copied
    cudaPointerAttributes pa;
    const bool on_dev = cudaPointerGetAttributes(&pa, points) == cudaSuccess &&
                        pa.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    DevBuf xb, flag;
    const double* X = points;
    if (!on_dev) {
        RCK(alloc(xb, (size_t)n * d * 8, st));
        RCU(cudaMemcpyAsync(xb.p, points, (size_t)n * d * 8, cudaMemcpyHostToDevice, st));
        X = xb.get<double>();
    }
    RCK(alloc(flag, 4, st));
    RCU(cudaMemsetAsync(flag.p, 0, 4, st));
    nonfinite_kernel<<<592, 256, 0, st>>>(X, n * (int64_t)d, flag.get<int32_t>());
    int32_t hflag = 0;
    RCU(cudaMemcpyAsync(&hflag, flag.p, 4, cudaMemcpyDeviceToHost, st));
    RCU(cudaStreamSynchronize(st));
    if (hflag) return isoc::set_error(ISOC_EINVAL, "points must be finite");

    // ---------------------------------------------------------- affinity
    const bool need_pass = !(sigma > 0.0) || alpha > 0.0;
    DevBuf stack, nnj, nnd, nnt, pv;
    RCK(alloc(nnj, (size_t)n * 4, st));
    RCK(alloc(nnd, (size_t)n * 8, st));
    RCK(alloc(nnt, (size_t)n, st));
    RCK(alloc(pv, (size_t)n * 8, st));
    double sig = sigma;
    if (need_pass) {
        RCK(alloc(stack, ISOC_FOLD_STACK_BYTES, st));
        RCK(isoc_sigma_partial(X, n, d, 0, n, alpha, stack.p, nnj.get<int32_t>(), nnd.get<double>(),
                               nnt.get<int8_t>(), pv.get<double>(), st));
        if (!(sigma > 0.0)) {
            double total = 0.0;
            RCK(isoc_sigma_finish(stack.p, 1, &total, st));
            sig = total / (double)(n * (n - 1));   // auto_sigma, affinity.py:233-241
            if (!(sig > 0.0)) return isoc::set_error(ISOC_EINVAL, "all points coincide; no usable distance scale");
        }
    } else {
        RCU(cudaMemsetAsync(pv.p, 0, (size_t)n * 8, st));
    }
    if (!(alpha > 0.0)) RCU(cudaMemsetAsync(pv.p, 0, (size_t)n * 8, st));
    double affinity_ms = now_ms() - t0;

    // --------------------------------------------------------------- MST
    t0 = now_ms();
    if (root < 0 || root >= n)
        return isoc::set_error(ISOC_EINVAL, "root must be in [0, %lld), got %lld", (long long)n, (long long)root);
    isoc_mst* h = nullptr;
    RCK(isoc_mst_create(X, n, d, 0, n, st, &h));
    struct MstGuard {
        isoc_mst* h;
        ~MstGuard() { isoc_mst_destroy(h); }
    } guard{h};
    DevBuf cmin, cedge, om, nn2j, nn2d, nn2t, u, v, w;
    RCK(alloc(cmin, (size_t)n * 8, st));
    RCK(alloc(cedge, (size_t)n * 8, st));
    RCK(alloc(om, (size_t)n * 8, st));
    RCK(alloc(nn2j, (size_t)n * 4, st));
    RCK(alloc(nn2d, (size_t)n * 8, st));
    RCK(alloc(nn2t, (size_t)n, st));
    int64_t comps = n, rounds = 0, ties = 0, rescans = 0;
    if (need_pass)
        RCK(one_round(h, n, 1, nnj.get<int32_t>(), nnd.get<double>(), nnt.get<int8_t>(),
                      cmin.get<uint64_t>(), cedge.get<uint64_t>(), &comps, &rounds, &ties, &rescans));
    const double tw = now_ms();
    RCK(isoc_omega_mst(X, n, d, 0, n, sig, h, om.get<double>(), nn2j.get<int32_t>(), nn2d.get<double>(),
                       nn2t.get<int8_t>(), st));
    RCU(cudaStreamSynchronize(st));
    const double omega_ms = now_ms() - tw;
    if (comps > 1)
        RCK(one_round(h, n, 1, nn2j.get<int32_t>(), nn2d.get<double>(), nn2t.get<int8_t>(),
                      cmin.get<uint64_t>(), cedge.get<uint64_t>(), &comps, &rounds, &ties, &rescans));
    while (comps > 1)
        RCK(one_round(h, n, 0, nullptr, nullptr, nullptr, cmin.get<uint64_t>(), cedge.get<uint64_t>(),
                      &comps, &rounds, &ties, &rescans));
    RCK(alloc(u, (size_t)(n - 1) * 4, st));
    RCK(alloc(v, (size_t)(n - 1) * 4, st));
    RCK(alloc(w, (size_t)(n - 1) * 8, st));
    RCK(isoc_mst_edges(h, u.get<int32_t>(), v.get<int32_t>(), w.get<double>()));
    // prim_mst's tie rule: an exact tie at a component minimum -> replay Prim
    // exactly (isoc_prim_edges); ISOC_MST=prim forces it (pipeline._tie_rule)
    const char* mst_env = std::getenv("ISOC_MST");
    if (ties > 0 || (mst_env && std::strcmp(mst_env, "prim") == 0))
        RCK(isoc_prim_edges(X, n, d, root, u.get<int32_t>(), v.get<int32_t>(), w.get<double>(), st));
    isoc_tree* tree = nullptr;
    RCK(isoc_tree_from_edges(u.get<int32_t>(), v.get<int32_t>(), w.get<double>(), n, root, sig, st, &tree));
    struct TreeGuard {
        isoc_tree* t;
        ~TreeGuard() { isoc_tree_destroy(t); }
    } tguard{tree};
    RCU(cudaStreamSynchronize(st));
    const double mst_ms = now_ms() - t0 - omega_ms;
    affinity_ms += omega_ms;

    t0 = now_ms();
    double ext[6];
    RCK(isoc_tree_set_weights(tree, om.get<double>(), pv.get<double>(), ext));
    affinity_ms += now_ms() - t0;
    const double phi_sum = ext[0], phi_min = ext[1], om_sum = ext[2], om_min = ext[3], p_sum = ext[4],
                 p_min = ext[5];

    // ------------------------------------------------- run_bisection
    t0 = now_ms();
    if (om_sum == 0.0 || om_min == 0.0) return isoc::set_error(ISOC_EINVAL, "float division by zero");
    const double alpha0 = (phi_min + p_min) / om_sum;
    const double beta0 = (phi_sum + p_sum) / om_min;
    int64_t t_budget = 1;
    if (beta0 > alpha0) {
        const double g = 2.0 * om_sum * om_sum * (beta0 - alpha0);
        const double f = phi_min + p_min;
        const double e = (beta0 - alpha0) / (1e-15 * (1.0 > beta0 ? 1.0 : beta0));
        if (!(g > 0.0) || !(f > 0.0) || !(e > 0.0)) return isoc::set_error(ISOC_EINVAL, "math domain error");
        const double t_gap = std::ceil(std::log2(g) - std::log2(f));
        const double t_eps = std::ceil(std::log2(e));
        const double tt = t_gap > t_eps ? t_gap : t_eps;
        t_budget = tt >= 128.0 ? 128 : (tt < 1.0 ? 1 : (int64_t)tt);
    }
    double lo = alpha0, hi = beta0;
    int wslot = -1;
    int64_t wj = 0, iters = 0;
    int32_t tlen = 0;
    auto record = [&](double mid, bool ok) {
        if (tlen < out->trace_cap) {
            if (out->trace_mid) out->trace_mid[tlen] = mid;
            if (out->trace_ok) out->trace_ok[tlen] = ok ? 1 : 0;
        }
        ++tlen;
    };
    auto sweep = [&](double N, bool& ok, int64_t& j, int& slot) -> int {
        slot = wslot < 0 ? 0 : 1 - wslot;
        RCK(isoc_decide(tree, N, k, slot, &j));
        ok = (j == k);
        return ISOC_OK;
    };
    auto stop_test = [](double a, double b) { return b - a <= 1e-15 * (1.0 > b ? 1.0 : b); };
    // speculation depth: as pipeline._speculation_depth (ISOC_SPEC_M overrides)
    int m = 1;
    {
        int64_t levels = 1, width = 0;
        RCK(isoc_tree_shape(tree, &levels, &width));
        int32_t cap = 16;
        RCK(isoc_decide_batch_capacity(tree, &cap));
        const int mmax = cap >= 63 ? 6 : 4;
        m = cap >= 63 ? 6 : ((n <= 64 * 1024 * (levels > 1 ? levels : 1) && width <= 262144) ? 4 : 1);
        if (const char* e = getenv("ISOC_SPEC_M")) {
            m = atoi(e);
            m = m < 1 ? 1 : (m > mmax ? mmax : m);
        }
    }
    if (m <= 1) {
        for (int64_t r = 0; r < t_budget; ++r) {
            if (stop_test(lo, hi)) break;
            const double mid = (lo + hi) / 2.0;
            bool ok;
            int64_t j;
            int slot;
            RCK(sweep(mid, ok, j, slot));
            ++iters;
            record(mid, ok);
            if (ok) {
                hi = mid;
                wslot = slot;
                wj = j;
            } else {
                lo = mid;
            }
        }
    } else {
        // speculative bisection: see pipeline.run_bisection
        bool have_w = false, stop = false;
        double wthr = 0.0;
        while (!stop && iters < t_budget) {
            double thr[64];
            int kid[64][2];
            int cnt = 0;
            const int64_t depth = (m < t_budget - iters) ? m : (t_budget - iters);
            // iterative build in the same preorder as the Python recursion
            struct Frame { double a, b; int depth, parent, side; };
            Frame stk[128];
            int sp = 0;
            stk[sp++] = {lo, hi, (int)depth, -1, 0};
            int root = -1;
            while (sp > 0) {
                const Frame f = stk[--sp];
                int idx = -1;
                if (f.depth > 0 && !stop_test(f.a, f.b)) {
                    const double mid = (f.a + f.b) / 2.0;
                    idx = cnt++;
                    thr[idx] = mid;
                    kid[idx][0] = kid[idx][1] = -1;
                    // push right first so the left subtree is built first (preorder)
                    stk[sp++] = {mid, f.b, f.depth - 1, idx, 1};
                    stk[sp++] = {f.a, mid, f.depth - 1, idx, 0};
                }
                if (f.parent < 0) root = idx;
                else kid[f.parent][f.side] = idx;
            }
            if (root < 0) break;
            int64_t js[64];
            RCK(isoc_decide_batch(tree, thr, cnt, k, js));
            int node = root;
            while (node >= 0) {
                if (stop_test(lo, hi)) {
                    stop = true;
                    break;
                }
                const double mid = thr[node];
                const bool ok = js[node] == k;
                ++iters;
                record(mid, ok);
                if (ok) {
                    hi = mid;
                    wthr = mid;
                    wj = js[node];
                    have_w = true;
                    node = kid[node][0];
                } else {
                    lo = mid;
                    node = kid[node][1];
                }
                if (iters >= t_budget) break;
            }
        }
        if (have_w) {
            int64_t j = 0;
            RCK(isoc_decide(tree, wthr, k, 0, &j));
            if (j != wj) return isoc::set_error(ISOC_ECUDA, "speculative sweep disagrees with the witness sweep");
            wslot = 0;
        }
    }
    if (wslot < 0) {
        bool ok;
        int64_t j;
        int slot;
        RCK(sweep(beta0, ok, j, slot));
        ++iters;
        record(beta0, ok);
        if (!ok) {
            const double bumped = beta0 * (1.0 + 1e-12);
            RCK(sweep(bumped, ok, j, slot));
            ++iters;
            record(bumped, ok);
        }
        if (!ok)
            return isoc::set_error(ISOC_EINFEASIBLE, "no feasible %lld-subpartition found within bracket (n=%lld, k=%lld)",
                                   (long long)k, (long long)n, (long long)k);
        wslot = slot;
        wj = j;
    }
    double miso = 0.0;
    RCK(isoc_witness(tree, wslot, k, out->labels, out->cut, out->eta, out->sparsities, &miso));
    const double partition_ms = now_ms() - t0;

    out->trace_len = tlen;
    out->iterations = iters;
    out->clusters_found = wj;
    out->miso = miso;
    out->sigma = sig;
    out->alpha_final = lo;
    out->beta_final = hi;
    out->timings_ms[0] = affinity_ms;
    out->timings_ms[1] = mst_ms;
    out->timings_ms[2] = partition_ms;
    out->timings_ms[3] = now_ms() - t_start;
    out->boruvka_rounds = rounds;
    out->exact_ties = ties;
    out->exact_rescans = rescans;
    return ISOC_OK;
}

}  // namespace

extern "C" int isoc_run(const double* points, int64_t n, int32_t d, int64_t k, double sigma, double alpha,
                        int64_t root, void* stream, isoc_run_out* out) {
    const int s = run_impl(points, n, d, k, sigma, alpha, root, (cudaStream_t)stream, out);
    isoc::note_launch();
    return s;
}
