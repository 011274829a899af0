"""Benchmark: points clustered/sec end-to-end at N=1M, d=64, k=20 (BASELINE.json).

One step = one full run_pipeline pass (exact sigma pass + Boruvka MST +
rooting + exact omega pass + extrema + bisection + witness labels/cost) over
one synthetic Gaussian-blob data set generated with the reference's
generator semantics (dataset.py:140-168, PCG64 seed 0).

  value  points/s with the points already resident in HBM (device tensor in)
  e2e    points/s through the public drop-in API with HOST numpy points in and
         host labels out (H2D + D2H inside the timed region)

Launch: python bench.py [--gpus N --steps K --warmup W]; for N > 1 under
torch.distributed.run (one process per GPU, rows sharded, NCCL MIN
all-reduce of the Boruvka keys).  --impl reference times the reference's
algorithm (the CPU oracle restatement, all host threads) on a bounded
row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": (2000, 2, 3),
    "c2": (100_000, 16, 10),
    "c3": (1_000_000, 64, 20),
    "c4": (200_000, 512, 50),
}
METRIC = "points clustered/sec end-to-end (N=1M,d=64,k=20) at 1/2/4/8 B200; MST-phase time"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS) + ["c5"])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--d", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-rows", type=int, default=0)
    return ap.parse_args()


def workload(args):
    n, d, k = CONFIGS[args.config]
    n = args.n or n
    d = args.d or d
    k = args.k or k
    return n, d, k


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed
    region by ONE background nvidia-smi process (no forks inside the region)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        import tempfile
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            lines = open(self.path).read().strip().splitlines()
        except Exception:
            lines = []
        for line in lines:
            s = [x.strip() for x in line.split(",")]
            try:
                sm.append(float(s[0]))
                mx = max(mx, float(s[1]))
                for nm, v in zip(names, s[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------- CPU side
def cpu_sample(X: np.ndarray, rows: int, threads: int):
    """Reference algorithm's O(n^2) per-point work on a bounded row sample.

    For `rows` points the CPU oracle (isoc_oracle.c, the reference's exact
    operation order) computes each point's full distance row (scipy order)
    and its full omega row (glibc exp + pow2 fold) -- the per-point work of
    distance_matrix/auto_sigma, prim_mst's relaxation and vertex_weights.
    Returns seconds for the sample; points/s = rows / seconds.
    """
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    orc.lib().oc_set_threads(threads)
    n = X.shape[0]
    t0 = time.perf_counter()
    orc.distance_rows(X, 0, rows)          # sigma / Prim rows
    orc.row_folds(X, 1.0, 0.0, 0, rows)    # omega rows
    return time.perf_counter() - t0


def pkg_generate_random(n, d, k, seed):
    """The package's generate_random (dataset.py:140-168 semantics)."""
    from paper_1702_04739_b200 import generate_random
    return generate_random(n, d, k, seed)


def synthetic_tree(n: int, seed: int):
    """C5 input: random recursive tree drawn vectorised as
    parent[perm[i]] = perm[floor(U_i * i)], flows 1-U[0,1), omega 2-U[0,1.9),
    p = 0 (the reference's tests/conftest.py:35-70 distributions)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    parent = np.full(n, -1, dtype=np.int64)
    perm = rng.permutation(n)
    if n > 1:
        i = np.arange(1, n, dtype=np.int64)
        parent[perm[1:]] = perm[np.minimum((rng.random(n - 1) * i).astype(np.int64), i - 1)]
    flows = np.zeros(n, dtype=np.float64)
    nonroot = parent != -1
    flows[nonroot] = 1.0 - rng.uniform(0.0, 1.0, int(nonroot.sum()))
    omega = 2.0 - rng.uniform(0.0, 1.9, n)
    return parent, flows, omega, np.zeros(n, dtype=np.float64)


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n, d, k = workload(args)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    orc.build()
    X, _ = orc.generate_random(n, d, k, 0)
    threads = os.cpu_count() or 1
    rows = args.cpu_sample_rows or max(8, int(2.0e9 / (n * max(d, 8))))
    rows = min(rows, n)
    for _ in range(max(0, args.warmup)):
        cpu_sample(X, max(1, rows // 8), threads)
    times = [cpu_sample(X, rows, threads) for _ in range(max(1, args.steps))]
    sec = statistics.median(times)
    val = rows / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3 * n / rows,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generate_random PCG64 seed 0)",
        "config": {"workload": f"c3-shaped blobs N={n} d={d} k={k}", "n": n, "d": d, "k": k},
        "cpu_baseline": {"value": val, "unit": "points/s", "cores": threads, "kind": "port",
                         "sample": f"{rows} of {n} points: exact distance row + omega row each "
                                   f"(oracle/isoc_oracle.c, OpenMP {threads} threads); "
                                   "extrapolated per point"},
        "e2e": {"value": val, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU side
KIND_NAMES = ["sigma_pass", "omega_pass", "boruvka_filter", "decide", "rescan", "bfs", "cost"]


def tree_phase_bench(args):
    """C5: tree phase only on a 50M-vertex random recursive tree, k = 100
    (tree_from_parent_list + extrema + par_solve_miso), vertices/s."""
    import torch
    import paper_1702_04739_b200 as pkg

    n = args.n or 50_000_000
    k = args.k or 100
    parent, flows, omega, p = synthetic_tree(n, 0)
    w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=0.0)

    def step():
        tree = pkg.tree_from_parent_list(parent, flows)
        ext = pkg.extrema(tree, w)
        return pkg.par_solve_miso(tree, w, ext, k)

    from paper_1702_04739_b200 import _lib
    import ctypes

    lib = _lib.load()
    lib.isoc_prof_read.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_longlong)]
    lib.isoc_launch_count.restype = ctypes.c_longlong
    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    sampler.start()
    lib.isoc_prof_enable(1)
    l0 = lib.isoc_launch_count()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = step()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    launches = lib.isoc_launch_count() - l0
    clocks = sampler.stop()
    kernels = {}
    for kind, name in enumerate(KIND_NAMES):
        tot = ctypes.c_double()
        cnt = ctypes.c_longlong()
        if lib.isoc_prof_read(kind, ctypes.byref(tot), ctypes.byref(cnt)) == 0 and cnt.value:
            kernels[name] = {"ms_total": tot.value / args.steps, "launches": cnt.value / args.steps}
    lib.isoc_prof_enable(0)
    # HBM roofline of the decision sweep (~45 algorithmic bytes
    # per vertex per sweep: f, omega, p in, parent / child ranges, codes and
    # the parents' folded omega / p out)
    roofline = None
    if "decide" in kernels:
        per_ms = kernels["decide"]["ms_total"] / max(1.0, kernels["decide"]["launches"])
        achieved = 45.0 * n / (per_ms * 1e-3) / 1e9
        peak = float(peaks().get("hbm_gbs") or 6536.4)
        roofline = {"kernel": "decide", "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": 1.721e9,
                    "traffic_unit": "bytes per launch (mean over the 78 sweeps of one step)",
                    "traffic_source": "profiles/round1_ncu_launches_decide_c5.csv (dram__bytes_read.sum + "
                                      "dram__bytes_write.sum per decide_kernel launch; mean 0.91 ms, 1.90 TB/s)",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "note": "algorithmic 45 B/vertex x n per sweep (SURVEY 8(d)); sweeps stop at the k-th cut, "
                            "so the measured DRAM traffic is lower; level-synchronous (grid barriers per level), "
                            "latency rather than bandwidth bounds it"}
    # CPU baseline: the oracle's tree phase (reference operation order) on a
    # 1M-vertex tree of the same generator, per vertex
    cpu = None
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as orc

        m = 1_000_000
        cp, cf, co, cpp = synthetic_tree(m, 0)
        t1 = time.perf_counter()
        orc.solve_tree(cp, cf, co, cpp, k)
        cs = time.perf_counter() - t1
        cpu = {"value": m / cs, "unit": "vertices/s", "cores": 1, "kind": "port",
               "sample": f"{m}-vertex random recursive tree (same generator), tree_from_parent_list + extrema "
                         "+ bisection in oracle/isoc_oracle.c (single thread)"}
    print(json.dumps({
        "metric": "tree-phase vertices/sec (C5: random spanning tree, 50M vertices, k=100)",
        "value": n * args.steps / el, "unit": "vertices/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic random recursive tree (PCG64 seed 0), flows 1-U, omega 2-1.9U, p=0",
        "config": {"workload": f"c5 tree phase N={n} k={k}", "n": n, "k": k},
        "iterations": res.iterations, "miso": res.miso, "kernels": kernels, "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": n * args.steps / el, "unit": "vertices/s",
                "h2d_bytes_per_step": n * 24, "d2h_bytes_per_step": n * 17},
        "gpu_launches": int(launches), "clocks": clocks}), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    if args.config == "c5":
        return tree_phase_bench(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1702_04739_b200 as pkg
    from paper_1702_04739_b200 import _lib
    from paper_1702_04739_b200 import pipeline as pl
    import ctypes

    lib = _lib.load()
    lib.isoc_launch_count.restype = ctypes.c_longlong
    lib.isoc_prof_read.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_longlong)]
    lib.isoc_peak_tflops.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]

    n, d, k = workload(args)
    X, _ = pkg_generate_random(n, d, k, 0)
    X = np.ascontiguousarray(X)
    Xdev = torch.from_numpy(X).pin_memory().cuda()
    torch.cuda.synchronize()

    def step_device():
        return pl.run_pipeline(Xdev, k)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up (also JIT-free: the library is prebuilt)
    for _ in range(args.warmup):
        run = step_device()
    barrier()

    # ---- timed region: device-resident input
    sampler = ClockSampler(local)
    sampler.start()
    lib.isoc_prof_enable(1)
    l0 = lib.isoc_launch_count()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    mst_ms = []
    for _ in range(args.steps):
        run = step_device()
        mst_ms.append(run.timings_ms["mst"])
    ev1.record()
    barrier()
    launches = lib.isoc_launch_count() - l0
    elapsed = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    clocks = sampler.stop()
    kernels = {}
    for kind, name in enumerate(KIND_NAMES):
        tot = ctypes.c_double()
        cnt = ctypes.c_longlong()
        if lib.isoc_prof_read(kind, ctypes.byref(tot), ctypes.byref(cnt)) == 0 and cnt.value:
            kernels[name] = {"ms_total": tot.value / args.steps, "launches": cnt.value / args.steps}
    lib.isoc_prof_enable(0)
    value = n * args.steps / elapsed

    # ---- e2e: host numpy in, host labels out, through the public API
    barrier()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        run_h = pkg.run_pipeline(X, k)
    e1.record()
    barrier()
    e2e_s = max_over_ranks(max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0))
    e2e_value = n * args.e2e_steps / e2e_s
    assert np.array_equal(run_h.result.labels, run.result.labels)
    h2d = X.nbytes
    d2h = 8 * n + n + 8 * n + 8 * k + 64   # labels, cut, eta, sparsities, scalars

    # ---- roofline of the dominant kernel
    fp32_peak = ctypes.c_double()
    fp64_peak = ctypes.c_double()
    lib.isoc_peak_tflops(0, ctypes.byref(fp32_peak))
    lib.isoc_peak_tflops(1, ctypes.byref(fp64_peak))
    rounds = run.mst_stats.get("boruvka_rounds", 0)
    # algorithmic flops per launch (per-unit 3*d fp64 flops): the
    # exact passes' unit is the UNORDERED pair, n(n-1)/2 of them split over the
    # ranks -- d_ij and d_ji are bitwise equal (x_i - x_j = -(x_j - x_i) exactly,
    # so the squares match), so one evaluation is the algorithm's minimum work;
    # SURVEY's ordered-pair view (n^2) is reported beside it. The filter: 2*d
    # per ordered pair it scans
    use_tc = d <= 512 and os.environ.get("ISOC_FILTER", "") != "ffma"
    unordered = n * (n - 1) / 2.0 / max(1, world)
    alg = {
        "sigma_pass": 3.0 * d * unordered,
        "omega_pass": 3.0 * d * unordered,
        # tcgen05 filter: 3 FP16 MMA passes (hi.hi, hi.lo, lo.hi) over K = 64 per atom per pair
        "boruvka_filter": (3 * 2.0 * 64 * ((d + 63) // 64) if use_tc else 2.0 * d) * n * n,
    }
    # the exact passes' fp64 ops cannot fuse (scipy's separately rounded
    # mul/add), so their ceiling is the DADD/DMUL issue rate = half the
    # measured DFMA flop rate
    fp64_op_peak = fp64_peak.value / 2.0
    # pairs the exact passes actually evaluate (one GPU: symmetric super-tiles
    # of 1024; sigma adds 128-wide leaf strips beyond each super-block)
    executed_pairs = {}
    if world == 1:
        # sigma: 2048-wide super-blocks of 16 x 16 tiles of 128 (+ a strip of 16
        # tiles per direction); omega: 1024-wide super-blocks, no strip
        sb, nt = 2048, 16
        nbs = -(-n // sb)
        tiles = 0
        for J in range(nbs):
            ext = 1 if J + 1 < nbs else 0
            tiles += J * (nt * nt + nt * ext + nt) + (nt * nt + nt * ext) if n >= 2048 else 0
        if n >= 2048:
            executed_pairs["sigma_pass"] = tiles * 128 * 128
        nbo = -(-n // 1024)
        executed_pairs["omega_pass"] = nbo * (nbo + 1) // 2 * 1024 * 1024
    tensor_peak = float(peaks().get("bf16_tflops") or 1590.0)   # fp16 dense = bf16 dense rate
    peak_for = {"sigma_pass": fp64_op_peak, "omega_pass": fp64_op_peak,
                "boruvka_filter": tensor_peak if use_tc else fp32_peak.value}
    dom = max(kernels, key=lambda kk: kernels[kk]["ms_total"]) if kernels else None
    roofline = None
    if dom in alg:
        per_launch_ms = kernels[dom]["ms_total"] / max(1.0, kernels[dom]["launches"])
        achieved = alg[dom] / (per_launch_ms * 1e-3) / 1e12
        roofline = {"kernel": dom,
                    "bound": ("tensor" if use_tc else "fp32") if dom == "boruvka_filter" else "fp64",
                    "achieved": achieved, "peak": peak_for[dom], "unit": "TFLOP/s",
                    "frac": achieved / peak_for[dom], "traffic": None,
                    "peak_source": (("MEASURED_PEAKS.json bf16_tflops (burst)" if use_tc else
                                     "measured FFMA microkernel (isoc_peak_tflops), this GPU")
                                    if dom == "boruvka_filter" else
                                    "measured DFMA microkernel / 2 (non-fusable DADD/DMUL issue "
                                    "rate), this GPU")}
        for kk, v in kernels.items():
            if kk in alg:
                pl_ms = v["ms_total"] / max(1.0, v["launches"])
                v["achieved_tflops"] = alg[kk] / (pl_ms * 1e-3) / 1e12
                v["frac_of_peak"] = v["achieved_tflops"] / peak_for[kk]
                if kk in ("sigma_pass", "omega_pass"):
                    v["ordered_pairs_view_tflops"] = 3.0 * d * n * n / max(1, world) / (pl_ms * 1e-3) / 1e12
                if kk in executed_pairs:
                    ex = 3.0 * d * executed_pairs[kk] / (pl_ms * 1e-3) / 1e12
                    v["executed"] = {"pairs": executed_pairs[kk], "tflops": ex,
                                     "frac_of_peak": ex / peak_for[kk]}
        # DRAM bytes per launch of the dominant kernel from the committed ncu
        # launch list of the same configuration (bench.py cannot run ncu itself)
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic_c3.json")))
            if tr.get("config") == f"c3 N={n} d={d} k={k}" and dom in tr:
                roofline["traffic"] = tr[dom]
                roofline["traffic_unit"] = "bytes per launch"
                roofline["traffic_source"] = tr["source"]
        except Exception:
            pass
        if dom in executed_pairs:
            roofline["executed"] = kernels[dom]["executed"]
            roofline["note"] = ("algorithmic = 3*d fp64 flops x n(n-1)/2 unordered pairs (d_ij == d_ji "
                                "bitwise, so one evaluation per pair is the minimum work); 'executed' adds "
                                "the pairs the tiling really evaluates (diagonal tiles, 128-column leaf "
                                "strip) -- the FP64 pipe's view; SURVEY 8(d)'s ordered-pair count (n^2) "
                                "would read 2x 'achieved'")

    if roofline is None and dom == "decide":
        # tiny inputs (C1): the tree phase dominates; HBM roofline of the
        # decision sweeps with the sequential-equivalent algorithmic bytes
        # (45 B per vertex per bisection step)
        steps_walked = max(1, int(run.result.iterations))
        achieved = 45.0 * n * steps_walked / (kernels["decide"]["ms_total"] * 1e-3) / 1e9
        peak = float(peaks().get("hbm_gbs") or 7700.0)
        roofline = {"kernel": "decide", "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "note": "level-synchronous sweeps over a narrow MST tree (hundreds of levels of a few "
                            "vertices): latency-bound, not bandwidth-bound; algorithmic bytes = 45 B x n per "
                            "bisection step walked"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rows = args.cpu_sample_rows or max(8, int(2.0e9 / (n * max(d, 8))))
        rows = min(rows, n)
        sec = cpu_sample(X, rows, threads)
        cpu = {"value": rows / sec, "unit": "points/s", "cores": threads, "kind": "port",
               "sample": f"{rows} of {n} points: exact distance row + omega row each "
                         f"(oracle/isoc_oracle.c, OpenMP {threads} threads); extrapolated per point"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_random PCG64 seed 0, Gaussian blobs)",
            "config": {"workload": f"c3 blobs N={n} d={d} k={k}" if args.config == "c3"
                       else f"{args.config} blobs N={n} d={d} k={k}",
                       "n": n, "d": d, "k": k, "parallelism": (f"symmetric super-tile ranges x{world} (rows owned per rank)" if world > 1 else "one GPU, symmetric super-tiles"),
                       "l2": "inputs larger than L2 (N*d*8 bytes) and an n^2 stream per step"},
            "mst_phase_ms": statistics.median(mst_ms) if mst_ms else None,
            "stage_ms": {kk: round(v, 2) for kk, v in run.timings_ms.items()},
            "mst_stats": run.mst_stats,
            "kernels": kernels,
            "roofline": roofline,
            "peaks_measured_tflops": {"fp32_ffma": fp32_peak.value, "fp64_dfma": fp64_peak.value,
                                      "tensor_bf16_file": tensor_peak,
                                      "hbm_gbs_file": peaks().get("hbm_gbs")},
            "filter": "tcgen05 3xFP16 split" if use_tc else "FP32 FFMA",
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
