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
all-reduce of the Boruvka keys).  `--gpus N` without WORLD_SIZE re-launches
itself under torch.distributed.run with N ranks (NCCL_DEBUG=INFO, INIT).

--impl reference times the reference's algorithm -- the CPU oracle port
(oracle/: scipy-order distances, numpy pairwise sigma, Prim, pow2 omega
folds, the bisection), all host threads -- on the same workload: directly
when N <= 46,340 (the reference's own dense cap), else on a measured ladder
N in {16,000, 32,000, 46,340} at the config's d with each phase fitted
(N^2: sigma, Prim, omega; N: partition) and extrapolated to N.

After the timed region the GPU result is compared bit for bit with the
committed oracle fixture of the config (tests/golden/full_<config>.json,
tools/oracle_full.py): "parity" in the JSON line.
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
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="end-to-end steps (default: as many as fit ~10 s, at most --steps, at least 1)")
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
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML (pynvml) polled from a background thread every 20 ms -- short timed
    regions (C1: a few ms per step) still get samples -- with one sample
    taken at start(); if NVML is unavailable, one background nvidia-smi
    process sampling every 200 ms (no forks inside the region)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None
        self.thread = None
        self.samples = []
        self.reasons = set()
        self.max_mhz = 0.0

    def _nvml_sample(self, nv, h):
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        for name, attr in self.REASONS:
            if bits & getattr(nv, attr, 0):
                self.reasons.add(name)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = [x.strip() for x in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if x.strip()]
            dev = self.index
            if self.index < len(vis) and vis[self.index].isdigit():
                dev = int(vis[self.index])   # NVML counts physical devices
            h = nv.nvmlDeviceGetHandleByIndex(dev)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._stop = threading.Event()
            self._nvml_sample(nv, h)

            def run():
                while not self._stop.wait(0.02):
                    self._nvml_sample(nv, h)
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
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
        if self.thread is not None:
            self._stop.set()
            self.thread.join(timeout=2)
            sm = self.samples
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz or None,
                    "reasons": sorted(self.reasons), "samples": len(sm), "source": "nvml 20 ms"}
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
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 200 ms"}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------- CPU side
LADDER = (16_000, 32_000, 46_340)   # up to the reference's dense cap (affinity.py:139-143)
PHASES_N2 = ("sigma", "prim", "omega")


def oracle_pipeline_timed(orc, X: np.ndarray, k: int) -> dict:
    """One run of the reference pipeline's algorithm on the host (the oracle
    port, pipeline.py:41-104 stage order), per-phase wall seconds:
    sigma = distance sum in scipy/numpy order (affinity.py:124-158, 233-241),
    prim = Prim with the reference's tie rule + flows + BFS (mst.py:128-181),
    omega = vertex_weights (affinity.py:175-201), partition = extrema +
    bisection + labels + cost (isoperim.py:222-308)."""
    t = {}
    t0 = time.perf_counter()
    sig = orc.auto_sigma_fast(X)
    t["sigma"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    tree = orc.prim_mst(X, sig, 0)
    t["prim"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    omega, _, _ = orc.omega_knn(X, sig, 1)
    t["omega"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    p = np.zeros(X.shape[0])
    orc.run_bisection(tree, omega, p, orc.extrema(tree, omega, p), k)
    t["partition"] = time.perf_counter() - t0
    t["total"] = sum(t.values())
    return t


def fit_ladder(points: list, n: int) -> dict:
    """Least-squares through the origin per phase: N^2 phases c = sum(t N^2) /
    sum(N^4); the partition c = sum(t N) / sum(N^2).  Returns the
    coefficients and the extrapolated per-phase seconds at n."""
    fit, extra = {}, {}
    for ph in PHASES_N2 + ("partition",):
        pw = 2 if ph in PHASES_N2 else 1
        num = sum(pt[ph] * pt["n"] ** pw for pt in points)
        den = sum(pt["n"] ** (2 * pw) for pt in points)
        fit[ph] = num / den
        extra[ph] = fit[ph] * n ** pw
    return {"coef_s_per_Npow": fit, "extrapolated_s": extra, "total_s": sum(extra.values())}


def cpu_reference(n: int, d: int, k: int, sizes, reps: int, threads: int, warmup: int = 1) -> dict:
    """Time the oracle port of the reference path on the host.  N <= 46,340:
    the workload itself, `reps` times (median).  Larger N: the ladder `sizes`
    at the same d and k, then the per-phase fit extrapolated to N."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    orc.build()
    orc.lib().oc_set_threads(threads)
    Xw, _ = orc.generate_random(min(n, 4000), d, k, 1)
    for _ in range(max(0, warmup)):
        oracle_pipeline_timed(orc, Xw, k)
    if n <= LADDER[-1]:
        X, _ = orc.generate_random(n, d, k, 0)
        runs = [oracle_pipeline_timed(orc, X, k) for _ in range(max(1, reps))]
        tot = statistics.median(r["total"] for r in runs)
        return {"seconds": tot, "direct": True, "runs": [round(r["total"], 4) for r in runs],
                "phases_s": {ph: round(statistics.median(r[ph] for r in runs), 4)
                             for ph in PHASES_N2 + ("partition",)},
                "sample": f"the whole workload (N={n}) run directly, median of {len(runs)}"}
    points = []
    for m in sizes:
        X, _ = orc.generate_random(m, d, k, 0)
        t = oracle_pipeline_timed(orc, X, k)
        t["n"] = m
        points.append(t)
    fit = fit_ladder(points, n)
    return {"seconds": fit["total_s"], "direct": False,
            "ladder": [{kk: (round(v, 4) if isinstance(v, float) else v) for kk, v in pt.items()}
                       for pt in points],
            "fit": {"model": "N^2 for sigma, Prim, omega; N for the partition (least squares)",
                    "coef_s_per_Npow": fit["coef_s_per_Npow"],
                    "extrapolated_s": {kk: round(v, 2) for kk, v in fit["extrapolated_s"].items()}},
            "sample": f"oracle port of the whole reference pipeline at N in {list(sizes)} (d={d}, k={k}), "
                      f"phases fitted and extrapolated to N={n}"}


def cpu_tree_reference(n: int, k: int, sizes) -> dict:
    """C5 host baseline: the oracle's tree phase (tree_from_parent_list +
    extrema + bisection; reference decide is sequential, isoperim.py:82-144)
    on a ladder of the same generator, fitted linearly in N."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc

    orc.build()
    pts = []
    for m in sizes:
        parent, flows, omega, p = orc.random_tree_instance(m, 0)
        t0 = time.perf_counter()
        orc.solve_tree(parent, flows, omega, p, k)
        pts.append({"n": m, "seconds": time.perf_counter() - t0})
    c = sum(q["seconds"] * q["n"] for q in pts) / sum(q["n"] ** 2 for q in pts)
    return {"seconds": c * n, "ladder": [{"n": q["n"], "seconds": round(q["seconds"], 3)} for q in pts],
            "fit": {"model": "linear in N", "coef_s_per_vertex": c},
            "sample": f"oracle tree phase at N in {list(sizes)} (same generator, k={k}), fitted linearly "
                      f"and extrapolated to N={n}; single thread (the reference decide is sequential)"}


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


def workload_label(args, n, d, k) -> str:
    if args.config == "c5":
        return f"c5 tree phase N={n} k={k}"
    return f"{args.config} blobs N={n} d={d} k={k}"


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    print(f"bench reference arm: rank {rank}/{world}", file=sys.stderr, flush=True)
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if args.config == "c5":
        n = args.n or 50_000_000
        k = args.k or 100
        ref = cpu_tree_reference(n, k, (1_000_000, 2_000_000, 4_000_000))
        metric, unit, cores = "tree-phase vertices/sec (C5: random spanning tree, 50M vertices, k=100)", \
            "vertices/s", 1
        config = {"workload": workload_label(args, n, 0, k), "n": n, "k": k}
    else:
        n, d, k = workload(args)
        ref = cpu_reference(n, d, k, LADDER, max(1, args.steps), threads, args.warmup)
        metric, unit, cores = METRIC, "points/s", threads
        config = {"workload": workload_label(args, n, d, k), "n": n, "d": d, "k": k}
    val = n / ref["seconds"]
    line = {
        "impl": "reference", "metric": metric, "value": val, "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ref["seconds"] * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generate_random PCG64 seed 0)" if args.config != "c5" else
                "synthetic random recursive tree (PCG64 seed 0)",
        "config": config,
        "cpu_baseline": {"value": val, "unit": unit, "cores": cores, "kind": "port",
                         "sample": ref["sample"], **{kk: v for kk, v in ref.items()
                                                     if kk in ("ladder", "fit", "runs", "phases_s")}},
        "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU side
KIND_NAMES = ["sigma_pass", "omega_pass", "boruvka_filter", "decide", "rescan", "bfs", "cost"]


def pinned_copy(a):
    """The e2e contract's inputs live in page-locked host memory: a pinned
    numpy array with a's contents (the library copies it straight to HBM)."""
    import torch
    a = np.ascontiguousarray(a)
    out = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True).numpy()
    np.copyto(out, a)
    return out


def tree_phase_bench(args):
    """C5: tree phase only on a 50M-vertex random recursive tree, k = 100
    (tree_from_parent_list + extrema + par_solve_miso), vertices/s."""
    import torch
    import paper_1702_04739_b200 as pkg

    n = args.n or 50_000_000
    k = args.k or 100
    parent, flows, omega, p = (pinned_copy(a) for a in synthetic_tree(n, 0))
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
                    "traffic_source": "profiles/round2_ncu_launches_decide_c5.csv (dram__bytes_read.sum + "
                                      "dram__bytes_write.sum per decide_kernel launch, 156 launches = 2 steps; "
                                      "mean 0.914 ms, 1.72 GB, 1.88 TB/s)",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "note": "algorithmic 45 B/vertex x n per sweep (SURVEY 8(d)); sweeps stop at the k-th cut, "
                            "so the measured DRAM traffic is lower; level-synchronous (grid barriers per level), "
                            "latency rather than bandwidth bounds it"}
    # CPU baseline: the oracle's tree phase (reference operation order) on a
    # ladder of trees of the same generator, fitted linearly in N
    cpu = None
    if not args.no_cpu_baseline:
        ref = cpu_tree_reference(n, k, (500_000, 1_000_000, 2_000_000))
        cpu = {"value": n / ref["seconds"], "unit": "vertices/s", "cores": 1, "kind": "port",
               "sample": ref["sample"], "ladder": ref["ladder"], "fit": ref["fit"]}
    tree = pkg.tree_from_parent_list(parent, flows)
    ext = pkg.extrema(tree, w)
    res = pkg.par_solve_miso(tree, w, ext, k)
    parity = fixture_parity("c5", n, 0, k, None, (res, tree, omega, ext))
    print(json.dumps({
        "metric": "tree-phase vertices/sec (C5: random spanning tree, 50M vertices, k=100)",
        "value": n * args.steps / el, "unit": "vertices/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic random recursive tree (PCG64 seed 0), flows 1-U, omega 2-1.9U, p=0",
        "config": {"workload": workload_label(args, n, 0, k), "n": n, "k": k},
        "iterations": res.iterations, "miso": res.miso, "kernels": kernels, "roofline": roofline,
        "cpu_baseline": cpu, "parity": parity,
        "e2e": {"value": n * args.steps / el, "unit": "vertices/s",
                "h2d_bytes_per_step": n * 24, "d2h_bytes_per_step": n * 17},
        "gpu_launches": int(launches), "clocks": clocks}), flush=True)


def fixture_parity(config: str, n: int, d: int, k: int, run, tree_res=None) -> dict:
    """Bitwise comparison with the committed oracle fixture of this config
    (tests/golden/full_<config>.json; tools/oracle_full.py), outside the
    timed region.  Points configs compare sigma, the tree arrays and MST
    edge set, omega, extrema, labels, cut, eta, sparsities, trace,
    iterations, alpha/beta and miso."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import digest as dg
    path = os.path.join(ROOT, "tests", "golden", f"full_{config}.json")
    if not os.path.exists(path):
        return {"status": "no-fixture", "fixture": os.path.relpath(path, ROOT)}
    want = dg.load(path)
    m = want["meta"]
    if m.get("n") != n or m.get("k") != k or (config != "c5" and m.get("d") != d):
        return {"status": "no-fixture", "fixture": os.path.relpath(path, ROOT), "why": "different n/d/k"}
    if config == "c5":
        res, tree, omega, ext = tree_res
        got = dg.result_digest(res, tree=tree, omega=omega,
                               extrema=[ext.phi_star_sum, ext.phi_star_min, ext.omega_star_sum,
                                        ext.omega_star_min, ext.p_star_sum, ext.p_star_min])
    else:
        e = run.extrema
        got = dg.result_digest(run.result, sigma=run.sigma, tree=run.tree, omega=run.omega_host(),
                               p=run.p_host(),
                               extrema=[e.phi_star_sum, e.phi_star_min, e.omega_star_sum, e.omega_star_min,
                                        e.p_star_sum, e.p_star_min])
    keys = [kk for kk in want if kk in got and kk != "meta"]
    bad = dg.compare(got, want, keys)
    return {"status": "fixture-match" if not bad else "MISMATCH", "fields_compared": len(keys),
            "differs": bad, "fixture": os.path.relpath(path, ROOT)}


def self_launch(args) -> bool:
    """--gpus N > 1 without a torch.distributed environment: re-run this
    command under torch.distributed.run with N ranks on this node."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
               NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    print("bench: self-launch " + " ".join(cmd), file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd, env=env))


def main():
    args = parse()
    self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; launch with torchrun "
                 f"--nproc-per-node {args.gpus} or without WORLD_SIZE")
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
    X = pinned_copy(X)
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

    # ---- e2e: host numpy in, host labels out, through the public API; short
    # steps are repeated (a single 0.1 s step would carry any one-off host
    # stall of the driver at full weight)
    e2e_steps = args.e2e_steps or max(1, min(args.steps, int(10.0 / max(elapsed / args.steps, 1e-3))))
    barrier()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(e2e_steps):
        run_h = pkg.run_pipeline(X, k)
    e1.record()
    barrier()
    e2e_s = max_over_ranks(max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0))
    e2e_value = n * e2e_steps / e2e_s
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
        # tcgen05 filter: 3 FP16 MMA passes (hi.hi, hi.lo, lo.hi) over K = 64 per atom per
        # (row, column) pair it scans; with the candidate lists later launches scan only
        # the refreshed rows, so the per-launch figure is the step's rows scanned x n
        # spread over its launches (the kernel line below divides by launches)
        "boruvka_filter": (3 * 2.0 * 64 * ((d + 63) // 64) if use_tc else 2.0 * d) * n *
                          (256.0 * run.mst_stats.get("filter_blocks_run", 0)
                           / max(1.0, kernels.get("boruvka_filter", {}).get("launches", 1.0))
                           if use_tc and run.mst_stats.get("filter_blocks_run") else n),
    }
    # the exact passes' fp64 ops cannot fuse (scipy's separately rounded
    # mul/add), so their ceiling is the DADD/DMUL issue rate = half the
    # measured DFMA flop rate
    fp64_op_peak = fp64_peak.value / 2.0
    # pairs the exact passes actually evaluate (one GPU: symmetric super-tiles;
    # sigma computes a 128-column leaf strip only for the row chains of each
    # wave's last column block -- every other straddling leaf is finished by
    # the merge from dumped distances)
    executed_pairs = {}
    if world == 1:
        # sigma: 2048-wide super-blocks of 16 x 16 tiles of 128, waves planned
        # as launch_sigma_sym_range does (64 GB of 1364-byte slots, >= 8
        # blocks); omega: 1024-wide super-blocks, no strip
        sb, nt = 2048, 16
        nbs = -(-n // sb)
        if n >= 2048:
            budget = (64 << 30) // (32 * 8 + 20 + 136 * 8)
            last = set()
            w0 = 0
            while w0 < nbs:
                yg = 8
                while w0 + yg < nbs and (yg + 1) * (n + sb * (w0 + yg + 1)) <= budget:
                    yg += 1
                w1 = min(w0 + yg, nbs)
                last.add(w1 - 1)
                w0 = w1
            tiles = sum((J + 1) * nt * (nt + (1 if (J in last and J + 1 < nbs) else 0)) for J in range(nbs))
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
            tr = json.load(open(os.path.join(ROOT, "profiles", "round2_traffic_c3.json")))
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
                                "the pairs the tiling really evaluates (diagonal tiles, the 128-column "
                                "leaf strip of each wave's last block) -- the FP64 pipe's view; SURVEY 8(d)'s ordered-pair count (n^2) "
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
        # bounded sample (~10-30 s of host work): the oracle port of the whole
        # reference pipeline on the ladder N = 16,000 / 32,000 / 46,340 (or the
        # workload itself when smaller), per phase, extrapolated with the
        # N^2 / N phase model -- the same measurement as --impl reference
        threads = os.cpu_count() or 1
        ref = cpu_reference(n, d, k, LADDER, 1, threads, 0)
        cpu = {"value": n / ref["seconds"], "unit": "points/s", "cores": threads, "kind": "port",
               "sample": ref["sample"], **{kk: v for kk, v in ref.items() if kk in ("ladder", "fit", "phases_s")}}

    parity = fixture_parity(args.config, n, d, k, run)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generate_random PCG64 seed 0, Gaussian blobs)",
            "config": {"workload": workload_label(args, n, d, k),
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
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "last_step_stage_ms": {kk: round(v, 2) for kk, v in run_h.timings_ms.items()}},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
