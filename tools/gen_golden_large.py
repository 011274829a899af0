"""Reference runs at the sizes SURVEY.md §7 step 1 asks the oracle to be pinned
at: the whole reference pipeline (its own stage functions, in run_pipeline's
order, src/pipeline.py:41-104) at N = 16,000 / 32,000 / 46,340 (the dense cap,
src/affinity.py:139-143), stored as compact digests (tests/digest.py) plus
the parent array and labels.  Also records the reference's per-stage wall
times on this container (8 cores, engine="par") for the CPU-baseline ladder.

Run in this container only (imports /root/reference):
    python tools/gen_golden_large.py [name ...]
Re-executes itself in numpy's pinned mode so np.exp
is glibc exp.  Writes tests/golden/large_<name>.json and .npz.
"""
from __future__ import annotations

import os
import subprocess
import sys
import time
from pathlib import Path

PIN = "AVX512F AVX512CD AVX512_SKX AVX512_CLX AVX512_CNL AVX512_ICL AVX512_SPR"
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"

# (name, n, d, k, seed[, sigma, alpha, root])
CASES = [
    ("n16000_d64_k20", 16000, 64, 20, 0),
    ("n32000_d16_k10", 32000, 16, 10, 0),
    ("n46340_d64_k20", 46340, 64, 20, 0),
    # the boundary's other arguments at scale: explicit sigma + root, alpha > 0
    ("n20000_d16_k8_sigma3_root777", 20000, 16, 8, 2, 3.0, 0.0, 777),
    ("n12000_d32_k12_alpha0.5", 12000, 32, 12, 3, "auto", 0.5, 0),
]


def main() -> None:
    if os.environ.get("NPY_DISABLE_CPU_FEATURES") != PIN:
        env = dict(os.environ, NPY_DISABLE_CPU_FEATURES=PIN)
        sys.exit(subprocess.call([sys.executable, __file__, *sys.argv[1:]], env=env))
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, str(ROOT / "tests"))
    import numpy as np
    import isoclust as ic
    import digest as dg

    only = set(sys.argv[1:]) or None
    workers = os.cpu_count()
    for case in CASES:
        name, n, d, k, seed = case[:5]
        sigma_arg, alpha, root = (case[5], case[6], case[7]) if len(case) > 5 else ("auto", 0.0, 0)
        if only and name not in only:
            continue
        pts, _ = ic.generate_random(n, d, k, seed)
        t = {}
        t0 = time.perf_counter()
        dist = ic.distance_matrix(pts, workers=workers)
        t["distance_matrix"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        sigma = ic.auto_sigma(dist) if sigma_arg == "auto" else float(sigma_arg)
        t["auto_sigma"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        tree = ic.prim_mst(dist, sigma, root)
        t["prim_mst"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        w = ic.node_weights(dist, sigma, alpha, workers=workers)
        ext = ic.extrema(tree, w)
        t["node_weights_extrema"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        res = ic.par_solve_miso(tree, w, ext, k, workers=workers)
        t["partition"] = time.perf_counter() - t0
        total_distance = ic.total_distance(tree, dist)
        dsum = float(dist.sum())
        del dist
        dig = dg.result_digest(
            res, sigma=sigma, tree=tree, omega=w.omega, p=w.p,
            extrema=[ext.phi_star_sum, ext.phi_star_min, ext.omega_star_sum, ext.omega_star_min,
                     ext.p_star_sum, ext.p_star_min],
            total_distance=total_distance)
        dig["dsum"] = dg.fbits(dsum)
        dig["meta"] = {
            "source": "reference isoclust run_pipeline stages (pinned numpy), tools/gen_golden_large.py",
            "n": n, "d": d, "k": k, "seed": seed, "sigma_arg": sigma_arg, "alpha": alpha, "root": root,
            "engine": "par", "workers": workers, "stage_seconds": {a: round(b, 3) for a, b in t.items()},
            "numpy": np.__version__, "cpu_count": os.cpu_count(),
        }
        dg.save(OUT / f"large_{name}.json", dig)
        np.savez_compressed(OUT / f"large_{name}.npz", parent=tree.parent.astype(np.int32),
                            labels=res.labels.astype(np.int8))
        print(name, "sigma", sigma, "miso", res.miso, "iters", res.iterations, t, file=sys.stderr,
              flush=True)


if __name__ == "__main__":
    main()
