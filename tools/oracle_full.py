"""Full-size oracle runs -> compact parity fixtures (test infrastructure).

Runs the CPU oracle (oracle/oracle.py run_pipeline_full: the reference's
operation order, vectorised across pairs, certified-unique MST) on the
BASELINE.json configs and writes tests/golden/full_<name>.json digests
(tests/digest.py).  Long-running at C3 (about an hour on 8 cores): run in the
background in the CPU container.
    python tools/oracle_full.py c3|c4|c5|<n> <d> <k> [seed]      (c1-c4: --seed S for another seed)
For n <= 46,340 `--check` compares against the reference digests
(tests/golden/large_*.json) instead of writing.
"""
from __future__ import annotations

import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import digest as dg  # noqa: E402
import oracle as orc  # noqa: E402

CONFIGS = {
    "c1": (2000, 2, 3, 0),
    "c2": (100_000, 16, 10, 0),
    "c3": (1_000_000, 64, 20, 0),
    "c4": (200_000, 512, 50, 0),
}
C5 = (50_000_000, 100, 0)


def points_digest(name, n, d, k, seed):
    pts, _ = orc.generate_random(n, d, k, seed)
    t0 = time.perf_counter()
    run = orc.run_pipeline_full(pts, k)
    wall = time.perf_counter() - t0
    o = run.out
    e = o.extrema
    dig = dg.result_digest(o.result, sigma=o.sigma, tree=o.tree, omega=o.omega, p=o.p,
                           extrema=[e.phi_star_sum, e.phi_star_min, e.omega_star_sum, e.omega_star_min,
                                    e.p_star_sum, e.p_star_min],
                           total_distance=run.total_distance)
    dig["meta"] = {
        "source": "CPU oracle run_pipeline_full (tools/oracle_full.py)", "config": name,
        "n": n, "d": d, "k": k, "seed": seed, "sigma_arg": "auto", "alpha": 0.0, "root": 0,
        "oracle_seconds": {a: round(b, 2) for a, b in run.seconds.items()}, "wall_s": round(wall, 1),
        "threads": orc.lib().oc_num_threads(), "isa": f"x86-64-v{orc.lib().ocf_isa()}",
        "mst_certificate": {"rounds": run.mst_stats["rounds"], "rescans": run.mst_stats["rescans"],
                            "rescans_per_round": run.mst_stats["rescans_per_round"],
                            "components_per_round": run.mst_stats["components_per_round"],
                            "unique_mst": True},
    }
    return dig


def tree_digest(n, k, seed):
    parent, flows, omega, p = orc.random_tree_instance(n, seed)
    t0 = time.perf_counter()
    res, tree, ext = orc.solve_tree(parent, flows, omega, p, k)
    wall = time.perf_counter() - t0
    dig = dg.result_digest(res, tree=tree, omega=omega,
                           extrema=[ext.phi_star_sum, ext.phi_star_min, ext.omega_star_sum,
                                    ext.omega_star_min, ext.p_star_sum, ext.p_star_min])
    dig["meta"] = {"source": "CPU oracle solve_tree (tools/oracle_full.py)", "config": "c5",
                   "n": n, "k": k, "seed": seed, "wall_s": round(wall, 1),
                   "generator": "oracle.random_tree_instance (vectorised random_parent_array law)"}
    return dig


def main(argv):
    check = "--check" in argv
    argv = [a for a in argv if a != "--check"]
    name = argv[0]
    seed_override = None
    if "--seed" in argv:
        i = argv.index("--seed")
        seed_override = int(argv[i + 1])
        del argv[i:i + 2]
    if name == "c5":
        n, k, seed = C5
        dig = tree_digest(n, k, seed)
    else:
        if name in CONFIGS:
            n, d, k, seed = CONFIGS[name]
            if seed_override is not None:
                seed = seed_override
                name = f"{name}_seed{seed}"
        else:
            n, d, k = (int(a) for a in argv[:3])
            seed = int(argv[3]) if len(argv) > 3 else 0
            name = f"n{n}_d{d}_k{k}"
        dig = points_digest(name, n, d, k, seed)
    if check:
        want = dg.load(os.path.join(ROOT, "tests", "golden", f"large_{name}.json"))
        bad = dg.compare(dig, want)
        print(json.dumps({"config": name, "equal_to_reference": not bad, "differs": bad,
                          "compared": sorted(k for k in want if k in dig and k != "meta"),
                          "meta": dig["meta"]}))
        return 0 if not bad else 1
    out = os.path.join(ROOT, "tests", "golden", f"full_{name}.json")
    dg.save(out, dig)
    print(json.dumps(dig["meta"]))
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
