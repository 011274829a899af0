"""Evidence run (not part of the test suite): the whole pipeline at large n
on the GPU against the CPU oracle (reference operation order, all host
threads), bit for bit: sigma, MST edge set and tree arrays, omega, labels,
miso, iterations, trace.  Usage: python tools/check_large.py N D K [seed]"""
import json
import sys
import time

sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import numpy as np

import oracle as orc
import paper_1702_04739_b200 as pkg

n, d, k = (int(a) for a in sys.argv[1:4])
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 0
pts, _ = orc.generate_random(n, d, k, seed)
t0 = time.perf_counter()
run = pkg.run_pipeline(pts, k)
t_gpu = time.perf_counter() - t0
t0 = time.perf_counter()
ref = orc.run_pipeline(pts, k)
t_cpu = time.perf_counter() - t0
bits = lambda a: np.asarray(a, dtype=np.float64).view(np.int64)
r, q = run.result, ref.result
checks = {
    "sigma": run.sigma == ref.sigma,
    "labels": bool(np.array_equal(r.labels, q.labels)),
    "miso": r.miso == q.miso,
    "iterations": r.iterations == q.iterations,
    "alpha_beta": (r.alpha_final, r.beta_final) == (q.alpha_final, q.beta_final),
    "trace": [m for m, _ in r.trace] == [m for m, _ in q.trace],
    "cut_eta": bool(np.array_equal(r.outcome.cut, q.outcome.cut) and np.array_equal(r.outcome.eta, q.outcome.eta)),
}
print(json.dumps({"n": n, "d": d, "k": k, "seed": seed, "gpu_s": round(t_gpu, 2), "cpu_oracle_s": round(t_cpu, 1),
                  "all_equal": all(checks.values()), "checks": checks, "mst_stats": run.mst_stats}))
