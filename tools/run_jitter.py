"""Diagnostic: run-to-run spread of run_pipeline on page-locked host input
(default C2: 100k x 16, k=10), 80 back-to-back runs after warm-up; prints the
median run and the slowest eight with their stage buckets and the omega-pass
time (profiles/round2_c2_host_jitter.txt).
python tools/run_jitter.py [n d k runs]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1702_04739_b200 as pkg  # noqa: E402

n, d, k, runs = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (100000, 16, 10, 80)))
X, _ = pkg.generate_random(n, d, k, 0)
X = bench.pinned_copy(X)
for _ in range(3):
    pkg.run_pipeline(X, k)
torch.cuda.synchronize()
rows = []
for _ in range(runs):
    t0 = time.perf_counter()
    r = pkg.run_pipeline(X, k)
    rows.append(((time.perf_counter() - t0) * 1e3, {a: round(b, 1) for a, b in r.timings_ms.items()},
                 r.mst_stats.get("omega_ms")))
rows.sort(key=lambda x: x[0])
print("median", rows[len(rows) // 2])
for x in rows[-8:]:
    print(x)
