"""Diagnostic: one warm-up + one timed run_pipeline at (n, d, k) for ncu
launch lists (ncu --metrics gpu__time_duration.sum ... python tools/one_pipeline.py n d k)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_1702_04739_b200 as pkg  # noqa: E402

n, d, k = (int(a) for a in sys.argv[1:4])
pts, _ = pkg.generate_random(n, d, k, 0)
import torch  # noqa: E402
X = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
for it in range(int(sys.argv[4]) if len(sys.argv) > 4 else 2):
    t0 = time.perf_counter()
    run = pkg.run_pipeline(X, k)
    torch.cuda.synchronize()
    print(f"run {it}: {time.perf_counter() - t0:.4f}s", run.timings_ms, run.mst_stats, flush=True)
