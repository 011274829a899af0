"""Stage timings of run_pipeline on synthetic blobs (diagnostic, not the bench)."""
import sys, time, json
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import oracle as orc
import paper_1702_04739_b200 as p
import torch
cfgs = [tuple(map(int, c.split(','))) for c in sys.argv[1:]] or [(100000, 16, 10)]
for n, d, k in cfgs:
    pts, _ = orc.generate_random(n, d, k, 0)
    run = p.run_pipeline(pts[: min(n, 4096)], k)  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    run = p.run_pipeline(pts, k)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    print(json.dumps({"n": n, "d": d, "k": k, "wall_s": round(el, 3), "timings_ms": {a: round(b, 1) for a, b in run.timings_ms.items()},
                      "mst": run.mst_stats, "iters": run.result.iterations, "miso": run.result.miso,
                      "residual": int((run.result.labels == 0).sum())}), flush=True)
