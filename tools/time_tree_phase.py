"""Per-stage wall times of the C5 tree phase (host arrays in, host results out)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1702_04739_b200 as pkg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
parent, flows, omega, p = bench.synthetic_tree(n, 0)
w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=0.0)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = pkg.tree_from_parent_list(parent, flows)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ext = pkg.extrema(tree, w)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res = pkg.par_solve_miso(tree, w, ext, 100)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"tree {1e3*(t1-t0):.1f} ms  extrema {1e3*(t2-t1):.1f} ms  solve {1e3*(t3-t2):.1f} ms  "
          f"total {1e3*(t3-t0):.1f} ms  iters {res.iterations}", flush=True)
if len(sys.argv) > 2:
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    tree = pkg.tree_from_parent_list(parent, flows)
    ext = pkg.extrema(tree, w)
    res = pkg.par_solve_miso(tree, w, ext, 100)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
