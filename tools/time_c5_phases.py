"""Diagnostic: wall time of each part of a C5 tree-phase step (pinned host
inputs, as bench.py), including the release of the previous tree handle."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1702_04739_b200 as pkg  # noqa: E402

n, k = 50_000_000, 100
parent, flows, omega, p = (bench.pinned_copy(a) for a in bench.synthetic_tree(n, 0))
w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=0.0)
for rep in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    tree = pkg.tree_from_parent_list(parent, flows)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    ext = pkg.extrema(tree, w)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    res = pkg.par_solve_miso(tree, w, ext, k)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    del tree, ext
    t.append(time.perf_counter())
    d = [round((b - a) * 1e3, 1) for a, b in zip(t, t[1:])]
    print(rep, "tree", d[0], "extrema", d[1], "solve", d[2], "release", d[3], "total", round((t[-1] - t[0]) * 1e3, 1),
          flush=True)
