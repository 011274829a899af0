"""Diagnostic: where a C5 tree-phase step spends its time (cProfile)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1702_04739_b200 as pkg  # noqa: E402

n, k = 50_000_000, 100
parent, flows, omega, p = (bench.pinned_copy(a) for a in bench.synthetic_tree(n, 0))
w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=0.0)


def step():
    tree = pkg.tree_from_parent_list(parent, flows)
    ext = pkg.extrema(tree, w)
    return pkg.par_solve_miso(tree, w, ext, k)


for _ in range(2):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    step()
torch.cuda.synchronize()
pr.disable()
print("wall per step", (time.perf_counter() - t0) / 3)
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
