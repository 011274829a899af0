"""Diagnostic: where the C5 tree-phase step spends its time (host + device)."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch
import oracle as orc
import paper_1702_04739_b200 as pkg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
parent, flows, omega, p = orc.random_tree_instance(n, 0)
w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=0.0)
def step():
    tree = pkg.tree_from_parent_list(parent, flows)
    ext = pkg.extrema(tree, w)
    return pkg.par_solve_miso(tree, w, ext, 100)
step(); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t = time.perf_counter(); step(); torch.cuda.synchronize(); el = time.perf_counter() - t
pr.disable()
print("step s", el)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
