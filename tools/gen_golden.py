"""Generate golden fixtures by running the REFERENCE implementation.

Run in this container only (it imports /root/reference/pkg/src):
    python tools/gen_golden.py
It re-executes itself with numpy's AVX-512 kernels disabled ("pinned mode",
SURVEY.md Appendix A.4), where np.exp is glibc exp bit for bit, so the
fixtures are reproducible by a CPU restatement and by the CUDA port.
Outputs tests/golden/*.npz (small; committed).  Nothing on the GPU box reads
/root/reference: tests consume only these files.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PIN = "AVX512F AVX512CD AVX512_SKX AVX512_CLX AVX512_CNL AVX512_ICL AVX512_SPR"
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"

# (name, n, d, k, seed, alpha, root, sigma)
PIPELINE_CASES = [
    ("c1_seed0", 2000, 2, 3, 0, 0.0, 0, "auto"),
    ("c1_seed1", 2000, 2, 3, 1, 0.0, 0, "auto"),
    ("d16_n1000", 1000, 16, 10, 0, 0.0, 0, "auto"),
    ("d64_n1500", 1500, 64, 20, 0, 0.0, 0, "auto"),
    ("d512_n600", 600, 512, 50, 0, 0.0, 0, "auto"),
    ("d5_n300_alpha1_root7", 300, 5, 6, 3, 1.0, 7, "auto"),
    ("d3_n50", 50, 3, 4, 7, 0.0, 0, "auto"),
    ("d2_n777_sigma2", 777, 2, 5, 11, 0.0, 3, 2.0),
    ("d13_n178", 178, 13, 3, 5, 0.0, 0, "auto"),
    # explicit small sigma: most flows exp(-d/sigma) underflow to subnormals / 0
    ("d5_n300_sigma0.02", 300, 5, 3, 0, 0.0, 0, 0.02),
    ("d5_n300_sigma0.05", 300, 5, 3, 0, 0.0, 0, 0.05),
]


def main() -> None:
    if os.environ.get("NPY_DISABLE_CPU_FEATURES") != PIN:
        env = dict(os.environ, NPY_DISABLE_CPU_FEATURES=PIN)
        sys.exit(subprocess.call([sys.executable, __file__, *sys.argv[1:]], env=env))
    only = None
    if len(sys.argv) > 2 and sys.argv[1] == "--only":
        only = set(sys.argv[2].split(","))
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, "/root/reference/pkg/tests")
    import numpy as np
    import isoclust as ic
    from conftest import random_instance  # the reference's own generator

    OUT.mkdir(parents=True, exist_ok=True)
    for name, n, d, k, seed, alpha, root, sigma in PIPELINE_CASES:
        if only is not None and name not in only:
            continue
        pts, _ = ic.generate_random(n, d, k, seed)
        run = ic.run_pipeline(pts, k, sigma=sigma, alpha=alpha, root=root, engine="seq")
        dist = ic.distance_matrix(pts, workers=1)
        tree = ic.prim_mst(dist, run.sigma, root)
        w = ic.node_weights(dist, run.sigma, alpha, workers=1)
        ext = ic.extrema(tree, w)
        r = run.result
        np.savez_compressed(
            OUT / f"pipe_{name}.npz",
            n=n, d=d, k=k, seed=seed, alpha=alpha, root=root,
            sigma_arg=(-1.0 if sigma == "auto" else float(sigma)),
            sigma=run.sigma, dsum=float(dist.sum()),
            parent=tree.parent, parent_flow=tree.parent_flow, depth=tree.depth,
            child_id=tree.child_id, bfs_order=tree.bfs_order, max_depth=tree.max_depth,
            total_distance=ic.total_distance(tree, dist),
            omega=w.omega, p=w.p,
            extrema=np.array([ext.phi_star_sum, ext.phi_star_min, ext.omega_star_sum,
                              ext.omega_star_min, ext.p_star_sum, ext.p_star_min]),
            labels=r.labels, miso=r.miso, iterations=r.iterations,
            alpha_final=r.alpha_final, beta_final=r.beta_final,
            trace_mid=np.array([t[0] for t in r.trace]),
            trace_ok=np.array([t[1] for t in r.trace], dtype=np.int8),
            cut=r.outcome.cut, eta=r.outcome.eta,
            sparsities=np.array(r.outcome.cluster_sparsities),
            row0=dist[0].copy(), rowlast=dist[n - 1].copy(),
        )
        print(name, "sigma", run.sigma, "miso", r.miso, "iters", r.iterations, file=sys.stderr)
    if only is not None:
        return

    # tree-phase instances from the reference's own random_instance
    rng = np.random.Generator(np.random.PCG64(20260814))
    trees = []
    for i in range(40):
        nn = int(rng.integers(3, 300))
        kk = int(rng.integers(1, 8))
        mode = "zero" if i % 2 == 0 else "alpha"
        tree, w = random_instance(rng, nn, alpha_mode=mode)
        ext = ic.extrema(tree, w)
        try:
            res = ic.par_solve_miso(tree, w, ext, kk, workers=1)
            ok = 1
        except ic.InfeasibleSubpartitionError:
            res, ok = None, 0
        rec = dict(parent=tree.parent, flows=tree.parent_flow, omega=w.omega, p=w.p, k=kk, ok=ok,
                   child_id=tree.child_id, depth=tree.depth, bfs_order=tree.bfs_order)
        if ok:
            rec.update(labels=res.labels, miso=res.miso, iterations=res.iterations,
                       alpha_final=res.alpha_final, beta_final=res.beta_final,
                       trace_mid=np.array([t[0] for t in res.trace]),
                       trace_ok=np.array([t[1] for t in res.trace], dtype=np.int8),
                       cut=res.outcome.cut, eta=res.outcome.eta,
                       sparsities=np.array(res.outcome.cluster_sparsities))
        trees.append(rec)
    np.savez_compressed(OUT / "trees_random_instance.npz",
                        **{f"t{i}_{key}": v for i, rec in enumerate(trees) for key, v in rec.items()},
                        count=len(trees))

    # one larger random recursive tree (reference generator, k=20)
    rng = np.random.Generator(np.random.PCG64(505))
    from conftest import random_parent_array
    nn = 20000
    parent = random_parent_array(rng, nn)
    flows = np.zeros(nn)
    nonroot = parent != -1
    flows[nonroot] = 1.0 - rng.uniform(0.0, 1.0, int(nonroot.sum()))
    tree = ic.tree_from_parent_list(parent, flows)
    omega = 2.0 - rng.uniform(0.0, 1.9, nn)
    w = ic.NodeWeights(omega=omega, p=np.zeros(nn), sigma=1.0, alpha=0.0)
    ext = ic.extrema(tree, w)
    res = ic.par_solve_miso(tree, w, ext, 20, workers=1)
    np.savez_compressed(OUT / "tree_rrt_n20000_k20.npz", parent=parent, flows=tree.parent_flow,
                        omega=omega, p=w.p, k=20, labels=res.labels, miso=res.miso,
                        iterations=res.iterations, alpha_final=res.alpha_final,
                        beta_final=res.beta_final,
                        trace_mid=np.array([t[0] for t in res.trace]),
                        trace_ok=np.array([t[1] for t in res.trace], dtype=np.int8),
                        cut=res.outcome.cut, eta=res.outcome.eta,
                        sparsities=np.array(res.outcome.cluster_sparsities),
                        child_id=tree.child_id, depth=tree.depth, bfs_order=tree.bfs_order)
    print("trees done", file=sys.stderr)


if __name__ == "__main__":
    main()
