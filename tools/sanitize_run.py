"""Small workloads that launch every kernel of the path once, for
compute-sanitizer (racecheck / synccheck / memcheck): tools/sanitize.sh.
  pipeline  n=3000 d=16 k=5: K1s sigma_sym, K2s omega_sym (+ round-2 minima),
            tcgen05 filter rounds, rescans, hook/jump, BFS rooting, batched
            and single decide sweeps, labels / cost
  d512      n=2500 d=512 k=8: the filter's streamed K atoms, row passes
  prim      the tie-rule replay (ISOC_MST=prim) and the dense stage API
  tree      a 20,000-vertex random recursive tree (tree_from_parent_list)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
import paper_1702_04739_b200 as pkg  # noqa: E402

what = sys.argv[1]
if what == "pipeline":
    pts, _ = orc.generate_random(3000, 16, 5, 0)
    run = pkg.run_pipeline(pts, 5)
    ref = orc.run_pipeline(pts, 5)
    assert np.array_equal(run.result.labels, ref.result.labels)
    print("pipeline ok", run.mst_stats)
elif what == "d512":
    pts, _ = orc.generate_random(2500, 512, 8, 1)
    run = pkg.run_pipeline(pts, 8)
    print("d512 ok", run.mst_stats)
elif what == "prim":
    os.environ["ISOC_MST"] = "prim"
    pts, _ = orc.generate_random(2100, 3, 4, 2)
    run = pkg.run_pipeline(pts, 4, root=7)
    D = pkg.distance_matrix(pts[:600])
    t = pkg.prim_mst(D, 1.0, 3)
    print("prim ok", run.mst_stats, int(t.max_depth))
elif what == "tree":
    parent, flows, omega, p = orc.random_tree_instance(20000, 3)
    tree = pkg.tree_from_parent_list(parent, flows)
    w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=0.0)
    res = pkg.par_solve_miso(tree, w, pkg.extrema(tree, w), 20)
    print("tree ok", res.iterations)
