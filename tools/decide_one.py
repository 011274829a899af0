"""One representative C5 decision sweep (for ncu): solve once, then sweep at
the final beta (a feasible threshold that runs to the k-th cut)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1702_04739_b200 as pkg  # noqa: E402
from paper_1702_04739_b200.pipeline import _attach  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
parent, flows, omega, p = bench.synthetic_tree(n, 0)
w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=0.0)
tree = pkg.tree_from_parent_list(parent, flows)
ext = pkg.extrema(tree, w)
res = pkg.par_solve_miso(tree, w, ext, 100)
dt = _attach(tree, w)
print("levels/width", dt.shape(), "beta", res.beta_final, flush=True)
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for thr in (res.beta_final, res.alpha_final, res.trace[0][0]):
    for _ in range(reps):
        torch.cuda.synchronize()
        st.record()
        j = dt.decide(thr, 100, 0)
        en.record()
        torch.cuda.synchronize()
    print(f"thr {thr:.6g} j {j} {st.elapsed_time(en):.3f} ms (event, default stream)", flush=True)
