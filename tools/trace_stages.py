"""Per-call wall time of every backend/device-tree call (diagnostic)."""
import sys, time, json, functools, collections
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch
import oracle as orc
import paper_1702_04739_b200 as p
from paper_1702_04739_b200 import engine
acc = collections.defaultdict(lambda: [0.0, 0])
def wrap(cls, name):
    f = getattr(cls, name)
    @functools.wraps(f)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); acc[f"{cls.__name__}.{name}"][0] += time.perf_counter() - t
        acc[f"{cls.__name__}.{name}"][1] += 1
        return r
    setattr(cls, name, g)
for n_ in ["to_device", "sigma_partial", "sigma_finish", "omega_mst", "mst_create", "mst_round_local",
           "mst_round_edges", "mst_round_finish", "mst_edges", "mst_destroy", "tree_from_edges"]:
    wrap(engine.CudaBackend, n_)
for n_ in ["set_weights", "decide", "witness"]:
    wrap(engine.DeviceTree, n_)
n, d, k = (int(x) for x in sys.argv[1:4])
pts, _ = orc.generate_random(n, d, k, 0)
X = torch.from_numpy(pts).cuda()
for rep in range(2):
    acc.clear()
    t = time.perf_counter(); run = p.run_pipeline(X, k); torch.cuda.synchronize()
    print("rep", rep, "total", round(time.perf_counter() - t, 3), {a: round(b, 1) for a, b in run.timings_ms.items()})
for kk, (s, c) in sorted(acc.items(), key=lambda x: -x[1][0]):
    print(f"{kk:40s} {s*1e3:10.1f} ms  x{c}")
