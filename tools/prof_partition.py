"""Diagnostic: per-call timings of the partition phase at a config (default
C3) over several pipeline runs -- each dt.decide / decide_batch call and the
final witness/labels step -- to find sporadic host-side stalls."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1702_04739_b200 as pkg
from paper_1702_04739_b200 import pipeline as pl
from paper_1702_04739_b200 import engine

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
X, _ = pkg.generate_random(n, d, k, 0)
Xdev = torch.from_numpy(np.ascontiguousarray(X)).cuda()

calls = []
DT = engine.DeviceTree
for name in ("decide", "decide_batch", "set_weights", "labels", "witness", "cost"):
    f = getattr(DT, name, None)
    if f is None:
        continue

    def wrap(f=f, name=name):
        def g(self, *a, **kw):
            t0 = time.perf_counter()
            r = f(self, *a, **kw)
            calls.append((name, (time.perf_counter() - t0) * 1e3))
            return r
        return g
    setattr(DT, name, wrap())

orig = pl.run_bisection


from cuda.bindings import runtime as cr


def pool_state():
    _, pool = cr.cudaDeviceGetDefaultMemPool(0)
    out = []
    for attr in (cr.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent, cr.cudaMemPoolAttr.cudaMemPoolAttrUsedMemCurrent):
        _, v = cr.cudaMemPoolGetAttribute(pool, attr)
        out.append(round(int(v) / 2**30, 2))
    _, free, tot = cr.cudaMemGetInfo()
    return out + [round(free / 2**30, 2), round(torch.cuda.memory_reserved() / 2**30, 2)]


def rb(*a, **kw):
    calls.append(("pool_reserved_used_free_torch_GB", pool_state()))
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    calls.append(("pre_sync", (time.perf_counter() - t0) * 1e3))
    t0 = time.perf_counter()
    r = orig(*a, **kw)
    calls.append(("run_bisection", (time.perf_counter() - t0) * 1e3))
    calls.append(("pool_after", pool_state()))
    return r


pl.run_bisection = rb
import gc
import os
if os.environ.get("NOGC"):
    gc.disable()
gc.callbacks.append(lambda phase, info: calls.append(("gc_" + phase + str(info.get("generation")), time.perf_counter() * 1e3)))
for rep in range(reps):
    calls.clear()
    run = pl.run_pipeline(Xdev, k)
    tot = {}
    for nm, ms in calls:
        tot.setdefault(nm, []).append(ms if isinstance(ms, list) else round(ms, 1))
    print(rep, {a: round(b, 1) for a, b in run.timings_ms.items()}, flush=True)
    for nm, v in tot.items():
        print("   ", nm, len(v), v[:20], flush=True)
