"""Diagnostic: wall time per decide_batch call on the C1 MST (63 thresholds)."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_1702_04739_b200 as pkg  # noqa: E402
from paper_1702_04739_b200 import pipeline as pl  # noqa: E402

pts, _ = pkg.generate_random(2000, 2, 3, 0)
run = pkg.run_pipeline(pts, 3)
dt = run.tree._device
thr, kids, root = pl._threshold_tree(run.result.alpha_final * 0.5, run.result.beta_final * 2.0, 6)
for cnt in (63, 15, 1):
    for _ in range(5):
        dt.decide_batch(thr[:cnt], 3)
    t0 = time.perf_counter()
    for _ in range(200):
        dt.decide_batch(thr[:cnt], 3)
    print(f"decide_batch x{cnt}: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us per call", flush=True)
t0 = time.perf_counter()
for _ in range(200):
    dt.decide(thr[0], 3, 0)
print(f"decide (witness): {(time.perf_counter() - t0) / 200 * 1e6:.1f} us per call")

# calibration: trivial API call, torch launch + sync, pageable copies
import ctypes  # noqa: E402
import torch  # noqa: E402
lib = pkg._lib.load()
lv, mw = ctypes.c_int64(), ctypes.c_int64()
t0 = time.perf_counter()
for _ in range(1000):
    lib.isoc_tree_shape(dt.h, ctypes.byref(lv), ctypes.byref(mw))
print(f"isoc_tree_shape: {(time.perf_counter() - t0) / 1000 * 1e6:.1f} us")
x = torch.zeros(8, device="cuda")
t0 = time.perf_counter()
for _ in range(1000):
    x.add_(1.0)
    torch.cuda.synchronize()
print(f"torch launch+sync: {(time.perf_counter() - t0) / 1000 * 1e6:.1f} us")
h = np.zeros(64)
t0 = time.perf_counter()
for _ in range(1000):
    x.copy_(torch.from_numpy(h[:8]).float())
    torch.cuda.synchronize()
print(f"torch small H2D+sync: {(time.perf_counter() - t0) / 1000 * 1e6:.1f} us")
cap = ctypes.c_int32()
t0 = time.perf_counter()
for _ in range(1000):
    lib.isoc_decide_batch_capacity(dt.h, ctypes.byref(cap))
print(f"isoc_decide_batch_capacity: {(time.perf_counter() - t0) / 1000 * 1e6:.1f} us")
