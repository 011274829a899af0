"""Diagnostic: per-step wall / event times of run_pipeline at C1 (device
input) with and without an nvidia-smi sampler running."""
import subprocess
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1702_04739_b200 as pkg  # noqa: E402

n, d, k = 2000, 2, 3
pts, _ = pkg.generate_random(n, d, k, 0)
X = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
for _ in range(5):
    pkg.run_pipeline(X, k)
torch.cuda.synchronize()


def loop(tag, steps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    tot = []
    for _ in range(steps):
        r = pkg.run_pipeline(X, k)
        tot.append(r.timings_ms["total"])
    e1.record()
    torch.cuda.synchronize()
    print(tag, "event ms/step", e0.elapsed_time(e1) / steps, "wall", (time.perf_counter() - t0) * 1e3 / steps,
          "internal", np.median(tot), flush=True)


loop("plain")
p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                     stdout=subprocess.DEVNULL)
time.sleep(0.5)
loop("with nvidia-smi")
p.terminate()
loop("plain again")
