"""Diagnostic: wall time of one sigma pass (sigma_partial) at n, d."""
import sys
import time

sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import numpy as np
import torch

from paper_1702_04739_b200 import pipeline

n, d = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(0)
pts = rng.standard_normal((n, d))
P = pipeline._Points(pts)
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    try:
        pipeline._sigma_pass(P, 0.0)
    except Exception as e:  # diagnostic runs may corrupt the result on purpose
        print("err", repr(e)[:100])
    torch.cuda.synchronize()
    print(n, d, "sigma_partial ms", round((time.perf_counter() - t) * 1e3, 1), flush=True)
