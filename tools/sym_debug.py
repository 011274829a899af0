"""Diagnostic: symmetric vs row sigma pass on assorted sizes."""
import os, sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import oracle as orc
from paper_1702_04739_b200 import pipeline
for n, d in [(2048, 3), (2049, 5), (3000, 16), (4099, 9), (4099, 16), (4099, 8), (5000, 9), (9000, 33)]:
    pts, _ = orc.generate_random(n, d, 4, 1)
    out = {}
    for mode in ("sym", "rows"):
        os.environ["ISOC_PASSES"] = mode
        P = pipeline._Points(pts)
        stack, (nj, nd, nt), _ = pipeline._sigma_pass(P, 0.0)
        try:
            s = pipeline._sigma_from_stack(P, stack)
        except Exception as e:
            s = repr(e)[:80]
        out[mode] = (s, nj.cpu().numpy(), nd.cpu().numpy(), nt.cpu().numpy())
    a, b = out["sym"], out["rows"]
    print(n, d, a[0] == b[0], a[0], b[0], [int((x != y).sum()) for x, y in zip(a[1:], b[1:])], flush=True)
