"""Diagnostic: per-row partial leaf stacks of the symmetric sigma pass
(isoc_sigma_sym_range over all blocks) for two builds of the library, and
the rows where they differ."""
import os
import sys

sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import numpy as np

import oracle as orc

n, d = int(sys.argv[1]), int(sys.argv[2])
out = sys.argv[3]
pts, _ = orc.generate_random(n, d, 3, 0)
from paper_1702_04739_b200 import pipeline
P = pipeline._Points(pts)
jlo, jhi = 0, (n + 1023) // 1024
vals, ids, cnt, m1, m2, j1 = P.b.sigma_sym_range(P.X, n, d, jlo, jhi)
np.savez(out, vals=vals.cpu().numpy(), ids=ids.cpu().numpy(), cnt=cnt.cpu().numpy())
if len(sys.argv) > 4:
    o = np.load(sys.argv[4])
    c0, c1 = o["cnt"], cnt.cpu().numpy()
    v0, v1 = o["vals"], vals.cpu().numpy()
    bad = [r for r in range(n) if c0[r] != c1[r] or not np.array_equal(v0[r, :c0[r]], v1[r, :c1[r]])]
    print("rows differing:", len(bad), bad[:20])
    for r in bad[:5]:
        print(r, c0[r], c1[r], v0[r, :c0[r]], v1[r, :c1[r]], o["ids"][r, :c0[r]], ids.cpu().numpy()[r, :c1[r]])
