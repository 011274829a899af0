"""Diagnostic: sigma-pass neighbours (round 1) and the omega pass's fused
round-2 minima at (n, d), saved to an npz for offline comparison."""
import sys

sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import numpy as np

import oracle as orc
from paper_1702_04739_b200 import pipeline

n, d, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
pts, _ = orc.generate_random(n, d, 20, 0)
P = pipeline._Points(pts)
b = P.b
stack, nn, _ = pipeline._sigma_pass(P, 0.0)
sigma = pipeline._sigma_from_stack(P, stack)
h = b.mst_create(P.X, n, d, 0, n)
cmin = b.mst_round_local(h, n, nn)
cedge = b.mst_round_edges(h, cmin)
b.mst_round_finish(h, cmin, cedge)
om, nn2 = b.omega_mst(P.X, n, d, 0, n, sigma, h)
b.mst_destroy(h)
np.savez(out, nn1=nn[0].cpu().numpy(), j2=nn2[0].cpu().numpy(), d2=nn2[1].cpu().numpy())
