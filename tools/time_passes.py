"""Diagnostic: CUDA-event times of the exact passes at (n, d) -- the sigma
pass and the omega pass with fused round-2 minima -- plus checksums of their
outputs, so kernel variants (ISOC_LIB_PATH=variants/X.so) can be timed side
by side and checked for identical results."""
import hashlib
import os
import sys

sys.path.insert(0, '.')
sys.path.insert(0, 'oracle')
import torch

import oracle as orc
from paper_1702_04739_b200 import pipeline

n, d = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
pts, _ = orc.generate_random(n, d, 20, 0)
P = pipeline._Points(pts)
b = P.b


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def digest(*ts):
    h = hashlib.sha1()
    for t in ts:
        h.update(t.cpu().numpy().tobytes())
    return h.hexdigest()[:12]


for _ in range(reps):
    (stack, nn, _), ms = timed(lambda: pipeline._sigma_pass(P, 0.0))
    print(f"sigma_pass n={n} d={d} ms={ms:.1f} nn={digest(*nn)} ties={int(nn[2].sum())} nnj={digest(nn[0])} nnd={digest(nn[1])}", flush=True)
if os.environ.get("NO_NN"):
    for _ in range(reps):
        _, ms = timed(lambda: pipeline._sigma_pass(P, 0.0, want_nn=False))
        print(f"sigma_pass(no nn) n={n} d={d} ms={ms:.1f}", flush=True)
sigma = pipeline._sigma_from_stack(P, stack)
h = b.mst_create(P.X, n, d, 0, n)
cmin = b.mst_round_local(h, n, nn)
cedge = b.mst_round_edges(h, cmin)
b.mst_round_finish(h, cmin, cedge)
for _ in range(reps):
    (om, nn2), ms = timed(lambda: b.omega_mst(P.X, n, d, 0, n, sigma, h))
    print(f"omega_mst n={n} d={d} ms={ms:.1f} omega={digest(om)} nn={digest(*nn2[:2])}", flush=True)
b.mst_destroy(h)
print(f"sigma={sigma!r}")
if os.environ.get("PLAIN_OMEGA"):
    for _ in range(reps):
        om, ms = timed(lambda: b.omega(P.X, n, d, 0, n, sigma))
        print(f"omega(plain) n={n} d={d} ms={ms:.1f} omega={digest(om)}", flush=True)
