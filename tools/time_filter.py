"""Diagnostic: CUDA-event time of the Boruvka filter kernel at (n, d): one
round on singleton components (filter launch timed by the library's
profiling events; the rest of the round is not)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import ctypes
import torch
import oracle as orc
from paper_1702_04739_b200 import pipeline, _lib
n, d = int(sys.argv[1]), int(sys.argv[2])
pts, _ = orc.generate_random(n, d, 20, 0)
P = pipeline._Points(pts)
b = P.b
lib = _lib.load()
for rep in range(3):
    h = b.mst_create(P.X, n, d, 0, n)
    lib.isoc_prof_enable(1)
    b.mst_round_local(h, n, None)
    torch.cuda.synchronize()
    tot, cnt = ctypes.c_double(), ctypes.c_longlong()
    lib.isoc_prof_read(2, ctypes.byref(tot), ctypes.byref(cnt))
    lib.isoc_prof_enable(0)
    pairs = n * n
    print(f"filter n={n} d={d} ms={tot.value:.2f} launches={cnt.value} "
          f"tensor TFLOP/s={3 * 2 * 64 * pairs / (tot.value * 1e-3) / 1e12:.0f}", flush=True)
    b.mst_destroy(h)
