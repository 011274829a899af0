"""Diagnostic: host->device paths for a large pageable numpy array."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1702_04739_b200 import pipeline
b = pipeline.backend()
a = np.random.default_rng(0).random(50_000_000)
cud = torch.cuda.cudart()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); d = b.to_device(a); torch.cuda.synchronize()
    t1 = time.perf_counter() - t
    t = time.perf_counter(); d2 = torch.from_numpy(a).to("cuda"); torch.cuda.synchronize(); t2 = time.perf_counter() - t
    t = time.perf_counter()
    ta = torch.from_numpy(a)
    r = cud.cudaHostRegister(ta.data_ptr(), a.nbytes, 0)
    t_reg = time.perf_counter() - t
    d3 = torch.empty_like(ta, device="cuda"); d3.copy_(ta, non_blocking=True); torch.cuda.synchronize()
    cud.cudaHostUnregister(ta.data_ptr())
    t3 = time.perf_counter() - t
    print(f"staged {t1*1e3:.1f} ms  pageable {t2*1e3:.1f} ms  register+copy {t3*1e3:.1f} ms (register {t_reg*1e3:.1f}, rc={r})", flush=True)
