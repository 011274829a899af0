"""Diagnostic: where a C1 run_pipeline spends its time (cProfile by
cumulative time, 20 runs after warm-up, device input)."""
import cProfile
import pstats
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1702_04739_b200 as pkg  # noqa: E402

pts, _ = pkg.generate_random(2000, 2, 3, 0)
X = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
for _ in range(5):
    pkg.run_pipeline(X, 3)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    pkg.run_pipeline(X, 3)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats(sys.argv[1] if len(sys.argv) > 1 else "tottime").print_stats(30)
