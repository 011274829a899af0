"""Small run_pipeline call for ncu captures (diagnostic)."""
import sys
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import oracle as orc
import paper_1702_04739_b200 as p
n, d, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (50000, 64, 20)))
pts, _ = orc.generate_random(n, d, k, 0)
run = p.run_pipeline(pts, k)
print(run.timings_ms, run.mst_stats)
