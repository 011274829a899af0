"""Reference-generated fixtures for the tie rule (prim_mst, mst.py:128-181;
min_reduce ties, _primitives.py:69-92): the reference's own Prim tree on

* an integer lattice with duplicates (many equal distances) through the dense
  stage API prim_mst(dist, sigma, root), and
* the two constructed instances of tests/test_gpu_parity.py (a round-2-only
  row tie; a round-1 unit-square tie under an explicit sigma).

Run in this container only (imports /root/reference), pinned numpy mode:
    python tools/gen_golden_ties.py      -> tests/golden/ties_*.npz
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PIN = "AVX512F AVX512CD AVX512_SKX AVX512_CLX AVX512_CNL AVX512_ICL AVX512_SPR"
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"


def main() -> None:
    if os.environ.get("NPY_DISABLE_CPU_FEATURES") != PIN:
        env = dict(os.environ, NPY_DISABLE_CPU_FEATURES=PIN)
        sys.exit(subprocess.call([sys.executable, __file__, *sys.argv[1:]], env=env))
    sys.path.insert(0, "/root/reference/pkg/src")
    import numpy as np
    import isoclust as ic

    def save(name, pts, sigma, root, k, with_pipeline):
        dist = ic.distance_matrix(pts, workers=1)
        sig = ic.auto_sigma(dist) if sigma == "auto" else float(sigma)
        tree = ic.prim_mst(dist, sig, root)
        extra = {}
        if with_pipeline:
            run = ic.run_pipeline(pts, k, sigma=sigma, root=root)
            extra = dict(labels=run.result.labels, miso=run.result.miso, iterations=run.result.iterations)
        np.savez_compressed(OUT / f"ties_{name}.npz", points=pts, sigma=sig, root=root, k=k,
                            sigma_arg=(-1.0 if sigma == "auto" else float(sigma)),
                            parent=tree.parent, child_id=tree.child_id, depth=tree.depth,
                            bfs_order=tree.bfs_order, parent_flow=tree.parent_flow, **extra)
        print(name, "parent[:8]", tree.parent[:8], file=sys.stderr)

    rng = np.random.default_rng(11)
    lat = rng.integers(0, 9, size=(700, 2)).astype(np.float64)
    lat[350] = lat[120]
    save("lattice_n700_root5", lat, "auto", 5, 4, False)

    pts, _ = ic.generate_random(2400, 2, 3, 5)
    six = np.array([[0, 0], [0, -1], [3, 4], [4, 3], [6, 3], [7, 3]], dtype=np.float64) + 1000.0
    save("round2_row_tie", np.concatenate([pts, six]), "auto", 2404, 3, True)
    pts, _ = ic.generate_random(2400, 2, 3, 6)
    sq = np.array([[0, 0], [1, 0], [0, 1], [1, 1]], dtype=np.float64) + 500.0
    save("round1_square_sigma1", np.concatenate([pts, sq]), 1.0, 2403, 3, True)


if __name__ == "__main__":
    main()
