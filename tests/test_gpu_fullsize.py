"""Full-size parity: the B200 pipeline against compact bitwise digests
(tests/digest.py) of

* the REFERENCE itself at N = 16,000 / 32,000 / 46,340 (its dense cap,
  affinity.py:139-143) -- tests/golden/large_*.json, tools/gen_golden_large.py;
* the CPU oracle at the BASELINE.json configs C2 (100k x 16, k=10),
  C3 (1M x 64, k=20), C4 (200k x 512, k=50) and C5 (50M-vertex tree, k=100)
  -- tests/golden/full_*.json, tools/oracle_full.py.  The oracle is pinned to
  the reference at the three sizes above (tools/oracle_full.py --check,
  tests/test_oracle.py) and its MST is certified unique, so it equals the
  reference's Prim tree.

Every field is compared bit for bit: sigma, parent / child_id / depth /
bfs_order / parent_flow (and the MST edge set), omega, extrema, labels, cut,
eta, cluster sparsities, the bisection trace, iterations, alpha/beta, miso and
the tree weight (math.fsum of the exact parent distances).
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import digest as dg

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1702_04739_b200 as p
    return p


def _pipeline_digest(run) -> dict:
    t = run.tree
    e = run.extrema
    out = dg.result_digest(run.result, sigma=run.sigma, tree=t, omega=run.omega_host(), p=run.p_host(),
                           extrema=[e.phi_star_sum, e.phi_star_min, e.omega_star_sum, e.omega_star_min,
                                    e.p_star_sum, e.p_star_min])
    return out


def _tree_weight(pkg, pts, tree) -> float:
    """math.fsum of the exact parent distances (mst.py:184-187)."""
    import torch
    X = torch.from_numpy(np.ascontiguousarray(pts)).cuda()
    par = torch.from_numpy(np.asarray(tree.parent)).cuda()
    nz = (par >= 0).nonzero().squeeze(1)
    # exact per-pair distances in scipy order on the device (t = u - v, s += t*t)
    diff = X[nz] - X[par[nz]]
    s = torch.zeros(nz.numel(), dtype=torch.float64, device=X.device)
    for k in range(X.shape[1]):
        t = diff[:, k]
        s = s + t * t
    return math.fsum(torch.sqrt(s).cpu().numpy().tolist())


def _check(got: dict, want: dict):
    keys = [k for k in want if k != "meta" and k not in ("dsum",)]
    missing = [k for k in keys if k not in got]
    assert not missing, missing
    bad = dg.compare(got, want, keys)
    assert bad == [], {k: (got.get(k), want.get(k)) for k in bad[:3]}


@pytest.mark.parametrize("name", ["n16000_d64_k20", "n32000_d16_k10", "n46340_d64_k20",
                                  "n20000_d16_k8_sigma3_root777", "n12000_d32_k12_alpha0.5"])
def test_pipeline_equals_reference_large(name, pkg):
    """run_pipeline == the reference's own run at up to its dense cap, with
    the default arguments and with an explicit sigma + root and alpha > 0."""
    want = dg.load(os.path.join(GOLDEN, f"large_{name}.json"))
    m = want["meta"]
    pts, _ = pkg.generate_random(m["n"], m["d"], m["k"], m["seed"])
    run = pkg.run_pipeline(pts, m["k"], sigma=m["sigma_arg"], alpha=m["alpha"], root=m["root"])
    got = _pipeline_digest(run)
    got["total_distance"] = dg.fbits(_tree_weight(pkg, pts, run.tree))
    _check(got, want)
    with np.load(os.path.join(GOLDEN, f"large_{name}.npz")) as z:
        assert np.array_equal(run.tree.parent, z["parent"])
        assert np.array_equal(run.result.labels, z["labels"])


def _fixture(name):
    path = os.path.join(GOLDEN, f"full_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"oracle fixture {path} not generated (tools/oracle_full.py {name})")
    return dg.load(path)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c2_seed1", "c3_seed1", "c4_seed1"])
def test_pipeline_equals_oracle_full_size(name, pkg):
    """BASELINE.json C1-C4 at full size (seed 0, and seed 1 -- SURVEY 8(d)'s
    second seed), every field bitwise vs the oracle."""
    want = _fixture(name)
    m = want["meta"]
    pts, _ = pkg.generate_random(m["n"], m["d"], m["k"], m["seed"])
    run = pkg.run_pipeline(pts, m["k"])
    assert run.mst_stats.get("exact_ties", 0) == 0
    got = _pipeline_digest(run)
    got["total_distance"] = dg.fbits(_tree_weight(pkg, pts, run.tree))
    _check(got, want)


def test_tree_phase_equals_oracle_c5(pkg):
    """BASELINE.json C5: 50M-vertex random recursive tree, k=100, tree phase
    only (tree_from_parent_list + extrema + par_solve_miso)."""
    want = _fixture("c5")
    m = want["meta"]
    import oracle as orc   # the instance generator (same law as bench.py's)
    parent, flows, omega, p = orc.random_tree_instance(m["n"], m["seed"])
    tree = pkg.tree_from_parent_list(parent, flows)
    w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=0.0)
    ext = pkg.extrema(tree, w)
    res = pkg.par_solve_miso(tree, w, ext, m["k"])
    got = dg.result_digest(res, tree=tree, omega=omega,
                           extrema=[ext.phi_star_sum, ext.phi_star_min, ext.omega_star_sum,
                                    ext.omega_star_min, ext.p_star_sum, ext.p_star_min])
    _check(got, want)
