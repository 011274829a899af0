"""The CPU oracle reproduces the reference bit for bit on its own outputs.

Fixtures in tests/golden were produced by running the reference
(/root/reference/pkg/src/isoclust, pinned numpy mode) via tools/gen_golden.py.
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from conftest import golden_pipeline_cases, load, random_instance_trees


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


@pytest.mark.parametrize("path", golden_pipeline_cases(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_oracle_pipeline_matches_reference(path, oracle_mod):
    g = load(path)
    n, d, k, seed = int(g["n"]), int(g["d"]), int(g["k"]), int(g["seed"])
    pts, _ = oracle_mod.generate_random(n, d, k, seed)
    # distances: first and last row bitwise (scipy order)
    assert np.array_equal(bits(oracle_mod.distance_rows(pts, 0, 1)[0]), bits(g["row0"]))
    assert np.array_equal(bits(oracle_mod.distance_rows(pts, n - 1, n)[0]), bits(g["rowlast"]))
    assert oracle_mod.flat_distance_sum(pts) == float(g["dsum"])
    sigma = "auto" if float(g["sigma_arg"]) < 0 else float(g["sigma_arg"])
    out = oracle_mod.run_pipeline(pts, k, sigma=sigma, alpha=float(g["alpha"]), root=int(g["root"]))
    assert out.sigma == float(g["sigma"])
    t = out.tree
    for name in ("parent", "depth", "child_id", "bfs_order"):
        assert np.array_equal(getattr(t, name), g[name]), name
    assert np.array_equal(bits(t.parent_flow), bits(g["parent_flow"]))
    assert math.fsum(t.parent_dist) == float(g["total_distance"])
    assert np.array_equal(bits(out.omega), bits(g["omega"]))
    assert np.array_equal(bits(out.p), bits(g["p"]))
    e = out.extrema
    assert [e.phi_star_sum, e.phi_star_min, e.omega_star_sum, e.omega_star_min, e.p_star_sum,
            e.p_star_min] == list(g["extrema"])
    r = out.result
    assert np.array_equal(r.labels, g["labels"])
    assert r.miso == float(g["miso"])
    assert r.iterations == int(g["iterations"])
    assert r.alpha_final == float(g["alpha_final"]) and r.beta_final == float(g["beta_final"])
    assert [m for m, _ in r.trace] == list(g["trace_mid"])
    assert [int(f) for _, f in r.trace] == list(g["trace_ok"])
    assert np.array_equal(r.outcome.cut, g["cut"]) and np.array_equal(r.outcome.eta, g["eta"])
    assert r.outcome.cluster_sparsities == list(g["sparsities"])


def test_oracle_tree_phase_matches_reference(oracle_mod):
    for rec in random_instance_trees():
        k = int(rec["k"])
        if not int(rec["ok"]):
            with pytest.raises(oracle_mod.InfeasibleSubpartitionError):
                oracle_mod.solve_tree(rec["parent"], rec["flows"], rec["omega"], rec["p"], k)
            continue
        res, tree, _ = oracle_mod.solve_tree(rec["parent"], rec["flows"], rec["omega"], rec["p"], k)
        assert np.array_equal(tree.child_id, rec["child_id"])
        assert np.array_equal(tree.bfs_order, rec["bfs_order"])
        assert np.array_equal(res.labels, rec["labels"])
        assert res.miso == float(rec["miso"])
        assert res.iterations == int(rec["iterations"])
        assert [m for m, _ in res.trace] == list(rec["trace_mid"])
        assert res.outcome.cluster_sparsities == list(rec["sparsities"])


def test_oracle_rrt_20000(oracle_mod):
    import os
    from conftest import GOLDEN
    g = load(os.path.join(GOLDEN, "tree_rrt_n20000_k20.npz"))
    res, tree, _ = oracle_mod.solve_tree(g["parent"], g["flows"], g["omega"], g["p"], int(g["k"]))
    assert np.array_equal(tree.bfs_order, g["bfs_order"])
    assert np.array_equal(res.labels, g["labels"])
    assert res.miso == float(g["miso"]) and res.iterations == int(g["iterations"])
    assert res.alpha_final == float(g["alpha_final"]) and res.beta_final == float(g["beta_final"])


def test_oracle_exp_matches_libm(oracle_mod):
    # the pinned-mode np.exp is glibc exp: compare against libm directly
    import ctypes
    libm = ctypes.CDLL("libm.so.6")
    libm.exp.restype = ctypes.c_double
    libm.exp.argtypes = [ctypes.c_double]
    rng = np.random.default_rng(3)
    xs = np.concatenate([-rng.random(20000) * 40, -rng.random(2000) * 800, (rng.random(2000) - 0.5) * 1500,
                         [0.0, -0.0, -1e-300, -745.2, -708.4, -709.9, 709.7, -1e-17]])
    got = oracle_mod.exp(xs)
    want = np.array([libm.exp(float(x)) for x in xs])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


def test_pairwise_sum_matches_numpy(oracle_mod):
    rng = np.random.default_rng(9)
    for n in (0, 1, 7, 8, 9, 127, 128, 129, 1000, 8193, 123457):
        a = rng.random(n) * 100
        assert oracle_mod.pairwise_sum(a) == float(np.sum(a))


def test_oracle_all_flows_underflow_raises_zero_division(oracle_mod):
    # with sigma so small that every exp(-d/sigma) underflows,
    # the reference's bracket (phi_min + p_min) / omega_sum raises Python's
    # ZeroDivisionError (isoperim.py:238-239; checked by running the reference
    # on this instance: run_pipeline(generate_random(300, 5, 3, 0), 3, sigma=1e-3))
    pts, _ = oracle_mod.generate_random(300, 5, 3, 0)
    with pytest.raises(ZeroDivisionError):
        oracle_mod.run_pipeline(pts, 3, sigma=1e-3)


# ------------------------------------------------ full-size oracle (isoc_fast.c)
@pytest.mark.parametrize("n,d", [(2, 3), (50, 3), (300, 5), (1000, 16), (600, 512), (2000, 2), (4099, 7)])
def test_fast_kernels_equal_scalar_oracle(n, d, oracle_mod):
    """ocf_* (vectorised across pairs) == the scalar restatement, bit for bit:
    the flat numpy sum, omega, and each row's K nearest (d, j)."""
    pts, _ = oracle_mod.generate_random(n, d, 5, 1)
    s = oracle_mod.flat_distance_sum(pts)
    assert oracle_mod.flat_distance_sum_fast(pts) == s
    sigma = s / (n * (n - 1))
    om, _ = oracle_mod.row_folds(pts, sigma)
    K = 8
    om2, kd, kj = oracle_mod.omega_knn(pts, sigma, K)
    assert np.array_equal(bits(om), bits(om2))
    D = oracle_mod.distance_rows(pts, 0, n)
    np.fill_diagonal(D, np.inf)
    want = np.argsort(D, axis=1, kind="stable")[:, :min(K, n - 1)]
    assert np.array_equal(kj[:, :want.shape[1]], want)
    assert np.array_equal(bits(kd[:, :want.shape[1]]), bits(np.take_along_axis(D, want, 1)))


@pytest.mark.parametrize("n,d,k,seed", [(300, 5, 4, 0), (2000, 2, 3, 0), (1500, 64, 20, 0),
                                        (600, 512, 50, 0), (5000, 16, 10, 3)])
def test_full_oracle_equals_scalar_oracle(n, d, k, seed, oracle_mod):
    """run_pipeline_full (certified Boruvka + rooting) == run_pipeline (Prim)."""
    pts, _ = oracle_mod.generate_random(n, d, k, seed)
    a = oracle_mod.run_pipeline(pts, k)
    b = oracle_mod.run_pipeline_full(pts, k).out
    assert a.sigma == b.sigma
    for name in ("parent", "depth", "child_id", "bfs_order"):
        assert np.array_equal(getattr(a.tree, name), getattr(b.tree, name)), name
    assert np.array_equal(bits(a.tree.parent_flow), bits(b.tree.parent_flow))
    assert np.array_equal(bits(a.omega), bits(b.omega))
    assert np.array_equal(a.result.labels, b.result.labels)
    assert a.result.miso == b.result.miso
    assert [m for m, _ in a.result.trace] == [m for m, _ in b.result.trace]


def test_full_oracle_rejects_ties(oracle_mod):
    """Integer lattice: many exact ties -> no uniqueness certificate."""
    g = np.arange(12, dtype=np.float64)
    pts = np.stack(np.meshgrid(g, g), -1).reshape(-1, 2)
    with pytest.raises(oracle_mod.TieError):
        oracle_mod.run_pipeline_full(pts, 3)


def test_full_oracle_matches_reference_16000(oracle_mod):
    """Pinned at SURVEY §7's size: the whole reference pipeline at N=16,000,
    d=64, k=20 (tests/golden/large_n16000_d64_k20.json, produced by the
    reference itself, tools/gen_golden_large.py) equals the full-size oracle
    in every field (sigma, dsum-derived sigma, tree arrays, omega, extrema,
    labels, cut, eta, sparsities, trace, alpha/beta, miso, tree weight).
    The 32,000 and 46,340 references are checked the same way by
    tools/oracle_full.py --check (8 s / 25 s on 8 cores; evidence in
    profiles/round2_oracle_pins.jsonl) and on the GPU side by
    tests/test_gpu_fullsize.py."""
    import digest as dg
    import os
    want = dg.load(os.path.join(os.path.dirname(__file__), "golden", "large_n16000_d64_k20.json"))
    meta = want["meta"]
    pts, _ = oracle_mod.generate_random(meta["n"], meta["d"], meta["k"], meta["seed"])
    run = oracle_mod.run_pipeline_full(pts, meta["k"])
    o = run.out
    e = o.extrema
    got = dg.result_digest(o.result, sigma=o.sigma, tree=o.tree, omega=o.omega, p=o.p,
                           extrema=[e.phi_star_sum, e.phi_star_min, e.omega_star_sum, e.omega_star_min,
                                    e.p_star_sum, e.p_star_min],
                           total_distance=run.total_distance)
    got["dsum"] = dg.fbits(oracle_mod.flat_distance_sum_fast(pts))
    assert dg.compare(got, want) == []
    assert len([k for k in want if k in got]) >= 24


@pytest.mark.parametrize("name", ["ties_lattice_n700_root5", "ties_round2_row_tie", "ties_round1_square_sigma1"])
def test_oracle_prim_tie_rule_matches_reference(name, oracle_mod):
    """The scalar oracle's Prim follows the reference's tie rule on tied
    inputs (tools/gen_golden_ties.py fixtures)."""
    g = load(os.path.join(os.path.dirname(__file__), "golden", f"{name}.npz"))
    t = oracle_mod.prim_mst(g["points"], float(g["sigma"]), int(g["root"]))
    for f in ("parent", "depth", "child_id", "bfs_order"):
        assert np.array_equal(getattr(t, f), g[f]), f
    assert np.array_equal(bits(t.parent_flow), bits(g["parent_flow"]))


def test_tie_constructions_first_tie_round(oracle_mod):
    """The constructed instances tie FIRST in the round they target (the
    certified Boruvka reports the round of its first tie)."""
    for name, rnd in [("ties_round2_row_tie", 2), ("ties_round1_square_sigma1", 1)]:
        g = load(os.path.join(os.path.dirname(__file__), "golden", f"{name}.npz"))
        with pytest.raises(oracle_mod.TieError, match=f"round {rnd}$"):
            oracle_mod.run_pipeline_full(g["points"], int(g["k"]), root=int(g["root"]))


def test_full_c1_fixture_is_the_reference_run():
    """The C1 oracle digest (tests/golden/full_c1.json, bench.py's C1 parity
    check) agrees with the reference's own C1 run (pipe_c1_seed0.npz)."""
    import digest as dg
    here = os.path.dirname(__file__)
    want = dg.load(os.path.join(here, "golden", "full_c1.json"))
    g = load(os.path.join(here, "golden", "pipe_c1_seed0.npz"))
    assert want["sigma"] == dg.fbits(float(g["sigma"]))
    assert want["miso"] == dg.fbits(float(g["miso"]))
    assert want["iterations"] == int(g["iterations"])
    assert want["labels"] == dg.ahash("labels", g["labels"])
    assert want["parent"] == dg.ahash("parent", g["parent"])
    assert want["omega"] == dg.ahash("omega", g["omega"])
    assert want["trace_mid"] == [dg.fbits(m) for m in g["trace_mid"]]
