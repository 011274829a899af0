"""brute_force_miso on the device (isoperim.py:324-390) against the
reference's own results (tests/golden/brute_force.npz, tools/gen_golden_brute.py)
and its known answers (reference tests/test_isoperim.py:194-225)."""
from __future__ import annotations

import itertools
import math

import numpy as np
import pytest

from conftest import GOLDEN, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_1702_04739_b200 as p
    return p


def _records():
    g = load(f"{GOLDEN}/brute_force.npz")
    return [{k.split("_", 1)[1]: v for k, v in g.items() if k.startswith(f"t{i}_")} for i in range(int(g["count"]))]


def _path(pkg):
    tree = pkg.tree_from_parent_list([1, 2, pkg.NO_VERTEX], [1.0, 0.1, 0.0])
    return tree, pkg.NodeWeights(omega=np.ones(3), p=np.zeros(3), sigma=1.0, alpha=0.0)


def test_known_answers(pkg):
    tree, w = _path(pkg)
    res = pkg.brute_force_miso(tree, w, 2)
    assert res.miso == 0.1
    assert res.outcome is None and res.iterations == 0 and res.trace == []
    assert res.alpha_final == res.beta_final == res.miso
    one = pkg.tree_from_parent_list([pkg.NO_VERTEX, 0], [0.0, 0.8])
    w1 = pkg.NodeWeights(omega=np.ones(2), p=np.zeros(2), sigma=1.0, alpha=0.0)
    assert pkg.brute_force_miso(one, w1, 1).miso == 0.0


def test_guards(pkg):
    tree, w = _path(pkg)
    with pytest.raises(pkg.InfeasibleSubpartitionError):
        pkg.brute_force_miso(tree, w, 4)
    with pytest.raises(TypeError):
        pkg.brute_force_miso(tree, w, 2.0)
    rng = np.random.default_rng(3)
    parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, 13)])
    big = pkg.tree_from_parent_list(parent, np.r_[0.0, rng.random(12)])
    wb = pkg.NodeWeights(omega=np.ones(13), p=np.zeros(13), sigma=1.0, alpha=0.0)
    with pytest.raises(ValueError, match="n <= 12"):
        pkg.brute_force_miso(big, wb, 2)


def test_matches_reference_goldens(pkg):
    recs = _records()
    assert len(recs) == 48
    for rec in recs:
        k = int(rec["k"])
        tree = pkg.tree_from_parent_list(rec["parent"], rec["flows"])
        w = pkg.NodeWeights(omega=rec["omega"], p=rec["p"], sigma=1.0, alpha=0.0)
        assert int(rec["ok"]) == 1
        res = pkg.brute_force_miso(tree, w, k)
        assert np.array_equal(res.labels, rec["labels"])
        assert res.miso == float(rec["miso"])


def _python_cost(lab, parent, flows, omega, p, k):
    worst = -math.inf
    for c in range(1, k + 1):
        mem = {i for i in range(len(lab)) if lab[i] == c}
        bnd = [flows[u] for u in range(len(lab)) if parent[u] != -1 and ((u in mem) != (parent[u] in mem))]
        worst = max(worst, (math.fsum(bnd) + math.fsum(p[i] for i in mem)) / math.fsum(omega[i] for i in mem))
    return worst


def test_matches_plain_enumeration(pkg):
    """reference tests/test_isoperim.py:217-225, with an itertools enumeration."""
    rng = np.random.default_rng(11)
    for _ in range(12):
        n = int(rng.integers(3, 7))
        k = int(rng.integers(1, 4))
        parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, n)])
        flows = np.r_[0.0, rng.uniform(0.05, 1.0, n - 1)]
        omega, p = rng.uniform(0.5, 2.0, n), rng.uniform(0.0, 0.3, n)
        tree = pkg.tree_from_parent_list(parent, flows)
        w = pkg.NodeWeights(omega=omega, p=p, sigma=1.0, alpha=1.0)
        best = min(_python_cost(lab, parent, flows, omega, p, k)
                   for lab in itertools.product(range(k + 1), repeat=n)
                   if all(c in lab for c in range(1, k + 1)))
        assert math.isclose(pkg.brute_force_miso(tree, w, k).miso, best, rel_tol=1e-12)


def test_largest_enumeration(pkg):
    """n = 12, k = 3: 4^12 = 16.8M labellings, every cluster recomputed."""
    rng = np.random.default_rng(12)
    parent = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, 12)])
    flows = np.r_[0.0, rng.uniform(0.05, 1.0, 11)]
    tree = pkg.tree_from_parent_list(parent, flows)
    w = pkg.NodeWeights(omega=rng.uniform(0.5, 2.0, 12), p=np.zeros(12), sigma=1.0, alpha=0.0)
    res = pkg.brute_force_miso(tree, w, 3)
    assert sorted(set(res.labels.tolist()) - {0}) == [1, 2, 3]
    assert res.miso == pkg.subpartition_cost(res.labels, tree, w)
    ext = pkg.extrema(tree, w)
    assert pkg.solve_miso(tree, w, ext, 3).miso >= res.miso * (1 - 1e-12)
