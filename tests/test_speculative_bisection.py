"""Host logic of the speculative bisection (pipeline.run_bisection) on CPU.

A fake device tree answers decision sweeps from a monotone feasibility rule
(j = k iff N >= threshold) and counts sweeps; the speculative walk (m = 2..4)
must reproduce the sequential loop of isoperim.py:222-308 exactly: the same
trace, iterations, alpha/beta and witness threshold, with fewer sweeps.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1702_04739_b200 import pipeline
from paper_1702_04739_b200.types import Extrema


class FakeTree:
    def __init__(self, n, k, cut_at, levels=40, width=1000):
        self.n, self.k, self.cut_at = n, k, cut_at
        self.levels, self.width = levels, width
        self.sweeps = 0
        self.decided = []
        self.slot_thr = {}

    def shape(self):
        return self.levels, self.width

    def _j(self, N):
        return self.k if N >= self.cut_at else self.k - 1

    def decide(self, N, k, slot):
        self.sweeps += 1
        self.decided.append(N)
        self.slot_thr[slot] = N
        return self._j(N)

    def decide_batch(self, thresholds, k):
        self.sweeps += 1
        return [self._j(t) for t in thresholds]

    def witness(self, slot, k):
        class W:
            pass
        w = W()
        w.cut = np.zeros(self.n, np.int8)
        w.eta = np.full(self.n, -1, np.int64)
        w.sparsities = [self.slot_thr[slot]] * k
        w.labels = np.zeros(self.n, np.int64)
        w.miso = self.slot_thr[slot]
        return w


def sequential(ext, k, n, cut_at):
    """The reference loop, verbatim."""
    import math
    a0 = (ext.phi_star_min + ext.p_star_min) / ext.omega_star_sum
    b0 = (ext.phi_star_sum + ext.p_star_sum) / ext.omega_star_min
    if b0 > a0:
        t = max(math.ceil(math.log2(2.0 * ext.omega_star_sum ** 2 * (b0 - a0))
                          - math.log2(ext.phi_star_min + ext.p_star_min)),
                math.ceil(math.log2((b0 - a0) / (1e-15 * max(1.0, b0)))))
    else:
        t = 1
    t = min(128, max(1, t))
    a, b, trace, wit = a0, b0, [], None
    for _ in range(t):
        if b - a <= 1e-15 * max(1.0, b):
            break
        mid = (a + b) / 2.0
        ok = mid >= cut_at
        trace.append((mid, ok))
        if ok:
            b, wit = mid, mid
        else:
            a = mid
    return a, b, trace, wit


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("seed", range(12))
def test_speculative_walk_equals_sequential(m, seed, monkeypatch):
    monkeypatch.setenv("ISOC_SPEC_M", str(m))
    rng = np.random.default_rng(seed)
    n, k = 1000, 5
    ext = Extrema(phi_star_sum=float(rng.uniform(10, 100)), phi_star_min=float(rng.uniform(1e-6, 1e-2)),
                  omega_star_sum=float(rng.uniform(100, 1000)), omega_star_min=float(rng.uniform(0.1, 1.0)),
                  p_star_sum=0.0, p_star_min=0.0)
    a0 = ext.phi_star_min / ext.omega_star_sum
    b0 = ext.phi_star_sum / ext.omega_star_min
    cut_at = float(a0 + (b0 - a0) * rng.uniform(0.01, 0.99) ** 3)
    tree = FakeTree(n, k, cut_at)
    res = pipeline.run_bisection(tree, ext, k, n)
    a, b, trace, wit = sequential(ext, k, n, cut_at)
    assert res.trace == trace
    assert res.iterations == len(trace)
    assert res.alpha_final == a and res.beta_final == b
    assert res.miso == wit
    if m > 1:
        assert tree.sweeps < len(trace) + 1 or len(trace) <= 2


def test_speculation_depth_heuristic(monkeypatch):
    monkeypatch.delenv("ISOC_SPEC_M", raising=False)
    assert pipeline._speculation_depth(FakeTree(1_000_000, 5, 0.0, levels=200, width=20_000)) == 4
    assert pipeline._speculation_depth(FakeTree(50_000_000, 5, 0.0, levels=35, width=4_000_000)) == 1


def test_threshold_tree_walks_equal_recursive_build():
    """pipeline._threshold_tree (level order) offers the walk exactly the
    midpoints of the recursive preorder build, for every outcome pattern."""
    import random
    from paper_1702_04739_b200.pipeline import BRACKET_EPS, _threshold_tree

    def build_rec(a0, b0, depth):
        thr, kids = [], []

        def build(a, b, d):
            if d == 0 or b - a <= BRACKET_EPS * max(1.0, b):
                return -1
            mid = (a + b) / 2.0
            idx = len(thr)
            thr.append(mid)
            kids.append(None)
            kids[idx] = (build(a, mid, d - 1), build(mid, b, d - 1))
            return idx
        return thr, kids, build(a0, b0, depth)

    def walk(thr, kids, root, pat):
        node, out, bit = root, [], 0
        while node >= 0:
            ok = (pat >> bit) & 1
            bit += 1
            out.append(thr[node])
            node = kids[node][0] if ok else kids[node][1]
        return out

    rng = random.Random(3)
    for _ in range(500):
        a = rng.random() * rng.choice([1e-8, 1.0, 1e3])
        b = a + rng.random() * rng.choice([1e-20, 1e-14, 1e-6, 1.0, 10.0])
        d = rng.randint(1, 6)
        t1, k1, r1 = build_rec(a, b, d)
        t2, k2, r2 = _threshold_tree(a, b, d)
        assert sorted(t1) == sorted(t2)
        for pat in range(1 << d):
            assert walk(t1, k1, r1, pat) == walk(t2, k2, r2, pat)
