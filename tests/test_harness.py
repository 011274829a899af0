"""Host harness (paper_1702_04739_b200/harness.py) against fixtures produced by
the reference's own dataset.py / evaluation.py / parengine.py
(tools/gen_golden_harness.py).  CPU only."""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, load

import paper_1702_04739_b200 as pkg

G = load(os.path.join(GOLDEN, "harness.npz"))


def test_generate_random_and_standardize_bitwise():
    for i in range(3):
        n, d, k, seed, spread = G[f"gen{i}_args"]
        pts, lab = pkg.generate_random(int(n), int(d), int(k), int(seed), float(spread))
        assert pts.tobytes() == G[f"gen{i}_points"].tobytes()
        assert np.array_equal(lab, G[f"gen{i}_labels"]) and lab.dtype == np.int64
        assert pkg.standardize(pts).tobytes() == G[f"gen{i}_std"].tobytes()
    assert np.array_equal(pkg.standardize([[1.0, 5.0], [2.0, 5.0], [4.0, 5.0]]), G["std_const"])


def test_generate_random_guards():
    for args, msg in [((5, 2, 0, 0), "k must be >= 1"), ((2, 2, 3, 0), "n must be >= max"),
                      ((5, 0, 2, 0), "d must be >= 1")]:
        with pytest.raises(ValueError, match=msg):
            pkg.generate_random(*args)
    with pytest.raises(ValueError, match="spread must be > 0"):
        pkg.generate_random(5, 2, 2, 0, spread=0.0)
    with pytest.raises(ValueError, match="2-d"):
        pkg.standardize(np.zeros(3))


def test_misclassification_rate_matches_reference():
    for i in range(6):
        got = pkg.misclassification_rate(G[f"mis{i}_pred"], G[f"mis{i}_truth"])
        assert got == float(G[f"mis{i}_rate"])
    assert pkg.misclassification_rate([0, 0, 0], [0, 1, 1]) == 1.0
    assert pkg.misclassification_rate([2, 2, 1], [0, 0, 1]) == 0.0
    with pytest.raises(ValueError, match="equal length"):
        pkg.misclassification_rate([1, 2], [0])
    with pytest.raises(ValueError, match=">= 0"):
        pkg.misclassification_rate([-1, 1], [0, 1])
    with pytest.raises(ValueError, match="contiguous"):
        pkg.misclassification_rate([1, 1], [0, 2])


def test_points_io_round_trip(tmp_path):
    ref_csv = os.path.join(GOLDEN, "harness_points.csv")
    pts, lab = pkg.generate_random(12, 3, 3, 5)
    out = tmp_path / "p.csv"
    pkg.save_points(str(out), pts, lab)
    assert out.read_bytes() == open(ref_csv, "rb").read()
    x, y = pkg.load_points(ref_csv, label_column=3)
    assert x.tobytes() == pts.tobytes() and y.tolist() == [0, 1, 2] * 4
    ws = tmp_path / "w.txt"
    pkg.save_points(str(ws), pts, format="whitespace")
    x2, none = pkg.load_points(str(ws), format="whitespace")
    assert none is None and x2.tobytes() == pts.tobytes()
    hdr = tmp_path / "h.csv"
    hdr.write_text("x,y,cls\n1,2,a\n\n3,4,b\n5,6,a\n")
    x3, y3 = pkg.load_points(str(hdr), label_column=2, header=True)
    assert x3.tolist() == [[1, 2], [3, 4], [5, 6]] and y3.tolist() == [0, 1, 0]
    lf = tmp_path / "l.txt"
    pkg.save_labels(str(lf), np.array([3, 0, 1]))
    assert pkg.load_labels(str(lf)).tolist() == [3, 0, 1]


@pytest.mark.parametrize("text,kw,msg", [
    ("1,2\n3\n", {}, "row 2: expected 2 columns, found 1"),
    ("1,2\n3,x\n", {}, r"row 2, column 2: could not parse 'x'"),
    ("1,2\n3,inf\n", {}, "non-finite value 'inf'"),
    ("1,2\n", {}, "need at least 2 data rows, found 1"),
    ("a\nb\n", {"label_column": 0}, "rows contain no coordinate columns"),
    ("1,2\n3,4\n", {"label_column": 5}, "label column 5 out of range for 2-column data"),
])
def test_load_points_errors(tmp_path, text, kw, msg):
    f = tmp_path / "bad.csv"
    f.write_text(text)
    with pytest.raises(pkg.DataFormatError, match=msg):
        pkg.load_points(str(f), **kw)
    with pytest.raises(ValueError, match="unknown format"):
        pkg.load_points(str(f), format="tsv")


def test_bench_csv_format(tmp_path):
    r = pkg.BenchRecord("rand-n10-d2-k2-s0", 10, 2, 2, "seq", 1, 1.23456, 2.0, 3.0, 6.5, 0.125, None)
    f = tmp_path / "b.csv"
    pkg.write_bench_csv([r], str(f))
    assert f.read_text() == (pkg.BENCH_CSV_HEADER + "\n"
                             "rand-n10-d2-k2-s0,10,2,2,seq,1,1.235,2.000,3.000,6.500,0.125,\n")
    with pytest.raises(ValueError, match="repetitions"):
        pkg.benchmark([10], [2], [2], ["seq"], [0], repetitions=0)


def test_depth_schedule_matches_reference(oracle_mod):
    for i in range(4):
        t = oracle_mod.tree_from_parent_list(G[f"ds{i}_parent"], G[f"ds{i}_flows"])
        ds = pkg.DepthSchedule.from_tree(t)
        assert ds.depths == G[f"ds{i}_depths"].tolist()
        assert np.array_equal(np.concatenate(ds.canonical_order), G[f"ds{i}_canonical"])
        assert [len(c) for c in ds.canonical_order] == G[f"ds{i}_canon_len"].tolist()
        groups = [g for lvl in ds.levels for g in lvl]
        assert np.array_equal(np.concatenate(groups), G[f"ds{i}_groups"])
        assert [len(g) for g in groups] == G[f"ds{i}_group_len"].tolist()
        assert [len(lvl) for lvl in ds.levels] == G[f"ds{i}_level_groups"].tolist()


def test_worker_pool_ordered():
    for w in (1, 3):
        assert pkg.WorkerPool(w).map(lambda c: c * c, range(7)) == [c * c for c in range(7)]
    with pytest.raises(ValueError):
        pkg.WorkerPool(0)
    assert math.isfinite(pkg.WorkerPool().workers)
