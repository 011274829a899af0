"""Host-side API mirrors the reference (no GPU needed): names, schema, errors
raised before any device work, worker resolution (pipeline.py / _primitives.py)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1702_04739_b200 as pkg
from paper_1702_04739_b200 import pipeline as pl
from paper_1702_04739_b200.types import DecisionOutcome, MisoResult, PipelineRun

REFERENCE_NAMES = [  # isoclust/__init__.py:71-122, the clustering-path subset
    "DecisionOutcome", "Extrema", "InfeasibleSubpartitionError", "MisoResult", "NO_VERTEX", "NodeWeights",
    "PipelineRun", "RootedTree", "WORKERS_ENV_VAR", "auto_sigma", "decide", "extrema", "miso_results_equal",
    "node_weights", "outcomes_equal", "par_decide", "par_solve_miso", "prim_mst", "resolve_workers",
    "run_pipeline", "solve_miso", "summarize", "total_distance", "tree_from_parent_list",
    "distance_matrix", "flow", "vertex_weights", "potentials", "sum_reduce", "min_reduce", "exclusive_scan",
    "extract_labels", "subpartition_cost", "reverse_bfs_order",
]


def test_reference_names_exported():
    for name in REFERENCE_NAMES:
        assert hasattr(pkg, name), name


def test_engine_rejected_before_device_use():
    with pytest.raises(ValueError):
        pkg.run_pipeline(np.zeros((4, 2)), 2, engine="gpu")


def test_point_validation_matches_reference():
    for bad in (np.zeros(5), np.zeros((1, 3)), np.zeros((4, 0)), np.array([[0.0, np.inf], [1.0, 2.0]])):
        with pytest.raises(ValueError):
            pl._validate_points(bad)


def test_k_validation():
    with pytest.raises(TypeError):
        pl._validate_k(2.0)
    with pytest.raises(TypeError):
        pl._validate_k(True)
    with pytest.raises(ValueError):
        pl._validate_k(0)
    pl._validate_k(np.int64(3))


def test_resolve_workers(monkeypatch):
    monkeypatch.setenv(pkg.WORKERS_ENV_VAR, "3")
    assert pkg.resolve_workers() == 3
    assert pkg.resolve_workers(5) == 5
    monkeypatch.setenv(pkg.WORKERS_ENV_VAR, "x")
    with pytest.raises(ValueError):
        pkg.resolve_workers()
    with pytest.raises(ValueError):
        pkg.resolve_workers(0)


def test_summarize_schema_matches_reference():
    labels = np.array([1, 1, 0, 2, 2, 2])
    res = MisoResult(miso=0.25, labels=labels, outcome=None, iterations=50, alpha_final=0.1,
                     beta_final=0.2, trace=[])
    run = PipelineRun(result=res, n=6, d=2, k=2, sigma=1.5, alpha=0.0, root=0, engine="seq", workers=1,
                      timings_ms={"affinity": 1.0, "mst": 2.0, "partition": 3.0, "total": 6.0004})
    s = pkg.summarize(run)
    assert list(s) == ["schema", "n", "d", "k", "miso", "iterations", "alpha_final", "beta_final",
                       "cluster_sizes", "residual_count", "sigma", "alpha", "root", "engine", "workers",
                       "timings_ms"]
    assert s["cluster_sizes"] == [2, 3] and s["residual_count"] == 1
    assert s["timings_ms"]["total"] == 6.0


def test_equality_helpers():
    a = DecisionOutcome(True, 2, np.array([1, 0], np.int8), np.array([0, -1]), [0.5, 0.25])
    b = DecisionOutcome(True, 2, np.array([1, 0], np.int8), np.array([0, -1]), [0.5, 0.25])
    assert pkg.outcomes_equal(a, b)
    b.cluster_sparsities[1] = 0.26
    assert not pkg.outcomes_equal(a, b)


def test_node_weights_validation():
    with pytest.raises(ValueError):
        pkg.NodeWeights(omega=np.ones(3), p=np.zeros(2), sigma=1.0, alpha=0.0)
    with pytest.raises(ValueError):
        pkg.NodeWeights(omega=np.ones(3), p=np.zeros(3), sigma=0.0, alpha=0.0)
    with pytest.raises(ValueError):
        pkg.NodeWeights(omega=np.ones(3), p=np.zeros(3), sigma=1.0, alpha=-1.0)


def test_dense_stage_api_validation_before_device_use():
    """The matrix-taking stage functions raise the reference's errors
    (affinity.py:84-98, 161-230, _primitives.py:127-145, isoperim.py:164-219)
    before any device work."""
    from paper_1702_04739_b200 import stages
    for bad in (np.zeros((3, 4)), np.zeros((1, 1)), np.ones((3, 3))):
        with pytest.raises(ValueError):
            stages._check_matrix_shape(bad)
    with pytest.raises(ValueError):
        pkg.vertex_weights(np.zeros((3, 3)), 0.0)
    with pytest.raises(ValueError):
        pkg.potentials(np.zeros((3, 3)), -1.0)
    assert np.array_equal(pkg.potentials(np.zeros((3, 3)), 0.0), np.zeros(3))
    with pytest.raises(ValueError):
        pkg.flow(1.0, 0.0)
    with pytest.raises(ValueError):
        pkg.flow(np.array([-1.0]), 1.0)
    with pytest.raises(ValueError):
        pkg.distance_matrix(np.zeros((10, 2)), max_points=5)
    with pytest.raises(TypeError):
        pkg.exclusive_scan(np.array([1.5]))
    with pytest.raises(ValueError):
        pkg.exclusive_scan(np.array([-1]))
    assert pkg.exclusive_scan(np.zeros(0, np.int64)).shape == (0,)
    with pytest.raises(ValueError):
        pkg.sum_reduce(np.zeros(0))
    with pytest.raises(ValueError):
        pkg.min_reduce(np.zeros((2, 2)))
    out = DecisionOutcome(feasible=False, clusters_found=1, cut=np.zeros(3, np.int8),
                          eta=np.full(3, -1, np.int64), cluster_sparsities=[])
    with pytest.raises(ValueError):
        pkg.extract_labels(out, 1)
