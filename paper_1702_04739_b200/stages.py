"""The reference's stage-level API on dense inputs, computed on the device.

isoclust exports stage functions that take a distance matrix
(/root/reference/pkg/src/isoclust/__init__.py:71-122): distance_matrix,
flow, vertex_weights, potentials, auto_sigma, node_weights,
validate_distance_matrix, prim_mst, total_distance, reverse_bfs_order, the
deterministic primitives sum_reduce / min_reduce / exclusive_scan, and the
witness helpers extract_labels / subpartition_cost.  These are the same
signatures, argument meanings and exceptions, backed by the kernels in
csrc/stages.cu (the matrix-free pipeline in pipeline.py never builds the
n x n matrix; these serve callers that hold one).  Results are bit-identical
to the reference in numpy's pinned exp mode.
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional

import numpy as np

from ._lib import check
from .engine import _ptr
from .pipeline import _rooted_tree_view, _validate_points, _device_tree, backend
from .types import NO_VERTEX, DecisionOutcome, NodeWeights, RootedTree

# affinity.py:23-24 -- beyond this the dense float64 matrix exceeds 16 GiB
MAX_POINTS = 46340


def _dev(a: np.ndarray, dtype):
    return backend().to_device(np.ascontiguousarray(a, dtype=dtype))


def _host(t) -> np.ndarray:
    return t.cpu().numpy()


def _check_matrix_shape(dist) -> np.ndarray:
    """affinity.py:84-98: square, at least 2 points, zero diagonal."""
    d = np.ascontiguousarray(dist, dtype=np.float64)
    if d.ndim != 2 or d.shape[0] != d.shape[1]:
        raise ValueError(f"distance matrix must be square, got shape {d.shape}")
    if d.shape[0] < 2:
        raise ValueError("distance matrix needs at least 2 points")
    if (np.diagonal(d) != 0).any():
        raise ValueError("distance matrix must have a zero diagonal")
    return d


def distance_matrix(points, *, workers: Optional[int] = None, max_points: int = MAX_POINTS) -> np.ndarray:
    """affinity.py:124-158: all pairwise Euclidean distances (scipy's
    operation order, exactly symmetric, zero diagonal), on the device."""
    x = _validate_points(points)
    n, d = x.shape
    if n > max_points:
        raise ValueError(
            f"n={n} exceeds the dense-matrix cap of {max_points} points "
            f"({8 * n * n / 2**30:.1f} GiB would be required)")
    b = backend()
    X = b.to_device(x)
    D = b.empty((n, n), b.torch.float64)
    check(b.lib.isoc_distance_matrix(_ptr(X), n, d, _ptr(D), b.stream))
    return _host(D)


def flow(distance, sigma: float):
    """affinity.py:161-172: exp(-d / sigma) (glibc exp, bitwise)."""
    if not (sigma > 0):
        raise ValueError(f"sigma must be > 0, got {sigma}")
    d = np.asarray(distance, dtype=np.float64)
    if (d < 0).any():
        raise ValueError("distance must be nonnegative")
    flat = np.ascontiguousarray(d.reshape(-1))
    b = backend()
    out = np.empty_like(flat)
    if flat.size:
        dv = b.to_device(flat)
        ov = b.empty((flat.size,), b.torch.float64)
        check(b.lib.isoc_flow(_ptr(dv), flat.size, float(sigma), _ptr(ov), b.stream))
        out = _host(ov)
    result = out.reshape(d.shape)
    return float(result) if np.isscalar(distance) or d.ndim == 0 else result


def vertex_weights(dist, sigma: float, *, workers: Optional[int] = None) -> np.ndarray:
    """affinity.py:175-201: omega[i] = pow2 fold over j != i of exp(-d_ij/sigma)."""
    d = _check_matrix_shape(dist)
    if not (sigma > 0):
        raise ValueError(f"sigma must be > 0, got {sigma}")
    b = backend()
    D = b.to_device(d)
    out = b.empty((d.shape[0],), b.torch.float64)
    check(b.lib.isoc_vertex_weights_dense(_ptr(D), d.shape[0], float(sigma), _ptr(out), b.stream))
    return _host(out)


def potentials(dist, alpha: float, *, workers: Optional[int] = None) -> np.ndarray:
    """affinity.py:204-230: p[i] = alpha * pow2 fold of row i (exact zeros at alpha = 0)."""
    d = _check_matrix_shape(dist)
    if alpha < 0:
        raise ValueError(f"alpha must be >= 0, got {alpha}")
    n = d.shape[0]
    if alpha == 0:
        return np.zeros(n, dtype=np.float64)
    b = backend()
    D = b.to_device(d)
    out = b.empty((n,), b.torch.float64)
    check(b.lib.isoc_potentials_dense(_ptr(D), n, float(alpha), _ptr(out), b.stream))
    return _host(out)


def auto_sigma(dist) -> float:
    """affinity.py:233-241: mean off-diagonal distance, float(d.sum()) / (n(n-1))
    with numpy's pairwise summation over the flat matrix."""
    d = _check_matrix_shape(dist)
    n = d.shape[0]
    b = backend()
    D = b.to_device(d)
    total = ctypes.c_double()
    check(b.lib.isoc_pairwise_sum(_ptr(D), n * n, ctypes.byref(total), b.stream))
    mean = float(total.value) / (n * (n - 1))
    if not (mean > 0):
        raise ValueError("all points coincide; no usable distance scale")
    return mean


def node_weights(dist, sigma: float, alpha: float = 0.0, *, workers: Optional[int] = None) -> NodeWeights:
    """affinity.py:244-257: vertex_weights and potentials of one matrix."""
    return NodeWeights(omega=vertex_weights(dist, sigma), p=potentials(dist, alpha),
                       sigma=float(sigma), alpha=float(alpha))


def validate_distance_matrix(dist) -> np.ndarray:
    """affinity.py:101-121: square, zero diagonal, finite, nonnegative, exactly symmetric."""
    d = _check_matrix_shape(dist)
    b = backend()
    D = b.to_device(d)
    flags = ctypes.c_int32()
    check(b.lib.isoc_validate_distance_matrix(_ptr(D), d.shape[0], ctypes.byref(flags), b.stream))
    f = flags.value
    if f & 1:
        raise ValueError("distance matrix must be finite")
    if f & 2:
        raise ValueError("distances must be nonnegative")
    if f & 4:
        raise ValueError("distance matrix must be exactly symmetric")
    return d


def prim_mst(dist, sigma: float, root: int = 0) -> RootedTree:
    """mst.py:128-181 on a distance matrix: the minimum spanning tree rooted at
    `root` with Prim's sibling ranks and parent flows.  Built by lexicographic
    Boruvka on the device (the same tree as Prim for distinct distances); when
    a round saw an exact tie at a component minimum, Prim itself is replayed
    on the matrix (isoc_prim_edges_dense), so ties follow the reference's rule."""
    d = validate_distance_matrix(dist)
    if not (sigma > 0):
        raise ValueError(f"sigma must be > 0, got {sigma}")
    n = d.shape[0]
    if not (0 <= root < n):
        raise ValueError(f"root must be in [0, {n}), got {root}")
    b = backend()
    torch = b.torch
    D = b.to_device(d)
    u = b.empty((n - 1,), torch.int32)
    v = b.empty((n - 1,), torch.int32)
    w = b.empty((n - 1,), torch.float64)
    ties = ctypes.c_int64()
    check(b.lib.isoc_mst_dense(_ptr(D), n, _ptr(u), _ptr(v), _ptr(w), ctypes.byref(ties), b.stream))
    if ties.value:
        # an exact tie at a component minimum: replay the reference's Prim on
        # the matrix (frontier ties -> smallest vertex, strict `<` relaxation)
        check(b.lib.isoc_prim_edges_dense(_ptr(D), n, root, _ptr(u), _ptr(v), _ptr(w), b.stream))
    dt = b.tree_from_edges(u, v, w, n, root, sigma)
    return _rooted_tree_view(dt, root)


def total_distance(tree: RootedTree, dist=None) -> float:
    """mst.py:184-187: math.fsum of the tree-edge distances.  With `dist` the
    distances are read from the matrix as the reference does; without it,
    from the exact parent-edge distances the device tree holds (matrix-free)."""
    nonroot = np.flatnonzero(tree.parent != NO_VERTEX)
    if dist is not None:
        return math.fsum(float(dist[u, tree.parent[u]]) for u in nonroot)
    pdist = _device_tree(tree).export()[6]
    return math.fsum(float(pdist[u]) for u in nonroot)


def reverse_bfs_order(tree: RootedTree) -> np.ndarray:
    """mst.py:68-75: leaves first, root last (the device tree's BFS order,
    children in child_id order, reversed)."""
    return np.array(tree.bfs_order, dtype=np.int64, copy=True)


def sum_reduce(values, pool=None) -> float:
    """_primitives.py:95-124: pow2 zero-padded adjacent-pair fold."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim != 1:
        raise ValueError(f"sum_reduce expects a 1-d array, got shape {v.shape}")
    if v.size == 0:
        raise ValueError("sum_reduce of an empty array")
    b = backend()
    out = ctypes.c_double()
    dv = b.to_device(v)
    check(b.lib.isoc_sum_reduce(_ptr(dv), v.size, ctypes.byref(out), b.stream))
    return float(out.value)


def min_reduce(values) -> tuple[float, int]:
    """_primitives.py:69-92: minimum and the smallest index attaining it."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim != 1:
        raise ValueError(f"min_reduce expects a 1-d array, got shape {v.shape}")
    if v.size == 0:
        raise ValueError("min_reduce of an empty array")
    b = backend()
    val, idx = ctypes.c_double(), ctypes.c_int64()
    dv = b.to_device(v)
    check(b.lib.isoc_min_reduce(_ptr(dv), v.size, ctypes.byref(val), ctypes.byref(idx), b.stream))
    return float(val.value), int(idx.value)


def exclusive_scan(values) -> np.ndarray:
    """_primitives.py:127-159: exclusive prefix sum of nonnegative integers."""
    a = np.asarray(values)
    if a.ndim != 1:
        raise ValueError(f"exclusive_scan expects a 1-d array, got shape {a.shape}")
    if a.size == 0:
        return np.zeros(0, dtype=np.int64)
    if not np.issubdtype(a.dtype, np.integer):
        raise TypeError(f"exclusive_scan expects integers, got dtype {a.dtype}")
    if (a < 0).any():
        raise ValueError("exclusive_scan requires nonnegative values")
    b = backend()
    src = b.to_device(a.astype(np.int64))
    out = b.empty((a.size,), b.torch.int64)
    check(b.lib.isoc_exclusive_scan(_ptr(src), a.size, _ptr(out), b.stream))
    return _host(out)


def extract_labels(outcome: DecisionOutcome, k: int) -> np.ndarray:
    """isoperim.py:164-181: labels 1..k by ascending cut-vertex index, 0 = residual."""
    if not outcome.feasible:
        raise ValueError("labels can only be extracted from a feasible outcome")
    if outcome.clusters_found != k:
        raise ValueError(f"outcome has {outcome.clusters_found} clusters, expected {k}")
    n = outcome.cut.shape[0]
    b = backend()
    cut = b.to_device(np.ascontiguousarray(outcome.cut, dtype=np.int8))
    eta = b.to_device(np.ascontiguousarray(outcome.eta, dtype=np.int64))
    out = b.empty((n,), b.torch.int64)
    check(b.lib.isoc_extract_labels(_ptr(cut), _ptr(eta), n, _ptr(out), b.stream))
    return _host(out)


def subpartition_cost(labels, tree: RootedTree, weights: NodeWeights) -> float:
    """isoperim.py:184-219: worst (boundary flow + potential) / mass over the
    clusters 1..k, with numpy's pairwise sums per cluster (device kernels)."""
    lab = np.asarray(labels, dtype=np.int64)
    if lab.ndim != 1 or lab.shape[0] != tree.n:
        raise ValueError(f"labels must be a length-{tree.n} array")
    if weights.n != tree.n:
        raise ValueError("weights and tree vertex counts differ")
    if (lab < 0).any():
        raise ValueError("labels must be nonnegative")
    k = int(lab.max())
    if k < 1:
        raise ValueError("no clusters: labels contain no value >= 1")
    sizes = np.bincount(lab, minlength=k + 1)
    empty = np.flatnonzero(sizes[1:] == 0)
    if empty.size:
        raise ValueError(f"cluster label {int(empty[0]) + 1} is empty")
    from .pipeline import _attach
    dt = _attach(tree, weights)
    return dt.cost(lab, k)


def brute_force_miso(tree: RootedTree, weights: NodeWeights, k: int):
    """isoperim.py:324-390: exhaustive search over every labelling of the
    vertices into {0, 1..k} (clusters need not be connected), for tiny
    instances (n <= 12, at most 2^26 labellings).  The enumeration runs on
    the device (brute_force_kernel, one labelling per thread); the winner is
    the smallest labelling code with the minimum worst sparsity, and miso is
    its exact cost recomputed by subpartition_cost, as in the reference."""
    from .pipeline import _validate_k
    from .types import MisoResult

    _validate_k(k)
    if tree.n != weights.n:
        raise ValueError(f"tree has {tree.n} vertices but weights have {weights.n}")
    n = tree.n
    if n > 12:
        raise ValueError(f"brute force supports n <= 12, got {n}")
    if k > n:
        from ._lib import InfeasibleSubpartitionError
        raise InfeasibleSubpartitionError(
            f"no feasible labeling: k={k} clusters require k <= n={n} vertices")
    if (k + 1) ** n > 1 << 26:
        raise ValueError(f"enumeration of {(k + 1) ** n} labelings exceeds the supported size")
    parent = np.where(np.asarray(tree.parent) == NO_VERTEX, -1, np.asarray(tree.parent))
    b = backend()
    code, worst = ctypes.c_int64(), ctypes.c_double()
    bufs = (_dev(parent, np.int32), _dev(tree.parent_flow, np.float64), _dev(weights.omega, np.float64),
            _dev(weights.p, np.float64))   # held until the call returns
    check(b.lib.isoc_brute_force_miso(*map(_ptr, bufs), n, int(k), ctypes.byref(code), ctypes.byref(worst),
                                      b.stream))
    if code.value < 0:
        from ._lib import InfeasibleSubpartitionError
        raise InfeasibleSubpartitionError(f"no feasible labeling found by enumeration (n={n}, k={k})")
    labels = (code.value // (k + 1) ** np.arange(n, dtype=np.int64)) % (k + 1)
    exact = subpartition_cost(labels, tree, weights)
    return MisoResult(miso=exact, labels=labels.astype(np.int64), outcome=None, iterations=0,
                      alpha_final=exact, beta_final=exact, trace=[])
