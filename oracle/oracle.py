"""CPU oracle for the isoperimetric-tree clustering path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline / --impl reference).  The product package never
imports this module.

The heavy arithmetic lives in isoc_oracle.c (restating the reference's
operation order bit for bit); this module restates the reference's Python
control flow on top of it:
  run_pipeline      /root/reference/pkg/src/isoclust/pipeline.py:41-104
  run_bisection     isoperim.py:222-308
  generate_random   dataset.py:140-168
  random_parent_array / random_instance   tests/conftest.py:35-70
Oracle results are pinned against fixtures produced by the reference itself
(tests/golden/, tools/gen_golden.py) in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

NO_VERTEX = -1
BRACKET_EPS = 1e-15
MAX_ITERATIONS = 128

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libisoc_oracle.so")
_lib = None


def build() -> str:
    """Compile libisoc_oracle.so (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double
        L.oc_exp.restype = D
        L.oc_exp.argtypes = [D]
        L.oc_exp_array.argtypes = [P, P, I64]
        L.oc_pair_distance.restype = D
        L.oc_pair_distance.argtypes = [P, I64, I64, I64]
        L.oc_distance_rows.argtypes = [P, I64, I64, I64, I64, P]
        L.oc_pairwise_sum.restype = D
        L.oc_pairwise_sum.argtypes = [P, I64]
        L.oc_flat_distance_sum.restype = D
        L.oc_flat_distance_sum.argtypes = [P, I64, I64]
        L.oc_row_folds.argtypes = [P, I64, I64, D, D, I64, I64, P, P]
        L.oc_sum_reduce.restype = D
        L.oc_sum_reduce.argtypes = [P, I64]
        L.oc_min_reduce.restype = D
        L.oc_min_reduce.argtypes = [P, I64, P]
        L.oc_prim.restype = ctypes.c_int
        L.oc_prim.argtypes = [P, I64, I64, I64, D, P, P, P, P, P, P]
        L.oc_tree_from_parent.restype = ctypes.c_int
        L.oc_tree_from_parent.argtypes = [P, I64, I64, P, P, P]
        L.oc_decide.restype = I64
        L.oc_decide.argtypes = [I64, I64, P, P, P, P, P, I64, D, P, P, P]
        L.oc_extract_labels.argtypes = [P, P, I64, P]
        L.oc_subpartition_cost.restype = D
        L.oc_subpartition_cost.argtypes = [P, I64, P, P, P, P]
        L.oc_num_threads.restype = ctypes.c_int
        L.oc_set_threads.argtypes = [ctypes.c_int]
        I = ctypes.c_int
        L.ocf_isa.restype = I
        L.ocf_flat_distance_sum.restype = D
        L.ocf_flat_distance_sum.argtypes = [P, I64, I]
        L.ocf_omega_knn.restype = I
        L.ocf_omega_knn.argtypes = [P, I64, I, D, I64, I64, I, P, P, P]
        L.ocf_rescan_rows.restype = I
        L.ocf_rescan_rows.argtypes = [P, I64, I, P, I64, P, I, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------------ data
def generate_random(n: int, d: int, k: int, seed: int, spread: float = 1.0):
    """dataset.py:140-168 (PCG64 blobs; point i in blob i % k)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    centers = rng.uniform(0.0, 10.0, size=(k, d))
    labels = np.arange(n, dtype=np.int64) % k
    points = centers[labels] + rng.normal(0.0, spread, size=(n, d))
    return points, labels


def random_parent_array(rng: np.random.Generator, n: int) -> np.ndarray:
    """tests/conftest.py:35-41 verbatim semantics (scalar draws; small n)."""
    parent = np.full(n, NO_VERTEX, dtype=np.int64)
    perm = rng.permutation(n)
    for i in range(1, n):
        parent[perm[i]] = perm[int(rng.integers(0, i))]
    return parent


def random_parent_array_fast(rng: np.random.Generator, n: int) -> np.ndarray:
    """C5 shape: the same recursive-tree law, vectorised as
    parent[perm[i]] = perm[floor(U_i * i)] so 50M vertices draw in seconds."""
    parent = np.full(n, NO_VERTEX, dtype=np.int64)
    perm = rng.permutation(n)
    if n > 1:
        i = np.arange(1, n, dtype=np.int64)
        picks = np.minimum((rng.random(n - 1) * i).astype(np.int64), i - 1)
        parent[perm[1:]] = perm[picks]
    return parent


def random_tree_instance(n: int, seed: int):
    """C5 generator: random recursive tree, flows 1-U[0,1),
    omega 2-U[0,1.9), p = 0 (tests/conftest.py:44-70 distributions)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    parent = random_parent_array_fast(rng, n)
    flows = np.zeros(n, dtype=np.float64)
    nonroot = parent != NO_VERTEX
    flows[nonroot] = 1.0 - rng.uniform(0.0, 1.0, int(nonroot.sum()))
    omega = 2.0 - rng.uniform(0.0, 1.9, n)
    p = np.zeros(n, dtype=np.float64)
    return parent, flows, omega, p


# ------------------------------------------------------------ structures
@dataclass
class Tree:
    parent: np.ndarray
    parent_flow: np.ndarray
    depth: np.ndarray
    child_id: np.ndarray
    bfs_order: np.ndarray
    root: int
    max_depth: int
    parent_dist: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return self.parent.shape[0]


@dataclass
class Extrema:
    phi_star_sum: float
    phi_star_min: float
    omega_star_sum: float
    omega_star_min: float
    p_star_sum: float
    p_star_min: float


@dataclass(eq=False)
class Outcome:
    feasible: bool
    clusters_found: int
    cut: np.ndarray
    eta: np.ndarray
    cluster_sparsities: list


@dataclass(eq=False)
class Result:
    miso: float
    labels: np.ndarray
    outcome: Optional[Outcome]
    iterations: int
    alpha_final: float
    beta_final: float
    trace: list = field(default_factory=list)


class InfeasibleSubpartitionError(RuntimeError):
    pass


# ------------------------------------------------------------- stages
def exp(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib().oc_exp_array(_p(x), _p(y), x.size)
    return y


def pair_distance(X: np.ndarray, i: int, j: int) -> float:
    X = np.ascontiguousarray(X, dtype=np.float64)
    return lib().oc_pair_distance(_p(X), X.shape[1], i, j)


def distance_rows(X: np.ndarray, lo: int, hi: int) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = np.empty((hi - lo, X.shape[0]), dtype=np.float64)
    lib().oc_distance_rows(_p(X), X.shape[0], X.shape[1], lo, hi, _p(out))
    return out


def pairwise_sum(a: np.ndarray) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().oc_pairwise_sum(_p(a), a.size)


def flat_distance_sum(X: np.ndarray) -> float:
    X = np.ascontiguousarray(X, dtype=np.float64)
    return lib().oc_flat_distance_sum(_p(X), X.shape[0], X.shape[1])


def auto_sigma(X: np.ndarray) -> float:
    """affinity.py:233-241 on the implicit distance matrix."""
    n = X.shape[0]
    total = flat_distance_sum(X)
    mean = total / (n * (n - 1))
    if not (mean > 0):
        raise ValueError("all points coincide; no usable distance scale")
    return mean


def row_folds(X: np.ndarray, sigma: float, alpha: float = 0.0, lo: int = 0, hi: Optional[int] = None):
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    hi = n if hi is None else hi
    omega = np.empty(hi - lo, dtype=np.float64)
    p = np.empty(hi - lo, dtype=np.float64)
    lib().oc_row_folds(_p(X), n, d, float(sigma), float(alpha), lo, hi, _p(omega), _p(p))
    return omega, p


def prim_mst(X: np.ndarray, sigma: float, root: int = 0) -> Tree:
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    parent = np.empty(n, np.int64)
    flow = np.empty(n, np.float64)
    depth = np.empty(n, np.int64)
    cid = np.empty(n, np.int64)
    order = np.empty(n, np.int64)
    pdist = np.empty(n, np.float64)
    rc = lib().oc_prim(_p(X), n, d, root, float(sigma), _p(parent), _p(flow), _p(depth), _p(cid),
                       _p(order), _p(pdist))
    if rc:
        raise ValueError("parent array does not describe one connected tree")
    return Tree(parent, flow, depth, cid, order, root, int(depth.max()), pdist)


def tree_from_parent_list(parent, parent_flow, root: Optional[int] = None) -> Tree:
    """mst.py:78-125."""
    par = np.ascontiguousarray(parent, dtype=np.int64).copy()
    flows = np.ascontiguousarray(parent_flow, dtype=np.float64).copy()
    n = par.shape[0]
    roots = np.flatnonzero(par == NO_VERTEX)
    if root is None:
        if roots.size != 1:
            raise ValueError(f"expected exactly one root sentinel, found {roots.size}")
        root = int(roots[0])
    flows[root] = 0.0
    depth = np.empty(n, np.int64)
    cid = np.empty(n, np.int64)
    order = np.empty(n, np.int64)
    if lib().oc_tree_from_parent(_p(par), n, root, _p(depth), _p(cid), _p(order)):
        raise ValueError("parent array does not describe one connected tree")
    return Tree(par, flows, depth, cid, order, root, int(depth.max()))


def sum_reduce(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().oc_sum_reduce(_p(a), a.size)


def min_reduce(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().oc_min_reduce(_p(a), a.size, None)


def extrema(tree: Tree, omega: np.ndarray, p: np.ndarray) -> Extrema:
    """affinity.py:260-279."""
    nonroot = np.arange(tree.n) != tree.root
    flows = np.ascontiguousarray(tree.parent_flow[nonroot])
    return Extrema(sum_reduce(flows), min_reduce(flows), sum_reduce(omega), min_reduce(omega),
                   sum_reduce(p), min_reduce(p))


def decide(tree: Tree, omega: np.ndarray, p: np.ndarray, k: int, N: float) -> Outcome:
    n = tree.n
    cut = np.zeros(n, np.int8)
    eta = np.empty(n, np.int64)
    sp = np.empty(max(k, 1), np.float64)
    om = np.ascontiguousarray(omega, dtype=np.float64)
    pp = np.ascontiguousarray(p, dtype=np.float64)
    j = lib().oc_decide(n, tree.root, _p(tree.parent), _p(tree.parent_flow), _p(tree.bfs_order),
                        _p(om), _p(pp), k, float(N), _p(cut), _p(eta), _p(sp))
    return Outcome(j == k, int(j), cut, eta, [float(v) for v in sp[:j]])


def extract_labels(outcome: Outcome) -> np.ndarray:
    labels = np.empty(outcome.cut.shape[0], np.int64)
    lib().oc_extract_labels(_p(outcome.cut), _p(outcome.eta), outcome.cut.shape[0], _p(labels))
    return labels


def subpartition_cost(labels, tree: Tree, omega, p) -> float:
    lab = np.ascontiguousarray(labels, dtype=np.int64)
    return lib().oc_subpartition_cost(_p(lab), lab.size, _p(tree.parent), _p(tree.parent_flow),
                                      _p(np.ascontiguousarray(omega)), _p(np.ascontiguousarray(p)))


def run_bisection(tree: Tree, omega, p, ext: Extrema, k: int, decide_fn=None) -> Result:
    """isoperim.py:222-308, same float expressions and fallbacks."""
    if decide_fn is None:
        decide_fn = lambda N: decide(tree, omega, p, k, N)  # noqa: E731
    alpha0 = (ext.phi_star_min + ext.p_star_min) / ext.omega_star_sum
    beta0 = (ext.phi_star_sum + ext.p_star_sum) / ext.omega_star_min
    if beta0 > alpha0:
        t_gap = math.ceil(math.log2(2.0 * ext.omega_star_sum**2 * (beta0 - alpha0))
                          - math.log2(ext.phi_star_min + ext.p_star_min))
        t_eps = math.ceil(math.log2((beta0 - alpha0) / (BRACKET_EPS * max(1.0, beta0))))
        t = max(t_gap, t_eps)
    else:
        t = 1
    t = min(MAX_ITERATIONS, max(1, t))
    alpha, beta = alpha0, beta0
    witness = None
    rounds = 0
    trace = []
    for _ in range(t):
        if beta - alpha <= BRACKET_EPS * max(1.0, beta):
            break
        mid = (alpha + beta) / 2.0
        out = decide_fn(mid)
        rounds += 1
        trace.append((mid, out.feasible))
        if out.feasible:
            beta = mid
            witness = out
        else:
            alpha = mid
    if witness is None:
        out = decide_fn(beta0)
        rounds += 1
        trace.append((beta0, out.feasible))
        if not out.feasible:
            bumped = beta0 * (1.0 + 1e-12)
            out = decide_fn(bumped)
            rounds += 1
            trace.append((bumped, out.feasible))
        if not out.feasible:
            raise InfeasibleSubpartitionError(f"no feasible {k}-subpartition found within bracket")
        witness = out
    labels = extract_labels(witness)
    miso = subpartition_cost(labels, tree, omega, p)
    return Result(miso, labels, witness, rounds, alpha, beta, trace)


@dataclass
class PipelineOut:
    result: Result
    tree: Tree
    omega: np.ndarray
    p: np.ndarray
    sigma: float
    extrema: Extrema


def run_pipeline(points, k: int, sigma="auto", alpha: float = 0.0, root: int = 0) -> PipelineOut:
    """pipeline.py:41-104 without the dense matrix (same arithmetic)."""
    X = np.ascontiguousarray(points, dtype=np.float64)
    sig = auto_sigma(X) if sigma == "auto" else float(sigma)
    tree = prim_mst(X, sig, root)
    omega, p = row_folds(X, sig, alpha)
    ext = extrema(tree, omega, p)
    res = run_bisection(tree, omega, p, ext, k)
    return PipelineOut(res, tree, omega, p, sig, ext)


def solve_tree(parent, flows, omega, p, k: int) -> tuple[Result, Tree, Extrema]:
    """C5 path: tree_from_parent_list + extrema + bisection."""
    tree = tree_from_parent_list(parent, flows)
    ext = extrema(tree, omega, p)
    return run_bisection(tree, omega, p, ext, k), tree, ext


# ------------------------------------------------ full-size oracle (C3/C4)
# isoc_fast.c kernels (same per-pair operation order, vectorised across
# pairs) + a certified Boruvka for Prim's edge set.  Used to produce the
# full-size parity fixtures (tools/oracle_full.py) and pinned against the
# reference at n = 16,000 / 32,000 / 46,340 (tests/test_oracle.py).

class TieError(RuntimeError):
    """A Boruvka component minimum was attained twice: the MST may not be
    unique, so the certified path cannot stand in for Prim (use prim_mst)."""


def flat_distance_sum_fast(X: np.ndarray) -> float:
    X = np.ascontiguousarray(X, dtype=np.float64)
    out = lib().ocf_flat_distance_sum(_p(X), X.shape[0], X.shape[1])
    if math.isnan(out):
        raise MemoryError("ocf_flat_distance_sum: allocation failed")
    return out


def auto_sigma_fast(X: np.ndarray) -> float:
    n = X.shape[0]
    mean = flat_distance_sum_fast(X) / (n * (n - 1))
    if not (mean > 0):
        raise ValueError("all points coincide; no usable distance scale")
    return mean


def omega_knn(X: np.ndarray, sigma: float, K: int = 32):
    """omega (vertex_weights, affinity.py:175-201; alpha = 0 so p = 0) and each
    row's K lexicographically smallest (d, j), j != i."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    omega = np.empty(n)
    kd = np.empty((n, K))
    kj = np.empty((n, K), np.int64)
    rc = lib().ocf_omega_knn(_p(X), n, d, float(sigma), 0, n, K, _p(omega), _p(kd), _p(kj))
    if rc:
        raise MemoryError("ocf_omega_knn: allocation failed")
    return omega, kd, kj


def mst_certified(X: np.ndarray, kd: np.ndarray, kj: np.ndarray, stats: Optional[dict] = None):
    """Prim's MST edge set (mst.py:128-181) via Boruvka with a uniqueness
    certificate: every round, every component's minimum outgoing edge is
    found exactly and must be the ONLY outgoing edge of that weight (else
    TieError).  A strictly lightest cut edge is in every MST, so the n-1
    certified edges are the unique MST = Prim's tree.  kd/kj (n x K, sorted
    by (d, j)) are refined in place by exact rescans of rows whose list
    cannot decide their component's minimum.  Returns (u, v, w) arrays."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    K = kd.shape[1]
    rows = np.arange(n)
    comp = np.arange(n, dtype=np.int32)
    eu = np.empty(0, np.int64)
    ev = np.empty(0, np.int64)
    ew = np.empty(0, np.float64)
    st = stats if stats is not None else {}
    st.update(rounds=0, rescans=0, rescans_per_round=[], components_per_round=[])
    ncomp = n
    while ncomp > 1:
        st["rounds"] += 1
        st["components_per_round"].append(int(ncomp))
        rescanned_this_round = 0
        for attempt in range(2):
            valid = kj >= 0
            ext = valid & (comp[np.where(valid, kj, 0)] != comp[:, None])
            has = ext.any(1)
            first = np.argmax(ext, 1)
            cand_d = np.where(has, kd[rows, first], np.inf)
            cand_j = np.where(has, kj[rows, first], -1)
            full = valid[:, K - 1]
            lb = np.where(full, kd[:, K - 1], np.inf)  # every unlisted j has d >= lb
            mult = (ext & (kd == cand_d[:, None])).sum(1)
            unsure = has & full & (kd[:, K - 1] == cand_d)  # unlisted j may tie the row min
            m = np.full(n, np.inf)
            np.minimum.at(m, comp, cand_d)
            mc = m[comp]
            need = (~has & (lb <= mc)) | (unsure & (cand_d <= mc))
            if not need.any():
                break
            if attempt == 1:
                raise TieError("more than K exact ties at a row minimum")
            idx = np.flatnonzero(need).astype(np.int64)
            nd = np.empty((idx.size, K))
            nj = np.empty((idx.size, K), np.int64)
            rc = lib().ocf_rescan_rows(_p(X), n, d, _p(idx), idx.size, _p(comp), K, _p(nd), _p(nj))
            if rc:
                raise MemoryError("ocf_rescan_rows: allocation failed")
            kd[idx] = nd
            kj[idx] = nj
            rescanned_this_round += idx.size
        st["rescans"] += rescanned_this_round
        st["rescans_per_round"].append(int(rescanned_this_round))
        # component minima: the attaining rows and their multiplicity
        at_min = has & (cand_d == mc)
        cnt = np.bincount(comp[at_min], weights=mult[at_min], minlength=n)
        if (cnt[comp[at_min]] > 1).any():
            raise TieError(f"exact tie at a component minimum in Boruvka round {st['rounds']}")
        a = rows[at_min]
        b = cand_j[at_min]
        w = cand_d[at_min]
        key = np.minimum(a, b) * n + np.maximum(a, b)
        key, first_idx = np.unique(key, return_index=True)
        eu = np.concatenate([eu, a[first_idx]])
        ev = np.concatenate([ev, b[first_idx]])
        ew = np.concatenate([ew, w[first_idx]])
        g = coo_matrix((np.ones(eu.size), (eu, ev)), shape=(n, n))
        ncomp, lab = connected_components(g, directed=False)
        comp = lab.astype(np.int32)
    if eu.size != n - 1:
        raise RuntimeError(f"certified Boruvka produced {eu.size} edges for n={n}")
    return eu, ev, ew


def root_tree(n: int, eu, ev, ew, root: int, sigma: float) -> Tree:
    """Root the MST edge set like prim_mst does (mst.py:128-181, 46-65):
    parent by BFS from root; child_id = rank of (d(p,u), u) among p's
    children (Prim's insertion order); bfs_order reversed."""
    a = np.concatenate([eu, ev]).astype(np.int64)
    b = np.concatenate([ev, eu]).astype(np.int64)
    w = np.concatenate([ew, ew])
    order = np.lexsort((b, w, a))
    a, b, w = a[order], b[order], w[order]
    start = np.searchsorted(a, np.arange(n + 1))
    parent = np.full(n, NO_VERTEX, np.int64)
    pdist = np.zeros(n)
    depth = np.zeros(n, np.int64)
    child_id = np.zeros(n, np.int64)
    seen = np.zeros(n, bool)
    seen[root] = True
    level = np.array([root], np.int64)
    out = [level]
    dep = 0
    while level.size:
        s, c = start[level], start[level + 1] - start[level]
        tot = int(c.sum())
        if tot == 0:
            break
        idx = np.arange(tot) - np.repeat(np.cumsum(c) - c, c) + np.repeat(s, c)
        src = np.repeat(level, c)
        dst = b[idx]
        keep = ~seen[dst]
        src, dst, wd = src[keep], dst[keep], w[idx][keep]
        dep += 1
        seen[dst] = True
        parent[dst] = src
        pdist[dst] = wd
        depth[dst] = dep
        # rank among siblings: dst is grouped by src (level order) and sorted by (w, b)
        grp_start = np.r_[0, np.flatnonzero(src[1:] != src[:-1]) + 1]
        pos = np.arange(dst.size)
        child_id[dst] = pos - np.repeat(grp_start, np.diff(np.r_[grp_start, dst.size]))
        level = dst
        out.append(level)
    root_first = np.concatenate(out)
    if root_first.size != n:
        raise ValueError("edge set does not span the points")
    flow = np.zeros(n)
    nonroot = parent != NO_VERTEX
    flow[nonroot] = exp((-pdist[nonroot]) / sigma)
    return Tree(parent, flow, depth, child_id, root_first[::-1].copy(), root, int(depth.max()), pdist)


@dataclass
class FullRun:
    out: PipelineOut
    total_distance: float
    mst_stats: dict
    seconds: dict


def run_pipeline_full(points, k: int, sigma="auto", root: int = 0, K: int = 32) -> FullRun:
    """run_pipeline (pipeline.py:41-104, alpha = 0) at full size: the same
    numbers as run_pipeline() above, with the n^2 passes vectorised and the
    MST edge set from the certified Boruvka (raises TieError when the MST
    is not provably unique)."""
    import time

    X = np.ascontiguousarray(points, dtype=np.float64)
    n = X.shape[0]
    sec = {}
    t0 = time.perf_counter()
    sig = auto_sigma_fast(X) if sigma == "auto" else float(sigma)
    sec["sigma"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    omega, kd, kj = omega_knn(X, sig, K)
    sec["omega_knn"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    st = {}
    eu, ev, ew = mst_certified(X, kd, kj, st)
    tree = root_tree(n, eu, ev, ew, root, sig)
    sec["mst"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    p = np.zeros(n)
    ext = extrema(tree, omega, p)
    res = run_bisection(tree, omega, p, ext, k)
    sec["partition"] = time.perf_counter() - t0
    return FullRun(PipelineOut(res, tree, omega, p, sig, ext), math.fsum(ew), st, sec)
