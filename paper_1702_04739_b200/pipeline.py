"""Drop-in clustering entry point and stage API on the B200 path.

`run_pipeline` keeps the reference signature and result type
(/root/reference/pkg/src/isoclust/pipeline.py:41-104): points and k in;
cluster labels (1..k), the residual mask (labels == 0) and the k-th
isoperimetric value (result.miso) out, plus the same four timing buckets.
Stages:
  affinity   K1 exact sigma pass (+ exact nearest neighbours = Boruvka
             round 1) and K2 exact omega pass       affinity.py:124-279
  mst        Boruvka rounds (FP32 filter + exact re-rank), rooting,
             parent flows                            mst.py:128-181
  partition  bisection over device decision sweeps   isoperim.py:222-308
Under torch.distributed (one process per GPU) rows are sharded for the
dense stages; the per-round Boruvka keys are MIN-all-reduced and the tree
phase runs replicated on every rank.  Results do not depend on the number of
GPUs.

The dense distance matrix of the reference is never formed, so the
reference's n <= 46,340 cap (affinity.py:23-24) does not apply.
"""
from __future__ import annotations

import math
import os
import time
import warnings
from typing import Callable, Optional, Union

import numpy as np

from ._lib import InfeasibleSubpartitionError
from .engine import Comm, CudaBackend, DeviceTree
from .types import (
    LazyRootedTree,
    BRACKET_EPS,
    MAX_ITERATIONS,
    NO_VERTEX,
    DecisionOutcome,
    Extrema,
    MisoResult,
    NodeWeights,
    PipelineRun,
    RootedTree,
)

ENGINES = ("seq", "par")
WORKERS_ENV_VAR = "ISOCLUST_WORKERS"

_BACKEND: Optional[CudaBackend] = None


def backend() -> CudaBackend:
    global _BACKEND
    if _BACKEND is None:
        _BACKEND = CudaBackend()
    return _BACKEND


def resolve_workers(workers: Optional[int] = None) -> int:
    """_primitives.py:25-41 (the count is recorded; it never changes results)."""
    if workers is None:
        env = os.environ.get(WORKERS_ENV_VAR, "").strip()
        if env:
            try:
                workers = int(env)
            except ValueError:
                raise ValueError(f"{WORKERS_ENV_VAR} must be an integer, got {env!r}") from None
        else:
            workers = os.cpu_count() or 1
    workers = int(workers)
    if workers < 1:
        raise ValueError(f"worker count must be >= 1, got {workers}")
    return workers


def _validate_points(points) -> np.ndarray:
    """affinity.py:70-81."""
    x = np.ascontiguousarray(points, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError(f"points must be a 2-d array, got shape {x.shape}")
    n, d = x.shape
    if n < 2:
        raise ValueError(f"need at least 2 points, got {n}")
    if d < 1:
        raise ValueError("points must have at least one coordinate")
    if not np.isfinite(x).all():
        raise ValueError("points must be finite")
    return x


def _validate_k(k) -> None:
    """isoperim.py:71-79."""
    if not isinstance(k, (int, np.integer)) or isinstance(k, bool):
        raise TypeError(f"k must be an integer, got {k!r}")
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")


# --------------------------------------------------------------- stages
def _is_device_tensor(points) -> bool:
    mod = type(points).__module__
    return mod.startswith("torch") and getattr(points, "is_cuda", False)


class _Points:
    """Points resident on the device plus this rank's row shard.

    Accepts host arrays (validated as affinity.py:70-81, then copied to HBM)
    or a CUDA torch tensor already resident in HBM (same validation on the
    device, no copy).
    """

    def __init__(self, points, comm: Optional[Comm] = None, b: Optional[CudaBackend] = None):
        self.b = b or backend()
        self.comm = comm or Comm()
        if _is_device_tensor(points):
            torch = self.b.torch
            X = points.to(torch.float64).contiguous()
            if X.dim() != 2:
                raise ValueError(f"points must be a 2-d array, got shape {tuple(X.shape)}")
            n, d = X.shape
            if n < 2:
                raise ValueError(f"need at least 2 points, got {n}")
            if d < 1:
                raise ValueError("points must have at least one coordinate")
            if not bool(torch.isfinite(X).all()):
                raise ValueError("points must be finite")
            self.host = None
            self.X = X
        else:
            self.host = _validate_points(points)
            self.X = self.b.to_device(self.host)
        self.n, self.d = (int(v) for v in self.X.shape)
        self.lo, self.hi = self.comm.rows(self.n)


def _sharded_symmetric(P: _Points, alpha: float = 0.0) -> bool:
    """Multi-GPU: the symmetric passes sharded by column-super-block ranges
    (each unordered pair once across the job) instead of row shards of the
    one-sided passes.  ISOC_SHARDED_SYM=0 selects the row shards."""
    return (P.comm.world > 1 and alpha == 0.0 and P.n >= 2048 and hasattr(P.b, "sigma_sym_range")
            and os.environ.get("ISOC_SHARDED_SYM", "1") != "0")


def _sigma_pass(P: _Points, alpha: float, want_nn: bool = True):
    if _sharded_symmetric(P, alpha):
        jlo, jhi = P.b.sym_block_range(P.n, P.comm.rank, P.comm.world)
        part = P.b.sigma_sym_range(P.X, P.n, P.d, jlo, jhi, want_nn)
        recv = tuple(None if t is None else P.comm.alltoall_rows(t, P.n) for t in part)
        stack, nn = P.b.sigma_rank_merge(P.X, P.n, P.d, P.lo, P.hi, recv, want_nn)
        p_loc = P.b.empty((P.hi - P.lo,), P.b.torch.float64).zero_()
        return stack, nn, p_loc
    if want_nn:
        return P.b.sigma_partial(P.X, P.n, P.d, P.lo, P.hi, alpha)
    return P.b.sigma_partial(P.X, P.n, P.d, P.lo, P.hi, alpha, want_nn=False)


def _omega_pass(P: _Points, sigma: float, h=None):
    """This rank's omega rows (and, with the MST handle h, the exact round-2
    minima).  Multi-GPU with the symmetric split: every rank evaluates its
    super-tile range once and sends each owner exactly the (row,
    super-block) subtrees it produced for that owner's rows (one all-to-all
    with per-peer split sizes per slot buffer); the owner folds them --
    bitwise the single-GPU result (each slot has one producer)."""
    if _sharded_symmetric(P):
        G, r = P.comm.world, P.comm.rank
        send, recv_counts = P.b.omega_shard_counts(P.n, G, r)
        ps, psm, psj = P.b.omega_sym_range(P.X, P.n, P.d, r, G, sigma, h)
        recv = [None if t is None else P.comm.alltoall_var(t, send, recv_counts) for t in (ps, psm, psj)]
        del ps, psm, psj
        return P.b.omega_rank_merge(P.n, r, G, *recv)
    if h is None:
        return P.b.omega(P.X, P.n, P.d, P.lo, P.hi, sigma), None
    return P.b.omega_mst(P.X, P.n, P.d, P.lo, P.hi, sigma, h)


def _round1_from_sigma(P: _Points) -> bool:
    """Borůvka round 1 from the sigma pass's exact nearest neighbours (default)
    or from the tensor-core filter (ISOC_ROUND1=filter: the symmetric sigma
    pass then skips the neighbour bookkeeping, ~6% of it, but singletons
    leave many uncertified rows to rescan -- a wash at n = 400k)."""
    return os.environ.get("ISOC_ROUND1", "nn") != "filter"


def _sigma_from_stack(P: _Points, stack) -> float:
    total = P.b.sigma_finish(P.comm.allgather_stack(stack))
    n = P.n
    mean = total / (n * (n - 1))
    if not (mean > 0):
        raise ValueError("all points coincide; no usable distance scale")
    return mean


def _boruvka(P: _Points, nn=None, sigma: Optional[float] = None) -> tuple:
    """MST edges on the device; returns (u, v, w, omega_local, stats).

    Round 1 uses the exact nearest neighbours of the sigma pass (when given);
    when `sigma` is given the exact omega pass runs right after round 1 and
    also yields round 2 (each row's exact minimum over other components);
    the remaining rounds use the FP32 filter + exact re-rank.  Per round each
    rank reduces its row shard to per-component 64-bit keys; two MIN
    all-reduces (weight bits, then packed endpoints of the rows that attain
    the minimum) make the lexicographic (d, min, max) winner global, after
    which hooking/contraction is replicated identically on every rank.
    """
    b, comm, n = P.b, P.comm, P.n
    h = b.mst_create(P.X, n, P.d, P.lo, P.hi)
    stats = {"boruvka_rounds": 0, "exact_ties": 0, "exact_rescans": 0, "omega_ms": 0.0}
    omega_loc = None

    def one_round(cand):
        cmin = b.mst_round_local(h, n, cand)
        comm.allreduce_min_(cmin)
        cedge = b.mst_round_edges(h, cmin)
        comm.allreduce_min_(cedge)
        c, t, r = b.mst_round_finish(h, cmin, cedge)
        stats["boruvka_rounds"] += 1
        stats["exact_ties"] += t
        stats["exact_rescans"] += r
        return c

    try:
        comps = n
        if nn is not None:
            comps = _progress(one_round(nn), comps, stats)
        if sigma is not None:
            t0 = time.perf_counter()
            omega_loc, nn2 = _omega_pass(P, sigma, h)
            if hasattr(b.torch, "cuda") and b.torch.cuda.is_available():
                b.torch.cuda.synchronize()
            stats["omega_ms"] = (time.perf_counter() - t0) * 1e3
            if comps > 1:
                comps = _progress(one_round(nn2), comps, stats)
        while comps > 1:
            comps = _progress(one_round(None), comps, stats)
        u, v, w = b.mst_edges(h, n)
        fs = getattr(b, "mst_filter_stats", lambda _h: None)(h)
        if fs is not None:
            stats["filter_blocks_run"], stats["filter_blocks_total"], stats["filter_rows_refreshed"] = fs
    finally:
        b.mst_destroy(h)
    if comm.world > 1:
        import torch

        tt = torch.tensor([stats["exact_ties"], stats["exact_rescans"]], dtype=torch.int64,
                          device=getattr(b, "device", "cpu"))
        comm.allreduce_sum_(tt)
        stats["exact_ties"], stats["exact_rescans"] = (int(x) for x in tt.tolist())
    return u, v, w, omega_loc, stats


def _tie_rule(P: _Points, u, v, w, stats: dict, root: int):
    """prim_mst's tie rule (mst.py:144-166, _primitives.py:69-92).

    The lexicographic Boruvka MST is the reference's Prim tree whenever every
    component minimum is unique.  When a round saw an
    exact distance tie (the count is global after the all-reduce, so every
    rank decides alike), Prim is replayed exactly on the device from `root`
    (isoc_prim_edges; X is replicated on every rank).  ISOC_MST=prim forces it.
    """
    stats["prim_replay"] = 0
    if stats["exact_ties"] or os.environ.get("ISOC_MST", "") == "prim":
        stats["prim_replay"] = 1
        return P.b.prim_edges(P.X, P.n, P.d, root)
    return u, v, w


def _progress(c: int, comps: int, stats: dict) -> int:
    if c >= comps:
        raise RuntimeError(f"Boruvka round {stats['boruvka_rounds']} made no progress ({c} components)")
    return c


def _rooted_tree_view(dt: DeviceTree, root: int) -> RootedTree:
    return LazyRootedTree(dt, root)


def auto_sigma_points(points) -> float:
    """auto_sigma (affinity.py:233-241) from points, matrix-free, bitwise:
    the mean off-diagonal distance with numpy's pairwise d.sum() order.
    (stages.auto_sigma takes a distance matrix, as the reference does.)"""
    P = _Points(points)
    stack, _, _ = _sigma_pass(P, 0.0)
    return _sigma_from_stack(P, stack)


def node_weights_points(points, sigma: float, alpha: float = 0.0) -> NodeWeights:
    """node_weights (vertex_weights + potentials, affinity.py:175-257) from
    points, matrix-free.  (stages.node_weights takes a distance matrix.)"""
    if not (sigma > 0):
        raise ValueError(f"sigma must be > 0, got {sigma}")
    if alpha < 0:
        raise ValueError(f"alpha must be >= 0, got {alpha}")
    P = _Points(points)
    om = P.comm.allgather_rows(_omega_pass(P, sigma)[0], P.n)
    if alpha > 0:
        _, _, p_loc = _sigma_pass(P, alpha)
        p = P.comm.allgather_rows(p_loc, P.n).cpu().numpy()
    else:
        p = np.zeros(P.n)
    return NodeWeights(omega=om.cpu().numpy(), p=p, sigma=float(sigma), alpha=float(alpha))


def minimum_spanning_tree(points, sigma: float, root: int = 0) -> RootedTree:
    """prim_mst (mst.py:128-181) from points: Boruvka on the device, rooted."""
    if not (sigma > 0):
        raise ValueError(f"sigma must be > 0, got {sigma}")
    P = _Points(points)
    if not (0 <= root < P.n):
        raise ValueError(f"root must be in [0, {P.n}), got {root}")
    u, v, w, _, stats = _boruvka(P)
    u, v, w = _tie_rule(P, u, v, w, stats, root)
    dt = P.b.tree_from_edges(u, v, w, P.n, root, sigma)
    return _rooted_tree_view(dt, root)


def tree_from_parent_list(parent, parent_flow, root: Optional[int] = None) -> RootedTree:
    """mst.py:78-125 on the device (sibling ranks by ascending vertex index).

    The sentinel count, a given root and the index range are validated on the
    device (isoc_tree_from_parent), raising ValueError like the reference."""
    # inputs are read, never mutated (the device keeps its own copies)
    par = np.ascontiguousarray(parent, dtype=np.int64)
    flows = np.ascontiguousarray(parent_flow, dtype=np.float64)
    n = par.shape[0]
    if par.ndim != 1 or flows.shape != par.shape:
        raise ValueError("parent and parent_flow must be 1-d arrays of equal length")
    if n == 0:
        raise ValueError("expected exactly one root sentinel, found 0")
    if root is not None and not (0 <= int(root) < n):
        raise ValueError("root does not match the parent array's sentinel")
    dt = backend().tree_from_parent(par, flows, root)
    return _rooted_tree_view(dt, dt.root)


def _device_tree(tree: RootedTree) -> DeviceTree:
    if tree._device is None:
        tree._device = backend().tree_from_parent(tree.parent, tree.parent_flow, tree.root,
                                                  child_id=tree.child_id)
    return tree._device


def extrema(tree: RootedTree, weights: NodeWeights) -> Extrema:
    """affinity.py:260-279 on the device (pow2 folds, bitwise)."""
    if tree.n != weights.n:
        raise ValueError(f"tree has {tree.n} vertices but weights have {weights.n}")
    dt = _device_tree(tree)
    b = dt.b
    return dt.set_weights(b.to_device(weights.omega), b.to_device(weights.p))


def _attach(tree: RootedTree, weights: NodeWeights) -> DeviceTree:
    dt = _device_tree(tree)
    if getattr(dt, "_weights_id", None) is not weights:
        b = dt.b
        dt.set_weights(b.to_device(weights.omega), b.to_device(weights.p))
        dt._weights_id = weights
    return dt


def _outcome(dt: DeviceTree, slot: int, k: int, j: int) -> tuple[DecisionOutcome, np.ndarray, float]:
    w = dt.witness(slot, k)
    out = DecisionOutcome(feasible=(j == k), clusters_found=j, cut=w.cut, eta=w.eta,
                          cluster_sparsities=w.sparsities[:j])
    return out, w.labels, w.miso


def decide(tree: RootedTree, weights: NodeWeights, k: int, N: float) -> DecisionOutcome:
    """One decision sweep (isoperim.py:82-144) on the device."""
    _validate_k(k)
    if tree.n != weights.n:
        raise ValueError(f"tree has {tree.n} vertices but weights have {weights.n}")
    if not math.isfinite(N):
        raise ValueError(f"threshold must be finite, got {N}")
    dt = _attach(tree, weights)
    j = dt.decide(N, k, 0)
    return _outcome(dt, 0, k, j)[0]


par_decide = decide


def _speculation_depth(dt: DeviceTree) -> int:
    """Bisection steps per batched sweep: 6 (63 thresholds, one warp each)
    on trees that fit one CTA's shared memory (C1), 4 (15 thresholds, one
    CTA group each) on latency-bound trees whose levels are narrow (MST trees of
    C1-C4), 1 (plain sequential sweeps, which stop at their own k-th cut) on
    wide trees (C5): there a 3-threshold sweep -- split CTAs or shared
    (decide_multi_kernel) -- costs 2.3x a single one.  ISOC_SPEC_M
    overrides."""
    cap = dt.batch_capacity() if hasattr(dt, "batch_capacity") else 16
    mmax = 6 if cap >= 63 else 4
    env = os.environ.get("ISOC_SPEC_M")
    if env is not None:
        return max(1, min(mmax, int(env)))
    if not hasattr(dt, "shape"):
        return 1
    if cap >= 63:
        return 6   # small tree: one warp per threshold, 63 thresholds cost one sweep
    levels, width = dt.shape()
    return 4 if dt.n <= 64 * 1024 * max(1, levels) and width <= 262144 else 1


_HEAP_KIDS: dict = {}


def _heap_kids(depth: int) -> list:
    """kids of the complete depth-`depth` tree in heap order (read-only, cached)."""
    kids = _HEAP_KIDS.get(depth)
    if kids is None:
        m = (1 << depth) - 1
        kids = [[2 * i + 1, 2 * i + 2] if 2 * i + 1 < m else [-1, -1] for i in range(m)]
        _HEAP_KIDS[depth] = kids
    return kids


def _threshold_tree(a0: float, b0: float, depth: int):
    """The midpoints the next `depth` bisection steps can visit from the
    bracket (a0, b0): node = (a + b) / 2 of its interval, children the
    halves (a, mid) and (mid, b); a node whose interval already passes the
    reference's stop test b - a <= 1e-15 * max(1, b) (isoperim.py:263-266)
    does not exist, nor do its descendants.  Built in level order.  Returns
    (thresholds, kids[node] = [left, right] or -1, root or -1)."""
    if depth >= 1 and (b0 - a0) / float(1 << (depth - 1)) > 4.0 * BRACKET_EPS * max(1.0, b0):
        # no interval of the tree can pass the stop test (each is at least
        # (b0 - a0) / 2^(depth-1) wide up to rounding, and b <= b0): the
        # complete tree in heap order, which is the level order below
        m = (1 << depth) - 1
        lo = [0.0] * m
        hi = [0.0] * m
        thr = [0.0] * m
        lo[0], hi[0] = a0, b0
        half = m >> 1
        for i in range(m):
            a, b = lo[i], hi[i]
            mid = (a + b) / 2.0
            thr[i] = mid
            if i < half:
                c = 2 * i + 1
                lo[c], hi[c], lo[c + 1], hi[c + 1] = a, mid, mid, b
        return thr, _heap_kids(depth), 0
    thr: list = []
    kids: list = []
    root = -1
    cur = [(a0, b0, -1, 0)]
    for _ in range(depth):
        nxt = []
        for a, b, par, side in cur:
            if b - a <= BRACKET_EPS * max(1.0, b):
                continue
            mid = (a + b) / 2.0
            idx = len(thr)
            thr.append(mid)
            kids.append([-1, -1])
            if par < 0:
                root = idx
            else:
                kids[par][side] = idx
            nxt.append((a, mid, idx, 0))
            nxt.append((mid, b, idx, 1))
        if not nxt:
            break
        cur = nxt
    return thr, kids, root


def run_bisection(dt: DeviceTree, ext: Extrema, k: int, n: int) -> MisoResult:
    """isoperim.py:222-308 with device decision sweeps.

    Same closed-form bracket, round budget, stop test, midpoint expression,
    witness rule and infeasible fallbacks as the reference; the witness's
    labels and exact cost are computed on the device once at the end.
    """
    _validate_k(k)
    alpha0 = (ext.phi_star_min + ext.p_star_min) / ext.omega_star_sum
    beta0 = (ext.phi_star_sum + ext.p_star_sum) / ext.omega_star_min
    if beta0 > alpha0:
        t_gap = math.ceil(
            math.log2(2.0 * ext.omega_star_sum**2 * (beta0 - alpha0))
            - math.log2(ext.phi_star_min + ext.p_star_min)
        )
        t_eps = math.ceil(math.log2((beta0 - alpha0) / (BRACKET_EPS * max(1.0, beta0))))
        t = max(t_gap, t_eps)
    else:
        t = 1
    t = min(MAX_ITERATIONS, max(1, t))

    alpha, beta = alpha0, beta0
    wslot: Optional[int] = None
    wj = 0
    rounds = 0
    trace: list = []

    def sweep(N: float) -> tuple[bool, int, int]:
        slot = 0 if wslot is None else 1 - wslot
        j = dt.decide(N, k, slot)
        return j == k, j, slot

    m = _speculation_depth(dt)
    if m <= 1:
        for _ in range(t):
            if beta - alpha <= BRACKET_EPS * max(1.0, beta):
                break
            mid = (alpha + beta) / 2.0
            ok, j, slot = sweep(mid)
            rounds += 1
            trace.append((mid, ok))
            if ok:
                beta = mid
                wslot, wj = slot, j
            else:
                alpha = mid
    else:
        # Speculative bisection: the thresholds the next m steps
        # can visit, built with the reference's own float recursion and stop
        # test, are swept in one batched pass; the walk then replays the
        # sequential loop on their outcomes.  The witness is re-derived at the
        # last feasible midpoint by one ordinary sweep.
        wthr = None
        stop = False
        while not stop and rounds < t:
            thr, kids, root = _threshold_tree(alpha, beta, min(m, t - rounds))
            if root < 0:
                break
            js = dt.decide_batch(thr, k)
            node = root
            while node >= 0:
                if beta - alpha <= BRACKET_EPS * max(1.0, beta):
                    stop = True
                    break
                mid = thr[node]
                j = js[node]
                ok = j == k
                rounds += 1
                trace.append((mid, ok))
                if ok:
                    beta = mid
                    wthr, wj = mid, j
                    node = kids[node][0]
                else:
                    alpha = mid
                    node = kids[node][1]
                if rounds >= t:
                    break
        if wthr is not None:
            j = dt.decide(wthr, k, 0)
            if j != wj:
                raise RuntimeError(f"speculative sweep disagrees with the witness sweep ({j} != {wj})")
            wslot = 0

    if wslot is None:
        ok, j, slot = sweep(beta0)
        rounds += 1
        trace.append((beta0, ok))
        if not ok:
            bumped = beta0 * (1.0 + 1e-12)
            ok, j, slot = sweep(bumped)
            rounds += 1
            trace.append((bumped, ok))
        if not ok:
            raise InfeasibleSubpartitionError(
                f"no feasible {k}-subpartition found within bracket (n={n}, k={k})"
            )
        wslot, wj = slot, j

    outcome, labels, miso = _outcome(dt, wslot, k, wj)
    return MisoResult(miso=miso, labels=labels, outcome=outcome, iterations=rounds,
                      alpha_final=alpha, beta_final=beta, trace=trace)


def solve_miso(tree: RootedTree, weights: NodeWeights, ext: Extrema, k: int) -> MisoResult:
    """Exact k-th isoperimetric number of the tree (isoperim.py:311-321)."""
    _validate_k(k)
    if tree.n != weights.n:
        raise ValueError(f"tree has {tree.n} vertices but weights have {weights.n}")
    dt = _attach(tree, weights)
    return run_bisection(dt, ext, k, tree.n)


def par_solve_miso(tree: RootedTree, weights: NodeWeights, ext: Extrema, k: int, *,
                   workers: Optional[int] = None) -> MisoResult:
    """parengine.py:212-232: same device engine (workers never change results)."""
    return solve_miso(tree, weights, ext, k)


# -------------------------------------------------------------- pipeline
def run_pipeline(
    points: np.ndarray,
    k: int,
    sigma: Union[str, float] = "auto",
    alpha: float = 0.0,
    root: int = 0,
    engine: str = "seq",
    workers: Optional[int] = None,
) -> PipelineRun:
    """Cluster a point set into k groups; returns the result with timings.

    Same contract as the reference (pipeline.py:41-104).  `engine` accepts
    "seq" and "par" (both run the device engine and return identical
    results); `workers` is recorded but, as in the reference, never changes
    results.  Under torch.distributed, every rank returns the same run.
    """
    if engine not in ENGINES:
        raise ValueError(f"engine must be one of {ENGINES}, got {engine!r}")
    x = points if _is_device_tensor(points) else np.asarray(points, dtype=np.float64)
    nworkers = resolve_workers(workers) if engine == "par" else 1
    b = backend()
    torch = b.torch

    t_start = time.perf_counter()
    t0 = time.perf_counter()
    P = _Points(x, b=b)
    n, d = P.n, P.d
    need_pass = sigma == "auto" or alpha > 0
    nn = None
    p_loc = None
    if need_pass:
        stack, nn, p_loc = _sigma_pass(P, float(alpha) if alpha > 0 else 0.0, _round1_from_sigma(P))
        sigma_val = _sigma_from_stack(P, stack) if sigma == "auto" else float(sigma)
    else:
        sigma_val = float(sigma)
    if not (sigma_val > 0):
        raise ValueError(f"sigma must be > 0, got {sigma_val}")
    affinity_ms = (time.perf_counter() - t0) * 1e3

    t0 = time.perf_counter()
    if not (0 <= root < n):
        raise ValueError(f"root must be in [0, {n}), got {root}")
    # the exact omega pass runs inside the MST loop (it also yields Boruvka
    # round 2); its time is booked under "affinity" like the reference's
    # node_weights
    u, v, w, om_loc, stats = _boruvka(P, nn, sigma=sigma_val)
    u, v, w = _tie_rule(P, u, v, w, stats, root)
    dt = b.tree_from_edges(u, v, w, n, root, sigma_val)
    torch.cuda.synchronize()
    mst_ms = (time.perf_counter() - t0) * 1e3 - stats["omega_ms"]
    affinity_ms += stats["omega_ms"]

    t0 = time.perf_counter()
    if alpha < 0:
        raise ValueError(f"alpha must be >= 0, got {alpha}")
    om = P.comm.allgather_rows(om_loc, n)
    if alpha > 0:
        p = P.comm.allgather_rows(p_loc, n)
    else:
        p = torch.zeros(n, dtype=torch.float64, device=b.device)
    ext = dt.set_weights(om, p)
    affinity_ms += (time.perf_counter() - t0) * 1e3

    t0 = time.perf_counter()
    result = run_bisection(dt, ext, k, n)
    partition_ms = (time.perf_counter() - t0) * 1e3
    total_ms = (time.perf_counter() - t_start) * 1e3

    return PipelineRun(
        result=result, n=n, d=d, k=k, sigma=sigma_val, alpha=float(alpha), root=root,
        engine=engine, workers=nworkers,
        timings_ms={"affinity": affinity_ms, "mst": mst_ms, "partition": partition_ms,
                    "total": total_ms},
        gpus=P.comm.world, mst_stats=stats,
        tree=LazyRootedTree(dt, root), extrema=ext, omega_device=om, p_device=p,
    )


def summarize(run: PipelineRun) -> dict:
    """JSON-ready summary (schema version 1, pipeline.py:107-128)."""
    labels = run.result.labels
    cluster_sizes = [int(np.sum(labels == c)) for c in range(1, run.k + 1)]
    return {
        "schema": 1,
        "n": run.n,
        "d": run.d,
        "k": run.k,
        "miso": run.result.miso,
        "iterations": run.result.iterations,
        "alpha_final": run.result.alpha_final,
        "beta_final": run.result.beta_final,
        "cluster_sizes": cluster_sizes,
        "residual_count": int(np.sum(labels == 0)),
        "sigma": run.sigma,
        "alpha": run.alpha,
        "root": run.root,
        "engine": run.engine,
        "workers": run.workers,
        "timings_ms": {k: round(v, 3) for k, v in run.timings_ms.items()},
    }
