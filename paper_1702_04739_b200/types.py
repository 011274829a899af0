"""Result and input containers with the reference's names and fields.

Mirrors /root/reference/pkg/src/isoclust: NodeWeights / Extrema
(affinity.py:31-67), RootedTree (mst.py:23-43), DecisionOutcome / MisoResult
(isoperim.py:37-68), PipelineRun (pipeline.py:25-38).  Host-side numpy
arrays, so results drop into code written against the reference.  A
RootedTree produced on the GPU also carries its device-resident layout
(`_device`) so the solver never re-uploads it.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Optional

import numpy as np

NO_VERTEX = -1

# isoperim.py:24, :27
BRACKET_EPS = 1e-15
MAX_ITERATIONS = 128


@dataclass
class NodeWeights:
    """Per-vertex similarity mass and isolation potential (affinity.py:31-55)."""

    omega: np.ndarray
    p: np.ndarray
    sigma: float
    alpha: float

    def __post_init__(self):
        self.omega = np.ascontiguousarray(self.omega, dtype=np.float64)
        self.p = np.ascontiguousarray(self.p, dtype=np.float64)
        if self.omega.shape != self.p.shape or self.omega.ndim != 1:
            raise ValueError(
                f"omega and p must be 1-d arrays of equal length, got "
                f"{self.omega.shape} and {self.p.shape}"
            )
        if not (self.sigma > 0):
            raise ValueError(f"sigma must be > 0, got {self.sigma}")
        if self.alpha < 0:
            raise ValueError(f"alpha must be >= 0, got {self.alpha}")

    @property
    def n(self) -> int:
        return self.omega.shape[0]


@dataclass
class Extrema:
    """Sums and minima of tree-edge flows, vertex masses and potentials."""

    phi_star_sum: float
    phi_star_min: float
    omega_star_sum: float
    omega_star_min: float
    p_star_sum: float
    p_star_min: float


@dataclass
class RootedTree:
    """Rooted spanning tree as parallel arrays (mst.py:23-43)."""

    parent: np.ndarray
    parent_flow: np.ndarray
    depth: np.ndarray
    child_id: np.ndarray
    bfs_order: np.ndarray
    root: int
    max_depth: int
    _device: Any = field(default=None, repr=False, compare=False)

    @property
    def n(self) -> int:
        return self.parent.shape[0]


class LazyRootedTree(RootedTree):
    """RootedTree whose arrays stay on the device until first read (one
    export of all five arrays); solve_miso / extrema use the device tree
    directly, so a caller that only wants the partition never pays the
    device-to-host copy of the tree."""

    _LAZY = ("parent", "parent_flow", "depth", "child_id", "bfs_order", "max_depth")

    def __init__(self, device_tree, root: int):
        object.__setattr__(self, "_device", device_tree)
        object.__setattr__(self, "root", int(root))

    def __getattr__(self, name):
        if name in LazyRootedTree._LAZY:
            parent, flow, depth, cid, order, max_depth, _ = self._device.export()
            for k, v in zip(LazyRootedTree._LAZY, (parent, flow, depth, cid, order, max_depth)):
                object.__setattr__(self, k, v)
            return object.__getattribute__(self, name)
        raise AttributeError(name)

    @property
    def n(self) -> int:
        return self._device.n


@dataclass(eq=False)
class DecisionOutcome:
    """Result of one threshold decision sweep (isoperim.py:37-50)."""

    feasible: bool
    clusters_found: int
    cut: np.ndarray
    eta: np.ndarray
    cluster_sparsities: list


@dataclass(eq=False)
class MisoResult:
    """Optimum value, witness labels and the bisection bracket (isoperim.py:53-68)."""

    miso: float
    labels: np.ndarray
    outcome: Optional[DecisionOutcome]
    iterations: int
    alpha_final: float
    beta_final: float
    trace: list = field(default_factory=list)


@dataclass
class PipelineRun:
    """One solved instance plus configuration and timings (pipeline.py:25-38)."""

    result: MisoResult
    n: int
    d: int
    k: int
    sigma: float
    alpha: float
    root: int
    engine: str
    workers: int
    timings_ms: dict
    # B200 extras (not in the reference): GPU count, MST statistics, and the
    # stage outputs kept on the device (read lazily: tree arrays on first
    # attribute access, omega via omega_host())
    gpus: int = 1
    mst_stats: dict = field(default_factory=dict)
    tree: Any = field(default=None, repr=False, compare=False)
    extrema: Optional[Extrema] = field(default=None, repr=False, compare=False)
    omega_device: Any = field(default=None, repr=False, compare=False)
    p_device: Any = field(default=None, repr=False, compare=False)

    def omega_host(self) -> np.ndarray:
        return self.omega_device.cpu().numpy()

    def p_host(self) -> np.ndarray:
        return self.p_device.cpu().numpy()


def outcomes_equal(a: DecisionOutcome, b: DecisionOutcome) -> bool:
    """Field-for-field (bitwise) equality (isoperim.py:393-402)."""
    return (
        a.feasible == b.feasible
        and a.clusters_found == b.clusters_found
        and np.array_equal(a.cut, b.cut)
        and np.array_equal(a.eta, b.eta)
        and len(a.cluster_sparsities) == len(b.cluster_sparsities)
        and all(x == y for x, y in zip(a.cluster_sparsities, b.cluster_sparsities))
    )


def miso_results_equal(a: MisoResult, b: MisoResult) -> bool:
    """Bitwise equality of two solver results incl. the trace (isoperim.py:405-423)."""
    outcomes = (a.outcome is None and b.outcome is None) or (
        a.outcome is not None and b.outcome is not None and outcomes_equal(a.outcome, b.outcome)
    )
    return (
        outcomes
        and a.miso == b.miso
        and np.array_equal(a.labels, b.labels)
        and a.iterations == b.iterations
        and a.alpha_final == b.alpha_final
        and a.beta_final == b.beta_final
        and a.trace == b.trace
    )
