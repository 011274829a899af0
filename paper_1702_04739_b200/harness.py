"""Host-side harness kept API-compatible with the reference (no kernels).

SURVEY.md 8(f) rank 4: the reference's point I/O (dataset.py), its
accuracy metric and timing harness (evaluation.py) and the two host
runtime objects its parallel engine exports (parengine.py DepthSchedule,
_primitives.py WorkerPool).  None of this is on the clustering hot path;
it exists so code written against `isoclust` finds the same names with the
same behaviour and error messages.  `benchmark` drives this package's
`run_pipeline` (the device engine).
"""
from __future__ import annotations

import csv
import io
import statistics
import sys
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Callable, Iterable, Optional, Sequence, Union

import numpy as np

from .pipeline import resolve_workers, run_pipeline
from .types import RootedTree

__all__ = [
    "BENCH_CSV_HEADER", "BenchRecord", "DataFormatError", "DepthSchedule", "WorkerPool", "benchmark",
    "class_count", "generate_random", "load_labels", "load_points", "misclassification_rate",
    "save_labels", "save_points", "standardize", "write_bench_csv",
]

_FORMATS = ("csv", "whitespace")


# ------------------------------------------------------------ dataset.py
class DataFormatError(ValueError):
    """Malformed input data (dataset.py:16-17); messages carry 1-based
    file row and column positions."""


def _check_format(format: str) -> str:
    if format not in _FORMATS:
        raise ValueError(f"unknown format {format!r}; expected 'csv' or 'whitespace'")
    return "," if format == "csv" else " "


def _rows_to_arrays(rows, label_column: Optional[int], path: str):
    """dataset.py:20-67: blank rows skipped, fixed width from the first data
    row, finite floats, label tokens mapped to ids by first appearance."""
    coords: list[list[float]] = []
    tokens: list[str] = []
    width = None
    for line_no, raw in rows:
        fields = [f.strip() for f in raw]
        if all(f == "" for f in fields):
            continue
        if width is None:
            width = len(fields)
            if label_column is not None and not 0 <= label_column < width:
                raise DataFormatError(f"{path}: label column {label_column} out of range for {width}-column data")
        elif len(fields) != width:
            raise DataFormatError(f"{path}: row {line_no}: expected {width} columns, found {len(fields)}")
        row: list[float] = []
        for col, tok in enumerate(fields):
            if col == label_column:
                tokens.append(tok)
                continue
            try:
                x = float(tok)
            except ValueError:
                raise DataFormatError(
                    f"{path}: row {line_no}, column {col + 1}: could not parse {tok!r} as a number") from None
            if not np.isfinite(x):
                raise DataFormatError(f"{path}: row {line_no}, column {col + 1}: non-finite value {tok!r}")
            row.append(x)
        coords.append(row)
    if len(coords) < 2:
        raise DataFormatError(f"{path}: need at least 2 data rows, found {len(coords)}")
    if not coords[0]:
        raise DataFormatError(f"{path}: rows contain no coordinate columns")
    points = np.asarray(coords, dtype=np.float64)
    if label_column is None:
        return points, None
    ids: dict[str, int] = {}
    return points, np.asarray([ids.setdefault(t, len(ids)) for t in tokens], dtype=np.int64)


def load_points(path: str, format: str = "csv", label_column: Optional[int] = None,
                header: bool = False) -> tuple[np.ndarray, Optional[np.ndarray]]:
    """dataset.py:70-100: read (points, labels) from delimited text."""
    _check_format(format)
    with open(path, "r", encoding="utf-8", newline="") as fh:
        lines = fh.read().splitlines()
    first = 1 if header else 0
    body = lines[first:]
    if format == "csv":
        parsed = csv.reader(io.StringIO("\n".join(body)))
    else:
        parsed = (line.split() for line in body)
    return _rows_to_arrays(((first + i + 1, r) for i, r in enumerate(parsed)), label_column, path)


def save_points(path: str, points: np.ndarray, labels: Optional[np.ndarray] = None, format: str = "csv") -> None:
    """dataset.py:103-125: repr() of each coordinate (round-trips exactly),
    optional trailing integer label column."""
    sep = _check_format(format)
    x = np.asarray(points, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError(f"points must be 2-d, got shape {x.shape}")
    if labels is not None and len(labels) != x.shape[0]:
        raise ValueError(f"labels length {len(labels)} does not match {x.shape[0]} points")
    out = []
    for i in range(x.shape[0]):
        fields = [repr(float(v)) for v in x[i]]
        if labels is not None:
            fields.append(str(int(labels[i])))
        out.append(sep.join(fields) + "\n")
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(out)


def save_labels(path: str, labels: np.ndarray) -> None:
    """dataset.py:128-132: one integer per line."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(f"{int(v)}\n" for v in np.asarray(labels).ravel())


def load_labels(path: str) -> np.ndarray:
    """dataset.py:135-137."""
    with open(path, "r", encoding="utf-8") as fh:
        return np.asarray([int(s) for s in fh if s.strip()], dtype=np.int64)


def generate_random(n: int, d: int, k: int, seed: int, spread: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """dataset.py:140-168: PCG64(seed) draws k centres U[0,10)^d, then
    N(0, spread) offsets for all n points at once; point i is in blob i % k.
    Bit-identical to the reference for the same arguments (the synthetic
    input of every BASELINE config)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    if n < max(2, k):
        raise ValueError(f"n must be >= max(2, k), got n={n}, k={k}")
    if d < 1:
        raise ValueError(f"d must be >= 1, got {d}")
    if not spread > 0:
        raise ValueError(f"spread must be > 0, got {spread}")
    gen = np.random.Generator(np.random.PCG64(seed))
    centres = gen.uniform(0.0, 10.0, size=(k, d))
    blob = np.arange(n, dtype=np.int64) % k
    noise = gen.normal(0.0, spread, size=(n, d))
    return centres[blob] + noise, blob


def standardize(points: np.ndarray) -> np.ndarray:
    """dataset.py:171-179: per-column z-score, zero-variance columns only centred."""
    x = np.asarray(points, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError(f"points must be 2-d, got shape {x.shape}")
    sd = x.std(axis=0)
    return (x - x.mean(axis=0)) / np.where(sd == 0.0, 1.0, sd)


def class_count(labels: np.ndarray) -> int:
    """dataset.py:182-191: number of classes of labels covering 0..c-1."""
    lab = np.asarray(labels, dtype=np.int64)
    if lab.size == 0:
        return 0
    c = int(lab.max()) + 1
    if lab.min() < 0 or np.unique(lab).size != c:
        raise ValueError("labels must cover the contiguous range 0..class_count-1")
    return c


# --------------------------------------------------------- evaluation.py
BENCH_CSV_HEADER = "dataset,n,d,k,engine,workers,affinity_ms,mst_ms,partition_ms,total_ms,miso,misclassification"


@dataclass
class BenchRecord:
    """evaluation.py:22-37: one dataset/engine measurement."""

    dataset: str
    n: int
    d: int
    k: int
    engine: str
    workers: int
    affinity_ms: float
    mst_ms: float
    partition_ms: float
    total_ms: float
    miso: float
    misclassification: Optional[float] = None


def misclassification_rate(pred, truth) -> float:
    """evaluation.py:40-70: 1 - (points matched by the best one-to-one
    cluster -> class assignment) / n; residual label 0 never matches."""
    from scipy.optimize import linear_sum_assignment

    p = np.asarray(pred, dtype=np.int64)
    t = np.asarray(truth, dtype=np.int64)
    if p.ndim != 1 or p.shape != t.shape:
        raise ValueError(f"pred and truth must be 1-d arrays of equal length, got {p.shape} and {t.shape}")
    if (p < 0).any():
        raise ValueError("predicted labels must be >= 0")
    if p.size == 0:
        raise ValueError("empty label arrays")
    classes = class_count(t)
    k = int(p.max())
    if k == 0:
        return 1.0
    sel = p > 0
    table = np.zeros((k, classes), dtype=np.int64)
    np.add.at(table, (p[sel] - 1, t[sel]), 1)
    r, c = linear_sum_assignment(-table)
    return 1.0 - int(table[r, c].sum()) / p.size


def _bench_one(name, points, truth, k, engine, repetitions, *, sigma, alpha, workers, root) -> BenchRecord:
    """evaluation.py:130-156: one discarded warm-up, then the median of
    each phase over `repetitions` runs."""
    run_pipeline(points, k, sigma, alpha, root, engine, workers)
    runs = [run_pipeline(points, k, sigma, alpha, root, engine, workers) for _ in range(repetitions)]
    med = {key: statistics.median(r.timings_ms[key] for r in runs) for key in ("affinity", "mst", "partition", "total")}
    last = runs[-1]
    return BenchRecord(dataset=name, n=last.n, d=last.d, k=k, engine=engine, workers=last.workers,
                       affinity_ms=med["affinity"], mst_ms=med["mst"], partition_ms=med["partition"],
                       total_ms=med["total"], miso=last.result.miso,
                       misclassification=misclassification_rate(last.result.labels, truth))


def benchmark(sizes: Sequence[int], dims: Sequence[int], ks: Sequence[int], engines: Sequence[str],
              seeds: Sequence[int], *, repetitions: int = 3, sigma: Union[str, float] = "auto",
              alpha: float = 0.0, workers: Optional[int] = None, spread: float = 1.0,
              root: int = 0) -> list[BenchRecord]:
    """evaluation.py:73-127: the (n, d, k, seed, engine) grid, one run at a
    time; invalid combinations are reported on stderr and skipped."""
    if repetitions < 1:
        raise ValueError(f"repetitions must be >= 1, got {repetitions}")
    if not sizes:
        raise ValueError("sizes must be nonempty")
    out: list[BenchRecord] = []
    for n in sizes:
        for d in dims:
            for k in ks:
                for seed in seeds:
                    name = f"rand-n{n}-d{d}-k{k}-s{seed}"
                    try:
                        points, truth = generate_random(n, d, k, seed, spread)
                    except ValueError as exc:
                        print(f"benchmark: skipping {name}: {exc}", file=sys.stderr)
                        continue
                    for engine in engines:
                        try:
                            out.append(_bench_one(name, points, truth, k, engine, repetitions, sigma=sigma,
                                                  alpha=alpha, workers=workers, root=root))
                        except ValueError as exc:
                            print(f"benchmark: skipping {name} ({engine}): {exc}", file=sys.stderr)
    return out


def write_bench_csv(records: Iterable[BenchRecord], path: str) -> None:
    """evaluation.py:159-169: fixed header; 3-decimal ms, repr() floats."""
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(BENCH_CSV_HEADER + "\n")
        for r in records:
            mis = "" if r.misclassification is None else repr(r.misclassification)
            fh.write(f"{r.dataset},{r.n},{r.d},{r.k},{r.engine},{r.workers},{r.affinity_ms:.3f},"
                     f"{r.mst_ms:.3f},{r.partition_ms:.3f},{r.total_ms:.3f},{r.miso!r},{mis}\n")


# ---------------------------------------------- host runtime objects
class WorkerPool:
    """_primitives.py:44-59: ordered map over a fixed chunk list on a
    bounded thread pool (results never depend on the worker count).  The
    device engine does not use it; it is exported for API compatibility."""

    def __init__(self, workers: Optional[int] = None):
        self.workers = resolve_workers(workers)

    def map(self, fn: Callable, chunks: Iterable) -> list:
        items = list(chunks)
        if self.workers == 1 or len(items) <= 1:
            return [fn(c) for c in items]
        with ThreadPoolExecutor(max_workers=self.workers) as ex:
            return list(ex.map(fn, items))


@dataclass(eq=False)
class DepthSchedule:
    """parengine.py:53-82: the level-synchronous sweep plan.  levels[i]
    lists the parent groups (ascending sibling rank) of depth
    max_depth - i; canonical_order[i] is that level in sweep order (groups
    reversed, descending sibling rank).  The device sweep (csrc/decide.cu)
    builds the same level ranges on the device; this host view is for
    callers that inspect the plan."""

    levels: list
    canonical_order: list
    depths: list

    @classmethod
    def from_tree(cls, tree: RootedTree) -> "DepthSchedule":
        order = np.asarray(tree.bfs_order)[::-1]
        dep = np.asarray(tree.depth)[order]
        par = np.asarray(tree.parent)
        levels, canonical, depths = [], [], []
        for lvl in range(int(tree.max_depth), -1, -1):
            members = order[dep == lvl]
            cuts = np.flatnonzero(np.diff(par[members]) != 0) + 1
            levels.append(list(np.split(members, cuts)))
            canonical.append(members[::-1].copy())
            depths.append(lvl)
        return cls(levels=levels, canonical_order=canonical, depths=depths)
