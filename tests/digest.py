"""Compact, bitwise fixture digests for full-size parity (test infrastructure).

A digest is a flat dict of scalars (floats stored by their IEEE bit pattern)
and SHA-256 hex strings of arrays in a canonical dtype, so a 1M- or 50M-vertex
result can be compared bit for bit against a committed fixture of a few KB.
Used by tools/gen_golden_large.py (reference runs), tools/oracle_full.py
(oracle runs at C3/C4/C5), tests/ and bench.py's post-timing parity check.
"""
from __future__ import annotations

import hashlib
import json
import struct

import numpy as np

# canonical dtypes: arrays are cast before hashing so int32/int64 device
# exports hash identically
CANON = {
    "parent": np.int64, "child_id": np.int64, "depth": np.int64, "bfs_order": np.int64,
    "parent_flow": np.float64, "omega": np.float64, "p": np.float64,
    "labels": np.int64, "cut": np.int8, "eta": np.int64,
}


def fbits(x: float) -> str:
    return struct.pack("<d", float(x)).hex()


def from_fbits(h: str) -> float:
    return struct.unpack("<d", bytes.fromhex(h))[0]


def ahash(name: str, a) -> str:
    arr = np.ascontiguousarray(np.asarray(a), dtype=CANON.get(name, None))
    return hashlib.sha256(arr.tobytes()).hexdigest()


def edge_set_hash(parent) -> str:
    """Hash of the undirected MST edge set {(min(u,p), max(u,p))}, sorted."""
    par = np.asarray(parent, dtype=np.int64)
    u = np.flatnonzero(par >= 0)
    a = np.minimum(u, par[u])
    b = np.maximum(u, par[u])
    key = np.sort(a * (1 << 32) + b)
    return hashlib.sha256(np.ascontiguousarray(key).tobytes()).hexdigest()


def result_digest(result, *, sigma=None, tree=None, omega=None, p=None, extrema=None,
                  total_distance=None) -> dict:
    """Digest of a MisoResult-like object plus the stage outputs that exist."""
    out = {
        "miso": fbits(result.miso),
        "iterations": int(result.iterations),
        "alpha_final": fbits(result.alpha_final),
        "beta_final": fbits(result.beta_final),
        "trace_mid": [fbits(m) for m, _ in result.trace],
        "trace_ok": [int(bool(ok)) for _, ok in result.trace],
        "labels": ahash("labels", result.labels),
        "label_counts": np.bincount(np.asarray(result.labels, dtype=np.int64)).tolist(),
        "cut": ahash("cut", result.outcome.cut),
        "cut_vertices": np.flatnonzero(np.asarray(result.outcome.cut)).tolist(),
        "eta": ahash("eta", result.outcome.eta),
        "sparsities": [fbits(s) for s in result.outcome.cluster_sparsities],
    }
    if sigma is not None:
        out["sigma"] = fbits(sigma)
    if tree is not None:
        for name in ("parent", "child_id", "depth", "bfs_order", "parent_flow"):
            out[name] = ahash(name, getattr(tree, name))
        out["edge_set"] = edge_set_hash(tree.parent)
        out["max_depth"] = int(tree.max_depth)
    if omega is not None:
        out["omega"] = ahash("omega", omega)
    if p is not None:
        out["p"] = ahash("p", p)
    if extrema is not None:
        out["extrema"] = [fbits(v) for v in extrema]
    if total_distance is not None:
        out["total_distance"] = fbits(total_distance)
    return out


def compare(got: dict, want: dict, keys=None) -> list:
    """Names of the fields (present in both, or in `keys`) that differ."""
    keys = keys if keys is not None else [k for k in want if k in got and k != "meta"]
    return [k for k in keys if got.get(k) != want.get(k)]


def load(path) -> dict:
    with open(path) as f:
        return json.load(f)


def save(path, digest: dict) -> None:
    with open(path, "w") as f:
        json.dump(digest, f, indent=1, sort_keys=True)
        f.write("\n")
