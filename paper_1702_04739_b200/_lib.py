"""ctypes binding of libisoclust_b200.so (include/isoclust_b200.h).

The library is built in-tree (paper_1702_04739_b200/csrc/Makefile).  There
is no CPU fallback: a missing library raises ImportError at first use, and
every non-zero status is mapped to the exception type the reference raises
for the same condition.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# ISOC_LIB_PATH: an alternative build of the same library (kernel variants
# timed side by side by tools/time_passes.py); never a CPU substitute
LIB_PATH = os.environ.get("ISOC_LIB_PATH") or os.path.join(_HERE, "libisoclust_b200.so")
CSRC = os.path.join(_HERE, "csrc")

ISOC_OK, ISOC_EINVAL, ISOC_ETYPE, ISOC_EINFEASIBLE, ISOC_ENOMEM, ISOC_ECUDA = range(6)
FOLD_STACK_BYTES = 1544
ROW_CAP = 40          # per-row leaf-stack entries of the sigma passes (csrc/kernels.h kRowCap)

_lock = threading.Lock()
_lib = None


class InfeasibleSubpartitionError(RuntimeError):
    """No k disjoint nonempty clusters exist under the search bracket
    (reference: isoperim.py:33)."""


def build(force: bool = False) -> str:
    """Compile the CUDA library for sm_100a (nvcc cross-compiles without a GPU)."""
    args = ["make", "-s", "-C", CSRC]
    if force:
        subprocess.run(args + ["clean"], check=True)
    subprocess.run(args, check=True)
    return LIB_PATH


P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
D = ctypes.c_double
PI64 = ctypes.POINTER(ctypes.c_int64)
PD = ctypes.POINTER(ctypes.c_double)

class RunOut(ctypes.Structure):
    """isoc_run_out (include/isoclust_b200.h)."""
    _fields_ = [("labels", P), ("cut", P), ("eta", P), ("sparsities", P), ("trace_mid", P),
                ("trace_ok", P), ("trace_cap", ctypes.c_int32), ("trace_len", ctypes.c_int32),
                ("iterations", I64), ("clusters_found", I64), ("miso", D), ("sigma", D),
                ("alpha_final", D), ("beta_final", D), ("timings_ms", D * 4),
                ("boruvka_rounds", I64), ("exact_ties", I64), ("exact_rescans", I64)]


# name -> (restype, argtypes)
SIGNATURES = {
    "isoc_version": (ctypes.c_int, []),
    "isoc_last_error": (ctypes.c_char_p, []),
    "isoc_sigma_partial": (ctypes.c_int, [P, I64, I32, I64, I64, D, P, P, P, P, P, P]),
    "isoc_sigma_finish": (ctypes.c_int, [P, I64, PD, P]),
    "isoc_sym_block_range": (ctypes.c_int, [I64, I32, I32, PI64, PI64]),
    "isoc_omega_block_range": (ctypes.c_int, [I64, I32, I32, PI64, PI64]),
    "isoc_sigma_sym_range": (ctypes.c_int, [P, I64, I32, I64, I64, P, P, P, P, P, P, P]),
    "isoc_sigma_rank_merge": (ctypes.c_int, [P, I64, I32, I64, I64, I32, P, P, P, P, P, P, P, P, P, P, P]),
    "isoc_omega": (ctypes.c_int, [P, I64, I32, I64, I64, D, P, P]),
    "isoc_omega_mst": (ctypes.c_int, [P, I64, I32, I64, I64, D, P, P, P, P, P, P]),
    "isoc_omega_shard_counts": (ctypes.c_int, [I64, I32, I32, P, P]),
    "isoc_omega_sym_range": (ctypes.c_int, [P, I64, I32, I32, I32, D, P, P, P, P, P]),
    "isoc_omega_rank_merge": (ctypes.c_int, [I64, I32, I32, P, P, P, P, P, P, P, P]),
    "isoc_distance_matrix": (ctypes.c_int, [P, I64, I32, P, P]),
    "isoc_flow": (ctypes.c_int, [P, I64, D, P, P]),
    "isoc_vertex_weights_dense": (ctypes.c_int, [P, I64, D, P, P]),
    "isoc_potentials_dense": (ctypes.c_int, [P, I64, D, P, P]),
    "isoc_pairwise_sum": (ctypes.c_int, [P, I64, PD, P]),
    "isoc_validate_distance_matrix": (ctypes.c_int, [P, I64, ctypes.POINTER(ctypes.c_int32), P]),
    "isoc_mst_dense": (ctypes.c_int, [P, I64, P, P, P, PI64, P]),
    "isoc_sum_reduce": (ctypes.c_int, [P, I64, PD, P]),
    "isoc_min_reduce": (ctypes.c_int, [P, I64, PD, PI64, P]),
    "isoc_exclusive_scan": (ctypes.c_int, [P, I64, P, P]),
    "isoc_extract_labels": (ctypes.c_int, [P, P, I64, P, P]),
    "isoc_brute_force_miso": (ctypes.c_int, [P, P, P, P, I32, I32, PI64, PD, P]),
    "isoc_mst_create": (ctypes.c_int, [P, I64, I32, I64, I64, P, ctypes.POINTER(P)]),
    "isoc_mst_round_local": (ctypes.c_int, [P, ctypes.c_int, P, P, P, P]),
    "isoc_mst_round_edges": (ctypes.c_int, [P, P, P]),
    "isoc_mst_round_finish": (ctypes.c_int, [P, P, P, PI64, PI64, PI64]),
    "isoc_mst_edges": (ctypes.c_int, [P, P, P, P]),
    "isoc_prim_edges": (ctypes.c_int, [P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, P, P, P, P]),
    "isoc_mst_filter_stats": (ctypes.c_int, [P, PI64, PI64, PI64]),
    "isoc_prim_edges_dense": (ctypes.c_int, [P, ctypes.c_int64, ctypes.c_int64, P, P, P, P]),
    "isoc_mst_destroy": (None, [P]),
    "isoc_tree_from_edges": (ctypes.c_int, [P, P, P, I64, I64, D, P, ctypes.POINTER(P)]),
    "isoc_tree_from_parent": (ctypes.c_int, [P, P, P, I64, I64, P, ctypes.POINTER(P)]),
    "isoc_tree_export": (ctypes.c_int, [P, P, P, P, P, P, PI64, P]),
    "isoc_tree_root": (ctypes.c_int, [P, PI64]),
    "isoc_tree_cost": (ctypes.c_int, [P, P, I64, PD]),
    "isoc_tree_set_weights": (ctypes.c_int, [P, P, P, P]),
    "isoc_decide": (ctypes.c_int, [P, D, I64, I32, PI64]),
    "isoc_witness": (ctypes.c_int, [P, I32, I64, P, P, P, P, PD]),
    "isoc_decide_batch_capacity": (ctypes.c_int, [P, P]),
    "isoc_decide_batch": (ctypes.c_int, [P, P, I32, I64, P]),
    "isoc_tree_shape": (ctypes.c_int, [P, PI64, PI64]),
    "isoc_tree_destroy": (None, [P]),
    "isoc_exp_dev": (ctypes.c_int, [P, P, I64, P]),
    "isoc_run": (ctypes.c_int, [P, I64, I32, I64, D, D, I64, P, ctypes.POINTER(RunOut)]),
    "isoc_release_cached_memory": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong)]),
    "isoc_launch_count": (ctypes.c_longlong, []),
    "isoc_prof_enable": (None, [ctypes.c_int]),
    "isoc_prof_read": (ctypes.c_int, [ctypes.c_int, PD, ctypes.POINTER(ctypes.c_longlong)]),
    "isoc_peak_tflops": (ctypes.c_int, [ctypes.c_int, PD]),
    "isoc_div_check": (ctypes.c_int, [ctypes.c_ulonglong, ctypes.c_ulonglong,
                                      ctypes.POINTER(ctypes.c_ulonglong), PD]),
    "isoc_fastpath_check": (ctypes.c_int, [ctypes.c_ulonglong, ctypes.c_ulonglong,
                                           ctypes.POINTER(ctypes.c_ulonglong), PD]),
}


def load():
    """Load the library (building it if the .so is absent and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            try:
                build()
            except Exception as exc:  # pragma: no cover - depends on toolchain
                raise ImportError(f"libisoclust_b200.so missing and build failed: {exc}") from exc
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("ISOC_LIB_PATH") and not hasattr(lib, name):
                continue   # an older variant build timed side by side (diagnostics only)
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    if status == ISOC_OK:
        return
    msg = load().isoc_last_error().decode(errors="replace")
    if status == ISOC_EINVAL:
        raise ValueError(msg)
    if status == ISOC_ETYPE:
        raise TypeError(msg)
    if status == ISOC_EINFEASIBLE:
        raise InfeasibleSubpartitionError(msg)
    if status == ISOC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"isoclust_b200: {msg}")


def run(points, k: int, sigma: float = 0.0, alpha: float = 0.0, root: int = 0) -> dict:
    """One-call C path (isoc_run): the whole pipeline on one GPU from host
    numpy points; sigma <= 0 means "auto".  Returns the outputs as a dict."""
    import numpy as np

    X = np.ascontiguousarray(points, dtype=np.float64)
    if X.ndim != 2:
        raise ValueError(f"points must be a 2-d array, got shape {X.shape}")
    if isinstance(k, bool) or not isinstance(k, (int, np.integer)):
        raise TypeError(f"k must be an integer, got {type(k).__name__}")
    n, d = X.shape
    cap = 256
    labels = np.empty(n, np.int64)
    cut = np.empty(n, np.int8)
    eta = np.empty(n, np.int64)
    sp = np.empty(max(int(k), 1), np.float64)
    tmid = np.empty(cap, np.float64)
    tok = np.empty(cap, np.uint8)
    out = RunOut()
    out.labels, out.cut, out.eta = labels.ctypes.data, cut.ctypes.data, eta.ctypes.data
    out.sparsities, out.trace_mid, out.trace_ok = sp.ctypes.data, tmid.ctypes.data, tok.ctypes.data
    out.trace_cap = cap
    check(load().isoc_run(X.ctypes.data, n, d, int(k), float(sigma), float(alpha), int(root), None,
                          ctypes.byref(out)))
    m = min(out.trace_len, cap)
    return {"labels": labels, "cut": cut, "eta": eta, "sparsities": [float(v) for v in sp[:out.clusters_found]],
            "trace": [(float(tmid[i]), bool(tok[i])) for i in range(m)], "iterations": int(out.iterations),
            "miso": float(out.miso), "sigma": float(out.sigma), "alpha_final": float(out.alpha_final),
            "beta_final": float(out.beta_final), "timings_ms": list(out.timings_ms),
            "mst_stats": {"boruvka_rounds": int(out.boruvka_rounds), "exact_ties": int(out.exact_ties),
                          "exact_rescans": int(out.exact_rescans)}}
