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
LIB_PATH = os.path.join(_HERE, "libisoclust_b200.so")
CSRC = os.path.join(_HERE, "csrc")

ISOC_OK, ISOC_EINVAL, ISOC_ETYPE, ISOC_EINFEASIBLE, ISOC_ENOMEM, ISOC_ECUDA = range(6)
FOLD_STACK_BYTES = 1544

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

# name -> (restype, argtypes)
SIGNATURES = {
    "isoc_version": (ctypes.c_int, []),
    "isoc_last_error": (ctypes.c_char_p, []),
    "isoc_sigma_partial": (ctypes.c_int, [P, I64, I32, I64, I64, D, P, P, P, P, P, P]),
    "isoc_sigma_finish": (ctypes.c_int, [P, I64, PD, P]),
    "isoc_omega": (ctypes.c_int, [P, I64, I32, I64, I64, D, P, P]),
    "isoc_omega_mst": (ctypes.c_int, [P, I64, I32, I64, I64, D, P, P, P, P, P, P]),
    "isoc_mst_create": (ctypes.c_int, [P, I64, I32, I64, I64, P, ctypes.POINTER(P)]),
    "isoc_mst_round_local": (ctypes.c_int, [P, ctypes.c_int, P, P, P, P]),
    "isoc_mst_round_edges": (ctypes.c_int, [P, P, P]),
    "isoc_mst_round_finish": (ctypes.c_int, [P, P, P, PI64, PI64, PI64]),
    "isoc_mst_edges": (ctypes.c_int, [P, P, P, P]),
    "isoc_mst_destroy": (None, [P]),
    "isoc_tree_from_edges": (ctypes.c_int, [P, P, P, I64, I64, D, P, ctypes.POINTER(P)]),
    "isoc_tree_from_parent": (ctypes.c_int, [P, P, P, I64, I64, P, ctypes.POINTER(P)]),
    "isoc_tree_export": (ctypes.c_int, [P, P, P, P, P, P, PI64, P]),
    "isoc_tree_set_weights": (ctypes.c_int, [P, P, P, P]),
    "isoc_decide": (ctypes.c_int, [P, D, I64, I32, PI64]),
    "isoc_witness": (ctypes.c_int, [P, I32, I64, P, P, P, P, PD]),
    "isoc_tree_destroy": (None, [P]),
    "isoc_exp_dev": (ctypes.c_int, [P, P, I64, P]),
    "isoc_launch_count": (ctypes.c_longlong, []),
    "isoc_prof_enable": (None, [ctypes.c_int]),
    "isoc_prof_read": (ctypes.c_int, [ctypes.c_int, PD, ctypes.POINTER(ctypes.c_longlong)]),
    "isoc_peak_tflops": (ctypes.c_int, [ctypes.c_int, PD]),
    "isoc_div_check": (ctypes.c_int, [ctypes.c_ulonglong, ctypes.c_ulonglong,
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
