"""Shared pytest setup: the `gpu` marker, golden-fixture loading, repo paths."""
from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def golden_pipeline_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "pipe_*.npz")))


def load(path):
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def random_instance_trees():
    g = load(os.path.join(GOLDEN, "trees_random_instance.npz"))
    out = []
    for i in range(int(g["count"])):
        out.append({k.split("_", 1)[1]: v for k, v in g.items() if k.startswith(f"t{i}_")})
    return out


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle as orc
    orc.build()
    return orc
