"""bench.py host logic on CPU: the --gpus self-launch (torch.distributed.run
with N ranks), the reference arm's JSON line, and the ladder fit."""
from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_gpus_flag_self_launches_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "c1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "torch.distributed.run" in out.stderr and "--nproc-per-node=2" in out.stderr
    assert "rank 0/2" in out.stderr and "rank 1/2" in out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1          # rank 0 alone prints
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["workload"] == "c1 blobs N=2000 d=2 k=3"
    assert line["cpu_baseline"]["kind"] == "port" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "4",
                          "--config", "c1"], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


def test_ladder_fit_is_exact_on_model_data():
    sys.path.insert(0, ROOT)
    import bench
    pts = [{"n": m, "sigma": 2e-9 * m * m, "prim": 3e-9 * m * m, "omega": 1e-9 * m * m,
            "partition": 5e-7 * m} for m in (16000, 32000, 46340)]
    fit = bench.fit_ladder(pts, 1_000_000)
    assert abs(fit["extrapolated_s"]["sigma"] - 2000.0) < 1e-6
    assert abs(fit["extrapolated_s"]["partition"] - 0.5) < 1e-9
    assert abs(fit["total_s"] - (2000 + 3000 + 1000 + 0.5)) < 1e-6


def test_fixture_parity_accepts_the_oracle_run_and_rejects_a_perturbed_one(oracle_mod):
    """bench.fixture_parity (the bench's post-timing parity check) on the C1
    oracle run: fixture-match; with one label changed: MISMATCH."""
    import types
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench

    pts, _ = oracle_mod.generate_random(2000, 2, 3, 0)
    out = oracle_mod.run_pipeline(pts, 3)
    e = out.extrema
    run = types.SimpleNamespace(
        result=out.result, sigma=out.sigma, tree=out.tree, extrema=e,
        omega_host=lambda: out.omega, p_host=lambda: out.p)
    got = bench.fixture_parity("c1", 2000, 2, 3, run)
    assert got["status"] == "fixture-match" and got["fields_compared"] >= 20, got
    bad = out.result.labels.copy()
    bad[0] = (bad[0] % 3) + 1
    run.result = types.SimpleNamespace(**{**out.result.__dict__, "labels": bad})
    got = bench.fixture_parity("c1", 2000, 2, 3, run)
    assert got["status"] == "MISMATCH" and "labels" in got["differs"]
