"""The O(1) pairwise-sum leaf successor (csrc/leaf.h) equals numpy's recursion.

Compiles tools/checks/leaf_check.cpp (host build of the same header the σ
kernel uses) and walks leaves for every total < 6000 plus random large
totals (including n*n), comparing start/length/heap id with the plain
descent of numpy's pairwise_sum split rule.
"""
import os
import subprocess

from conftest import ROOT


def test_leaf_successor_matches_descent(tmp_path):
    exe = str(tmp_path / "leaf_check")
    subprocess.run(["/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++", "-O2", "-std=c++17",
                    "-I", os.path.join(ROOT, "paper_1702_04739_b200", "csrc"),
                    os.path.join(ROOT, "tools", "checks", "leaf_check.cpp"), "-o", exe], check=True)
    out = subprocess.run([exe, "6000", "300"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bad=0" in out.stdout
