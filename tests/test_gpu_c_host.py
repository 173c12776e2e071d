"""libmpcore from a plain C host (tests/c/dist_solve.c, include/mpcore.h
only): NCCL bootstrap, the distributed LU + solve at one rank and the
one-call solve, bitwise equal, built with gcc against the in-tree library."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_host_dist_solve(tmp_path):
    pkg = os.path.join(ROOT, "paper_2107_12550_b200")
    exe = str(tmp_path / "dist_solve")
    subprocess.run(["gcc", "-O2", "-o", exe,
                    os.path.join(ROOT, "tests", "c", "dist_solve.c"),
                    "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include",
                    "-L", pkg, "-l:libmpcore.so",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm",
                    "-Wl,-rpath," + pkg], check=True)
    r = subprocess.run([exe, "768"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bitwise-vs-one-call yes" in r.stdout
