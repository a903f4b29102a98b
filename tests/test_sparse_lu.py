"""The product crossover's basis factorization (third_party/eigen_subset
SparseLU: sparse left-looking LU with threshold pivoting) -- compiled and run
on the host; the reference's own test_simplex / test_crossover suites over it
run in tests/test_reference_suites.py."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sparse_lu_residuals_singularity_and_fill(tmp_path):
    exe = tmp_path / "sparse_lu_check"
    cc = subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "third_party", "eigen_subset"),
                         os.path.join(ROOT, "tests", "native", "sparse_lu_check.cpp"), "-o", str(exe)],
                        capture_output=True, text=True)
    if cc.returncode != 0:
        pytest.fail(cc.stderr[-2000:])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout[-3000:]
