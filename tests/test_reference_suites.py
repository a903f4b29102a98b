"""CPU: the reference's OWN doctest suites (proj/tests/test_{kernels,scaling,
kkt,pdhg,standard_form,simplex,crossover}.cpp), compiled unmodified against the Eigen/doctest
API shims by oracle/Makefile, must pass. This pins the shim — and therefore
oracle/_ref and the golden fixtures made from it — to the reference's own
expectations."""
import os
import subprocess

import pytest

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
SUITES = ["test_kernels", "test_scaling", "test_kkt", "test_pdhg", "test_standard_form",
          "test_simplex", "test_crossover"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes(suite):
    exe = os.path.join(REF, suite)
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout
