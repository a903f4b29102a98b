"""GPU: the reference's own test_pdhg.cpp suite (12 TEST_CASEs, unmodified),
linked against integration/run_pdhg_cuda.cpp — cclp::run_pdhg re-implemented
over the C ABI — so every run_pdhg call in the reference's tests executes on
the B200 engine (oracle/Makefile `dropin`)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "test_pdhg_gpu")


def test_reference_pdhg_suite_on_gpu_engine():
    if not os.path.exists(EXE):
        pytest.skip("drop-in binary not built (needs /root/reference at build time)")
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout
