import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# the engine's development knobs (csrc/host_util.cuh dev_knob) are read only with
# this switch; some tests force layouts through them
os.environ.setdefault("CCLP_CU_DEV_KNOBS", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a engine)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()
