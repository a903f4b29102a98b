"""GPU: the sm_100a engine against the golden fixtures made by the REFERENCE
itself (tests/golden/make_golden.py via oracle/_ref).

Bars (north_star): iterates within 1e-6 relative at equal iteration counts
(fp64), iterations-to-converge within 5%; Ruiz factors and the kernel-level
matvec (reference summation order) bit-exact."""
import glob
import os

import numpy as np
import pytest

from paper_2510_24429_b200.lp import LinearProgram
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, run_pdhg

pytestmark = pytest.mark.gpu
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
REL_TOL = 1e-6


def lp_from(g):
    return LinearProgram(int(g["m"]), int(g["n"]), g["colptr"], g["rowind"], g["val"], g["c"],
                         g["row_lower"], g["row_upper"], g["col_lower"], g["col_upper"])


def rel(a, b):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    return 0.0 if d == 0 else d / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(params=GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def golden(request):
    return np.load(request.param)


def test_kernels_bit_exact(golden):
    lp = lp_from(golden)
    with Engine(lp) as e:
        assert np.array_equal(e.matvec(golden["mv_x"]), golden["ax"])
        assert np.array_equal(e.matvec_transpose(golden["mv_y"]), golden["aty"])
        r, s = e.ruiz(10)
        assert np.array_equal(r, golden["ruiz_r"]) and np.array_equal(s, golden["ruiz_s"])
        assert e.estimate_norm(100, 0) == pytest.approx(float(golden["norm100"]), rel=1e-12)


@pytest.mark.parametrize("exact", [False, True])
def test_run_pdhg_against_reference(golden, exact):
    lp = lp_from(golden)
    thr = list(golden["thresholds"])
    with Engine(lp) as e:
        for it in golden["budgets"]:
            snaps = []
            res = e.solve(PdhgConfig(max_iterations=int(it), exact_spmv=exact), thresholds=thr,
                          sink=snaps.append)
            stop, iters, restarts, _ = golden[f"it{it}_stats"]
            assert int(res.stop) == stop
            if it < 20000 or stop != 0:  # equal iteration budgets
                assert res.iterations == iters and res.restarts == restarts
                assert rel(res.iterate.x, golden[f"it{it}_x"]) <= REL_TOL
                assert rel(res.iterate.y, golden[f"it{it}_y"]) <= REL_TOL
                assert rel(res.iterate.z, golden[f"it{it}_z"]) <= REL_TOL
            else:  # run to convergence: iteration counts within 5%
                assert abs(res.iterations - iters) <= 0.05 * iters
            meta = golden[f"it{it}_snap_meta"]
            assert [s.iteration for s in snaps] == [int(mm[3]) for mm in meta]
            assert [s.threshold for s in snaps] == [mm[0] for mm in meta]
            for k, s in enumerate(snaps):
                assert rel(s.iterate.x, golden[f"it{it}_snap{k}_x"]) <= REL_TOL
