"""GPU: long-row segmentation of the iteration SpMV (power-law row lengths,
SURVEY.md §8(a) 'merge-path on long rows'). Rows longer than 256*G nonzeros
are summed as fixed 4096-element segments by whole warps and combined in
segment order, so the result depends on the matrix only. Checked against the
CPU oracle at equal iteration counts (north_star tolerance 1e-6 relative)
and for run-to-run bit-identity."""
import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.lp import INF, LinearProgram, csc_from_triplets
from paper_2510_24429_b200.pdhg import PdhgConfig, PdhgStopReason, run_pdhg

pytestmark = pytest.mark.gpu

REL_TOL = 1e-6


def rel(a, b):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    return d / max(np.linalg.norm(b), 1e-300) if d > 0 else 0.0


def dense_rows_lp(m=300, n=40_000, dense=(0, 7, 150), seed=11):
    """Short random rows plus a few rows touching every column (length n),
    known optimum as in C2."""
    rng = np.random.default_rng(seed)
    r = rng.integers(0, m, size=6 * n)
    c = np.repeat(np.arange(n), 6)
    rows = [r, np.repeat(np.array(dense), n)]
    cols = [c, np.tile(np.arange(n), len(dense))]
    rows.append(np.arange(m))
    perm = rng.permutation(n)
    cols.append(perm[:m])
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rng.uniform(-2, 2, size=rows.size)
    vals[-m:] = rng.uniform(2, 3, size=m)
    colptr, rowind, val = csc_from_triplets(m, n, rows, cols, vals)
    return lpgen._known_optimum(colptr.astype(np.int64), rowind, val, m, n, perm[:m], rng,
                                "dense_rows")[0]


@pytest.fixture(scope="module")
def long_lp():
    return dense_rows_lp()


@pytest.mark.parametrize("iters", [0, 1, 25])
def test_long_rows_equal_iteration_parity(long_lp, iters, oracle):
    lp = long_lp
    res = run_pdhg(lp, PdhgConfig(max_iterations=iters))
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=iters))
    assert res.iterations == ref["iterations"]
    assert res.restarts == ref["restarts"]
    for a, b in ((res.iterate.x, ref["x"]), (res.iterate.y, ref["y"]), (res.iterate.z, ref["z"])):
        assert rel(a, b) <= REL_TOL


def test_long_rows_rerun_bit_identical(long_lp):
    a = run_pdhg(long_lp, PdhgConfig(max_iterations=300))
    b = run_pdhg(long_lp, PdhgConfig(max_iterations=300))
    assert np.array_equal(a.iterate.x, b.iterate.x)
    assert np.array_equal(a.iterate.y, b.iterate.y)


def test_long_rows_exact_mode_matches_fast(long_lp):
    fast = run_pdhg(long_lp, PdhgConfig(max_iterations=50))
    exact = run_pdhg(long_lp, PdhgConfig(max_iterations=50, exact_spmv=True))
    assert rel(fast.iterate.x, exact.iterate.x) <= 1e-9
    assert rel(fast.iterate.y, exact.iterate.y) <= 1e-9


def test_powerlaw_c5xs_parity(oracle):
    """C5 at 1/100 scale (5M nnz, rows up to ~3.6k): equal-iteration parity."""
    lp = lpgen.make_config("C5xs")
    res = run_pdhg(lp, PdhgConfig(max_iterations=20))
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=20))
    assert res.iterations == ref["iterations"] == 20
    assert rel(res.iterate.x, ref["x"]) <= REL_TOL
    assert rel(res.iterate.y, ref["y"]) <= REL_TOL


@pytest.fixture
def small_panels(monkeypatch):
    """Force column panels on small LPs (production: panels of 48 MB of x,
    i.e. only when x exceeds ~3 panels; C5 has 9)."""
    monkeypatch.setenv("CCLP_CU_PANEL_BYTES", "16384")


@pytest.mark.parametrize("iters", [1, 30])
def test_column_panels_parity(small_panels, iters, oracle):
    lp = lpgen.make_config("C5xs")  # 500k columns -> 245 panels of 2k columns
    res = run_pdhg(lp, PdhgConfig(max_iterations=iters))
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=iters))
    assert res.iterations == ref["iterations"]
    assert rel(res.iterate.x, ref["x"]) <= REL_TOL
    assert rel(res.iterate.y, ref["y"]) <= REL_TOL


def test_column_panels_rerun_and_exact(small_panels, long_lp):
    a = run_pdhg(long_lp, PdhgConfig(max_iterations=200))
    b = run_pdhg(long_lp, PdhgConfig(max_iterations=200))
    assert np.array_equal(a.iterate.x, b.iterate.x)
    exact = run_pdhg(long_lp, PdhgConfig(max_iterations=200, exact_spmv=True))
    assert rel(a.iterate.x, exact.iterate.x) <= 1e-9
