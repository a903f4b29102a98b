"""GPU: the speculative row product (row_step, iter_kernels.cuh). On the
single-device loop with the SELL-G row product, step t's A x_{t+1} starts on
the no-restart candidate while the last block of k_primal(t-1) still runs the
decision tail, and is recomputed from the restart candidate in the steps that
restart. Per-row order is unchanged, so every iterate, report, restart,
snapshot and stop equals the waiting form's (CCLP_CU_SPEC=0, a development
knob) exactly — including the stops that return state t-1 or state t while
the speculative product has already written state t+1's ax slot."""
import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, Tolerances

pytestmark = pytest.mark.gpu


def solve(lp, monkeypatch, spec, thresholds=(), tol=None, **kw):
    monkeypatch.setenv("CCLP_CU_SPEC", "1" if spec else "0")
    # the SELL-G row product (chosen by timing in production): pinned here so
    # the speculative form is the one under test on every box
    monkeypatch.setenv("CCLP_CU_SELL_ROWS", "2")
    snaps = []
    with Engine(lp) as eng:
        res = eng.solve(PdhgConfig(**kw), tol or Tolerances(), thresholds=thresholds, sink=snaps.append)
        on = eng.describe()["speculative_rows"]
    return res, snaps, on


def same(a, b, sa=(), sb=()):
    assert (a.iterations, a.restarts, a.stop) == (b.iterations, b.restarts, b.stop)
    for u, v in ((a.iterate.x, b.iterate.x), (a.iterate.y, b.iterate.y), (a.iterate.z, b.iterate.z)):
        assert np.array_equal(u, v)
    assert a.report.maxresid_rel == b.report.maxresid_rel and a.report.rel_gap == b.report.rel_gap
    assert [s.iteration for s in sa] == [s.iteration for s in sb]
    for s, t in zip(sa, sb):
        assert np.array_equal(s.iterate.x, t.iterate.x) and np.array_equal(s.iterate.y, t.iterate.y)


@pytest.fixture(scope="module")
def random_lp():
    # C2 at half size: SELL-G rows (near-uniform rows), the speculative form
    return lpgen.random_equality_lp(50000, 250000, 10, seed=11)[0]


def test_speculative_rows_active_on_sell_rows(random_lp, monkeypatch):
    _, _, on = solve(random_lp, monkeypatch, True, max_iterations=10)
    assert on
    _, _, off = solve(random_lp, monkeypatch, False, max_iterations=10)
    assert not off


@pytest.mark.parametrize("iters", [1, 2, 3, 65, 1500])
def test_speculative_identical_at_iteration_limit(random_lp, monkeypatch, iters):
    """Stop at max_iterations (state t returned; the speculative product of
    step t has written state t+1's slot) at batch edges and mid-batch."""
    a, sa, on = solve(random_lp, monkeypatch, True, max_iterations=iters, thresholds=[1e-1, 3e-2])
    b, sb, _ = solve(random_lp, monkeypatch, False, max_iterations=iters, thresholds=[1e-1, 3e-2])
    assert on
    same(a, b, sa, sb)


def test_speculative_identical_with_restarts(random_lp, monkeypatch):
    """Restarting steps recompute the row product from the restart candidate."""
    a, sa, _ = solve(random_lp, monkeypatch, True, max_iterations=4000, thresholds=[1e-1, 1e-2, 1e-3])
    b, sb, _ = solve(random_lp, monkeypatch, False, max_iterations=4000, thresholds=[1e-1, 1e-2, 1e-3])
    assert a.restarts > 0
    same(a, b, sa, sb)


def test_speculative_identical_to_convergence(monkeypatch):
    lp = lpgen.random_equality_lp(20000, 100000, 12, seed=5)[0]
    a, _, on = solve(lp, monkeypatch, True, max_iterations=200_000, tol=Tolerances(eps_rel=1e-5))
    b, _, _ = solve(lp, monkeypatch, False, max_iterations=200_000, tol=Tolerances(eps_rel=1e-5))
    assert a.stop.name == "kConverged"
    same(a, b)


def test_speculative_identical_check_interval(random_lp, monkeypatch):
    a, _, _ = solve(random_lp, monkeypatch, True, max_iterations=700, check_interval=64)
    b, _, _ = solve(random_lp, monkeypatch, False, max_iterations=700, check_interval=64)
    same(a, b)


def test_speculative_numerical_error_returns_pre_step_state(monkeypatch):
    """A non-finite step returns the pre-step state (pdhg.cpp:128-130): its ax
    slot is not the one the speculative product of the next step writes (with
    two ping-pong slots it would be)."""
    lp = lpgen.random_equality_lp(50000, 250000, 10, seed=11)[0]
    lp.c[0] = 1e308  # overflows the first primal step (test_gpu_parity.py's recipe)
    kw = dict(max_iterations=50, scaling_iterations=0, step_scale=1.0)
    a, _, on = solve(lp, monkeypatch, True, **kw)
    b, _, _ = solve(lp, monkeypatch, False, **kw)
    assert on and int(a.stop) == 5 and a.stop == b.stop
    assert a.iterations == b.iterations and a.error_iteration == b.error_iteration
    for u, v in ((a.iterate.x, b.iterate.x), (a.iterate.y, b.iterate.y), (a.iterate.z, b.iterate.z)):
        assert np.array_equal(u, v, equal_nan=True)
    assert np.array_equal(np.array([a.report.maxresid_rel, a.report.rel_gap]),
                          np.array([b.report.maxresid_rel, b.report.rel_gap]), equal_nan=True)


def test_bench_config_takes_the_fast_paths():
    """C2 (the bench workload): SELL-G rows with the speculative row product
    and SELL-32 columns — the layouts the measured numbers come from."""
    lp = lpgen.make_config("C2")
    with Engine(lp) as eng:
        eng.begin(PdhgConfig())
        eng.advance(10)
        d = eng.describe()
    assert d["sell_rows_block"] > 0 and d["sell_cols_block"] > 0 and d["speculative_rows"]
