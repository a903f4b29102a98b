"""GPU: the two forms of the streaming epilogues k_dual / k_primal
(iter_kernels.cuh): operand streams through the shared-memory ring of bulk
async copies (bulk_stream, long vectors) or loaded by the threads
(reg_stream, short vectors). Each thread visits the same elements in the same
order in both, so the report partials, every decision and every iterate are
identical — the choice (Context::bulk_epilogue, by vector length) never
changes a result."""
import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, Tolerances

pytestmark = pytest.mark.gpu


def solve(lp, monkeypatch, form, **kw):
    monkeypatch.setenv("CCLP_CU_EPI", form)
    thresholds = kw.pop("thresholds", ())
    snaps = []
    with Engine(lp) as eng:
        res = eng.solve(PdhgConfig(**kw), Tolerances(), thresholds=thresholds, sink=snaps.append)
    return res, snaps


def lps():
    return [("eq40x90", lpgen.small_equality_lp(40, 90, 0.2, 7)[0]),
            ("transport20x30", lpgen.transportation_lp(20, 30, seed=3)),
            ("random2k", lpgen.random_equality_lp(2000, 10000, 8, seed=9)[0]),
            # more than 148 x 512 x 4 columns: the ring refills its stages
            ("random60k", lpgen.random_equality_lp(60000, 400000, 6, seed=11)[0])]


@pytest.mark.parametrize("name,lp", lps())
def test_bulk_and_register_epilogues_identical(name, lp, monkeypatch):
    a, sa = solve(lp, monkeypatch, "bulk", max_iterations=600, thresholds=[1e-1, 1e-2])
    b, sb = solve(lp, monkeypatch, "reg", max_iterations=600, thresholds=[1e-1, 1e-2])
    assert a.iterations == b.iterations and a.restarts == b.restarts and a.stop == b.stop
    for u, v in ((a.iterate.x, b.iterate.x), (a.iterate.y, b.iterate.y), (a.iterate.z, b.iterate.z)):
        assert np.array_equal(u, v)
    assert a.report.maxresid_rel == b.report.maxresid_rel and a.report.rel_gap == b.report.rel_gap
    assert [s.iteration for s in sa] == [s.iteration for s in sb]
    for s, t in zip(sa, sb):
        assert np.array_equal(s.iterate.x, t.iterate.x) and np.array_equal(s.iterate.y, t.iterate.y)


def test_epilogues_identical_to_convergence(monkeypatch):
    lp = lpgen.small_equality_lp(40, 90, 0.2, 7)[0]
    a, _ = solve(lp, monkeypatch, "bulk", max_iterations=100_000)
    b, _ = solve(lp, monkeypatch, "reg", max_iterations=100_000)
    assert a.iterations == b.iterations and a.stop == b.stop
    assert np.array_equal(a.iterate.x, b.iterate.x)


def _degenerate_lps():
    from paper_2510_24429_b200.lp import LinearProgram
    inf = np.inf
    c = np.array([1.0, -1.0, 0.0])
    return [("no_nonzeros", LinearProgram(2, 3, np.zeros(4, np.int32), np.zeros(0, np.int32), np.zeros(0), c,
                                          np.zeros(2), np.zeros(2), np.array([0.0, -inf, 0.0]),
                                          np.array([inf, 2.0, 1.0]))),
            ("no_rows", LinearProgram(0, 3, np.zeros(4, np.int32), np.zeros(0, np.int32), np.zeros(0), c,
                                      np.zeros(0), np.zeros(0), np.array([0.0, -5.0, 0.0]),
                                      np.array([inf, 2.0, 1.0])))]


@pytest.mark.parametrize("name,lp", _degenerate_lps())
@pytest.mark.parametrize("form", ["reg", "bulk"])
def test_degenerate_shapes_match_oracle(name, lp, form, monkeypatch, oracle):
    """No nonzeros / no rows: empty tiles in both epilogue forms, ||A|| = 0."""
    res, _ = solve(lp, monkeypatch, form, max_iterations=50)
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=50))
    assert res.iterations == ref["iterations"] and res.stop.name == "kConverged" and ref["stop"] == "converged"
    assert np.allclose(res.iterate.x, ref["x"], rtol=0, atol=1e-12)
