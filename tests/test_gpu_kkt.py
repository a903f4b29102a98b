"""GPU: the verification side — relative_report and
absolute_violation (kkt.cpp:106-149) of arbitrary iterates computed on the
device (cclp_cu_relative_report), against the reference's own
relative_report (oracle/_ref) and the plain-C restatement. Products use the
reference-order SpMV, so maxima are exact; sums are reduced in a different
(fixed) order and agree to 1e-12 relative."""
import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.lp import INF, LinearProgram
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, REPORT_FIELDS

pytestmark = pytest.mark.gpu

EXACT = ("rp_inf", "rd_inf", "complementarity")


def _lps():
    yield "two_var", lpgen.two_var_lp()
    yield "small", lpgen.small_equality_lp(30, 70, 0.2, seed=3)[0]
    yield "transport", lpgen.transportation_lp(15, 25, seed=2)
    lp = lpgen.small_equality_lp(25, 60, 0.25, seed=8)[0]
    rng = np.random.default_rng(8)
    cl, cu = lp.col_lower.copy(), lp.col_upper.copy()
    kinds = rng.integers(0, 4, lp.n)  # free, lower only, upper only, boxed
    cl[kinds == 0], cu[kinds == 0] = -INF, INF
    cu[kinds == 1] = INF
    cl[kinds == 2], cu[kinds == 2] = -INF, rng.uniform(0, 3, (kinds == 2).sum())
    cl[kinds == 3], cu[kinds == 3] = -1.0, rng.uniform(0, 3, (kinds == 3).sum())
    yield "mixed_bounds", LinearProgram(lp.m, lp.n, lp.colptr, lp.rowind, lp.val, lp.c,
                                        lp.row_lower, lp.row_upper, cl, cu)


def _iterates(lp, rng):
    yield rng.normal(size=lp.n), rng.normal(size=lp.m), rng.normal(size=lp.n)
    yield np.zeros(lp.n), np.zeros(lp.m), np.zeros(lp.n)
    x = np.clip(rng.normal(size=lp.n), lp.col_lower, lp.col_upper)
    yield x, rng.normal(size=lp.m), np.where(rng.random(lp.n) < 0.5, 0.0, rng.normal(size=lp.n))


def _close(a, b, name):
    if name in EXACT:
        assert a == b, (name, a, b)
    else:
        assert a == pytest.approx(b, rel=1e-12, abs=1e-12), (name, a, b)


@pytest.mark.parametrize("name,lp", list(_lps()))
def test_relative_report_matches_reference(name, lp, reference, oracle):
    rng = np.random.default_rng(1)
    with Engine(lp) as eng:
        for x, y, z in _iterates(lp, rng):
            rep, av = eng.relative_report(x, y, z)
            ref = reference.relative_report(lp, x, y, z)
            res = oracle.relative_report(lp, x, y, z)
            for f in REPORT_FIELDS:
                _close(getattr(rep, f), ref[f], f)
                _close(getattr(rep, f), res[f], f)
            assert av == max(rep.rp_inf, rep.rd_inf, rep.complementarity)


def test_relative_report_of_a_solve_matches_the_solver():
    """The report the solver returns for its result equals an independent
    device recomputation on the returned iterate (C2 at 1/10 size)."""
    lp = lpgen.random_equality_lp(10_000, 50_000, 10, seed=4)[0]
    with Engine(lp) as eng:
        res = eng.solve(PdhgConfig(max_iterations=3000))
        rep, _ = eng.relative_report(res.iterate.x, res.iterate.y, res.iterate.z)
    for f in ("rel_primal", "rel_dual", "rel_gap", "maxresid_rel", "primal_objective", "dual_objective"):
        assert getattr(rep, f) == pytest.approx(getattr(res.report, f), rel=1e-9, abs=1e-12), f


def test_relative_report_rejects_inequality_rows():
    lp = lpgen.small_equality_lp(10, 20, 0.3, seed=1)[0]
    ru = lp.row_upper.copy()
    ru[0] += 1.0
    ineq = LinearProgram(lp.m, lp.n, lp.colptr, lp.rowind, lp.val, lp.c, lp.row_lower, ru,
                         lp.col_lower, lp.col_upper)
    with Engine(ineq) as eng:
        with pytest.raises(Exception):
            eng.relative_report(np.zeros(lp.n), np.zeros(lp.m), np.zeros(lp.n))
