"""CPU: cclp::run_race and friends (race.hpp:86-129, SPEC.md "[MODULE] race")
as implemented in integration/run_race.cpp, with the SPEC's examples: the
threshold ladder, the thread split, the deterministic simulation, and a real
race over the reference's CPU run_pdhg + run_crossover (librace_cpu.so)."""
import pytest

from integration import race
from paper_2510_24429_b200 import lpgen

pytestmark = pytest.mark.skipif(not race.available("cpu"),
                                reason="integration/lib/librace_cpu.so not built (needs /root/reference at build time)")


def test_schedule_thresholds_examples():
    assert race.schedule_thresholds(1e-6, 1e-2, 0.1) == [1e-2, 1e-3, 1e-4, 1e-5]
    assert race.schedule_thresholds(1e-8, 1e-4, 0.1) == [1e-4, 1e-5, 1e-6, 1e-7]
    assert race.schedule_thresholds(1e-4, 1e-4, 0.1) == []
    with pytest.raises(ValueError):
        race.schedule_thresholds(1e-6, 1e-2, 1.5)


def test_reserve_threads_examples():
    assert race.reserve_threads(4, 16) == (12, 4)
    assert race.reserve_threads(4, 2) == (1, 1)


def test_simulated_later_faster_worker_wins():
    # {1e-2: 100 ms, 1e-3: 10 ms launched 20 ms later} -> 1e-3 wins at 30 ms
    trace = [5e-3] * 20 + [5e-4] * 200
    out = race.simulate(trace, 1e-3, {1e-2: (0.100, True), 1e-3: (0.010, True)})
    assert out["status"] == "solved"
    assert out["winner"] == "1e-03"
    assert out["wall_s"] == pytest.approx(0.030)
    assert out["pdhg_stop"] == "won-by-crossover"
    st = {w["threshold"]: w["status"] for w in out["workers"]}
    assert st == {"1e-02": "cancelled", "1e-03": "success"}


def test_simulated_baseline_main_wins_and_no_workers():
    trace = [5e-3] * 10 + [1e-7]
    out = race.simulate(trace, 1e-3, {1e-2: (0.001, True)}, main=(0.05, True), mode="baseline")
    assert out["status"] == "solved" and out["winner"] == "main" and out["main_won"]
    assert out["workers"] == []


def test_simulated_failed_verification_and_pool():
    trace = [5e-3] * 5 + [5e-4] * 5 + [5e-5] * 200
    out = race.simulate(trace, 1e-3, {1e-2: (1.0, False), 1e-3: (1.0, True), 1e-4: (0.001, True)},
                        pool=1)
    # pool of one: 1e-3 and 1e-4 arrive while 1e-2 runs and are dropped; 1e-2
    # then fails verification and PDHG never converges -> pdhg-limit
    assert [w["threshold"] for w in out["workers"]] == ["1e-02"]
    assert out["status"] == "pdhg-limit"


def test_cpu_race_two_var_and_transport():
    out = race.run_race(lpgen.two_var_lp(), kind="cpu")
    assert out["status"] == "solved"
    assert out["objective"] == pytest.approx(2.0, abs=1e-6)
    lp = lpgen.transportation_lp(8, 12, seed=3)
    base = race.run_race(lp, kind="cpu", mode="baseline")
    conc = race.run_race(lp, kind="cpu", mode="concurrent")
    assert base["status"] == conc["status"] == "solved"
    assert base["winner"] == "main"
    assert conc["objective"] == pytest.approx(base["objective"], rel=1e-9)


def _general_lp(m, n, seed, density=0.2):
    """Mixed row types: equality, <=, >=, ranged; a few empty columns."""
    import numpy as np
    from paper_2510_24429_b200.lp import INF, LinearProgram, csc_from_triplets
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < density
    mask[:, ::7] = False  # empty columns
    r, c = np.nonzero(mask)
    cp, ri, v = csc_from_triplets(m, n, r, c, rng.uniform(0.5, 2.0, r.size))
    kind = rng.integers(0, 4, m)
    b = rng.uniform(-1, 1, m)
    rl = np.where(kind == 2, -INF, b)
    ru = np.where(kind == 1, INF, np.where(kind == 3, b + 1.0, b))
    return LinearProgram(m, n, cp, ri, v, rng.normal(size=n), rl, ru,
                         np.zeros(n), np.where(rng.random(n) < 0.3, 4.0, INF))


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("maximize,named", [(False, False), (True, False), (False, True)])
def test_direct_standard_form_equals_reference(seed, maximize, named):
    """The race's O(nnz) to_standard_form_direct (integration/
    standard_form_direct.cpp) is field-for-field the reference's
    to_standard_form (standard_form.cpp:23-104)."""
    lp = _general_lp(23 + seed, 41 + 3 * seed, seed)
    ok, why = race.standard_form_check(lp, maximize, named)
    assert ok, why
    eq = lpgen.transportation_lp(5, 7, seed=seed)  # slack-free too
    ok, why = race.standard_form_check(eq, maximize, named)
    assert ok, why


def test_direct_standard_form_rejects_free_row():
    import numpy as np
    from paper_2510_24429_b200.lp import INF
    lp = _general_lp(10, 20, 3)
    lp.row_lower = lp.row_lower.copy()
    lp.row_upper = lp.row_upper.copy()
    lp.row_lower[4], lp.row_upper[4] = -INF, INF
    with pytest.raises(ValueError):
        race.standard_form_check(lp)


# ---- the scalable crossover (integration/crossover_scalable.cpp) -----------
@pytest.mark.parametrize("make", [lambda: lpgen.transportation_lp(20, 30, seed=3),
                                  lambda: lpgen.transportation_lp(20, 30, seed=4),
                                  lambda: lpgen.small_equality_lp(40, 90, 0.2, 7)[0],
                                  lambda: lpgen.two_var_lp()])
def test_scalable_crossover_race_matches_reference_crossover(make):
    """The race with the scalable crossover (sparse LU crash and factors,
    sparse etas, host pricing) ends on the reference crossover's basis."""
    lp = make()
    ref = race.run_race(lp, kind="cpu", mode="baseline", crossover="reference")
    sc = race.run_race(lp, kind="cpu", mode="baseline", crossover="scalable")
    race.set_crossover("cpu", "reference")
    assert ref["status"] == sc["status"] == "solved"
    assert sc["basic"] == ref["basic"]
    assert sc["objective"] == pytest.approx(ref["objective"], rel=1e-9, abs=1e-9)


@pytest.mark.parametrize("eps", [1e-2, 1e-4])
def test_scalable_crossover_from_snapshots_matches_reference(eps):
    """From the same PDHG iterate (the oracle's, at a ladder tolerance) both
    crossovers verify the same basis; the scalable one is the faster."""
    from oracle.pyoracle import Restatement
    from paper_2510_24429_b200 import lp as lpm
    std = lpm.to_standard_form(lpgen.transportation_lp(60, 150, seed=1))
    r = Restatement().run_pdhg(std, tol=dict(eps_rel=eps))
    a = race.crossover(std, r["x"], r["y"], r["z"], r["report"]["maxresid_rel"], crossover="reference")
    b = race.crossover(std, r["x"], r["y"], r["z"], r["report"]["maxresid_rel"], crossover="scalable")
    assert a["status"] == b["status"] == "success"
    assert a["basic"] == b["basic"]
    assert b["objective"] == pytest.approx(a["objective"], rel=1e-9)
    assert b["crash_accepted"] <= std.m and b["host_prices"] >= 1


def test_scalable_crossover_rejects_dependent_candidates_like_the_reference():
    """Duplicate columns: the second copy is dependent on the first and is
    rejected by the crash exactly as build_basis does (crossover.cpp:131-133)."""
    import numpy as np
    from paper_2510_24429_b200.lp import LinearProgram
    # min x0 + x1 + 3 x2 s.t. x0 + x1 + x2 = 2, x0 + x1 - x2 = 0 ; x0 and x1 identical columns
    colptr = np.array([0, 2, 4, 6], np.int32)
    rowind = np.array([0, 1, 0, 1, 0, 1], np.int32)
    val = np.array([1.0, 1.0, 1.0, 1.0, 1.0, -1.0])
    lp = LinearProgram(2, 3, colptr, rowind, val, np.array([1.0, 1.0, 3.0]), np.array([2.0, 0.0]),
                       np.array([2.0, 0.0]), np.zeros(3), np.full(3, np.inf), name="DUP")
    x = np.array([0.5, 0.5, 1.0]); y = np.array([2.0, -1.0]); z = np.array([0.0, 0.0, 0.0])
    a = race.crossover(lp, x, y, z, 1e-3, crossover="reference")
    b = race.crossover(lp, x, y, z, 1e-3, crossover="scalable")
    assert a["status"] == b["status"]
    assert a["basic"] == b["basic"]
