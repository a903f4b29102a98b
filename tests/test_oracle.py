"""CPU: the C restatement (oracle/cclp_oracle.c) pinned against the reference.

* golden fixtures (tests/golden/*.npz, produced by the reference's own code via
  tests/golden/make_golden.py) — bit for bit;
* the live reference build (oracle/_ref) when present — bit for bit;
* the reference's known-answer tests (test_pdhg.cpp, test_kkt.cpp,
  test_kernels.cpp, test_scaling.cpp) restated on the oracle.
"""
import glob
import os

import numpy as np
import pytest

from oracle.pyoracle import REPORT_FIELDS, STOP_NAMES
from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.lp import INF, LinearProgram

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def lp_from(g):
    return LinearProgram(int(g["m"]), int(g["n"]), g["colptr"], g["rowind"], g["val"], g["c"],
                         g["row_lower"], g["row_upper"], g["col_lower"], g["col_upper"])


@pytest.fixture(params=GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def golden(request):
    return np.load(request.param)


def test_golden_present():
    assert len(GOLDEN) >= 8


def test_golden_kernels_bit_exact(golden, oracle):
    lp = lp_from(golden)
    assert np.array_equal(oracle.matvec(lp, golden["mv_x"]), golden["ax"])
    assert np.array_equal(oracle.matvec_transpose(lp, golden["mv_y"]), golden["aty"])
    r, s, sv = oracle.ruiz(lp, 10)
    assert np.array_equal(r, golden["ruiz_r"])
    assert np.array_equal(s, golden["ruiz_s"])
    assert np.array_equal(sv, golden["ruiz_val"])
    assert oracle.estimate_norm(lp, 100, 0) == float(golden["norm100"])


def test_golden_run_pdhg_bit_exact(golden, oracle):
    lp = lp_from(golden)
    thr = list(golden["thresholds"])
    for it in golden["budgets"]:
        res = oracle.run_pdhg(lp, config=dict(max_iterations=int(it)), thresholds=thr)
        st = golden[f"it{it}_stats"]
        assert STOP_NAMES.index(res["stop"]) == st[0]
        assert res["iterations"] == st[1] and res["restarts"] == st[2]
        assert np.array_equal(res["x"], golden[f"it{it}_x"])
        assert np.array_equal(res["y"], golden[f"it{it}_y"])
        assert np.array_equal(res["z"], golden[f"it{it}_z"])
        rep = np.array([res["report"][f] for f in REPORT_FIELDS])
        assert np.array_equal(rep, golden[f"it{it}_report"])
        meta = golden[f"it{it}_snap_meta"]
        assert len(res["snapshots"]) == len(meta)
        for k, s in enumerate(res["snapshots"]):
            assert [s["threshold"], s["maxresid"], float(s["from_average"]), s["iteration"]] == \
                list(meta[k])
            assert np.array_equal(s["x"], golden[f"it{it}_snap{k}_x"])


def test_live_reference_bit_exact(oracle, reference):
    for seed in range(3):
        lp = lpgen.small_equality_lp(12, 30, 0.3, 100 + seed)[0]
        a = oracle.run_pdhg(lp, config=dict(max_iterations=3000), thresholds=[1e-2, 1e-3])
        b = reference.run_pdhg(lp, config=dict(max_iterations=3000), thresholds=[1e-2, 1e-3])
        assert a["stop"] == b["stop"] and a["iterations"] == b["iterations"]
        assert a["restarts"] == b["restarts"]
        assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])
        assert a["report"] == b["report"]
        rng = np.random.default_rng(seed)
        x, y, z = rng.standard_normal(lp.n), rng.standard_normal(lp.m), rng.standard_normal(lp.n)
        assert oracle.relative_report(lp, x, y, z) == reference.relative_report(lp, x, y, z)


def test_transportation_c1_reference_parity(oracle, reference):
    lp = lpgen.transportation_lp()
    a = oracle.run_pdhg(lp, config=dict(max_iterations=50))
    b = reference.run_pdhg(lp, config=dict(max_iterations=50))
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])


# ---- the reference's known-answer tests, restated on the oracle -------------

def row_lp(vals, m=1, rows=None):
    n = len(vals)
    rows = rows if rows is not None else [0] * n
    return LinearProgram(m, n, np.arange(n + 1, dtype=np.int32), np.array(rows, np.int32),
                         np.array(vals, float), np.ones(n), np.ones(m), np.ones(m), np.zeros(n),
                         np.full(n, INF))


def test_norm_known_answers(oracle):
    # test_pdhg.cpp:13-25
    assert oracle.estimate_norm(row_lp([1.0, 1.0]), 50, 1) == pytest.approx(np.sqrt(2), rel=1e-12)
    assert oracle.estimate_norm(row_lp([1.0, 1.0, 1.0], 3, [0, 1, 2]), 10, 1) == \
        pytest.approx(1.0, rel=1e-12)
    assert oracle.estimate_norm(row_lp([3.0, 4.0], 2, [0, 1]), 100, 1) == pytest.approx(4.0, rel=1e-10)


def test_norm_within_one_percent_of_svd(oracle):
    # test_pdhg.cpp:27-39
    rng = np.random.default_rng(3)
    for rep in range(25):
        lp = lpgen.small_equality_lp(int(rng.integers(2, 20)), int(rng.integers(2, 20)), 0.5,
                                     rep)[0]
        truth = np.linalg.svd(lp.dense(), compute_uv=False)[0]
        assert abs(oracle.estimate_norm(lp, 50, rep) - truth) <= 0.01 * truth


def test_two_var_first_step_and_convergence(oracle):
    # test_pdhg.cpp:41-49, 107-120, 122-136
    lp = lpgen.two_var_lp()
    res = oracle.run_pdhg(lp, thresholds=[1e-2, 1e-3])
    assert res["stop"] == "converged" and res["report"]["maxresid_rel"] <= 1e-6
    assert abs(res["x"][0] - 2.0) < 1e-4 and abs(res["x"][1]) < 1e-4
    snaps = res["snapshots"]
    assert [s["threshold"] for s in snaps] == [1e-2, 1e-3]
    assert snaps[0]["iteration"] < snaps[1]["iteration"]
    assert oracle.run_pdhg(lp, config=dict(max_iterations=0))["iterations"] == 0


def test_report_hand_evaluated_ratios(oracle):
    # test_kkt.cpp:61-75: all-zero iterate on the two-variable LP
    rep = oracle.relative_report(lpgen.two_var_lp(), np.zeros(2), np.zeros(1), np.zeros(2))
    assert rep["rel_primal"] == pytest.approx(2.0 / 3.0, rel=1e-15)
    assert rep["rel_dual"] == pytest.approx(np.sqrt(5) / (1 + np.sqrt(5)), rel=1e-15)
    assert rep["rel_gap"] == 0.0
    # test_kkt.cpp:49-59: the optimal pair has zero residuals
    rep = oracle.relative_report(lpgen.two_var_lp(), np.array([2.0, 0.0]), np.array([1.0]),
                                 np.array([0.0, 1.0]))
    assert rep["maxresid_rel"] == 0.0


def test_ruiz_powers_of_two_and_equilibrated(oracle):
    # test_scaling.cpp:70-99
    rng = np.random.default_rng(5)
    for rep in range(10):
        lp = lpgen.small_equality_lp(6, 11, 0.4, rep)[0]
        lp.val = lp.val * 10.0 ** rng.integers(-3, 4, size=lp.nnz)
        r, s, sv = oracle.ruiz(lp, 20)
        assert np.all(np.log2(r) == np.floor(np.log2(r)))
        assert np.all(np.log2(s) == np.floor(np.log2(s)))
        cols = np.repeat(np.arange(lp.n), np.diff(lp.colptr))
        rowmax = np.zeros(lp.m)
        np.maximum.at(rowmax, lp.rowind, np.abs(sv))
        colmax = np.zeros(lp.n)
        np.maximum.at(colmax, cols, np.abs(sv))
        for mx in (rowmax, colmax):
            nz = mx[mx > 0]
            assert np.all((nz >= 0.5) & (nz < 2.0))


def test_eigen_redux_order(oracle):
    # dot/norm follow Eigen 3.4's 2x2-packet reduction, not a sequential sum
    a = np.array([1e16, 1.0, -1e16, 1.0, 1.0])
    b = np.ones(5)
    p0a = (a[0] + a[4 - 4]) if False else None  # noqa: F841 (documentation only)
    # packets: p0=(a0,a1), p1=(a2,a3); p0+=p1 -> (a0+a2, a1+a3); hsum; tail a4
    expect = ((a[0] + a[2]) + (a[1] + a[3])) + a[4]
    assert oracle.dot(a, b) == expect
    assert oracle.norm(np.array([3.0, 4.0])) == 5.0


def test_gaussian_start_matches_libstdcxx(reference, oracle):
    # the restated mt19937_64 + normal_distribution drives the same ||A||
    lp = lpgen.small_equality_lp(30, 70, 0.2, 9)[0]
    for seed in (0, 1, 12345):
        assert oracle.estimate_norm(lp, 20, seed) == reference.estimate_norm(lp, 20, seed)


def test_preconditions(oracle):
    lp = lpgen.two_var_lp()
    with pytest.raises(ValueError):
        oracle.run_pdhg(lp, thresholds=[1e-3, 1e-2])
    with pytest.raises(ValueError):
        oracle.run_pdhg(lp, tol=dict(eps_rel=0.5))
    with pytest.raises(ValueError):
        oracle.run_pdhg(lp, config=dict(check_interval=0))
