"""GPU at BASELINE.json's full sizes (C2, C3, C4, C5s) through properties
that do not need a full CPU solve (the CPU oracle would take minutes to
hours there), plus the loop's control paths on small LPs:

* C2: equal-iteration parity against the CPU oracle itself (20 iterations),
  and the first ladder snapshot (1e-2, iteration 681) against its synchronous
  snapshot;
  C3 (20), C4 (5) and C5s (20) the same, against the plain-C restatement of the
  reference (bit-exact to the reference's own build, tests/test_oracle.py).
* Convergence against fixtures made by the reference's own run_pdhg
  (tests/golden/make_convergence.py): C1 to 1e-6 and C2 to 1e-4 -- iterations
  within 5 % (north_star) and the restart counts.
* C3/C4/C5s: the returned report equals the oracle's independent
  relative_report (kkt.cpp:50-149) recomputed on the returned iterate;
  reruns are bit-identical; C4 sharded (P = 2, halo exchange) is
  bit-identical to one device.
* cancel / time limit / check_interval > 1 / the iteration log.
"""
import re
import threading
import time

import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import (Engine, PdhgConfig, PdhgStopReason, ShardedEngine,
                                        run_pdhg)

pytestmark = pytest.mark.gpu

REPORT_KEYS = ["rp_norm2", "rd_norm2", "rp_inf", "rd_inf", "primal_objective", "dual_objective",
               "gap_abs", "rel_primal", "rel_dual", "rel_gap", "maxresid_rel", "complementarity"]


def rel(a, b):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    return d / max(np.linalg.norm(b), 1e-300) if d > 0 else 0.0


@pytest.fixture(scope="module")
def lps():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = lpgen.make_config(name)
        return cache[name]
    return get


def test_c2_full_size_equal_iteration_parity(lps, oracle):
    lp = lps("C2")
    res = run_pdhg(lp, PdhgConfig(max_iterations=20))
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=20))
    assert res.iterations == ref["iterations"] == 20
    assert rel(res.iterate.x, ref["x"]) <= 1e-6
    assert rel(res.iterate.y, ref["y"]) <= 1e-6
    assert rel(res.iterate.z, ref["z"]) <= 1e-6


def test_c2_full_size_snapshot_parity(lps, oracle):
    """The ladder's first snapshot at full C2 size (iteration 681 at 1e-2),
    extracted by the iteration kernels into a device slot while the loop runs
    on: the same iteration, threshold and iterate as the restatement's
    synchronous snapshot (pdhg.cpp:346-358)."""
    lp = lps("C2")
    snaps = []
    res = run_pdhg(lp, PdhgConfig(max_iterations=700), thresholds=[1e-2], sink=snaps.append)
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=700), thresholds=[1e-2])
    assert res.iterations == ref["iterations"] == 700
    assert len(snaps) == len(ref["snapshots"]) == 1
    s, r = snaps[0], ref["snapshots"][0]
    assert s.iteration == r["iteration"] and s.threshold == r["threshold"]
    assert s.from_average == bool(r["from_average"])
    for a, b in ((s.iterate.x, r["x"]), (s.iterate.y, r["y"]), (s.iterate.z, r["z"])):
        assert rel(a, b) <= 1e-6
    assert rel(res.iterate.x, ref["x"]) <= 1e-6


@pytest.mark.parametrize("name,iters", [("C3", 20), ("C4", 5), ("C5s", 20)])
def test_full_size_equal_iteration_parity(name, iters, lps, oracle):
    """north_star: x, y, z within 1e-6 relative after equal iteration counts,
    on BASELINE.json's own configs (the oracle's setup -- 10 Ruiz passes and 100
    power iterations -- dominates its minute of CPU time here)."""
    lp = lps(name)
    res = run_pdhg(lp, PdhgConfig(max_iterations=iters))
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=iters))
    assert res.iterations == ref["iterations"] == iters
    assert res.restarts == ref["restarts"]
    assert res.stop == PdhgStopReason.kIterationLimit and ref["stop"] == "iteration-limit"
    assert rel(res.iterate.x, ref["x"]) <= 1e-6
    assert rel(res.iterate.y, ref["y"]) <= 1e-6
    assert rel(res.iterate.z, ref["z"]) <= 1e-6
    for k in ("rel_primal", "rel_dual", "rel_gap"):
        assert getattr(res.report, k) == pytest.approx(ref["report"][k], rel=1e-6, abs=1e-12), k


def _fixture(config, eps):
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                     f"convergence_{config}_{eps:.0e}.json")
    if not os.path.exists(p):
        pytest.skip(f"{p} not generated")
    with open(p) as f:
        return json.load(f)


@pytest.mark.parametrize("name,eps", [("C1", 1e-6), ("C2", 1e-4)])
def test_convergence_matches_reference_fixture(name, eps, lps):
    """Iterations-to-converge within 5 % of the reference's own run_pdhg
    (north_star), same stop, and the restart count within one."""
    from paper_2510_24429_b200.pdhg import Tolerances
    fx = _fixture(name, eps)
    ref = fx["reference"]
    lp = lps(name)
    assert (lp.m, lp.n, lp.nnz) == (fx["m"], fx["n"], fx["nnz"])
    res = run_pdhg(lp, PdhgConfig(), Tolerances(eps_rel=eps))
    assert res.stop == PdhgStopReason.kConverged and ref["stop"] == "converged"
    assert abs(res.iterations - ref["iterations"]) <= 0.05 * ref["iterations"], \
        (res.iterations, ref["iterations"])
    assert abs(res.restarts - ref["restarts"]) <= 1, (res.restarts, ref["restarts"])
    assert res.report.maxresid_rel <= eps
    assert res.report.primal_objective == pytest.approx(ref["report"]["primal_objective"],
                                                        rel=10 * eps)


@pytest.mark.parametrize("name", ["C3", "C4", "C5s"])
def test_full_size_report_matches_independent_kkt(name, lps, oracle):
    lp = lps(name)
    a = run_pdhg(lp, PdhgConfig(max_iterations=300))
    b = run_pdhg(lp, PdhgConfig(max_iterations=300))
    assert np.array_equal(a.iterate.x, b.iterate.x) and np.array_equal(a.iterate.y, b.iterate.y)
    kkt = oracle.relative_report(lp, a.iterate.x, a.iterate.y, a.iterate.z)
    for k in REPORT_KEYS:
        got = getattr(a.report, k)
        assert got == pytest.approx(kkt[k], rel=1e-9, abs=1e-12 * (1 + abs(kkt[k]))), k
    # the device verification entry point (cclp_cu_relative_report) on the same iterate
    with Engine(lp) as eng:
        dev, _ = eng.relative_report(a.iterate.x, a.iterate.y, a.iterate.z)
    for k in REPORT_KEYS:
        assert getattr(dev, k) == pytest.approx(kkt[k], rel=1e-11, abs=1e-12 * (1 + abs(kkt[k]))), k


def test_c4_full_size_sharded_bit_identical(lps):
    lp = lps("C4")
    cfg = PdhgConfig(max_iterations=60)
    one = run_pdhg(lp, cfg)
    with ShardedEngine(lp, 2) as eng:
        sh = eng.solve(cfg)
        assert eng.describe()["halo_x"]
    assert np.array_equal(sh.iterate.x, one.iterate.x)
    assert np.array_equal(sh.iterate.y, one.iterate.y)


def test_cancel_stops_the_loop():
    lp = lpgen.random_equality_lp(5000, 20000, 8, seed=3)[0]
    import ctypes
    flag = (ctypes.c_uint8 * 1)(0)
    threading.Timer(0.3, lambda: flag.__setitem__(0, 1)).start()
    t = time.perf_counter()
    res = run_pdhg(lp, PdhgConfig(max_iterations=10**9), cancel=flag)
    assert res.stop == PdhgStopReason.kCancelled
    assert time.perf_counter() - t < 20
    assert res.iterations > 0


def test_time_limit_stops_the_loop():
    lp = lpgen.random_equality_lp(5000, 20000, 8, seed=3)[0]
    res = run_pdhg(lp, PdhgConfig(max_iterations=10**9, time_limit=0.5))
    assert res.stop == PdhgStopReason.kTimeLimit
    assert res.seconds < 10


@pytest.mark.parametrize("interval", [2, 7])
def test_check_interval_parity(interval, oracle):
    lp = lpgen.small_equality_lp(40, 90, 0.2, 7)[0]
    res = run_pdhg(lp, PdhgConfig(max_iterations=20000, check_interval=interval))
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=20000, check_interval=interval))
    assert res.stop.name == {"converged": "kConverged",
                             "iteration-limit": "kIterationLimit"}[ref["stop"]]
    assert res.iterations == ref["iterations"]
    assert res.iterations % interval == 0
    assert rel(res.iterate.x, ref["x"]) <= 1e-6


def test_iteration_log_format():
    lines = []
    lp = lpgen.small_equality_lp(40, 90, 0.2, 7)[0]
    res = run_pdhg(lp, PdhgConfig(max_iterations=500, log_interval=100, log=lines.append))
    # pdhg.cpp:332-340: "%lld\t%.6e\t%.6e\t%.6e\t%.3f\n" every log_interval checks
    pat = re.compile(r"^(\d+)\t(\S+e[+-]\d\d)\t(\S+e[+-]\d\d)\t(\S+e[+-]\d\d)\t\d+\.\d{3}\n$")
    its = [int(pat.match(ln).group(1)) for ln in lines]
    assert its == [k for k in range(0, res.iterations + 1, 100)]  # check(0) included, as upstream


def test_in_graph_phase_profile_splits_the_iteration():
    """cclp_cu_phase_profile: the four phases measured inside the graphs add
    up to the event-timed iteration (bench.py's kernel split)."""
    lp = lpgen.random_equality_lp(20000, 100000, 10, seed=2)[0]
    with Engine(lp) as eng:
        eng.begin(PdhgConfig())
        eng.advance(256)
        ms = eng.advance(512)
        ph = eng.phase_profile()
    assert ph["steps"] >= 64
    parts = [ph[k] for k in ("spmv_rows", "dual", "spmv_cols", "primal")]
    assert all(v > 0 for v in parts), ph
    per_iter_us = ms * 1e3 / 512
    assert 0.6 * per_iter_us <= sum(parts) <= 1.4 * per_iter_us, (sum(parts), per_iter_us)
