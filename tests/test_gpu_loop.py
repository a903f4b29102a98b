"""GPU: the loop's host/device protocol (pdhg.cpp:300-377).

* cancel is polled every iteration (pdhg.cpp:301): a preset flag stops at
  iteration 0 before the first check (no snapshot), and a flag raised
  mid-batch stops inside the batch, on a pass boundary, with the state the
  reference returns (the current iterate, pdhg.cpp:301-305);
* ladder snapshots are taken by the kernels and copied out while the device
  keeps iterating: a slow sink does not stall the loop, the snapshots still
  equal the CPU oracle's, and a sink that raises stops the loop and the
  exception propagates (the reference's synchronous sink would unwind
  run_pdhg the same way).
"""
import ctypes
import threading
import time

import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, PdhgStopReason, Tolerances, run_pdhg

pytestmark = pytest.mark.gpu


def rel(a, b):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    return d / max(np.linalg.norm(b), 1e-300) if d > 0 else 0.0


@pytest.fixture(scope="module")
def mid_lp():
    return lpgen.random_equality_lp(20000, 100000, 10, seed=7)[0]


def test_preset_cancel_stops_before_the_first_check(oracle):
    lp = lpgen.small_equality_lp(40, 90, 0.2, 7)[0]
    flag = (ctypes.c_uint8 * 1)(1)
    snaps = []
    # a threshold that check(0) would cross: the cancel poll comes first
    res = run_pdhg(lp, PdhgConfig(max_iterations=1000), thresholds=[1e9], sink=snaps.append,
                   cancel=flag)
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=1000), thresholds=[1e9], cancel=True)
    assert res.stop == PdhgStopReason.kCancelled and ref["stop"] == "cancelled"
    assert res.iterations == ref["iterations"] == 0
    assert snaps == [] and ref["snapshots"] == []
    assert rel(res.iterate.x, ref["x"]) <= 1e-12
    assert rel(res.iterate.z, ref["z"]) <= 1e-12


def test_cancel_stops_inside_a_batch(mid_lp):
    k = 2048  # iterations per device batch: a host-side poll could only stop on multiples
    flag = (ctypes.c_uint8 * 1)(0)
    threading.Timer(0.4, lambda: flag.__setitem__(0, 1)).start()
    cfg = PdhgConfig(max_iterations=10**8, poll_interval=k)
    t = time.perf_counter()
    res = run_pdhg(mid_lp, cfg, Tolerances(eps_rel=1e-13, eps_cross=1e-2), cancel=flag)
    assert res.stop == PdhgStopReason.kCancelled
    assert time.perf_counter() - t < 30
    assert res.iterations > 0 and res.iterations % k != 0, res.iterations
    # the returned view is the state at that pass boundary: the same iterate
    # as a run limited to that many iterations (unless check(t) restarted,
    # which changes the limit run's returned iterate, pdhg.cpp:359-368)
    lim = run_pdhg(mid_lp, PdhgConfig(max_iterations=res.iterations),
                   Tolerances(eps_rel=1e-13, eps_cross=1e-2))
    assert lim.iterations == res.iterations
    if lim.restarts == res.restarts:
        assert np.array_equal(lim.iterate.x, res.iterate.x)
        assert np.array_equal(lim.iterate.y, res.iterate.y)


def test_slow_sink_does_not_stall_the_device(mid_lp):
    tol = Tolerances(eps_rel=1e-13, eps_cross=1e-1)
    with Engine(mid_lp) as eng:
        cfg = PdhgConfig(max_iterations=40000)
        base = eng.solve(cfg, tol)
        calls = []

        def slow(s):
            calls.append((s.iteration, time.perf_counter()))
            time.sleep(0.4)

        res = eng.solve(cfg, tol, thresholds=[1e-1, 1e-2], sink=slow)
    assert len(calls) == 2 and res.iterations == base.iterations
    assert np.array_equal(res.iterate.x, base.iterate.x)  # snapshots never perturb the iterates
    # device loop time unchanged by the 0.8 s the sink slept (a halting loop
    # would add it); allow 10 % + 20 ms of noise
    assert res.loop_seconds < base.loop_seconds * 1.10 + 0.02, (res.loop_seconds, base.loop_seconds)


def test_snapshots_match_the_oracle_with_inline_extraction(oracle):
    lp = lpgen.small_equality_lp(40, 90, 0.2, 7)[0]
    thr = [1e-1, 1e-2, 1e-3, 1e-4, 1e-5]
    snaps = []
    res = run_pdhg(lp, PdhgConfig(max_iterations=20000), thresholds=thr, sink=snaps.append)
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=20000), thresholds=thr)
    assert res.iterations == ref["iterations"]
    assert [s.iteration for s in snaps] == [s["iteration"] for s in ref["snapshots"]]
    for a, b in zip(snaps, ref["snapshots"]):
        assert a.threshold == b["threshold"] and a.from_average == b["from_average"]
        assert a.maxresid == pytest.approx(b["maxresid"], rel=1e-6)
        for u, v in ((a.iterate.x, b["x"]), (a.iterate.y, b["y"]), (a.iterate.z, b["z"])):
            assert rel(u, v) <= 1e-6


def test_snapshot_at_the_last_iteration_is_delivered(oracle):
    # a threshold crossed at the final check (iteration limit): no step follows
    # to extract it on the device, the host does
    lp = lpgen.small_equality_lp(40, 90, 0.2, 7)[0]
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=20000), thresholds=[1e-3])
    t = ref["snapshots"][0]["iteration"]
    snaps = []
    res = run_pdhg(lp, PdhgConfig(max_iterations=t), thresholds=[1e-3], sink=snaps.append)
    assert res.iterations == t and [s.iteration for s in snaps] == [t]
    assert rel(snaps[0].iterate.x, ref["snapshots"][0]["x"]) <= 1e-6


def test_sink_exception_stops_the_loop_and_propagates(mid_lp):
    class Boom(RuntimeError):
        pass

    def sink(_s):
        raise Boom("sink failed")

    t = time.perf_counter()
    with pytest.raises(Boom):
        run_pdhg(mid_lp, PdhgConfig(max_iterations=10**8, poll_interval=256),
                 Tolerances(eps_rel=1e-13, eps_cross=1e-1), thresholds=[1e-1], sink=sink)
    assert time.perf_counter() - t < 30  # 1e8 iterations would take hours
