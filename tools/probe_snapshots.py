"""Snapshot copy-out cost (north_star (3), pdhg.cpp:346-358): the same solve
with and without the tolerance ladder, loop seconds and iterations/s of each,
and the iterations at which the snapshots were taken. With the ladder the
kernels extract each snapshot into a device slot and a side stream copies it
to pinned memory while the loop runs on, so the two rates should agree.

    python tools/probe_snapshots.py [C2 C3 ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, Tolerances  # noqa: E402

LADDER = [1e-2, 1e-3, 1e-4, 1e-5]
ITERS = {"C1": 20_000, "C2": 8_000, "C3": 16_000, "C4": 600}

for name in sys.argv[1:] or ["C2", "C3"]:
    lp = lpgen.make_config(name)
    its = ITERS.get(name, 2000)
    cfg = PdhgConfig(max_iterations=its)
    tol = Tolerances(eps_rel=1e-12)  # never converges: the same number of iterations in both runs
    with Engine(lp) as eng:
        # warm: tuning, graphs and the pinned staging sets of the snapshots
        eng.solve(PdhgConfig(max_iterations=50), tol, thresholds=[1e30], sink=lambda s: None)
        out = {}
        # alternating arms, the faster of two runs each
        for arm, thr in (("no_ladder", []), ("ladder", LADDER), ("no_ladder", []), ("ladder", LADDER)):
            snaps = []
            t0 = time.perf_counter()

            def sink(s, t0=t0, snaps=snaps):
                snaps.append((s.iteration, s.threshold, round(time.perf_counter() - t0, 4)))

            res = eng.solve(cfg, tol, thresholds=thr, sink=sink)
            if arm not in out or res.loop_seconds < out[arm]["loop_s"]:
                out[arm] = {"iterations": res.iterations, "loop_s": res.loop_seconds,
                            "iters_per_s": res.iterations / res.loop_seconds, "snapshots": snaps}
        out["rate_ratio_ladder_over_plain"] = out["ladder"]["iters_per_s"] / out["no_ladder"]["iters_per_s"]
        out["snapshot_bytes"] = 8 * (2 * lp.n + lp.m)
        print(json.dumps({"config": name, "m": lp.m, "n": lp.n, "nnz": lp.nnz, **out}), flush=True)
