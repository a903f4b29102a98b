"""Crossover scalability on the B200 box.

For LPs past C1's size, one B200 PDHG solve to `eps` on the standard form,
then from that iterate:
  * the scalable crossover (integration/crossover_scalable.cpp) with pricing
    on the B200 (cclp_cu_price) and with host pricing;
  * the reference's run_crossover (dense etas, crossover.cpp:101-150,
    factorization.cpp:110-139) in a subprocess under a time limit (skipped
    above --ref-max-m rows: its crash holds m dense etas of length m);
and the full race end to end (GPU PDHG + concurrent scalable crossover).
One JSON line per (LP, arm) on stdout.

    python tools/crossover_scale.py [--eps 1e-4] [--ref-timeout 300]
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from integration import race  # noqa: E402
from paper_2510_24429_b200 import lp as lpm  # noqa: E402
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import PdhgConfig, Tolerances, run_pdhg  # noqa: E402

CASES = {
    "C1": lambda: lpm.to_standard_form(lpgen.transportation_lp(200, 500, seed=1)),
    "T1000x3000": lambda: lpm.to_standard_form(lpgen.transportation_lp(1000, 3000, seed=1)),
    "T2000x5000": lambda: lpm.to_standard_form(lpgen.transportation_lp(2000, 5000, seed=1)),
    "MCF2000x4": lambda: lpgen.multicommodity_lp(nodes=2000, arcs_per_node=6, commodities=4, side_rows=2000,
                                                 side_per_var=2, seed=3),
    "C2": lambda: lpgen.make_config("C2"),
    "MCF10000x8": lambda: lpgen.multicommodity_lp(nodes=10000, arcs_per_node=8, commodities=8, side_rows=8000,
                                                  side_per_var=3, seed=3),
}

REF_CHILD = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from integration import race
from paper_2510_24429_b200.lp import LinearProgram
d = np.load(sys.argv[2])
lp = LinearProgram(int(d["m"]), int(d["n"]), d["colptr"], d["rowind"], d["val"], d["c"], d["b"], d["b"],
                   d["l"], d["u"])
o = race.crossover(lp, d["x"], d["y"], d["z"], float(d["thr"]), crossover="reference", kind="cpu")
print(json.dumps(o))
"""


def emit(**kw):
    kw.pop("basic", None)
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eps", type=float, default=1e-4)
    ap.add_argument("--cases", default=",".join(c for c in CASES if c != "C2"))
    ap.add_argument("--ref-timeout", type=float, default=300.0)
    ap.add_argument("--ref-max-m", type=int, default=12000)
    ap.add_argument("--no-race", action="store_true")
    args = ap.parse_args()
    for name in args.cases.split(","):
        std = CASES[name]()
        t = time.perf_counter()
        res = run_pdhg(std, PdhgConfig(max_iterations=2_000_000, time_limit=300.0), Tolerances(eps_rel=args.eps))
        pdhg_s = time.perf_counter() - t
        emit(case=name, arm="pdhg_b200", m=std.m, n=std.n, nnz=std.nnz, eps=args.eps, seconds=pdhg_s,
             iterations=res.iterations, stop=res.stop.name, maxresid=res.report.maxresid_rel)
        x, y, z = res.iterate.x, res.iterate.y, res.iterate.z
        thr = res.report.maxresid_rel
        basics = {}
        for arm in ("scalable-device", "scalable"):
            o = race.crossover(std, x, y, z, thr, crossover=arm, kind="gpu")
            basics[arm] = o["basic"]
            emit(case=name, arm=f"crossover_{arm}", m=std.m, **o)
        if std.m <= args.ref_max_m:
            with tempfile.TemporaryDirectory() as td:
                f = os.path.join(td, "snap.npz")
                np.savez(f, m=std.m, n=std.n, colptr=std.colptr, rowind=std.rowind, val=std.val, c=std.c,
                         b=std.row_lower, l=std.col_lower, u=std.col_upper, x=x, y=y, z=z, thr=thr)
                t = time.perf_counter()
                try:
                    p = subprocess.run([sys.executable, "-c", REF_CHILD, ROOT, f], capture_output=True, text=True,
                                       timeout=args.ref_timeout)
                    o = json.loads(p.stdout.strip().splitlines()[-1])
                    same = o["basic"] == basics["scalable-device"]
                    emit(case=name, arm="crossover_reference", m=std.m, same_basis_as_scalable=same, **o)
                except subprocess.TimeoutExpired:
                    emit(case=name, arm="crossover_reference", m=std.m, status="DNF",
                         seconds=time.perf_counter() - t, note=f"killed at {args.ref_timeout:.0f} s")
        else:
            emit(case=name, arm="crossover_reference", m=std.m, status="not run",
                 note=f"dense etas: m^2 doubles = {8 * std.m ** 2 / 1e9:.1f} GB and O(m^3) crash")
        if not args.no_race:
            t = time.perf_counter()
            out = race.run_race(std, kind="gpu", mode="concurrent", eps_rel=1e-6, time_limit=600.0,
                                crossover="scalable-device")
            emit(case=name, arm="race_b200_concurrent", m=std.m, wall_s=time.perf_counter() - t,
                 status=out.get("status"), winner=out.get("winner"), objective=out.get("objective"),
                 device_prices=race.pricing_counts("gpu")[0])


if __name__ == "__main__":
    main()
