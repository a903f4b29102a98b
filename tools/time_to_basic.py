"""Time to a verified basic solution (BASELINE metric): the
race (PDHG + concurrent crossover, integration/run_race.cpp) with the B200
run_pdhg versus the same race with the reference's CPU run_pdhg, on C1
(transportation 200 x 500) by default. Prints one JSON line per arm."""
import json
import sys
import time

sys.path.insert(0, ".")
from integration import race  # noqa: E402
from paper_2510_24429_b200 import lpgen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
arms = sys.argv[2].split(",") if len(sys.argv) > 2 else ["gpu", "cpu"]
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["concurrent", "baseline"]
limit = float(sys.argv[4]) if len(sys.argv) > 4 else 900.0
lp = lpgen.make_config(cfg)
if "gpu" in arms:  # warm the engine (module load, context, pool)
    race.run_race(lpgen.two_var_lp(), kind="gpu")
for kind in arms:
    for mode in modes:
        t = time.perf_counter()
        out = race.run_race(lp, kind=kind, mode=mode, time_limit=limit)
        wall = time.perf_counter() - t
        print(json.dumps({"config": cfg, "pdhg": kind, "mode": mode, "wall_s": wall,
                          "status": out["status"], "winner": out["winner"],
                          "objective": out["objective"], "pdhg_stop": out["pdhg_stop"],
                          "pdhg_iterations": out["pdhg_iterations"], "race_wall_s": out["wall_s"],
                          "workers": out["workers"], "n_basic": len(out["basic"]),
                          "basic_hash": hash(tuple(out["basic"]))}), flush=True)
