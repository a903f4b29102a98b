"""Time to a relative tolerance on a config (the BASELINE metric's
time-to-1e-4): one end-to-end solve through run_pdhg from pinned host
buffers, with a time limit. One JSON line per (config, eps).

    python tools/time_to_tol.py C3 1e-4 150
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import PdhgConfig, Tolerances, run_pdhg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
limit = float(sys.argv[3]) if len(sys.argv) > 3 else 150.0
lp, _keep = bench.pinned_copy(lpgen.make_config(cfg))
run_pdhg(lp, PdhgConfig(max_iterations=10))  # warm (module, pool)
t = time.perf_counter()
res = run_pdhg(lp, PdhgConfig(max_iterations=10_000_000, time_limit=limit), Tolerances(eps_rel=eps))
wall = time.perf_counter() - t
print(json.dumps({"config": cfg, "m": lp.m, "n": lp.n, "nnz": lp.nnz, "eps_rel": eps, "seconds": wall,
                  "iterations": res.iterations, "restarts": res.restarts, "stop": res.stop.name,
                  "maxresid_rel": res.report.maxresid_rel, "time_limit": limit}), flush=True)
