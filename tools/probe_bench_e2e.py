"""Replicates bench.py's e2e leg with per-solve phase timings."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, run_pdhg  # noqa: E402

lp = lpgen.make_config("C2")
torch.cuda.set_device(0)
use_pinned = len(sys.argv) < 2 or sys.argv[1] != "pageable"
plp, keep = bench.pinned_copy(lp) if use_pinned else (lp, None)
run_pdhg(plp, PdhgConfig(max_iterations=10))
for rep in range(3):
    t = time.perf_counter()
    eng = Engine(plp)
    t1 = time.perf_counter()
    res = eng.solve(PdhgConfig(max_iterations=2000))
    t2 = time.perf_counter()
    ph = eng.describe()["phase_seconds"]
    eng.close()
    t3 = time.perf_counter()
    print(f"pinned={use_pinned} create {1e3*(t1-t):.1f} solve {1e3*(t2-t1):.1f} close {1e3*(t3-t2):.1f} ms")
    print("   " + ", ".join(f"{k} {v*1e3:.1f}" for k, v in ph.items()), flush=True)
for rep in range(2):
    t = time.perf_counter()
    r = run_pdhg(plp, PdhgConfig(max_iterations=2000))
    print(f"run_pdhg: {1e3*(time.perf_counter()-t):.1f} ms it={r.iterations}", flush=True)
