"""Phase breakdown of an end-to-end solve (create -> solve -> download)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
lp = lpgen.make_config(cfgname)
if "--pinned" in sys.argv:  # the bench's e2e input: the LP in pinned host buffers
    import bench
    lp, _keep = bench.pinned_copy(lp)
for rep in range(3):
    t = time.perf_counter()
    eng = Engine(lp)
    t_create = time.perf_counter() - t
    t = time.perf_counter()
    res = eng.solve(PdhgConfig(max_iterations=iters))
    t_solve = time.perf_counter() - t
    ph = eng.describe()["phase_seconds"]
    t = time.perf_counter()
    eng.close()
    t_close = time.perf_counter() - t
    print(f"rep {rep}: create {t_create*1e3:.1f} ms, solve {t_solve*1e3:.1f} ms, close {t_close*1e3:.1f} ms, "
          f"iters {res.iterations}, loop {res.loop_seconds*1e3:.1f} ms", flush=True)
    print("   " + ", ".join(f"{k} {v*1e3:.1f}" for k, v in ph.items()), flush=True)
