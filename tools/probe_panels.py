"""C5 column-panel size sweep (dev probe): us/iteration for several panel
byte budgets (CCLP_CU_PANEL_BYTES), one generated LP."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
t = time.time()
lp = lpgen.make_config(cfg)
print("gen", cfg, lp.m, lp.n, lp.nnz, f"{time.time() - t:.1f}s", flush=True)
for mb in [int(a) for a in sys.argv[2:]] or [32, 48, 64, 80]:
    os.environ["CCLP_CU_DEV_KNOBS"] = "1"
    os.environ["CCLP_CU_PANEL_BYTES"] = str(mb << 20)
    eng = Engine(lp)
    eng.begin(PdhgConfig())
    eng.advance(3)
    ms = eng.advance(10)
    d = eng.describe()
    print(f"panel {mb} MB: {ms / 10 * 1e3:.1f} us/iteration, grid_r {d.get('spmv_rows_grid_x10_rpg')}", flush=True)
    eng.close()
