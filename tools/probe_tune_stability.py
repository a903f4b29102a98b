"""Stability of the timing-based layout and geometry choices: fresh engines on
a config, the chosen SELL block shapes / grids and the in-graph phase split.

    python tools/probe_tune_stability.py C2:6 C3:3 C4:2
"""
import sys
sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig
for name, reps in ((a.split(":")[0], int(a.split(":")[1])) for a in (sys.argv[1:] or ["C2:6", "C3:3"])):
    lp = lpgen.make_config(name)
    for r in range(reps):
        with Engine(lp) as eng:
            eng.begin(PdhgConfig())
            eng.advance(300)
            ms = eng.advance(300)
            d = eng.describe()
            ph = eng.phase_profile()
            print(name, r, "rows block", d["sell_rows_block"], "cols block", d["sell_cols_block"],
                  "grids", d["spmv_rows_grid_x10_rpg"], d["spmv_cols_grid_x10_rpg"],
                  "us/it %.2f" % (ms / 300 * 1e3),
                  " ".join(f"{k} {v:.2f}" for k, v in ph.items() if k != "steps"), flush=True)
