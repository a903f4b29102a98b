import sys
sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig
for name, reps in (("C2", 6), ("C3", 3)):
    lp = lpgen.make_config(name)
    for r in range(reps):
        with Engine(lp) as eng:
            eng.begin(PdhgConfig())
            eng.advance(300)
            ms = eng.advance(300)
            d = eng.describe()
            ph = eng.phase_profile()
            print(name, r, "block", d["sell_rows_block"], "us/it %.2f" % (ms / 300 * 1e3), "rows %.2f" % ph["spmv_rows"], flush=True)
