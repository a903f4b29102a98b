"""compute-sanitizer target (dev): small solves through every kernel path
added late in round 1 — SELL-32 columns, SELL-G rows (forced), long rows and
columns, sharded, relative_report, .cscb ingest."""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.lp import write_cscb  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, run_pdhg, run_pdhg_sharded  # noqa: E402
from test_gpu_longrows import dense_rows_lp  # noqa: E402
from test_gpu_sell import dense_cols_lp  # noqa: E402

os.environ["CCLP_CU_DEV_KNOBS"] = "1"
os.environ["CCLP_CU_SELL"] = "1"
os.environ["CCLP_CU_SELL_ROWS"] = "2"
lps = [lpgen.small_equality_lp(40, 90, 0.2, 7)[0], lpgen.random_equality_lp(2000, 10000, 8, seed=9)[0],
       dense_rows_lp(), dense_cols_lp()]
for lp in lps:
    r = run_pdhg(lp, PdhgConfig(max_iterations=100))
    s = run_pdhg_sharded(lp, 2, PdhgConfig(max_iterations=100))
    assert np.array_equal(r.iterate.x, s.iterate.x)
    with Engine(lp) as e:
        rep, av = e.relative_report(r.iterate.x, r.iterate.y, r.iterate.z)
    d = tempfile.mkdtemp()
    p = os.path.join(d, "a.cscb")
    write_cscb(lp, p)
    with Engine.from_file(p) as e:
        f = e.solve(PdhgConfig(max_iterations=100))
    assert np.array_equal(f.iterate.x, r.iterate.x)
# round 2: the speculative row product (three ax slots) with a ladder and restarts
with Engine(lpgen.random_equality_lp(2000, 10000, 8, seed=9)[0]) as e:
    snaps = []
    from paper_2510_24429_b200.pdhg import Tolerances  # noqa: E402
    e.solve(PdhgConfig(max_iterations=1500), Tolerances(), thresholds=[1e-1, 1e-2], sink=snaps.append)
print("sanitize smoke ok")
