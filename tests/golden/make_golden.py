"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, the
reference's own sources compiled against the Eigen-API shim).

Run in the build container (needs /root/reference at build time):
    make -C oracle ref && python tests/golden/make_golden.py

Each fixture holds a small LP (CSC + bounds) and the reference's outputs on
it: matvec / matvec_transpose of a seeded vector, Ruiz factors, the norm
estimate, and run_pdhg results (x, y, z, report, stop, iterations, restarts,
snapshots) at several iteration budgets. tests/test_oracle.py pins the C
restatement to these bit for bit; tests/test_gpu_parity.py checks the GPU
engine against them within the north-star tolerance.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import REPORT_FIELDS, STOP_NAMES, Reference  # noqa: E402
from paper_2510_24429_b200 import lpgen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
BUDGETS = [0, 1, 10, 100, 1000, 20000]


def cases():
    yield "twovar", lpgen.two_var_lp(), [1e-2, 1e-3]
    for seed in range(3):
        yield f"eq6x12_s{seed}", lpgen.small_equality_lp(6, 12, 0.5, seed)[0], [1e-2, 1e-4]
    yield "eq40x90", lpgen.small_equality_lp(40, 90, 0.2, 7)[0], [1e-2, 1e-4]
    yield "transport8x12", lpgen.transportation_lp(8, 12, seed=11), [1e-2, 1e-4]
    ub = lpgen.small_equality_lp(10, 25, 0.4, 3)[0]
    ub.col_upper = np.where(np.arange(ub.n) % 3 == 0, 1.5, ub.col_upper)  # boxed columns
    yield "boxed10x25", ub, [1e-2]
    fr = lpgen.small_equality_lp(8, 16, 0.4, 4)[0]
    fr.col_lower = np.where(np.arange(fr.n) % 5 == 1, -np.inf, fr.col_lower)  # free columns
    yield "free8x16", fr, [1e-2]


def main():
    R = Reference()
    for name, lp, thr in cases():
        rng = np.random.default_rng(123)
        x = rng.standard_normal(lp.n)
        y = rng.standard_normal(lp.m)
        out = dict(m=lp.m, n=lp.n, colptr=lp.colptr, rowind=lp.rowind, val=lp.val, c=lp.c,
                   row_lower=lp.row_lower, row_upper=lp.row_upper, col_lower=lp.col_lower,
                   col_upper=lp.col_upper, mv_x=x, mv_y=y, ax=R.matvec(lp, x),
                   aty=R.matvec_transpose(lp, y), norm100=R.estimate_norm(lp, 100, 0),
                   thresholds=np.array(thr), budgets=np.array(BUDGETS))
        r, s, sv = R.ruiz(lp, 10)
        out.update(ruiz_r=r, ruiz_s=s, ruiz_val=sv)
        for it in BUDGETS:
            res = R.run_pdhg(lp, config=dict(max_iterations=it), thresholds=thr)
            out[f"it{it}_x"] = res["x"]
            out[f"it{it}_y"] = res["y"]
            out[f"it{it}_z"] = res["z"]
            out[f"it{it}_report"] = np.array([res["report"][f] for f in REPORT_FIELDS])
            out[f"it{it}_stats"] = np.array([STOP_NAMES.index(res["stop"]), res["iterations"],
                                             res["restarts"], res["error_iteration"]])
            snaps = res["snapshots"]
            out[f"it{it}_snap_meta"] = np.array(
                [[s["threshold"], s["maxresid"], float(s["from_average"]), s["iteration"]]
                 for s in snaps]).reshape(-1, 4)
            for k, s in enumerate(snaps):
                out[f"it{it}_snap{k}_x"] = s["x"]
                out[f"it{it}_snap{k}_y"] = s["y"]
                out[f"it{it}_snap{k}_z"] = s["z"]
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, lp.m, lp.n, lp.nnz, "final", STOP_NAMES[out[f"it{BUDGETS[-1]}_stats"][0]],
              out[f"it{BUDGETS[-1]}_stats"][1])


if __name__ == "__main__":
    main()
