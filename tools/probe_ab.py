"""A/B of one development knob (csrc/host_util.cuh dev_knob) on the device loop:
us per iteration (CUDA graph, best of 3) and the in-graph phase split, per
config and knob value. Knobs read at begin() share one engine per config;
`--fresh` builds an engine per value (knobs read at create, e.g. the G).

    python tools/probe_ab.py CCLP_CU_SELLG_PIPE 0,2,4 C2 C3
    python tools/probe_ab.py --fresh CCLP_CU_G_ROWS 4,2 C4
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CCLP_CU_DEV_KNOBS"] = "1"
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig  # noqa: E402

args = sys.argv[1:]
fresh = "--fresh" in args
args = [a for a in args if a != "--fresh"]
knob, values = args[0], args[1].split(",")


def run(eng, name, v, rep, B, its):
    eng.begin(PdhgConfig())
    eng.advance(200)
    best = min(eng.advance(its) / its for _ in range(3))
    ph = eng.phase_profile()
    print(f"{name} {knob}={v} pass {rep}: {best * 1e3:8.2f} us/it  B_iter frac "
          f"{B / (best * 1e-3) / 1e9 / 6471.4:.3f}  "
          + " ".join(f"{k}={x:.2f}" for k, x in ph.items() if k != "steps"), flush=True)


for name in args[2:] or ["C2"]:
    lp = lpgen.make_config(name)
    B = 24 * lp.nnz + 20 * (lp.m + lp.n) + 8
    its = max(200, int(4e11 / (24 * lp.nnz)) // 10)
    if fresh:
        for rep in range(2):
            for v in values:
                os.environ[knob] = v
                with Engine(lp) as eng:
                    run(eng, name, v, rep, B, its)
    else:
        with Engine(lp) as eng:
            for rep in range(2):  # two passes over the values, alternating
                for v in values:
                    os.environ[knob] = v
                    run(eng, name, v, rep, B, its)
