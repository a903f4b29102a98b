"""A/B of two builds of the engine library on the device loop (one process
per library, alternating): us per iteration and the in-graph phase split.

    python tools/probe_libs.py a.so b.so C2 [C3 ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys
sys.path.insert(0, sys.argv[1])
from paper_2510_24429_b200 import pdhg, lpgen
pdhg.load_library(sys.argv[2])
lp = lpgen.make_config(sys.argv[3])
its = max(200, int(4e11 / (24 * lp.nnz)) // 10)
with pdhg.Engine(lp) as eng:
    eng.begin(pdhg.PdhgConfig())
    eng.advance(200)
    best = min(eng.advance(its) / its for _ in range(3))
    ph = eng.phase_profile()
print(f"{sys.argv[3]} {sys.argv[2].split('/')[-1]}: {best * 1e3:.2f} us/it " +
      " ".join(f"{k}={v:.2f}" for k, v in ph.items() if k != "steps"), flush=True)
"""
libs, cfgs = sys.argv[1:3], sys.argv[3:] or ["C2"]
for cfg in cfgs:
    for rep in range(2):
        for lib in libs:
            subprocess.run([sys.executable, "-c", CHILD, ROOT, os.path.abspath(lib), cfg], check=True)
