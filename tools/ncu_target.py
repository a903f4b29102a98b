"""Minimal driver for ncu: engine setup on a config, then N eagerly launched
iterations (k_spmv_rows, k_dual, k_spmv_cols, k_primal per iteration)."""
import sys

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
eng = Engine(lpgen.make_config(cfg))
eng.begin(PdhgConfig())
eng.profile_kernels(iters)
eng.close()
