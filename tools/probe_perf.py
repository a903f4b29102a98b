"""Performance probe (not the bench): device loop rate and per-kernel times
with algorithmic bytes, for one config."""
import sys
import time

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
t = time.time()
lp = lpgen.make_config(cfgname)
m, n, nnz = lp.m, lp.n, lp.nnz
print("gen", cfgname, m, n, nnz, f"{time.time()-t:.2f}s", flush=True)
eng = Engine(lp)
eng.begin(PdhgConfig())
d = eng.describe()
print({k: v for k, v in d.items() if k != "phase_seconds"}, flush=True)
eng.advance(100)
its = max(50, int(2e11 / (24 * nnz)) // 10)
ms = eng.advance(its)
B = 24 * nnz + 20 * (m + n) + 8
print(f"advance {its}: {ms/its*1e3:.2f} us/it, {its/ms*1e3:.0f} it/s, B_iter {B/1e6:.1f} MB "
      f"-> {B/(ms/its*1e-3)/1e9:.0f} GB/s", flush=True)
pk = eng.profile_kernels(50)
kb = dict(spmv_rows=12 * nnz + 4 * (m + 1) + 8 * n + 8 * m,
          spmv_cols=12 * nnz + 4 * (n + 1) + 8 * m + 8 * n,
          dual=8 * m * 10, primal=8 * n * 12)
for k, v in pk.items():
    print(f"  {k:10s} {v*1e3:9.2f} us  {kb[k]/1e6:8.1f} MB  {kb[k]/(v*1e-3)/1e9:7.0f} GB/s", flush=True)
eng.close()
