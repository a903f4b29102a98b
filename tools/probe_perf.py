"""Quick performance probe (not the bench): C2 device loop, per-kernel times,
time-to-tolerance, reference CPU timing."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, Tolerances  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
t = time.time()
lp = lpgen.make_config(cfgname)
print("gen", cfgname, lp.m, lp.n, lp.nnz, f"{time.time()-t:.2f}s", flush=True)
t = time.time()
eng = Engine(lp)
print("create", f"{time.time()-t:.3f}s", eng.describe(), flush=True)
t = time.time()
eng.begin(PdhgConfig())
print("begin", f"{time.time()-t:.3f}s", flush=True)
eng.advance(200)
for it in (1000, 1000):
    ms = eng.advance(it)
    print(f"advance {it}: {ms:.2f} ms -> {it/ms*1e3:.0f} it/s, {ms/it*1e3:.2f} us/it", flush=True)
pk = eng.profile_kernels(200)
print("kernels: " + ", ".join(f"{k} {v*1e3:.2f} us" for k, v in pk.items()), flush=True)
d = eng.describe()
print(f"last cols body (start->finalize) {d['last_cols_body_ns']/1e3:.2f} us, finalize {d['last_finalize_ns']/1e3:.2f} us", flush=True)
nnz, m, n = lp.nnz, lp.m, lp.n
B = 24 * nnz + 20 * (m + n) + 8
print(f"B_iter {B/1e6:.1f} MB; at advance rate: {B/(ms/it*1e-3)/1e9:.0f} GB/s", flush=True)
for eps in ():
    t = time.time()
    res = eng.solve(PdhgConfig(max_iterations=200000), Tolerances(eps_rel=eps))
    print(f"solve eps={eps}: stop={res.stop.name} it={res.iterations} restarts={res.restarts} "
          f"wall={time.time()-t:.3f}s setup={res.setup_seconds:.3f}s loop={res.loop_seconds:.3f}s "
          f"maxresid={res.report.maxresid_rel:.3e} obj={res.report.primal_objective:.10g}", flush=True)
eng.close()
if len(sys.argv) > 2:
    from oracle.pyoracle import Reference
    R = Reference()
    for S in (0, int(sys.argv[2])):
        t = time.time()
        r = R.run_pdhg(lp, config=dict(max_iterations=S))
        print(f"ref max_iter={S}: {time.time()-t:.2f}s stop={r['stop']} it={r['iterations']}", flush=True)
