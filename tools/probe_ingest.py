"""LP ingest: engine creation from in-memory arrays vs from a binary CSC file
(.cscb, page-cache warm after the first read), per config."""
import os
import sys
import tempfile
import time

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402
from paper_2510_24429_b200.lp import write_cscb  # noqa: E402
from paper_2510_24429_b200.pdhg import Engine  # noqa: E402

for cfgname in sys.argv[1:] or ["C2", "C4"]:
    lp = lpgen.make_config(cfgname)
    d = tempfile.mkdtemp()
    p = os.path.join(d, cfgname + ".cscb")
    t = time.perf_counter()
    write_cscb(lp, p)
    t_write = time.perf_counter() - t
    size = os.path.getsize(p)
    Engine(lp).close()  # context/driver warm-up
    for rep in range(3):
        t = time.perf_counter()
        e = Engine(lp)
        t_arr = time.perf_counter() - t
        e.close()
        t = time.perf_counter()
        e = Engine.from_file(p)
        t_file = time.perf_counter() - t
        e.close()
        print(f"{cfgname} rep {rep}: file {size/1e6:.0f} MB (write {t_write:.2f} s); create from arrays "
              f"{t_arr*1e3:.1f} ms, from .cscb {t_file*1e3:.1f} ms ({size/t_file/1e9:.2f} GB/s)", flush=True)
    os.remove(p)
