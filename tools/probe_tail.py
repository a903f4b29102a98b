import sys
sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig
for name in sys.argv[1:]:
    with Engine(lpgen.make_config(name)) as eng:
        eng.begin(PdhgConfig())
        eng.advance(500)
        vals = []
        for _ in range(20):
            eng.advance(7)
            d = eng.describe()
            vals.append((-d["last_cols_body_ns"], d["last_finalize_ns"]))
        vals.sort(key=lambda v: v[1])
        med = vals[len(vals) // 2]
        ph = eng.phase_profile()
        print(name, "reduce+ctrl load ns", med[0], "finalize total ns", med[1], "decide ns", med[1] - med[0], ph)
