"""Standard-form construction for the race: the reference's triplet rebuild
(to_standard_form, standard_form.cpp:23-104) vs the O(nnz) append
(integration/standard_form_direct.cpp), on a general-form LP of the given size
(half the rows inequalities). CPU only."""
import sys

import numpy as np

sys.path.insert(0, ".")
from integration import race  # noqa: E402
from paper_2510_24429_b200.lp import INF, LinearProgram  # noqa: E402

m, n, k = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (200_000, 1_000_000, 10)))
rng = np.random.default_rng(0)
rows = np.sort(rng.integers(0, m, (n, k)), axis=1)
keep = np.concatenate([np.ones((n, 1), bool), rows[:, 1:] != rows[:, :-1]], axis=1)
cnt = keep.sum(1)
colptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
rowind = rows[keep].astype(np.int32)
val = rng.uniform(0.5, 2.0, rowind.size)
b = rng.uniform(-1, 1, m)
ru = np.where(np.arange(m) % 2 == 0, b, b + 1.0)
lp = LinearProgram(m, n, colptr, rowind, val, rng.normal(size=n), b, ru, np.zeros(n), np.full(n, INF))
ok, why, (t_ref, t_dir) = race.standard_form_check(lp, timings=True)
print(f"m={m} n={n} nnz={rowind.size}: equal={ok} {why} reference {t_ref:.3f} s, direct {t_dir:.3f} s "
      f"({t_ref / t_dir:.1f}x)")
