"""GPU: crossover pricing on the device — cclp_cu_price against
a restatement of the reference's price() (simplex.cpp:266-296) whose column
dots come from the reference's own matvec_transpose (kernels.cpp, the same
sequential order as EngineModel::column_dot, basis.cpp:35-42). The pick
(entering column, direction, violation) must be identical: Dantzig and Bland,
phase 1 and 2, skip sets, logical columns."""
import time

import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import Engine

pytestmark = pytest.mark.gpu


def ref_price(lp, d_struct, y, status, skip, phase1, dtol, bland):
    """simplex.cpp:266-296 over the EngineModel's n + m columns."""
    n, m = lp.n, lp.m
    pick = (-1, 0, 0.0)
    for j in range(n + m):
        st = status[j]
        if st in "BX" or (skip is not None and skip[j]):
            continue
        cost = 0.0 if phase1 else (lp.c[j] if j < n else 0.0)
        d = cost - (d_struct[j] if j < n else y[j - n])
        if st == "L" and d < -dtol:
            viol, dr = -d, 1
        elif st == "U" and d > dtol:
            viol, dr = d, -1
        elif st == "Z" and abs(d) > dtol:
            viol, dr = abs(d), (1 if d < 0.0 else -1)
        else:
            continue
        if bland:
            if pick[0] < 0:
                pick = (j, dr, viol)
        elif viol > pick[2]:
            pick = (j, dr, viol)
    return pick


def lps():
    return [("transport", lpgen.transportation_lp(15, 25, seed=2)),
            ("small", lpgen.small_equality_lp(30, 80, 0.2, seed=4)[0]),
            ("random", lpgen.random_equality_lp(500, 2500, 6, seed=3)[0])]


@pytest.mark.parametrize("name,lp", lps())
@pytest.mark.parametrize("phase1", [False, True])
@pytest.mark.parametrize("bland", [False, True])
def test_price_matches_reference(name, lp, phase1, bland, reference):
    rng = np.random.default_rng(7)
    with Engine(lp) as eng:
        for trial in range(4):
            y = rng.normal(size=lp.m)
            if trial == 3:  # ties: duplicate violations across columns
                y = np.round(y)
            status = "".join(rng.choice(list("BLUXZ"), size=lp.n + lp.m, p=[.2, .4, .2, .1, .1]))
            skip = (rng.random(lp.n + lp.m) < 0.1) if trial % 2 else None
            d_struct = reference.matvec_transpose(lp, y)
            want = ref_price(lp, d_struct, y, status, skip, phase1, 1e-9, bland)
            got = eng.price(y, status, skip, phase1=phase1, dtol=1e-9, bland=bland)
            assert got == want, (trial, got, want)


def test_price_none_violating(reference):
    lp = lpgen.transportation_lp(10, 12, seed=1)
    with Engine(lp) as eng:
        assert eng.price(np.zeros(lp.m), "B" * (lp.n + lp.m)) == (-1, 0, 0.0)


def test_price_c2_size_speed(reference):
    """C2-sized pricing (600k columns): the device pick equals the
    restatement's; records both times (device call incl. transfers)."""
    lp = lpgen.make_config("C2")
    rng = np.random.default_rng(3)
    y = rng.normal(size=lp.m)
    status = np.where(rng.random(lp.n + lp.m) < 0.7, ord("L"), ord("B")).astype(np.uint8).tobytes().decode()
    d_struct = reference.matvec_transpose(lp, y)
    t = time.perf_counter()
    dcost = lp.c - d_struct  # vectorised restatement for the large case (same values)
    st = np.frombuffer(status.encode(), np.uint8)[:lp.n]
    viol = np.where((st == ord("L")) & (dcost < -1e-9), -dcost, 0.0)
    j = int(np.argmax(viol)) if viol.max() > 0 else -1
    t_cpu = time.perf_counter() - t
    with Engine(lp) as eng:
        eng.price(y, status)  # warm
        t = time.perf_counter()
        e, dr, v = eng.price(y, status)
        t_gpu = time.perf_counter() - t
    logical = np.frombuffer(status.encode(), np.uint8)[lp.n:]
    lv = np.where((logical == ord("L")) & (y > 1e-9), y, 0.0)  # logical: d = 0 - y
    if lv.max() > viol.max():
        j = lp.n + int(np.argmax(lv))
    assert e == j
    print(f"price C2: device {t_gpu * 1e3:.2f} ms (incl. transfers), numpy restatement {t_cpu * 1e3:.2f} ms")
