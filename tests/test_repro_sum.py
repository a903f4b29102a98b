"""The setup's partition-independent sums (repro_consts / k_repro_sum,
csrc/setup_kernels.cuh), restated in numpy: the same IEEE operations, so the
properties checked here -- every level sum exact, hence the result identical
for any split into blocks / shards and any summation order, and accurate to
well below one ulp of the plain sum -- are the ones the sharded setup relies
on to stay bit-identical to one device."""
import math

import numpy as np
import pytest


def consts(M, N):
    if not (M > 0.0) or not (M <= 1.7e308) or N <= 0:
        return None
    k = 1
    while (1 << k) <= N:
        k += 1
    _, e = math.frexp(M)
    E1 = e + k
    E2 = E1 - 53 + k
    E3 = E2 - 53 + k
    if E1 > 1020 or E3 < -1000:
        return None
    return [math.ldexp(1.5, E1), math.ldexp(1.5, E2), math.ldexp(1.5, E3)]


def level_sums(v, T, order):
    """Exact level sums of the terms v, accumulated in `order` (a permutation)."""
    S = [0.0, 0.0, 0.0]
    rem = v.copy()
    for lv in range(3):
        x = (T[lv] + rem) - T[lv]
        rem = rem - x
        acc = 0.0
        for i in order:
            acc += float(x[i])
        S[lv] = acc
    return S


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_any_split_and_order_gives_the_same_double(seed):
    rng = np.random.default_rng(seed)
    n = 4000
    v = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))
    terms = v * v if seed == 0 else v * rng.standard_normal(n)
    M = float(np.max(np.abs(terms)))
    T = consts(M, n)
    whole = level_sums(terms, T, range(n))
    ref = (whole[0] + whole[1]) + whole[2]
    for trial in range(5):
        cuts = np.sort(rng.choice(np.arange(1, n), size=rng.integers(1, 8), replace=False))
        parts = np.split(np.arange(n), cuts)
        S = [0.0, 0.0, 0.0]
        for p in parts[::-1]:  # shards combined in any order
            ps = level_sums(terms, T, rng.permutation(p))
            S = [a + b for a, b in zip(S, ps)]
        assert (S[0] + S[1]) + S[2] == ref
    exact = math.fsum(terms.tolist())
    assert abs(ref - exact) <= 1e-15 * max(abs(exact), 1e-300) + 1e-300 or ref == exact
