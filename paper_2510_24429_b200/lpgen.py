"""Seeded synthetic LP generators for the benchmark configurations.

BASELINE.json `configs` / SURVEY.md §8(d):
  C1 transportation 200 x 500       (m=700, n=100,700 with slacks, nnz=200,700)
  C2 random equality LP             (m=100k, n=500k, nnz=5M)
  C3 multicommodity flow            (~2M vars, ~20M nnz)
  C4 staircase / block-angular      (~10M vars, ~100M nnz)
  C5 power-law row lengths          (~50M vars, ~500M nnz)

C2 and C5 follow the known-optimum construction of the reference's test
generator `generate_equality_lp` (proj/tests/test_util.hpp:71-112): a
complementary triple (x*, y*, z*) with x* > 0 on an m-column support, z* > 0
off it, c = A'y* + z*, b = A x*, so c'x* is the optimal value. All
generators are O(nnz) numpy; every output is an equality-form LP as
`to_standard_form` (standard_form.cpp:23-104) would produce it.
"""
from __future__ import annotations

import numpy as np

from .lp import INF, LinearProgram, csc_from_triplets, to_standard_form


def two_var_lp() -> LinearProgram:
    """test_util.hpp:20-34: min x1 + 2 x2 s.t. x1 + x2 = 2, x >= 0."""
    return LinearProgram(1, 2, np.array([0, 1, 2], np.int32), np.array([0, 0], np.int32),
                         np.array([1.0, 1.0]), np.array([1.0, 2.0]), np.array([2.0]),
                         np.array([2.0]), np.zeros(2), np.full(2, INF), name="TWOVAR")


def _distinct_rows(rng, m: int, n: int, k: int) -> np.ndarray:
    """k distinct row indices per column, sorted; shape (n, k)."""
    rows = rng.integers(0, m, size=(n, k), dtype=np.int64)
    rows.sort(axis=1)
    while True:
        dup = np.any(rows[:, 1:] == rows[:, :-1], axis=1)
        if not dup.any():
            return rows
        idx = np.nonzero(dup)[0]
        fresh = rng.integers(0, m, size=(idx.size, k), dtype=np.int64)
        fresh.sort(axis=1)
        rows[idx] = fresh


def _nonzero_uniform(rng, size, lo=-2.0, hi=2.0):
    v = rng.uniform(lo, hi, size=size)
    v[v == 0.0] = 1.0
    return v


def _known_optimum(A_colptr, A_rowind, A_val, m, n, support, rng, name):
    """c = A'y* + z*, b = A x* (test_util.hpp:90-111)."""
    import scipy.sparse as sp

    A = sp.csc_matrix((A_val, A_rowind, A_colptr), shape=(m, n))
    x_star = np.zeros(n)
    z_star = np.zeros(n)
    on = np.zeros(n, dtype=bool)
    on[support] = True
    x_star[on] = rng.uniform(0.5, 2.0, size=int(on.sum()))
    z_star[~on] = rng.uniform(0.5, 2.0, size=int((~on).sum()))
    y_star = rng.uniform(-1.0, 1.0, size=m)
    c = A.T @ y_star + z_star
    b = A @ x_star
    lp = LinearProgram(m, n, A_colptr.astype(np.int32), A_rowind.astype(np.int32),
                       A_val.astype(np.float64), c, b.copy(), b.copy(), np.zeros(n),
                       np.full(n, INF), name=name)
    return lp, x_star, y_star, z_star


def random_equality_lp(m: int = 100_000, n: int = 500_000, nnz_per_col: int = 10,
                       seed: int = 2):
    """C2: random sparse equality LP with a unique optimum by construction.

    Each column gets `nnz_per_col` distinct rows with values U(-2,2); the m
    support columns (a seeded permutation, as in test_util.hpp:84-87) carry a
    band-diagonal entry of magnitude U(2,3) at their own row so that the basis
    B is nonsingular. Returns (lp, x*, y*, z*)."""
    rng = np.random.default_rng(seed)
    k = nnz_per_col
    perm = rng.permutation(n)
    support = perm[:m]
    rows = _distinct_rows(rng, m, n, k)
    vals = _nonzero_uniform(rng, (n, k))
    # band diagonal for the support: support column perm[i] holds row i. A
    # column lacking its diagonal row gets it in place of its first entry,
    # which keeps the rows distinct.
    diag_rows = np.arange(m)
    sc = support
    r_sc = rows[sc]
    has = np.any(r_sc == diag_rows[:, None], axis=1)
    r_sc[~has, 0] = diag_rows[~has]
    r_sc.sort(axis=1)
    rows[sc] = r_sc
    is_diag = np.zeros((n, k), dtype=bool)
    is_diag[sc] = rows[sc] == diag_rows[:, None]
    mag = rng.uniform(2.0, 3.0, size=(n, k))
    sign = np.where(rng.random((n, k)) < 0.5, -1.0, 1.0)
    vals = np.where(is_diag, sign * mag, vals)
    colptr = np.arange(0, n * k + 1, k, dtype=np.int64)
    return _known_optimum(colptr, rows.reshape(-1), vals.reshape(-1), m, n, support, rng,
                          f"random_{m}x{n}")


def small_equality_lp(m: int, n: int, density: float = 0.5, seed: int = 0):
    """Small instance in the style of test_util.hpp:71-112 (random_sparse with
    a j % m diagonal band so no column is empty)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < density
    r, cidx = np.nonzero(mask)
    v = _nonzero_uniform(rng, r.size)
    rows = np.concatenate([np.arange(n) % m, r])
    cols = np.concatenate([np.arange(n), cidx])
    vals = np.concatenate([np.ones(n), v])
    colptr, rowind, val = csc_from_triplets(m, n, rows, cols, vals)
    perm = rng.permutation(n)
    return _known_optimum(colptr.astype(np.int64), rowind, val, m, n, perm[:m], rng,
                          f"small_{m}x{n}")


def transportation_lp(sources: int = 200, sinks: int = 500, seed: int = 1) -> LinearProgram:
    """C1: supply rows sum_j x_ij <= s_i, demand rows sum_i x_ij >= d_j,
    x >= 0, costs U(1,100); s_i ~ U(50,150), d_j ~ U(10,50) rescaled to
    sum d = 0.9 sum s. Returned in standard form (one slack per row)."""
    rng = np.random.default_rng(seed)
    S, D = sources, sinks
    s = rng.uniform(50.0, 150.0, size=S)
    d = rng.uniform(10.0, 50.0, size=D)
    d *= 0.9 * s.sum() / d.sum()
    cost = rng.uniform(1.0, 100.0, size=S * D)
    n = S * D
    m = S + D
    # column (i, j) = i*D + j has rows i and S + j (ascending)
    rowind = np.empty(2 * n, dtype=np.int32)
    rowind[0::2] = np.repeat(np.arange(S), D)
    rowind[1::2] = S + np.tile(np.arange(D), S)
    colptr = np.arange(0, 2 * n + 1, 2, dtype=np.int32)
    rl = np.concatenate([np.full(S, -INF), d])
    ru = np.concatenate([s, np.full(D, INF)])
    gen = LinearProgram(m, n, colptr, rowind, np.ones(2 * n), cost, rl, ru, np.zeros(n),
                        np.full(n, INF), name=f"transport_{S}x{D}")
    return to_standard_form(gen)


CONFIGS = {
    "C1": dict(kind="transportation", sources=200, sinks=500, seed=1),
    "C2": dict(kind="random", m=100_000, n=500_000, nnz_per_col=10, seed=2),
}


def make_config(name: str) -> LinearProgram:
    spec = dict(CONFIGS[name])
    kind = spec.pop("kind")
    if kind == "transportation":
        return transportation_lp(**spec)
    if kind == "random":
        return random_equality_lp(**spec)[0]
    raise KeyError(name)
