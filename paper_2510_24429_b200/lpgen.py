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


def multicommodity_lp(nodes: int = 10_000, arcs_per_node: int = 10, commodities: int = 20,
                      side_rows: int = 100_000, side_per_var: int = 7, seed: int = 3):
    """C3: multicommodity flow on a ring-local random digraph.

    Flow variables x[k, e] >= 0 (commodity-major), conservation rows
    (k, v): out - in = d[k, v] (equality), capacity rows sum_k x[k, e] <= cap_e
    and `side_rows` budget rows sum w x <= B over random (k, e) sets, each flow
    variable in `side_per_var` of them (~10 nnz per flow variable). Arcs join
    v to v + offset with small offsets (plus 5% long-range arcs), so the
    matrix has the locality of a real network. Feasible and bounded by
    construction: demands, capacities and budgets are set from a random
    positive flow x0 with margins; costs are U(1, 10) > 0. Returned in
    standard form (one slack per inequality row)."""
    rng = np.random.default_rng(seed)
    V, K = nodes, commodities
    E = V * arcs_per_node
    tail = np.repeat(np.arange(V), arcs_per_node)
    off = rng.integers(1, 33, size=E) * np.where(rng.random(E) < 0.5, -1, 1)
    far = rng.random(E) < 0.05
    off[far] = rng.integers(1, V, size=int(far.sum()))
    head = (tail + off) % V
    head = np.where(head == tail, (head + 1) % V, head)
    nf = K * E
    # conservation: column (k, e) has +1 at row k*V + tail, -1 at row k*V + head
    kk = np.repeat(np.arange(K), E)
    ee = np.tile(np.arange(E), K)
    r_tail = kk * V + tail[ee]
    r_head = kk * V + head[ee]
    # capacity rows K*V + e
    r_cap = K * V + ee
    # side rows: K*V + E + s
    S = side_rows
    r_side = K * V + E + rng.integers(0, S, size=(nf, side_per_var))
    w_side = rng.uniform(0.5, 2.0, size=(nf, side_per_var))
    rows = np.concatenate([r_tail[:, None], r_head[:, None], r_cap[:, None], r_side], axis=1)
    vals = np.concatenate([np.ones((nf, 1)), -np.ones((nf, 1)), np.ones((nf, 1)), w_side], axis=1)
    order = np.argsort(rows, axis=1, kind="stable")
    rows = np.take_along_axis(rows, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    # merge duplicate side rows within a column (sum, as make_sparse would)
    dup = np.zeros_like(rows, dtype=bool)
    dup[:, 1:] = rows[:, 1:] == rows[:, :-1]
    if dup.any():
        for j in np.nonzero(dup.any(axis=1))[0]:
            r, v = rows[j], vals[j]
            ur, inv = np.unique(r, return_inverse=True)
            sv = np.zeros(ur.size)
            np.add.at(sv, inv, v)
            pad = rows.shape[1] - ur.size
            rows[j] = np.concatenate([ur, np.full(pad, -1)])
            vals[j] = np.concatenate([sv, np.zeros(pad)])
    m = K * V + E + S
    keep = rows >= 0
    counts = keep.sum(axis=1)
    colptr = np.zeros(nf + 1, dtype=np.int64)
    colptr[1:] = np.cumsum(counts)
    rowind = rows[keep].astype(np.int32)
    val = vals[keep]
    import scipy.sparse as sp
    A = sp.csc_matrix((val, rowind, colptr), shape=(m, nf))
    x0 = rng.uniform(0.1, 1.0, size=nf)
    act = A @ x0
    rl = np.empty(m)
    ru = np.empty(m)
    ncons = K * V
    rl[:ncons] = act[:ncons]
    ru[:ncons] = act[:ncons]
    rl[ncons:] = -INF
    ru[ncons:] = act[ncons:] * rng.uniform(1.05, 1.5, size=m - ncons)
    c = rng.uniform(1.0, 10.0, size=nf)
    gen = LinearProgram(m, nf, colptr.astype(np.int32), rowind, val, c, rl, ru, np.zeros(nf),
                        np.full(nf, INF), name=f"mcf_{V}x{K}")
    return to_standard_form(gen)


def staircase_lp(stages: int = 1000, cols_per_stage: int = 10_000, rows_per_stage: int = 5_000,
                 own_per_col: int = 6, next_per_col: int = 4, seed: int = 4):
    """C4: staircase / block-angular LP. Stage t has `cols_per_stage` columns
    and `rows_per_stage` rows; a column of stage t has `own_per_col` entries in
    stage t's rows and `next_per_col` in stage t+1's rows (the last stage links
    to none), values U(-2, 2). Known optimum as in C2 (test_util.hpp:71-112):
    each row's band-diagonal support column carries a U(2,3) entry."""
    rng = np.random.default_rng(seed)
    T, nc, nr = stages, cols_per_stage, rows_per_stage
    n, m = T * nc, T * nr
    stage = np.repeat(np.arange(T), nc)
    k1, k2 = own_per_col, next_per_col
    own = _distinct_rows(rng, nr, n, k1) + (stage * nr)[:, None]
    nxt = _distinct_rows(rng, nr, n, k2) + ((stage + 1) * nr)[:, None]
    last = stage == T - 1
    rows = np.concatenate([own, nxt], axis=1)
    vals = _nonzero_uniform(rng, rows.shape)
    # support: in each stage the first nr columns (after a seeded shuffle) own
    # row (stage*nr + i) as a band diagonal
    perm_in_stage = np.argsort(rng.random((T, nc)), axis=1)
    support_local = perm_in_stage[:, :nr]  # (T, nr)
    support = (support_local + (np.arange(T) * nc)[:, None]).reshape(-1)
    diag_rows = np.arange(m)
    r_sc = rows[support, :k1]
    has = np.any(r_sc == diag_rows[:, None], axis=1)
    r_sc[~has, 0] = diag_rows[~has]
    rows[support, :k1] = r_sc
    is_diag = np.zeros(rows.shape, dtype=bool)
    is_diag[support, :k1] = rows[support, :k1] == diag_rows[:, None]
    vals = np.where(is_diag, np.where(rng.random(rows.shape) < 0.5, -1.0, 1.0) *
                    rng.uniform(2.0, 3.0, size=rows.shape), vals)
    keep = np.ones(rows.shape, dtype=bool)
    keep[last, k1:] = False
    order = np.argsort(np.where(keep, rows, np.iinfo(np.int64).max), axis=1, kind="stable")
    rows = np.take_along_axis(rows, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    keep = np.take_along_axis(keep, order, axis=1)
    counts = keep.sum(axis=1)
    colptr = np.zeros(n + 1, dtype=np.int64)
    colptr[1:] = np.cumsum(counts)
    return _known_optimum(colptr, rows[keep], vals[keep], m, n, support, rng,
                          f"staircase_{T}x{nc}")


def powerlaw_lp(m: int = 10_000_000, n: int = 50_000_000, nnz: int = 500_000_000,
                alpha: float = 1.8, min_len: int = 8, max_len: int | None = None, seed: int = 5):
    """C5: power-law row lengths: row lengths follow a
    truncated Pareto law with exponent `alpha` (P(L >= k) ~ k^(1-alpha), from
    `min_len` up to `max_len`, default n/50), rescaled to `nnz` in total;
    columns uniform (distinct within a row), values U(-2,2). Known optimum as
    in C2 (test_util.hpp:71-112): the m support columns perm[:m] carry a
    band-diagonal U(2,3) entry at their own row. One int64 sort of the keys
    col*m + row gives the CSC directly. Returns (lp, x*, y*, z*)."""
    rng = np.random.default_rng(seed)
    max_len = max_len or max(min_len + 1, n // 50)
    u = rng.random(m)
    L = min_len * u ** (-1.0 / (alpha - 1.0))
    L = np.minimum(L, max_len)
    L = np.maximum(1, np.rint(L * ((nnz - m) / L.sum()))).astype(np.int64)
    L = np.minimum(L, max_len)
    diff = (nnz - m) - int(L.sum())  # exact total: spread the residual over rows
    if diff != 0:
        idx = rng.choice(m, size=abs(diff), replace=abs(diff) > m)
        np.add.at(L, idx, 1 if diff > 0 else -1)
        L = np.maximum(L, 1)
    perm = rng.permutation(n)
    support = perm[:m]
    rows = np.repeat(np.arange(m, dtype=np.int64), L)
    cols = rng.integers(0, n, size=rows.size, dtype=np.int64)
    # key*2 + flag: the diagonal entry (flag 0) sorts first among equal keys
    keys = np.concatenate([(cols * m + rows) * 2 + 1,
                           (support.astype(np.int64) * m + np.arange(m)) * 2])
    del rows, cols
    keys.sort(kind="stable")
    first = np.ones(keys.size, dtype=bool)
    first[1:] = (keys[1:] >> 1) != (keys[:-1] >> 1)
    keys = keys[first]
    is_diag = (keys & 1) == 0
    keys >>= 1
    rowind = (keys % m).astype(np.int32)
    col_of = keys // m
    del keys
    colptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(col_of, minlength=n), out=colptr[1:])
    del col_of
    vals = _nonzero_uniform(rng, rowind.size)
    nd = int(is_diag.sum())
    vals[is_diag] = np.where(rng.random(nd) < 0.5, -1.0, 1.0) * rng.uniform(2.0, 3.0, size=nd)
    return _known_optimum(colptr, rowind, vals, m, n, support, rng, f"powerlaw_{m}x{n}")


CONFIGS = {
    "C1": dict(kind="transportation", sources=200, sinks=500, seed=1),
    "C2": dict(kind="random", m=100_000, n=500_000, nnz_per_col=10, seed=2),
    "C3": dict(kind="mcf", nodes=10_000, arcs_per_node=10, commodities=20, side_rows=100_000,
               side_per_var=7, seed=3),
    "C4": dict(kind="staircase", stages=1000, cols_per_stage=10_000, rows_per_stage=5_000,
               own_per_col=6, next_per_col=4, seed=4),
    "C5": dict(kind="powerlaw", m=10_000_000, n=50_000_000, nnz=500_000_000, seed=5),
    # C5 at 1/10 and 1/100 scale: the same row-length law for tests and probes
    "C5s": dict(kind="powerlaw", m=1_000_000, n=5_000_000, nnz=50_000_000, seed=5),
    "C5xs": dict(kind="powerlaw", m=100_000, n=500_000, nnz=5_000_000, seed=5),
}


def make_config(name: str) -> LinearProgram:
    spec = dict(CONFIGS[name])
    kind = spec.pop("kind")
    if kind == "transportation":
        return transportation_lp(**spec)
    if kind == "random":
        return random_equality_lp(**spec)[0]
    if kind == "mcf":
        return multicommodity_lp(**spec)
    if kind == "staircase":
        return staircase_lp(**spec)[0]
    if kind == "powerlaw":
        return powerlaw_lp(**spec)[0]
    raise KeyError(name)
