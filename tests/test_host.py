"""CPU: host-side LP handling (lp.py, lpgen.py) against the reference's rules."""
import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.lp import INF, LinearProgram, csc_from_triplets, to_standard_form


def test_make_sparse_semantics():
    # kernels.cpp:20-27 / test_kernels.cpp:50-57: duplicates summed, zeros pruned
    colptr, rowind, val = csc_from_triplets(2, 2, [0, 0, 1, 1], [0, 0, 1, 0], [1.0, 2.0, 0.0, -1.0])
    assert list(colptr) == [0, 2, 2]
    assert list(rowind) == [0, 1] and list(val) == [3.0, -1.0]


def test_validate_rejects_bad_structure():
    lp = lpgen.two_var_lp()
    lp.validate()
    bad = lpgen.two_var_lp()
    bad.val = np.array([1.0, 0.0])
    with pytest.raises(ValueError):
        bad.validate()
    crossed = lpgen.two_var_lp()
    crossed.col_lower = np.array([1.0, 0.0])
    crossed.col_upper = np.array([0.0, INF])
    with pytest.raises(ValueError):
        crossed.validate()


def test_standard_form_le_row():
    # test_standard_form.cpp:29-43: x1 + x2 <= 4 gains a [0, inf) slack, b = 4
    gen = LinearProgram(1, 2, np.array([0, 1, 2], np.int32), np.array([0, 0], np.int32),
                        np.ones(2), np.array([1.0, 0.0]), np.array([-INF]), np.array([4.0]),
                        np.zeros(2), np.full(2, INF))
    s = to_standard_form(gen)
    assert s.n == 3 and s.row_lower[0] == 4.0 and s.row_upper[0] == 4.0
    assert s.col_lower[2] == 0.0 and s.col_upper[2] == INF
    assert s.all_rows_equality()


def test_standard_form_ge_row_and_max():
    gen = LinearProgram(1, 1, np.array([0, 1], np.int32), np.array([0], np.int32), np.ones(1),
                        np.array([3.0]), np.array([2.0]), np.array([INF]), np.zeros(1),
                        np.full(1, INF))
    s = to_standard_form(gen, maximize=True)
    assert s.row_lower[0] == 2.0 and s.col_lower[1] == -INF and s.col_upper[1] == 0.0
    assert s.c[0] == -3.0


def test_transportation_shape_c1():
    lp = lpgen.transportation_lp()
    assert (lp.m, lp.n, lp.nnz) == (700, 100_700, 200_700)
    assert lp.all_rows_equality()
    lp.validate()


@pytest.mark.parametrize("m,n", [(5, 10), (30, 80)])
def test_known_optimum_satisfies_kkt(m, n, oracle):
    lp, xs, ys, zs = lpgen.small_equality_lp(m, n, 0.4, 1)
    rep = oracle.relative_report(lp, xs, ys, zs)
    assert rep["maxresid_rel"] < 1e-12


def test_random_lp_c2_shape_small():
    lp, xs, ys, zs = lpgen.random_equality_lp(m=2000, n=10_000, nnz_per_col=10, seed=2)
    lp.validate()
    assert lp.nnz == 100_000 and lp.all_rows_equality()
    A = lp.dense()
    assert np.allclose(A @ xs, lp.row_lower)
    assert np.allclose(A.T @ ys + zs, lp.c)
    assert np.all(xs * zs == 0)
