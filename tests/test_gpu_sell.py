"""GPU: the SELL-32 column product (k_spmv_cols_sell; engine.cu
build_sell_cols), chosen by the matrix (near-uniform column lengths: slices
padded to at most 1.25x the nonzeros); CCLP_CU_SELL=1 is the default. Each column is summed by one lane in ascending
position — the reference's own order — so: equal-iteration parity with the
oracle, sharded solves bit-identical to one device, long columns (left to the
segment path) handled, and the result within rounding of the CSR column
kernel."""
import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.lp import csc_from_triplets
from paper_2510_24429_b200.pdhg import PdhgConfig, run_pdhg, run_pdhg_sharded

pytestmark = pytest.mark.gpu


def rel(a, b):
    d = np.linalg.norm(np.asarray(a) - np.asarray(b))
    return d / max(np.linalg.norm(b), 1e-300) if d > 0 else 0.0


@pytest.fixture(autouse=True)
def sell(monkeypatch):
    monkeypatch.setenv("CCLP_CU_SELL", "1")


def dense_cols_lp(m=2000, n=20_000, dense=(3, 500, 19_000), seed=13):
    """Short random columns plus a few columns touching every row."""
    rng = np.random.default_rng(seed)
    rows = [rng.integers(0, m, size=6 * n), np.tile(np.arange(m), len(dense)), np.arange(m)]
    perm = rng.permutation(n)
    cols = [np.repeat(np.arange(n), 6), np.repeat(np.array(dense), m), perm[:m]]
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rng.uniform(-2, 2, size=rows.size)
    vals[-m:] = rng.uniform(2, 3, size=m)
    colptr, rowind, val = csc_from_triplets(m, n, rows, cols, vals)
    return lpgen._known_optimum(colptr.astype(np.int64), rowind, val, m, n, perm[:m], rng,
                                "dense_cols")[0]


def lps():
    return [("eq40x90", lpgen.small_equality_lp(40, 90, 0.2, 7)[0]),
            ("transport20x30", lpgen.transportation_lp(20, 30, seed=3)),
            ("random2k", lpgen.random_equality_lp(2000, 10000, 8, seed=9)[0]),
            ("dense_cols", dense_cols_lp())]


@pytest.mark.parametrize("name,lp", lps())
@pytest.mark.parametrize("iters", [1, 40])
def test_sell_equal_iteration_parity(name, lp, iters, oracle):
    res = run_pdhg(lp, PdhgConfig(max_iterations=iters))
    ref = oracle.run_pdhg(lp, config=dict(max_iterations=iters))
    assert res.iterations == ref["iterations"]
    for a, b in ((res.iterate.x, ref["x"]), (res.iterate.y, ref["y"]), (res.iterate.z, ref["z"])):
        assert rel(a, b) <= 1e-9


@pytest.mark.parametrize("name,lp", lps())
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("mode", ["contig", "small", "gs"])
def test_sell_sharded_bit_identical(name, lp, P, mode, monkeypatch):
    """Every slice-to-warp deal (block-contiguous 1024 / 256, grid-stride)
    gives the same sums: shards and one device agree bit for bit."""
    monkeypatch.setenv("CCLP_CU_SELL_MODE", mode)
    cfg = PdhgConfig(max_iterations=200)
    one = run_pdhg(lp, cfg)
    sh = run_pdhg_sharded(lp, P, cfg)
    assert sh.iterations == one.iterations and sh.stop == one.stop
    assert np.array_equal(sh.iterate.x, one.iterate.x)
    assert np.array_equal(sh.iterate.y, one.iterate.y)


@pytest.mark.parametrize("name,lp", lps())
def test_sell_rerun_identical_and_close_to_csr(name, lp, monkeypatch):
    cfg = PdhgConfig(max_iterations=200)
    a = run_pdhg(lp, cfg)
    b = run_pdhg(lp, cfg)
    assert np.array_equal(a.iterate.x, b.iterate.x) and np.array_equal(a.iterate.y, b.iterate.y)
    monkeypatch.setenv("CCLP_CU_SELL", "0")
    c = run_pdhg(lp, cfg)
    assert rel(a.iterate.x, c.iterate.x) <= 1e-9 and rel(a.iterate.y, c.iterate.y) <= 1e-9


# ---- SELL-G products (k_spmv_rows_sellg, k_spmv_cols_sellg): chosen by
# timing, so they must be bit-identical to the CSR-G kernels;
# CCLP_CU_SELL_ROWS=2 / CCLP_CU_SELLG_COLS=2 force them.

def _long_rows_lp():
    from test_gpu_longrows import dense_rows_lp
    return dense_rows_lp()


@pytest.mark.parametrize("name", ["eq40x90", "transport20x30", "random2k", "dense_cols", "long_rows"])
def test_sellg_rows_bit_identical_to_csr(name, monkeypatch):
    lp = _long_rows_lp() if name == "long_rows" else dict(lps())[name]
    cfg = PdhgConfig(max_iterations=150)
    monkeypatch.setenv("CCLP_CU_SELL", "0")
    monkeypatch.setenv("CCLP_CU_SELL_ROWS", "0")
    monkeypatch.setenv("CCLP_CU_SELLG_COLS", "0")
    a = run_pdhg(lp, cfg)
    monkeypatch.setenv("CCLP_CU_SELL_ROWS", "2")
    monkeypatch.setenv("CCLP_CU_SELLG_COLS", "2")  # both sides in SELL-G slices
    b = run_pdhg(lp, cfg)
    sh = run_pdhg_sharded(lp, 2, cfg)
    assert a.iterations == b.iterations == sh.iterations
    for u, v in ((a.iterate.x, b.iterate.x), (a.iterate.y, b.iterate.y), (a.iterate.x, sh.iterate.x)):
        assert np.array_equal(u, v)
