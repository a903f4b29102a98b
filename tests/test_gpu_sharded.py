"""GPU: the row-block sharded solve in its one-GPU form -
P shards in one process exchanging by device copies, the same kernels and
launch order as the NCCL path. Each shard computes its rows of A x and A'y
completely, so the iterates must be bit-identical to the single-device engine
at equal iteration counts (the report sums are combined per shard, so the
reports agree to rounding)."""
import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import (PdhgConfig, PdhgStopReason, ShardedEngine, Tolerances,
                                        run_pdhg, run_pdhg_sharded)

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["push", "gather"], autouse=True)
def transport(request, monkeypatch):
    """Every sharded test runs over both transports: the fused push (P2P
    stores inside the producing kernels + epoch flags) and the gathers
    (device copies / NCCL)."""
    monkeypatch.setenv("CCLP_CU_TRANSPORT", request.param)
    return request.param


def lps():
    return [("eq40x90", lpgen.small_equality_lp(40, 90, 0.2, 7)[0]),
            ("transport20x30", lpgen.transportation_lp(20, 30, seed=3)),
            ("random2k", lpgen.random_equality_lp(2000, 10000, 8, seed=9)[0])]


@pytest.mark.parametrize("name,lp", lps())
@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_sharded_bit_identical_to_single(name, lp, P):
    cfg = PdhgConfig(max_iterations=300)
    one = run_pdhg(lp, cfg)
    sh = run_pdhg_sharded(lp, P, cfg)
    assert sh.iterations == one.iterations
    assert sh.restarts == one.restarts
    assert sh.stop == one.stop
    assert np.array_equal(sh.iterate.x, one.iterate.x)
    assert np.array_equal(sh.iterate.y, one.iterate.y)
    assert np.array_equal(sh.iterate.z, one.iterate.z)
    assert sh.report.maxresid_rel == pytest.approx(one.report.maxresid_rel, rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_converges_like_single(P):
    lp = lpgen.small_equality_lp(40, 90, 0.2, 7)[0]
    one = run_pdhg(lp, PdhgConfig(max_iterations=20000))
    sh = run_pdhg_sharded(lp, P, PdhgConfig(max_iterations=20000))
    assert sh.stop == one.stop == PdhgStopReason.kConverged
    assert sh.iterations == one.iterations
    assert np.array_equal(sh.iterate.x, one.iterate.x)


def test_sharded_snapshots_match():
    lp = lpgen.two_var_lp()
    a, b = [], []
    one = run_pdhg(lp, thresholds=[1e-2, 1e-3], sink=a.append)
    sh = run_pdhg_sharded(lp, 1, thresholds=[1e-2, 1e-3], sink=b.append)
    assert [s.iteration for s in a] == [s.iteration for s in b]
    for s, t in zip(a, b):
        assert np.array_equal(s.iterate.x, t.iterate.x)
    assert sh.iterations == one.iterations


def test_sharded_long_rows_and_bounds():
    lp = lpgen.make_config("C5xs")
    cfg = PdhgConfig(max_iterations=40)
    one = run_pdhg(lp, cfg)
    sh = run_pdhg_sharded(lp, 3, cfg)
    assert np.array_equal(sh.iterate.x, one.iterate.x)
    assert np.array_equal(sh.iterate.y, one.iterate.y)
    with ShardedEngine(lp, 3) as eng:
        d = eng.describe()
    assert d["shards"] == 3 and d["row_bounds"][-1] == lp.m and d["col_bounds"][-1] == lp.n


def test_sharded_measurement_hooks():
    lp = lpgen.random_equality_lp(2000, 10000, 8, seed=9)[0]
    with ShardedEngine(lp, 2) as eng:
        eng.begin(PdhgConfig())
        ms = eng.advance(50)
    assert ms > 0


def test_nccl_transport_one_rank_matches_single():
    """The NCCL transport (ncclAllGather in place, captured in the CUDA graph)
    with a one-rank communicator: identical iterates to the one-device engine."""
    from paper_2510_24429_b200.pdhg import nccl_unique_id
    lp = lpgen.random_equality_lp(2000, 10000, 8, seed=9)[0]
    cfg = PdhgConfig(max_iterations=200)
    one = run_pdhg(lp, cfg)
    with ShardedEngine(lp, 1, rank=0, nranks=1, nccl_id=nccl_unique_id()) as eng:
        sh = eng.solve(cfg)
    assert sh.iterations == one.iterations
    assert np.array_equal(sh.iterate.x, one.iterate.x)
    assert np.array_equal(sh.iterate.y, one.iterate.y)


@pytest.mark.parametrize("P", [2, 3, 4])
def test_halo_exchange_staircase_bit_identical(P):
    """A staircase LP (C4's structure) needs only the neighbouring stage's x
    and y: the halo exchange replaces the all-gathers and the iterates stay
    bit-identical to one device."""
    lp = lpgen.staircase_lp(stages=24, cols_per_stage=300, rows_per_stage=150, seed=6)[0]
    cfg = PdhgConfig(max_iterations=300)
    one = run_pdhg(lp, cfg)
    with ShardedEngine(lp, P) as eng:
        sh = eng.solve(cfg)
        d = eng.describe()
    assert d["halo_x"] and d["halo_y"]
    assert d["halo_x_volume"] < lp.n and d["halo_y_volume"] < lp.m
    assert sh.iterations == one.iterations and sh.restarts == one.restarts
    assert np.array_equal(sh.iterate.x, one.iterate.x)
    assert np.array_equal(sh.iterate.y, one.iterate.y)


@pytest.mark.parametrize("P", [2, 3])
def test_sharded_column_panels_bit_identical(P, monkeypatch):
    """Column panels (forced small here; C5 uses 9 of 48 MB) are defined on the
    original column space and take the full matrix's G, so the sharded sums
    equal the single-device sums."""
    monkeypatch.setenv("CCLP_CU_PANEL_BYTES", "65536")
    lp = lpgen.make_config("C5xs")
    cfg = PdhgConfig(max_iterations=40)
    one = run_pdhg(lp, cfg)
    sh = run_pdhg_sharded(lp, P, cfg)
    assert np.array_equal(sh.iterate.x, one.iterate.x)
    assert np.array_equal(sh.iterate.y, one.iterate.y)


@pytest.mark.parametrize("P", [2, 4])
def test_shards_hold_only_their_slices_and_setup_is_bit_identical(P):
    """No device copy of the full LP: shard p holds only the nonzeros of its
    row block of A and its column block of A' (sum = nnz, each ~ nnz/P), and
    the distributed setup (Ruiz over all-gathered scales, the power iteration
    over the shards, reproducible sums) gives the single device's
    ||A||, omega, tau and sigma bit for bit."""
    lp = lpgen.staircase_lp(stages=32, cols_per_stage=400, rows_per_stage=200, seed=6)[0]
    cfg = PdhgConfig(max_iterations=50)
    one = run_pdhg(lp, cfg)
    with ShardedEngine(lp, P) as eng:
        sh = eng.solve(cfg)
        d = eng.describe()
    loc = d["local_shards"]
    assert [s["rank"] for s in loc] == list(range(P))
    assert sum(s["nnz_rows"] for s in loc) == lp.nnz
    assert sum(s["nnz_cols"] for s in loc) == lp.nnz
    for s in loc:
        assert s["nnz_rows"] <= 1.25 * lp.nnz / P and s["nnz_cols"] <= 1.25 * lp.nnz / P
    for k in ("norm_estimate", "omega", "tau", "sigma"):
        assert getattr(sh, k) == getattr(one, k), k
    assert np.array_equal(sh.iterate.x, one.iterate.x)
    assert np.array_equal(sh.iterate.y, one.iterate.y)
