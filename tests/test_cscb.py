"""LP ingest from the binary CSC file (.cscb).

CPU: the writer/reader round trip, header checks, and the C-ABI entry point's
error path on a bad file (no device needed to reject a file). GPU: a solve of
an engine created from the file is bit-identical to one created from arrays."""
import os

import numpy as np
import pytest

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.lp import CSCB_MAGIC, read_cscb, write_cscb
from paper_2510_24429_b200.pdhg import Engine, PdhgConfig


def _lps():
    yield "two_var", lpgen.two_var_lp()
    yield "c2_small", lpgen.random_equality_lp(60, 140, 4, seed=5)[0]
    yield "ragged", lpgen.small_equality_lp(33, 71, density=0.13, seed=9)[0]


@pytest.mark.parametrize("name,lp", list(_lps()))
def test_round_trip(tmp_path, name, lp):
    p = str(tmp_path / f"{name}.cscb")
    write_cscb(lp, p)
    back = read_cscb(p)
    assert (back.m, back.n, back.nnz) == (lp.m, lp.n, lp.nnz)
    for f in ("colptr", "rowind", "val", "c", "row_lower", "row_upper", "col_lower", "col_upper"):
        a, b = np.asarray(getattr(lp, f)), np.asarray(getattr(back, f))
        assert a.shape == b.shape and np.array_equal(a, b, equal_nan=True), f
    with open(p, "rb") as fh:
        assert fh.read(8) == CSCB_MAGIC
    assert os.path.getsize(p) % 8 == 0


def test_bad_magic_rejected(tmp_path):
    p = str(tmp_path / "bad.cscb")
    with open(p, "wb") as fh:
        fh.write(b"NOTACSCB" + bytes(24))
    with pytest.raises(ValueError):
        read_cscb(p)


def test_abi_rejects_bad_files(tmp_path):
    import ctypes as C
    from paper_2510_24429_b200.pdhg import load_library
    L = load_library()
    ctx = C.c_void_p()
    missing = str(tmp_path / "missing.cscb").encode()
    assert L.cclp_cu_create_from_file(missing, 0, C.byref(ctx), None, None) != 0
    bad = tmp_path / "bad.cscb"
    bad.write_bytes(b"NOTACSCB" + bytes(24))
    assert L.cclp_cu_create_from_file(str(bad).encode(), 0, C.byref(ctx), None, None) != 0
    # truncated: header promises more than the file holds
    good = str(tmp_path / "good.cscb")
    write_cscb(lpgen.small_equality_lp(20, 50, seed=1)[0], good)
    with open(good, "rb") as fh:
        data = fh.read()
    trunc = tmp_path / "trunc.cscb"
    trunc.write_bytes(data[:len(data) // 2])
    assert L.cclp_cu_create_from_file(str(trunc).encode(), 0, C.byref(ctx), None, None) != 0
    assert not ctx.value


@pytest.mark.gpu
@pytest.mark.parametrize("name,lp", list(_lps()))
def test_solve_from_file_matches_arrays(tmp_path, name, lp):
    p = str(tmp_path / f"{name}.cscb")
    write_cscb(lp, p)
    cfg = PdhgConfig(max_iterations=3000)
    with Engine(lp) as a:
        ra = a.solve(cfg)
    with Engine.from_file(p) as b:
        rb = b.solve(cfg)
    assert ra.iterations == rb.iterations and ra.stop == rb.stop
    assert np.array_equal(ra.iterate.x, rb.iterate.x)
    assert np.array_equal(ra.iterate.y, rb.iterate.y)


def test_round_trip_empty_matrix(tmp_path):
    """A matrix with no nonzeros (and an LP with no rows) survives the format."""
    from paper_2510_24429_b200.lp import INF, LinearProgram
    lp = LinearProgram(3, 4, np.zeros(5, np.int32), np.zeros(0, np.int32), np.zeros(0),
                       np.arange(4.0), np.ones(3), np.ones(3), np.zeros(4), np.full(4, INF))
    p = str(tmp_path / "empty.cscb")
    write_cscb(lp, p)
    back = read_cscb(p)
    assert (back.m, back.n, back.nnz) == (3, 4, 0)
    assert np.array_equal(back.c, lp.c) and np.all(np.isinf(back.col_upper))
    norows = LinearProgram(0, 2, np.zeros(3, np.int32), np.zeros(0, np.int32), np.zeros(0),
                           np.ones(2), np.zeros(0), np.zeros(0), np.zeros(2), np.ones(2))
    write_cscb(norows, p)
    back = read_cscb(p)
    assert (back.m, back.n, back.nnz) == (0, 2, 0) and np.array_equal(back.col_upper, np.ones(2))
