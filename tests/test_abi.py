"""CPU: the C-ABI library builds, loads without a GPU and exports every symbol
include/cclp_cu.h declares; host-only entry points behave."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cclp_cu.h")
LIB = os.path.join(ROOT, "paper_2510_24429_b200", "libcclp_cuda.so")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(cclp_cu_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2510_24429_b200 import build
        build.build()
    return C.CDLL(LIB)


def test_header_declares_the_run_pdhg_boundary():
    syms = declared_symbols()
    for s in ("cclp_cu_run_pdhg", "cclp_cu_create", "cclp_cu_solve", "cclp_cu_destroy",
              "cclp_cu_matvec", "cclp_cu_matvec_transpose", "cclp_cu_ruiz",
              "cclp_cu_estimate_norm"):
        assert s in syms


def test_every_declared_symbol_is_exported(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_mirror_lists_every_symbol():
    from paper_2510_24429_b200.pdhg import EXPORTED_SYMBOLS
    assert sorted(EXPORTED_SYMBOLS) == declared_symbols()


def test_stop_strings(lib):
    # to_string(PdhgStopReason), pdhg.cpp:28-44
    lib.cclp_cu_stop_string.restype = C.c_char_p
    got = [lib.cclp_cu_stop_string(i).decode() for i in range(7)]
    assert got == ["converged", "iteration-limit", "time-limit", "cancelled",
                   "won-by-crossover", "numerical-error", "unknown"]


def test_default_config_matches_reference(lib):
    from paper_2510_24429_b200.pdhg import PdhgConfig, Tolerances, _Config, _Tol
    c = _Config()
    lib.cclp_cu_default_config(C.byref(c))
    d = PdhgConfig()
    # pdhg.hpp:29-42
    assert (c.step_scale, c.primal_weight, c.restart_factor, c.norm_iterations,
            c.scaling_iterations, c.max_iterations, c.check_interval, c.seed) == \
        (d.step_scale, d.primal_weight, d.restart_factor, d.norm_iterations,
         d.scaling_iterations, d.max_iterations, d.check_interval, d.seed) == \
        (0.9, 0.0, 0.5, 100, 10, 2000000, 1, 0)
    t = _Tol()
    lib.cclp_cu_default_tolerances(C.byref(t))
    assert (t.eps_rel, t.eps_abs, t.eps_cross, t.decrement) == (1e-6, 1e-6, 1e-2, 0.1)
    assert Tolerances() == Tolerances(t.eps_rel, t.eps_abs, t.eps_cross, t.decrement)


def test_struct_layouts_match_header():
    """ctypes mirrors must match the C structs field for field."""
    from paper_2510_24429_b200 import pdhg
    src = open(HEADER).read()
    for cname, py in (("cclp_cu_config", pdhg._Config), ("cclp_cu_result", pdhg._Result),
                      ("cclp_cu_snapshot", pdhg._Snapshot), ("cclp_cu_lp", pdhg._LP)):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + cname + ";", src).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        fields = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            names = decl.split(None, 1)[1] if not decl.startswith("const") else \
                decl.split(None, 2)[2]
            for nm in names.split(","):
                fields.append(nm.strip().lstrip("*").strip())
        assert [f[0] for f in py._fields_] == fields, cname


def test_create_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_24429_b200 import lpgen
    from paper_2510_24429_b200.pdhg import Engine
    with pytest.raises(RuntimeError):
        Engine(lpgen.two_var_lp())


def test_no_cpu_fallback_in_product():
    """The product path never imports the oracle."""
    for f in os.listdir(os.path.join(ROOT, "paper_2510_24429_b200")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "paper_2510_24429_b200", f)).read()
            assert "oracle" not in src.replace("# ", ""), f


@pytest.mark.parametrize("seed,n", [(0, 1), (0, 7), (3, 1000), (12345, 200001), (7, 3_000_001)])
def test_gaussian_start_matches_oracle(seed, n):
    """The engine's two-stage start vector equals the oracle's sequential
    mt19937_64 + normal_distribution restatement bit for bit (host only)."""
    import numpy as np

    from oracle.pyoracle import Restatement
    from paper_2510_24429_b200.pdhg import gaussian_start
    ours = gaussian_start(seed, n)
    ref = Restatement().gaussian_start(seed, n)
    assert np.array_equal(ours.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("case,msg", [
    ("colptr0", "colptr[0] != 0"),
    ("decreasing", "decreasing column offsets"),
    ("range", "row index out of range"),
    ("negative", "row index out of range"),
    ("unsorted", "unsorted or duplicate row indices"),
    ("duplicate", "unsorted or duplicate row indices"),
])
def test_create_rejects_malformed_csc_before_touching_the_device(lib, case, msg):
    """LinearProgram::validate's CSC checks (lp.cpp:71-83) run on the host in
    cclp_cu_create, so a bad matrix is EINVAL (no GPU needed) instead of an
    out-of-bounds gather on the device."""
    import numpy as np

    from paper_2510_24429_b200.pdhg import _LP
    colptr = np.array([0, 2, 3], np.int32)
    rowind = np.array([0, 1, 1], np.int32)
    if case == "colptr0":
        colptr = np.array([1, 2, 3], np.int32)
    elif case == "decreasing":
        colptr = np.array([0, 3, 2], np.int32)
    elif case == "range":
        rowind = np.array([0, 2, 1], np.int32)
    elif case == "negative":
        rowind = np.array([0, -1, 1], np.int32)
    elif case == "unsorted":
        rowind = np.array([1, 0, 1], np.int32)
    elif case == "duplicate":
        rowind = np.array([1, 1, 1], np.int32)
    val = np.ones(3)
    v2, v1 = np.zeros(2), np.zeros(2)
    dp = C.POINTER(C.c_double)
    ip = C.POINTER(C.c_int32)
    lp = _LP(2, 2, colptr.ctypes.data_as(ip), rowind.ctypes.data_as(ip), val.ctypes.data_as(dp),
             v2.ctypes.data_as(dp), v1.ctypes.data_as(dp), v1.ctypes.data_as(dp),
             v2.ctypes.data_as(dp), v2.ctypes.data_as(dp))
    ctx = C.c_void_p()
    lib.cclp_cu_last_error.restype = C.c_char_p
    assert lib.cclp_cu_create(C.byref(lp), 0, C.byref(ctx)) == 1  # CCLP_CU_EINVAL
    assert msg in lib.cclp_cu_last_error().decode()
    assert not ctx.value


def test_iteration_kernels_keep_no_stack_frame():
    """The per-iteration kernels take IterParams (~2 KB) by value; a helper that
    is not inlined copies it into a per-thread stack frame on every launch (a
    50% slowdown of the epilogues, measured). Guard it from the cubin."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(LIB) or not os.path.exists(tool):
        pytest.skip("library or cuobjdump missing")
    out = subprocess.run([tool, "-res-usage", LIB], capture_output=True, text=True).stdout
    seen = 0
    for fn, stack in re.findall(r"Function (\S+):\s*\n\s*REG:\d+ STACK:(\d+)", out):
        if re.search(r"k_(spmv_rows|spmv_cols|dual|primal|finalize)", fn):
            seen += 1
            assert int(stack) <= 16, (fn, stack)
    assert seen >= 6
