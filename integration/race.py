"""ctypes bridge to cclp::run_race (integration/run_race.cpp via
integration/race_capi.cpp), built by `make -C integration` into
integration/lib/librace_gpu.so (run_pdhg = the B200 engine) and
integration/lib/librace_cpu.so (run_pdhg = the reference's CPU loop); the
crossover is the reference's run_crossover in both, over the product's sparse
LU (third_party/eigen_subset). Used by tests/ and
tools/time_to_basic.py."""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBS = {"gpu": os.path.join(ROOT, "integration", "lib", "librace_gpu.so"),
        "cpu": os.path.join(ROOT, "integration", "lib", "librace_cpu.so")}
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_cache = {}


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def lib(kind: str):
    if kind not in _cache:
        L = C.CDLL(LIBS[kind])
        L.cclp_race_last_error.restype = C.c_char_p
        L.cclp_race_run.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int,
                                    C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                    C.c_longlong, C.c_char_p, C.c_int]
        L.cclp_race_schedule.argtypes = [C.c_double, C.c_double, C.c_double, _dp, C.c_int]
        L.cclp_race_reserve.argtypes = [C.c_int, C.c_int, _ip, _ip]
        L.cclp_race_simulate.argtypes = [_dp, C.c_int, C.c_double, _dp, _dp, _ip, C.c_int, C.c_double,
                                         C.c_int, C.c_int, C.c_double, C.c_double, C.c_int,
                                         C.c_double, C.c_char_p, C.c_int]
        L.cclp_race_standard_form_check.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp, _dp,
                                                    _dp, _dp, C.c_int, C.c_int, _dp]
        L.cclp_race_set_crossover.argtypes = [C.c_int, C.c_int]
        L.cclp_race_crossover.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                          C.c_double, C.c_double, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.cclp_race_pricing_counts.argtypes = [C.POINTER(C.c_longlong)]
        _cache[kind] = L
    return _cache[kind]


def standard_form_check(lp, maximize: bool = False, named: bool = False, kind: str = "cpu",
                        timings: bool = False):
    """(equal, reason[, (t_reference_s, t_direct_s)]): the race's O(nnz)
    standard form against the reference's to_standard_form
    (standard_form.cpp:23-104) on `lp`."""
    import numpy as np
    L = lib(kind)
    a = [np.ascontiguousarray(x, t) for x, t in (
        (lp.colptr, np.int32), (lp.rowind, np.int32), (lp.val, np.float64), (lp.c, np.float64),
        (lp.row_lower, np.float64), (lp.row_upper, np.float64), (lp.col_lower, np.float64),
        (lp.col_upper, np.float64))]
    ptr = [x.ctypes.data_as(_ip if x.dtype == np.int32 else _dp) for x in a]
    t = np.zeros(2)
    rc = L.cclp_race_standard_form_check(lp.m, lp.n, *ptr, int(maximize), int(named),
                                         t.ctypes.data_as(_dp))
    if rc == 2:
        raise ValueError(L.cclp_race_last_error().decode())
    out = (rc == 0, L.cclp_race_last_error().decode())
    return out + ((float(t[0]), float(t[1])),) if timings else out


CROSSOVER = {"reference": 0, "scalable": 1, "scalable-device": 2}


def set_crossover(kind: str, crossover: str, device: int = 0) -> None:
    """The race's crossover (race_capi.cpp cclp_race_set_crossover): the
    reference's run_crossover, or crossover_scalable.cpp with host or B200
    pricing. Library defaults: gpu -> scalable-device, cpu -> reference."""
    L = lib(kind)
    if L.cclp_race_set_crossover(CROSSOVER[crossover], device) != 0:
        raise RuntimeError(L.cclp_race_last_error().decode())


def crossover(std_lp, x, y, z, threshold: float, crossover: str = "scalable", eps_abs: float = 1e-6,
              kind: str = "cpu", device: int = 0) -> dict:
    """One run_crossover on an equality-form LP from the iterate (x, y, z):
    status, sorted basic set, objective, pivots, seconds and the scalable
    engine's statistics (race_capi.cpp cclp_race_crossover)."""
    L = lib(kind)
    k = [np.ascontiguousarray(std_lp.colptr, np.int32), np.ascontiguousarray(std_lp.rowind, np.int32)]
    d = [np.ascontiguousarray(a, np.float64) for a in (std_lp.val, std_lp.c, std_lp.row_lower, std_lp.col_lower,
                                                       std_lp.col_upper, x, y, z)]
    cap = 64 * 1024 + 24 * std_lp.m
    buf = C.create_string_buffer(cap)
    rc = L.cclp_race_crossover(std_lp.m, std_lp.n, k[0].ctypes.data_as(_ip), k[1].ctypes.data_as(_ip),
                               *[a.ctypes.data_as(_dp) for a in d], threshold, eps_abs, CROSSOVER[crossover],
                               device, buf, cap)
    if rc != 0:
        raise RuntimeError(L.cclp_race_last_error().decode())
    return json.loads(buf.value.decode())


def pricing_counts(kind: str) -> tuple:
    """(device, host) pricing calls made by scalable crossovers so far."""
    out = (C.c_longlong * 2)()
    lib(kind).cclp_race_pricing_counts(out)
    return int(out[0]), int(out[1])


def run_race(lp, kind: str = "gpu", mode: str = "concurrent", eps_rel: float = 1e-6,
             eps_cross: float = 1e-2, eps_abs: float = 1e-6, time_limit: float = 3600.0,
             pool: int = 4, max_iterations: int = 2_000_000, crossover: str = None) -> dict:
    L = lib(kind)
    if crossover is not None:
        set_crossover(kind, crossover)
    k = [np.ascontiguousarray(lp.colptr, np.int32), np.ascontiguousarray(lp.rowind, np.int32)]
    d = [np.ascontiguousarray(a, np.float64) for a in (lp.val, lp.c, lp.row_lower, lp.row_upper,
                                                       lp.col_lower, lp.col_upper)]
    cap = 64 * 1024 + 32 * (lp.n + lp.m)
    buf = C.create_string_buffer(cap)
    rc = L.cclp_race_run(lp.m, lp.n, k[0].ctypes.data_as(_ip), k[1].ctypes.data_as(_ip),
                         *[a.ctypes.data_as(_dp) for a in d], 1 if mode == "concurrent" else 0,
                         eps_rel, eps_cross, eps_abs, time_limit, pool, max_iterations, buf, cap)
    if rc != 0:
        raise RuntimeError(L.cclp_race_last_error().decode())
    return json.loads(buf.value.decode())


def schedule_thresholds(eps_rel: float, eps_cross: float, decrement: float, kind: str = "cpu"):
    out = (C.c_double * 64)()
    n = lib(kind).cclp_race_schedule(eps_rel, eps_cross, decrement, out, 64)
    if n < 0:
        raise ValueError(lib(kind).cclp_race_last_error().decode())
    return list(out[:n])


def reserve_threads(pool: int, cores: int, kind: str = "cpu"):
    a, b = C.c_int32(), C.c_int32()
    lib(kind).cclp_race_reserve(pool, cores, C.byref(a), C.byref(b))
    return a.value, b.value


def simulate(trace, sec_per_iter, workers: dict, main=(0.0, True), mode="concurrent",
             eps_rel=1e-6, eps_cross=1e-2, pool=4, time_limit=3600.0, kind: str = "cpu") -> dict:
    L = lib(kind)
    tr = np.ascontiguousarray(trace, np.float64)
    thr = np.ascontiguousarray(list(workers.keys()), np.float64)
    dur = np.ascontiguousarray([w[0] for w in workers.values()], np.float64)
    ok = np.ascontiguousarray([1 if w[1] else 0 for w in workers.values()], np.int32)
    buf = C.create_string_buffer(1 << 16)
    rc = L.cclp_race_simulate(tr.ctypes.data_as(_dp), tr.size, sec_per_iter, thr.ctypes.data_as(_dp),
                              dur.ctypes.data_as(_dp), ok.ctypes.data_as(_ip), thr.size, main[0],
                              1 if main[1] else 0, 1 if mode == "concurrent" else 0, eps_rel,
                              eps_cross, pool, time_limit, buf, 1 << 16)
    if rc != 0:
        raise RuntimeError(L.cclp_race_last_error().decode())
    return json.loads(buf.value.decode())
