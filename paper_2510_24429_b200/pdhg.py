"""Python mirror of the reference's PDHG interface over the sm_100a engine.

Same names, argument meaning and error behaviour as
``cclp::run_pdhg`` (proj/include/cclp/pdhg.hpp:29-142, proj/src/pdhg.cpp):

  * ``PdhgConfig`` / ``Tolerances`` / ``ResidualReport`` / ``PdhgSnapshot`` /
    ``PdhgResult`` / ``PdhgStopReason`` — field-for-field.
  * ``run_pdhg(std_lp, config, tol, thresholds, sink, cancel)`` raises
    ``ValueError`` where the reference throws ``std::invalid_argument``
    (non-equality LP, bad tolerances, non-decreasing thresholds); a non-finite
    iterate is reported as ``PdhgStopReason.kNumericalError``.
  * The sink is called synchronously on the calling thread with a snapshot
    whose arrays are copies.

Every call goes through ``libcclp_cuda.so`` (include/cclp_cu.h); there is no
CPU path. Importing this module on a machine without a GPU works; calling it
raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
import threading
from typing import Callable, Optional, Sequence

import numpy as np

from .lp import LinearProgram

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CCLP_CU_LIB", os.path.join(HERE, "libcclp_cuda.so"))

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class _LP(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("colptr", _ip), ("rowind", _ip),
                ("val", _dp), ("c", _dp), ("row_lower", _dp), ("row_upper", _dp),
                ("col_lower", _dp), ("col_upper", _dp)]


class _Config(C.Structure):
    _fields_ = [("step_scale", C.c_double), ("primal_weight", C.c_double),
                ("restart_factor", C.c_double), ("time_limit", C.c_double),
                ("norm_iterations", C.c_int32), ("scaling_iterations", C.c_int32),
                ("max_iterations", C.c_int64), ("check_interval", C.c_int32),
                ("seed", C.c_uint64), ("log_interval", C.c_int64),
                ("deterministic", C.c_int32), ("poll_interval", C.c_int32),
                ("exact_spmv", C.c_int32)]


class _Tol(C.Structure):
    _fields_ = [("eps_rel", C.c_double), ("eps_abs", C.c_double), ("eps_cross", C.c_double),
                ("decrement", C.c_double)]


REPORT_FIELDS = ["rp_norm2", "rd_norm2", "rp_inf", "rd_inf", "primal_objective",
                 "dual_objective", "gap_abs", "rel_primal", "rel_dual", "rel_gap",
                 "maxresid_rel", "complementarity"]


class _Report(C.Structure):
    _fields_ = [(f, C.c_double) for f in REPORT_FIELDS]


class _Snapshot(C.Structure):
    _fields_ = [("x", _dp), ("y", _dp), ("z", _dp), ("m", C.c_int32), ("n", C.c_int32),
                ("threshold", C.c_double), ("maxresid", C.c_double),
                ("from_average", C.c_int32), ("iteration", C.c_int64)]


class _Result(C.Structure):
    _fields_ = [("stop", C.c_int32), ("iterations", C.c_int64), ("restarts", C.c_int64),
                ("error_iteration", C.c_int64), ("seconds", C.c_double), ("report", _Report),
                ("norm_estimate", C.c_double), ("omega", C.c_double), ("tau", C.c_double),
                ("sigma", C.c_double), ("setup_seconds", C.c_double),
                ("loop_seconds", C.c_double), ("kernel_launches", C.c_int64)]


_SINK = C.CFUNCTYPE(None, C.POINTER(_Snapshot), C.c_void_p)
_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class _HostComm(C.Structure):
    _fields_ = [("allgather", _ALLGATHER), ("user", C.c_void_p)]
_LOG = C.CFUNCTYPE(None, C.c_char_p, C.c_void_p)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Loads libcclp_cuda.so; raises if it was not built (no fallback)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(f"{path} is missing: build it with "
                               "`python -m paper_2510_24429_b200.build` (no CPU fallback)")
        L = C.CDLL(path)
        L.cclp_cu_last_error.restype = C.c_char_p
        L.cclp_cu_stop_string.restype = C.c_char_p
        L.cclp_cu_stop_string.argtypes = [C.c_int32]
        L.cclp_cu_default_config.argtypes = [C.POINTER(_Config)]
        L.cclp_cu_default_tolerances.argtypes = [C.POINTER(_Tol)]
        L.cclp_cu_create.argtypes = [C.POINTER(_LP), C.c_int, C.POINTER(C.c_void_p)]
        L.cclp_cu_destroy.argtypes = [C.c_void_p]
        L.cclp_cu_request_cancel.argtypes = [C.c_void_p]
        L.cclp_cu_sharded_request_cancel.argtypes = [C.c_void_p]
        L.cclp_cu_price.argtypes = [C.c_void_p, _dp, C.c_char_p, C.c_void_p, C.c_int32, C.c_double,
                                     C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_double)]
        L.cclp_cu_relative_report.argtypes = [C.c_void_p, _dp, _dp, _dp, C.POINTER(_Report),
                                               C.POINTER(C.c_double)]
        L.cclp_cu_create_from_file.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p),
                                               C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.cclp_cu_solve.argtypes = [C.c_void_p, C.POINTER(_Config), C.POINTER(_Tol), _dp, C.c_int32,
                                    _SINK, C.c_void_p, C.POINTER(C.c_uint8), _LOG, C.c_void_p,
                                    _dp, _dp, _dp, C.POINTER(_Result)]
        L.cclp_cu_matvec.argtypes = [C.c_void_p, _dp, _dp]
        L.cclp_cu_matvec_transpose.argtypes = [C.c_void_p, _dp, _dp]
        L.cclp_cu_ruiz.argtypes = [C.c_void_p, C.c_int32, _dp, _dp]
        L.cclp_cu_estimate_norm.argtypes = [C.c_void_p, C.c_int32, C.c_uint64, _dp]
        L.cclp_cu_begin.argtypes = [C.c_void_p, C.POINTER(_Config), C.POINTER(_Tol)]
        L.cclp_cu_advance.argtypes = [C.c_void_p, C.c_int64, _dp]
        L.cclp_cu_profile_kernels.argtypes = [C.c_void_p, C.c_int64, _dp]
        L.cclp_cu_phase_profile.argtypes = [C.c_void_p, _dp, C.POINTER(C.c_int64)]
        L.cclp_cu_stream.restype = C.c_void_p
        L.cclp_cu_stream.argtypes = [C.c_void_p]
        L.cclp_cu_describe.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]
        L.cclp_cu_gaussian_start.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.cclp_cu_gaussian_start.restype = None
        L.cclp_cu_partition.argtypes = [_ip, C.c_int32, C.c_int32, _ip]
        L.cclp_cu_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
        L.cclp_cu_sharded_create.argtypes = [C.POINTER(_LP), C.c_int, C.c_int32, C.c_int32, C.c_int32,
                                             C.POINTER(C.c_uint8), C.POINTER(C.c_void_p)]
        L.cclp_cu_sharded_solve.argtypes = [C.c_void_p, C.POINTER(_Config), C.POINTER(_Tol), _dp,
                                            C.c_int32, _SINK, C.c_void_p, C.POINTER(C.c_uint8), _dp,
                                            _dp, _dp, C.POINTER(_Result)]
        L.cclp_cu_sharded_begin.argtypes = [C.c_void_p, C.POINTER(_Config), C.POINTER(_Tol)]
        L.cclp_cu_sharded_advance.argtypes = [C.c_void_p, C.c_int64, _dp]
        L.cclp_cu_sharded_describe.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int32]
        L.cclp_cu_sharded_destroy.argtypes = [C.c_void_p]
        L.cclp_cu_sharded_create_hostcomm.argtypes = [C.POINTER(_LP), C.c_int, C.c_int32, C.c_int32,
                                                      C.POINTER(_HostComm), C.POINTER(C.c_void_p)]
        _lib = L
        return L


EXPORTED_SYMBOLS = [
    "cclp_cu_last_error", "cclp_cu_stop_string", "cclp_cu_default_config",
    "cclp_cu_default_tolerances", "cclp_cu_create", "cclp_cu_destroy", "cclp_cu_solve",
    "cclp_cu_run_pdhg", "cclp_cu_matvec", "cclp_cu_matvec_transpose", "cclp_cu_ruiz",
    "cclp_cu_estimate_norm", "cclp_cu_begin", "cclp_cu_advance", "cclp_cu_profile_kernels", "cclp_cu_phase_profile",
    "cclp_cu_stream", "cclp_cu_describe", "cclp_cu_gaussian_start", "cclp_cu_partition",
    "cclp_cu_nccl_unique_id", "cclp_cu_sharded_create", "cclp_cu_sharded_solve",
    "cclp_cu_sharded_begin", "cclp_cu_sharded_advance", "cclp_cu_sharded_describe",
    "cclp_cu_sharded_destroy", "cclp_cu_sharded_create_hostcomm", "cclp_cu_create_from_file",
    "cclp_cu_relative_report", "cclp_cu_price", "cclp_cu_request_cancel",
    "cclp_cu_sharded_request_cancel",
]


# Host phase timings reported by cclp_cu_describe (context.cuh, Context::phase).
PHASES = ["upload", "csr_build", "partition_tune", "norms", "ruiz", "scale_values", "power_norm",
          "init_check0", "graph_build", "loop", "result_download"]


class PdhgStopReason(enum.IntEnum):
    """pdhg.hpp:44-51."""
    kConverged = 0
    kIterationLimit = 1
    kTimeLimit = 2
    kCancelled = 3
    kWonByCrossover = 4
    kNumericalError = 5


_STOP_STRINGS = ["converged", "iteration-limit", "time-limit", "cancelled", "won-by-crossover",
                 "numerical-error"]


def to_string(reason: PdhgStopReason) -> str:
    """pdhg.cpp:28-44."""
    return _STOP_STRINGS[int(reason)] if 0 <= int(reason) < 6 else "unknown"


@dataclasses.dataclass
class PdhgConfig:
    """pdhg.hpp:29-42 (+ engine knobs: poll_interval = iterations per device
    batch; exact_spmv = reference-order SpMV sums, bit-identical products)."""
    step_scale: float = 0.9
    primal_weight: float = 0.0
    restart_factor: float = 0.5
    norm_iterations: int = 100
    scaling_iterations: int = 10
    max_iterations: int = 2_000_000
    time_limit: float = float("inf")
    check_interval: int = 1
    seed: int = 0
    log_interval: int = 0
    log: Optional[Callable[[str], None]] = None
    deterministic: bool = True
    poll_interval: int = 0
    exact_spmv: bool = False

    def _c(self) -> _Config:
        return _Config(self.step_scale, self.primal_weight, self.restart_factor, self.time_limit,
                       self.norm_iterations, self.scaling_iterations, self.max_iterations,
                       self.check_interval, self.seed, self.log_interval,
                       1 if self.deterministic else 0, self.poll_interval,
                       1 if self.exact_spmv else 0)


@dataclasses.dataclass
class Tolerances:
    """kkt.hpp:32-41."""
    eps_rel: float = 1e-6
    eps_abs: float = 1e-6
    eps_cross: float = 1e-2
    decrement: float = 0.1

    def validate(self) -> None:
        """kkt.cpp:26-37."""
        if not (0.0 < self.decrement < 1.0):
            raise ValueError("tolerances: decrement must be in (0,1)")
        if not (self.eps_rel > 0.0 and self.eps_rel <= self.eps_cross):
            raise ValueError("tolerances: need 0 < eps_rel <= eps_cross")
        if not self.eps_abs > 0.0:
            raise ValueError("tolerances: eps_abs must be positive")


@dataclasses.dataclass
class ResidualReport:
    """kkt.hpp:43-58."""
    rp_norm2: float = 0.0
    rd_norm2: float = 0.0
    rp_inf: float = 0.0
    rd_inf: float = 0.0
    primal_objective: float = 0.0
    dual_objective: float = 0.0
    gap_abs: float = 0.0
    rel_primal: float = 0.0
    rel_dual: float = 0.0
    rel_gap: float = 0.0
    maxresid_rel: float = 0.0
    complementarity: float = 0.0

    def to_json(self) -> str:
        import json
        return json.dumps(dataclasses.asdict(self))


@dataclasses.dataclass
class Iterate:
    """kkt.hpp:25-30."""
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    k: int = 0


@dataclasses.dataclass
class PdhgSnapshot:
    """pdhg.hpp:111-117."""
    iterate: Iterate
    threshold: float
    maxresid: float
    from_average: bool
    iteration: int


@dataclasses.dataclass
class PdhgResult:
    """pdhg.hpp:121-129, plus engine diagnostics."""
    iterate: Iterate
    report: ResidualReport
    stop: PdhgStopReason
    iterations: int
    restarts: int
    seconds: float
    error_iteration: int = -1
    norm_estimate: float = 0.0
    omega: float = 0.0
    tau: float = 0.0
    sigma: float = 0.0
    setup_seconds: float = 0.0
    loop_seconds: float = 0.0
    kernel_launches: int = 0


def _check(L, rc: int) -> None:
    if rc == 0:
        return
    msg = L.cclp_cu_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 3:
        raise MemoryError(msg)
    raise RuntimeError(msg)


class Engine:
    """A device-resident LP (cclp_cu_ctx): upload + CSR build once, then
    solves, kernel-level calls and measurement hooks."""

    def __init__(self, lp: LinearProgram, device: int = 0):
        self.L = load_library()
        self.lp = lp
        self._keep = dict(colptr=np.ascontiguousarray(lp.colptr, np.int32),
                          rowind=np.ascontiguousarray(lp.rowind, np.int32),
                          val=np.ascontiguousarray(lp.val, np.float64),
                          c=np.ascontiguousarray(lp.c, np.float64),
                          rl=np.ascontiguousarray(lp.row_lower, np.float64),
                          ru=np.ascontiguousarray(lp.row_upper, np.float64),
                          cl=np.ascontiguousarray(lp.col_lower, np.float64),
                          cu=np.ascontiguousarray(lp.col_upper, np.float64))
        k = self._keep
        d = lambda a: a.ctypes.data_as(_dp)  # noqa: E731
        i = lambda a: a.ctypes.data_as(_ip)  # noqa: E731
        self._lp = _LP(lp.m, lp.n, i(k["colptr"]), i(k["rowind"]), d(k["val"]), d(k["c"]),
                       d(k["rl"]), d(k["ru"]), d(k["cl"]), d(k["cu"]))
        self.ctx = C.c_void_p()
        _check(self.L, self.L.cclp_cu_create(C.byref(self._lp), device, C.byref(self.ctx)))

    @classmethod
    def from_file(cls, path: str, device: int = 0) -> "Engine":
        """LP ingest from a binary CSC file (lp.write_cscb): mapped and streamed
        to the device by the engine; the host keeps only a memory map."""
        from .lp import read_cscb
        self = cls.__new__(cls)
        self.L = load_library()
        self.lp = read_cscb(path)
        self._keep = {}
        self.ctx = C.c_void_p()
        m, n = C.c_int32(), C.c_int32()
        _check(self.L, self.L.cclp_cu_create_from_file(path.encode(), device, C.byref(self.ctx),
                                                       C.byref(m), C.byref(n)))
        return self

    def relative_report(self, x, y, z):
        """relative_report and absolute_violation (kkt.cpp:106-149) of the
        iterate on this (equality-form, unscaled) LP, computed on the device.
        Returns (ResidualReport, absolute_violation)."""
        xs = [np.ascontiguousarray(a, np.float64) for a in (x, y, z)]
        rep, av = _Report(), C.c_double()
        _check(self.L, self.L.cclp_cu_relative_report(self.ctx, *(a.ctypes.data_as(_dp) for a in xs),
                                                      C.byref(rep), C.byref(av)))
        return ResidualReport(**{f: getattr(rep, f) for f in REPORT_FIELDS}), av.value

    def price(self, y, status, skip=None, phase1: bool = False, dtol: float = 1e-9, bland: bool = False):
        """price() of the reference's simplex (simplex.cpp:266-296) on the
        device. `status`: n+m ColStatus chars (bytes or str) over the
        structural then logical columns; `skip`: optional n+m booleans.
        Returns (entering or -1, direction, violation)."""
        yv = np.ascontiguousarray(y, np.float64)
        st = status.encode() if isinstance(status, str) else bytes(status)
        sk = None if skip is None else np.ascontiguousarray(skip, np.uint8)
        e, d, v = C.c_int64(), C.c_int32(), C.c_double()
        _check(self.L, self.L.cclp_cu_price(self.ctx, yv.ctypes.data_as(_dp), st,
                                            None if sk is None else sk.ctypes.data_as(C.c_void_p),
                                            int(phase1), dtol, int(bland), C.byref(e), C.byref(d),
                                            C.byref(v)))
        return int(e.value), int(d.value), float(v.value)

    def close(self) -> None:
        if self.ctx:
            self.L.cclp_cu_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- kernel-level -----------------------------------------------------
    def matvec(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.lp.m)
        _check(self.L, self.L.cclp_cu_matvec(self.ctx, x.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
        return out

    def matvec_transpose(self, y) -> np.ndarray:
        y = np.ascontiguousarray(y, np.float64)
        out = np.empty(self.lp.n)
        _check(self.L, self.L.cclp_cu_matvec_transpose(self.ctx, y.ctypes.data_as(_dp),
                                                       out.ctypes.data_as(_dp)))
        return out

    def ruiz(self, iterations: int = 10):
        r, s = np.empty(self.lp.m), np.empty(self.lp.n)
        _check(self.L, self.L.cclp_cu_ruiz(self.ctx, iterations, r.ctypes.data_as(_dp),
                                           s.ctypes.data_as(_dp)))
        return r, s

    def estimate_norm(self, iterations: int = 100, seed: int = 0) -> float:
        out = C.c_double()
        _check(self.L, self.L.cclp_cu_estimate_norm(self.ctx, iterations, seed, C.byref(out)))
        return out.value

    # ---- solve --------------------------------------------------------------
    def solve(self, config: Optional[PdhgConfig] = None, tol: Optional[Tolerances] = None,
              thresholds: Sequence[float] = (), sink=None, cancel=None) -> PdhgResult:
        config = config or PdhgConfig()
        tol = tol or Tolerances()
        lp = self.lp
        thr = np.ascontiguousarray(list(thresholds), np.float64)
        x, y, z = np.empty(lp.n), np.empty(lp.m), np.empty(lp.n)
        res = _Result()
        errors = []

        def _sink(sp, _u):
            try:
                s = sp.contents
                it = Iterate(np.ctypeslib.as_array(s.x, (lp.n,)).copy() if lp.n else np.empty(0),
                             np.ctypeslib.as_array(s.y, (lp.m,)).copy() if lp.m else np.empty(0),
                             np.ctypeslib.as_array(s.z, (lp.n,)).copy() if lp.n else np.empty(0),
                             int(s.iteration))
                if sink is not None:
                    sink(PdhgSnapshot(it, s.threshold, s.maxresid, bool(s.from_average),
                                      int(s.iteration)))
            except BaseException as e:  # stop the loop now, re-raise after the solve
                errors.append(e)
                self.L.cclp_cu_request_cancel(self.ctx)

        def _log(line, _u):
            if config.log is not None:
                config.log(line.decode())

        cb = _SINK(_sink)
        lg = _LOG(_log)
        flag = cancel if cancel is not None else (C.c_uint8 * 1)(0)
        rc = self.L.cclp_cu_solve(self.ctx, C.byref(config._c()), C.byref(_Tol(
            tol.eps_rel, tol.eps_abs, tol.eps_cross, tol.decrement)),
            thr.ctypes.data_as(_dp) if thr.size else None, thr.size, cb, None,
            C.cast(flag, C.POINTER(C.c_uint8)), lg, None, x.ctypes.data_as(_dp),
            y.ctypes.data_as(_dp), z.ctypes.data_as(_dp), C.byref(res))
        _check(self.L, rc)
        if errors:
            raise errors[0]
        rep = ResidualReport(**{f: getattr(res.report, f) for f in REPORT_FIELDS})
        return PdhgResult(Iterate(x, y, z, int(res.iterations)), rep,
                          PdhgStopReason(res.stop), int(res.iterations), int(res.restarts),
                          float(res.seconds), int(res.error_iteration), res.norm_estimate,
                          res.omega, res.tau, res.sigma, res.setup_seconds, res.loop_seconds,
                          int(res.kernel_launches))

    # ---- measurement hooks ------------------------------------------------
    def begin(self, config: Optional[PdhgConfig] = None, tol: Optional[Tolerances] = None):
        config = config or PdhgConfig()
        tol = tol or Tolerances()
        _check(self.L, self.L.cclp_cu_begin(self.ctx, C.byref(config._c()), C.byref(_Tol(
            tol.eps_rel, tol.eps_abs, tol.eps_cross, tol.decrement))))

    def advance(self, iters: int) -> float:
        ms = C.c_double()
        _check(self.L, self.L.cclp_cu_advance(self.ctx, iters, C.byref(ms)))
        return ms.value

    def profile_kernels(self, iters: int) -> dict:
        """Average ms per launch of the four iteration kernels."""
        out = (C.c_double * 4)()
        _check(self.L, self.L.cclp_cu_profile_kernels(self.ctx, iters, out))
        return dict(zip(["spmv_rows", "dual", "spmv_cols", "primal"], list(out)))

    def phase_profile(self) -> dict:
        """Median microseconds per step of rows / dual / cols / primal as they
        ran inside the loop's CUDA graphs (in-kernel %globaltimer stamps of the
        last 128 steps), plus the number of steps they cover."""
        out = (C.c_double * 4)()
        steps = C.c_int64()
        _check(self.L, self.L.cclp_cu_phase_profile(self.ctx, out, C.byref(steps)))
        d = dict(zip(["spmv_rows", "dual", "spmv_cols", "primal"], list(out)))
        d["steps"] = steps.value
        return d

    def stream_ptr(self) -> int:
        return int(self.L.cclp_cu_stream(self.ctx) or 0)

    def describe(self) -> dict:
        keys = ["m", "n", "nnz", "group_rows", "group_cols", "spmv_rows_grid_x10_rpg",
                "spmv_cols_grid_x10_rpg", "launches",
                "last_cols_body_ns", "last_finalize_ns"]
        out = (C.c_int64 * (len(keys) + len(PHASES) + 3))()
        self.L.cclp_cu_describe(self.ctx, out, len(out))
        d = dict(zip(keys, list(out)))
        d["phase_seconds"] = {k: out[len(keys) + i] * 1e-9 for i, k in enumerate(PHASES)}
        d["sell_rows_block"] = int(out[len(keys) + len(PHASES)])  # 0: CSR-G row kernel
        d["sell_cols_block"] = int(out[len(keys) + len(PHASES) + 1])
        d["speculative_rows"] = bool(out[len(keys) + len(PHASES) + 2])  # row_step after begin()
        return d


def gaussian_start(seed: int, n: int) -> np.ndarray:
    """The power iteration's start vector (pdhg.cpp:49-52), host-side."""
    L = load_library()
    v = np.empty(n)
    L.cclp_cu_gaussian_start(seed, n, v.ctypes.data_as(_dp))
    return v


def partition(ptr, parts: int) -> np.ndarray:
    """The nnz-balanced split of rows used for the shards (host only)."""
    L = load_library()
    ptr = np.ascontiguousarray(ptr, np.int32)
    out = np.empty(parts + 1, np.int32)
    _check(L, L.cclp_cu_partition(ptr.ctypes.data_as(_ip), ptr.size - 1, parts,
                                  out.ctypes.data_as(_ip)))
    return out


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0), to be broadcast to the other ranks."""
    L = load_library()
    buf = (C.c_uint8 * 128)()
    _check(L, L.cclp_cu_nccl_unique_id(buf))
    return bytes(buf)


class ShardedEngine:
    """Row-block sharded solve (cclp_cu_sharded).

    nranks == 1: `nshards` shards in this process on `device` (exchanges by
    device copies); nranks > 1: one shard per process over NCCL, `nccl_id`
    from rank 0's nccl_unique_id(); or, with `host_allgather(bytes) -> [bytes
    per rank]` (e.g. over torch.distributed gloo), one shard per process with
    the push transport over CUDA IPC and no NCCL."""

    def __init__(self, lp: LinearProgram, nshards: int = 1, device: int = 0, rank: int = 0,
                 nranks: int = 1, nccl_id: Optional[bytes] = None, host_allgather=None):
        self.L = load_library()
        self.lp = lp
        self._keep = dict(colptr=np.ascontiguousarray(lp.colptr, np.int32),
                          rowind=np.ascontiguousarray(lp.rowind, np.int32),
                          val=np.ascontiguousarray(lp.val, np.float64),
                          c=np.ascontiguousarray(lp.c, np.float64),
                          rl=np.ascontiguousarray(lp.row_lower, np.float64),
                          ru=np.ascontiguousarray(lp.row_upper, np.float64),
                          cl=np.ascontiguousarray(lp.col_lower, np.float64),
                          cu=np.ascontiguousarray(lp.col_upper, np.float64))
        k = self._keep
        d = lambda a: a.ctypes.data_as(_dp)  # noqa: E731
        i = lambda a: a.ctypes.data_as(_ip)  # noqa: E731
        self._lp = _LP(lp.m, lp.n, i(k["colptr"]), i(k["rowind"]), d(k["val"]), d(k["c"]),
                       d(k["rl"]), d(k["ru"]), d(k["cl"]), d(k["cu"]))
        idbuf = None
        if nccl_id is not None:
            idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        self.ctx = C.c_void_p()
        if host_allgather is not None:
            # host_allgather(bytes) -> list of bytes objects, one per rank (rank order)
            def _ag(inp, nbytes, out, _u):
                try:
                    parts = host_allgather(C.string_at(inp, nbytes))
                    blob = b"".join(parts)
                    C.memmove(out, blob, len(blob))
                    return 0
                except Exception:
                    return 1
            self._ag = _ALLGATHER(_ag)
            self._hc = _HostComm(self._ag, None)
            _check(self.L, self.L.cclp_cu_sharded_create_hostcomm(
                C.byref(self._lp), device, rank, nranks, C.byref(self._hc), C.byref(self.ctx)))
            return
        _check(self.L, self.L.cclp_cu_sharded_create(C.byref(self._lp), device, nshards, rank,
                                                     nranks, idbuf, C.byref(self.ctx)))

    def close(self) -> None:
        if self.ctx:
            self.L.cclp_cu_sharded_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def describe(self) -> dict:
        out = (C.c_int64 * 256)()
        self.L.cclp_cu_sharded_describe(self.ctx, out, 256)
        P = int(out[0])
        rb = list(out[1:P + 2])
        cb = list(out[P + 2:2 * P + 3])
        o = 2 * P + 3
        nloc = int(out[o + 5])
        local = [dict(rank=int(out[o + 6 + 3 * k]), nnz_rows=int(out[o + 7 + 3 * k]),
                      nnz_cols=int(out[o + 8 + 3 * k])) for k in range(nloc)]
        return dict(shards=P, row_bounds=rb, col_bounds=cb, launches=int(out[o]),
                    halo_x=bool(out[o + 1]), halo_x_volume=int(out[o + 2]),
                    halo_y=bool(out[o + 3]), halo_y_volume=int(out[o + 4]), local_shards=local)

    def solve(self, config: Optional[PdhgConfig] = None, tol: Optional[Tolerances] = None,
              thresholds: Sequence[float] = (), sink=None, cancel=None) -> PdhgResult:
        config = config or PdhgConfig()
        tol = tol or Tolerances()
        lp = self.lp
        thr = np.ascontiguousarray(list(thresholds), np.float64)
        x, y, z = np.empty(lp.n), np.empty(lp.m), np.empty(lp.n)
        res = _Result()
        errors = []

        def _sink(sp, _u):
            try:
                s = sp.contents
                it = Iterate(np.ctypeslib.as_array(s.x, (lp.n,)).copy() if lp.n else np.empty(0),
                             np.ctypeslib.as_array(s.y, (lp.m,)).copy() if lp.m else np.empty(0),
                             np.ctypeslib.as_array(s.z, (lp.n,)).copy() if lp.n else np.empty(0),
                             int(s.iteration))
                if sink is not None:
                    sink(PdhgSnapshot(it, s.threshold, s.maxresid, bool(s.from_average),
                                      int(s.iteration)))
            except BaseException as e:  # stop the loop now, re-raise after the solve
                errors.append(e)
                self.L.cclp_cu_sharded_request_cancel(self.ctx)

        cb = _SINK(_sink)
        flag = cancel if cancel is not None else (C.c_uint8 * 1)(0)
        rc = self.L.cclp_cu_sharded_solve(
            self.ctx, C.byref(config._c()), C.byref(_Tol(tol.eps_rel, tol.eps_abs, tol.eps_cross,
                                                         tol.decrement)),
            thr.ctypes.data_as(_dp) if thr.size else None, thr.size, cb, None,
            C.cast(flag, C.POINTER(C.c_uint8)), x.ctypes.data_as(_dp), y.ctypes.data_as(_dp),
            z.ctypes.data_as(_dp), C.byref(res))
        _check(self.L, rc)
        if errors:
            raise errors[0]
        rep = ResidualReport(**{f: getattr(res.report, f) for f in REPORT_FIELDS})
        return PdhgResult(Iterate(x, y, z, int(res.iterations)), rep,
                          PdhgStopReason(res.stop), int(res.iterations), int(res.restarts),
                          float(res.seconds), int(res.error_iteration), res.norm_estimate,
                          res.omega, res.tau, res.sigma, res.setup_seconds, res.loop_seconds,
                          int(res.kernel_launches))

    def begin(self, config: Optional[PdhgConfig] = None, tol: Optional[Tolerances] = None):
        config = config or PdhgConfig()
        tol = tol or Tolerances()
        _check(self.L, self.L.cclp_cu_sharded_begin(self.ctx, C.byref(config._c()), C.byref(
            _Tol(tol.eps_rel, tol.eps_abs, tol.eps_cross, tol.decrement))))

    def advance(self, iters: int) -> float:
        ms = C.c_double()
        _check(self.L, self.L.cclp_cu_sharded_advance(self.ctx, iters, C.byref(ms)))
        return ms.value


def run_pdhg_sharded(std_lp: LinearProgram, nshards: int, config: Optional[PdhgConfig] = None,
                     tol: Optional[Tolerances] = None, thresholds: Sequence[float] = (),
                     sink=None, cancel=None, device: int = 0) -> PdhgResult:
    """run_pdhg over `nshards` row-block shards in this process (one GPU)."""
    if not std_lp.all_rows_equality():
        raise ValueError("run_pdhg: LP must be in equality form")
    (tol or Tolerances()).validate()
    with ShardedEngine(std_lp, nshards, device) as eng:
        return eng.solve(config, tol, thresholds, sink, cancel)


def run_pdhg(std_lp: LinearProgram, config: Optional[PdhgConfig] = None,
             tol: Optional[Tolerances] = None, thresholds: Sequence[float] = (),
             sink: Optional[Callable[[PdhgSnapshot], None]] = None, cancel=None,
             device: int = 0) -> PdhgResult:
    """cclp::run_pdhg (pdhg.hpp:138-142) on the B200 engine."""
    if not std_lp.all_rows_equality():
        raise ValueError("run_pdhg: LP must be in equality form")
    (tol or Tolerances()).validate()
    with Engine(std_lp, device) as eng:
        return eng.solve(config, tol, thresholds, sink, cancel)
