"""ctypes bindings to the CPU oracle — TEST INFRASTRUCTURE ONLY.

Two checkers, both CPU:
  * `Restatement` -> oracle/liboracle.so: the plain-C restatement
    (cclp_oracle.c) of the reference's run_pdhg path; builds from this repo
    alone, so it is available on the GPU box.
  * `Reference`   -> oracle/_ref/libcclp_ref.so: the reference's own sources
    (/root/reference/proj/src/*.cpp) compiled here against the Eigen-API shim
    (oracle/Makefile). Present wherever it was built and shipped.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcclp_ref.so")

STOP_NAMES = ["converged", "iteration-limit", "time-limit", "cancelled", "won-by-crossover",
              "numerical-error"]
REPORT_FIELDS = ["rp_norm2", "rd_norm2", "rp_inf", "rd_inf", "primal_objective",
                 "dual_objective", "gap_abs", "rel_primal", "rel_dual", "rel_gap",
                 "maxresid_rel", "complementarity"]

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(_dp)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int32).ctypes.data_as(_ip)


class _LP(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_int), ("colptr", _ip), ("rowind", _ip), ("val", _dp),
                ("c", _dp), ("row_lower", _dp), ("row_upper", _dp), ("col_lower", _dp),
                ("col_upper", _dp)]


class _Config(C.Structure):
    _fields_ = [("step_scale", C.c_double), ("primal_weight", C.c_double),
                ("restart_factor", C.c_double), ("time_limit", C.c_double),
                ("norm_iterations", C.c_int), ("scaling_iterations", C.c_int),
                ("max_iterations", C.c_int64), ("check_interval", C.c_int),
                ("seed", C.c_uint64)]


class _Tol(C.Structure):
    _fields_ = [("eps_rel", C.c_double), ("eps_abs", C.c_double), ("eps_cross", C.c_double),
                ("decrement", C.c_double)]


class _Report(C.Structure):
    _fields_ = [(f, C.c_double) for f in REPORT_FIELDS]


class _Snapshot(C.Structure):
    _fields_ = [("threshold", C.c_double), ("maxresid", C.c_double), ("from_average", C.c_int),
                ("iteration", C.c_int64), ("x", _dp), ("y", _dp), ("z", _dp)]


class _Result(C.Structure):
    _fields_ = [("stop", C.c_int), ("iterations", C.c_int64), ("restarts", C.c_int64),
                ("error_iteration", C.c_int64), ("seconds", C.c_double), ("report", _Report),
                ("tau", C.c_double), ("sigma", C.c_double), ("norm_estimate", C.c_double),
                ("omega", C.c_double)]


class _Trace(C.Structure):
    _fields_ = [("restart_iters", _i64p), ("restart_cap", C.c_int64),
                ("n_restarts_logged", C.c_int64), ("trace", _dp), ("trace_cap", C.c_int64),
                ("n_trace", C.c_int64)]


_SINK = C.CFUNCTYPE(None, C.POINTER(_Snapshot), C.c_void_p)

DEFAULT_CONFIG = dict(step_scale=0.9, primal_weight=0.0, restart_factor=0.5,
                      time_limit=float("inf"), norm_iterations=100, scaling_iterations=10,
                      max_iterations=2_000_000, check_interval=1, seed=0)
DEFAULT_TOL = dict(eps_rel=1e-6, eps_abs=1e-6, eps_cross=1e-2, decrement=0.1)


def build_restatement() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "restate"], check=True)


def _keep(lp):
    """Contiguous typed copies that stay alive while ctypes pointers exist."""
    return dict(colptr=np.ascontiguousarray(lp.colptr, np.int32),
                rowind=np.ascontiguousarray(lp.rowind, np.int32),
                val=np.ascontiguousarray(lp.val, np.float64),
                c=np.ascontiguousarray(lp.c, np.float64),
                rl=np.ascontiguousarray(lp.row_lower, np.float64),
                ru=np.ascontiguousarray(lp.row_upper, np.float64),
                cl=np.ascontiguousarray(lp.col_lower, np.float64),
                cu=np.ascontiguousarray(lp.col_upper, np.float64))


class Restatement:
    """The plain-C restatement (liboracle.so)."""

    def __init__(self, path: str = RESTATE_SO):
        if not os.path.exists(path):
            build_restatement()
        self.lib = L = C.CDLL(path)
        L.oracle_dot.restype = C.c_double
        L.oracle_dot.argtypes = [_dp, _dp, C.c_int64]
        L.oracle_norm.restype = C.c_double
        L.oracle_norm.argtypes = [_dp, C.c_int64]
        L.oracle_pow2_sqrt.restype = C.c_double
        L.oracle_pow2_sqrt.argtypes = [C.c_double]
        L.oracle_estimate_norm.restype = C.c_double
        L.oracle_estimate_norm.argtypes = [C.POINTER(_LP), C.c_int, C.c_uint64]
        L.oracle_gaussian_start.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.oracle_matvec.argtypes = [C.POINTER(_LP), _dp, _dp]
        L.oracle_matvec_transpose.argtypes = [C.POINTER(_LP), _dp, _dp]
        L.oracle_ruiz.argtypes = [C.POINTER(_LP), C.c_int, _dp, _dp, _dp]
        L.oracle_relative_report.argtypes = [C.POINTER(_LP), _dp, _dp, _dp, C.POINTER(_Report)]
        L.oracle_run_pdhg.restype = C.c_int
        L.oracle_run_pdhg.argtypes = [C.POINTER(_LP), C.POINTER(_Config), C.POINTER(_Tol), _dp,
                                      C.c_int, _SINK, C.c_void_p, C.POINTER(C.c_uint8), _dp, _dp,
                                      _dp, C.POINTER(_Result), C.POINTER(_Trace)]
        L.oracle_last_error.restype = C.c_char_p

    @staticmethod
    def _lp(lp, keep):
        return _LP(lp.m, lp.n, _i(keep["colptr"]), _i(keep["rowind"]), _d(keep["val"]),
                   _d(keep["c"]), _d(keep["rl"]), _d(keep["ru"]), _d(keep["cl"]), _d(keep["cu"]))

    def matvec(self, lp, x):
        k = _keep(lp)
        out = np.empty(lp.m)
        x = np.ascontiguousarray(x, np.float64)
        self.lib.oracle_matvec(C.byref(self._lp(lp, k)), _d(x), _d(out))
        return out

    def matvec_transpose(self, lp, y):
        k = _keep(lp)
        out = np.empty(lp.n)
        y = np.ascontiguousarray(y, np.float64)
        self.lib.oracle_matvec_transpose(C.byref(self._lp(lp, k)), _d(y), _d(out))
        return out

    def dot(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        return self.lib.oracle_dot(_d(a), _d(b), a.size)

    def norm(self, a):
        a = np.ascontiguousarray(a, np.float64)
        return self.lib.oracle_norm(_d(a), a.size)

    def ruiz(self, lp, iterations=10):
        k = _keep(lp)
        r, s, sv = np.empty(lp.m), np.empty(lp.n), np.empty(max(lp.nnz, 1))
        self.lib.oracle_ruiz(C.byref(self._lp(lp, k)), iterations, _d(r), _d(s), _d(sv))
        return r, s, sv[:lp.nnz]

    def gaussian_start(self, seed, n):
        v = np.empty(n)
        self.lib.oracle_gaussian_start(seed, n, _d(v))
        return v

    def estimate_norm(self, lp, iterations=100, seed=0):
        k = _keep(lp)
        return self.lib.oracle_estimate_norm(C.byref(self._lp(lp, k)), iterations, seed)

    def relative_report(self, lp, x, y, z):
        k = _keep(lp)
        rep = _Report()
        xs = [np.ascontiguousarray(v, np.float64) for v in (x, y, z)]
        self.lib.oracle_relative_report(C.byref(self._lp(lp, k)), _d(xs[0]), _d(xs[1]),
                                        _d(xs[2]), C.byref(rep))
        return {f: getattr(rep, f) for f in REPORT_FIELDS}

    def run_pdhg(self, lp, config=None, tol=None, thresholds=(), cancel=False,
                 trace_cap=0, restart_cap=100000):
        cfg = dict(DEFAULT_CONFIG, **(config or {}))
        tl = dict(DEFAULT_TOL, **(tol or {}))
        k = _keep(lp)
        x, y, z = np.empty(lp.n), np.empty(lp.m), np.empty(lp.n)
        thr = np.ascontiguousarray(thresholds, np.float64)
        snaps = []

        def sink(sp, _user):
            s = sp.contents
            snaps.append(dict(threshold=s.threshold, maxresid=s.maxresid,
                              from_average=bool(s.from_average), iteration=s.iteration,
                              x=np.ctypeslib.as_array(s.x, (lp.n,)).copy(),
                              y=np.ctypeslib.as_array(s.y, (lp.m,)).copy() if lp.m else np.empty(0),
                              z=np.ctypeslib.as_array(s.z, (lp.n,)).copy()))
        cb = _SINK(sink)
        res = _Result()
        rit = np.zeros(max(restart_cap, 1), np.int64)
        tr = np.zeros(3 * max(trace_cap, 1))
        trace = _Trace(rit.ctypes.data_as(_i64p), restart_cap, 0, _d(tr), trace_cap, 0)
        flag = (C.c_uint8 * 1)(1 if cancel else 0)
        rc = self.lib.oracle_run_pdhg(C.byref(self._lp(lp, k)), C.byref(_Config(**cfg)),
                                      C.byref(_Tol(**tl)), _d(thr) if thr.size else None,
                                      thr.size, cb, None, flag, _d(x), _d(y), _d(z),
                                      C.byref(res), C.byref(trace))
        if rc != 0:
            raise ValueError(self.lib.oracle_last_error().decode())
        return dict(x=x, y=y, z=z, stop=STOP_NAMES[res.stop], iterations=res.iterations,
                    restarts=res.restarts, error_iteration=res.error_iteration,
                    seconds=res.seconds,
                    report={f: getattr(res.report, f) for f in REPORT_FIELDS},
                    tau=res.tau, sigma=res.sigma, norm_estimate=res.norm_estimate,
                    omega=res.omega, snapshots=snaps,
                    restart_iters=rit[:trace.n_restarts_logged].copy(),
                    trace=tr[:3 * trace.n_trace].reshape(-1, 3).copy())


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The reference's own run_pdhg, built by oracle/Makefile into _ref/."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        self.lib = L = C.CDLL(path)
        L.cclp_ref_last_error.restype = C.c_char_p
        csc = [C.c_int, C.c_int, _ip, _ip, _dp]
        lpargs = csc + [_dp, _dp, _dp, _dp, _dp]
        L.cclp_ref_matvec.argtypes = csc + [_dp, _dp]
        L.cclp_ref_matvec_transpose.argtypes = csc + [_dp, _dp]
        L.cclp_ref_estimate_norm.argtypes = csc + [C.c_int, C.c_uint64, _dp]
        L.cclp_ref_ruiz.argtypes = lpargs + [C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.cclp_ref_relative_report.argtypes = lpargs + [_dp, _dp, _dp, _dp]
        L.cclp_ref_run_pdhg.argtypes = lpargs + [_dp, _i64p, _dp, _dp, C.c_int,
                                                 C.POINTER(C.c_uint8), _dp, _dp, _dp, _dp, _i64p,
                                                 _dp, _dp, _dp, _dp, _dp, _ip]

    def _check(self, rc):
        if rc == 1:
            raise ValueError(self.lib.cclp_ref_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.lib.cclp_ref_last_error().decode())

    @staticmethod
    def _csc(lp, k):
        return [lp.m, lp.n, _i(k["colptr"]), _i(k["rowind"]), _d(k["val"])]

    @classmethod
    def _lpargs(cls, lp, k):
        return cls._csc(lp, k) + [_d(k["c"]), _d(k["rl"]), _d(k["ru"]), _d(k["cl"]), _d(k["cu"])]

    def matvec(self, lp, x):
        k = _keep(lp)
        out = np.empty(lp.m)
        x = np.ascontiguousarray(x, np.float64)
        self._check(self.lib.cclp_ref_matvec(*self._csc(lp, k), _d(x), _d(out)))
        return out

    def matvec_transpose(self, lp, y):
        k = _keep(lp)
        out = np.empty(lp.n)
        y = np.ascontiguousarray(y, np.float64)
        self._check(self.lib.cclp_ref_matvec_transpose(*self._csc(lp, k), _d(y), _d(out)))
        return out

    def estimate_norm(self, lp, iterations=100, seed=0):
        k = _keep(lp)
        out = (C.c_double * 1)()
        self._check(self.lib.cclp_ref_estimate_norm(*self._csc(lp, k), iterations, seed, out))
        return out[0]

    def ruiz(self, lp, iterations=10):
        k = _keep(lp)
        r, s, sv = np.empty(lp.m), np.empty(lp.n), np.empty(max(lp.nnz, 1))
        sc, sb = np.empty(lp.n), np.empty(lp.m)
        self._check(self.lib.cclp_ref_ruiz(*self._lpargs(lp, k), iterations, _d(r), _d(s),
                                           _d(sv), _d(sc), _d(sb)))
        return r, s, sv[:lp.nnz]

    def relative_report(self, lp, x, y, z):
        k = _keep(lp)
        rep = np.empty(12)
        xs = [np.ascontiguousarray(v, np.float64) for v in (x, y, z)]
        self._check(self.lib.cclp_ref_relative_report(*self._lpargs(lp, k), _d(xs[0]),
                                                      _d(xs[1]), _d(xs[2]), _d(rep)))
        return dict(zip(REPORT_FIELDS, rep.tolist()))

    def run_pdhg(self, lp, config=None, tol=None, thresholds=(), cancel=False,
                 keep_snapshots=True):
        cfg = dict(DEFAULT_CONFIG, **(config or {}))
        tl = dict(DEFAULT_TOL, **(tol or {}))
        k = _keep(lp)
        dcfg = np.array([cfg["step_scale"], cfg["primal_weight"], cfg["restart_factor"],
                         cfg["time_limit"]])
        icfg = np.array([cfg["norm_iterations"], cfg["scaling_iterations"],
                         cfg["max_iterations"], cfg["check_interval"], cfg["seed"]], np.int64)
        tolv = np.array([tl["eps_rel"], tl["eps_abs"], tl["eps_cross"], tl["decrement"]])
        thr = np.ascontiguousarray(thresholds, np.float64)
        nt = thr.size
        x, y, z = np.empty(lp.n), np.empty(lp.m), np.empty(lp.n)
        rep = np.empty(12)
        stats = np.zeros(4, np.int64)
        secs = np.zeros(1)
        ks = nt if keep_snapshots else 0
        sx, sy, sz = np.empty(max(ks * lp.n, 1)), np.empty(max(ks * lp.m, 1)), np.empty(max(ks * lp.n, 1))
        meta = np.empty(4 * max(nt, 1))
        ns = (C.c_int * 1)()
        flag = (C.c_uint8 * 1)(1 if cancel else 0)
        self._check(self.lib.cclp_ref_run_pdhg(
            *self._lpargs(lp, k), _d(dcfg), icfg.ctypes.data_as(_i64p), _d(tolv),
            _d(thr) if nt else None, nt, flag, _d(x), _d(y), _d(z), _d(rep),
            stats.ctypes.data_as(_i64p), _d(secs), _d(sx) if ks else None,
            _d(sy) if ks else None, _d(sz) if ks else None, _d(meta), ns))
        snaps = []
        for i in range(ns[0]):
            s = dict(threshold=meta[4 * i], maxresid=meta[4 * i + 1],
                     from_average=bool(meta[4 * i + 2]), iteration=int(meta[4 * i + 3]))
            if ks:
                s.update(x=sx[i * lp.n:(i + 1) * lp.n].copy(), y=sy[i * lp.m:(i + 1) * lp.m].copy(),
                         z=sz[i * lp.n:(i + 1) * lp.n].copy())
            snaps.append(s)
        return dict(x=x, y=y, z=z, stop=STOP_NAMES[stats[0]], iterations=int(stats[1]),
                    restarts=int(stats[2]), error_iteration=int(stats[3]), seconds=float(secs[0]),
                    report=dict(zip(REPORT_FIELDS, rep.tolist())), snapshots=snaps)
