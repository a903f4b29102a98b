"""Command-line front end (SPEC.md "[MODULE] bench_cli") over
cclp::run_race with the B200 run_pdhg:

  python -m integration.cli solve <model.mps[.gz]|model.cscb> [--mode baseline|concurrent]
      [--eps-rel 1e-6] [--eps-cross 1e-2] [--eps-abs 1e-6] [--decrement 0.1]
      [--workers 4] [--time-limit 3600] [--seed S] [--write-basis FILE]
      [--write-solution FILE] [--json] [--pdhg gpu|cpu]
  python -m integration.cli bench <dir> [same flags] [--shift 1.0]
      [--out report.json] [--csv report.csv]

Exit codes (SPEC): 0 solved, 2 time limit, 3 numerical failure, 4 input
error. `bench` runs every model in baseline and concurrent mode, one after
the other, and reports shifted geometric means (shift 1 s), the performance
ratio baseline/concurrent, wins / losses / ties at +-10%, and the histogram
of winning launch thresholds ("main" last). Time-limit runs enter the means
at the limit value (SPEC design decision)."""
from __future__ import annotations

import argparse
import csv
import ctypes as C
import io
import json
import math
import os
import sys
import time

from integration import race

EXIT_SOLVED, EXIT_TIME, EXIT_NUMERIC, EXIT_INPUT = 0, 2, 3, 4


def shifted_geomean(times, shift: float = 1.0) -> float:
    """exp(mean(ln(t_i + shift))) - shift (SPEC; achterberg07)."""
    times = list(times)
    if not times:
        raise ValueError("shifted_geomean of an empty list")
    if shift <= 0 or any(t < 0 for t in times):
        raise ValueError("shifted_geomean needs times >= 0 and shift > 0")
    return math.exp(sum(math.log(t + shift) for t in times) / len(times)) - shift


def classify_win_loss(baseline: float, candidate: float) -> str:
    """win if candidate <= 0.9 baseline, loss if >= 1.1 baseline, else tie."""
    if candidate <= 0.9 * baseline:
        return "win"
    if candidate >= 1.1 * baseline:
        return "loss"
    return "tie"


def solve_file(path: str, mode: str = "concurrent", eps_rel=1e-6, eps_cross=1e-2, eps_abs=1e-6,
               decrement=0.1, workers=4, time_limit=3600.0, seed=0, basis_out="",
               solution_out="", pdhg="gpu"):
    """Returns (exit code, outcome dict or error string)."""
    L = race.lib(pdhg)
    L.cclp_race_solve_file.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_double, C.c_int, C.c_double, C.c_ulonglong, C.c_char_p,
                                       C.c_char_p, C.c_char_p, C.c_int]
    buf = C.create_string_buffer(1 << 20)
    t = time.perf_counter()
    rc = L.cclp_race_solve_file(path.encode(), 1 if mode == "concurrent" else 0, eps_rel, eps_cross,
                                eps_abs, decrement, workers, time_limit, seed, basis_out.encode(),
                                solution_out.encode(), buf, 1 << 20)
    wall = time.perf_counter() - t
    if rc == EXIT_INPUT:
        return rc, L.cclp_race_last_error().decode()
    out = json.loads(buf.value.decode()) if buf.value else {}
    out["cli_wall_s"] = wall
    return rc, out


def write_mps(lp, path: str, name: str = "LP", pdhg: str = "cpu") -> None:
    """The reference's write_mps (mps.hpp:50) for an LP in arrays."""
    import numpy as np
    L = race.lib(pdhg)
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
    L.cclp_race_write_mps.argtypes = [C.c_int, C.c_int, ip, ip, dp, dp, dp, dp, dp, dp, C.c_char_p,
                                      C.c_char_p]
    k = [np.ascontiguousarray(lp.colptr, np.int32), np.ascontiguousarray(lp.rowind, np.int32)]
    d = [np.ascontiguousarray(a, np.float64) for a in (lp.val, lp.c, lp.row_lower, lp.row_upper,
                                                       lp.col_lower, lp.col_upper)]
    rc = L.cclp_race_write_mps(lp.m, lp.n, k[0].ctypes.data_as(ip), k[1].ctypes.data_as(ip),
                               *[a.ctypes.data_as(dp) for a in d], name.encode(), path.encode())
    if rc != 0:
        raise RuntimeError(L.cclp_race_last_error().decode())


def summarize(records, shift: float = 1.0, time_limit: float = 3600.0) -> dict:
    """BenchSummary from per-(model, mode) records (SPEC bench_cli)."""
    def t_of(r):
        return r["wall_s"] if r["status"] == "solved" else time_limit
    by = {}
    for r in records:
        by.setdefault(r["model"], {})[r["mode"]] = r
    models = sorted(by)
    base = [t_of(by[mdl]["baseline"]) for mdl in models if "baseline" in by[mdl]]
    conc = [t_of(by[mdl]["concurrent"]) for mdl in models if "concurrent" in by[mdl]]
    sgm_b = shifted_geomean(base, shift) if base else None
    sgm_c = shifted_geomean(conc, shift) if conc else None
    wins = losses = ties = 0
    for mdl in models:
        if "baseline" in by[mdl] and "concurrent" in by[mdl]:
            c = classify_win_loss(t_of(by[mdl]["baseline"]), t_of(by[mdl]["concurrent"]))
            wins += c == "win"
            losses += c == "loss"
            ties += c == "tie"
    hist = {}
    for mdl in models:
        r = by[mdl].get("concurrent")
        if r and r["status"] == "solved":
            hist[r["winner"]] = hist.get(r["winner"], 0) + 1
    order = sorted([k for k in hist if k != "main"], key=lambda s: -float(s)) + \
        (["main"] if "main" in hist else [])
    return {"models": len(models), "shift": shift,
            "sgm": {"baseline": sgm_b, "concurrent": sgm_c},
            "performance_ratio": (sgm_b / sgm_c) if sgm_b and sgm_c else None,
            "wins": wins, "losses": losses, "ties": ties,
            "histogram": {k: hist[k] for k in order}, "records": records}


def emit_report(summary: dict, fmt: str) -> str:
    if fmt == "json":
        return json.dumps(summary, indent=1)
    if fmt == "csv":
        s = io.StringIO()
        w = csv.writer(s)
        w.writerow(["model", "mode", "wall_s", "status", "winner", "pdhg_iterations", "pivots",
                    "violation"])
        for r in summary["records"]:
            w.writerow([r["model"], r["mode"], r["wall_s"], r["status"], r.get("winner", ""),
                        r.get("pdhg_iterations", ""), r.get("pivots", ""), r.get("violation", "")])
        return s.getvalue()
    raise ValueError(f"unknown report format {fmt!r}")


def _common(ap):
    ap.add_argument("--mode", default="concurrent", choices=["baseline", "concurrent"])
    ap.add_argument("--eps-rel", type=float, default=1e-6)
    ap.add_argument("--eps-cross", type=float, default=1e-2)
    ap.add_argument("--eps-abs", type=float, default=1e-6)
    ap.add_argument("--decrement", type=float, default=0.1)
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--time-limit", type=float, default=3600.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--pdhg", default="gpu", choices=["gpu", "cpu"])


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="cclp-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve")
    s.add_argument("model")
    _common(s)
    s.add_argument("--write-basis", default="")
    s.add_argument("--write-solution", default="")
    s.add_argument("--json", action="store_true")
    b = sub.add_parser("bench")
    b.add_argument("dir")
    _common(b)
    b.add_argument("--shift", type=float, default=1.0)
    b.add_argument("--out", default="")
    b.add_argument("--csv", default="")
    a = ap.parse_args(argv)
    kw = dict(eps_rel=a.eps_rel, eps_cross=a.eps_cross, eps_abs=a.eps_abs, decrement=a.decrement,
              workers=a.workers, time_limit=a.time_limit, seed=a.seed, pdhg=a.pdhg)
    if a.cmd == "solve":
        if not os.path.exists(a.model):
            print(f"input error: {a.model} not found", file=sys.stderr)
            return EXIT_INPUT
        rc, out = solve_file(a.model, a.mode, basis_out=a.write_basis,
                             solution_out=a.write_solution, **kw)
        if rc == EXIT_INPUT:
            print(f"input error: {out}", file=sys.stderr)
            return rc
        if a.json:
            print(json.dumps(out))
        else:
            print(f"{out.get('model')}: {out['status']} objective {out['objective']:.12g} "
                  f"winner {out['winner']} in {out['cli_wall_s']:.3f} s "
                  f"({out['pdhg_iterations']} PDHG iterations)")
        return rc
    files = sorted(f for f in os.listdir(a.dir) if f.endswith((".mps", ".mps.gz", ".cscb")))
    if not files:
        print(f"input error: no .mps or .cscb files in {a.dir}", file=sys.stderr)
        return EXIT_INPUT
    records = []
    for f in files:
        for mode in ("baseline", "concurrent"):
            rc, out = solve_file(os.path.join(a.dir, f), mode, **kw)
            if rc == EXIT_INPUT:
                records.append(dict(model=f, mode=mode, wall_s=a.time_limit, status="input-error"))
                continue
            records.append(dict(model=f, mode=mode, wall_s=out["cli_wall_s"], status=out["status"],
                                winner=out["winner"], pdhg_iterations=out["pdhg_iterations"],
                                pivots=out.get("pivots"), violation=out.get("violation")))
    summary = summarize(records, a.shift, a.time_limit)
    if a.out:
        open(a.out, "w").write(emit_report(summary, "json"))
    if a.csv:
        open(a.csv, "w").write(emit_report(summary, "csv"))
    print(json.dumps({k: v for k, v in summary.items() if k != "records"}))
    return EXIT_SOLVED


if __name__ == "__main__":
    sys.exit(main())
