"""Benchmark: PDHG iterations/s of the B200 engine on BASELINE.json configs[1]
(C2: synthetic random sparse equality LP, m=100k, n=500k, 5M nnz, fp64).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one batch of `--iters-per-step` (500) PDHG iterations (reference loop
body, check_interval = 1: both residual reports, restart and stop decisions
every iteration) on device-resident state. `value` = total iterations / max
over ranks of the device time of the K timed steps (CUDA events on the engine
stream). `e2e` = the same metric through the public C-ABI call
(cclp_cu_run_pdhg via paper_2510_24429_b200.pdhg.run_pdhg) from pinned host
buffers: LP upload, CSR build, Ruiz, ||A||, the loop and the result download
are all inside the timed region. The working set (~180 MB) exceeds the
126 MB L2, so no flush is needed between steps.

Multi-GPU (torchrun, N>1): C2 fits one GPU, so ranks run independent
replicas ("replicas only" for C1-C3); value sums iterations over
ranks, time is the max over ranks. `--workload C4|C5|C5s` with N>1 runs the
row-block sharded solve instead (one shard per rank; each iteration the
producing kernels store y, x and the report sums straight into the peers'
buffers over NVLink (CUDA IPC), or NCCL all-gathers / halo exchanges with
CCLP_CU_TRANSPORT=gather; iterates bit-identical to one GPU): value =
iterations/s of that one solve (strong scaling), device time max over ranks.

Every N > 1 replica line also carries `partitioned`: C4 (configs[3], 100M nnz)
row-block sharded over the N ranks (5 x 50 iterations, device time max over
ranks, per-GPU fraction of the HBM roofline); at N = 1 it is the single
engine's C4 line (`per_config`).

The roofline's per-kernel times are the kernels' durations inside the CUDA
graph (in-kernel %globaltimer stamps, cclp_cu_phase_profile), with the eager
per-launch event timing reported beside them.

`--impl reference` times the reference's own run_pdhg (oracle/_ref, built
from /root/reference's sources) on one pinned host core of rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PDHG iterations/s (C2 random LP 100k x 500k, 5M nnz, fp64, check every iteration)"
UNIT = "iter/s"
CONFIG_NAME = "C2"


def algorithmic_bytes(m: int, n: int, nnz: int) -> dict:
    """B_iter = 24 nnz + 20 (m+n) + 8, split per kernel:
    row kernel (A x): 12 nnz + 4(m+1) + 8n (x) + 8m (ax);
    column kernel (A'y): 12 nnz + 4(n+1) + 8m (y) + 8n (aty)."""
    return dict(iteration=24 * nnz + 20 * (m + n) + 8,
                rows=12 * nnz + 4 * (m + 1) + 8 * n + 8 * m,
                cols=12 * nnz + 4 * (n + 1) + 8 * m + 8 * n)


def kernel_table(m: int, n: int, nnz: int, ph: dict, dsc: dict) -> list:
    """(kernel, algorithmic bytes per launch, in-graph us, SpMV side) of the
    four kernels one iteration launches (DESIGN.md §4 table)."""
    ab = algorithmic_bytes(m, n, nnz)
    return [("k_spmv_rows_sellg" if dsc.get("sell_rows_block") else "k_spmv_rows", ab["rows"], ph["spmv_rows"], "rows"),
            ("k_dual", 80 * m, ph["dual"], None),
            ("k_spmv_cols_sell" if dsc.get("sell_cols_block") else "k_spmv_cols", ab["cols"], ph["spmv_cols"], "cols"),
            ("k_primal", 96 * n, ph["primal"], None)]


def l2_roofline(lp, dom: str, dom_ms: float, clocks: dict, kernel: str = "") -> dict:
    rows = dom == "rows"
    out_len, vec_len = (lp.m, lp.n) if rows else (lp.n, lp.m)
    traffic = 44.0 * lp.nnz + 4.0 * (out_len + 1) + 8.0 * out_len
    mhz = clocks.get("sm_mhz") or 1965.0
    cap = 6300.0 * mhz * 1e6 / 1e9  # GB/s
    achieved = traffic / (dom_ms * 1e-3) / 1e9
    return {"bound": "l2_sectors", "kernel": kernel or f"k_spmv_{dom}", "bytes_per_launch": traffic,
            "achieved": achieved, "peak": cap, "unit": "GB/s", "frac": achieved / cap,
            "model": "12 B stream + 32 B L2 sector per gathered nonzero + row pointers + output; "
                     "cap 6300 B/clk x SM clock"}


def bench_config(lp, workload: str, world: int, sharded: bool = False) -> dict:
    """The workload description both arms print (identical keys and values)."""
    return {"workload": workload, "m": lp.m, "n": lp.n, "nnz": lp.nnz, "check_interval": 1,
            "parallelism": (f"row-block sharded x{world}" if sharded else
                            ("replicas" if world > 1 else "single")),
            "l2": "working set > 126 MB L2, no flush"}


def pinned_core():
    """Run the CPU baselines on ONE host core (the reference loop is
    single-threaded; 1 pinned core). Returns (core, host_cores)."""
    host = os.cpu_count() or 1
    try:
        allowed = sorted(os.sched_getaffinity(0))
        return allowed[-1], host, allowed
    except Exception:
        return None, host, None


class OneCore:
    def __enter__(self):
        self.core, self.host, self.allowed = pinned_core()
        if self.core is not None:
            os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        if self.allowed is not None:
            os.sched_setaffinity(0, set(self.allowed))


CPU_NOTE = ("the reference's own sources (proj/src/*.cpp, unmodified) compiled against the "
            "repo's Eigen-API subset (third_party/eigen_subset, built by oracle/Makefile): Eigen 3.4 "
            "is not installed on the box")


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t = time.time()  # the timed region starts once the sampler is live
            while not self.lines and time.time() - t < 5.0:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# Test mode for the N > 1 code paths on a single-GPU box: every rank on
# device 0, the process group over gloo, and the sharded arm's control
# exchange through it (host all-gather) instead of NCCL.
ONE_DEVICE = os.environ.get("CCLP_BENCH_ONE_DEVICE") == "1"


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if ONE_DEVICE else int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1 and args.impl != "reference":
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group(backend="gloo" if ONE_DEVICE else "nccl")
        pg = dist
    return world, rank, local, pg


def barrier(pg):
    if pg is not None:
        pg.barrier()


def allreduce_max(pg, v: float, device) -> float:
    if pg is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if ONE_DEVICE else device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(pg, v: float, device) -> float:
    if pg is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if ONE_DEVICE else device)
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


def pinned_copy(lp):
    """The LP's arrays in pinned host memory (the e2e input buffers)."""
    import torch
    from paper_2510_24429_b200.lp import LinearProgram

    def pin(a, dt):
        t = torch.empty(a.shape, dtype=dt, pin_memory=True)
        t.numpy()[...] = a
        return t

    keep = [pin(lp.colptr, torch.int32), pin(lp.rowind, torch.int32), pin(lp.val, torch.float64),
            pin(lp.c, torch.float64), pin(lp.row_lower, torch.float64),
            pin(lp.row_upper, torch.float64), pin(lp.col_lower, torch.float64),
            pin(lp.col_upper, torch.float64)]
    arrs = [k.numpy() for k in keep]
    return LinearProgram(lp.m, lp.n, *arrs, name=lp.name), keep


def cpu_reference_rate(lp, iters: int, use_ref: bool = True):
    """Loop-only iterations/s of the reference run_pdhg: (T(S) - T(0)) / S, on
    one pinned host core."""
    from oracle.pyoracle import Reference, Restatement, reference_available
    kind = "reference" if (use_ref and reference_available()) else "port"
    impl = Reference() if kind == "reference" else Restatement()
    with OneCore() as oc:
        t = time.perf_counter()
        impl.run_pdhg(lp, config=dict(max_iterations=0))
        t0 = time.perf_counter() - t
        t = time.perf_counter()
        r = impl.run_pdhg(lp, config=dict(max_iterations=iters))
        ts = time.perf_counter() - t
    return dict(value=r["iterations"] / max(ts - t0, 1e-9), setup_s=t0, total_s=ts,
                iterations=r["iterations"], kind=kind, core=oc.core, host_cores=oc.host)


def run_reference_arm(args, world, rank, pg):
    from paper_2510_24429_b200 import lpgen
    if rank != 0:  # the reference is a single-process CPU code: rank 0 only
        return
    lp = lpgen.make_config(CONFIG_NAME)
    from oracle.pyoracle import Reference, Restatement, reference_available
    kind = "reference" if reference_available() else "port"
    impl = Reference() if kind == "reference" else Restatement()
    S = args.ref_iters
    with OneCore() as oc:
        t = time.perf_counter()
        impl.run_pdhg(lp, config=dict(max_iterations=0))  # setup only: Ruiz + ||A|| + check(0)
        t_setup = time.perf_counter() - t
        for _ in range(max(args.warmup - 1, 0)):
            impl.run_pdhg(lp, config=dict(max_iterations=1))
        loop_s, iters = 0.0, 0
        for _ in range(args.steps):
            t = time.perf_counter()
            r = impl.run_pdhg(lp, config=dict(max_iterations=S))
            loop_s += max(time.perf_counter() - t - t_setup, 1e-9)
            iters += r["iterations"]
    v = iters / loop_s
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * loop_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, paper_2510_24429_b200/lpgen.py)",
        "config": bench_config(lp, CONFIG_NAME, world),
        "iters_per_step": S,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "host_cores": oc.host,
                         "kind": kind,
                         "sample": f"C2, {args.steps} x run_pdhg(max_iterations={S}) minus its "
                                   f"setup ({t_setup:.2f} s: Ruiz + power iteration), on 1 of "
                                   f"{oc.host} host cores (sched_setaffinity to core {oc.core}; "
                                   f"the reference has no threading); {CPU_NOTE}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


SHARDED_WORKLOADS = ("C3", "C4", "C5", "C5s")


def metric_for(workload: str) -> str:
    if workload == CONFIG_NAME:
        return METRIC
    return f"PDHG iterations/s ({workload} synthetic LP, fp64, check every iteration)"


def _fresh_nccl_id(pg, rank, dev):
    """A new NCCL unique id from rank 0, broadcast over the process group."""
    import torch
    from paper_2510_24429_b200.pdhg import nccl_unique_id
    idt = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    pg.broadcast(idt, src=0)
    return bytes(idt.cpu().numpy().tobytes())


def run_sharded_arm(args, world, rank, local, pg, emit=True, workload=None, steps=None, iters=None,
                    e2e=True):
    """N ranks, one row-block shard each (cclp_cu_sharded over NCCL). With
    emit=False the line is returned (rank 0) instead of printed: the
    `partitioned` record of a replica run."""
    import torch
    from paper_2510_24429_b200 import lpgen
    from paper_2510_24429_b200.pdhg import PdhgConfig, ShardedEngine, nccl_unique_id

    dev = torch.device("cuda", local)
    workload = workload or args.workload
    lp = lpgen.make_config(workload)
    if ONE_DEVICE:
        def host_allgather(blob: bytes):
            parts = [None] * world
            pg.all_gather_object(parts, blob)
            return parts
        make = lambda src: ShardedEngine(src, 1, device=local, rank=rank, nranks=world,  # noqa: E731
                                         host_allgather=host_allgather)
    else:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        pg.broadcast(idt, src=0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
        make = lambda src: ShardedEngine(src, 1, device=local, rank=rank, nranks=world,  # noqa: E731
                                         nccl_id=nccl_id if src is lp else _fresh_nccl_id(pg, rank, dev))
    t_setup = time.perf_counter()
    eng = make(lp)
    eng.begin(PdhgConfig())
    t_setup = allreduce_max(pg, time.perf_counter() - t_setup, dev)
    K, W, I = steps or args.steps, args.warmup, iters or args.iters_per_step
    for _ in range(W):
        eng.advance(I)
    torch.cuda.synchronize(dev)
    barrier(pg)
    with ClockSampler(local) as clk:
        dev_ms = sum(eng.advance(I) for _ in range(K))
    barrier(pg)
    t_max = allreduce_max(pg, dev_ms, dev)
    d = eng.describe()
    eng.close()
    value = K * I / (t_max * 1e-3)
    B = 24 * lp.nnz + 20 * (lp.m + lp.n) + 8
    peak, peak_kind = measured_peak_gbs()
    if not e2e:
        if rank != 0:
            return None
        return {"workload": workload, "m": lp.m, "n": lp.n, "nnz": lp.nnz, "shards": world,
                "iters_per_s": value, "us_per_iteration": t_max * 1e3 / (K * I), "iters_timed": K * I,
                "setup_s_incl_create": t_setup,
                "iteration_frac_per_gpu": B * value / 1e9 / world / peak,
                "row_bounds": d["row_bounds"], "col_bounds": d["col_bounds"],
                "halo_x": d["halo_x"], "halo_y": d["halo_y"],
                "slice_nnz": [(s_["nnz_rows"], s_["nnz_cols"]) for s_ in d["local_shards"]],
                "transport": "push (P2P stores over CUDA IPC)" if ONE_DEVICE else "NCCL / push",
                "clocks": clk.summary()}
    # e2e: every rank builds its shard engine from the LP in pinned host
    # memory and solves `--e2e-iters` iterations, result gathered to every
    # rank (upload, slicing, setup, loop, download); max over ranks
    plp, _keep = pinned_copy(lp)
    cfg = PdhgConfig(max_iterations=args.e2e_iters)
    barrier(pg)
    t = time.perf_counter()
    with make(plp) as e2:
        res = e2.solve(cfg)
    e2e_t = allreduce_max(pg, time.perf_counter() - t, dev)
    e2e_value = res.iterations / e2e_t
    if rank == 0:
        line = {
            "metric": metric_for(workload), "value": value, "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": t_max / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, paper_2510_24429_b200/lpgen.py)",
            "config": {"workload": workload, "m": lp.m, "n": lp.n, "nnz": lp.nnz,
                       "iters_per_step": I, "check_interval": 1,
                       "parallelism": f"row-block sharded x{world} (NCCL all-gather)",
                       "row_bounds": d["row_bounds"], "col_bounds": d["col_bounds"],
                       "l2": "matrix >> 126 MB L2, no flush"},
            "us_per_iteration": t_max * 1e3 / (K * I),
            "roofline": {"bound": "hbm", "achieved": B * value / 1e9 / world, "peak": peak,
                         "unit": "GB/s", "frac": B * value / 1e9 / world / peak,
                         "traffic": None, "kernel": "whole iteration, per GPU",
                         "bytes_per_launch": B, "peak_kind": peak_kind},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": sum(a.nbytes for a in (plp.colptr, plp.rowind, plp.val, plp.c,
                                                                 plp.row_lower, plp.row_upper,
                                                                 plp.col_lower, plp.col_upper)),
                    "d2h_bytes_per_step": 8 * (2 * lp.n + lp.m), "iters_per_step": args.e2e_iters,
                    "includes": "per rank: shard engine from pinned host LP, setup, loop, full result"},
            "gpu_launches": int(d["launches"]),
            "clocks": clk.summary(),
        }
        if ONE_DEVICE:
            line["config"]["parallelism"] = f"row-block sharded x{world} on ONE device (test mode)"
        print(json.dumps(line), flush=True)


def per_config_line(name: str, args, local: int) -> dict:
    """The >= 10M-nnz configs (north_star's 50 % target) in the same run:
    device-resident iterations/s through the same loop, the in-graph kernel
    split, the dominant kernel's and the iteration's fraction of the measured
    HBM peak, and the clocks sampled during that timed region."""
    import torch
    from paper_2510_24429_b200 import lpgen
    from paper_2510_24429_b200.pdhg import Engine, PdhgConfig
    lp = lpgen.make_config(name)
    I = max(20, int(args.iters_per_step * 5_000_000 / lp.nnz))
    K = 5
    peak, peak_kind = measured_peak_gbs()
    with Engine(lp, device=local) as eng:
        eng.begin(PdhgConfig())
        for _ in range(3):
            eng.advance(I)
        torch.cuda.synchronize(local)
        with ClockSampler(local) as clk:
            ms = sum(eng.advance(I) for _ in range(K))
        ph = eng.phase_profile()
        dsc = eng.describe()
    ab = algorithmic_bytes(lp.m, lp.n, lp.nnz)
    iter_us = ms * 1e3 / (K * I)
    ks = kernel_table(lp.m, lp.n, lp.nnz, ph, dsc)
    dom_kernel, dom_bytes, dom_us, _ = max(ks, key=lambda k: k[2])
    dom_gbs = dom_bytes / (dom_us * 1e-6) / 1e9
    it_gbs = ab["iteration"] / (iter_us * 1e-6) / 1e9
    del lp
    return {"m": dsc.get("m"), "n": dsc.get("n"), "nnz": dsc.get("nnz"),
            "iters_per_s": K * I / (ms * 1e-3), "us_per_iteration": iter_us,
            "iters_timed": K * I,
            "kernels_us": {k: ph[k] for k in ("spmv_rows", "dual", "spmv_cols", "primal")},
            "kernels_timing": f"in-graph stamps, median of {ph['steps']} steps",
            "kernels": {k: {"us": us, "bytes_per_launch": b, "frac": b / (us * 1e-6) / 1e9 / peak}
                        for k, b, us, _ in ks if us > 0},
            "dominant": {"kernel": dom_kernel, "bytes_per_launch": dom_bytes, "achieved": dom_gbs,
                         "frac": dom_gbs / peak},
            "iteration": {"bytes": ab["iteration"], "achieved": it_gbs, "frac": it_gbs / peak},
            "peak": peak, "peak_kind": peak_kind, "clocks": clk.summary()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--iters-per-step", type=int, default=500)
    ap.add_argument("--e2e-iters", type=int, default=2000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-iters", type=int, default=20)
    ap.add_argument("--cpu-iters", type=int, default=200)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--per-config", default="C3,C4",
                    help="extra configs timed in the same N=1 run ('' to skip)")
    ap.add_argument("--partitioned", default="C4",
                    help="config of the per-N partitioned record ('' to skip)")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-tolerance solves (profiling runs)")
    ap.add_argument("--workload", default=CONFIG_NAME,
                    help="C2 (default, configs[1]); C3/C4/C5/C5s: with N>1 the sharded solve")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world, rank, local, pg = dist_setup(args)
    if args.impl == "reference":
        run_reference_arm(args, world, rank, pg)
        return
    if world > 1 and args.workload in SHARDED_WORKLOADS:
        run_sharded_arm(args, world, rank, local, pg)
        pg.destroy_process_group()
        return

    import torch
    from paper_2510_24429_b200 import lpgen
    from paper_2510_24429_b200.pdhg import Engine, PdhgConfig, Tolerances, run_pdhg

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lp = lpgen.make_config(args.workload)
    eng = Engine(lp, device=local)
    eng.begin(PdhgConfig())
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=dev)
    K, W, I = args.steps, args.warmup, args.iters_per_step
    for _ in range(W):
        eng.advance(I)
    launches0 = eng.describe()["launches"]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    barrier(pg)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        lib_ms = 0.0
        for _ in range(K):
            lib_ms += eng.advance(I)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    barrier(pg)
    dev_ms = ev0.elapsed_time(ev1)
    launches = eng.describe()["launches"] - launches0
    t_max = allreduce_max(pg, dev_ms, dev)
    total_iters = allreduce_sum(pg, float(K * I), dev)
    value = total_iters / (t_max * 1e-3)

    # per-kernel device time for the roofline: the split of the timed graph
    # iterations themselves (in-kernel %globaltimer stamps, median over the
    # last 128 steps); the eager per-kernel event timing is kept beside it
    ph = eng.phase_profile()
    pk_eager = eng.profile_kernels(100)
    pk = {k: ph[k] * 1e-3 for k in ("spmv_rows", "dual", "spmv_cols", "primal")}
    ab = algorithmic_bytes(lp.m, lp.n, lp.nnz)
    dsc = eng.describe()
    # the kernels that actually ran (SELL layouts: engine.cu)
    ks = kernel_table(lp.m, lp.n, lp.nnz, ph, dsc)
    dom_kernel, dom_bytes, dom_us, dom = max(ks, key=lambda k: k[2])
    dom_ms = dom_us * 1e-3
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peak_gbs()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(args.workload, {}).get(dom_kernel)
    except Exception:
        pass
    iter_us = dev_ms * 1e3 / (K * I)
    eng.close()

    # e2e: public API from pinned host buffers, upload..download timed
    plp, _keep = pinned_copy(lp)
    h2d = sum(a.nbytes for a in (plp.colptr, plp.rowind, plp.val, plp.c, plp.row_lower,
                                 plp.row_upper, plp.col_lower, plp.col_upper))
    d2h = 8 * (2 * lp.n + lp.m)
    cfg = PdhgConfig(max_iterations=args.e2e_iters)
    run_pdhg(plp, PdhgConfig(max_iterations=10), device=local)  # warm
    barrier(pg)
    e2e_t, e2e_it = 0.0, 0
    for _ in range(args.e2e_steps):
        t = time.perf_counter()
        res = run_pdhg(plp, cfg, device=local)
        e2e_t += time.perf_counter() - t
        e2e_it += res.iterations
    e2e_t = allreduce_max(pg, e2e_t, dev)
    e2e_total = allreduce_sum(pg, float(e2e_it), dev)
    e2e_value = e2e_total / e2e_t

    # time to tolerance (one solve, rank 0)
    ttt = None
    if rank == 0 and lp.nnz <= 25_000_000 and not args.no_ttt:  # ~1 s on C2; C4/C5 would take minutes
        t = time.perf_counter()
        r4 = run_pdhg(plp, PdhgConfig(max_iterations=200000),
                      tol=Tolerances(eps_rel=1e-4),
                      device=local)
        ttt = {"eps_rel": 1e-4, "seconds": time.perf_counter() - t, "iterations": r4.iterations,
               "stop": r4.stop.name, "restarts": r4.restarts}
        t = time.perf_counter()
        r6 = run_pdhg(plp, PdhgConfig(max_iterations=400000), tol=Tolerances(eps_rel=1e-6),
                      device=local)
        ttt = [ttt, {"eps_rel": 1e-6, "seconds": time.perf_counter() - t,
                     "iterations": r6.iterations, "stop": r6.stop.name, "restarts": r6.restarts}]

    # the partitioned path (north_star (4)) at this N: C4 row-block sharded
    # over the N ranks (N = 1: the single engine's C4 line below)
    partitioned = None
    if world > 1 and args.partitioned:
        torch.cuda.synchronize(dev)
        partitioned = run_sharded_arm(args, world, rank, local, pg, emit=False, workload=args.partitioned,
                                      steps=5, iters=50, e2e=False)

    per_config = None
    if rank == 0 and world == 1 and args.per_config:
        per_config = {c: per_config_line(c, args, local) for c in args.per_config.split(",") if c}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_iters = max(3, int(args.cpu_iters * 5_000_000 / max(lp.nnz, 1)))
        cb = cpu_reference_rate(lp, cpu_iters)
        cpu = {"value": cb["value"], "unit": UNIT, "cores": 1, "host_cores": cb["host_cores"],
               "kind": cb["kind"],
               "sample": f"{args.workload}, run_pdhg(max_iterations={cpu_iters}) minus "
                         f"run_pdhg(max_iterations=0) ({cb['setup_s']:.2f} s setup), on 1 of "
                         f"{cb['host_cores']} host cores (sched_setaffinity to core {cb['core']}; "
                         f"the reference loop is single-threaded); {CPU_NOTE}"}

    if rank == 0:
        line = {
            "metric": metric_for(args.workload), "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": t_max / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, paper_2510_24429_b200/lpgen.py)",
            "config": bench_config(lp, args.workload, world),
            "iters_per_step": I,
            "us_per_iteration": iter_us,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": dom_kernel,
                         "kernel_us": dom_ms * 1e3, "bytes_per_launch": dom_bytes,
                         "peak_kind": peak_kind,
                         "iteration": {"bytes": ab["iteration"],
                                       "achieved": ab["iteration"] / (iter_us * 1e-6) / 1e9,
                                       "frac": ab["iteration"] / (iter_us * 1e-6) / 1e9 / peak},
                         "kernels_us": {k: v * 1e3 for k, v in pk.items()},
                         "kernels": {k: {"us": us, "bytes_per_launch": b,
                                         "frac": b / (us * 1e-6) / 1e9 / peak}
                                     for k, b, us, _ in ks if us > 0},
                         "kernels_timing": f"in-graph: block-0 %globaltimer stamps after each "
                                           f"kernel's PDL wait, median of {ph['steps']} steps",
                         "kernels_us_eager": {k: v * 1e3 for k, v in pk_eager.items()}},
            # the bound the SpMV actually meets on gather-heavy LPs: L2 traffic of
            # 12 B stream + one 32 B sector per gathered nonzero (+ the vectors),
            # against the LTS throughput cap (~6,300 B/clk, B300_MICROARCH.md) at
            # the sampled SM clock
            "l2_roofline": (l2_roofline(lp, dom, dom_ms, clk.summary(), dom_kernel)
                            if dom is not None else None),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "iters_per_step": args.e2e_iters,
                    "includes": "upload, CSR build, Ruiz, ||A|| power iteration, loop, download"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "time_to_tolerance": ttt,
            "cpu_baseline": cpu,
        }
        if per_config:
            line["per_config"] = per_config
            if args.partitioned in per_config:
                partitioned = dict(per_config[args.partitioned], shards=1, workload=args.partitioned)
        if partitioned:
            line["partitioned"] = partitioned
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
