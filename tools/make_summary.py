"""Writes profiles/<round>/SUMMARY.md from the evidence files in that
directory (bench line, reference arm, ncu summaries, launch list, probes).

    python tools/make_summary.py r2
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r2"
D = os.path.join(ROOT, "profiles", rnd)


def last_json(name):
    with open(os.path.join(D, name)) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def text(name, default=""):
    p = os.path.join(D, name)
    return open(p).read().strip() if os.path.exists(p) else default


b = last_json("bench_c2.json")
r = last_json("bench_ref_c2.json")
ro = b["roofline"]
ku = ro["kernels_us"]
lines = text("launches_c2.md").splitlines()[:12]
snap = [json.loads(x) for x in text("probe_snapshots.jsonl").splitlines() if x.strip()]
c2snap = next((s for s in snap if s["config"] == "C2"), None)

out = [f"# {rnd} evidence (B200, 1 GPU)", "",
       "Commands (`gpurun`; `tools/round_measure.sh [tests] [bench] [ncu]` for the suite, the bench and ncu):", "",
       "    python -m pytest tests -m gpu -x -q                    -> gputests_tail.txt",
       "    python bench.py                                        -> bench_c2.json",
       "    python bench.py --impl reference --steps 2 --warmup 3  -> bench_ref_c2.json",
       "    ncu --metrics gpu__time_duration.sum --clock-control none --csv \\",
       "        --log-file launches_c2.csv python tools/ncu_target.py C2 200  -> launches_c2.md",
       "    ncu --set full --clock-control none --import-source on \\",
       "        -k regex:\"k_spmv_rows|k_spmv_cols|k_dual|k_primal\" -s 8 -c 4 python tools/ncu_target.py C2|C3|C4 5",
       "                                                           -> ncu_full_C*.md, ../ncu_traffic.json",
       "    python tools/probe_perf.py C2|C3|C4|C5s                -> probe_c2_c3_c4_c5s.txt",
       "    python tools/probe_snapshots.py C2 C3                  -> probe_snapshots.jsonl",
       "    python tools/probe_e2e.py C2                           -> probe_e2e_c2.txt",
       "    python tools/crossover_scale.py [--cases C2 --no-race] -> crossover_scale.jsonl, crossover_c2.jsonl",
       "    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py -> sanitize_memcheck.txt", "",
       f"GPU tests: {text('gputests_tail.txt')}", "",
       "## Bench line (C2, configs[1]: m=100k, n=500k, 5M nnz, fp64, check every iteration)", "",
       "| quantity | value |", "|---|---|",
       f"| device loop (`value`, {b['steps']} steps x {b['iters_per_step']} iterations) | **{b['value']:,.0f} it/s** "
       f"({b['us_per_iteration']:.1f} us/iteration) |",
       f"| end to end through the C ABI (`e2e`: pinned host buffers, upload..download, "
       f"{b['e2e']['iters_per_step']:,} iterations incl. setup) | **{b['e2e']['value']:,.0f} it/s** |",
       f"| reference `run_pdhg`, 1 pinned host core (`--impl reference`, same box) | {r['value']:.1f} it/s "
       f"(e2e ratio **{b['e2e']['value'] / r['value']:.0f}x**) |",
       f"| bench `cpu_baseline` (same reference build, in the bench process) | {b['cpu_baseline']['value']:.1f} it/s |",
       f"| in-graph split (us): rows / dual / cols / primal | {ku['spmv_rows']:.1f} / {ku['dual']:.1f} / "
       f"{ku['spmv_cols']:.1f} / {ku['primal']:.1f} |",
       f"| dominant `{ro['kernel']}`: algorithmic {ro['bytes_per_launch'] / 1e6:.1f} MB / {ro['kernel_us']:.1f} us "
       f"| **{ro['frac']:.3f}** of the measured {ro['peak']:.0f} GB/s (L2-sector model {b['l2_roofline']['frac']:.2f}) |",
       "| per kernel fraction of the HBM peak | "
       + ", ".join(f"{k} {v['frac']:.2f}" for k, v in ro.get("kernels", {}).items()) + " |",
       f"| iteration (B_iter {ro['iteration']['bytes'] / 1e6:.0f} MB) | {ro['iteration']['frac']:.3f} |",
       f"| ncu DRAM traffic of the dominant kernel per launch | "
       + (f"{ro['traffic'] / 1e6:.1f} MB" if ro.get("traffic") else "n/a") + " |"]
if b.get("time_to_tolerance"):
    t4, t6 = b["time_to_tolerance"]
    out.append(f"| time to 1e-4 / 1e-6 (full solves, end to end) | {t4['seconds']:.2f} s ({t4['iterations']:,} it) / "
               f"{t6['seconds']:.1f} s ({t6['iterations']:,} it) |")
out.append(f"| clocks during the timed region | {b['clocks']['sm_mhz']:.0f} MHz of {b['clocks']['sm_max_mhz']:.0f}, "
           f"reasons {b['clocks']['reasons']} |")
ttt = [json.loads(x) for x in text("time_to_tol_c3_c4.jsonl").splitlines() if x.strip()]
if ttt:
    out += ["", "Time to 1e-4 end to end (`tools/time_to_tol.py`, `time_to_tol_c3_c4.jsonl`): "
            + "; ".join(f"{t['config']} {t['seconds']:.1f} s ({t['iterations']:,} iterations, {t['restarts']} restarts)"
                        for t in ttt) + "."]
out += ["", "## Per configuration (same bench run, `per_config`; in-graph kernel split)", "",
        "| config | nnz | us / iteration | B_iter fraction | rows | dual | cols | primal | dominant (fraction) |",
        "|---|---|---|---|---|---|---|---|---|"]
for c, v in b.get("per_config", {}).items():
    k = v["kernels_us"]
    out.append(f"| {c} | {v['nnz'] / 1e6:.1f}M | {v['us_per_iteration']:.1f} | **{v['iteration']['frac']:.3f}** | "
               f"{k['spmv_rows']:.1f} | {k['dual']:.1f} | {k['spmv_cols']:.1f} | {k['primal']:.1f} | "
               f"`{v['dominant']['kernel']}` ({v['dominant']['frac']:.2f}) |")
out += ["", "Probe on the same box (`probe_c2_c3_c4_c5s.txt`, CUDA graph, best of 3): ",
        "```", text("probe_c2_c3_c4_c5s.txt"), "```", "",
        "## ncu --set full", ""]
for c in ("C2", "C3", "C4"):
    t = text(f"ncu_full_{c}.md")
    if t:
        out += [t, ""]
out += ["`k_dual<1>`/`k_primal<1>` are the bulk-copy forms (512 threads, one block per SM, a 112-128 KB shared-memory",
        "ring; SASS `UBLKCP` bulk copies and `SYNCS` mbarrier waits); `<0>` the thread-load forms C2 takes.", "",
        "## Launch list, C2 (`tools/ncu_target.py C2 200`: setup + 200 eager iterations; cold, serialized — compare shares; under ncu the geometry tuning picks the 256-thread SELL variants)",
        ""] + lines + ["",
        "The setup's power iteration (100 x: two SpMVs, `k_repro_max`, `k_repro_sum`, `k_div_scalar`) dominates the list.", ""]
if c2snap:
    out += ["## Snapshots do not stall the loop (`probe_snapshots.jsonl`)", "",
            f"C2, {c2snap['ladder']['iterations']:,} iterations with and without the 1e-2...1e-5 ladder (snapshots at "
            f"iterations {', '.join(str(s[0]) for s in c2snap['ladder']['snapshots'])}, "
            f"{c2snap['snapshot_bytes'] / 1e6:.1f} MB each, extracted by the kernels into device slots and copied on a "
            f"side stream while the loop runs): loop rate ratio **{c2snap['rate_ratio_ladder_over_plain']:.3f}**.", ""]
out += ["## Crossover scalability and time to basic", "",
        "`crossover_scale.jsonl` (DESIGN.md §7): the scalable crossover finds the reference crossover's basis on every LP the",
        "reference can run, 0.36 s vs 28.8 s (m = 4,000) and 1.45 s vs 171.9 s (m = 7,000) with pricing on the B200.",
        "`crossover_c2.jsonl`: on C2 (m = 100k, a random LP) the crossover from the 1e-4 iterate does not finish in 14 min",
        "and the race in 11 min (the crash LU of a random 100k basis fills in); the reference's dense etas need 80 GB.", "",
        "## Experiments not adopted (`history/`)", "",
        "* `r2_fused_halfsteps.txt` — SpMV + epilogue fused kernels: slower on every config.",
        "* `r2_smem_panel_spmv_c2.txt` — x staged in shared memory by TMA, column panels: slower than the L1 gathers.",
        "* `r2_sellg_pipe_and_g.txt` — pipelined SELL-G loop, G = 2 on C4 rows, length-sorted SELL-G windows, adaptive",
        "  bulk tiles, k_select_x grid, parallel bulk issue: none faster; the cancel poll costs nothing.",
        "* `r2_staged_rows.txt` — the CSR-G row product's matrix stream through a bulk-copy shared-memory ring",
        "  (bit-identical; block-synchronous ring much slower on C4/C5s), and 8 loads in flight per lane (slower).",
        "* `r2_epilogue_bulk_vs_reg.txt`, `r2_ab_primal_bulk.txt` — the bulk-copy epilogues (adopted on long vectors).", ""]
open(os.path.join(D, "SUMMARY.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
