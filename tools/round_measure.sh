#!/bin/bash
# One GPU call that refreshes the round's evidence: bench (C2), the reference
# arm, a per-config probe, the ncu launch list of the bench workload and one
# `ncu --set full` capture of each iteration kernel (C2 and C4).
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1
for c in C2 C3 C4 C5s; do timeout 300 python tools/probe_perf.py $c; done > gpurun_out/probe_all.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python tools/ncu_target.py C2 20 > /dev/null 2>&1
for c in C2 C4; do
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_spmv_rows|k_spmv_cols|k_dual|k_primal" -s 8 -c 4 \
    -o gpurun_out/full_$c python tools/ncu_target.py $c 5 > gpurun_out/ncu_$c.log 2>&1
done
ls -la gpurun_out
