#!/bin/bash
# One GPU call that refreshes the round's evidence: the GPU test suite, bench
# (C2 + per_config C3/C4), the reference arm, the ncu launch list of the bench
# workload and one `ncu --set full` capture of the iteration kernels (C2-C4).
#   tools/round_measure.sh [tests] [bench] [ncu]   (default: all three)
set -x
mkdir -p gpurun_out
ARGS=("$@")
want() {
  [ ${#ARGS[@]} -eq 0 ] && return 0
  for a in "${ARGS[@]}"; do [ "$a" = "$1" ] && return 0; done
  return 1
}
if want tests; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests_rc=$?"
  tail -3 gpurun_out/gputests.log
fi
if want bench; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
  timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1
fi
if want ncu; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python tools/ncu_target.py C2 200 > /dev/null 2>&1
  for c in C2 C3 C4; do
    timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"k_spmv_rows|k_spmv_cols|k_dual|k_primal" -s 8 -c 4 \
      -o gpurun_out/full_$c python tools/ncu_target.py $c 5 > gpurun_out/ncu_$c.log 2>&1
  done
fi
ls -la gpurun_out
