# C2 ncu (launch list and one --set full capture of the iteration kernels)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python tools/ncu_target.py C2 20 > /dev/null 2>&1; echo "launch_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_spmv_rows|k_spmv_cols|k_dual|k_primal" -s 8 -c 4 \
    -o gpurun_out/full_C2 python tools/ncu_target.py C2 5 > gpurun_out/ncu_C2.log 2>&1; echo "full_rc=$?"
