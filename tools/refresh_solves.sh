# Time to 1e-4 on C3/C4 and the snapshot-ladder rate on C2/C3 (evidence refresh)
mkdir -p gpurun_out
timeout 600 python tools/probe_snapshots.py C2 C3 > gpurun_out/probe_snapshots.jsonl 2> gpurun_out/probe_snapshots.err; echo "snap_rc=$?"
timeout 400 python tools/time_to_tol.py C3 1e-4 200 > gpurun_out/time_to_tol_c3_c4.jsonl 2> gpurun_out/ttt.err; echo "c3_rc=$?"
timeout 300 python tools/time_to_tol.py C4 1e-4 150 >> gpurun_out/time_to_tol_c3_c4.jsonl 2>> gpurun_out/ttt.err; echo "c4_rc=$?"
cat gpurun_out/probe_snapshots.jsonl gpurun_out/time_to_tol_c3_c4.jsonl
