mkdir -p gpurun_out
timeout 600 python tools/probe_ab.py --fresh CCLP_CU_SELL 1,2 C2 > gpurun_out/ab8.txt 2>&1
timeout 600 python tools/probe_ab.py --fresh CCLP_CU_SELLG_COLS 2,0 C2 >> gpurun_out/ab8.txt 2>&1
cat gpurun_out/ab8.txt
