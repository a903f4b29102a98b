mkdir -p gpurun_out
CCLP_CU_SELL_ROWS=2 timeout 900 python tools/probe_ab.py --fresh CCLP_CU_G_ROWS 1,2,4,8 C2 C3 > gpurun_out/ab9.txt 2>&1
cat gpurun_out/ab9.txt
