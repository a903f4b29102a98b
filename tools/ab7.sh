mkdir -p gpurun_out
timeout 1200 python tools/probe_libs.py ab_libs/cur.so ab_libs/nopipe_minb2.so C3 C4 > gpurun_out/ab7.txt 2>&1
timeout 600 python tools/probe_libs.py ab_libs/cur.so ab_libs/nopipe.so C3 >> gpurun_out/ab7.txt 2>&1
cat gpurun_out/ab7.txt
