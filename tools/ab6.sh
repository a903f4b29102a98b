mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_speculative.py -x -q > gpurun_out/spec_tests.log 2>&1; echo "spec_tests_rc=$?"; tail -15 gpurun_out/spec_tests.log
timeout 900 python tools/probe_libs.py ab_libs/base.so ab_libs/spec.so C2 C3 C4 > gpurun_out/ab6.txt 2>&1; cat gpurun_out/ab6.txt
