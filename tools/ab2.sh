mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python tools/probe_libs.py ab_libs/base.so ab_libs/spec.so C2 C3 C4 > gpurun_out/ab2.txt 2>&1; echo "ab_rc=$?"; cat gpurun_out/ab2.txt | tail -20
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests_rc=$?"; tail -15 gpurun_out/gputests.log
