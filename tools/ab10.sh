mkdir -p gpurun_out
for lib in cur st6 st3; do
  echo "== $lib" >> gpurun_out/ab10.txt
  CCLP_CU_LIB=ab_libs/$lib.so timeout 600 python tools/probe_ab.py --fresh CCLP_CU_EPI bulk,reg C2 C3 >> gpurun_out/ab10.txt 2>&1
done
cat gpurun_out/ab10.txt
