# round-2: K6 CONSTC prologue-only form; store-pattern diagnostics (ideal v2 stores)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_debug_checks.py -q -x -m gpu > gpurun_out/r2_tests_k6c2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_tests_k6c2.log
for rep in 1 2; do for m in 1 0; do for c in C3 C4; do echo -n "const=$m "; LAMFAST_K6_CONST=$m timeout 300 python tools/k6_ab.py $c 3; done; done; done > gpurun_out/r2_k6_const2.txt 2>&1
grep standard gpurun_out/r2_k6_const2.txt
for rep in 1 2; do for v in default storeonly v2test v2testso; do
  lib=paper_1905_05417_b200/lib/liblamfast_b200.so; [ $v != default ] && lib=build/ptv/$v/liblamfast_b200.so
  echo -n "$v C4: "; LAMFAST_LIB=$lib timeout 120 python tools/run_steps.py --config C4 --steps 20 2>&1 | tail -1 | cut -c1-110
done; done > gpurun_out/r2_v2test.txt 2>&1
grep -v "^+" gpurun_out/r2_v2test.txt
