# round-2: K6 two-phase phase-1 occupancy variants
set -x
for v in default tp2m3 tp1m3 tp1m4; do for c in C3 C4; do
  lib=paper_1905_05417_b200/lib/liblamfast_b200.so; [ $v != default ] && lib=build/k6v/$v/liblamfast_b200.so
  echo -n "$v "; LAMFAST_LIB=$lib timeout 300 python tools/k6_ab.py $c 3; done; done > gpurun_out/r2_k6_occ.txt 2>&1
grep standard gpurun_out/r2_k6_occ.txt
timeout 900 python -m pytest tests/test_gpu_ranges.py tests/test_gpu_acceptance.py tests/test_gpu_debug_checks.py -q -x -m gpu > gpurun_out/r2_tests_k6batch.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_tests_k6batch.log
