# round-2: K2b phase 1 block per element over terms
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py tests/test_gpu_fuzz.py -q -x -m gpu > gpurun_out/r2_tests_k2b2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_tests_k2b2.log
for rep in 1 2; do for v in default k2p2m2 k2p4m1; do for c in C3 C4 C2; do
  lib=paper_1905_05417_b200/lib/liblamfast_b200.so; [ $v != default ] && lib=build/k2bv/$v/liblamfast_b200.so
  echo -n "$v $c: "; LAMFAST_LIB=$lib timeout 120 python tools/run_steps.py --config $c --geometry bilinear --steps 10 2>&1 | tail -1 | cut -c1-100; done; done; done > gpurun_out/r2_k2b_v2.txt 2>&1
grep -v "^+" gpurun_out/r2_k2b_v2.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_k2b_launches_v2.csv python tools/run_steps.py --config C3 --geometry bilinear --steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
