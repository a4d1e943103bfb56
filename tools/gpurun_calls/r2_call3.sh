# round-2: K6 rewrite (tau + pair groups) parity and A/B; ncu of the e3 combine
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_fuzz.py tests/test_gpu_debug_checks.py -q -x -m gpu > gpurun_out/r2_tests_k6.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_tests_k6.log
for v in p4m1 p2m2 p3m1 p2m1; do for c in C3 C4; do LAMFAST_LIB=build/k6v/$v/liblamfast_b200.so timeout 300 python tools/k6_ab.py $c 3; done; done > gpurun_out/r2_k6_ab.txt 2>&1
cat gpurun_out/r2_k6_ab.txt
LAMFAST_EFORM_MIN_TERMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_e3 -c 1 -o gpurun_out/r2_ncu_e3_c4 python tools/run_steps.py --config C4 --steps 1 > gpurun_out/r2_ncu_e3.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_standard -c 1 -o gpurun_out/r2_ncu_k6_c3 python tools/k6_ab.py C3 1 > gpurun_out/r2_ncu_k6.log 2>&1; echo "ncu k6 rc=$?"
