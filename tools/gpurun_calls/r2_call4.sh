# round-2: lane-transposed coefficient combine (k_combine_coef): parity, A/B, ncu
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py tests/test_gpu_ranges.py -q -x -m gpu > gpurun_out/r2_tests_coef.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_tests_coef.log
STEPS=20 timeout 900 bash tools/ab_eform.sh > gpurun_out/r2_coef.txt 2>&1; echo "ab rc=$?"
head -16 gpurun_out/r2_coef.txt | cut -c1-120
LAMFAST_EFORM_MIN_TERMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_coef -c 1 -o gpurun_out/r2_ncu_coef_c4 python tools/run_steps.py --config C4 --steps 1 > gpurun_out/r2_ncu_coef.log 2>&1; echo "ncu rc=$?"
