# round-2: coef kernel with double-buffered cp.async staging
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py tests/test_gpu_ranges.py -q -x -m gpu -k "coefficient or many_terms or decompose or kernel_families or range" > gpurun_out/r2_tests_coef5.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_tests_coef5.log
for rep in 1 2; do for c in C4 C3; do for dec in "" "--decompose"; do echo -n "coef $c $dec: "; LAMFAST_EFORM_MIN_TERMS=1 timeout 120 python tools/run_steps.py --config $c --steps 20 $dec 2>&1 | tail -1 | cut -c1-110; done; done; done > gpurun_out/r2_coef_v5.txt 2>&1
grep -v "^+" gpurun_out/r2_coef_v5.txt
LAMFAST_EFORM_MIN_TERMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_coef -c 1 -o gpurun_out/r2_ncu_coef_v5_c4 python tools/run_steps.py --config C4 --steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
