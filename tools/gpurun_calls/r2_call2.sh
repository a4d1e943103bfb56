# round-2 check: e3 coefficient form, pattern kernel registers, drop-in THP
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py tests/test_gpu_ranges.py tests/test_dropin.py tests/test_gpu_fuzz.py -q -x -m gpu > gpurun_out/r2_tests_e3.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_tests_e3.log
for c in C4 C3 C2; do timeout 120 python tools/time_pattern.py $c; done > gpurun_out/r2_pattern.txt 2>&1
STEPS=20 timeout 900 bash tools/ab_eform.sh > gpurun_out/r2_eform_e3.txt 2>&1; echo "eform rc=$?"
timeout 300 ./build/dropin_e2e C4 3 > gpurun_out/r2_dropin_e2e.txt 2>&1; echo "dropin rc=$?"
cat gpurun_out/r2_pattern.txt gpurun_out/r2_dropin_e2e.txt
