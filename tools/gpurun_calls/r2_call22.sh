# round-2: K6 phase 1 KP/MINB chosen by layout; batch-aligned slabs bitwise; timing
set -x
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_ranges.py tests/test_gpu_acceptance.py tests/test_gpu_parity.py tests/test_gpu_debug_checks.py -q -x -m gpu -k "standard or bitwise or range or acceptance or kernel_families or slab" > gpurun_out/r2_tests_k6sel.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_tests_k6sel.log
for c in C3 C4 C2; do timeout 300 python tools/k6_ab.py $c 3; done > gpurun_out/r2_k6_sel.txt 2>&1
grep standard gpurun_out/r2_k6_sel.txt
