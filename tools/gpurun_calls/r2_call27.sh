# round-2: K2b phase-1 tables precomputed by a separate kernel
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py tests/test_gpu_fuzz.py tests/test_gpu_ranges.py -q -x -m gpu > gpurun_out/r2_tests_k2btab.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_tests_k2btab.log
for rep in 1 2; do for c in C3 C4 C2; do echo -n "$c: "; timeout 120 python tools/run_steps.py --config $c --geometry bilinear --steps 10 2>&1 | tail -1 | cut -c1-100; done; done > gpurun_out/r2_k2b_tab.txt 2>&1
grep -v "^+" gpurun_out/r2_k2b_tab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_k2b_tab_launches.csv python tools/run_steps.py --config C3 --geometry bilinear --steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
