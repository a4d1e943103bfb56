# round-2: two-phase K6 (local blocks + gather) vs coloured: parity and timing
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_ranges.py tests/test_gpu_debug_checks.py tests/test_gpu_fuzz.py -q -x -m gpu > gpurun_out/r2_tests_k6tp.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_tests_k6tp.log
for rep in 1 2; do for m in twophase coloured; do for c in C3 C4; do echo -n "$m "; LAMFAST_K6=$m timeout 300 python tools/k6_ab.py $c 3; done; done; done > gpurun_out/r2_k6_twophase.txt 2>&1
grep standard gpurun_out/r2_k6_twophase.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r2_k6tp_launches.csv python tools/k6_ab.py C3 1 > /dev/null 2>&1; echo "ncu rc=$?"
