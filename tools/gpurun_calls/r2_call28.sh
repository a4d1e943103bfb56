# round-2: planar K6 scratch layout
set -x
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_ranges.py tests/test_gpu_acceptance.py tests/test_gpu_parity.py tests/test_gpu_debug_checks.py -q -x -m gpu -k "standard or bitwise or range or acceptance or kernel_families or slab" > gpurun_out/r2_tests_k6planar.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_tests_k6planar.log
for rep in 1 2; do for c in C3 C4; do timeout 300 python tools/k6_ab.py $c 3; done; done > gpurun_out/r2_k6_planar.txt 2>&1
grep standard gpurun_out/r2_k6_planar.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_k6_planar_launches.csv python tools/k6_ab.py C3 1 > /dev/null 2>&1; echo "ncu rc=$?"
