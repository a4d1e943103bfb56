# round-2: K6 phase 1 with constant-bank tables (affine) vs shared-memory tables
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_debug_checks.py -q -x -m gpu > gpurun_out/r2_tests_k6c.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_tests_k6c.log
for rep in 1 2; do for m in 1 0; do for c in C3 C4; do echo -n "const=$m "; LAMFAST_K6_CONST=$m timeout 300 python tools/k6_ab.py $c 3; done; done; done > gpurun_out/r2_k6_const.txt 2>&1
grep standard gpurun_out/r2_k6_const.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_standard_local -c 1 -o gpurun_out/r2_ncu_k6local_c3 python tools/k6_ab.py C3 1 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench_c4_v3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline --no-standard > /dev/null 2>&1; echo "ncu2 rc=$?"
