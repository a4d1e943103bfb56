# round-2: coef kernel variants, K6 prefetch A/B, CPU ply trend, reference arm line
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py -q -x -m gpu -k "coefficient or many_terms or decompose or kernel_families or standard or acceptance" > gpurun_out/r2_tests_c5.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_tests_c5.log
for v in ku0 ku1; do for c in C4 C3; do for dec in "" "--decompose"; do echo -n "$v $c $dec: "; LAMFAST_LIB=build/coefv/$v/liblamfast_b200.so LAMFAST_EFORM_MIN_TERMS=1 timeout 120 python tools/run_steps.py --config $c --steps 20 $dec 2>&1 | tail -1 | cut -c1-110; done; done; done > gpurun_out/r2_coef_v2.txt 2>&1
cat gpurun_out/r2_coef_v2.txt
for v in pf0 pf1; do for c in C3 C4; do LAMFAST_LIB=build/k6v/$v/liblamfast_b200.so timeout 300 python tools/k6_ab.py $c 3; done; done > gpurun_out/r2_k6_pf.txt 2>&1
cat gpurun_out/r2_k6_pf.txt
timeout 600 python tools/cpu_ply_trend.py C4 2 9 32 > gpurun_out/r2_cpu_ply_trend.txt 2>&1; cat gpurun_out/r2_cpu_ply_trend.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference_arm.json 2> gpurun_out/r2_bench_reference_arm.err; echo "ref rc=$?"; tail -c 1500 gpurun_out/r2_bench_reference_arm.json
