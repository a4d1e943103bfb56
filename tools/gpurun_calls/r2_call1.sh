set -x
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2_bench_default.err
STEPS=20 timeout 900 bash tools/ab_eform.sh > gpurun_out/r2_eform.txt 2>&1; echo "eform rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline --no-standard > gpurun_out/r2_ncu_launch.log 2>&1; echo "ncu rc=$?"
