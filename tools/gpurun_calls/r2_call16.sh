# round-2 checkpoint 2: smoke, full GPU suite, default bench, launch list, ncu of the bench's top kernel
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke2.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke2.log
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/r2_gputests_full2.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/r2_gputests_full2.log
timeout 900 python bench.py > gpurun_out/r2_bench_ckpt2.json 2> gpurun_out/r2_bench_ckpt2.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r2_bench_ckpt2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches_bench_c4_v2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline > gpurun_out/r2_ncu_launch2.log 2>&1; echo "ncu rc=$?"
