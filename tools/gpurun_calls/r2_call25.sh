# round-2 final validation: smoke, full GPU suite, default bench, reference arm, launch list, ncu --set full of the bench's top kernel
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_final_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r2_final_gputests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2_final_gputests.log
timeout 900 python bench.py > gpurun_out/r2_final_bench.json 2> gpurun_out/r2_final_bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r2_final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_final_ref.json 2> gpurun_out/r2_final_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline --no-standard > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_combine_b -c 1 -o gpurun_out/r2_final_ncu_combine_c4 python bench.py --steps 1 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline --no-standard > /dev/null 2>&1; echo "ncu2 rc=$?"
