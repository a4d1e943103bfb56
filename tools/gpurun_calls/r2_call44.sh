# round-2 final validation (2): smoke, full GPU suite, default bench, reference arm, launch list, ncu --set full
# of the bench's top kernel, per-config bench lines, C5 stream against the column threads
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_final2_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r2_final2_gputests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2_final2_gputests.log
timeout 900 python bench.py > gpurun_out/r2_final2_bench.json 2> gpurun_out/r2_final2_bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r2_final2_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_final2_ref.json 2> gpurun_out/r2_final2_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_final2_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline --no-standard > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_combine_b -c 1 -o gpurun_out/r2_final2_ncu_combine_c4 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline --no-standard > /dev/null 2>&1; echo "ncu2 rc=$?"
timeout 600 python bench.py --config C3 --no-c5 --no-dropin --no-cpu-baseline > gpurun_out/r2_final2_bench_c3.json 2> /dev/null; echo "c3 rc=$?"
timeout 900 python tools/c5_stream_threads.py default 8 6 > gpurun_out/r2_c5_stream_threads.txt 2>&1; cat gpurun_out/r2_c5_stream_threads.txt | tail -4
