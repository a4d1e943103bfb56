# round-2: full GPU suite + default bench on the restored default (entry-owned combine)
set -x
timeout 2400 python -m pytest tests -q -x -m gpu > gpurun_out/r2_gputests_call35.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_gputests_call35.log
timeout 600 python bench.py > gpurun_out/r2_bench_call35.json 2> gpurun_out/r2_bench_call35.err; echo "bench rc=$?"; cat gpurun_out/r2_bench_call35.json | cut -c1-600
