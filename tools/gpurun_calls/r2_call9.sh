# round-2: host-written columns for one-shot calls: tests + e2e A/B
set -x
timeout 900 python -m pytest tests/test_gpu_ranges.py tests/test_dropin.py tests/test_reftests.py tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/r2_tests_hostcols.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_tests_hostcols.log
timeout 900 python bench.py --no-c5 --no-standard --no-cpu-baseline --e2e-steps 5 > gpurun_out/r2_bench_hostcols.json 2> gpurun_out/r2_bench_hostcols.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r2_bench_hostcols.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2_bench_hostcols.json').read().strip().splitlines()[-1])
print(json.dumps(d['e2e'], indent=1)); print(json.dumps(d['e2e_dropin']))
PY
