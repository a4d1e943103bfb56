# round-2: NT-store host columns, sink path host columns: tests + e2e
set -x
timeout 900 python -m pytest tests/test_gpu_ranges.py tests/test_dropin.py -q -x -m gpu > gpurun_out/r2_tests_hostcols2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_tests_hostcols2.log
timeout 900 python bench.py --no-standard --no-cpu-baseline --e2e-steps 5 > gpurun_out/r2_bench_hostcols2.json 2> gpurun_out/r2_bench_hostcols2.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r2_bench_hostcols2.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2_bench_hostcols2.json').read().strip().splitlines()[-1])
print(json.dumps(d['e2e'], indent=1)); print(json.dumps(d['e2e_dropin'])); print(json.dumps(d['c5'].get('e2e_stream')))
PY
