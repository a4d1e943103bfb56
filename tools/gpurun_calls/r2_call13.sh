# round-2: C5 function-range cut parity, debug checks, 2-rank gloo line (C5 leg collective-safe)
set -x
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_debug_checks.py -q -x -m gpu --durations=5 > gpurun_out/r2_tests_c5range.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/r2_tests_c5range.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 > gpurun_out/r2_bench_2rank_gloo_v2.json 2> gpurun_out/r2_bench_2rank_gloo_v2.err; echo "2rank rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2_bench_2rank_gloo_v2.json').read().strip().splitlines()[-1])
print(json.dumps(d.get('c5'))[:1500]); print(d['verify'])
PY
