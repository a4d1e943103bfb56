# round-2: 2-rank code-path check of the multi-rank bench line (gloo, both ranks on one GPU), reference arm under torchrun,
# C5 stream and drop-in with the final thread defaults
set -x
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 > gpurun_out/r2_bench_2rank_gloo_final.json 2> gpurun_out/r2_bench_2rank_gloo_final.err; echo "2rank rc=$?"; tail -c 400 gpurun_out/r2_bench_2rank_gloo_final.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2_bench_2rank_gloo_final.json').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','n_gpus','ms_per_step','scaling')}, d['config']['workload'])
print('c5', {k:d['c5'].get(k) for k in ('value','ms_per_step','per_rank_ms','balance')} if d.get('c5') else None)
print('verify', d.get('verify'))
PY
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2_ref_arm_2rank.json 2> gpurun_out/r2_ref_arm_2rank.err; echo "ref 2rank rc=$?"; cat gpurun_out/r2_ref_arm_2rank.json | cut -c1-300
timeout 900 python tools/c5_stream_threads.py default 16 > gpurun_out/r2_c5_stream_threads2.txt 2>&1; tail -2 gpurun_out/r2_c5_stream_threads2.txt
timeout 300 build/dropin_e2e C4 3 | cut -c1-140
