# round-2 checkpoint: smoke, full GPU suite, default bench, 2-rank gloo code-path line
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r2_gputests_full.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2_gputests_full.log
timeout 900 python bench.py > gpurun_out/r2_bench_ckpt.json 2> gpurun_out/r2_bench_ckpt.err; echo "bench rc=$?"; tail -c 400 gpurun_out/r2_bench_ckpt.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 > gpurun_out/r2_bench_2rank_gloo.json 2> gpurun_out/r2_bench_2rank_gloo.err; echo "2rank rc=$?"; tail -c 600 gpurun_out/r2_bench_2rank_gloo.err
