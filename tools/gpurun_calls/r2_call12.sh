# round-2: K2b phase-1 pair groups A/B (bilinear geometry), parity
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py -q -x -m gpu -k "skew or general or bilinear or inplane or kernel_families or maximum or mixed" > gpurun_out/r2_tests_k2b.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_tests_k2b.log
for rep in 1 2; do for v in k2p1m2 k2p2m2 k2p4m2 k2p4m1; do for c in C3 C4; do echo -n "$v $c: "; LAMFAST_LIB=build/k2bv/$v/liblamfast_b200.so timeout 120 python tools/run_steps.py --config $c --geometry bilinear --steps 10 2>&1 | tail -1 | cut -c1-120; done; done; done > gpurun_out/r2_k2b_ab.txt 2>&1
grep -v "^+" gpurun_out/r2_k2b_ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_k2b_launches.csv python tools/run_steps.py --config C3 --geometry bilinear --steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
