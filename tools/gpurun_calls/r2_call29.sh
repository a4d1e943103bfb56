# round-2: ncu --set full of the C3 per-term combine (NT=4 path) and the C5 family
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_b -c 1 -o gpurun_out/r2_ncu_combine_c3 python tools/run_steps.py --config C3 --steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
