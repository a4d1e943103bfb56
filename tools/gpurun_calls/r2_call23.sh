# round-2: ncu of the K2b element kernel and gather (C3 bilinear)
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_inplane -c 2 -o gpurun_out/r2_ncu_k2b_c3 python tools/run_steps.py --config C3 --geometry bilinear --steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
