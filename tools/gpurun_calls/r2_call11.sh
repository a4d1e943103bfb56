# round-2: per-term combine: store-only ceiling of the current pattern, ncu source capture
set -x
for rep in 1 2; do for v in default storeonly; do for c in C4 C3; do
  lib=paper_1905_05417_b200/lib/liblamfast_b200.so; [ $v = storeonly ] && lib=build/ptv/storeonly/liblamfast_b200.so
  echo -n "$v $c: "; LAMFAST_LIB=$lib timeout 120 python tools/run_steps.py --config $c --steps 20 2>&1 | tail -1 | cut -c1-120
done; done; done > gpurun_out/r2_storeonly.txt 2>&1
grep -v "^+" gpurun_out/r2_storeonly.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_b -c 1 -o gpurun_out/r2_ncu_combine_c4 python tools/run_steps.py --config C4 --steps 1 > gpurun_out/r2_ncu_combine.log 2>&1; echo "ncu rc=$?"
