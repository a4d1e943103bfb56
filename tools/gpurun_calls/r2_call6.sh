# round-2: coef sets-per-thread variants; per-term vs coef threshold sweep
set -x
for v in ns1 ns2a ns2b ns2c; do for c in C4 C3; do echo -n "$v $c: "; LAMFAST_LIB=build/coefv/$v/liblamfast_b200.so LAMFAST_EFORM_MIN_TERMS=1 timeout 120 python tools/run_steps.py --config $c --steps 20 2>&1 | tail -1 | cut -c1-110; done; done > gpurun_out/r2_coef_ns.txt 2>&1
cat gpurun_out/r2_coef_ns.txt
for c in C4 C3; do for n in 3 4 5 6 7 8; do for m in 1000 1; do echo -n "$c distinct=$n min_terms=$m: "; LAMFAST_EFORM_MIN_TERMS=$m timeout 120 python tools/run_steps.py --config $c --distinct $n --steps 20 2>&1 | tail -1 | cut -c1-110; done; done; done > gpurun_out/r2_coef_threshold.txt 2>&1
cat gpurun_out/r2_coef_threshold.txt
LAMFAST_LIB=build/coefv/ns2a/liblamfast_b200.so LAMFAST_EFORM_MIN_TERMS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_coef -c 1 -o gpurun_out/r2_ncu_coef_ns2a_c4 python tools/run_steps.py --config C4 --steps 1 > gpurun_out/r2_ncu_coef2.log 2>&1; echo "ncu rc=$?"
