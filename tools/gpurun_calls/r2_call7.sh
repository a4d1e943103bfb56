# round-2: coef staging rewrite; NS variants; NS=2 parity
set -x
LAMFAST_LIB=build/coefv/ns2a/liblamfast_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "coefficient or many_terms or decompose" > gpurun_out/r2_tests_ns2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_tests_ns2.log
for rep in 1 2; do for v in ns1 ns2a ns2d; do for c in C4 C3; do echo -n "$v $c: "; LAMFAST_LIB=build/coefv/$v/liblamfast_b200.so LAMFAST_EFORM_MIN_TERMS=1 timeout 120 python tools/run_steps.py --config $c --steps 20 2>&1 | tail -1 | cut -c1-110; done; done; done > gpurun_out/r2_coef_ns_v3.txt 2>&1
grep -v "^+" gpurun_out/r2_coef_ns_v3.txt
