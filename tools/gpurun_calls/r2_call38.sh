# round-2: drop-in CSR vectors sized without a zero fill: drop-in tests, reference suites, drop-in e2e (C4, C3)
set -x
timeout 900 python -m pytest tests/test_dropin.py tests/test_reftests.py -q -x -m gpu > gpurun_out/r2_tests_dropin_uninit.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_tests_dropin_uninit.log
(
echo "# build/dropin_e2e: lamfast::assembleFast -> StiffnessMatrix (std::vector). uninit = default (vectors sized without a zero fill), zero = LAMFAST_DROPIN_ZERO_FILL=1 (value-initialising resize, round-2 checkpoint behaviour)"
for rep in 1 2; do
echo -n "uninit C4: "; timeout 300 build/dropin_e2e C4 3
echo -n "zero   C4: "; LAMFAST_DROPIN_ZERO_FILL=1 timeout 300 build/dropin_e2e C4 3
done
echo -n "uninit C3: "; timeout 300 build/dropin_e2e C3 3
echo -n "zero   C3: "; LAMFAST_DROPIN_ZERO_FILL=1 timeout 300 build/dropin_e2e C3 3
) > gpurun_out/r2_dropin_e2e_uninit.txt 2>&1
cat gpurun_out/r2_dropin_e2e_uninit.txt
