# round-2: combine grid order (row chunks fastest): parity, A/B, t_chunk on the C5 family
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ranges.py tests/test_gpu_fuzz.py tests/test_gpu_debug_checks.py tests/test_gpu_acceptance.py -q -x -m gpu > gpurun_out/r2_tests_gridorder.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_tests_gridorder.log
run() { timeout 300 python tools/run_steps.py --config $1 --steps 20 $2 $3 $4 2>&1 | tail -1 | cut -c1-130; }
(
for rep in 1 2; do for c in C4 C3 C2 "C4 --distinct 16" "C3 --distinct 16"; do
  echo -n "x=entry blocks (before) $c: "; LAMFAST_LIB=build/var/noswap/liblamfast_b200.so run $c
  echo -n "x=row chunks (default) $c: "; run $c
done; done
for tc in 0 48 64 96 128; do
  if [ $tc = 0 ]; then unset LAMFAST_TCHUNK; else export LAMFAST_TCHUNK=$tc; fi
  echo -n "C5/96 plies x=row chunks tchunk=$tc: "; run C5 --plies 96
  echo -n "C5/96 plies x=entry blocks tchunk=$tc: "; LAMFAST_LIB=build/var/noswap/liblamfast_b200.so run C5 --plies 96
done
) > gpurun_out/r2_grid_order.txt 2>&1
grep -v "^+" gpurun_out/r2_grid_order.txt
