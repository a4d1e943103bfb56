# round-2: DMMA position-owned combine, rows ordered by term mask + contiguous weight staging: parity, A/B, ncu
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py tests/test_gpu_fuzz.py tests/test_gpu_acceptance.py tests/test_gpu_ranges.py -q -x -m gpu > gpurun_out/r2_tests_mma2.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2_tests_mma2.log
V=build/var
run() { timeout 120 python tools/run_steps.py --config $1 --steps 20 $2 $3 $4 2>&1 | tail -1 | cut -c1-150; }
(
for rep in 1 2; do for c in C4 C3; do
  echo -n "entry $c: "; LAMFAST_COMBINE=entry run $c
  echo -n "mma $c: "; run $c
  echo -n "mma A=32 $c: "; LAMFAST_POS_ALIGN=32 run $c
  echo -n "mma A=4 $c: "; LAMFAST_POS_ALIGN=4 run $c
  echo -n "mma smem40 $c: "; LAMFAST_POS_SMEM_KB=40 run $c
  echo -n "mma ntile8 $c: "; LAMFAST_LIB=$V/nt8m2/liblamfast_b200.so run $c
  echo -n "mma ntile4 minb4 smem50 $c: "; LAMFAST_POS_SMEM_KB=50 LAMFAST_LIB=$V/nt4m4/liblamfast_b200.so run $c
done; done
echo -n "entry C2: "; LAMFAST_COMBINE=entry run C2
echo -n "mma C2: "; run C2
echo -n "entry C5/32: "; LAMFAST_COMBINE=entry run C5 --plies 32
echo -n "mma C5/32: "; run C5 --plies 32
echo -n "entry C4 bilinear: "; LAMFAST_COMBINE=entry run C4 --geometry bilinear
echo -n "mma C4 bilinear: "; run C4 --geometry bilinear
for n in 5 7; do
echo -n "entry C4 distinct $n: "; LAMFAST_COMBINE=entry run C4 --distinct $n
echo -n "mma C4 distinct $n: "; run C4 --distinct $n
done
) > gpurun_out/r2_mma_ab2.txt 2>&1
grep -v "^+" gpurun_out/r2_mma_ab2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_mma -c 1 -o gpurun_out/r2_mma2_c4 -f python tools/run_steps.py --config C4 --steps 1 > gpurun_out/ncu_mma.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_mma -c 1 -o gpurun_out/r2_mma2_c3 -f python tools/run_steps.py --config C3 --steps 1 > gpurun_out/ncu_mma.log 2>&1; echo "ncu rc=$?"
