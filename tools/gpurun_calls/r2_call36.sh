# round-2: DMMA position-owned combine v3 (split operands per neighbour, 4 position groups per warp,
# 32-bit shared addressing): parity with LAMFAST_COMBINE=pos, A/B against the entry-owned kernel, ncu
set -x
V=build/var
export LAMFAST_LIB=$V/mma3/liblamfast_b200.so
LAMFAST_COMBINE=pos timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_acceptance.py tests/test_gpu_ranges.py -q -x -m gpu > gpurun_out/r2_tests_mma3.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2_tests_mma3.log
run() { timeout 120 python tools/run_steps.py --config $1 --steps 20 $2 $3 $4 2>&1 | tail -1 | cut -c1-150; }
LAMFAST_COMBINE=pos LAMFAST_POS_DEBUG=1 timeout 120 python tools/run_steps.py --config C4 --steps 1 2>&1 | grep -E "combine_pos|job" | head -12 > gpurun_out/r2_mma3_jobs.txt
(
for rep in 1 2; do for c in C4 C3; do
  echo -n "entry $c: "; run $c
  echo -n "mma3 $c: "; LAMFAST_COMBINE=pos run $c
  echo -n "mma3 A=4 $c: "; LAMFAST_COMBINE=pos LAMFAST_POS_ALIGN=4 run $c
  echo -n "mma3 smem40 $c: "; LAMFAST_COMBINE=pos LAMFAST_POS_SMEM_KB=40 run $c
  echo -n "mma3 G1 $c: "; LAMFAST_COMBINE=pos LAMFAST_LIB=$V/mma3g1/liblamfast_b200.so run $c
  echo -n "mma3 G8 $c: "; LAMFAST_COMBINE=pos LAMFAST_LIB=$V/mma3g8/liblamfast_b200.so run $c
  echo -n "mma3 storeonly $c: "; LAMFAST_COMBINE=pos LAMFAST_LIB=$V/mma3so/liblamfast_b200.so run $c
done; done
echo -n "entry C5/32: "; run C5 --plies 32
echo -n "mma3 C5/32: "; LAMFAST_COMBINE=pos run C5 --plies 32
echo -n "entry C2: "; run C2
echo -n "mma3 C2: "; LAMFAST_COMBINE=pos run C2
) > gpurun_out/r2_mma3_ab.txt 2>&1
grep -v "^+" gpurun_out/r2_mma3_ab.txt
LAMFAST_COMBINE=pos timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_mma -c 1 -o gpurun_out/r2_mma3_c4 -f python tools/run_steps.py --config C4 --steps 1 > gpurun_out/ncu_mma3.log 2>&1; echo "ncu rc=$?"
