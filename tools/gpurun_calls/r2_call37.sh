# round-2: DMMA position-owned combine v4 (incremental decode over a warp's consecutive groups,
# cp.async staging, rows-first class alignment): parity, A/B, ncu
set -x
V=build/var
export LAMFAST_LIB=$V/mma4/liblamfast_b200.so
LAMFAST_COMBINE=pos timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_acceptance.py tests/test_gpu_ranges.py -q -x -m gpu > gpurun_out/r2_tests_mma4.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2_tests_mma4.log
run() { timeout 200 python tools/run_steps.py --config $1 --steps 20 $2 $3 $4 2>&1 | tail -1 | cut -c1-150; }
(
for rep in 1 2; do for c in C4 C3; do
  echo -n "entry $c: "; run $c
  echo -n "mma4 G8 $c: "; LAMFAST_COMBINE=pos run $c
  echo -n "mma4 G8 smem40 $c: "; LAMFAST_COMBINE=pos LAMFAST_POS_SMEM_KB=40 run $c
  echo -n "mma4 G4 $c: "; LAMFAST_COMBINE=pos LAMFAST_LIB=$V/mma4g4/liblamfast_b200.so run $c
  echo -n "mma4 G16 $c: "; LAMFAST_COMBINE=pos LAMFAST_LIB=$V/mma4g16/liblamfast_b200.so run $c
  echo -n "mma4 storeonly $c: "; LAMFAST_COMBINE=pos LAMFAST_LIB=$V/mma4so/liblamfast_b200.so run $c
done; done
echo -n "entry C5/64: "; run C5 --plies 64
echo -n "mma4 C5/64: "; LAMFAST_COMBINE=pos run C5 --plies 64
echo -n "mma4 G16 C5/64: "; LAMFAST_COMBINE=pos LAMFAST_LIB=$V/mma4g16/liblamfast_b200.so run C5 --plies 64
echo -n "entry C2: "; run C2
echo -n "mma4 C2: "; LAMFAST_COMBINE=pos run C2
) > gpurun_out/r2_mma4_ab.txt 2>&1
grep -v "^+" gpurun_out/r2_mma4_ab.txt
LAMFAST_COMBINE=pos LAMFAST_POS_DEBUG=1 timeout 120 python tools/run_steps.py --config C5 --plies 64 --steps 1 2>&1 | grep -E "combine_pos|job" | head -12 > gpurun_out/r2_mma4_jobs_c5.txt
LAMFAST_COMBINE=pos timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_mma -c 1 -o gpurun_out/r2_mma4_c4 -f python tools/run_steps.py --config C4 --steps 1 > gpurun_out/ncu_mma4.log 2>&1; echo "ncu rc=$?"
