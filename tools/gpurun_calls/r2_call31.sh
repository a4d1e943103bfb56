# round-2: position-owned combine (k_combine_pos): parity, then A/B against the entry-owned kernel
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py tests/test_gpu_fuzz.py tests/test_gpu_acceptance.py tests/test_gpu_ranges.py -q -x -m gpu > gpurun_out/r2_tests_pos.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2_tests_pos.log
LAMFAST_POS_DEBUG=1 timeout 120 python tools/run_steps.py --config C4 --steps 1 2>&1 | grep -E "combine_pos|job|step" | head -40 > gpurun_out/r2_pos_jobs_c4.txt
LAMFAST_POS_DEBUG=1 timeout 120 python tools/run_steps.py --config C3 --steps 1 2>&1 | grep -E "combine_pos|job|step" | head -60 > gpurun_out/r2_pos_jobs_c3.txt
(
timeout 120 python tools/run_steps.py --config C4 --steps 1 --calibrate | grep calibrate
for rep in 1 2; do for c in C4 C3; do
  echo -n "entry $c: "; LAMFAST_COMBINE=entry timeout 120 python tools/run_steps.py --config $c --steps 20 2>&1 | tail -1
  for A in 0 32 16 4 1; do
    echo -n "pos A=$A $c: "; LAMFAST_POS_ALIGN=$A timeout 120 python tools/run_steps.py --config $c --steps 20 2>&1 | tail -1
  done
done; done
for c in C2 C1; do
  echo -n "entry $c: "; LAMFAST_COMBINE=entry timeout 120 python tools/run_steps.py --config $c --steps 50 2>&1 | tail -1
  echo -n "pos $c: "; timeout 120 python tools/run_steps.py --config $c --steps 50 2>&1 | tail -1
done
echo -n "entry C5/32: "; LAMFAST_COMBINE=entry timeout 200 python tools/run_steps.py --config C5 --plies 32 --steps 10 2>&1 | tail -1
echo -n "pos C5/32: "; timeout 200 python tools/run_steps.py --config C5 --plies 32 --steps 10 2>&1 | tail -1
echo -n "entry C4 bilinear: "; LAMFAST_COMBINE=entry timeout 200 python tools/run_steps.py --config C4 --geometry bilinear --steps 10 2>&1 | tail -1
echo -n "pos C4 bilinear: "; timeout 200 python tools/run_steps.py --config C4 --geometry bilinear --steps 10 2>&1 | tail -1
for n in 5 7; do
echo -n "entry C4 distinct $n: "; LAMFAST_COMBINE=entry timeout 200 python tools/run_steps.py --config C4 --distinct $n --steps 10 2>&1 | tail -1
echo -n "pos C4 distinct $n: "; timeout 200 python tools/run_steps.py --config C4 --distinct $n --steps 10 2>&1 | tail -1
done
) > gpurun_out/r2_pos_ab.txt 2>&1
cat gpurun_out/r2_pos_ab.txt | cut -c1-200
