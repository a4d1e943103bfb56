# round-2: slot form of the per-term combine (k_combine_slots): parity, A/B against per-term / coefficient forms
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_debug_checks.py tests/test_gpu_ranges.py -q -x -m gpu > gpurun_out/r2_tests_slots.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2_tests_slots.log
run() { timeout 200 python tools/run_steps.py --config $1 --steps 20 $2 $3 $4 2>&1 | tail -1 | cut -c1-150; }
(
for rep in 1 2; do
for n in 5 6 7 8 16; do
  echo -n "C4 distinct $n slots: "; run C4 --distinct $n
  echo -n "C4 distinct $n other: "; LAMFAST_SLOTS_MIN_TERMS=1000 run C4 --distinct $n
done
for n in 6 16; do
  echo -n "C3 distinct $n slots: "; run C3 --distinct $n
  echo -n "C3 distinct $n other: "; LAMFAST_SLOTS_MIN_TERMS=1000 run C3 --distinct $n
done
for c in C4 C3 C2; do
  echo -n "$c native per-term: "; run $c
  echo -n "$c native slots: "; LAMFAST_SLOTS_MIN_TERMS=1 run $c
done
done
echo -n "C5/32 native per-term: "; run C5 --plies 32
echo -n "C5/32 native slots: "; LAMFAST_SLOTS_MIN_TERMS=1 run C5 --plies 32
) > gpurun_out/r2_slots_ab.txt 2>&1
grep -v "^+" gpurun_out/r2_slots_ab.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_slots -c 1 -o gpurun_out/r2_slots_c4d16 -f python tools/run_steps.py --config C4 --distinct 16 --steps 1 > gpurun_out/ncu_slots.log 2>&1; echo "ncu rc=$?"
