# round-2: slot form with branch-free two-slot rows (L_t = 3 / 3 and 5): A/B
set -x
V=build/var
run() { timeout 200 python tools/run_steps.py --config $1 --steps 20 $2 $3 $4 2>&1 | tail -1 | cut -c1-150; }
(
for rep in 1 2; do for c in "C4 --distinct 16" "C4 --distinct 6" "C3 --distinct 16" "C3 --distinct 6"; do
  echo -n "$c default: "; run $c
  echo -n "$c masked L3: "; LAMFAST_LIB=$V/slm3/liblamfast_b200.so run $c
  echo -n "$c masked L3+5: "; LAMFAST_LIB=$V/slm35/liblamfast_b200.so run $c
done; done
for c in C4 C3; do
  echo -n "$c native per-term: "; run $c
  echo -n "$c native slots: "; LAMFAST_SLOTS_MIN_TERMS=1 run $c
  echo -n "$c native slots masked L3: "; LAMFAST_SLOTS_MIN_TERMS=1 LAMFAST_LIB=$V/slm3/liblamfast_b200.so run $c
  echo -n "$c native slots masked L3+5: "; LAMFAST_SLOTS_MIN_TERMS=1 LAMFAST_LIB=$V/slm35/liblamfast_b200.so run $c
done
) > gpurun_out/r2_slots_masked.txt 2>&1
grep -v "^+" gpurun_out/r2_slots_masked.txt
