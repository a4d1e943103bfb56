# round-2: decompose_angles folded per ply configuration on affine maps: full GPU suite, timing
set -x
timeout 2400 python -m pytest tests -q -x -m gpu > gpurun_out/r2_tests_fold.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/r2_tests_fold.log
run() { timeout 200 python tools/run_steps.py --config $1 --steps 20 $2 $3 $4 2>&1 | tail -1 | cut -c1-150; }
(
for rep in 1 2; do for c in C4 C3 C2; do
  echo -n "$c direct: "; run $c
  echo -n "$c decompose folded: "; run $c --decompose
  echo -n "$c decompose unfolded (coefficient form): "; LAMFAST_FOLD_DECOMPOSE=0 run $c --decompose
done; done
echo -n "C4 16 angles decompose folded: "; run C4 --distinct 16 --decompose
echo -n "C4 16 angles decompose unfolded: "; LAMFAST_FOLD_DECOMPOSE=0 run C4 --distinct 16 --decompose
) > gpurun_out/r2_fold_ab.txt 2>&1
grep -v "^+" gpurun_out/r2_fold_ab.txt
