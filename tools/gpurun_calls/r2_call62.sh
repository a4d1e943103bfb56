# round-2: grid order + ~100-row chunks for many entry blocks: full-size parity, timing
set -x
timeout 2400 python -m pytest tests -q -x -m gpu > gpurun_out/r2_tests_gridorder2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_tests_gridorder2.log
run() { timeout 300 python tools/run_steps.py --config $1 --steps 20 $2 $3 $4 2>&1 | tail -1 | cut -c1-130; }
(
for rep in 1 2; do for c in C4 C3 "C5 --plies 96" "C5 --plies 64" "C5 --plies 32"; do
  echo -n "before (x=entry blocks, 48-row chunks) $c: "; LAMFAST_TCHUNK=48 LAMFAST_LIB=build/var/noswap/liblamfast_b200.so run $c
  echo -n "default $c: "; run $c
done; done
) > gpurun_out/r2_grid_order2.txt 2>&1
grep -v "^+" gpurun_out/r2_grid_order2.txt
timeout 900 python bench.py --no-e2e --no-dropin --no-cpu-baseline --no-standard > gpurun_out/r2_bench_gridorder.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/r2_bench_gridorder.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['c5']['value'],d['c5']['ms_per_step'],d['c5']['roofline']['frac'],d['clocks'])"
