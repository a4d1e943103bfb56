# Re-measures every number the round's profiles/ summaries quote (one B200), into gpurun_out/:
#   bench lines C4 (default, full), C3, C5; per-config report CSV (fast / standard / Voigt-free);
#   bilinear-map (general in-plane path) steps; launch list of the default bench command.
set -x
python bench.py > gpurun_out/r2rr_bench_c4.log 2>&1
python bench.py --config C3 --no-e2e --no-cpu-baseline --no-standard > gpurun_out/r2rr_bench_c3.log 2>&1
python bench.py --config C5 --no-e2e --no-cpu-baseline --no-standard --steps 10 > gpurun_out/r2rr_bench_c5.log 2>&1
python -m paper_1905_05417_b200.report --configs C1 C2 C3 C4 --backends fast standard voigt_free --repetitions 3 > gpurun_out/r2rr_report.csv 2> gpurun_out/r2rr_report.err
for c in C2 C3 C4; do python tools/run_steps.py --config $c --geometry bilinear --steps 10; done > gpurun_out/r2rr_bilinear.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2rr_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-standard > /dev/null 2>&1
