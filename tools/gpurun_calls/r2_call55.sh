# round-2 closing refresh of the per-config numbers and the slot-form ncu
set -x
timeout 900 python bench.py --config C5 --no-e2e --no-cpu-baseline --no-standard --no-dropin --steps 10 > gpurun_out/r2_closing_bench_c5.json 2> /dev/null; echo "c5 rc=$?"
timeout 1200 python -m paper_1905_05417_b200.report --configs C1 C2 C3 C4 --backends fast standard voigt_free --repetitions 3 > gpurun_out/r2_closing_report.csv 2> gpurun_out/r2_closing_report.err; echo "report rc=$?"
for c in C2 C3 C4; do timeout 200 python tools/run_steps.py --config $c --geometry bilinear --steps 10 2>&1 | tail -1; done > gpurun_out/r2_closing_bilinear.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_slots -c 1 -o gpurun_out/r2_slots3_c4d16 -f python tools/run_steps.py --config C4 --distinct 16 --steps 1 > /dev/null 2>&1; echo "ncu rc=$?"
cat gpurun_out/r2_closing_bilinear.txt; head -20 gpurun_out/r2_closing_report.csv
