# round-2 last run on the final library: smoke, GPU suite, default bench line, launch list, ncu of the top kernel
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r2_last_gputests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_last_gputests.log
timeout 900 python bench.py > gpurun_out/r2_last_bench.json 2> gpurun_out/r2_last_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_last_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline --no-standard > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_combine_b -c 1 -o gpurun_out/r2_last_ncu_combine_c4 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-c5 --no-dropin --no-cpu-baseline --no-standard > /dev/null 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_combine_b -c 1 -o gpurun_out/r2_last_ncu_combine_c3 -f python tools/run_steps.py --config C3 --steps 1 > /dev/null 2>&1; echo "ncu3 rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2_last_bench.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['pcie_frac'], d['e2e_dropin']['ms_mean'], {k:(round(v['ms_per_step'],3),v['form']) for k,v in d['many_terms'].items()}, d['c5']['value'], d['c5']['ms_per_step'], d['c5']['roofline']['frac'], d['c5']['e2e_stream']['ms'], d['clocks'])
PY
