# round-2 closing run on the final commit: smoke, full GPU suite, default bench line
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/r2_closing_gputests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2_closing_gputests.log
timeout 900 python bench.py > gpurun_out/r2_closing_bench.json 2> gpurun_out/r2_closing_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2_closing_bench.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['pcie_frac'], d['e2e_dropin']['ms_mean'], {k:(v['ms_per_step'],v['form']) for k,v in d['many_terms'].items()}, d['c5']['value'], d['c5']['e2e_stream']['ms'], d['clocks'])
PY
