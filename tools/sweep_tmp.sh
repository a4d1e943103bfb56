for c in C3 C4 C2; do
  echo -n "$c bilinear "; python tools/run_steps.py --config $c --geometry bilinear --steps 10 2>&1 | tail -1
  echo -n "$c "; python tools/run_steps.py --config $c --steps 10 2>&1 | tail -1
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x 2>&1 | tail -1
