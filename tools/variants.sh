for c in C4 C3 C2; do
  for m in 1 2 3 0; do echo -n "ws=$m "; LAMFAST_WS=$m python tools/run_steps.py --config $c --steps 20; done
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
