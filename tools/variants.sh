for c in C4 C3 C2; do
  for m in staged direct tma; do echo -n "$m "; LAMFAST_STORE=$m python tools/run_steps.py --config $c --steps 20; done
done
python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
