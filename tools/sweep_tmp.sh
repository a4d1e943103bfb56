for tc in 0 32 48 64 80 96 128 257; do
  echo -n "C4 tchunk=$tc "; LAMFAST_TCHUNK=$tc python tools/run_steps.py --config C4 --steps 20 2>&1 | tail -1
done
for tc in 0 32 64 129; do
  echo -n "C3 tchunk=$tc "; LAMFAST_TCHUNK=$tc python tools/run_steps.py --config C3 --steps 20 2>&1 | tail -1
done
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
