for tc in 0 32 43 48 64 65 80 129; do
  echo -n "C3 tchunk=$tc "; LAMFAST_TCHUNK=$tc python tools/run_steps.py --config C3 --steps 20 2>&1 | tail -1
done
for tc in 0 48 52 64; do
  echo -n "C4 tchunk=$tc "; LAMFAST_TCHUNK=$tc python tools/run_steps.py --config C4 --steps 20 2>&1 | tail -1
done
