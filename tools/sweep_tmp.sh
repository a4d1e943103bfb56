for c in C4 C3 C2 C1; do
  echo -n "$c "; python tools/run_steps.py --config $c --steps 20 2>&1 | tail -1
done
echo -n "C5p32 "; python tools/run_steps.py --config C5 --plies 32 --steps 10 2>&1 | tail -1
echo -n "C4 bilinear "; python tools/run_steps.py --config C4 --geometry bilinear --steps 10 2>&1 | tail -1
python -m pytest tests -m gpu -q -x 2>&1 | tail -2
