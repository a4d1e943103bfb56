for c in C2 C3 C4; do
  for tc in 0 4 8 16 32 64 129 257; do echo -n "tchunk=$tc "; LAMFAST_TCHUNK=$tc python tools/run_steps.py --config $c --steps 20; done
done
