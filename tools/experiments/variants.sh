for c in C4 C3; do
  for m in 1 2 0; do echo -n "ws=$m "; LAMFAST_WS=$m python tools/run_steps.py --config $c --steps 20; done
done
