for c in C4 C3; do for tc in 0 32 48 64 80 96 128; do echo -n "tchunk=$tc "; LAMFAST_TCHUNK=$tc python tools/run_steps.py --config $c --steps 20; done; done
