# A/B of the general-geometry in-plane operators (K2b), all two-phase except the last:
# register-blocked element kernel (default), scalar element kernel, DMMA element kernel,
# coloured in-place form.
for c in C3 C4 C2; do
  for v in default scalar mma coloured; do
    echo -n "$v "; LAMFAST_K2B=$v python tools/run_steps.py --config $c --geometry bilinear --steps 10
  done
done
