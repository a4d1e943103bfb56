# A/B of the general-geometry in-plane operators (K2b): two-phase with the scalar element
# kernel (default), two-phase with the DMMA element kernel, coloured in-place form.
for c in C3 C4 C2; do
  for v in default mma coloured; do
    echo -n "$v "; LAMFAST_K2B=$v python tools/run_steps.py --config $c --geometry bilinear --steps 10
  done
done
