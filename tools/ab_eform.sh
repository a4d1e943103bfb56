# A/B of the combine's coefficient form (E-form) against the per-term form
# (LAMFAST_EFORM_MIN_TERMS picks the smallest term count that takes the
# E-form; 1000 = never, i.e. per-term with read-modify-write passes above 8).
s=${STEPS:-20}
for rep in 1 2; do
for c in C4 C3; do
  for m in 1000 1; do
    echo -n "$c default min_terms=$m "; LAMFAST_EFORM_MIN_TERMS=$m python tools/run_steps.py --config $c --steps $s 2>&1 | tail -1
    echo -n "$c decompose min_terms=$m "; LAMFAST_EFORM_MIN_TERMS=$m python tools/run_steps.py --config $c --decompose --steps $s 2>&1 | tail -1
  done
  for n in 8 16; do
    for m in 1000 1; do
      echo -n "$c distinct=$n min_terms=$m "; LAMFAST_EFORM_MIN_TERMS=$m python tools/run_steps.py --config $c --distinct $n --steps $s 2>&1 | tail -1
    done
  done
done
done
