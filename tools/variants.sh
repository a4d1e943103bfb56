python tools/run_steps.py --config C4 --steps 3 --calibrate | head -2
for v in A SO A SO; do
  if [ $v = A ]; then L=paper_1905_05417_b200/lib/liblamfast_b200.so; else L=build/var$v/lib.so; fi
  for c in C4 C3; do echo -n "$v "; LAMFAST_LIB=$L python tools/run_steps.py --config $c --steps 20; done
done
