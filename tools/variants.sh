for v in A NK M3 M3NK A NK; do
  if [ $v = A ]; then L=paper_1905_05417_b200/lib/liblamfast_b200.so; else L=build/var$v/lib.so; fi
  for c in C4 C3; do echo -n "$v "; LAMFAST_LIB=$L python tools/run_steps.py --config $c --steps 20; done
done
