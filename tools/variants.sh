nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/var_clocks.csv &
SMI=$!
nvidia-smi -q | grep -iE "serial|bus id|product name" | head -4
python tools/run_steps.py --config C4 --steps 10 --calibrate
for v in A C A C; do
  if [ $v = A ]; then L=paper_1905_05417_b200/lib/liblamfast_b200.so; else L=build/var$v/lib.so; fi
  for c in C4 C3; do echo -n "$v "; LAMFAST_LIB=$L python tools/run_steps.py --config $c --steps 20; done
done
kill $SMI
