# round-2: position-owned combine, variants (straight-line term sets, store-only bound, one position per thread) + ncu
set -x
V=build/var
run() { timeout 120 python tools/run_steps.py --config $1 --steps 20 2>&1 | tail -1 | cut -c1-150; }
(
for rep in 1 2; do for c in C4 C3; do
  echo -n "entry $c: "; LAMFAST_COMBINE=entry run $c
  echo -n "pos switch $c: "; run $c
  echo -n "pos switch smem100 $c: "; LAMFAST_POS_SMEM_KB=100 run $c
  echo -n "pos noswitch $c: "; LAMFAST_LIB=$V/noswitch/liblamfast_b200.so run $c
  echo -n "pos storeonly $c: "; LAMFAST_LIB=$V/storeonly/liblamfast_b200.so run $c
  echo -n "pos storeonly A=1 $c: "; LAMFAST_POS_ALIGN=1 LAMFAST_LIB=$V/storeonly/liblamfast_b200.so run $c
  echo -n "pos storeonly smem100 $c: "; LAMFAST_POS_SMEM_KB=100 LAMFAST_LIB=$V/storeonly/liblamfast_b200.so run $c
  echo -n "pos ept1 minb3 $c: "; LAMFAST_LIB=$V/ept1m3/liblamfast_b200.so run $c
  echo -n "pos ept1 minb4 $c: "; LAMFAST_LIB=$V/ept1m4/liblamfast_b200.so run $c
  echo -n "pos ept1 minb4 smem50 $c: "; LAMFAST_POS_SMEM_KB=50 LAMFAST_LIB=$V/ept1m4/liblamfast_b200.so run $c
done; done
) > gpurun_out/r2_pos_ab2.txt 2>&1
grep -v "^+" gpurun_out/r2_pos_ab2.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_combine_pos -c 1 -o gpurun_out/r2_pos_c4 -f python tools/run_steps.py --config C4 --steps 1 > gpurun_out/ncu_pos.log 2>&1; echo "ncu rc=$?"
