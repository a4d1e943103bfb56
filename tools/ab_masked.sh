# A/B of combine-kernel build variants: build/var_*/liblamfast_b200.so vs the default lib.
# Build a variant first, e.g.
#   make -C paper_1905_05417_b200/csrc BUILD=../../build/var_sh OUT=../../build/var_sh/liblamfast_b200.so \
#        EXTRA=-DLF_SH32 ../../build/var_sh/liblamfast_b200.so
# usage: bash tools/ab_masked.sh "default old sh" "C4 C3"
VARS=${1:-"default old"}
CFGS=${2:-"C4 C3"}
for rep in 1 2; do
for c in $CFGS; do
  for v in $VARS; do
    lib=build/var_$v/liblamfast_b200.so; [ $v = default ] && lib=paper_1905_05417_b200/lib/liblamfast_b200.so
    extra=""; [ $c = C5 ] && extra="--plies 32"
    echo -n "$v "; LAMFAST_LIB=$lib python tools/run_steps.py --config $c --steps 20 $extra
  done
done
done
