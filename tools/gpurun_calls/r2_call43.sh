# round-2: drop-in e2e against the host thread counts (columns, staging copies); C-ABI e2e with the new default
set -x
(
echo "# build/dropin_e2e C4 2 (ms_mean) against LAMFAST_COL_THREADS x LAMFAST_COPY_THREADS; default = columns 4 (quarter of 16 cores), copies 16"
echo -n "default: "; timeout 300 build/dropin_e2e C4 2 | cut -c1-120
for col in 2 4 8; do for cp in 4 8 12 16; do
  echo -n "col $col copy $cp: "; LAMFAST_COL_THREADS=$col LAMFAST_COPY_THREADS=$cp timeout 300 build/dropin_e2e C4 2 | cut -c1-120
done; done
) > gpurun_out/r2_dropin_threads.txt 2>&1
grep -v "^+" gpurun_out/r2_dropin_threads.txt
timeout 600 python tools/e2e_col_threads.py C4 2>&1 | head -3
