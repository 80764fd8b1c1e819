#!/bin/bash
# GPU-box helper: fwd kernel cycles for each library given ("" = in-tree), with the
# environment of the caller (e.g. WF_FWD_SPLIT=1)
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for v in "$@"; do
  echo "== ${v:-main}"
  WF_LIB_PATH=$v timeout -s KILL 300 ncu --metrics $M --clock-control none -k regex:wf_block_fwd -s 1 -c 1 --csv python tools/kprof.py 2>/dev/null | \
    python -c "
import csv,sys
rows=[r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value'); ki=h.index('Kernel Name')
print(rows[1][ki][:36], ' '.join(r[mi].split('.')[0]+'='+r[vi] for r in rows[1:]))"
done
