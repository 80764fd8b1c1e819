#!/bin/bash
# GPU-box helper: duration, cycles, clock and tensor-pipe share of the block kernels for each
# library given (""= in-tree).  usage: tools/ncu_quick.sh [lib.so ...]
LIBS=("$@"); [ ${#LIBS[@]} -eq 0 ] && LIBS=("")
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for v in "${LIBS[@]}"; do
  echo "== ${v:-main}"
  WF_LIB_PATH=$v timeout -s KILL 300 ncu --metrics $M --clock-control none -k regex:wf_block -s 2 -c 2 --csv python tools/kprof.py 2>/dev/null | \
    python -c "
import csv,sys
rows=[r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
for r in rows[1:]: print(r[ki][:40], r[mi], r[vi])"
done
