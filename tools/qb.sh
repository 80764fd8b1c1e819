#!/bin/bash
# GPU-box helper: quick single-GPU bench of library variants, interleaved (R rounds).
# usage: tools/qb.sh [lib.so ...]   ("" = the in-tree libwf.so)
R=${R:-2}
LIBS=("$@"); [ ${#LIBS[@]} -eq 0 ] && LIBS=("")
for r in $(seq $R); do
  for v in "${LIBS[@]}"; do
    WF_LIB_PATH=$v timeout -s KILL 120 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e $EXTRA 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('${v:-main}', 'fwd %.2f bwd %.2f' % (k['block_fwd'], k['block_bwd']), 'total %.0f TF/s' % d['value'], 'sm %s MHz' % d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
