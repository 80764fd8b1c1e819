#!/bin/bash
# GPU-box helper: quick single-GPU bench of library variants, interleaved (R rounds), for the
# GPT (32K causal) and DiT (64K full 16x72) workloads.  usage: tools/qb.sh [lib.so ...]
# ("" = the in-tree libwf.so); WL="gpt dit" selects workloads.
R=${R:-2}
WL=${WL:-gpt dit}
LIBS=("$@"); [ ${#LIBS[@]} -eq 0 ] && LIBS=("")
for r in $(seq $R); do
  for w in $WL; do
    for v in "${LIBS[@]}"; do
      if [ $w = gpt ]; then S=32768; else S=65536; fi
      WF_LIB_PATH=$v timeout -s KILL 180 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e \
        --workload $w --seq $S $EXTRA 2>&1 | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$w', '${v:-main}', 'fwd %.3f bwd %.3f' % (k['block_fwd'], k['block_bwd']), 'fwdTF %.0f bwdTF %.0f' % (d['fwd_kernel_tflops'], d['bwd_kernel_tflops']), 'total %.0f TF/s' % d['value'], 'sm %s MHz' % d['clocks']['sm_mhz'], d['clocks']['reasons'])" || echo "$w ${v:-main} FAILED"
    done
  done
done
