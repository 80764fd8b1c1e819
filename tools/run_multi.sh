#!/bin/bash
# GPU-box helper: one multi-GPU bench line per C (NG GPUs), compact summary.
NG=${NG:-2}
for C in ${CS:-1 2}; do
  timeout -s KILL ${TO:-150} python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 295$NG$C bench.py --gpus $NG --steps ${STEPS:-10} --warmup 3 --C $C --no-e2e $EXTRA 2>gpurun_out/b_p${NG}_c$C.err | tail -1 > gpurun_out/b_p${NG}_c$C.json
  python -c "import json;d=json.load(open('gpurun_out/b_p${NG}_c$C.json'));print('P',d['n_gpus'],'C',d['config']['C'],round(d['value']),round(d['ms_per_step'],2),{k:round(v,2) for k,v in d['kernel_ms_per_step'].items()},d['exposed_comm'],{k:round(v,2) for k,v in d['phase_ms_per_step'].items()})" || tail -5 gpurun_out/b_p${NG}_c$C.err
done
