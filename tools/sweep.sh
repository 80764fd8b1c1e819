#!/bin/bash
# GPU-box helper: the BASELINE metric grid on the GPUs of one box (NG = 2 or 4):
# GPT 32x128 causal and DiT 16x72 full for every valid C, plus the long-context sweep
# (C = NG vs C = 1).  One JSON line per run -> gpurun_out/sweep_p$NG.jsonl
NG=${NG:-4}
OUT=gpurun_out/sweep_p$NG.jsonl
: > $OUT
run() {  # args: C workload seq
  timeout -s KILL 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $NG --steps 5 --warmup 3 --no-cpu --no-e2e \
    --C $1 --workload $2 --seq $3 2>/dev/null | grep '^{' >> $OUT || echo "{\"failed\": \"C=$1 $2 N=$3\"}" >> $OUT
}
for C in 1 2 4; do
  [ $((NG % C)) -ne 0 ] && continue
  run $C gpt 0
  run $C dit 0
done
for N in 16384 65536 131072 262144 524288; do
  run 1 gpt $N
  run $NG gpt $N
done
python - <<'PY'
import json, os
p = f"gpurun_out/sweep_p{os.environ.get('NG', '4')}.jsonl"
for line in open(p):
    d = json.loads(line)
    if "failed" in d:
        print("FAILED", d["failed"]); continue
    c, pa = d["config"], d["parallel"]; ex = d.get("exposed_comm") or {}
    print(f"{c['workload'][:38]:38} P={pa['P']} C={pa['C']} {d['tflops_per_gpu']:7.1f} TF/s/GPU "
          f"frac(burst) {d['frac_of_peak_per_gpu']['burst']:.3f} bwd-kernel {d['roofline']['frac']:.3f} "
          f"exposed {ex.get('frac', 0):.3f}")
PY
