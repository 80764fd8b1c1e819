#!/bin/bash
# GPU-box helper: NCCL P2P settings vs phase bandwidth (P=4, C=2).
run() {
  env "$@" timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29600 bench.py --gpus 4 --steps 5 --warmup 3 --C 2 --no-e2e 2>/dev/null | tail -1 > gpurun_out/env.json
  python -c "import json;d=json.load(open('gpurun_out/env.json'));print('$*', round(d['value']),round(d['ms_per_step'],2),d['exposed_comm']['frac'],{k:round(v,2) for k,v in d['phase_ms_per_step'].items()})"
}
run A=1
run NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32
run NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32 NCCL_P2P_NVL_CHUNKSIZE=4194304
run NCCL_P2P_USE_CUDA_MEMCPY=1
run NCCL_NCHANNELS_PER_PEER=32
