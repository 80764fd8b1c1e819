"""GPU-box helper: WallFacer Transformer layer (GPT-7B shape: hidden 4096, 32 x 128, FFN
16384 = 4H, causal; LayerNorm + GELU FeedForward) forward + backward throughput, tokens/s and model TFLOP/s, max over ranks.

    python tools/layer_bench.py [--N 32768]
    torchrun --nproc-per-node 4 tools/layer_bench.py --N 65536 --C 2
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00611_b200 as wf  # noqa: E402
from paper_2407_00611_b200.layer import LayerWeights, WallFacerLayer, layer_flops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=32768)
    ap.add_argument("--C", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--no-checkpoint", action="store_true")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    H, h, d, F = 4096, 32, 128, 4 * 4096
    N, P = a.N, world
    n = N // P
    W = LayerWeights.random(H, h, d, F, seed=1)
    ctx = wf.Context(P, a.C, rank=rank)
    layer = WallFacerLayer(ctx, W, h, d, causal=True, checkpoint=not a.no_checkpoint)
    g = torch.Generator(device="cuda").manual_seed(rank)
    x = torch.randn((n, H), generator=g, device="cuda").to(torch.bfloat16)
    dy = torch.randn((n, H), generator=g, device="cuda").to(torch.bfloat16)

    def step():
        y, saved = layer.forward(x, N)
        layer.backward(dy, saved, N)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / a.steps], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    fl = layer_flops(N, H, h, d, F, True)
    if rank == 0:
        print(json.dumps({"workload": "wallfacer_layer_gpt7b", "N": N, "P": P, "C": a.C, "checkpoint": not a.no_checkpoint,
                          "ms_per_step": ms, "tokens_per_s": N / (ms / 1e3),
                          "model_tflops_per_gpu": fl / P / (ms / 1e3) / 1e12,
                          "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
