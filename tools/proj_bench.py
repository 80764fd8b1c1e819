"""GPU-box helper: projection GEMM throughput (ours vs cuBLAS via torch.matmul) and, under
torchrun, the fused projection + team gather vs projection then separate gather, each
followed by the attention forward (GPT-7B layer shape: hidden 4096, 32 x 128, causal).

    python tools/proj_bench.py                       # 1 GPU: GEMM only
    torchrun --nproc-per-node 4 tools/proj_bench.py --C 2
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00611_b200 as wf  # noqa: E402


def timeit(fn, steps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda", dtype=torch.float64)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--C", type=int, default=2)
    ap.add_argument("--rows", type=int, default=16384)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    H, h, d = 4096, 32, 128
    E = h * d
    n = a.rows
    g = torch.Generator(device="cuda").manual_seed(rank)
    x = torch.randn((n, H), generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn((3 * E, H), generator=g, device="cuda") * H ** -0.5).to(torch.bfloat16)
    out = {}
    if world == 1:
        y = torch.empty((n, 3 * E), dtype=torch.bfloat16, device="cuda")
        t_ours = timeit(lambda: wf.gemm_bf16(x, w, y))
        t_cublas = timeit(lambda: torch.matmul(x, w.t(), out=y))
        fl = 2.0 * n * 3 * E * H
        out = {"gemm": f"{n}x{3 * E}x{H}", "ours_ms": t_ours, "ours_tflops": fl / t_ours / 1e9,
               "cublas_ms": t_cublas, "cublas_tflops": fl / t_cublas / 1e9}
    else:
        P, C = world, a.C
        N = n * P
        ctx = wf.Context(P, C, rank=rank)
        q, k, v = (torch.empty((n, h, d), dtype=torch.bfloat16, device="cuda") for _ in range(3))
        o = torch.empty_like(q)
        lse = torch.empty((h, n), dtype=torch.float32, device="cuda")
        y = torch.empty((n, 3 * E), dtype=torch.bfloat16, device="cuda")

        def fused():
            ctx.qkv_proj(x, w, N, h, d, True, q=q, k=k, v=v)
            ctx.fwd(q, k, v, N, True, o=o, lse=lse)

        def separate():
            wf.gemm_bf16(x, w, y)
            yq = y.view(n, 3, h, d)
            q.copy_(yq[:, 0])
            k.copy_(yq[:, 1])
            v.copy_(yq[:, 2])
            ctx.fwd(q, k, v, N, True, o=o, lse=lse)

        def fwd_only():
            ctx.fwd(q, k, v, N, True, o=o, lse=lse)

        out = {"P": P, "C": C, "N": N, "fused_ms": timeit(fused, 5, 2), "separate_ms": timeit(separate, 5, 2),
               "fwd_only_ms": timeit(fwd_only, 5, 2)}
        ctx.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
