"""GPU-box stress test of the real multi-rank path (launched with torchrun): many fwd+bwd
calls per (C, schedule, mask, N) with shape changes in between (workspace re-carve and
IPC re-mapping), checking that O is bit-identical across repeats (the forward is
deterministic) and that dQ/dK/dV stay finite.  Prints one line per configuration."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00611_b200 as wf  # noqa: E402
from paper_2407_00611_b200.scheduler import variants  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
iters = int(os.environ.get("ITERS", "30"))
h, d = 8, 128
for C, sched in variants(world):
    ctx = wf.Context(world, C, rank=rank)
    if sched:
        ctx.set_schedule(sched)
    t0 = time.time()
    ok = True
    for N in (2048 * world, 1024 * world, 4096 * world):
        for causal in (True, False):
            n = N // world
            g = torch.Generator(device="cuda").manual_seed(rank * 7 + N)
            q, k, v, do = (torch.randn((n, h, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
            ref = None
            for it in range(iters):
                o, lse = ctx.fwd(q, k, v, N, causal)
                dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, causal)
                if it == 0:
                    torch.cuda.synchronize()
                    ref = o.clone()
                elif it == iters - 1:
                    torch.cuda.synchronize()
                    ok = ok and bool(torch.equal(o, ref))
                    ok = ok and all(bool(torch.isfinite(x.float()).all()) for x in (dq, dk, dv))
    ctx.close()
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(f"C={C} sched={sched}: {'ok' if flag.item() else 'MISMATCH'} ({time.time() - t0:.1f} s, "
              f"{iters * 6} fwd+bwd calls)", flush=True)
dist.destroy_process_group()
