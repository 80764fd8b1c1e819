"""Debug: real multi-GPU run of every C for P = #GPUs, per-rank errors vs the oracle and
CommTrace diff (GPU box helper; launched with torchrun)."""
import os, sys
from collections import Counter
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, ".")
import paper_2407_00611_b200 as wf
from oracle.dense import attention_bwd
from oracle.sharding import unit_positions
from oracle.schedule import simulate_forward, simulate_backward
from wf_inputs import make_qkv_do, to_f64

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
h, d = 2, 128
for C in [int(c) for c in os.environ.get("CS", "1 2 4").split()]:
    for causal in (True, False):
        N = 512 * world
        qg, kg, vg, dog = make_qkv_do(N, h, d, seed=21, peaky=True)
        idx = torch.from_numpy(unit_positions(rank, world, N, causal))
        qs, ks, vs, dos = (t[idx].contiguous().cuda() for t in (qg, kg, vg, dog))
        ctx = wf.Context(world, C, rank=rank)
        direct = os.environ.get("SCHED") == "direct" and C > 1 and C * C <= world
        if direct:
            ctx.set_schedule(wf.SCHED_DIRECT_PULL)
        o, lse = ctx.fwd(qs, ks, vs, N, causal)
        dq, dk, dv = ctx.bwd(dos, qs, ks, vs, o, lse, N, causal)
        torch.cuda.synchronize()
        tr = ctx.trace()
        ctx.close()
        res = [x.cpu() for x in (o, lse, dq, dk, dv)]
        allres = [None] * world
        dist.all_gather_object(allres, (res, tr))
        if rank == 0:
            dq_r, dk_r, dv_r, o_r, l_r = attention_bwd(to_f64(qg), to_f64(kg), to_f64(vg), to_f64(dog), causal=causal)
            line = []
            trace = []
            for r, (rs, t) in enumerate(allres):
                pos = unit_positions(r, world, N, causal)
                o_, l_, dq_, dk_, dv_ = (x.double().numpy() for x in rs)
                e = [np.abs(o_ - o_r[pos]).max(), np.abs(l_ - l_r[:, pos]).max()] + \
                    [np.abs(g - ref[pos]).max() / np.abs(ref).max() for g, ref in ((dq_, dq_r), (dk_, dk_r), (dv_, dv_r))]
                line.append("r%d " % r + " ".join("%.3g" % x for x in e))
                trace += t
            _, _, ef, _ = simulate_forward(N, None, None, world, C, causal, compute=False, heads=h, head_dim=d,
                                           direct=direct)
            _, _, _, eb = simulate_backward(N, None, None, None, None, None, world, C, causal, compute=False, heads=h,
                                            head_dim=d, direct=direct)
            ref = Counter((e.pas, e.kind, e.step, e.src, e.dst, e.block, e.nbytes) for e in ef + eb)
            got = Counter(trace)
            print(f"C={C} causal={causal} trace_ok={got == ref}", " | ".join(line), flush=True)
            if got != ref:
                print("  missing", list((ref - got).elements())[:5], "extra", list((got - ref).elements())[:5])
dist.destroy_process_group()
