"""GPU-box helper: bandwidth of the peer-memory transport at P ranks.

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/transport_bw.py --N 65536

For each team size C (every valid C <= 4 unless --C): fwd + bwd steps of the GPT shape are
traced with CUPTI (torch.profiler); every copy-engine peer copy the library issues
(`Memcpy PtoP` / DtoD over the IPC mapping) is timed on its own -- its duration excludes
the flag waits -- so bytes / duration is the achieved NVLink rate per message, reported
per size bucket against 900 GB/s per direction.  Beside it: the library's own per-phase
device times (wf_phase_times, which include the waits for the slowest peer), the bytes
each phase moved according to this rank's CommTrace, and the exposed-communication
fraction (the same steps with every transfer skipped).  Writes gpurun_out/transport_p{P}.json.
"""
import argparse
import json
import os
import sys
from collections import defaultdict

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_2407_00611_b200 as wf  # noqa: E402
from paper_2407_00611_b200.scheduler import candidates  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=65536)
ap.add_argument("--C", type=int, default=0)
ap.add_argument("--steps", type=int, default=3)
args = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
lr = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(lr)
dev = torch.device("cuda", lr)
dist.init_process_group("nccl", device_id=dev)
P, N, h, d = world, args.N, 32, 128
n = N // P
g = torch.Generator(device=dev).manual_seed(1234 + rank)
q, k, v, do = (torch.randn((n, h, d), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
o, lse = torch.empty_like(q), torch.empty((h, n), dtype=torch.float32, device=dev)
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)


def barrier():
    dist.barrier()
    torch.cuda.synchronize()


def allmax(x):
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


from torch.profiler import ProfilerActivity, profile  # noqa: E402

result = {"P": P, "N": N, "heads": h, "head_dim": d, "per_C": {}}
for C in ([args.C] if args.C else candidates(P)):
    ctx = wf.Context(P, C, rank=rank)

    def step():
        ctx.fwd(q, k, v, N, True, o=o, lse=lse)
        ctx.bwd(do, q, k, v, o, lse, N, True, dq=dq, dk=dk, dv=dv)

    for _ in range(3):
        step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    barrier()
    ms = allmax(e0.elapsed_time(e1)) / args.steps
    ctx.set_debug(1)
    barrier()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    barrier()
    ms_nt = allmax(e0.elapsed_time(e1)) / args.steps
    ctx.set_debug(0)
    ctx.set_profiling(True)
    ctx.phase_times()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            step()
        barrier()
    phase = {kk: vv / args.steps for kk, vv in ctx.phase_times().items()}
    ctx.set_profiling(False)
    tr = ctx.trace()  # this rank's sends of the last fwd + bwd
    sent = defaultdict(int)
    for (_pas, kind, _s, src, dst, _b, nbytes) in tr:
        sent[kind] += nbytes
    path = f"gpurun_out/transport_trace_r{rank}.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") == "gpu_memcpy"]
    buckets = defaultdict(lambda: [0, 0.0, 0])  # size bucket -> bytes, us, count
    for e in ev:
        nb = e["args"].get("bytes", 0)
        if nb <= 0 or e["dur"] <= 0:
            continue
        kind = e["name"]
        b = f"{kind} {'<1MiB' if nb < 2 ** 20 else ('<64MiB' if nb < 2 ** 26 else '>=64MiB')}"
        buckets[b][0] += nb
        buckets[b][1] += e["dur"]
        buckets[b][2] += 1
    copies = {b: {"GB_per_s": x[0] / (x[1] * 1e3), "bytes_per_step": x[0] / args.steps,
                  "copies_per_step": x[2] / args.steps, "busy_ms_per_step": x[1] / 1e3 / args.steps}
              for b, x in buckets.items()}
    rec = {"ms_per_step": ms, "ms_per_step_no_transfer": ms_nt, "exposed_frac": max(0.0, (ms - ms_nt) / ms),
           "copies_by_size": copies, "phase_ms_per_step": phase, "bytes_sent_per_step_by_kind": dict(sent)}
    allrec = [None] * world
    dist.all_gather_object(allrec, rec)
    result["per_C"][C] = allrec
    ctx.close()
    barrier()

if rank == 0:
    json.dump(result, open(f"gpurun_out/transport_p{P}.json", "w"), indent=1)
    for C, recs in result["per_C"].items():
        r0 = recs[0]
        print(f"P={P} C={C}: {r0['ms_per_step']:.2f} ms/step, no-transfer {r0['ms_per_step_no_transfer']:.2f}, "
              f"exposed {100 * r0['exposed_frac']:.1f} %")
        for b, x in sorted(r0["copies_by_size"].items()):
            print(f"   rank0 {b}: {x['GB_per_s']:.0f} GB/s over {x['copies_per_step']:.0f} copies/step, "
                  f"{x['bytes_per_step'] / 2 ** 20:.0f} MiB/step")
dist.destroy_process_group()
