"""GPU-box helper: a CUPTI (torch.profiler) timeline of bench-shaped fwd+bwd steps, one per
rank, summarised per stream: kernel and copy time by name, and the largest idle gaps on the
stream the block kernels run on (with the activity on either side).

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/trace_step.py --N 65536 --C 4
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

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=65536)
ap.add_argument("--C", type=int, default=0)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--sched", type=int, default=0)
ap.add_argument("--out", default="gpurun_out/trace")
args = ap.parse_args()

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
lr = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(lr)
dev = torch.device("cuda", lr)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
P, N, h, d = world, args.N, args.heads, 128
C = args.C or P
n = N // P
g = torch.Generator(device=dev).manual_seed(1234 + rank)
q, k, v, do = (torch.randn((n, h, d), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
o, lse = torch.empty_like(q), torch.empty((h, n), dtype=torch.float32, device=dev)
dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
ctx = wf.Context(P, C, rank=rank)
if args.sched:
    ctx.set_schedule(args.sched)


def step():
    ctx.fwd(q, k, v, N, True, o=o, lse=lse)
    ctx.bwd(do, q, k, v, o, lse, N, True, dq=dq, dk=dk, dv=dv)


def barrier():
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


for _ in range(4):
    step()
barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.steps):
    step()
e1.record()
barrier()
plain_ms = e0.elapsed_time(e1) / args.steps

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(args.steps):
        step()
    barrier()
os.makedirs(args.out, exist_ok=True)
path = f"{args.out}/rank{rank}.json"
prof.export_chrome_trace(path)

ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in
      ("kernel", "gpu_memcpy", "gpu_memset")]
by_stream = defaultdict(list)
for e in ev:
    by_stream[e["args"].get("stream", e.get("tid"))].append(e)
t0 = min(e["ts"] for e in ev)
t1 = max(e["ts"] + e["dur"] for e in ev)
lines = [f"rank {rank}: P={P} C={C} N={N} plain {plain_ms:.2f} ms/step, traced span {(t1 - t0) / 1e3 / args.steps:.2f} ms/step"]
main = max(by_stream, key=lambda s: sum(e["dur"] for e in by_stream[s] if "wf_block" in e["name"]))
for s, es in sorted(by_stream.items(), key=lambda kv: -sum(e["dur"] for e in kv[1])):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for e in es:
        nm = e["name"].split("(")[0].split("<")[0][:40]
        tot[nm] += e["dur"]
        cnt[nm] += 1
    busy = sum(tot.values()) / 1e3 / args.steps
    lines.append(f"  stream {s}{' (block kernels)' if s == main else ''}: busy {busy:.2f} ms/step")
    for nm, t in sorted(tot.items(), key=lambda kv: -kv[1])[:8]:
        lines.append(f"    {t / 1e3 / args.steps:8.3f} ms  x{cnt[nm] // args.steps:3d}  {nm}")
es = sorted(by_stream[main], key=lambda e: e["ts"])
gaps = []
for a, b in zip(es, es[1:]):
    gap = b["ts"] - (a["ts"] + a["dur"])
    if gap > 0:
        gaps.append((gap, a["name"][:40], b["name"][:40], (a["ts"] + a["dur"] - t0) / 1e3))
idle = sum(x[0] for x in gaps) / 1e3 / args.steps
lines.append(f"  block-kernel stream idle between its launches: {idle:.2f} ms/step; largest gaps:")
for gap, an, bn, at in sorted(gaps, reverse=True)[:12]:
    lines.append(f"    {gap / 1e3:7.3f} ms at {at:7.2f}  after {an}  before {bn}")
txt = "\n".join(lines)
outs = [None] * world
if world > 1:
    dist.all_gather_object(outs, txt)
else:
    outs = [txt]
if rank == 0:
    print("\n".join(outs))
    open(f"{args.out}/summary.txt", "w").write("\n".join(outs) + "\n")
ctx.close()
if world > 1:
    dist.destroy_process_group()
