"""GPU-box helper: the copy-engine ceiling of one GPU-to-GPU peer copy over NVLink 5, for
the transport comparison of DESIGN.md section 1a: a 512 MiB copy GPU0 -> GPU1 issued as one
cudaMemcpyAsync, or split into 2 / 4 / 8 chunks on as many streams (copy engines).
Prints GB/s per variant (CUDA events on the issuing streams, best of 5)."""
import json

import torch

n = 512 * 2 ** 20
src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
dst = torch.empty(n, dtype=torch.uint8, device="cuda:1")
res = {}
for parts in (1, 2, 4, 8):
    streams = [torch.cuda.Stream(device="cuda:0") for _ in range(parts)]
    best = 0.0
    for _ in range(5):
        torch.cuda.synchronize("cuda:0")
        torch.cuda.synchronize("cuda:1")
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream("cuda:0"))
        ch = n // parts
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dst[i * ch:(i + 1) * ch].copy_(src[i * ch:(i + 1) * ch], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream("cuda:0").wait_stream(s)
        e1.record(torch.cuda.current_stream("cuda:0"))
        torch.cuda.synchronize("cuda:0")
        best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
    res[parts] = best
    print(f"{parts} stream(s): {best:.0f} GB/s")
json.dump(res, open("gpurun_out/p2p_ceiling.json", "w"))
