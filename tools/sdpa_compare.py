"""GPU-box helper: context numbers for the library attention in this image, same shape and
FLOP convention as bench.py (GPT 32K causal 32x128 and DiT 64K full 16x72, one GPU): torch's
scaled_dot_product_attention forward + backward in bf16 (torch picks its backend, cuDNN or
flash, on B200), timed with CUDA events after warm-up.  Not a baseline the driver uses.

    python tools/sdpa_compare.py
"""
import json

import torch
import torch.nn.functional as F


def run(N, h, d, causal, steps=10, warmup=3):
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v, do = (torch.randn((1, h, N, d), generator=g, device="cuda", dtype=torch.bfloat16) for _ in range(4))
    q.requires_grad_(True)
    k.requires_grad_(True)
    v.requires_grad_(True)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    fwd_ms, bwd_ms = [], []

    def step(timed):
        if timed:
            ev[0].record()
        o = F.scaled_dot_product_attention(q, k, v, is_causal=causal)
        if timed:
            ev[1].record()
        o.backward(do)
        if timed:
            ev[2].record()
            torch.cuda.synchronize()
            fwd_ms.append(ev[0].elapsed_time(ev[1]))
            bwd_ms.append(ev[1].elapsed_time(ev[2]))

    for _ in range(warmup):
        step(False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step(False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    for _ in range(3):
        step(True)
    flops = 4.0 * N * N * h * d * (0.5 if causal else 1.0) * 3.5
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        step(False)
        torch.cuda.synchronize()
    kernels = sorted({e.name[:80] for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA})
    return {"N": N, "heads": h, "head_dim": d, "causal": causal, "ms_per_step": ms, "tflops": flops / ms / 1e9,
            "fwd_ms": min(fwd_ms), "bwd_ms": min(bwd_ms), "kernels": kernels}


if __name__ == "__main__":
    for cfg in ((32768, 32, 128, True), (65536, 16, 72, False)):
        try:
            print(json.dumps({"impl": "torch.sdpa", **run(*cfg)}))
        except Exception as e:  # noqa: BLE001 -- report and continue (e.g. an unsupported head dim)
            print(json.dumps({"impl": "torch.sdpa", "N": cfg[0], "head_dim": cfg[2], "error": str(e)[:200]}))
