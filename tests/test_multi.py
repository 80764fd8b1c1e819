"""Multi-process tests of the N > 1 path.

* CPU (gloo, world_size 2): the host side of a real multi-rank job -- rank 0 creates the
  NCCL id through the C ABI, torch.distributed broadcasts it, every rank computes its own
  CommTrace (wf_plan_trace, rank-filtered) and the union over ranks equals the oracle's
  literal schedule simulation.
* GPU, one device shared by P processes (gloo bootstrap, wf_init_bootstrap): the REAL
  peer-memory transport of DESIGN.md §1a -- CUDA-IPC-mapped workspaces, copy-engine
  pushes, release/acquire flags, in-place pulls of the merge and sums, ring-slot acks --
  runs between processes exactly as between GPUs, only time-sliced on one device.  So the
  driver's single-GPU `-m gpu` run covers it: values against the fp64 dense oracle, each
  rank's trace against the oracle's records of that rank, back-to-back calls, the fused
  projection gather, and WF_ERR_COMM after a peer stops signalling.
* GPU, one process per GPU (NCCL bootstrap; `gpurun --gpus 2` or more, `multigpu`): the
  same jobs over NVLink.
PAPER.md:179-185 (Alg. 1 ring and reduce-scatter), P:203-205 (backward), P:335 (double
buffering).
"""
import os
import socket
from collections import Counter

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.schedule import simulate_backward, simulate_forward


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_events(P, C, N, h, d, causal):
    _, _, ef, _ = simulate_forward(N, None, None, P, C, causal, compute=False, heads=h, head_dim=d)
    _, _, _, eb = simulate_backward(N, None, None, None, None, None, P, C, causal, compute=False, heads=h, head_dim=d)
    return [(e.pas, e.kind, e.step, e.src, e.dst, e.block, e.nbytes) for e in ef + eb]


def _cpu_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes
        from paper_2407_00611_b200._lib import WfUid, lib
        import paper_2407_00611_b200 as wf
        uid = WfUid()
        if rank == 0:
            assert lib().wf_get_uid(ctypes.byref(uid)) == 0
        t = torch.tensor(list(bytes(uid.bytes)), dtype=torch.uint8)
        dist.broadcast(t, src=0)
        got = bytes(t.tolist())
        allu = [None] * world
        dist.all_gather_object(allu, got)
        traces = {}
        for P, C in ((2, 2), (4, 2), (8, 2), (8, 4), (4, 1)):
            # the P ranks of the simulated job are split across the world processes
            mine = []
            for r in range(rank, P, world):
                mine += wf.plan_trace(P, C, 512 * P, 2, 64, rank=r)
            parts = [None] * world
            dist.all_gather_object(parts, mine)
            traces[(P, C)] = [e for p in parts for e in p]
        if rank == 0:
            q.put((allu, traces))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_host_path():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allu, traces = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(set(allu)) == 1 and any(allu[0])
    for (P, C), tr in traces.items():
        assert Counter(tr) == Counter(_oracle_events(P, C, 512 * P, 2, 64, False)), (P, C)


# ---------------------------------------------------------------------- GPU jobs
H, D = 2, 128


def _job_attn(wf, rank, world, C, N, causal, repeat=1):
    """Real fwd + bwd of this rank's shard (repeat > 1: back to back, no host sync)."""
    from wf_inputs import make_qkv_do
    from oracle.sharding import unit_positions
    qg, kg, vg, dog = make_qkv_do(N, H, D, seed=21, peaky=True)
    idx = torch.from_numpy(unit_positions(rank, world, N, causal))
    qs, ks, vs, dos = (t[idx].contiguous().cuda() for t in (qg, kg, vg, dog))
    ctx = wf.Context(world, C, rank=rank)
    outs = []
    for _ in range(repeat):
        o, lse = ctx.fwd(qs, ks, vs, N, causal)
        dq, dk, dv = ctx.bwd(dos, qs, ks, vs, o, lse, N, causal)
        outs.append([x.clone() for x in (o, lse, dq, dk, dv)])
    torch.cuda.synchronize()
    tr = ctx.trace()
    ctx.close()
    first = [x.float().cpu().numpy() for x in outs[0]]  # numpy: no shared-memory tensors across processes
    same_o = all(torch.equal(x[0], outs[0][0]) and torch.equal(x[1], outs[0][1]) for x in outs)
    g0 = torch.cat([x.float().flatten() for x in outs[0][2:]])
    gdev = max(float((torch.cat([y.float().flatten() for y in x[2:]]) - g0).abs().max()) for x in outs)
    return first, tr, same_o, gdev / float(g0.abs().max())


def _job_proj(wf, rank, world, C, N, causal):
    """wf_qkv_proj's fused gather vs a plain forward on the same Q/K/V: identical results and
    traces."""
    from wf_inputs import make_x_w
    from oracle.sharding import unit_positions
    Hd = 192
    xg, w = make_x_w(N, Hd, H, D, seed=4)
    idx = torch.from_numpy(unit_positions(rank, world, N, causal))
    xs = xg[idx].contiguous().cuda()
    ctx = wf.Context(world, C, rank=rank)
    qs, ks, vs = ctx.qkv_proj(xs, w.cuda(), N, H, D, causal)
    o1, l1 = ctx.fwd(qs, ks, vs, N, causal)
    torch.cuda.synchronize()
    tr1 = ctx.trace()
    ctx.close()
    ctx = wf.Context(world, C, rank=rank)
    o2, l2 = ctx.fwd(qs.clone(), ks.clone(), vs.clone(), N, causal)
    torch.cuda.synchronize()
    tr2 = ctx.trace()
    ctx.close()
    return bool(torch.equal(o1, o2) and torch.equal(l1, l2)), sorted(tr1) == sorted(tr2)


def _job_failure(wf, rank, world, C, N):
    """Rank 1 stops calling after one collective call; rank 0's next call waits for it,
    times out (1 s), and the call after that returns WF_ERR_COMM (no trap, no hang)."""
    from wf_inputs import make_qkv_do
    from oracle.sharding import unit_positions
    qg, kg, vg, _ = make_qkv_do(N, H, D, seed=3)
    idx = torch.from_numpy(unit_positions(rank, world, N, True))
    qs, ks, vs = (t[idx].contiguous().cuda() for t in (qg, kg, vg))
    ctx = wf.Context(world, C, rank=rank, timeout_s=1.0)
    ctx.fwd(qs, ks, vs, N, True)
    torch.cuda.synchronize()
    dist.barrier()
    res = None
    if rank == 0:
        ctx.fwd(qs, ks, vs, N, True)   # rank 1 never joins: its waits time out
        torch.cuda.synchronize()       # returns: no trap, the context is usable
        try:
            ctx.fwd(qs, ks, vs, N, True)
            res = "no error"
        except wf.WFError as e:
            res = str(e)
        torch.cuda.synchronize()
    dist.barrier()
    if rank != 0:  # the live rank frees first (its finalize barrier signals into rank 0's workspace)
        ctx.close()
    dist.barrier()
    if rank == 0:  # WF_ERR_COMM is sticky: finalize skips the collective barrier
        ctx.close()
    return res


def _gpu_worker(rank, world, port, shared, jobs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = 0 if shared else rank
    torch.cuda.set_device(dev)
    if shared:   # P processes on one GPU: host bootstrap (wf_init_bootstrap) over gloo
        dist.init_process_group("gloo", rank=rank, world_size=world)
    else:        # one process per GPU: NCCL bootstrap (wf_init)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    try:
        import paper_2407_00611_b200 as wf
        out = []
        for job in jobs:
            kind, args = job[0], job[1:]
            fn = {"attn": _job_attn, "proj": _job_proj, "fail": _job_failure}[kind]
            out.append(fn(wf, rank, world, *args))
        allres = [None] * world
        dist.all_gather_object(allres, out)
        if rank == 0:
            q.put(allres)
    finally:
        dist.destroy_process_group()


def _spawn(world, shared, jobs, timeout=900):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, shared, jobs, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        allres = q.get(timeout=timeout)
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.exitcode is None:
                p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return allres  # [rank][job]


_REF = {}


def _reference(N, causal):
    from oracle.dense import attention_bwd
    from wf_inputs import make_qkv_do, to_f64
    if (N, causal) not in _REF:
        qg, kg, vg, dog = make_qkv_do(N, H, D, seed=21, peaky=True)
        dq_r, dk_r, dv_r, o_r, l_r = attention_bwd(to_f64(qg), to_f64(kg), to_f64(vg), to_f64(dog), causal=causal)
        _REF[(N, causal)] = (o_r, l_r, dq_r, dk_r, dv_r)
    return _REF[(N, causal)]


def _check_attn(world, C, N, causal, per_rank):
    from oracle.sharding import unit_positions
    o_r, l_r, dq_r, dk_r, dv_r = _reference(N, causal)
    trace = []
    for r, (res, tr, same_o, gdev) in enumerate(per_rank):
        pos = unit_positions(r, world, N, causal)
        o, lse, dq, dk, dv = (np.asarray(x, dtype=np.float64) for x in res)
        assert np.abs(o - o_r[pos]).max() <= 2e-2, (C, causal, r)
        assert np.abs(lse - l_r[:, pos]).max() <= 1e-2, (C, causal, r)
        for g, ref in ((dq, dq_r), (dk, dk_r), (dv, dv_r)):
            assert np.abs(g - ref[pos]).max() / np.abs(ref).max() <= 2e-2, (C, causal, r)
        assert all(e[3] == r for e in tr)
        # back-to-back calls: the forward is bit-identical; gradients agree to bf16 rounding
        # of fp32 sums taken in a different order (a corrupted ring slot would be O(1))
        assert same_o and gdev < 1e-2, (C, causal, r, same_o, gdev)
        trace += tr
    assert Counter(trace) == Counter(_oracle_events(world, C, N, H, D, causal)), (C, causal)


# ---------------------------------------------------------------------- one GPU, P processes
@pytest.mark.gpu
def test_real_transport_shared_gpu_p4():
    """P = 4 ranks on one GPU: ring (C = 1, R = 4), paper regime (C = 2 = sqrt P, R = 1) and
    the extension (C = 4, unit-pipelined with partial pushes), causal and full, each call
    repeated back to back; then the fused projection gather."""
    world, N = 4, 2048
    cases = [(1, True), (2, True), (4, True), (1, False), (4, False)]
    jobs = [("attn", C, N, causal, 3) for C, causal in cases] + [("proj", 2, N, True), ("proj", 4, N, True)]
    allres = _spawn(world, True, jobs)
    for i, (C, causal) in enumerate(cases):
        _check_attn(world, C, N, causal, [allres[r][i] for r in range(world)])
    for j in (len(cases), len(cases) + 1):
        assert all(same and tr for same, tr in (allres[r][j] for r in range(world))), j


@pytest.mark.gpu
def test_real_transport_shared_gpu_p2():
    """P = 2: the plain ring (C = 1, R = 2) and the extension C = 2 (slice = own unit)."""
    world, N = 2, 1024
    cases = [(1, True), (2, True), (2, False)]
    allres = _spawn(world, True, [("attn", C, N, causal, 2) for C, causal in cases])
    for i, (C, causal) in enumerate(cases):
        _check_attn(world, C, N, causal, [allres[r][i] for r in range(world)])


@pytest.mark.gpu
@pytest.mark.parametrize("C", [1, 2])
def test_peer_timeout_reports_err_comm(C):
    """async communication failures surface as WF_ERR_COMM on the next call."""
    allres = _spawn(2, True, [("fail", C, 1024)], timeout=600)
    msg = allres[0][0]
    assert msg.startswith("wf status 5") and "did not signal" in msg, msg


# ---------------------------------------------------------------------- one process per GPU
@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("C", [1, 2, 4])
@pytest.mark.parametrize("causal", [True, False])
def test_real_transport_multi_gpu(C, causal):
    world = min(torch.cuda.device_count(), 4)
    if world % C:
        pytest.skip("C must divide the GPU count")
    N = 512 * world
    allres = _spawn(world, False, [("attn", C, N, causal, 4)])
    _check_attn(world, C, N, causal, [allres[r][0] for r in range(world)])


@pytest.mark.gpu
@pytest.mark.multigpu
def test_real_path_multi_tile_units():
    """C = GPU count (unit-pipelined, partial pushes) with units of 16 query tiles per rank."""
    world = min(torch.cuda.device_count(), 4)
    N = 2048 * world
    allres = _spawn(world, False, [("attn", world, N, True, 2)])
    _check_attn(world, world, N, True, [allres[r][0] for r in range(world)])


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("C", [2, 4])
def test_fused_projection_gather_real_path(C):
    world = min(torch.cuda.device_count(), 4)
    if world % C:
        pytest.skip("C must divide the GPU count")
    allres = _spawn(world, False, [("proj", C, 512 * world, True)])
    assert all(same and tr for same, tr in (allres[r][0] for r in range(world))), allres
