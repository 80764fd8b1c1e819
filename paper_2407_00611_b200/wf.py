"""Thin torch-facing binding of libwf.so (argument marshalling only).

Every step of the hot path runs inside libwf.so's CUDA kernels; torch supplies
device memory, streams and (for multi-GPU) the process group that broadcasts
the NCCL id.  Names follow include/wf.h.
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import ALLGATHER_FN, KINDS, WfEvent, WfUid, lib

__all__ = ["WFError", "block_fwd", "block_bwd", "Context", "plan", "plan_trace", "shard_ranges"]


class WFError(RuntimeError):
    pass


def _check(st, ctx=None):
    if st != 0:
        msg = lib().wf_last_error(ctx)
        raise WFError(f"wf status {st}: {msg.decode() if msg else ''}")


def _ptr(t):
    if t is None:
        return None
    if not t.is_contiguous():
        raise WFError("tensor arguments must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _i32arr(xs):
    if xs is None:
        return None, 0
    arr = (ctypes.c_int32 * len(xs))(*[int(x) for x in xs])
    return arr, len(xs)


def _backend(group):
    import torch.distributed as dist
    return dist.get_backend(group)


def _bf16(t, name):
    if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
        raise WFError(f"{name}: need a contiguous CUDA bf16 tensor")
    return t


def block_fwd(q, k, v, causal=False, chunk=0, qstart=None, kstart=None, o_in=None, lse_in=None,
              out_f32=False, out_bf16=True):
    """One forward_iteration on the current device: returns (o_f32|None, o_bf16|None, lse)."""
    nq, h, d = q.shape
    nk = k.shape[0]
    of = torch.empty((nq, h, d), dtype=torch.float32, device=q.device) if out_f32 else None
    ob = torch.empty((nq, h, d), dtype=torch.bfloat16, device=q.device) if out_bf16 else None
    lse = torch.empty((h, nq), dtype=torch.float32, device=q.device)
    qs, nqs = _i32arr(qstart)
    ks, nks = _i32arr(kstart)
    _check(lib().wf_block_fwd(_ptr(_bf16(q, "q")), _ptr(_bf16(k, "k")), _ptr(_bf16(v, "v")), nq, nk, h, d,
                              int(causal), int(chunk), qs, nqs, ks, nks, _ptr(o_in), _ptr(lse_in), _ptr(of), _ptr(ob),
                              _ptr(lse), _stream()))
    return of, ob, lse


def gemm_bf16(a, b, y=None, a_mn=False, b_mn=False):
    """Y[m, n] = sum_k A(m, k) B(n, k) on the tensor cores (wf_gemm_bf16_t).
    a: [M, K] (or [K, M] with a_mn), b: [N, K] (or [K, N] with b_mn), bf16 -> y [M, N] bf16."""
    M, K = (a.shape[1], a.shape[0]) if a_mn else a.shape
    N = b.shape[1] if b_mn else b.shape[0]
    y = torch.empty((M, N), dtype=torch.bfloat16, device=a.device) if y is None else y
    _check(lib().wf_gemm_bf16_t(_ptr(_bf16(a, "a")), int(a_mn), _ptr(_bf16(b, "b")), int(b_mn), M, N, K,
                                _ptr(_bf16(y, "y")), _stream()))
    return y


def layernorm_fwd(x, w, b, eps=1e-5, y=None):
    """y = (x - mean) rstd w + b (wf_layernorm_fwd); returns (y, mean, rstd) (fp32 [rows])."""
    rows, H = x.shape
    y = torch.empty_like(x) if y is None else y
    mean = torch.empty((rows,), dtype=torch.float32, device=x.device)
    rstd = torch.empty((rows,), dtype=torch.float32, device=x.device)
    _check(lib().wf_layernorm_fwd(_ptr(_bf16(x, "x")), _ptr(_bf16(w, "w")), _ptr(_bf16(b, "b")), rows, H, float(eps),
                                  _ptr(_bf16(y, "y")), _ptr(mean), _ptr(rstd), _stream()))
    return y, mean, rstd


def layernorm_bwd(dy, x, w, mean, rstd, dw, db, dres=None, dx=None):
    """dx (+ dres) and dw, db += (wf_layernorm_bwd); dw, db fp32 [H] accumulate."""
    rows, H = x.shape
    dx = torch.empty_like(x) if dx is None else dx
    _check(lib().wf_layernorm_bwd(_ptr(_bf16(dy, "dy")), _ptr(_bf16(x, "x")), _ptr(_bf16(w, "w")), _ptr(mean),
                                  _ptr(rstd), _ptr(dres), rows, H, _ptr(_bf16(dx, "dx")), _ptr(dw), _ptr(db),
                                  _stream()))
    return dx


def gelu_fwd(u, h=None):
    h = torch.empty_like(u) if h is None else h
    _check(lib().wf_gelu_fwd(_ptr(_bf16(u, "u")), u.numel(), _ptr(_bf16(h, "h")), _stream()))
    return h


def gelu_bwd(dh, u, du=None):
    du = torch.empty_like(u) if du is None else du
    _check(lib().wf_gelu_bwd(_ptr(_bf16(dh, "dh")), _ptr(_bf16(u, "u")), u.numel(), _ptr(_bf16(du, "du")),
                             _stream()))
    return du


def add_bf16(a, b, y=None):
    y = torch.empty_like(a) if y is None else y
    _check(lib().wf_add_bf16(_ptr(_bf16(a, "a")), _ptr(_bf16(b, "b")), a.numel(), _ptr(y), _stream()))
    return y


def pack3(a, b, c, y=None):
    rows = a.shape[0]
    E = a.numel() // rows
    y = torch.empty((rows, 3 * E), dtype=torch.bfloat16, device=a.device) if y is None else y
    _check(lib().wf_pack3_bf16(_ptr(_bf16(a, "a")), _ptr(b), _ptr(c), rows, E, _ptr(y), _stream()))
    return y


def block_bwd(q, k, v, do, lse, dsum, dq_acc, dk_acc, dv_acc, causal=False, chunk=0, qstart=None, kstart=None,
              accumulate=False):
    """One flash-attention backward step on the current device (in place on the accumulators)."""
    nq, h, d = q.shape
    nk = k.shape[0]
    qs, nqs = _i32arr(qstart)
    ks, nks = _i32arr(kstart)
    _check(lib().wf_block_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(do), _ptr(lse), _ptr(dsum), nq, nk, h, d, int(causal),
                              int(chunk), qs, nqs, ks, nks, _ptr(dq_acc), _ptr(dk_acc), _ptr(dv_acc), int(accumulate),
                              _stream()))


def plan(P, C, rank):
    out = (ctypes.c_int32 * 6)()
    _check(lib().wf_plan(P, C, rank, out))
    return dict(send=out[0], recv=out[1], next=out[2], last=out[3], R=out[4], regime="paper" if out[5] == 0 else "ext")


def _events(buf, n):
    return [(e.pas, KINDS[e.kind], e.step, e.src, e.dst, e.block, e.nbytes) for e in buf[:n]]


SCHED_GATHER_SHUFFLE, SCHED_DIRECT_PULL = 0, 1


def plan_trace(P, C, N, heads, head_dim, rank=-1, sched=SCHED_GATHER_SHUFFLE):
    n = ctypes.c_size_t(0)
    _check(lib().wf_plan_trace_sched(P, C, N, heads, head_dim, rank, sched, None, 0, ctypes.byref(n)))
    buf = (WfEvent * max(1, n.value))()
    _check(lib().wf_plan_trace_sched(P, C, N, heads, head_dim, rank, sched, buf, n.value, ctypes.byref(n)))
    return _events(buf, n.value)


def shard_ranges(P, rank, N, causal):
    out = (ctypes.c_int64 * 4)()
    _check(lib().wf_shard_ranges(P, rank, N, int(causal), out))
    return list(out)


def workspace_bytes(P, C, N, heads, head_dim, causal):
    """Device workspace bytes one rank allocates for this shape (wf_workspace_bytes)."""
    out = ctypes.c_size_t(0)
    _check(lib().wf_workspace_bytes(P, C, N, heads, head_dim, int(causal), ctypes.byref(out)))
    return int(out.value)


def _host_allgather(P, group):
    """wf_allgather_fn over torch.distributed (the bootstrap of wf_init_bootstrap)."""
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    def fn(inp, out, nbytes, user):
        try:
            t = torch.frombuffer(bytearray(ctypes.string_at(inp, nbytes)), dtype=torch.uint8).to(dev)
            outs = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(P)]
            dist.all_gather(outs, t, group=group)
            data = torch.cat(outs).cpu().numpy().tobytes()
            ctypes.memmove(out, data, P * nbytes)
            return 0
        except Exception:  # pragma: no cover - reported as WF_ERR_COMM by the library
            return 1

    return ALLGATHER_FN(fn)


class Context:
    """A wf_ctx: real (one rank of a torch.distributed job) or emulated (all P ranks on one GPU).

    Real mode bootstraps the peer-memory transport through NCCL (wf_init) when the process
    group is NCCL, and through the group's host all-gather (wf_init_bootstrap) otherwise --
    e.g. gloo, which lets several ranks share one GPU in tests."""

    def __init__(self, P, C, rank=0, emulated=False, group=None, topology=0, timeout_s=None):
        self.P, self.C, self.rank, self.emulated = P, C, rank, emulated
        self._ag = None
        h = ctypes.c_void_p()
        if emulated:
            _check(lib().wf_init_emulated(P, C, ctypes.byref(h)))
        elif P > 1 and _backend(group) != "nccl":
            self._ag = _host_allgather(P, group)
            _check(lib().wf_init_bootstrap(P, C, topology, rank, ctypes.cast(self._ag, ctypes.c_void_p), None,
                                           ctypes.byref(h)))
        else:
            uid = WfUid()
            if P > 1:
                import torch.distributed as dist
                if rank == 0:
                    _check(lib().wf_get_uid(ctypes.byref(uid)))
                t = torch.tensor(list(bytes(uid.bytes)), dtype=torch.uint8)
                if dist.get_backend(group) == "nccl":
                    t = t.cuda()
                dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
                for i, b in enumerate(t.cpu().tolist()):
                    uid.bytes[i] = b
            _check(lib().wf_init(P, C, topology, rank, ctypes.byref(uid), ctypes.byref(h)))
        self.h = h
        if timeout_s is not None:
            _check(lib().wf_set_timeout(self.h, float(timeout_s)), self.h)

    def _check_rows(self, rows, N, what):
        want = N if self.emulated else N // self.P
        if N % self.P or rows != want:
            raise WFError(f"{what}: {rows} rows, expected {want} (N = {N}, P = {self.P}, "
                          f"{'emulated: all ranks stacked' if self.emulated else 'one rank shard'})")

    def _lse_shape(self, rows, h):
        return (self.P, h, rows // self.P) if self.emulated else (h, rows)

    def fwd(self, q, k, v, N, causal, o=None, lse=None):
        rows, h, d = q.shape
        self._check_rows(rows, N, "fwd")
        for t, name in ((q, "q"), (k, "k"), (v, "v")):
            _bf16(t, name)
            if t.shape != q.shape:
                raise WFError(f"fwd: {name} shape {tuple(t.shape)} != q shape {tuple(q.shape)}")
        o = torch.empty_like(q) if o is None else _bf16(o, "o")
        lse_shape = self._lse_shape(rows, h)
        lse = torch.empty(lse_shape, dtype=torch.float32, device=q.device) if lse is None else lse
        if o.shape != q.shape or tuple(lse.shape) != lse_shape or lse.dtype != torch.float32 or not lse.is_contiguous():
            raise WFError("fwd: o must match q; lse must be contiguous fp32 " + str(lse_shape))
        _check(lib().wf_attn_fwd(self.h, _ptr(q), _ptr(k), _ptr(v), N, h, d, int(causal), _ptr(o), _ptr(lse),
                                 _stream()), self.h)
        return o, lse

    def qkv_proj(self, x, w, N, heads, head_dim, causal, q=None, k=None, v=None):
        """Alg. 1 l.1 AllGather_QKVmatmul (wf_qkv_proj): x [rows, hidden], w [3 heads head_dim, hidden]
        -> q, k, v [rows, heads, head_dim]; with C > 1 the team gather rides on the GEMM epilogue."""
        rows, hidden = x.shape
        self._check_rows(rows, N, "qkv_proj")
        if tuple(w.shape) != (3 * heads * head_dim, hidden):
            raise WFError(f"qkv_proj: w shape {tuple(w.shape)} != {(3 * heads * head_dim, hidden)}")
        q = torch.empty((rows, heads, head_dim), dtype=torch.bfloat16, device=x.device) if q is None else q
        k = torch.empty_like(q) if k is None else k
        v = torch.empty_like(q) if v is None else v
        _check(lib().wf_qkv_proj(self.h, _ptr(_bf16(x, "x")), _ptr(_bf16(w, "w")), N, hidden, heads, head_dim,
                                 int(causal), _ptr(q), _ptr(k), _ptr(v), _stream()), self.h)
        return q, k, v

    def bwd(self, do, q, k, v, o, lse, N, causal, dq=None, dk=None, dv=None):
        rows, h, d = q.shape
        self._check_rows(rows, N, "bwd")
        for t, name in ((do, "do"), (q, "q"), (k, "k"), (v, "v"), (o, "o")):
            _bf16(t, name)
            if t.shape != q.shape:
                raise WFError(f"bwd: {name} shape {tuple(t.shape)} != q shape {tuple(q.shape)}")
        lse_shape = self._lse_shape(rows, h)
        if tuple(lse.shape) != lse_shape or lse.dtype != torch.float32 or not lse.is_contiguous():
            raise WFError("bwd: lse must be contiguous fp32 " + str(lse_shape))
        dq = torch.empty_like(q) if dq is None else _bf16(dq, "dq")
        dk = torch.empty_like(k) if dk is None else _bf16(dk, "dk")
        dv = torch.empty_like(v) if dv is None else _bf16(dv, "dv")
        for t, name in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
            if t.shape != q.shape:
                raise WFError(f"bwd: {name} shape {tuple(t.shape)} != q shape {tuple(q.shape)}")
        _check(lib().wf_attn_bwd(self.h, _ptr(do), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), N, h, d,
                                 int(causal), _ptr(dq), _ptr(dk), _ptr(dv), _stream()), self.h)
        return dq, dk, dv

    def trace(self):
        n = ctypes.c_size_t(0)
        _check(lib().wf_get_trace(self.h, None, 0, ctypes.byref(n)), self.h)
        buf = (WfEvent * max(1, n.value))()
        _check(lib().wf_get_trace(self.h, buf, n.value, ctypes.byref(n)), self.h)
        return _events(buf, n.value)

    def set_schedule(self, sched):
        """SCHED_GATHER_SHUFFLE (the paper's Alg. 1 l.1-2) or SCHED_DIRECT_PULL (wf_set_schedule)."""
        _check(lib().wf_set_schedule(self.h, int(sched)), self.h)

    def set_debug(self, flags):
        """flags: 1 = skip every inter-rank transfer (timing of exposed communication only)."""
        _check(lib().wf_set_debug(self.h, int(flags)), self.h)

    def set_profiling(self, on=True):
        _check(lib().wf_set_profiling(self.h, int(on)), self.h)

    def kernel_times(self):
        """(fwd_ms, bwd_ms, fwd_launches, bwd_launches) since profiling was enabled / last call."""
        out = (ctypes.c_double * 4)()
        _check(lib().wf_kernel_times(self.h, out), self.h)
        return out[0], out[1], int(out[2]), int(out[3])

    def phase_times(self):
        """{kind: device ms} of the message phases since profiling was enabled / last call."""
        out = (ctypes.c_double * len(KINDS))()
        _check(lib().wf_phase_times(self.h, out, len(KINDS)), self.h)
        return {k: out[i] for i, k in enumerate(KINDS) if out[i] > 0}

    def kernel_launches(self):
        return int(lib().wf_kernel_launches(self.h))

    def close(self):
        if self.h:
            lib().wf_finalize(self.h)
            self.h = None
        self._ag = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
