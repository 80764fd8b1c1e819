"""Thin torch-facing binding of libwf.so (argument marshalling only).

Every step of the hot path runs inside libwf.so's CUDA kernels; torch supplies
device memory, streams and (for multi-GPU) the process group that broadcasts
the NCCL id.  Names follow include/wf.h.
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import KINDS, WfEvent, WfUid, lib

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


def rmsnorm_fwd(x, w, eps=1e-5, y=None, rstd=None):
    """y = x rstd w (wf_rmsnorm_fwd); returns (y, rstd fp32 [rows])."""
    rows, H = x.shape
    y = torch.empty_like(x) if y is None else y
    rstd = torch.empty((rows,), dtype=torch.float32, device=x.device) if rstd is None else rstd
    _check(lib().wf_rmsnorm_fwd(_ptr(_bf16(x, "x")), _ptr(_bf16(w, "w")), rows, H, float(eps), _ptr(y), _ptr(rstd),
                                _stream()))
    return y, rstd


def rmsnorm_bwd(dy, x, w, rstd, dw, dres=None, dx=None):
    """dx (+ dres) and dw += (wf_rmsnorm_bwd); dw fp32 [H] accumulates."""
    rows, H = x.shape
    dx = torch.empty_like(x) if dx is None else dx
    _check(lib().wf_rmsnorm_bwd(_ptr(_bf16(dy, "dy")), _ptr(x), _ptr(w), _ptr(rstd), _ptr(dres), rows, H, _ptr(dx),
                                _ptr(dw), _stream()))
    return dx


def swiglu_fwd(gu, h=None):
    rows, F2 = gu.shape
    h = torch.empty((rows, F2 // 2), dtype=torch.bfloat16, device=gu.device) if h is None else h
    _check(lib().wf_swiglu_fwd(_ptr(_bf16(gu, "gu")), rows, F2 // 2, _ptr(h), _stream()))
    return h


def swiglu_bwd(dh, gu, dgu=None):
    rows, F2 = gu.shape
    dgu = torch.empty_like(gu) if dgu is None else dgu
    _check(lib().wf_swiglu_bwd(_ptr(_bf16(dh, "dh")), _ptr(gu), rows, F2 // 2, _ptr(dgu), _stream()))
    return dgu


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


class Context:
    """A wf_ctx: real (one rank of a torch.distributed job) or emulated (all P ranks on one GPU)."""

    def __init__(self, P, C, rank=0, emulated=False, group=None, topology=0):
        self.P, self.C, self.rank, self.emulated = P, C, rank, emulated
        h = ctypes.c_void_p()
        if emulated:
            _check(lib().wf_init_emulated(P, C, ctypes.byref(h)))
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

    def fwd(self, q, k, v, N, causal, o=None, lse=None):
        rows, h, d = q.shape
        o = torch.empty_like(q) if o is None else o
        lse_shape = (self.P, h, rows // self.P) if self.emulated else (h, rows)
        lse = torch.empty(lse_shape, dtype=torch.float32, device=q.device) if lse is None else lse
        _check(lib().wf_attn_fwd(self.h, _ptr(q), _ptr(k), _ptr(v), N, h, d, int(causal), _ptr(o), _ptr(lse),
                                 _stream()), self.h)
        return o, lse

    def qkv_proj(self, x, w, N, heads, head_dim, causal, q=None, k=None, v=None):
        """Alg. 1 l.1 AllGather_QKVmatmul (wf_qkv_proj): x [rows, hidden], w [3 heads head_dim, hidden]
        -> q, k, v [rows, heads, head_dim]; with C > 1 the team gather rides on the GEMM epilogue."""
        rows, hidden = x.shape
        q = torch.empty((rows, heads, head_dim), dtype=torch.bfloat16, device=x.device) if q is None else q
        k = torch.empty_like(q) if k is None else k
        v = torch.empty_like(q) if v is None else v
        _check(lib().wf_qkv_proj(self.h, _ptr(_bf16(x, "x")), _ptr(_bf16(w, "w")), N, hidden, heads, head_dim,
                                 int(causal), _ptr(q), _ptr(k), _ptr(v), _stream()), self.h)
        return q, k, v

    def bwd(self, do, q, k, v, o, lse, N, causal, dq=None, dk=None, dv=None):
        rows, h, d = q.shape
        dq = torch.empty_like(q) if dq is None else dq
        dk = torch.empty_like(k) if dk is None else dk
        dv = torch.empty_like(v) if dv is None else dv
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

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
