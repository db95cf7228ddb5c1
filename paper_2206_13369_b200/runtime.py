"""Host-side plumbing shared by the solvers: input coercion/upload, output
conversion, and the collective wrapper used for row-sharded runs."""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist


_NATIVE = {}  # (group, device) -> native NCCL communicator handle (one per process group)


def _native_comm(group, world, rank):
    """The library's own NCCL communicator for this group (mlr_comm_create),
    built once: rank 0's unique id travels by ONE torch.distributed broadcast,
    after which every per-iteration collective is a direct ncclAllReduce /
    ncclAllGather call on the plan stream (include/mlr_b200.h)."""
    from . import _lib
    dev = torch.cuda.current_device()
    # keyed by the process group object as well as its shape: a destroyed and
    # re-created group gets a new communicator
    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    key = (id(pg), dev, world, rank)
    if key in _NATIVE:
        return _NATIVE[key]
    lib = _lib.load()
    if not lib.mlr_comm_available():
        _NATIVE[key] = None
        return None
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        _lib.check(lib.mlr_comm_unique_id(ctypes.c_void_p(uid.data_ptr())))
    t = uid.cuda()
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    uid.copy_(t.cpu())
    h = ctypes.c_void_p()
    _lib.check(lib.mlr_comm_create(ctypes.c_void_p(uid.data_ptr()), world, rank, dev, ctypes.byref(h)))
    _NATIVE[key] = h
    return h


class Comm:
    """Collectives of the row-sharded solvers.  On GPUs over an NCCL process
    group they run on the library's own NCCL communicator (ctypes ->
    mlr_comm_allreduce / mlr_comm_allgather on the current stream; torch.
    distributed only carries the one-time unique-id exchange).  Over gloo
    (CPU tests, ranks sharing one device) they go through torch.distributed,
    staging CUDA tensors through host memory.  A world of one makes every
    call a no-op."""

    def __init__(self, group=None, enabled=None, force_native=None):
        if force_native is None:  # tests: run a one-rank NCCL group through the native collectives
            force_native = os.environ.get("MLR_FORCE_NATIVE_NCCL") == "1"
        if enabled is None:
            enabled = dist.is_available() and dist.is_initialized()
        self.enabled = bool(enabled)
        self.group = group
        self.world = dist.get_world_size(group) if self.enabled else 1
        self.rank = dist.get_rank(group) if self.enabled else 0
        self.native = None
        if (self.world > 1 or force_native) and self.enabled and torch.cuda.is_available() \
                and dist.get_backend(group) == "nccl" and os.environ.get("MLR_NATIVE_NCCL", "1") != "0":
            self.native = _native_comm(group, self.world, self.rank)  # force_native: one-rank NCCL (tests)

    def _host(self, t):
        """gloo works on host tensors: stage CUDA tensors through host memory."""
        return self.world > 1 and t.is_cuda and dist.get_backend(self.group) != "nccl"

    def _nat(self, t):
        return self.native is not None and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()

    def _native_reduce(self, t, op):
        from . import _lib
        _lib.check(_lib.load().mlr_comm_allreduce(self.native, ctypes.c_void_p(t.data_ptr()), t.numel(), 8, op,
                                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return t

    def sum(self, t):
        if self._nat(t):
            return self._native_reduce(t, 0)
        if self.world > 1:
            if self._host(t):
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def max(self, t):
        if self._nat(t):
            return self._native_reduce(t, 2)
        if self.world > 1:
            if self._host(t):
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.MAX, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def check_replicated(self, t, what):
        """Debug (MLR_VERIFY_REPLICATED=1): the all-reduced buffer every rank
        feeds its replicated eigensolver / LMO must be bitwise identical on
        all ranks (NCCL's all-reduce guarantees it; this checks it).  Raises
        RuntimeError naming the first rank that differs."""
        if self.world <= 1:
            return
        bits = t.contiguous().view(torch.int64)
        h = torch.stack([bits.sum(), (bits * torch.arange(1, bits.numel() + 1, device=bits.device)).sum()])
        hd = h
        out = torch.zeros(2 * self.world, dtype=torch.int64, device=h.device)
        if self._host(h) or not h.is_cuda or self.native is None:
            parts = [torch.empty_like(hd.cpu()) for _ in range(self.world)]
            dist.all_gather(parts, hd.cpu() if self._host(h) else hd, group=self.group)
            out = torch.cat([x.to(out.device) for x in parts])
        else:
            dist.all_gather_into_tensor(out, hd, group=self.group)
        got = out.view(self.world, 2).cpu()
        for r in range(1, self.world):
            if not torch.equal(got[r], got[0]):
                raise RuntimeError(f"replicated {what} differs between rank 0 and rank {r}")

    def gather(self, out, t):
        """out (world * t.numel()) <- concatenation of every rank's t."""
        if self._nat(t) and self._nat(out):
            from . import _lib
            _lib.check(_lib.load().mlr_comm_allgather(
                self.native, ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), t.numel(), 8,
                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        elif self.world > 1:
            if dist.get_backend(self.group) == "nccl":
                dist.all_gather_into_tensor(out, t, group=self.group)
            else:
                h = t.cpu()
                parts = [torch.empty_like(h) for _ in range(self.world)]
                dist.all_gather(parts, h, group=self.group)
                out.copy_(torch.cat(parts))
        else:
            out.copy_(t)
        return out


SINGLE = Comm(enabled=False)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2206_13369_b200 requires a CUDA (sm_100a) device; no CPU fallback exists")


def as_device_matrix(x, name="d", precision="auto"):
    """Validate like as_matrix (linalg.py:48-57, finiteness is checked on the
    device) and return (tensor on GPU, kind) where kind records how to give
    results back: "numpy", "torch-cpu" or "torch-cuda"."""
    require_cuda()
    if isinstance(x, torch.Tensor):
        kind = "torch-cuda" if x.is_cuda else "torch-cpu"
        t = x
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        if t.dim() != 2:
            raise ValueError(f"{name} must be 2-D, got ndim={t.dim()}")
        if t.shape[0] < 1 or t.shape[1] < 1:
            raise ValueError(f"{name} must have positive dimensions, got {tuple(t.shape)}")
        if not t.is_cuda:
            t = t.to(torch.device("cuda", torch.cuda.current_device()), non_blocking=t.is_pinned())
        return _with_precision(t.contiguous(), precision), kind
    a = np.asarray(x)
    if a.dtype != np.float32:
        a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={a.ndim}")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"{name} must have positive dimensions, got {a.shape}")
    t = torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", torch.cuda.current_device()))
    return _with_precision(t, precision), "numpy"


def _with_precision(t, precision):
    """PcpOptions / CpcpOptions.precision: "auto" keeps the input's type
    (float32 or float64), "float64" / "float32" convert on the device."""
    if precision not in ("auto", "float64", "float32"):
        raise ValueError(f"precision must be one of ('auto', 'float64', 'float32'), got {precision!r}")
    if precision == "float64" and t.dtype != torch.float64:
        return t.to(torch.float64)
    if precision == "float32" and t.dtype != torch.float32:
        return t.to(torch.float32)
    return t


def give_back_all(ts, kind):
    """Results on the caller's side.  Host results land in pinned buffers
    through queued non-blocking copies and one synchronisation, so the
    device-to-host transfer runs at copy-engine speed instead of through
    pageable staging (numpy results are views of the pinned buffers)."""
    if kind == "torch-cuda":
        return list(ts)
    outs, dev = [], None
    for t in ts:
        if not t.is_cuda:
            outs.append(t)
            continue
        h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
        dev = t.device
    if dev is not None:
        torch.cuda.current_stream(dev).synchronize()
    return outs if kind == "torch-cpu" else [h.numpy() for h in outs]


def give_back(t, kind):
    return give_back_all([t], kind)[0]
