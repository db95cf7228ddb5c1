"""Host-side plumbing shared by the solvers: input coercion/upload, output
conversion, and the collective wrapper used for row-sharded runs."""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class Comm:
    """Collectives over a torch.distributed group (NCCL on GPUs, gloo on CPU);
    a world of one makes every call a no-op."""

    def __init__(self, group=None, enabled=None):
        if enabled is None:
            enabled = dist.is_available() and dist.is_initialized()
        self.enabled = bool(enabled)
        self.group = group
        self.world = dist.get_world_size(group) if self.enabled else 1
        self.rank = dist.get_rank(group) if self.enabled else 0

    def _host(self, t):
        """gloo works on host tensors: stage CUDA tensors through host memory."""
        return self.world > 1 and t.is_cuda and dist.get_backend(self.group) != "nccl"

    def sum(self, t):
        if self.world > 1:
            if self._host(t):
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def max(self, t):
        if self.world > 1:
            if self._host(t):
                h = t.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.MAX, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return t

    def gather(self, out, t):
        """out (world * t.numel()) <- concatenation of every rank's t."""
        if self.world > 1:
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


def as_device_matrix(x, name="d"):
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
        return t.contiguous(), kind
    a = np.asarray(x)
    if a.dtype != np.float32:
        a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={a.ndim}")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"{name} must have positive dimensions, got {a.shape}")
    t = torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", torch.cuda.current_device()))
    return t, "numpy"


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
