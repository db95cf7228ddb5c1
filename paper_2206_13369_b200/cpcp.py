"""ML-CPCP drop-in: ``ml_fwt_solve`` (reference cpcp.py:480-515, loop
cpcp.py:326-456) on B200.

Per iteration the host enqueues
``lmo -> [all-reduce dots] -> update -> gram -> [all-reduce, all-gather] -> finalize``;
the corner decisions, the exact box QP (cpcp.py:202-231), the bound updates
and the 5-iteration convergence window all run on the device.
"""

from __future__ import annotations

import dataclasses
import warnings

import numpy as np
import torch

from .api_types import CpcpOptions, CpcpState, IterationRecord, ObservationMask
from .backend import CudaCpcp
from .chain import build_chain, resolve_coarse_width
from .runtime import SINGLE, Comm, as_device_matrix, give_back


# When set to a list, solves record per-phase CUDA-event timings into it.
TIMING_SINK = None


def run_fwt(be, comm, D, maskbits, m_global, opts, radius, check_every):
    st = be.input_stats(D)
    comm.sum(st[2:3])
    if st[2].item() > 0:
        raise ValueError("d contains non-finite entries")
    opts.validate()
    S = be.empty(tuple(D.shape), D.dtype)
    be.start(D, maskbits, S, opts.lambda_l, opts.lambda_s, opts.tol, radius, opts.max_iters, opts.time_budget)
    nn, ns = be.stats_slice()
    be.gram()
    comm.sum(be.red[:ns])
    comm.gather(be.amax_all, be.amax)
    be.begin()
    while True:
        for _ in range(check_every):
            be.lmo()
            comm.sum(be.dots)
            be.update(D, maskbits, S)
            be.gram()
            comm.sum(be.red[:ns])
            comm.gather(be.amax_all, be.amax)
            be.finalize()
        state = be.state()
        if state["done"]:
            break
    k = state["k"]
    L = be.empty(tuple(D.shape), D.dtype)
    be.outputs(L)
    hist, objs = be.history(k)
    return L, S, state, hist, objs


def _check_every(opts):
    if opts.check_every is not None:
        return max(1, int(opts.check_every))
    return 1 if opts.time_budget is not None else 8


def _warn_unsupported(opts):
    if opts.track_oracle_atoms:
        raise NotImplementedError("track_oracle_atoms is not available on the GPU path")
    if opts.collect_rank:
        warnings.warn("collect_rank is not computed on the GPU path; rank_l is reported as -1",
                      RuntimeWarning, stacklevel=3)


def _state_from(L, S, st, hist, objs, kind):
    history = [IterationRecord(i + 1, float(h[0]), float(h[1]), int(round(h[2])), float(h[3]), float(h[4]))
               for i, h in enumerate(hist)]
    return CpcpState(l=give_back(L, kind), s=give_back(S, kind), t_l=float(st["t_l"]), t_s=float(st["t_s"]),
                     u_l=float(st["u_l"]), u_s=float(st["u_s"]), iter=int(st["k"]), history=history,
                     objective_history=[float(x) for x in objs], converged=st["done"] == 1)


def _mask_bits(mask, shape, device, rows=None):
    if mask is None:
        return None
    obs = mask.observed if isinstance(mask, ObservationMask) else np.asarray(mask).astype(bool)
    if rows is not None:
        obs = obs[rows]
    if obs.shape != tuple(shape):
        raise ValueError("mask shape does not match data")
    bits = ObservationMask(obs).packed_bits()
    return torch.from_numpy(bits.view(np.int32)).to(device)


def ml_fwt_solve(d, mask=None, opts=None):
    """Multilevel Frank-Wolfe thresholding (drop-in for mlrpca.ml_fwt_solve)."""
    if opts is None:
        raise ValueError("CpcpOptions with penalty weights is required")
    D, kind = as_device_matrix(d, "d")
    m, n = D.shape
    _warn_unsupported(opts)
    with torch.cuda.device(D.device):
        nh = resolve_coarse_width(n, m, opts.levels, opts.rank_guess)
        chain = build_chain(n, nh)
        radius = 1.0 / chain.sigma_max()
        bits = _mask_bits(mask, (m, n), D.device)
        be = CudaCpcp(chain, m, m, 0, D.dtype == torch.float32, opts.max_iters, 1, D.device)
        if TIMING_SINK is not None:
            be.set_timing(True)
        try:
            out = run_fwt(be, SINGLE, D, bits, m, opts, radius, _check_every(opts))
            if TIMING_SINK is not None:
                t = be.timing()
                t["iters"] = out[2]["k"]
                TIMING_SINK.append(t)
        finally:
            be.close()
    return _state_from(*out, kind)


def fwt_solve(d, mask=None, opts=None):
    """Full-width Frank-Wolfe thresholding (drop-in for mlrpca.fwt_solve,
    reference cpcp.py:459-477): the nuclear-ball linear minimisation step uses the leading
    singular triple of the full gradient.  It is the same device loop as
    ``ml_fwt_solve`` on the identity chain (R = I, radius 1), which the
    reference itself reproduces bit for bit (ml_fwt_solve with levels = n)."""
    if opts is None:
        raise ValueError("CpcpOptions with penalty weights is required")
    D, _ = as_device_matrix(d, "d")
    n = D.shape[1]
    full = dataclasses.replace(opts, levels=n)
    return ml_fwt_solve(d, mask, full)


def ml_fwt_solve_rows(d_local, mask_local, opts, m_global, row0, group=None):
    """Row-sharded ML-FWT: rows [row0, row0 + m_local) of the global problem
    on this rank; K_g, the stats, the QP dots and the l1 arg-max are combined
    over ``group``."""
    if opts is None:
        raise ValueError("CpcpOptions with penalty weights is required")
    D, kind = as_device_matrix(d_local, "d")
    m, n = D.shape
    comm = Comm(group)
    _warn_unsupported(opts)
    with torch.cuda.device(D.device):
        chain = build_chain(n, resolve_coarse_width(n, m_global, opts.levels, opts.rank_guess))
        radius = 1.0 / chain.sigma_max()
        bits = _mask_bits(mask_local, (m, n), D.device)
        be = CudaCpcp(chain, m, m_global, row0, D.dtype == torch.float32, opts.max_iters, comm.world, D.device)
        try:
            out = run_fwt(be, comm, D, bits, m_global, opts, radius, _check_every(opts))
        finally:
            be.close()
    return _state_from(*out, kind)


__all__ = ["ml_fwt_solve", "fwt_solve", "ml_fwt_solve_rows", "CpcpOptions"]
