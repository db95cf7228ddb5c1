"""ML-CPCP drop-in: ``ml_fwt_solve`` (reference cpcp.py:480-515, loop
cpcp.py:326-456) on B200.

Per iteration the host enqueues
``lmo -> [all-reduce dots] -> update -> gram -> [all-reduce, all-gather] -> finalize``;
the corner decisions, the exact box QP (cpcp.py:202-231), the bound updates
and the 5-iteration convergence window all run on the device.
"""

from __future__ import annotations

import dataclasses
import os

import numpy as np
import torch

from . import _lib
from .api_types import CpcpOptions, CpcpState, IterationRecord, ObservationMask
from .backend import CudaCpcp, CudaSpectrum, chain_cholesky
from .chain import build_chain, resolve_coarse_width
from .runtime import SINGLE, Comm, as_device_matrix, give_back, give_back_all


# When set to a list, solves record per-phase CUDA-event timings into it.
TIMING_SINK = None
VERIFY_REPLICATED = os.environ.get("MLR_VERIFY_REPLICATED") == "1"  # see pcp.VERIFY_REPLICATED
# When set to a list, solves append their final device state (dict of
# mlr_cpcp_state: k, corner flags, the l1 arg-max (i_s, j_s), ...): tests.
STATE_SINK = None


class RankProbe:
    """collect_rank (reference cpcp.py:434-439): the numerical rank of the
    fine iterate L = L_H R^T after each update, i.e. #{sigma_i(L) >
    sigma_1(L) max(m, n) eps}.  sigma(L) = sigma(L_H C) with C C^T = R^T R,
    computed on the device by the two-pass spectrum plan (warm-started across
    iterations) and recorded by the finalize step as the iteration's rank_l.
    FP32 plans keep an FP64 shadow of L_H (same rank-1 updates, unrounded):
    the reference runs in float64, and FP32 rounding noise would otherwise
    count as rank."""

    def __init__(self, be, chain, comm, m_global, f32, device):
        self.comm = comm
        self.be = be
        lh, ld, done, self.slot = be.rank_binding()
        self.shadow = None
        if f32:
            self.shadow = torch.zeros((be.m_local, chain.n_coarse), dtype=torch.float64, device=device)
            lh, ld = self.shadow.data_ptr(), self.shadow.stride(0)
        self.lh, self.ld = lh, ld
        identity = chain.n_coarse == chain.n_fine and chain.n_factors == 0
        C = None if identity else chain_cholesky(chain, device)
        self.spec = CudaSpectrum(be.m_local, chain.n_coarse, False, device, C=C, skip_ptr=done)
        self.rel = max(m_global, chain.n_fine) * np.finfo(np.float64).eps

    def step(self):
        sp = self.spec
        if self.shadow is not None:
            self.be.rank_shadow(self.shadow)
        sp.gram(self.lh, self.ld)
        self.comm.sum(sp.red)
        sp.rotate(self.lh, self.ld)
        self.comm.sum(sp.red2)
        sp.finish(self.rel, rank_ptr=self.slot)

    def close(self):
        self.spec.close()


def run_fwt(be, comm, D, maskbits, m_global, opts, radius, check_every, probe=None, atoms=None):
    """Row-block host loop shared by the single-GPU and sharded entry points.
    ``probe`` records collect_rank; ``atoms`` (a list) receives the LMO factors
    (u, v) of every iteration for track_oracle_atoms."""
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
    pending = None
    while True:
        for _ in range(check_every):
            be.lmo()
            if atoms is not None:
                uv = (be.empty((be.m_local,), torch.float64), be.empty((be.nh,), torch.float64))
                be.atom_copy(*uv)
                atoms.append(uv)
            comm.sum(be.dots)
            be.update(D, maskbits, S)
            if probe is not None:
                probe.step()
            be.gram()
            comm.sum(be.red[:ns])
            comm.gather(be.amax_all, be.amax)
            if VERIFY_REPLICATED:
                comm.check_replicated(be.red[:ns], "K_g + stats")
                comm.check_replicated(be.amax_all, "arg-max records")
            be.finalize()
        # pipelined polling (see pcp.run_ialm)
        token = be.snapshot()
        if pending is not None:
            state = be.read_snapshot(pending)
            if state["done"]:
                break
        pending = token
    k = state["k"]
    L = be.empty(tuple(D.shape), D.dtype)
    be.outputs(L)
    hist, objs = be.history(k)
    return L, S, state, hist, objs


def _check_every(opts):
    if opts.check_every is not None:
        return max(1, int(opts.check_every))
    return 1 if opts.time_budget is not None else 8


def _oracle_atoms(be, atoms, out, kind):
    """track_oracle_atoms (cpcp.py:355-360): the dense LMO atom of every
    iteration (this rank's rows), expanded on the device from the saved
    factors; None on the P[D] = 0 early exit, like the reference."""
    if atoms is None:
        return None
    st = out[2]
    k = st["k"]
    if st["done"] == 1 and k == 1 and out[4][0] == 0.0 and out[3][0][0] == 0.0:
        return None
    res = []
    for u, v in atoms[:k]:
        a = be.empty((be.m_local, be.n), torch.float64)
        be.atom_dense(u, v, a)
        res.append(give_back(a, kind))
    return res


def _state_from(L, S, st, hist, objs, kind, atoms=None):
    history = [IterationRecord(i + 1, float(h[0]), float(h[1]), int(round(h[2])), float(h[3]), float(h[4]))
               for i, h in enumerate(hist)]
    l, s = give_back_all([L, S], kind)
    return CpcpState(l=l, s=s, t_l=float(st["t_l"]), t_s=float(st["t_s"]),
                     u_l=float(st["u_l"]), u_s=float(st["u_s"]), iter=int(st["k"]), history=history,
                     objective_history=[float(x) for x in objs], converged=st["done"] == 1, oracle_atoms=atoms)


def _mask_bits(mask, shape, device, rows=None):
    """The observation pattern as bit-packed rows on ``device`` (uint32 words,
    bit j & 31 of word j >> 5).  ``mask``: an ObservationMask, a boolean array,
    or a boolean / uint8 CUDA tensor (a mask already resident in HBM).  The
    bytes are packed on the device (``mlr_mask_pack``); a host mask crosses
    PCIe as one byte per entry."""
    if mask is None:
        return None
    if isinstance(mask, torch.Tensor):
        obs = mask if rows is None else mask[rows]
        if obs.dtype not in (torch.bool, torch.uint8):
            obs = obs != 0
        if tuple(obs.shape) != tuple(shape):
            raise ValueError("mask shape does not match data")
        obs = obs.to(device).contiguous()
    else:
        obs = mask.observed if isinstance(mask, ObservationMask) else np.asarray(mask)
        if obs.dtype != np.bool_:
            obs = obs.astype(bool)
        if rows is not None:
            obs = obs[rows]
        if obs.shape != tuple(shape):
            raise ValueError("mask shape does not match data")
        obs = torch.from_numpy(np.ascontiguousarray(obs).view(np.uint8)).to(device)
    m, n = shape
    words = (n + 31) // 32
    bits = torch.empty((m, words), dtype=torch.int32, device=device)
    if m:
        with torch.cuda.device(device):
            _lib.check(_lib.load().mlr_mask_pack(obs.data_ptr(), n, m, n, bits.data_ptr(), words,
                                                 torch.cuda.current_stream().cuda_stream))
    return bits


def ml_fwt_solve(d, mask=None, opts=None):
    """Multilevel Frank-Wolfe thresholding (drop-in for mlrpca.ml_fwt_solve)."""
    if opts is None:
        raise ValueError("CpcpOptions with penalty weights is required")
    D, kind = as_device_matrix(d, "d", opts.precision)
    m, n = D.shape
    with torch.cuda.device(D.device):
        nh = resolve_coarse_width(n, m, opts.levels, opts.rank_guess)
        chain = build_chain(n, nh)
        radius = 1.0 / chain.sigma_max()
        bits = _mask_bits(mask, (m, n), D.device)
        be = CudaCpcp(chain, m, m, 0, D.dtype == torch.float32, opts.max_iters, 1, D.device)
        if TIMING_SINK is not None:
            be.set_timing(True)
        probe = RankProbe(be, chain, SINGLE, m, D.dtype == torch.float32, D.device) if opts.collect_rank else None
        atoms = [] if opts.track_oracle_atoms else None
        try:
            out = run_fwt(be, SINGLE, D, bits, m, opts, radius, _check_every(opts), probe, atoms)
            atoms = _oracle_atoms(be, atoms, out, kind)
            if TIMING_SINK is not None:
                t = be.timing()
                t["iters"] = out[2]["k"]
                TIMING_SINK.append(t)
        finally:
            if probe is not None:
                probe.close()
            be.close()
    if STATE_SINK is not None:
        STATE_SINK.append(dict(out[2]))
    return _state_from(*out, kind, atoms)


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
    D, kind = as_device_matrix(d_local, "d", opts.precision)
    m, n = D.shape
    comm = Comm(group)
    with torch.cuda.device(D.device):
        chain = build_chain(n, resolve_coarse_width(n, m_global, opts.levels, opts.rank_guess))
        radius = 1.0 / chain.sigma_max()
        bits = _mask_bits(mask_local, (m, n), D.device)
        be = CudaCpcp(chain, m, m_global, row0, D.dtype == torch.float32, opts.max_iters, comm.world, D.device)
        probe = RankProbe(be, chain, comm, m_global, D.dtype == torch.float32, D.device) if opts.collect_rank else None
        atoms = [] if opts.track_oracle_atoms else None
        try:
            out = run_fwt(be, comm, D, bits, m_global, opts, radius, _check_every(opts), probe, atoms)
            atoms = _oracle_atoms(be, atoms, out, kind)
        finally:
            if probe is not None:
                probe.close()
            be.close()
    if STATE_SINK is not None:
        STATE_SINK.append(dict(out[2]))
    return _state_from(*out, kind, atoms)


__all__ = ["ml_fwt_solve", "fwt_solve", "ml_fwt_solve_rows", "CpcpOptions"]
