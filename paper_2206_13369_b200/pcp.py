"""ML-PCP drop-in: ``ml_ialm_solve`` (reference pcp.py:213-309) and the
full-width ``ialm_solve`` (pcp.py:118-197) on B200.

The host loop mirrors the reference's structure and stopping rules; every
arithmetic step runs in the CUDA library.  Per iteration the host enqueues
``svt -> update -> gram -> [all-reduce] -> finalize`` and polls the
device-side stopping flag every ``check_every`` iterations, so the GPU is
never idle waiting for Python.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from .api_types import IterationRecord, MultilevelDiagnostics, PcpOptions, PcpState, SvdError
from .backend import CudaPcp, CudaSpectrum
from .chain import build_chain, resolve_coarse_width
from .runtime import SINGLE, Comm, as_device_matrix, give_back, give_back_all

LANCZOS_TOL = 1e-15
# Debug: check that the all-reduced Gram every rank feeds its replicated
# Jacobi is bitwise identical across ranks (runtime.Comm.check_replicated).
VERIFY_REPLICATED = os.environ.get("MLR_VERIFY_REPLICATED") == "1"

# When set to a list, solves record per-phase CUDA-event timings into it
# (one dict per solve; used by bench.py for the roofline figures).
TIMING_SINK = None


def _zero_state(shape, kind, like):
    z = torch.zeros(shape, dtype=like.dtype, device=like.device)
    rec = IterationRecord(1, 0.0, 0.0, 0, 0.0, 0.0)
    return PcpState(l=give_back(z, kind), s=give_back(z.clone(), kind), y=give_back(z.clone(), kind), mu=0.0,
                    iter=1, history=[rec], mu_history=[], converged=True)


def _jacobi_tol(opts, f32):
    if opts.jacobi_tol is not None:
        return float(opts.jacobi_tol)
    # FP32 data carries ~6e-8 relative noise; a 1e-6 relative off-diagonal
    # test leaves relF(L) vs the FP64 reference unchanged on C2 (4.8e-6 vs 4.7e-6
    # at 1e-9) and saves ~10% of the sweeps (tools/gpu/jacobi_tol_sweep.py)
    return 1e-6 if f32 else 64 * np.finfo(np.float64).eps


def run_ialm(be, comm, D, m_global, n, opts, lam, check_every, coarse=None):
    """Row-block host loop shared by the single-GPU and sharded entry points.

    ``coarse`` (a list) receives a copy of the coarse iterate L_H after every
    SVT step (collect_diagnostics).  Returns (L, S, Y, state dict, history
    array) or None for a zero D."""
    st3 = be.input_stats(D)
    comm.sum(st3[0:1])
    comm.max(st3[1:2])
    comm.sum(st3[2:3])
    sumsq, _, bad = st3[:3].tolist()
    if bad > 0:
        raise ValueError("d contains non-finite entries")
    if sumsq == 0.0:
        return None
    opts.validate()
    # sigma_1(D) by Lanczos on D^T D (pcp.py:100, 114).  float32 data only
    # needs sigma_1 far below its own rounding (6e-8): mu0 = 1.25/sigma_1 scales
    # every later mu, and a 1e-9 relative error in theta moves mu0 by ~1e-9
    lz_tol = LANCZOS_TOL if D.dtype == torch.float64 else 1e-9
    be.lanczos_init()
    steps = 0
    # one rank: the whole run is one cooperative kernel; otherwise batches of
    # steps with the all-reduce in between and pipelined polling (batch j + 1
    # is queued before batch j's state is read; steps after convergence are
    # no-ops on the device)
    run_whole = comm.world == 1 and getattr(be, "lanczos_run_available", lambda: False)()
    if run_whole:
        be.lanczos_run(D, lz_tol)
    pending = None
    while not run_whole:
        for _ in range(4):
            w = be.lanczos_matvec(D)
            comm.sum(w)
            be.lanczos_update(w, lz_tol)
            steps += 1
        token = be.snapshot()
        if pending is not None and be.read_snapshot(pending)[1]["done"]:
            break
        pending = token
        if steps > 2 * n + 24:
            raise SvdError("Lanczos estimate of sigma_1(D) did not converge", iterations=steps)
    f32 = D.dtype == torch.float32
    Y = [be.empty(tuple(D.shape), D.dtype), be.empty(tuple(D.shape), D.dtype)]
    be.start(D, Y[0], lam, opts.mu0, opts.rho, opts.tol_feasibility, opts.max_iters, opts.time_budget,
             _jacobi_tol(opts, f32), 60)
    nn, ns = be.stats_slice()
    be.gram(0)
    comm.sum(be.red[:nn])
    calls = 0
    pending = None
    while True:
        for _ in range(check_every):
            be.svt()
            if coarse is not None:
                z = be.empty((D.shape[0], be.nh), D.dtype)
                be.coarse_copy(z)
                coarse.append(z)
            be.update(D, Y[calls % 2], Y[(calls + 1) % 2])
            calls += 1
            be.gram(1)
            comm.sum(be.red[:ns])
            if VERIFY_REPLICATED:
                comm.check_replicated(be.red[:ns], "coarse Gram + stats")
            be.finalize()
        # pipelined polling: the next batch is queued before this one's state
        # is read; once done, every further step is a no-op on the device
        token = be.snapshot()
        if pending is not None:
            st = be.read_snapshot(pending)[0]
            if st["done"]:
                break
        pending = token
    if st["done"] == 3:
        raise SvdError("coarse Jacobi eigensolver did not converge", iterations=-st["jac_sweeps"])
    k = st["k"]
    L = be.empty(tuple(D.shape), D.dtype)
    S = be.empty(tuple(D.shape), D.dtype)
    be.outputs(D, Y[(k - 1) % 2], L, S)
    hist = be.history(k)
    return L, S, Y[k % 2], st, hist


def diagnostics(be, comm, chain, coarse, k, m_global):
    """collect_diagnostics (reference pcp.py:298-306): epsilon_bound of the
    final coarse iterate (multilevel.py:248-265) and the alignment errors
    delta_j = <L_H^j (R^T R - I), L_H^j - restrict(L_final)>, with
    restrict(L_final) = L_H^final R^T R.  All on the device: one streaming
    pass per delta, and the two-pass spectrum plan for sigma(L_H^final)."""
    zs = coarse[:k]
    zf = zs[-1]
    dev = zf.device
    deltas = torch.zeros(k, dtype=torch.float64, device=dev)
    work = torch.zeros(int(be.lib.mlr_pcp_delta_work_doubles()), dtype=torch.float64, device=dev)
    for j, z in enumerate(zs):
        be.delta(z, zf, deltas[j:j + 1], work)
    comm.sum(deltas)
    f32 = zf.dtype == torch.float32
    nh = chain.n_coarse
    spec = CudaSpectrum(zf.shape[0], nh, f32, dev)
    try:
        spec.gram(zf.data_ptr(), zf.stride(0))
        comm.sum(spec.red)
        spec.rotate(zf.data_ptr(), zf.stride(0))
        comm.sum(spec.red2)
        # k-th largest sigma(L_H) pairs with the k-th smallest sigma(R)
        pair = torch.zeros(spec.np_, dtype=torch.float64)
        pair[:nh] = torch.from_numpy(1.0 - chain.composite_sigmas()[::-1].copy())
        pair = pair.to(dev)
        out = torch.zeros(2, dtype=torch.float64, device=dev)
        eps = np.finfo(np.float32 if f32 else np.float64).eps
        spec.finish(max(m_global, nh) * eps, rank_ptr=out[1:].data_ptr(), pair_w=pair, wsum_out=out[:1])
        epsilon = float(out[0].item())
    finally:
        spec.close()
    return MultilevelDiagnostics(epsilon=epsilon, delta_history=[float(x) for x in deltas.tolist()])


def _state_from(L, S, Yk, st, hist, kind):
    history = [IterationRecord(i + 1, float(h[0]), float(h[1]), int(round(h[2])), float(h[3]), float(h[4]))
               for i, h in enumerate(hist)]
    l, s, y = give_back_all([L, S, Yk], kind)
    return PcpState(l=l, s=s, y=y, mu=float(st["mu_final"]),
                    iter=int(st["k"]), history=history, mu_history=[float(x) for x in hist[:, 5]],
                    converged=st["done"] == 1)


def ml_ialm_solve(d, opts=None):
    """Multilevel inexact ALM (drop-in for mlrpca.ml_ialm_solve).

    ``d`` may be a numpy array (any dtype coercible to float64; float32 input
    runs the FP32 path), or a torch tensor (CPU or CUDA; results stay on the
    input's side).  ``opts.levels`` is the coarse width n_H, as in the
    reference.  Raises ValueError / LevelError / SvdError like the reference.
    """
    opts = opts if opts is not None else PcpOptions()
    D, kind = as_device_matrix(d, "d", opts.precision)
    m, n = D.shape
    lam = opts.lam if opts.lam is not None else 1.0 / np.sqrt(max(m, n))
    diag = None
    with torch.cuda.device(D.device):
        opts_checked = _checked_width(n, m, opts)
        chain = build_chain(n, opts_checked)
        be = CudaPcp(chain, m, m, D.dtype == torch.float32, opts.max_iters, D.device)
        if TIMING_SINK is not None:
            be.set_timing(True)
        coarse = [] if opts.collect_diagnostics else None
        try:
            out = run_ialm(be, SINGLE, D, m, n, opts, lam, _check_every(opts), coarse)
            if coarse is not None and out is not None:
                diag = diagnostics(be, SINGLE, chain, coarse, out[3]["k"], m)
            if TIMING_SINK is not None:
                t = be.timing()
                t["iters"] = out[3]["k"] if out is not None else 0
                t["jac_sweeps"] = [int(x) for x in out[4][:, 6]] if out is not None else []
                t["lanczos_steps"] = be.lanczos_state()["k"] + 1
                TIMING_SINK.append(t)
        finally:
            be.close()
    if out is None:
        return _zero_state(tuple(D.shape), kind, D)
    state = _state_from(*out, kind)
    state.diagnostics = diag
    return state


def ialm_solve(d, opts=None):
    """Full-width inexact ALM (drop-in for mlrpca.ialm_solve, reference
    pcp.py:118-197).

    Runs the ML-PCP device loop on the identity chain (n_H = n, so the
    restriction is exact) with the truncated SVT enabled: only the top ``sv``
    singular values take part, and ``sv`` adapts each iteration exactly as
    the reference's svd_truncated bookkeeping does (pcp.py:132-138,
    160-165).  PCP is transpose-symmetric (lam, mu0, the dual start and both
    shrinkages are), so a wide ``d`` is solved as its transpose and the
    Gram stays min(m, n) square.
    """
    opts = opts if opts is not None else PcpOptions()
    D, kind = as_device_matrix(d, "d", opts.precision)
    m, n = D.shape
    lam = opts.lam if opts.lam is not None else 1.0 / np.sqrt(max(m, n))
    wide = n > m
    if wide:
        D = D.t().contiguous()
        m, n = n, m
    kmax = n
    cap = min(opts.svd_budget or kmax, kmax)
    sv0 = min(opts.rank_guess + 1, cap)
    with torch.cuda.device(D.device):
        chain = build_chain(n, n)
        be = CudaPcp(chain, m, m, D.dtype == torch.float32, opts.max_iters, D.device)
        be.set_truncation(sv0, cap)
        if TIMING_SINK is not None:
            be.set_timing(True)
        try:
            out = run_ialm(be, SINGLE, D, m, n, opts, lam, _check_every(opts))
            if TIMING_SINK is not None:
                t = be.timing()
                t["iters"] = out[3]["k"] if out is not None else 0
                t["jac_sweeps"] = [int(x) for x in out[4][:, 6]] if out is not None else []
                t["lanczos_steps"] = be.lanczos_state()["k"] + 1
                TIMING_SINK.append(t)
        finally:
            be.close()
    if out is None:
        shape = (n, m) if wide else (m, n)
        return _zero_state(shape, kind, D)
    if wide:
        L, S, Yk, st, hist = out
        out = (L.t().contiguous(), S.t().contiguous(), Yk.t().contiguous(), st, hist)
    return _state_from(*out, kind)


def _checked_width(n, m, opts):
    return resolve_coarse_width(n, m, opts.levels, opts.rank_guess)


def _check_every(opts):
    if opts.check_every is not None:
        return max(1, int(opts.check_every))
    return 1 if opts.time_budget is not None else 4


def ml_ialm_solve_rows(d_local, opts, m_global, group=None):
    """Row-sharded ML-IALM: this rank holds rows of the global m_global x n
    iterate; K = A^T A and the per-iteration reductions are all-reduced over
    ``group`` (NCCL).  Returns a PcpState whose arrays are this rank's rows."""
    D, kind = as_device_matrix(d_local, "d", opts.precision)
    m, n = D.shape
    comm = Comm(group)
    lam = opts.lam if opts.lam is not None else 1.0 / np.sqrt(max(m_global, n))
    diag = None
    with torch.cuda.device(D.device):
        chain = build_chain(n, _checked_width(n, m_global, opts))
        be = CudaPcp(chain, m, m_global, D.dtype == torch.float32, opts.max_iters, D.device)
        if TIMING_SINK is not None:
            be.set_timing(True)
        coarse = [] if opts.collect_diagnostics else None
        try:
            out = run_ialm(be, comm, D, m_global, n, opts, lam, _check_every(opts), coarse)
            if coarse is not None and out is not None:
                diag = diagnostics(be, comm, chain, coarse, out[3]["k"], m_global)
            if TIMING_SINK is not None:
                t = be.timing()
                t["iters"] = out[3]["k"] if out is not None else 0
                t["jac_sweeps"] = [int(x) for x in out[4][:, 6]] if out is not None else []
                t["lanczos_steps"] = be.lanczos_state()["k"] + 1
                TIMING_SINK.append(t)
        finally:
            be.close()
    if out is None:
        return _zero_state(tuple(D.shape), kind, D)
    state = _state_from(*out, kind)
    state.diagnostics = diag
    return state
