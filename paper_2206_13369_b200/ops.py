"""Single-operation GPU entry points (used by tests and by callers who need the
restriction operators on device data).

``restrict`` / ``prolong`` mirror multilevel.restrict / multilevel.prolong
(multilevel.py:212-245); ``eigh_psd`` exposes the coarse Jacobi eigensolver;
``singular_values`` / ``matrix_rank`` expose the two-pass spectrum plan used
by the rank telemetry (collect_rank, collect_diagnostics).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .backend import CudaSpectrum
from .chain import Chain
from .runtime import as_device_matrix, give_back


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def restrict(x, chain: Chain):
    """x (m x n_fine) @ R -> (m x n_coarse)."""
    X, kind = as_device_matrix(x, "x")
    if X.shape[1] != chain.n_fine:
        raise ValueError(f"matrix has {X.shape[1]} columns, chain expects {chain.n_fine}")
    lib = _lib.load()
    h = chain.device_handle(X.device.index)
    np_ = lib.mlr_chain_padded_width(h)
    out = torch.empty((X.shape[0], np_), dtype=X.dtype, device=X.device)
    _lib.check(lib.mlr_restrict(h, X.shape[0], int(X.dtype == torch.float32), ctypes.c_void_p(X.data_ptr()),
                                X.stride(0), ctypes.c_void_p(out.data_ptr()), _stream()))
    return give_back(out[:, :chain.n_coarse].contiguous(), kind)


def prolong(x_h, chain: Chain):
    """x_h (m x n_coarse) @ R^T -> (m x n_fine)."""
    XH, kind = as_device_matrix(x_h, "x_h")
    if XH.shape[1] != chain.n_coarse:
        raise ValueError(f"matrix has {XH.shape[1]} columns, chain expects {chain.n_coarse}")
    lib = _lib.load()
    h = chain.device_handle(XH.device.index)
    np_ = lib.mlr_chain_padded_width(h)
    pad = torch.zeros((XH.shape[0], np_), dtype=XH.dtype, device=XH.device)
    pad[:, :chain.n_coarse] = XH
    out = torch.empty((XH.shape[0], chain.n_fine), dtype=XH.dtype, device=XH.device)
    _lib.check(lib.mlr_prolong(h, XH.shape[0], int(XH.dtype == torch.float32), ctypes.c_void_p(pad.data_ptr()),
                               ctypes.c_void_p(out.data_ptr()), out.stride(0), _stream()))
    return give_back(out, kind)


def eigh_psd(b, tol=None, max_sweeps=60):
    """Eigen-decomposition of a symmetric PSD matrix by the one-sided block
    Jacobi kernel.  Returns (eigenvalues, eigenvectors-as-columns, sweeps),
    eigenvalues sorted descending."""
    B, kind = as_device_matrix(b, "b")
    n = B.shape[0]
    if B.shape[1] != n:
        raise ValueError("b must be square")
    B = B.to(torch.float64)
    np_ = ((n + 63) // 64) * 64
    Bp = torch.zeros((np_, np_), dtype=torch.float64, device=B.device)
    Bp[:n, :n] = B
    lib = _lib.load()
    V = torch.empty_like(Bp)
    lam = torch.empty(np_, dtype=torch.float64, device=B.device)
    work = torch.empty(int(lib.mlr_eigh_work_doubles(np_)), dtype=torch.float64, device=B.device)
    info = np.zeros(1, dtype=np.int32)
    tol = 64 * np.finfo(np.float64).eps if tol is None else float(tol)
    _lib.check(lib.mlr_eigh_psd(np_, ctypes.c_void_p(Bp.data_ptr()), ctypes.c_void_p(V.data_ptr()),
                                ctypes.c_void_p(lam.data_ptr()), tol, int(max_sweeps),
                                ctypes.c_void_p(work.data_ptr()), info.ctypes.data, _stream()))
    # padded columns are zero in X, so rotations never touch them: columns
    # [0, n) of V span the real coordinates
    order = torch.argsort(lam[:n], descending=True)
    return (give_back(lam[:n][order].contiguous(), kind), give_back(V[:n, :n][:, order].contiguous(), kind),
            int(info[0]))


def _spectrum(x, rel):
    X, kind = as_device_matrix(x, "x")
    if X.shape[1] > X.shape[0]:
        X = X.t().contiguous()
    m, n = X.shape
    f32 = X.dtype == torch.float32
    with torch.cuda.device(X.device):
        sp = CudaSpectrum(m, n, f32, X.device)
        try:
            sig = torch.zeros(sp.np_, dtype=torch.float64, device=X.device)
            rank = torch.zeros(1, dtype=torch.float64, device=X.device)
            sp.gram(X.data_ptr(), X.stride(0))
            sp.rotate(X.data_ptr(), X.stride(0))
            sp.finish(rel, sig_out=sig, rank_ptr=rank.data_ptr())
            torch.cuda.current_stream().synchronize()
        finally:
            sp.close()
    return sig[:n], int(rank.item()), kind


def singular_values(x):
    """All min(m, n) singular values of x, descending, accurate to ~eps * sigma_1
    (Gram + Jacobi, then Jacobi on the Gram of the rotated columns)."""
    sig, _, kind = _spectrum(x, 0.0)
    return give_back(sig.contiguous(), kind)


def matrix_rank(x):
    """#{sigma_i > sigma_1 * max(m, n) * eps(dtype)} (numpy.linalg.matrix_rank's
    default tolerance; the reference's rank_l column, cpcp.py:434-439)."""
    X, _ = as_device_matrix(x, "x")
    eps = np.finfo(np.float32 if X.dtype == torch.float32 else np.float64).eps
    return _spectrum(X, max(X.shape) * eps)[1]
