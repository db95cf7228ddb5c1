"""Host-side restriction chain (built once per solve) and its device upload.

Same operator as the reference's ``build_chain`` (multilevel.py:125-179):
the composite of halving interpolation factors (multilevel.py:23-57), scaled
by its exact spectral norm.  Every fine row of the composite has at most two
adjacent nonzeros, so the device receives it as a 2-tap stencil
``(c0[j], w0[j], w1[j])`` plus the tridiagonal of ``G_R = R^T R``; the
reference instead multiplies by the dense ``n x n_H`` matrix
(pcp.py:236, cpcp.py:503).
"""

from __future__ import annotations

import ctypes
import functools
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib


class LevelError(ValueError):
    """No coarse level satisfies the requested constraints (multilevel.py:19-20)."""


def coarse_sizes(n):
    """Widths reachable from ``n`` by repeated halving (multilevel.py:60-65)."""
    out = [int(n)]
    while out[-1] > 1:
        out.append((out[-1] + 1) // 2)
    return out


def _factor_taps(n):
    """Taps of one halving factor (multilevel.py:23-57) as, per fine row i,
    the list of (coarse column, weight)."""
    if n < 2:
        raise ValueError(f"fine size must be >= 2, got {n}")
    nh = (n + 1) // 2
    odd = n & 1
    rows = [[] for _ in range(n)]
    last = nh - 2 if odd else nh - 1
    for j in range(last + 1):
        if j == 0:
            taps = ((0, 1.0), (1, 1.0), (2, 0.5))
        elif j == nh - 1:
            taps = ((n - 2, 0.5), (n - 1, 1.0))
        else:
            taps = ((2 * j, 0.5), (2 * j + 1, 1.0), (2 * j + 2, 0.5))
        for i, w in taps:
            if i < n and not (odd and i == n - 1):
                rows[i].append((j, w))
    if odd:
        rows[n - 1].append((nh - 1, 1.0))
    return rows


def interpolation_dense(n):
    """Dense (n, ceil(n/2)) halving factor (for tests / small sizes)."""
    rows = _factor_taps(n)
    out = np.zeros((n, (n + 1) // 2))
    for i, taps in enumerate(rows):
        for j, w in taps:
            out[i, j] += w
    return out


def _compose(n, target):
    """Raw (unnormalised) composite as per-row sparse dicts {col: weight}."""
    cur = [{i: 1.0} for i in range(n)]
    size = n
    nfac = 0
    while size > target:
        taps = _factor_taps(size)
        nxt = []
        for row in cur:
            acc = {}
            for mid, w in row.items():
                for c, v in taps[mid]:
                    acc[c] = acc.get(c, 0.0) + w * v
            nxt.append(acc)
        cur = nxt
        size = (size + 1) // 2
        nfac += 1
    return cur, nfac


@dataclass
class Chain:
    """Normalised composite restriction R (n x n_coarse) in stencil form."""

    n_fine: int
    n_coarse: int
    n_factors: int
    spectral_norm: float
    c0: np.ndarray      # int32 [n]
    w0: np.ndarray      # float64 [n]
    w1: np.ndarray      # float64 [n]
    g_diag: np.ndarray  # float64 [n_coarse]
    g_off: np.ndarray   # float64 [n_coarse - 1]
    _dev: dict = field(default_factory=dict, repr=False)

    def dense(self):
        r = np.zeros((self.n_fine, self.n_coarse))
        j = np.arange(self.n_fine)
        r[j, self.c0] += self.w0
        nz = self.w1 != 0
        r[j[nz], self.c0[nz] + 1] += self.w1[nz]
        return r

    def sigma_max(self):
        """Largest singular value of R (cpcp.py:502 uses 1/sigma_1 as radius).

        R^T R is tridiagonal: dense eigvalsh for small n_H (bit-for-bit the
        reference's call), LAPACK bisection on the tridiagonal for large n_H
        (the dense solve is O(n_H^3)); the identity chain is exactly 1."""
        if self.n_coarse == self.n_fine and not np.any(self.g_off) and np.all(self.g_diag == 1.0):
            return 1.0
        if self.n_coarse > 512:
            from scipy.linalg import eigvalsh_tridiagonal
            k = self.n_coarse - 1
            top = eigvalsh_tridiagonal(self.g_diag, self.g_off, select="i", select_range=(k, k))[0]
            return float(np.sqrt(max(top, 0.0)))
        g = np.diag(self.g_diag) + np.diag(self.g_off, 1) + np.diag(self.g_off, -1)
        return float(np.sqrt(max(np.linalg.eigvalsh(g)[-1], 0.0)))

    def composite_sigmas(self):
        """All singular values of R, descending (multilevel.py:90-95); from the
        tridiagonal R^T R (host-side chain setup, like sigma_max)."""
        if self.n_coarse == self.n_fine and not np.any(self.g_off) and np.all(self.g_diag == 1.0):
            return np.ones(self.n_coarse)
        from scipy.linalg import eigvalsh_tridiagonal
        lam = eigvalsh_tridiagonal(self.g_diag, self.g_off) if self.n_coarse > 1 else self.g_diag.copy()
        return np.sqrt(np.maximum(lam, 0.0))[::-1].copy()

    def device_handle(self, device_index):
        """Chain tables on the given CUDA device (uploaded once, cached)."""
        h = self._dev.get(device_index)
        if h is None:
            import torch
            lib = _lib.load()
            with torch.cuda.device(device_index):
                out = ctypes.c_void_p()
                c0 = np.ascontiguousarray(self.c0, dtype=np.int32)
                w0 = np.ascontiguousarray(self.w0)
                w1 = np.ascontiguousarray(self.w1)
                gd = np.ascontiguousarray(self.g_diag)
                go = np.ascontiguousarray(self.g_off if self.g_off.size else np.zeros(1))
                _lib.check(lib.mlr_chain_create(
                    self.n_fine, self.n_coarse, c0.ctypes.data, w0.ctypes.data, w1.ctypes.data,
                    gd.ctypes.data, go.ctypes.data, ctypes.byref(out)))
            h = out.value
            self._dev[device_index] = h
        return h

    def __del__(self):
        try:
            lib = _lib._lib
            if lib is not None:
                for h in self._dev.values():
                    lib.mlr_chain_destroy(h)
        except Exception:
            pass


_CACHE: dict = {}


@functools.lru_cache(maxsize=16)
def build_chain(n, n_coarse_target):
    """Normalised chain from ``n`` down to ``n_coarse_target`` (reachable by
    repeated halving; ``n`` itself gives the identity).  Mirrors the checks
    and error messages of multilevel.build_chain."""
    n, target = int(n), int(n_coarse_target)
    if n < 1 or target < 1:
        raise ValueError("sizes must be positive")
    key = (n, target)
    if key in _CACHE:
        return _CACHE[key]
    sizes = coarse_sizes(n)
    if target not in sizes:
        above = [s for s in sizes if s > target]
        below = [s for s in sizes if s < target]
        near = ([str(min(above))] if above else []) + ([str(max(below))] if below else [])
        raise ValueError(
            f"coarse size {target} is not reachable from {n} by repeated "
            f"halving; nearest reachable sizes: {' and '.join(near)}")
    rows, nfac = _compose(n, target)
    # the raw composite's Gram (dyadic, formed exactly) gives sigma_1 like the
    # reference's eigvalsh of (raw^T raw) (multilevel.py:160-164)
    c0 = np.empty(n, dtype=np.int32)
    r0 = np.empty(n)
    r1 = np.zeros(n)
    for j, row in enumerate(rows):
        cols = sorted(c for c, w in row.items() if w != 0.0)
        if not cols or len(cols) > 2 or (len(cols) == 2 and cols[1] != cols[0] + 1):
            raise RuntimeError("composite restriction is not a 2-tap stencil")
        c0[j] = cols[0]
        r0[j] = row[cols[0]]
        if len(cols) == 2:
            r1[j] = row[cols[1]]
    graw = np.zeros((target, target))
    np.add.at(graw, (c0, c0), r0 * r0)
    has1 = r1 != 0
    np.add.at(graw, (c0[has1] + 1, c0[has1] + 1), r1[has1] * r1[has1])
    np.add.at(graw, (c0[has1], c0[has1] + 1), r0[has1] * r1[has1])
    np.add.at(graw, (c0[has1] + 1, c0[has1]), r0[has1] * r1[has1])
    if nfac == 0 and target == n:
        spectral = 1.0  # no coarsening: raw = I and eigvalsh(I) is exactly 1
    else:
        spectral = float(np.sqrt(max(np.linalg.eigvalsh(graw)[-1], 0.0)))
    if spectral == 0.0:
        raise ValueError("composite operator is zero; cannot normalize")
    # scipy divides a sparse array by a scalar as a multiply by its reciprocal
    inv = 1.0 / spectral
    w0 = r0 * inv
    w1 = r1 * inv
    gd = np.zeros(target)
    go = np.zeros(max(target - 1, 0))
    np.add.at(gd, c0, w0 * w0)
    np.add.at(gd, c0[has1] + 1, w1[has1] * w1[has1])
    if target > 1:
        np.add.at(go, c0[has1], w0[has1] * w1[has1])
    ch = Chain(n, target, nfac, spectral, c0, w0, w1, gd, go)
    _CACHE[key] = ch
    return ch


def select_levels(n, rank_guess, r_needed, m):
    """Smallest reachable n_H > max(rank_guess, r_needed) (multilevel.py:182-209)."""
    n, m, rank_guess, r_needed = int(n), int(m), int(rank_guess), int(r_needed)
    if rank_guess < 1 or m < 1:
        raise ValueError("rank_guess and m must be positive")
    floor = max(rank_guess, r_needed)
    cands = [s for s in coarse_sizes(n) if s > floor]
    if not cands:
        raise LevelError(
            f"no coarse level reachable from n={n} satisfies "
            f"n_H > max(rank_guess, r_needed) = {floor}")
    best = min(cands)
    if best > (m + 1) / 2:
        warnings.warn(
            f"coarse size {best} violates n_H <= (m+1)/2 = {(m + 1) / 2}; "
            "the rank bound cannot be certified for this problem",
            RuntimeWarning, stacklevel=3)
    return best


def resolve_coarse_width(n, m, levels, rank_guess):
    """``levels`` is the coarse width n_H (pcp.py:200-210, cpcp.py:492-500)."""
    if levels is not None:
        if levels < 1:
            raise LevelError(
                f"coarse size {levels} is invalid: the rank bound "
                f"requires rank(L) <= n_H <= (m+1)/2 with n_H >= 1")
        return int(levels)
    return select_levels(n, rank_guess, 1, m)
