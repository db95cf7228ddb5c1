"""CPU oracle for the multilevel PCP / CPCP hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain numpy/scipy restatement of the reference package
``mlrpca`` 0.1.0 (``/root/reference/pkg/src/mlrpca``), limited to what the
two multilevel solvers execute.  It exists so that

  * ``tests/`` can check the CUDA path against the reference algorithm on the
    GPU box (where ``/root/reference`` is absent),
  * ``bench.py --impl reference`` / the ``cpu_baseline`` leg can time the
    reference algorithm on the box's host cores (``kind: "port"``),
  * ``__graft_entry__.smoke()`` has a checker.

Nothing in ``paper_2206_13369_b200/`` imports this module; the product path
must never route through it.

Pinning: ``tests/test_oracle_pinning.py`` checks this restatement against the
reference's own known-answer tests (``pkg/tests/test_linalg.py``,
``pkg/tests/test_multilevel.py``) and against golden vectors produced by the
real reference (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``).
The restatement follows the reference's floating-point operation order, so on
the same numpy/scipy build the solver outputs agree bit for bit.

Every function cites the reference ``file:line`` it restates; paths are
relative to ``pkg/src/mlrpca/``.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse.linalg
import scipy.sparse as sp

# --------------------------------------------------------------------------
# linalg.py
# --------------------------------------------------------------------------


def as_matrix(x, name="x"):
    """linalg.py:48-57 — finite, 2-D, positive-dims float64."""
    arr = np.asarray(x, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={arr.ndim}")
    if min(arr.shape) < 1:
        raise ValueError(f"{name} must have positive dimensions, got {arr.shape}")
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains non-finite entries")
    return arr


def soft_threshold(x, tau):
    """linalg.py:60-72 — sign(x)*max(|x|-tau, 0), same op order."""
    if tau < 0:
        raise ValueError(f"threshold must be nonnegative, got {tau}")
    x = np.asarray(x, dtype=np.float64)
    mag = np.abs(x)
    mag -= tau
    np.maximum(mag, 0.0, out=mag)
    return np.copysign(mag, x, out=mag)


def svd_full(x):
    """linalg.py:86-99 (+ _fix_signs 75-83): thin SVD, sigma descending."""
    x = as_matrix(x)
    try:
        u, s, vt = np.linalg.svd(x, full_matrices=False)
    except np.linalg.LinAlgError:
        u, s, vt = scipy.linalg.svd(x, full_matrices=False, lapack_driver="gesvd")
    v = vt.T
    if u.shape[1]:
        peak = np.argmax(np.abs(u), axis=0)
        sgn = np.sign(u[peak, np.arange(u.shape[1])])
        sgn[sgn == 0] = 1.0
        u, v = u * sgn, v * sgn
    return u, s, v


def svt(x, tau):
    """linalg.py:128-142 — (z, rank); ties sigma == tau are not counted."""
    if tau < 0:
        raise ValueError(f"threshold must be nonnegative, got {tau}")
    u, s, v = svd_full(x)
    k = int(np.count_nonzero(s > tau))
    if k == 0:
        return np.zeros_like(np.asarray(x, dtype=np.float64)), 0
    return (u[:, :k] * (s[:k] - tau)) @ v[:, :k].T, k


# --------------------------------------------------------------------------
# multilevel.py
# --------------------------------------------------------------------------


class LevelError(ValueError):
    """multilevel.py:19-20."""


def build_interpolation(n):
    """multilevel.py:23-57 — one halving factor, shape (n, ceil(n/2)).

    Coarse column j injects weight 1 at fine row 2j+1 and 1/2 at 2j, 2j+2
    (column 0 also weight 1 at row 0; the last column of an even n gets
    (n-2: 1/2, n-1: 1)); for odd n the final fine row is reserved for a unit
    injection from the trailing coarse column.
    """
    n = int(n)
    if n < 2:
        raise ValueError(f"fine size must be >= 2, got {n}")
    nh = (n + 1) // 2
    odd = n % 2 == 1
    last_regular = nh - 2 if odd else nh - 1
    entries = []
    for j in range(last_regular + 1):
        if j == 0:
            taps = ((0, 1.0), (1, 1.0), (2, 0.5))
        elif j == nh - 1:
            taps = ((n - 2, 0.5), (n - 1, 1.0))
        else:
            taps = ((2 * j, 0.5), (2 * j + 1, 1.0), (2 * j + 2, 0.5))
        for i, w in taps:
            if i < n and not (odd and i == n - 1):
                entries.append((i, j, w))
    if odd:
        entries.append((n - 1, nh - 1, 1.0))
    rows = [e[0] for e in entries]
    cols = [e[1] for e in entries]
    vals = [e[2] for e in entries]
    return sp.csr_array((vals, (rows, cols)), shape=(n, nh))


def coarse_sizes(n):
    """multilevel.py:60-65."""
    out = [int(n)]
    while out[-1] > 1:
        out.append((out[-1] + 1) // 2)
    return out


@dataclass
class Chain:
    """multilevel.py:68-102 (RestrictionChain), reduced to what solvers use."""

    n_fine: int
    n_coarse: int
    composite: sp.csr_array
    raw_composite: sp.csr_array
    spectral_norm: float
    n_factors: int
    _cho: tuple | None = field(default=None, repr=False)
    _sig: np.ndarray | None = field(default=None, repr=False)

    def gram_cho(self):
        """multilevel.py:97-102."""
        if self._cho is None:
            g = (self.composite.T @ self.composite).toarray()
            self._cho = scipy.linalg.cho_factor(g)
        return self._cho

    def composite_sigmas(self):
        """multilevel.py:90-95."""
        if self._sig is None:
            self._sig = np.linalg.svd(self.composite.toarray(), compute_uv=False)
        return self._sig


def build_chain(n, target, normalize=True):
    """multilevel.py:125-179."""
    n, target = int(n), int(target)
    if n < 1 or target < 1:
        raise ValueError("sizes must be positive")
    sizes = coarse_sizes(n)
    if target not in sizes:
        above = [s for s in sizes if s > target]
        below = [s for s in sizes if s < target]
        near = ([str(min(above))] if above else []) + ([str(max(below))] if below else [])
        raise ValueError(
            f"coarse size {target} is not reachable from {n} by repeated "
            f"halving; nearest reachable sizes: {' and '.join(near)}")
    factors = []
    size = n
    while size > target:
        factors.append(build_interpolation(size))
        size = (size + 1) // 2
    raw = sp.csr_array(sp.identity(n, format="csr"))
    for f in factors:
        raw = sp.csr_array(raw @ f)
    lam_max = np.linalg.eigvalsh((raw.T @ raw).toarray())[-1]
    spectral = float(np.sqrt(max(lam_max, 0.0)))
    if normalize:
        if spectral == 0.0:
            raise ValueError("composite operator is zero; cannot normalize")
        comp = sp.csr_array(raw / spectral)
    else:
        comp = raw
    return Chain(n, target, comp, raw, spectral, len(factors))


def select_levels(n, rank_guess, r_needed, m):
    """multilevel.py:182-209."""
    n, m, rank_guess, r_needed = int(n), int(m), int(rank_guess), int(r_needed)
    if rank_guess < 1 or m < 1:
        raise ValueError("rank_guess and m must be positive")
    floor = max(rank_guess, r_needed)
    ok = [s for s in coarse_sizes(n) if s > floor]
    if not ok:
        raise LevelError(
            f"no coarse level reachable from n={n} satisfies "
            f"n_H > max(rank_guess, r_needed) = {floor}")
    best = min(ok)
    if best > (m + 1) / 2:
        warnings.warn(
            f"coarse size {best} violates n_H <= (m+1)/2 = {(m + 1) / 2}; "
            "the rank bound cannot be certified for this problem",
            RuntimeWarning, stacklevel=2)
    return best


def restrict(x, chain):
    """multilevel.py:212-219."""
    return as_matrix(x) @ chain.composite


def prolong(x_h, chain):
    """multilevel.py:238-245."""
    return as_matrix(x_h) @ chain.composite.T


def restrict_least_squares(x, chain):
    """multilevel.py:222-235."""
    return scipy.linalg.cho_solve(chain.gram_cho(), (as_matrix(x) @ chain.composite).T).T


# --------------------------------------------------------------------------
# pcp.py — multilevel inexact ALM
# --------------------------------------------------------------------------


@dataclass
class Record:
    """pcp.py:57-66 (IterationRecord)."""

    iter: int
    feasibility_gap: float
    objective: float
    rank_l: int
    sparsity_s: float
    wall_seconds: float


@dataclass
class PcpResult:
    """pcp.py:69-81 (PcpState) minus diagnostics."""

    l: np.ndarray
    s: np.ndarray
    y: np.ndarray
    mu: float
    iter: int
    history: list
    mu_history: list
    converged: bool
    n_coarse: int = 0
    sigma1: float = 0.0
    diagnostics: tuple = None   # (epsilon, delta_history) with collect_diagnostics


def epsilon_bound(l_h, chain):
    """multilevel.py:248-265: sum_k sigma_k(L_H) (1 - sigma_{n_H-k+1}(R)), k <= rank(L_H)."""
    s_l = svd_full(as_matrix(l_h))[1]
    r_h = int(np.count_nonzero(s_l > s_l[0] * max(l_h.shape) * np.finfo(float).eps))
    if r_h == 0:
        return 0.0
    s_r = chain.composite_sigmas()
    return float(np.sum(s_l[:r_h] * (1.0 - s_r[::-1][:r_h])))


def _coarse_width(n, m, levels, rank_guess):
    """pcp.py:200-210 / cpcp.py:492-500."""
    if levels is not None:
        if levels < 1:
            raise LevelError(
                f"coarse size {levels} is invalid: the rank bound "
                f"requires rank(L) <= n_H <= (m+1)/2 with n_H >= 1")
        return int(levels)
    return select_levels(n, rank_guess, 1, m)


def ml_ialm(d, lam=None, mu0=None, rho=1.5, tol=1e-7, max_iters=500,
            rank_guess=5, levels=None, time_budget=None, collect_diagnostics=False):
    """pcp.py:213-309 (ml_ialm_solve) with pcp.py:95-115 inlined.

    Returns PcpResult.  Option validation follows pcp.py:42-54.
    """
    d = as_matrix(d, "d")
    m, n = d.shape
    if np.linalg.norm(d, "fro") == 0.0:          # pcp.py:229-230, 105-109
        z = np.zeros_like(d)
        return PcpResult(z, z.copy(), z.copy(), 0.0, 1,
                         [Record(1, 0.0, 0.0, 0, 0.0, 0.0)], [], True)
    if lam is not None and lam <= 0:
        raise ValueError("lam must be positive")
    if mu0 is not None and mu0 <= 0:
        raise ValueError("mu0 must be positive")
    if rho <= 1:
        raise ValueError("rho must exceed 1")
    if tol <= 0:
        raise ValueError("tol_feasibility must be positive")
    if max_iters < 1:
        raise ValueError("max_iters must be positive")
    if rank_guess < 1:
        raise ValueError("rank_guess must be positive")
    lam = lam if lam is not None else 1.0 / np.sqrt(max(m, n))     # pcp.py:99
    sigma1 = np.linalg.norm(d, 2)                                  # pcp.py:100
    mu = mu0 if mu0 is not None else 1.25 / sigma1                 # pcp.py:101
    chain = build_chain(n, _coarse_width(n, m, levels, rank_guess), True)
    rd = chain.composite.toarray()                                 # pcp.py:236
    cho = chain.gram_cho()
    d_norm = np.linalg.norm(d, "fro")                              # pcp.py:238
    s_mat = np.zeros_like(d)
    y = d / max(np.linalg.norm(d, 2), np.max(np.abs(d)) / lam)     # pcp.py:112-115
    buf = np.empty_like(d)
    hist, mus, iterates = [], [], []
    done = False
    t0 = time.perf_counter()
    k = 0
    l_mat = np.zeros_like(d)
    l_h = np.zeros((m, chain.n_coarse))
    for k in range(1, max_iters + 1):                              # pcp.py:248
        mus.append(mu)
        inv = 1.0 / mu
        np.multiply(y, inv, out=buf)                               # pcp.py:252-255
        buf += d
        buf -= s_mat
        m_h = scipy.linalg.cho_solve(cho, (buf @ rd).T).T
        u_h, sig, v_h = svd_full(m_h)                              # pcp.py:257
        rank = int(np.count_nonzero(sig > inv))                    # pcp.py:258
        if rank == 0:
            l_h = np.zeros((m, chain.n_coarse))
            l_mat = np.zeros_like(d)
            nuc = 0.0
        else:
            kept = sig[:rank] - inv
            l_h = (u_h[:, :rank] * kept) @ v_h[:, :rank].T
            l_mat = l_h @ rd.T
            nuc = float(np.sum(kept))
        if collect_diagnostics:                                    # pcp.py:268-269
            iterates.append(l_h)
        np.multiply(y, inv, out=buf)                               # pcp.py:272-275
        buf += d
        buf -= l_mat
        s_mat = soft_threshold(buf, lam * inv)
        np.subtract(d, l_mat, out=buf)                             # pcp.py:277-282
        buf -= s_mat
        gap = float(np.linalg.norm(buf, "fro") / d_norm)
        buf *= mu
        y += buf
        mu *= rho
        hist.append(Record(k, gap, nuc + lam * float(np.sum(np.abs(s_mat))), rank,
                           float(np.count_nonzero(s_mat)) / (m * n),
                           time.perf_counter() - t0))
        if gap <= tol:
            done = True
            break
        if time_budget is not None and hist[-1].wall_seconds >= time_budget:
            break
    diag = None
    if collect_diagnostics:                                        # pcp.py:298-306
        ref = restrict(l_mat, chain)
        drift = (chain.composite.T @ chain.composite).toarray() - np.eye(chain.n_coarse)
        deltas = [float(np.sum((lh @ drift) * (lh - ref))) for lh in iterates]
        diag = (epsilon_bound(l_h, chain) if np.any(l_h) else 0.0, deltas)
    return PcpResult(l_mat, s_mat, y, mu, k, hist, mus, done,
                     chain.n_coarse, float(sigma1), diag)


def lanczos_sigma1(d, steps=80, seed=0):
    """sigma_1(d) by Lanczos on d^T d with full reorthogonalisation (numpy).
    Bench setup only: the reference takes sigma_1 from a full SVD
    (pcp.py:100, 114; ~260 s each at 20000^2), which a bounded CPU sample of
    the loop leaves out."""
    m, n = d.shape
    q = np.random.default_rng(seed).standard_normal(n)
    qs = [q / np.linalg.norm(q)]
    alpha, beta = [], []
    theta = 0.0
    for k in range(min(steps, n)):
        w = d.T @ (d @ qs[-1])
        a = float(qs[-1] @ w)
        alpha.append(a)
        for v in qs:                      # full reorthogonalisation
            w -= (v @ w) * v
        b = float(np.linalg.norm(w))
        t = np.diag(alpha) + np.diag(beta, 1) + np.diag(beta, -1)
        theta_new = float(np.linalg.eigvalsh(t)[-1])
        if k > 3 and abs(theta_new - theta) <= 1e-15 * theta_new or b == 0.0:
            theta = theta_new
            break
        theta = theta_new
        beta.append(b)
        qs.append(w / b)
    return float(np.sqrt(theta))


def ml_ialm_steps(d, sigma1, lam=None, rho=1.5, levels=None, rank_guess=5):
    """Generator form of the ml_ialm loop (pcp.py:248-296, same operations as
    ml_ialm above) for bounded CPU samples in bench.py: yields (k, gap, rank)
    after every iteration and keeps iterating past the tolerance (an
    iteration's work does not depend on it).  sigma1 is supplied by the
    caller (see lanczos_sigma1)."""
    d = as_matrix(d, "d")
    m, n = d.shape
    lam = lam if lam is not None else 1.0 / np.sqrt(max(m, n))     # pcp.py:99
    mu = 1.25 / sigma1                                             # pcp.py:101
    chain = build_chain(n, _coarse_width(n, m, levels, rank_guess), True)
    rd = chain.composite.toarray()                                 # pcp.py:236
    cho = chain.gram_cho()
    d_norm = np.linalg.norm(d, "fro")                              # pcp.py:238
    s_mat = np.zeros_like(d)
    y = d / max(sigma1, np.max(np.abs(d)) / lam)                   # pcp.py:112-115
    buf = np.empty_like(d)
    k = 0
    while True:
        k += 1
        inv = 1.0 / mu
        np.multiply(y, inv, out=buf)                               # pcp.py:252-255
        buf += d
        buf -= s_mat
        m_h = scipy.linalg.cho_solve(cho, (buf @ rd).T).T
        u_h, sig, v_h = svd_full(m_h)                              # pcp.py:257
        rank = int(np.count_nonzero(sig > inv))                    # pcp.py:258
        if rank == 0:
            l_mat = np.zeros_like(d)
        else:
            kept = sig[:rank] - inv
            l_mat = ((u_h[:, :rank] * kept) @ v_h[:, :rank].T) @ rd.T
        np.multiply(y, inv, out=buf)                               # pcp.py:272-275
        buf += d
        buf -= l_mat
        s_mat = soft_threshold(buf, lam * inv)
        np.subtract(d, l_mat, out=buf)                             # pcp.py:277-282
        buf -= s_mat
        gap = float(np.linalg.norm(buf, "fro") / d_norm)
        buf *= mu
        y += buf
        mu *= rho
        _ = float(np.sum(np.abs(s_mat))), np.count_nonzero(s_mat)  # pcp.py:284-291 telemetry
        yield k, gap, rank


DENSE_SVD_LIMIT = 256   # linalg.py:16


def svd_truncated(x, r):
    """linalg.py:102-125: leading r triplets; dense LAPACK when
    min(m, n) <= 256 or r >= min(m, n), else ARPACK (svds, v0 = ones)."""
    x = as_matrix(x)
    k = min(x.shape)
    r = int(r)
    if not 1 <= r <= k:
        raise ValueError(f"rank must satisfy 1 <= r <= {k}, got {r}")
    if k <= DENSE_SVD_LIMIT or r >= k:
        u, s, v = svd_full(x)
        return u[:, :r], s[:r], v[:, :r]
    u, s, vt = scipy.sparse.linalg.svds(x, k=r, v0=np.ones(min(x.shape)))
    order = np.argsort(s)[::-1]
    u, v = u[:, order], vt[order].T
    if u.shape[1]:
        peak = np.argmax(np.abs(u), axis=0)
        sgn = np.sign(u[peak, np.arange(u.shape[1])])
        sgn[sgn == 0] = 1.0
        u, v = u * sgn, v * sgn
    return u, s[order], v


def ialm(d, lam=None, mu0=None, rho=1.5, tol=1e-7, max_iters=500, rank_guess=5,
         svd_budget=None, time_budget=None):
    """pcp.py:118-197 (ialm_solve): inexact ALM with the adaptive truncated SVD."""
    d = as_matrix(d, "d")
    m, n = d.shape
    if np.linalg.norm(d, "fro") == 0.0:
        z = np.zeros_like(d)
        return PcpResult(z, z.copy(), z.copy(), 0.0, 1, [Record(1, 0.0, 0.0, 0, 0.0, 0.0)], [], True)
    lam = lam if lam is not None else 1.0 / np.sqrt(max(m, n))     # pcp.py:99
    sigma1 = np.linalg.norm(d, 2)                                  # pcp.py:100
    mu = mu0 if mu0 is not None else 1.25 / sigma1                 # pcp.py:101
    kmax = min(m, n)
    cap = min(svd_budget or kmax, kmax)                            # pcp.py:132-133
    d_norm = np.linalg.norm(d, "fro")
    s_mat = np.zeros_like(d)
    y = d / max(np.linalg.norm(d, 2), np.max(np.abs(d)) / lam)     # pcp.py:112-115
    sv = min(rank_guess + 1, cap)                                  # pcp.py:138
    work = np.empty_like(d)
    hist, mus = [], []
    done = False
    t0 = time.perf_counter()
    k = 0
    l_mat = np.zeros_like(d)
    for k in range(1, max_iters + 1):                              # pcp.py:145
        mus.append(mu)
        inv = 1.0 / mu
        np.multiply(y, inv, out=work)
        work += d
        work -= s_mat
        u, sig, v = svd_truncated(work, sv)                        # pcp.py:153
        rank = int(np.count_nonzero(sig > inv))
        if rank == 0:
            l_mat = np.zeros_like(d)
            nuc = 0.0
        else:
            shrunk = sig[:rank] - inv
            l_mat = (u[:, :rank] * shrunk) @ v[:, :rank].T
            nuc = float(np.sum(shrunk))
        if sig[-1] > inv:                                          # pcp.py:160-165
            sv = min(sv + 5, cap)
        else:
            sv = max(min(rank + 1, cap), 1)
        np.multiply(y, inv, out=work)
        work += d
        work -= l_mat
        s_mat = soft_threshold(work, lam * inv)
        np.subtract(d, l_mat, out=work)
        work -= s_mat
        gap = float(np.linalg.norm(work, "fro") / d_norm)
        work *= mu
        y += work
        mu *= rho
        hist.append(Record(k, gap, nuc + lam * float(np.sum(np.abs(s_mat))), rank,
                           float(np.count_nonzero(s_mat)) / (m * n), time.perf_counter() - t0))
        if gap <= tol:
            done = True
            break
        if time_budget is not None and hist[-1].wall_seconds >= time_budget:
            break
    return PcpResult(l_mat, s_mat, y, mu, k, hist, mus, done, n, float(sigma1))


# --------------------------------------------------------------------------
# cpcp.py — multilevel Frank-Wolfe thresholding
# --------------------------------------------------------------------------


def l1_argmax(g):
    """cpcp.py:155-161 — column-major first-occurrence tie break."""
    a = np.abs(g)
    rows = np.argmax(a, axis=0)
    j = int(np.argmax(a[rows, np.arange(g.shape[1])]))
    return int(rows[j]), j


def _coord_min(quad, lin):
    """cpcp.py:195-199."""
    if quad <= 0.0:
        return 1.0 if lin < 0.0 else 0.0
    return float(min(max(-lin / quad, 0.0), 1.0))


def box_qp(aa, bb, ab, la, lb, fallback=None):
    """cpcp.py:202-231 — exact 2-variable QP over the unit box."""
    def q(x, y):
        return 0.5 * (aa * x * x + 2 * ab * x * y + bb * y * y) + la * x + lb * y

    det = aa * bb - ab * ab
    best = None
    if det > 0.0:
        x = (-la * bb + lb * ab) / det
        y = (-lb * aa + la * ab) / det
        if 0.0 <= x <= 1.0 and 0.0 <= y <= 1.0:
            best = (x, y)
    if best is None:
        x = y = 0.0
        for _ in range(200):
            xn = _coord_min(aa, la + ab * y)
            yn = _coord_min(bb, lb + ab * xn)
            stop = abs(xn - x) <= 1e-12 and abs(yn - y) <= 1e-12
            x, y = xn, yn
            if stop:
                break
        best = (x, y)
    if fallback is not None:
        gf = float(min(max(fallback, 0.0), 1.0))
        if q(gf, gf) < q(*best):
            best = (gf, gf)
    return best


class LeadingTriple:
    """cpcp.py:288-323 — warm-started power iteration for sigma_1."""

    def __init__(self, cols, rtol=1e-6, max_passes=40):
        self.v = np.ones(cols) / np.sqrt(cols)
        self.rtol = rtol
        self.max_passes = max_passes
        self.passes = []

    def __call__(self, g):
        v = self.v
        prev = -1.0
        u = None
        nw = 0.0
        p = 0
        for p in range(1, self.max_passes + 1):
            gu = g @ v
            s2 = float(gu.dot(gu))
            if s2 == 0.0:
                self.passes.append(p)
                return None, 0.0, None
            u = gu / np.sqrt(s2)
            w = g.T @ u
            nw = float(np.sqrt(w.dot(w)))
            if nw == 0.0:
                self.passes.append(p)
                return None, 0.0, None
            v = w / nw
            if abs(s2 - prev) <= self.rtol * s2:
                break
            prev = s2
        self.passes.append(p)
        self.v = v
        return u, nw, v


@dataclass
class CpcpResult:
    """cpcp.py:94-112 (CpcpState)."""

    l: np.ndarray
    s: np.ndarray
    t_l: float
    t_s: float
    u_l: float
    u_s: float
    iter: int
    history: list
    objective_history: list
    converged: bool
    n_coarse: int = 0
    power_passes: list | None = None
    oracle_atoms: list | None = None


def _converged(objs, tol, window=5):
    """cpcp.py:280-285."""
    if len(objs) <= window:
        return False
    prev = objs[-1 - window]
    return prev - objs[-1] <= tol * max(abs(prev), np.finfo(float).tiny)


def ml_fwt(d, observed, lambda_l, lambda_s, tol=1e-3, max_iters=2000,
           rank_guess=5, levels=None, time_budget=None, collect_rank=True, track_oracle_atoms=False):
    """cpcp.py:480-515 (ml_fwt_solve) driving cpcp.py:326-456 (_run_fwt).

    ``observed`` is a boolean m x n array or None (fully observed).
    """
    d = as_matrix(d, "d")
    m, n = d.shape
    if lambda_l <= 0 or lambda_s <= 0:
        raise ValueError("penalty weights must be positive")
    if tol <= 0:
        raise ValueError("tol must be positive")
    if max_iters < 1:
        raise ValueError("max_iters must be positive")
    nh = _coarse_width(n, m, levels, rank_guess)
    chain = build_chain(n, nh, True)                              # cpcp.py:501
    radius = 1.0 / float(chain.composite_sigmas()[0])             # cpcp.py:502
    rd = chain.composite.toarray()
    triple = LeadingTriple(chain.n_coarse)

    def lmo(g):                                                   # cpcp.py:506-513
        g_h = g @ rd
        u, sig, v = triple(g_h)
        if u is None:
            return np.zeros_like(g), 0.0
        return ((-radius) * np.outer(u, v)) @ rd.T, -radius * sig

    if observed is not None:
        observed = np.asarray(observed).astype(bool)
        if observed.shape != d.shape:
            raise ValueError("mask shape does not match data")
    mf = observed.astype(np.float64) if observed is not None else None

    def proj(x):                                                  # cpcp.py:47-61
        return np.where(observed, x, 0.0) if observed is not None else x.copy()

    pd = proj(d)                                                  # cpcp.py:121-131
    sq0 = float(np.sum(pd * pd))
    u_l, u_s = sq0 / (2.0 * lambda_l), sq0 / (2.0 * lambda_s)
    l = np.zeros_like(d)
    s = np.zeros_like(d)
    t_l = t_s = 0.0
    hist, objs = [], []
    t0 = time.perf_counter()
    if u_l == 0.0:                                                # cpcp.py:348-350
        hist.append(Record(1, 0.0, 0.0, 0, 0.0, 0.0))
        return CpcpResult(l, s, 0.0, 0.0, 0.0, 0.0, 1, hist, [0.0], True, nh, [])
    r = proj(d)                                                   # cpcp.py:352-354
    pd_norm = float(np.sqrt(r.ravel().dot(r.ravel())))
    np.negative(r, out=r)
    done = False
    k = 0
    atoms = [] if track_oracle_atoms else None                   # cpcp.py:355
    for k in range(1, max_iters + 1):                             # cpcp.py:357
        m_l, val_l = lmo(r)
        if atoms is not None:                                     # cpcp.py:359-360
            atoms.append(m_l.copy())
        i_s, j_s = l1_argmax(r)
        val_s = -abs(float(r[i_s, j_s]))
        cl = lambda_l < -val_l                                    # cpcp.py:365-368
        cs = lambda_s < -val_s
        v_tl = u_l if cl else 0.0
        v_ts = u_s if cs else 0.0
        if cl:                                                    # cpcp.py:371-385
            a = u_l * m_l
            a -= l
        else:
            a = -l
        if mf is not None:
            a *= mf
            b = s * mf
            np.negative(b, out=b)
        else:
            b = -s
        spike = -u_s * np.sign(r[i_s, j_s]) if cs else 0.0
        if cs:
            b[i_s, j_s] += spike
        rr = r.ravel()
        ga, gb = box_qp(float(a.ravel().dot(a.ravel())),          # cpcp.py:387-395
                        float(b.ravel().dot(b.ravel())),
                        float(a.ravel().dot(b.ravel())),
                        float(a.ravel().dot(rr)) + lambda_l * (v_tl - t_l),
                        float(b.ravel().dot(rr)) + lambda_s * (v_ts - t_s),
                        2.0 / (k + 2.0))
        l *= 1.0 - ga                                             # cpcp.py:399-411
        if cl:
            m_l *= ga * u_l
            l += m_l
        s *= 1.0 - gb
        if cs:
            s[i_s, j_s] += gb * spike
        t_l += ga * (v_tl - t_l)
        t_s += gb * (v_ts - t_s)
        a *= ga
        r += a
        b *= gb
        r += b
        w = s - r                                                 # cpcp.py:414-421
        s_new = soft_threshold(w, lambda_s)
        ds = s_new - s
        if mf is not None:
            ds *= mf
        r += ds
        s = s_new
        t_s = float(np.abs(s).sum())
        if k % 64 == 0:                                           # cpcp.py:423-427
            r = l + s
            r -= d
            if mf is not None:
                r *= mf
        sq = float(r.ravel().dot(r.ravel()))                      # cpcp.py:429-432
        obj = 0.5 * sq + lambda_l * t_l + lambda_s * t_s
        u_l, u_s = min(u_l, obj / lambda_l), min(u_s, obj / lambda_s)
        objs.append(obj)
        if collect_rank:                                          # cpcp.py:434-439
            sv = np.linalg.svd(l, compute_uv=False)
            rank = int(np.count_nonzero(sv > sv[0] * max(m, n) * np.finfo(float).eps)) \
                if sv[0] > 0 else 0
        else:
            rank = -1
        hist.append(Record(k, float(np.sqrt(sq)) / pd_norm, obj, rank,
                           float(np.count_nonzero(s)) / (m * n),
                           time.perf_counter() - t0))
        if _converged(objs, tol):
            done = True
            break
        if time_budget is not None and hist[-1].wall_seconds >= time_budget:
            break
    return CpcpResult(l, s, t_l, t_s, u_l, u_s, k, hist, objs, done, nh,
                      triple.passes, atoms)


# --------------------------------------------------------------------------
# BASELINE.json configs: the seeded synthetic generators
# live in one place, paper_2206_13369_b200/datasets.py (input data, not
# reference arithmetic); re-exported here so tests and fixtures scripts can
# take inputs and the checker from one module.
# --------------------------------------------------------------------------
from paper_2206_13369_b200.datasets import CONFIGS, gaussian_rpca, make_config, video_rpca  # noqa: E402,F401
