"""Option, record and state types with the reference's names and semantics.

Field-for-field mirrors of ``PcpOptions`` / ``IterationRecord`` /
``PcpState`` (pcp.py:20-81), ``CpcpOptions`` / ``CpcpState`` /
``ObservationMask`` (cpcp.py:23-112) and ``SvdError`` (linalg.py:19-30).
Extra fields are appended with defaults so reference call sites work
unchanged; they only tune the GPU path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class SvdError(RuntimeError):
    """Eigen/SVD iteration failed to converge (linalg.py:19-30)."""

    def __init__(self, message, iterations=None):
        super().__init__(message)
        self.iterations = iterations


PRECISIONS = ("auto", "float64", "float32")


def check_precision(p):
    if p not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}, got {p!r}")


@dataclass
class PcpOptions:
    """pcp.py:20-54.  ``levels`` is the coarse WIDTH n_H (pcp.py:200-210).

    GPU-only extras: ``jacobi_tol`` (relative off-diagonal stopping level of
    the coarse eigensolver; default 64*eps for float64 data, 1e-6 for
    float32), ``check_every`` (iterations between host polls of the
    device-side stopping flag; 1 when ``time_budget`` is set) and
    ``precision``: "auto" (default) computes and returns in the input's
    floating type (float32 stays float32, anything else float64);
    "float64" reproduces the reference exactly in that respect (every input
    is coerced to float64, linalg.py:48-57, and results are float64);
    "float32" computes in FP32 for any input."""

    lam: float | None = None
    mu0: float | None = None
    rho: float = 1.5
    tol_feasibility: float = 1e-7
    max_iters: int = 500
    rank_guess: int = 5
    levels: int | None = None
    svd_budget: int | None = None
    collect_diagnostics: bool = False
    time_budget: float | None = None
    jacobi_tol: float | None = None
    check_every: int | None = None
    precision: str = "auto"

    def validate(self):
        check_precision(self.precision)
        if self.lam is not None and self.lam <= 0:
            raise ValueError("lam must be positive")
        if self.mu0 is not None and self.mu0 <= 0:
            raise ValueError("mu0 must be positive")
        if self.rho <= 1:
            raise ValueError("rho must exceed 1")
        if self.tol_feasibility <= 0:
            raise ValueError("tol_feasibility must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be positive")
        if self.rank_guess < 1:
            raise ValueError("rank_guess must be positive")


@dataclass
class IterationRecord:
    """pcp.py:57-66."""

    iter: int
    feasibility_gap: float
    objective: float
    rank_l: int
    sparsity_s: float
    wall_seconds: float


@dataclass
class MultilevelDiagnostics:
    """multilevel.py:105-122."""

    epsilon: float
    delta_history: list

    @property
    def delta_max(self):
        if not self.delta_history:
            return 0.0
        return float(max(0.0, max(self.delta_history)))


@dataclass
class PcpState:
    """pcp.py:69-81.  Arrays are numpy for host input, torch (on the input's
    device) for CUDA-tensor input."""

    l: object
    s: object
    y: object
    mu: float
    iter: int
    history: list
    mu_history: list
    converged: bool
    diagnostics: MultilevelDiagnostics | None = None


class ObservationMask:
    """cpcp.py:23-53 — entrywise observation pattern."""

    def __init__(self, observed):
        observed = np.asarray(observed)
        if observed.ndim != 2:
            raise ValueError("mask must be 2-D")
        self.observed = observed.astype(bool)
        self.rows, self.cols = self.observed.shape

    @classmethod
    def full(cls, rows, cols):
        return cls(np.ones((rows, cols), dtype=bool))

    @classmethod
    def random(cls, rows, cols, fraction, rng):
        if not 0.0 <= fraction <= 1.0:
            raise ValueError("fraction must lie in [0, 1]")
        count = int(round(fraction * rows * cols))
        flat = np.zeros(rows * cols, dtype=bool)
        flat[rng.choice(rows * cols, size=count, replace=False)] = True
        return cls(flat.reshape(rows, cols))

    def project(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.shape != self.observed.shape:
            raise ValueError(
                f"matrix shape {x.shape} does not match mask {self.observed.shape}")
        return np.where(self.observed, x, 0.0)

    def packed_bits(self, rows=None):
        """Bit-packed rows (uint32 words, bit j&31 of word j>>5) for the GPU."""
        obs = self.observed if rows is None else self.observed[rows]
        by = np.packbits(obs, axis=1, bitorder="little")
        words = (obs.shape[1] + 31) // 32
        pad = words * 4 - by.shape[1]
        if pad:
            by = np.concatenate([by, np.zeros((by.shape[0], pad), dtype=np.uint8)], axis=1)
        return np.ascontiguousarray(by).view("<u4")


@dataclass
class CpcpOptions:
    """cpcp.py:64-91 (no defaults for the penalty weights)."""

    lambda_l: float
    lambda_s: float
    tol: float = 1e-3
    max_iters: int = 2000
    rank_guess: int = 5
    levels: int | None = None
    time_budget: float | None = None
    collect_rank: bool = True
    track_oracle_atoms: bool = False
    check_every: int | None = None
    precision: str = "auto"  # as PcpOptions.precision

    def validate(self):
        check_precision(self.precision)
        if self.lambda_l <= 0 or self.lambda_s <= 0:
            raise ValueError("penalty weights must be positive")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be positive")


@dataclass
class CpcpState:
    """cpcp.py:94-112."""

    l: object
    s: object
    t_l: float
    t_s: float
    u_l: float
    u_s: float
    iter: int
    history: list
    objective_history: list
    converged: bool
    oracle_atoms: list | None = None
