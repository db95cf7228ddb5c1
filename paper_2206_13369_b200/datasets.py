"""Seeded synthetic inputs for the BASELINE.json configs.

No public dataset is involved: C1/C2/C3/C5 are Gaussian-factor low-rank plus
uniform sparse corruptions, C4 is a synthetic 240x320x1000 "video" stack
with the shapes and distributions BASELINE.json states.  Draw order is
fixed (U, V, support, values, mask) so every process regenerates the same
matrix from the seed.
"""

from __future__ import annotations

import numpy as np


def gaussian_rpca(m, n, rank, eta, seed, observe=None):
    """D = U V^T + S0 with U, V ~ N(0, 1/n); S0 has floor(eta*m*n) entries
    uniform in [-1, 1] on a uniformly random support; optional Bernoulli
    observation mask (D zeroed off-mask)."""
    rng = np.random.default_rng(seed)
    scale = 1.0 / np.sqrt(n)
    u = rng.standard_normal((m, rank)) * scale
    v = rng.standard_normal((n, rank)) * scale
    low = u @ v.T
    cnt = int(np.floor(eta * m * n))
    pos = rng.choice(m * n, size=cnt, replace=False)
    vals = rng.uniform(-1.0, 1.0, size=cnt)
    sparse = np.zeros(m * n)
    sparse[pos] = vals
    d = low + sparse.reshape(m, n)
    mask = None
    if observe is not None:
        mask = rng.random((m, n)) < observe
        d = np.where(mask, d, 0.0)
    return d, mask


def video_rpca(seed, height=240, width=320, frames=1000, rank=5, squares=5, side=20, observe=0.7):
    """C4: rank-5 nonnegative background (U[0,1] factors scaled by 1/max)
    plus five drifting 20x20 U[0,1] squares per frame, pixel (r, c) of frame
    f at matrix entry (r + c*height, f); Bernoulli(observe) mask."""
    rng = np.random.default_rng(seed)
    m = height * width
    u = rng.uniform(0.0, 1.0, size=(m, rank))
    v = rng.uniform(0.0, 1.0, size=(frames, rank))
    bg = u @ v.T
    bg /= bg.max()
    pos = np.stack([rng.uniform(0, height - side, squares), rng.uniform(0, width - side, squares)], axis=1)
    vel = rng.integers(1, 4, size=(squares, 2)) * rng.choice([-1, 1], size=(squares, 2))
    fg = np.zeros((m, frames))
    hi = np.array([height - side, width - side], dtype=np.float64)
    for f in range(frames):
        for q in range(squares):
            r0, c0 = int(pos[q, 0]), int(pos[q, 1])
            idx = (np.arange(r0, r0 + side)[:, None] + np.arange(c0, c0 + side)[None, :] * height).ravel()
            fg[idx, f] += rng.uniform(0.0, 1.0, size=side * side)
        pos += vel
        for ax in range(2):
            low = pos[:, ax] < 0
            high = pos[:, ax] > hi[ax]
            pos[low, ax] = -pos[low, ax]
            pos[high, ax] = 2 * hi[ax] - pos[high, ax]
            vel[low | high, ax] *= -1
    d = bg + fg
    mask = rng.random((m, frames)) < observe
    return np.where(mask, d, 0.0), mask


CONFIGS = {
    "C1": dict(solver="pcp", m=500, n=500, rank=25, eta=0.10, n_coarse=125, tol=1e-7, dtype="float64"),
    "C2": dict(solver="pcp", m=2000, n=2000, rank=100, eta=0.10, n_coarse=250, tol=1e-6, dtype="float32"),
    "C3": dict(solver="cpcp", m=4000, n=4000, rank=200, eta=0.10, observe=0.8, n_coarse=500, tol=1e-6,
               dtype="float32"),
    "C4": dict(solver="cpcp", video=True, m=76800, n=1000, n_coarse=125, tol=1e-6, dtype="float32"),
    "C5": dict(solver="pcp", m=20000, n=20000, rank=200, eta=0.05, n_coarse=1250, tol=1e-5, dtype="float32"),
}


def make_config(name, seed=0):
    """(d, mask) for a BASELINE config; FP32 configs are rounded to float32."""
    c = CONFIGS[name]
    if c.get("video"):
        d, mask = video_rpca(seed)
    else:
        d, mask = gaussian_rpca(c["m"], c["n"], c["rank"], c["eta"], seed, c.get("observe"))
    return d.astype(c["dtype"]), mask
