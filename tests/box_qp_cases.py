"""Box-QP cases shared by the oracle pin (CPU) and the device test (GPU):
every branch of _solve_box_qp (cpcp.py:202-231) -- interior stationary
point, det <= 0, a stationary point outside the box, coordinate descent
with quad <= 0, the fallback step winning and losing, no fallback."""
import numpy as np


def cases(seed=5, n_random=400):
    rows = [
        (2.0, 3.0, 0.5, -1.0, -1.0, 0.5),      # interior
        (1.0, 1.0, 1.0, -0.5, -0.5, 0.5),      # det = 0
        (1.0, 1.0, 2.0, -1.0, 0.3, 0.25),      # det < 0
        (2.0, 3.0, 0.5, -10.0, 2.0, 0.1),      # stationary point outside the box
        (0.0, 0.0, 0.0, -1.0, 1.0, 0.4),       # quad <= 0 both
        (-1.0, 2.0, 0.0, 0.5, -0.5, 0.7),      # negative curvature in ga
        (1e-300, 1e-300, 0.0, -1e-300, 1e-300, 0.5),
        (4.0, 1.0, 1.9, -3.0, -1.0, 1.0),      # fallback clipped to 1
        (4.0, 1.0, 1.9, -3.0, -1.0, -0.5),     # fallback clipped to 0
        (5.0, 5.0, 0.1, -0.2, -0.3, float("nan")),  # no fallback
    ]
    rng = np.random.default_rng(seed)
    for _ in range(n_random):
        a = rng.standard_normal(2) * 10 ** rng.uniform(-3, 3, 2)
        aa, bb = abs(a[0]), abs(a[1])
        ab = rng.standard_normal() * np.sqrt(aa * bb) * rng.uniform(0, 1.5)
        la, lb = rng.standard_normal(2) * 10 ** rng.uniform(-3, 3, 2)
        fb = rng.uniform(-0.2, 1.2) if rng.random() < 0.8 else float("nan")
        rows.append((aa, bb, ab, la, lb, fb))
    return np.array(rows, dtype=np.float64)
