"""Small solves covering every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): ML-PCP FP64 (cluster Jacobi, rank-0
certificate) and FP32 (fast rows, tcgen05 reconstruction), ML-CPCP with a
mask, the cooperative-grid Jacobi (n_p = 640), the long-row Lanczos kernel,
the frame-stack layout kernels.  Checks results loosely (sanitizer runs are
about memory/race errors)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2206_13369_b200 as pkg  # noqa: E402
from oracle import mlrpca_oracle as O  # noqa: E402

which = sys.argv[1:] or ["pcp64", "pcp32", "cpcp", "coop", "lzlong", "frames"]
if "pcp64" in which:
    d, _ = O.gaussian_rpca(120, 96, 6, 0.1, 3)
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=24, max_iters=12))
    print("pcp64", st.iter, flush=True)
if "pcp32" in which:
    d, _ = O.gaussian_rpca(300, 256, 8, 0.1, 4)
    st = pkg.ml_ialm_solve(d.astype(np.float32), pkg.PcpOptions(levels=64, max_iters=10, tol_feasibility=1e-6))
    print("pcp32", st.iter, flush=True)
if "cpcp" in which:
    d, mask = O.gaussian_rpca(100, 80, 4, 0.1, 5, observe=0.8)
    lam = 1 / np.sqrt(100)
    st = pkg.ml_fwt_solve(d.astype(np.float32), pkg.ObservationMask(mask), pkg.CpcpOptions(
        lambda_l=lam, lambda_s=lam / 10, max_iters=15, levels=20, collect_rank=False))
    print("cpcp", st.iter, flush=True)
if "coop" in which:
    rng = np.random.default_rng(1)
    a = rng.standard_normal((660, 640))
    lam, v, sw = pkg.eigh_psd(a.T @ a, max_sweeps=3)
    print("coop sweeps", sw, flush=True)
if "lzlong" in which:
    d, _ = O.gaussian_rpca(40, 4100, 3, 0.1, 6)
    st = pkg.ml_ialm_solve(d.astype(np.float32), pkg.PcpOptions(max_iters=2))
    print("lzlong", st.iter, flush=True)
if "frames" in which:
    raster = np.random.default_rng(2).integers(0, 256, (5, 24, 32), dtype=np.uint8)
    x = pkg.frames.frames_to_matrix(raster)
    back = pkg.frames.matrix_to_frames(x, 24, 32)
    print("frames", bool(np.array_equal(np.asarray(back), raster)), flush=True)
