"""Full-width ialm_solve vs ml_ialm_solve on C1 / C2 (device-resident input):
iterations, wall time per solve, per-phase CUDA-event totals, and the CPU
oracle's full-width IALM iteration count for C1."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2206_13369_b200 as pkg  # noqa: E402
from paper_2206_13369_b200 import pcp as P  # noqa: E402
from paper_2206_13369_b200.datasets import CONFIGS, make_config  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2"]:
    c = CONFIGS[name]
    d, _ = make_config(name)
    D = torch.from_numpy(d).cuda()
    for label, fn, opts in [
        ("ialm", pkg.ialm_solve, pkg.PcpOptions(lam=1 / np.sqrt(c["m"]), tol_feasibility=c["tol"])),
        ("ml_ialm", pkg.ml_ialm_solve, pkg.PcpOptions(lam=1 / np.sqrt(c["m"]), tol_feasibility=c["tol"],
                                                      levels=c["n_coarse"])),
    ]:
        fn(D, opts)
        torch.cuda.synchronize()
        P.TIMING_SINK = []
        t0 = time.perf_counter()
        st = fn(D, opts)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ph = P.TIMING_SINK[-1]
        P.TIMING_SINK = None
        print(name, label, "iters", st.iter, "rank", st.history[-1].rank_l, "conv", st.converged,
              f"{dt * 1e3:.1f} ms", {k: round(v[0], 2) for k, v in ph.items() if isinstance(v, tuple)},
              "sweeps", ph["jac_sweeps"][:6], flush=True)
