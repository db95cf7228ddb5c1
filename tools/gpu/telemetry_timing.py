"""Cost of the reference's telemetry options on the GPU path:
collect_rank (ML-CPCP, C3 / C4 shapes, first 60 iterations) and
collect_diagnostics (ML-PCP, C2)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2206_13369_b200 as pkg  # noqa: E402
from paper_2206_13369_b200.datasets import CONFIGS, make_config  # noqa: E402


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


for name in ["C3", "C4"]:
    c = CONFIGS[name]
    d, mask = make_config(name)
    D = torch.from_numpy(d).cuda()
    m, n = d.shape
    lam = 1 / np.sqrt(m)
    for rank in (False, True):
        opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(m), tol=c["tol"], max_iters=60,
                               levels=c["n_coarse"], collect_rank=rank)
        st, dt = timed(lambda: pkg.ml_fwt_solve(D, pkg.ObservationMask(mask), opts))
        print(name, "collect_rank", rank, "iters", st.iter, f"{dt / st.iter * 1e3:.3f} ms/iter",
              "ranks", [h.rank_l for h in st.history][::10], flush=True)

c = CONFIGS["C2"]
d, _ = make_config("C2")
D = torch.from_numpy(d).cuda()
for diag in (False, True):
    opts = pkg.PcpOptions(lam=1 / np.sqrt(2000), tol_feasibility=c["tol"], levels=c["n_coarse"],
                          collect_diagnostics=diag)
    st, dt = timed(lambda: pkg.ml_ialm_solve(D, opts))
    extra = (st.diagnostics.epsilon, st.diagnostics.delta_max) if diag else None
    print("C2 collect_diagnostics", diag, "iters", st.iter, f"{dt * 1e3:.1f} ms", extra, flush=True)
