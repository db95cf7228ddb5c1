"""Jacobi stopping tolerance vs sweeps / time / parity on a BASELINE config
(default C5): solves with jacobi_tol in argv (FP32 default 1e-6) and compares
each against the reference fixture (tests/golden/c5_pcp.npz: sketches, fixed
rows, rank column) when present, else against the first tolerance's solve."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2206_13369_b200 as pkg  # noqa: E402
from paper_2206_13369_b200 import pcp as P  # noqa: E402
from paper_2206_13369_b200.datasets import CONFIGS, make_config  # noqa: E402

name = os.environ.get("CFG", "C5")
tols = [float(x) for x in sys.argv[1:]] or [1e-6, 1e-5]
c = CONFIGS[name]
d, _ = make_config(name)
m, n = d.shape
D = torch.from_numpy(d).cuda()
del d
fx = os.path.join(os.path.dirname(__file__), "..", "..", "tests", "golden", f"{name.lower()}_pcp.npz")
g = np.load(fx) if os.path.exists(fx) else None
rng = np.random.default_rng(77)
q = torch.from_numpy(rng.standard_normal(n)).cuda()
p = torch.from_numpy(rng.standard_normal(m)).cuda()


def relf(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-300))


base = None
for jt in tols:
    opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c["tol"], levels=c["n_coarse"], jacobi_tol=jt)
    pkg.ml_ialm_solve(D, opts)
    sink = []
    P.TIMING_SINK = sink
    torch.cuda.synchronize()
    t = time.time()
    st = pkg.ml_ialm_solve(D, opts)
    torch.cuda.synchronize()
    dt = time.time() - t
    P.TIMING_SINK = None
    L64, S64 = st.l.double(), st.s.double()
    sk = {"l_q": (L64 @ q).cpu().numpy(), "l_p": (p @ L64).cpu().numpy(), "s_q": (S64 @ q).cpu().numpy(),
          "s_p": (p @ S64).cpu().numpy()}
    ranks = [h.rank_l for h in st.history]
    if g is not None:
        ref = {k: g[k] for k in sk}
        ref_ranks = [int(x) for x in g["h_rank"]]
        ref_iter = int(g["iter"])
    else:
        if base is None:
            base = (sk, ranks, st.iter)
        ref, ref_ranks, ref_iter = base
    errs = {k: relf(sk[k], ref[k]) for k in sk}
    s = sink[0]
    print(f"{name} jtol {jt:.0e}: iters {st.iter}/{ref_iter} ranks_equal {ranks == ref_ranks} "
          f"relF sketches {max(errs.values()):.2e} solve {dt * 1e3:.1f} ms jacobi {s['jacobi'][0]:.1f} ms "
          f"sweeps {sum(s['jac_sweeps'])} {list(s['jac_sweeps'])}", flush=True)
    del L64, S64, st
