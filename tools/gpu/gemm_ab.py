"""Per-phase timings that are GEMM-bound (gram, recon, pre, post) on C2 and C5
(first iterations), for A/B builds via MLR_LIB_PATH."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import pcp as P
from paper_2206_13369_b200.datasets import make_config, CONFIGS
for name, its in (('C2', 500), ('C5', 3)):
    d, _ = make_config(name); c = CONFIGS[name]; m, n = d.shape
    D = torch.from_numpy(d).cuda()
    opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'], max_iters=its)
    pkg.ml_ialm_solve(D, opts)
    sink = []; P.TIMING_SINK = sink
    st = pkg.ml_ialm_solve(D, opts)
    P.TIMING_SINK = None
    s = sink[0]
    print(name, 'iters', st.iter, {k: round(s[k][0] / s['iters'], 4) for k in ('gram', 'pre', 'post', 'recon', 'jacobi')}, flush=True)
    del D
