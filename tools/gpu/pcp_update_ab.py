"""Repeatable timing of the ML-PCP fused row pass (update phase) on one
config, three repeats, for A/B builds (MLR_LIB_PATH)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import pcp as P
from paper_2206_13369_b200.datasets import make_config, CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
d, _ = make_config(name); c = CONFIGS[name]; m, n = d.shape
D = torch.from_numpy(d).cuda()
opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'],
                      max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 500)
pkg.ml_ialm_solve(D, opts)
res = []
for rep in range(3):
    sink = []; P.TIMING_SINK = sink
    st = pkg.ml_ialm_solve(D, opts)
    P.TIMING_SINK = None
    s = sink[0]
    res.append(round(s['update'][0] / s['iters'], 4))
print(name, 'iters', st.iter, 'update ms/iter', res, flush=True)
