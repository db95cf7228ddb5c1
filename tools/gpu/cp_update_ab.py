"""Repeatable timing of the ML-CPCP update kernel on C4 (300 iterations,
CUDA-event phase timers), three repeats for A/B comparisons."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import cpcp as CP
from paper_2206_13369_b200.datasets import make_config, CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else 'C4'
d, mask = make_config(name); c = CONFIGS[name]; m, n = d.shape
D = torch.from_numpy(d).cuda(); om = pkg.ObservationMask(mask)
lam = 1 / np.sqrt(max(m, n))
opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=c['tol'], max_iters=300,
                       levels=c['n_coarse'], collect_rank=False)
pkg.ml_fwt_solve(D, om, opts)
res = []
for rep in range(3):
    sink = []; CP.TIMING_SINK = sink
    st = pkg.ml_fwt_solve(D, om, opts)
    CP.TIMING_SINK = None
    s = sink[0]
    res.append({k: round(v[0] / s['iters'], 4) for k, v in s.items() if isinstance(v, tuple)})
print(name, 'iters', st.iter, 'update ms/iter', [r['update'] for r in res], 'dots', [r['dots'] for r in res], flush=True)
