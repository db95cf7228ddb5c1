"""Fixed vs per-iteration cost of the ML-CPCP solves: CUDA-event time of
ml_fwt_solve at several max_iters (D and the mask resident on the device)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import make_config, CONFIGS

for name in sys.argv[1:] or ['C4', 'C3']:
    d, mask = make_config(name); c = CONFIGS[name]; m, n = d.shape
    D = torch.from_numpy(d).cuda(); om = pkg.ObservationMask(mask)
    lam = 1 / np.sqrt(max(m, n))
    res = []
    for its in (10, 10, 100, 200, 300):
        opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=c['tol'], max_iters=its,
                               levels=c['n_coarse'], collect_rank=False)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        st = pkg.ml_fwt_solve(D, om, opts)
        b.record()
        torch.cuda.synchronize()
        res.append((st.iter, a.elapsed_time(b)))
    print(name, [(i, round(t, 2)) for i, t in res], 'per-iteration ms (100 -> 300): %.4f' % ((res[-1][1] - res[2][1]) / (res[-1][0] - res[2][0])), flush=True)
