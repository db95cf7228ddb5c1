"""One ML-PCP solve per named config (for an ncu launch list of the
tridiagonal eigensolver kernels: ncu -k regex:trd_ ...)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import make_config, CONFIGS

for name in sys.argv[1:] or ['C2']:
    d, _ = make_config(name)
    c = CONFIGS[name]
    m, n = d.shape
    D = torch.from_numpy(d).cuda()
    opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'])
    st = pkg.ml_ialm_solve(D, opts)
    torch.cuda.synchronize()
    print(name, 'iters', st.iter, flush=True)
