"""Full-width fwt_solve on C3-shaped data: per-phase ms/iteration (matvec LMO
vs the n x n Gram path with MLR_CPCP_FINE=0)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import cpcp as CP
from paper_2206_13369_b200.datasets import make_config, CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else 'C3'
its = int(sys.argv[2]) if len(sys.argv) > 2 else 100
d, mask = make_config(name)
m, n = d.shape
D = torch.from_numpy(d).cuda()
om = pkg.ObservationMask(mask)
lam = 1 / np.sqrt(max(m, n))
opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=CONFIGS[name]['tol'], max_iters=its,
                       collect_rank=False, check_every=8)
pkg.fwt_solve(D, om, pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=1e-6, max_iters=5,
                                     collect_rank=False))
sink = []
CP.TIMING_SINK = sink
torch.cuda.synchronize()
t = time.time()
st = pkg.fwt_solve(D, om, opts)
torch.cuda.synchronize()
dt = time.time() - t
CP.TIMING_SINK = None
s = sink[0]
it = s['iters']
print(name, 'full-width iters', st.iter, 'solve %.3fs' % dt, 'ms/iter %.3f' % (1e3 * dt / st.iter),
      {k: round(v[0] / it, 4) for k, v in s.items() if isinstance(v, tuple)}, 'obj', st.objective_history[-1], flush=True)
