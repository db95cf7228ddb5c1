import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200.datasets import make_config, CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else 'C1'
d, _ = make_config(name); c = CONFIGS[name]
opts = pkg.PcpOptions(lam=1/np.sqrt(c['m']), tol_feasibility=c['tol'], levels=c['n_coarse'], max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 500)
st = pkg.ml_ialm_solve(torch.from_numpy(d).cuda(), opts)
torch.cuda.synchronize()
print('iters', st.iter)
