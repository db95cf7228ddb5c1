"""Per-iteration rank and Jacobi sweeps of an ML-PCP solve (history columns)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import pcp as P
from paper_2206_13369_b200.datasets import make_config, CONFIGS
for name in sys.argv[1:]:
    d, _ = make_config(name); c = CONFIGS[name]; m, n = d.shape
    D = torch.from_numpy(d).cuda()
    opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'])
    sink = []; P.TIMING_SINK = sink
    st = pkg.ml_ialm_solve(D, opts)
    P.TIMING_SINK = None
    print(name, 'ranks', [h.rank_l for h in st.history], 'sweeps', sink[0].get('jac_sweeps'), flush=True)
