"""cProfile of one ML-PCP solve plus its phase timers: host-side fixed cost."""
import cProfile
import pstats
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
opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'])
for _ in range(2):
    pkg.ml_ialm_solve(D, opts)
torch.cuda.synchronize()
sink = []
P.TIMING_SINK = sink
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); st = pkg.ml_ialm_solve(D, opts); b.record(); torch.cuda.synchronize()
P.TIMING_SINK = None
t = sink[0]
ph = {k: round(v[0], 3) for k, v in t.items() if isinstance(v, tuple)}
print(name, 'solve ms %.2f' % a.elapsed_time(b), 'phase sum %.2f' % sum(ph.values()), ph)
pr = cProfile.Profile()
pr.enable()
pkg.ml_ialm_solve(D, opts)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(14)
