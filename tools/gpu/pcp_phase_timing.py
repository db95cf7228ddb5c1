"""Per-phase CUDA-event timing of full ML-PCP solves: total ms per solve and
launch count for every phase (second solve, after a warm-up)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import pcp as P
from paper_2206_13369_b200.datasets import make_config, CONFIGS

for name in sys.argv[1:] or ['C1', 'C2']:
    d, _ = make_config(name)
    c = CONFIGS[name]
    m, n = d.shape
    D = torch.from_numpy(d).cuda()
    opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'])
    pkg.ml_ialm_solve(D, opts)
    sink = []
    P.TIMING_SINK = sink
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    st = pkg.ml_ialm_solve(D, opts)
    stop.record()
    torch.cuda.synchronize()
    P.TIMING_SINK = None
    t = sink[0]
    phases = {k: (round(v[0], 3), v[1]) for k, v in t.items() if isinstance(v, tuple)}
    print(name, 'iters', st.iter, 'solve ms %.2f' % start.elapsed_time(stop), 'lanczos steps', t['lanczos_steps'],
          'phase ms (total, launches):', phases, flush=True)
