import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import pcp as P
from paper_2206_13369_b200.datasets import make_config, CONFIGS
which = sys.argv[1:] or ['C3', 'C4', 'C5']
for name in which:
    t = time.time(); d, mask = make_config(name); tgen = time.time() - t
    c = CONFIGS[name]; m, n = d.shape
    D = torch.from_numpy(d).cuda()
    torch.cuda.synchronize()
    if c['solver'] == 'pcp':
        opts = pkg.PcpOptions(lam=1/np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'])
        sink = []; P.TIMING_SINK = sink
        t = time.time(); st = pkg.ml_ialm_solve(D, opts); torch.cuda.synchronize(); dt = time.time() - t
        P.TIMING_SINK = None
        s = sink[0]; it = s['iters']
        print(name, 'gen %.1fs' % tgen, 'iters', st.iter, 'conv', st.converged, 'solve %.3fs' % dt, 'gap', st.history[-1].feasibility_gap,
              'rank', st.history[-1].rank_l, 'per-iter ms', {k: round(v[0]/it, 3) for k, v in s.items() if isinstance(v, tuple)}, 'sweeps', s['jac_sweeps'][:5], s['jac_sweeps'][-5:], 'lanczos', s['lanczos_steps'], flush=True)
    else:
        lam = 1/np.sqrt(max(m, n))
        opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam/np.sqrt(max(m, n)), tol=c['tol'], max_iters=5000, levels=c['n_coarse'], collect_rank=False)
        om = pkg.ObservationMask(mask)
        t = time.time(); st = pkg.ml_fwt_solve(D, om, opts); torch.cuda.synchronize(); dt = time.time() - t
        print(name, 'gen %.1fs' % tgen, 'iters', st.iter, 'conv', st.converged, 'solve %.3fs' % dt, 'ms/iter %.3f' % (1e3*dt/st.iter), 'obj', st.objective_history[-1], 'fg', st.history[-1].feasibility_gap, 'sparsity', st.history[-1].sparsity_s, flush=True)
