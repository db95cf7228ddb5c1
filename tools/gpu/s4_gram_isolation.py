"""Is the C5 Gram slower inside the solve than alone?  Times mlr_pcp_gram
(gram128 + slice sum) with CUDA events: 20 launches back to back, and 20
launches each preceded by a fused update pass (the iteration's order)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import pcp as P
from paper_2206_13369_b200.backend import CudaPcp
from paper_2206_13369_b200.chain import build_chain
from paper_2206_13369_b200.datasets import make_config, CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else 'C5'
d, _ = make_config(name); c = CONFIGS[name]; m, n = d.shape
D = torch.from_numpy(d).cuda()
opts = pkg.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c['tol'], levels=c['n_coarse'])
chain = build_chain(n, P._checked_width(n, m, opts))
be = CudaPcp(chain, m, m, True, opts.max_iters, D.device)
be.set_timing(True)  # the library's own phase timer, read at the end
st3 = be.input_stats(D)
be.lanczos_init()
if be.lanczos_run_available():
    be.lanczos_run(D, 1e-9)
else:
    for _ in range(140):  # steps past convergence are no-ops on the device
        be.lanczos_update(be.lanczos_matvec(D), 1e-9)
Y = [be.empty(tuple(D.shape), D.dtype), be.empty(tuple(D.shape), D.dtype)]
be.start(D, Y[0], opts.lam, opts.mu0, opts.rho, opts.tol_feasibility, opts.max_iters, opts.time_budget, P._jacobi_tol(opts, True), 60)
def ev():
    return torch.cuda.Event(enable_timing=True)


e = [ev() for _ in range(4)]
e[0].record(); be.gram(0); e[1].record(); be.svt(); be.update(D, Y[0], Y[1]); e[2].record(); be.gram(1); e[3].record(); be.finalize()
torch.cuda.synchronize()
print(name, 'first gram(0) after start: %.3f ms, first gram(1): %.3f ms' % (e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])))


tot = 0.0
for _ in range(20):
    a, b = ev(), ev()
    a.record(); be.gram(1); b.record(); torch.cuda.synchronize()
    tot += a.elapsed_time(b)
print(name, 'gram alone, back to back: %.3f ms' % (tot / 20))
tot = 0.0
for i in range(20):
    be.update(D, Y[(i + 1) % 2], Y[i % 2])
    a, b = ev(), ev()
    a.record(); be.gram(1); b.record(); torch.cuda.synchronize()
    tot += a.elapsed_time(b)
print(name, 'gram right after an update pass: %.3f ms' % (tot / 20))
# sustained: 150 x (update + gram) queued without host synchronisation
pairs = []
for i in range(150):
    be.update(D, Y[(i + 1) % 2], Y[i % 2])
    a, b = ev(), ev()
    a.record(); be.gram(1); b.record()
    pairs.append((a, b))
torch.cuda.synchronize()
ts = [a.elapsed_time(b) for a, b in pairs]
print(name, 'gram after update, 150 queued pairs: first 10 %.3f ms, last 50 %.3f ms' % (sum(ts[:10]) / 10, sum(ts[-50:]) / 50))
# the solve's own order: svt + update + gram + finalize
pairs = []
for i in range(12):
    be.svt(); be.update(D, Y[(i + 1) % 2], Y[i % 2])
    a, b = ev(), ev()
    a.record(); be.gram(1); b.record(); be.finalize()
    pairs.append((a, b))
torch.cuda.synchronize()
ts = [a.elapsed_time(b) for a, b in pairs]
print(name, 'gram inside 12 queued iterations (svt, update, gram, finalize):', ' '.join('%.3f' % t for t in ts))
t = be.timing()
print(name, 'library phase timer:', {k: (round(v[0], 3), v[1], round(v[0] / max(v[1], 1), 4)) for k, v in t.items() if isinstance(v, tuple)})
be.close()
