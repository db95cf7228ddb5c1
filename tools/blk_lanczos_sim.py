"""Block-Lanczos pass counts for sigma_1 (numpy, full reorthogonalisation):
how many passes over D a block of b vectors needs at the 1e-9 tolerance of
the GPU Lanczos.  Usage: python tools/blk_lanczos_sim.py C2"""
import sys, numpy as np, scipy.linalg
sys.path.insert(0, '/root/repo')
from paper_2206_13369_b200.datasets import make_config
name = sys.argv[1]
d, _ = make_config(name); d = d.astype(np.float64)
m, n = d.shape
s_true = np.linalg.norm(d, 2) if name in ('C1','C2') else None
A = lambda X: d.T @ (d @ X)
def block_lanczos(b, tol=1e-9, maxp=200, seed=0):
    rng = np.random.default_rng(seed)
    Q = np.linalg.qr(rng.standard_normal((n, b)))[0]
    Qs = [Q]; As = []; Bs = []
    Qprev = np.zeros((n, b)); Bprev = np.zeros((b, b))
    th_prev = None; hits = 0
    for p in range(1, maxp + 1):
        W = A(Q) - Qprev @ Bprev.T
        Aj = Q.T @ W
        W = W - Q @ Aj
        # full reorth against all previous blocks (numpy, for the experiment)
        for Qo in Qs:
            W -= Qo @ (Qo.T @ W)
        Qn, Bj = np.linalg.qr(W)
        As.append(Aj); Bs.append(Bj)
        k = len(As)
        T = np.zeros((k * b, k * b))
        for i in range(k):
            T[i*b:(i+1)*b, i*b:(i+1)*b] = As[i]
            if i + 1 < k:
                T[(i+1)*b:(i+2)*b, i*b:(i+1)*b] = Bs[i]
                T[i*b:(i+1)*b, (i+1)*b:(i+2)*b] = Bs[i].T
        th = np.linalg.eigvalsh(T)[-1]
        if th_prev is not None and abs(th - th_prev) <= tol * th:
            hits += 1
            if hits >= 2:
                return p, np.sqrt(th)
        else:
            hits = 0
        th_prev = th
        Qprev, Bprev, Q = Q, Bj, Qn
        Qs.append(Q)
    return maxp, np.sqrt(th)
for b in ([int(x) for x in sys.argv[2:]] or [1, 2, 4, 8, 16]):
    p, s = block_lanczos(b)
    print(name, 'block', b, 'passes', p, 'sigma1', s, 'err', (abs(s - s_true) / s_true) if s_true else None, flush=True)
