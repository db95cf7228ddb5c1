import sys, numpy as np, ctypes, torch
sys.path.insert(0, '/root/repo')
import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import ops
for n in (256, 300, 320, 384, 500):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n + 40, n))
    B = a.T @ a
    ev = np.linalg.eigvalsh(B)[::-1]
    lam, V, sweeps = ops.eigh_psd(B)
    lam = np.sort(np.asarray(lam))[::-1][:n]
    print(n, 'err %.3e' % (np.abs(lam - ev).max() / ev[0]), 'sweeps', sweeps, flush=True)
