"""CPU experiment: Jacobi sweeps per ML-PCP iteration under the current
relative off-diagonal test vs an SVT-aware test (Daleckii-Krein bound of the
error an unresolved pair leaves in L_H = M_H f(B)).

Runs the C2 ML-IALM in FP64 numpy (the oracle's iteration), and at every
iteration warm-starts a cyclic round-robin Jacobi on B~ = V^T B V from the
previous eigenvectors.  Prints sweeps and the L_H / rank / nuclear error of
each criterion.  Not product code.

    python tools/jacobi_criterion_sim.py [C2|small] [tolB]
"""
import sys

import numpy as np
import scipy.linalg

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import mlrpca_oracle as O  # noqa: E402


def rr_pairs(n):
    idx = list(range(n))
    rounds = []
    for _ in range(n - 1):
        rounds.append((np.array(idx[: n // 2]), np.array(idx[n // 2:][::-1])))
        idx = [idx[0]] + [idx[-1]] + idx[1:-1]
    return rounds


def jacobi(Bt, V, rounds, stop):
    """Cyclic Jacobi; stop(B, p, q) -> per-pair measure; sweep converged when
    max measure over the sweep <= 1 (measure is pre-scaled)."""
    B = Bt.copy()
    V = V.copy()
    sweeps = 0
    while sweeps < 60:
        sweeps += 1
        mx = 0.0
        for p, q in rounds:
            a, b, g = B[p, p], B[q, q], B[p, q]
            mx = max(mx, float(np.max(stop(a, b, g))))
            d = b - a
            h = np.sqrt(d * d + 4 * g * g)
            with np.errstate(divide="ignore", invalid="ignore"):
                t = np.where(g != 0, 2 * g / np.where(d >= 0, d + h, d - h), 0.0)
            c = 1 / np.sqrt(1 + t * t)
            s = c * t
            Bp, Bq = B[p, :].copy(), B[q, :].copy()
            B[p, :] = c[:, None] * Bp - s[:, None] * Bq
            B[q, :] = s[:, None] * Bp + c[:, None] * Bq
            Bp, Bq = B[:, p].copy(), B[:, q].copy()
            B[:, p] = Bp * c - Bq * s
            B[:, q] = Bp * s + Bq * c
            Vp, Vq = V[:, p].copy(), V[:, q].copy()
            V[:, p] = Vp * c - Vq * s
            V[:, q] = Vp * s + Vq * c
        if mx <= 1.0:
            break
    return B, V, sweeps


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    tolB = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
    if cfg == "C2":
        d, _ = O.gaussian_rpca(2000, 2000, 100, 0.10, 0)
        d = d.astype(np.float32).astype(np.float64)
        levels, tol = 250, 1e-6
    else:
        d, _ = O.gaussian_rpca(600, 600, 30, 0.10, 0)
        levels, tol = 150, 1e-6
    m, n = d.shape
    lam = 1 / np.sqrt(max(m, n))
    sigma1 = np.linalg.norm(d, 2)
    mu = 1.25 / sigma1
    chain = O.build_chain(n, levels, True)
    rd = chain.composite.toarray()
    cho = chain.gram_cho()
    dn = np.linalg.norm(d)
    s_mat = np.zeros_like(d)
    y = d / max(sigma1, np.max(np.abs(d)) / lam)
    nH = chain.n_coarse
    rounds = rr_pairs(nH)
    VA = np.eye(nH)
    VB = np.eye(nH)
    tolJ = 1e-6
    tot = {"A": 0, "B": 0}
    for k in range(1, 60):
        tau = 1 / mu
        m_h = scipy.linalg.cho_solve(cho, ((d - s_mat + y / mu) @ rd).T).T
        Bm = m_h.T @ m_h
        lam_ex, V_ex = np.linalg.eigh(Bm)
        sig_ex = np.sqrt(np.maximum(lam_ex, 0))
        fex = np.where(sig_ex > tau, 1 - tau / np.maximum(sig_ex, 1e-300), 0.0)
        W_ex = (V_ex * fex) @ V_ex.T
        LH_ex = m_h @ W_ex
        rank_ex = int(np.sum(sig_ex > tau))
        nuc_ex = float(np.sum(np.maximum(sig_ex - tau, 0)))
        sig1 = sig_ex[-1]
        early = 0.03 * np.sqrt(tolJ)

        def stopA(a, b, g):
            r = np.abs(g) / np.sqrt(np.maximum(a * b, 1e-300))
            return np.where(r <= early, 0.5, r / early)  # converged-enough test

        def stopB(a, b, g):
            sa, sb = np.sqrt(np.maximum(a, 0)), np.sqrt(np.maximum(b, 0))
            fa = np.where(sa > tau, 1 - tau / np.maximum(sa, 1e-300), 0.0)
            fb = np.where(sb > tau, 1 - tau / np.maximum(sb, 1e-300), 0.0)
            dl = a - b
            with np.errstate(divide="ignore", invalid="ignore"):
                dd = np.where(np.abs(dl) > 1e-12 * np.maximum(a, b), (fa - fb) / dl,
                              tau / (2 * np.maximum(np.maximum(sa, sb), tau) ** 3))
            w = np.abs(g) * np.abs(dd) * np.maximum(sa, sb) / sig1
            # the diagonal itself (rank / nuclear): second-order g^2/|a-b| near tau^2
            return w / tolB

        out = {}
        for name, stop, V0 in (("A", stopA, VA), ("B", stopB, VB)):
            Bt = V0.T @ Bm @ V0
            Bd, V, sw = jacobi(Bt, V0, rounds, stop)
            lamd = np.diag(Bd)
            order = np.argsort(-lamd)
            lamd, V = lamd[order], V[:, order]
            sg = np.sqrt(np.maximum(lamd, 0))
            f = np.where(sg > tau, 1 - tau / np.maximum(sg, 1e-300), 0.0)
            LH = m_h @ ((V * f) @ V.T)
            err = np.linalg.norm(LH - LH_ex) / max(np.linalg.norm(LH_ex), 1e-300)
            rk = int(np.sum(sg > tau))
            nuc = float(np.sum(np.maximum(sg - tau, 0)))
            out[name] = (sw, err, rk, nuc)
            tot[name] += sw
            if name == "A":
                VA = V
            else:
                VB = V
        print(f"it {k:2d} rank {rank_ex:3d}  A: {out['A'][0]} sw err {out['A'][1]:.1e} rk {out['A'][2]} "
              f"|  B: {out['B'][0]} sw err {out['B'][1]:.1e} rk {out['B'][2]} dnuc {abs(out['B'][3]-nuc_ex)/max(nuc_ex,1e-300):.1e}",
              flush=True)
        # advance the exact iteration
        l_mat = LH_ex @ rd.T
        s_mat = O.soft_threshold(d - l_mat + y / mu, lam / mu)
        res = d - l_mat - s_mat
        gap = np.linalg.norm(res) / dn
        y = y + mu * res
        mu *= 1.5
        if gap <= tol:
            break
    print("total sweeps", tot)


if __name__ == "__main__":
    main()
