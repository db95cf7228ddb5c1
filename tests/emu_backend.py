"""CPU emulation of the CUDA backends (TEST INFRASTRUCTURE ONLY).

Implements the same per-step interface as ``paper_2206_13369_b200.backend``
(CudaPcp / CudaCpcp) with numpy on CPU torch tensors, following the device
algorithm step for step (Gram-based coarse SVT, exact residual
recomputation, coarse evaluation of the QP dots, Gram power iteration).  It
lets the product host loops (``run_ialm`` / ``run_fwt``) and their
row-sharded collectives run under gloo on a CPU-only machine, and checks the
GPU formulation itself against the oracle.
"""

from __future__ import annotations

import time

import numpy as np
import torch


def _np(t):
    return t.numpy()


class _Base:
    def __init__(self, chain, m_local, f32):
        self.chain = chain
        self.R = chain.dense()
        self.f32 = bool(f32)
        self.dt = np.float32 if f32 else np.float64
        self.nh = chain.n_coarse
        self.np_ = ((self.nh + 63) // 64) * 64
        self.n = chain.n_fine
        self.m_local = int(m_local)
        self.device = torch.device("cpu")

    def empty(self, shape, dtype):
        return torch.zeros(shape, dtype=dtype)

    # pipelined polling: the emulation is synchronous, so a snapshot is the
    # state at the time it is taken
    def snapshot(self):
        if hasattr(self, "lanczos_state"):
            return (self.state() if hasattr(self, "st") else None, self.lanczos_state())
        return self.state()

    def read_snapshot(self, token):
        return token

    def _budget_flag(self):
        """This rank's time-budget flag, summed across ranks with the stats
        (mirrors stats_reduce_kernel / cp_part_reduce)."""
        st = self.st
        wall = time.perf_counter() - st["t0"] + getattr(self, "clock_skew", 0.0)
        return 1.0 if st["time_budget"] >= 0 and wall >= st["time_budget"] else 0.0

    def close(self):
        pass

    def _restrict(self, x):
        out = np.zeros((x.shape[0], self.np_))
        out[:, :self.nh] = x.astype(np.float64) @ self.R
        return out.astype(self.dt)

    def _prolong(self, xh):
        return (xh[:, :self.nh].astype(np.float64) @ self.R.T).astype(self.dt)


class EmuPcp(_Base):
    def __init__(self, chain, m_local, m_global, f32, max_iters, device=None):
        super().__init__(chain, m_local, f32)
        self.m_global = int(m_global)
        self.max_iters = int(max_iters)
        nn = self.np_ * self.np_
        self.red = torch.zeros(max(nn + 8, self.n + 8), dtype=torch.float64)
        self.stats = torch.zeros(4, dtype=torch.float64)
        self.lz_w = torch.zeros(self.n, dtype=torch.float64)
        G = chain.dense().T @ chain.dense()
        self.Gi = np.linalg.inv(G)
        self.V = np.eye(self.np_)
        self.hist = np.zeros((max_iters, 8))

    # ---- init
    def input_stats(self, D):
        d = _np(D).astype(np.float64)
        fin = np.isfinite(d)
        v = np.where(fin, d, 0.0)
        self.stats[0] = float(np.sum(v * v))
        self.stats[1] = float(np.max(np.abs(v))) if v.size else 0.0
        self.stats[2] = float(np.count_nonzero(~fin))
        return self.stats

    def lanczos_init(self):
        self.lz = {"Q": [np.ones(self.n) / np.sqrt(self.n)], "a": [], "b": [], "theta": 0.0, "stable": 0,
                   "done": 0, "sigma1": 0.0}

    def lanczos_matvec(self, D):
        if self.lz["done"]:
            return self.lz_w
        d = _np(D).astype(np.float64)
        self.lz_w.copy_(torch.from_numpy(d.T @ (d @ self.lz["Q"][-1])))
        return self.lz_w

    def lanczos_update(self, w, tol):
        z = self.lz
        if z["done"]:
            return
        w = _np(w).copy()
        q = z["Q"][-1]
        a = float(q @ w)
        w -= a * q
        if z["b"]:
            w -= z["b"][-1] * z["Q"][-2]
        Q = np.array(z["Q"])
        for _ in range(2):
            w -= Q.T @ (Q @ w)
        b = float(np.linalg.norm(w))
        z["a"].append(a)
        T = np.diag(z["a"]) + np.diag(z["b"], 1) + np.diag(z["b"], -1)
        th = float(np.linalg.eigvalsh(T)[-1])
        rel = abs(th - z["theta"]) / th if z["theta"] > 0 else 1.0
        z["theta"] = th
        z["stable"] = z["stable"] + 1 if rel <= tol else 0
        k = len(z["a"]) - 1
        if (z["stable"] >= 2 and k >= 3) or b == 0.0 or k + 1 >= min(500, max(8, self.n)):
            z["done"] = 1
            z["sigma1"] = np.sqrt(max(th, 0.0))
            return
        z["b"].append(b)
        z["Q"].append(w / b)

    def lanczos_state(self):
        return {"k": len(self.lz["a"]), "done": self.lz["done"], "sigma1": self.lz["sigma1"],
                "theta": self.lz["theta"]}

    def start(self, D, Y0, lam, mu0, rho, tol, max_iters, time_budget, jac_tol, jac_max_sweeps):
        sumsq, maxabs = float(self.stats[0]), float(self.stats[1])
        s1 = self.lz["sigma1"]
        mu = mu0 if mu0 else 1.25 / s1
        self.st = {"lam": lam, "rho": rho, "tol": tol, "d_norm": np.sqrt(sumsq), "mu": mu, "k": 1, "done": 0,
                   "status": 0, "rank": 0, "nuclear": 0.0, "mu_last": mu, "mu_final": mu, "max_iters": max_iters,
                   "time_budget": -1.0 if time_budget is None else float(time_budget), "t0": time.perf_counter(),
                   "sigma1": s1,
                   "scale": max(s1, maxabs / lam)}
        d = _np(D)
        y = (d.astype(np.float64) / self.st["scale"]).astype(self.dt)
        Y0.copy_(torch.from_numpy(y))
        inv = self.dt(1.0 / mu)
        self.A = self._restrict(y * inv + d)

    def stats_slice(self):
        nn = self.np_ * self.np_
        return nn, nn + 4

    def gram(self, with_stats):
        nn = self.np_ * self.np_
        A = self.A.astype(np.float64)
        self.red[:nn] = torch.from_numpy((A.T @ A).ravel())
        if with_stats:
            self.red[nn:nn + 3] = torch.from_numpy(self.part)
            self.red[nn + 3] = self._budget_flag()

    def finalize(self):
        st = self.st
        if st["done"]:
            return
        nn = self.np_ * self.np_
        res2, l1, nnz, budget_hit = _np(self.red[nn:nn + 4]).tolist()
        k = st["k"]
        gap = np.sqrt(res2) / st["d_norm"]
        wall = time.perf_counter() - st["t0"]
        self.hist[k - 1] = [gap, st["nuclear"] + st["lam"] * l1, st["rank"],
                            nnz / (self.m_global * self.n), wall, st["mu"], 0, nnz]
        st["mu_last"] = st["mu"]
        st["mu_final"] = st["mu"] * st["rho"]
        if gap <= st["tol"]:
            st["done"] = 1
        elif k >= st["max_iters"] or budget_hit > 0:
            st["done"] = 2
        else:
            st["k"] = k + 1
            st["mu"] *= st["rho"]

    def svt(self):
        st = self.st
        if st["done"]:
            return
        nn = self.np_ * self.np_
        K = _np(self.red[:nn]).reshape(self.np_, self.np_)[:self.nh, :self.nh]
        B = self.Gi @ K @ self.Gi
        lam, V = np.linalg.eigh(B)
        tau = 1.0 / st["mu"]
        s = np.sqrt(np.maximum(lam, 0.0))
        keep = s > tau
        f = np.where(keep, (s - tau) / np.where(s > 0, s, 1.0), 0.0)
        st["rank"] = int(np.count_nonzero(keep))
        st["nuclear"] = float(np.sum(s[keep] - tau))
        W = self.Gi @ (V * f) @ V.T
        Z = np.zeros((self.A.shape[0], self.np_))
        Z[:, :self.nh] = self.A[:, :self.nh].astype(np.float64) @ W
        self.Z = Z.astype(self.dt)

    def update(self, D, Yin, Yout):
        st = self.st
        if st["done"]:
            return
        d, y = _np(D), _np(Yin)
        dt = self.dt
        inv, mu = dt(1.0 / st["mu"]), dt(st["mu"])
        thr = dt(st["lam"] * (1.0 / st["mu"]))
        inv_next = dt(1.0 / (st["mu"] * st["rho"]))
        L = self._prolong(self.Z)
        w = y * inv + d - L
        s = (np.sign(w) * np.maximum(np.abs(w) - thr, 0)).astype(dt)
        res = (d - L) - s
        yn = y + res * mu
        Yout.copy_(torch.from_numpy(yn))
        self.part = np.array([float(np.sum(res.astype(np.float64) ** 2)), float(np.sum(np.abs(s), dtype=np.float64)),
                              float(np.count_nonzero(s))])
        self.A = self._restrict(yn * inv_next + d - s)

    def outputs(self, D, Yprev, L, S):
        st = self.st
        d, y = _np(D), _np(Yprev)
        dt = self.dt
        inv = dt(1.0 / st["mu_last"])
        thr = dt(st["lam"] * (1.0 / st["mu_last"]))
        Lm = self._prolong(self.Z)
        w = y * inv + d - Lm
        L.copy_(torch.from_numpy(Lm))
        S.copy_(torch.from_numpy((np.sign(w) * np.maximum(np.abs(w) - thr, 0)).astype(dt)))

    def state(self):
        st = self.st
        return {"k": st["k"], "done": st["done"], "status": st["status"], "rank": st["rank"], "mu": st["mu"],
                "mu_final": st["mu_final"], "mu_last": st["mu_last"], "nuclear": st["nuclear"],
                "sigma1": st["sigma1"], "d_norm": st["d_norm"], "jac_sweeps": 1}

    def history(self, count):
        return self.hist[:count].copy()


def _coord_min(quad, lin):
    if quad <= 0.0:
        return 1.0 if lin < 0.0 else 0.0
    return min(max(-lin / quad, 0.0), 1.0)


def _box_qp(aa, bb, ab, la, lb, fb):
    def q(x, y):
        return 0.5 * (aa * x * x + 2 * ab * x * y + bb * y * y) + la * x + lb * y
    det = aa * bb - ab * ab
    best = None
    if det > 0.0:
        x = (-la * bb + lb * ab) / det
        y = (-lb * aa + la * ab) / det
        if 0.0 <= x <= 1.0 and 0.0 <= y <= 1.0:
            best = (x, y)
    if best is None:
        x = y = 0.0
        for _ in range(200):
            xn = _coord_min(aa, la + ab * y)
            yn = _coord_min(bb, lb + ab * xn)
            stop = abs(xn - x) <= 1e-12 and abs(yn - y) <= 1e-12
            x, y = xn, yn
            if stop:
                break
        best = (x, y)
    gf = min(max(fb, 0.0), 1.0)
    if q(gf, gf) < q(*best):
        best = (gf, gf)
    return best


class EmuCpcp(_Base):
    def __init__(self, chain, m_local, m_global, row0, f32, max_iters, world, device=None):
        super().__init__(chain, m_local, f32)
        self.m_global, self.row0 = int(m_global), int(row0)
        self.max_iters = int(max_iters)
        nn = self.np_ * self.np_
        self.red = torch.zeros(nn + 8, dtype=torch.float64)
        self.amax = torch.zeros(4, dtype=torch.float64)
        self.amax_all = torch.zeros(4 * int(world), dtype=torch.float64)
        self.dots = torch.zeros(3, dtype=torch.float64)
        self.mstats = torch.zeros(4, dtype=torch.float64)
        self.hist = np.zeros((max_iters, 8))
        self.objs = np.zeros(max_iters)

    def input_stats(self, D):
        d = _np(D).astype(np.float64)
        self.mstats[2] = float(np.count_nonzero(~np.isfinite(d)))
        return self.mstats

    def _mask(self, maskbits, m):
        if maskbits is None:
            return np.ones((m, self.n), dtype=bool)
        by = _np(maskbits).view(np.uint8)
        return np.unpackbits(by, axis=1, bitorder="little")[:, :self.n].astype(bool)

    def _fine(self, d, obs, S, Lh, init):
        dt = self.dt
        if init:
            r = np.where(obs, -d, 0).astype(dt)
            sn = np.zeros_like(d)
        else:
            st = self.st
            L = self._prolong(Lh)
            sh = (dt(1.0 - st["gb"]) * S).astype(dt)
            if st["corner_s"]:
                li = st["i_s"] - self.row0
                if 0 <= li < sh.shape[0]:
                    sh[li, st["j_s"]] += dt(st["gb"] * st["spike"])
            rh = (L + sh) - d
            w = np.where(obs, sh - rh, sh)
            sn = (np.sign(w) * np.maximum(np.abs(w) - dt(st["lam_s"]), 0)).astype(dt)
            r = np.where(obs, (L + sn) - d, 0).astype(dt)
        r64, s64 = r.astype(np.float64), sn.astype(np.float64)
        self.part = np.array([np.sum(r64 * r64), np.sum(np.abs(s64)), np.count_nonzero(sn), np.sum(s64 * s64),
                              np.sum(s64 * r64)])
        self.GH = self._restrict(r)
        self.SH = self._restrict(sn)
        a = np.abs(r64)
        if a.size:
            cols = np.argmax(a, axis=0)
            vals = a[cols, np.arange(a.shape[1])]
            j = int(np.argmax(vals))
            i = int(cols[j])
            self.amax.copy_(torch.tensor([a[i, j], r64[i, j], s64[i, j], float(j * self.m_global + self.row0 + i)]))
        else:
            self.amax.copy_(torch.tensor([0.0, 0.0, 0.0, -1.0]))
        return sn

    def start(self, D, maskbits, S, lam_l, lam_s, tol, radius, max_iters, time_budget):
        m = D.shape[0]
        self.obs = self._mask(maskbits, m)
        self.st = {"lam_l": lam_l, "lam_s": lam_s, "tol": tol, "radius": radius, "max_iters": max_iters,
                   "time_budget": -1.0 if time_budget is None else float(time_budget), "t_l": 0.0, "t_s": 0.0, "k": 0, "done": 0, "status": 0,
                   "ga": 0.0, "gb": 0.0, "corner_l": False, "corner_s": False, "t0": time.perf_counter(),
                   "passes": 0}
        self.LH = np.zeros((m, self.np_), dtype=self.dt)
        self.v = np.zeros(self.np_)
        self.v[:self.nh] = 1.0 / np.sqrt(self.nh)
        S.zero_()
        self._fine(_np(D), self.obs, None, None, True)

    def stats_slice(self):
        nn = self.np_ * self.np_
        return nn, nn + 6

    def gram(self):
        if self.st["done"]:
            return
        nn = self.np_ * self.np_
        g = self.GH.astype(np.float64)
        self.red[:nn] = torch.from_numpy((g.T @ g).ravel())
        self.red[nn:nn + 5] = torch.from_numpy(self.part)
        self.red[nn + 5] = self._budget_flag()

    def begin(self):
        nn = self.np_ * self.np_
        sq = float(self.red[nn])
        st = self.st
        st.update(u_l=sq / (2 * st["lam_l"]), u_s=sq / (2 * st["lam_s"]), pd_norm=np.sqrt(sq), sq=sq, ss=0.0, sr=0.0,
                  k=1)
        if st["u_l"] == 0.0:
            st["done"] = 1

    def lmo(self):
        st = self.st
        if st["done"]:
            return
        nn = self.np_ * self.np_
        K = _np(self.red[:nn]).reshape(self.np_, self.np_)
        v = self.v.copy()
        prev, none, p = -1.0, False, 0
        vin = v
        s2 = nw = 0.0
        for p in range(1, 41):
            kv = K @ v
            s2 = float(v @ kv)
            kvn = float(np.linalg.norm(kv))
            if s2 <= 0.0 or kvn == 0.0:
                none = True
                break
            nw = kvn / np.sqrt(s2)
            vin = v
            v = kv / kvn
            stop = abs(s2 - prev) <= 1e-6 * s2
            prev = s2
            if stop:
                break
        if not none:
            self.v = v
        st.update(none=none, s2=s2, sigma=nw, passes=p)
        self.vin = vin
        recs = _np(self.amax_all).reshape(-1, 4)
        best = None
        for rec in recs:
            if rec[3] < 0:
                continue
            if best is None or rec[0] > best[0] or (rec[0] == best[0] and rec[3] < best[3]):
                best = rec
        if best is None:
            best = np.array([0.0, 0.0, 0.0, 0.0])
        idx = int(best[3])
        st["j_s"], st["i_s"] = idx // self.m_global, idx % self.m_global
        st["r_is"], st["s_is"] = float(best[1]), float(best[2])
        val_l = 0.0 if none else -st["radius"] * nw
        st["corner_l"] = st["lam_l"] < -val_l
        st["corner_s"] = st["lam_s"] < abs(st["r_is"])
        st["v_tl"] = st["u_l"] if st["corner_l"] else 0.0
        st["v_ts"] = st["u_s"] if st["corner_s"] else 0.0
        st["coef"] = -st["radius"] * st["u_l"] if st["corner_l"] else 0.0
        st["spike"] = -st["u_s"] * np.sign(st["r_is"]) if st["corner_s"] else 0.0
        # coarse dots
        g = self.GH.astype(np.float64)[:, :self.nh]
        u = np.zeros(g.shape[0]) if none else g @ vin[:self.nh] / np.sqrt(s2)
        self.u = u
        E = st["coef"] * np.outer(u, self.v[:self.nh]) - self.LH.astype(np.float64)[:, :self.nh]
        a = np.where(self.obs, E @ self.R.T, 0.0)
        aa = float(np.sum(a * a))
        ab = -float(np.sum(E * self.SH.astype(np.float64)[:, :self.nh]))
        ar = float(np.sum(E * g))
        li = st["i_s"] - self.row0
        if st["corner_s"] and 0 <= li < a.shape[0]:
            ab += st["spike"] * a[li, st["j_s"]]
        self.dots.copy_(torch.tensor([aa, ab, ar]))

    def update(self, D, maskbits, S):
        st = self.st
        if st["done"]:
            return
        aa, ab, ar = _np(self.dots).tolist()
        bb, br = st["ss"], -st["sr"]
        if st["corner_s"]:
            bb += st["spike"] ** 2 - 2 * st["spike"] * st["s_is"]
            br += st["spike"] * st["r_is"]
        la = ar + st["lam_l"] * (st["v_tl"] - st["t_l"])
        lb = br + st["lam_s"] * (st["v_ts"] - st["t_s"])
        ga, gb = _box_qp(aa, bb, ab, la, lb, 2.0 / (st["k"] + 2.0))
        st["ga"], st["gb"] = ga, gb
        st["t_l"] += ga * (st["v_tl"] - st["t_l"])
        st["t_s"] += gb * (st["v_ts"] - st["t_s"])
        lh = (1 - ga) * self.LH.astype(np.float64)
        lh[:, :self.nh] += ga * st["coef"] * np.outer(self.u, self.v[:self.nh])
        self.LH = lh.astype(self.dt)
        sn = self._fine(_np(D), self.obs, _np(S), self.LH, False)
        S.copy_(torch.from_numpy(sn))

    def finalize(self):
        st = self.st
        if st["done"]:
            return
        nn = self.np_ * self.np_
        sq, l1, nnz, ss, sr, budget_hit = _np(self.red[nn:nn + 6]).tolist()
        st.update(sq=sq, ss=ss, sr=sr, t_s=l1)
        obj = 0.5 * sq + st["lam_l"] * st["t_l"] + st["lam_s"] * st["t_s"]
        st["u_l"] = min(st["u_l"], obj / st["lam_l"])
        st["u_s"] = min(st["u_s"], obj / st["lam_s"])
        k = st["k"]
        self.objs[k - 1] = obj
        wall = time.perf_counter() - st["t0"]
        self.hist[k - 1] = [np.sqrt(sq) / st["pd_norm"], obj, -1, nnz / (self.m_global * self.n), wall, st["ga"],
                            st["gb"], st["passes"]]
        conv = k > 5 and self.objs[k - 6] - obj <= st["tol"] * max(abs(self.objs[k - 6]), np.finfo(float).tiny)
        if conv:
            st["done"] = 1
        elif k >= st["max_iters"] or budget_hit > 0:
            st["done"] = 2
        else:
            st["k"] = k + 1

    def outputs(self, L):
        L.copy_(torch.from_numpy(self._prolong(self.LH)))

    def state(self):
        st = self.st
        keys = ("k", "done", "status", "t_l", "t_s", "u_l", "u_s")
        return {k: st.get(k, 0) for k in keys}

    def history(self, count):
        return self.hist[:count].copy(), self.objs[:count].copy()
