"""Golden fixtures for the full-size BASELINE configs C3, C4 and C5, produced
by the REAL reference package (/root/reference/pkg/src/mlrpca) in the build
container.  The GPU box regenerates the same inputs from the seeded
generators (paper_2206_13369_b200/datasets.py) and compares against these
summaries, so nothing here has to travel except the small .npz files.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_large.py [C5] [C3] [C4] [small]

What is stored (fine planes are far too large to commit):
* iteration count, mu, the full history columns (gap / objective / rank /
  sparsity), mu or objective history;
* Frobenius norms of L, S (and Y for PCP);
* seeded Gaussian sketches L q, p^T L, S q, p^T S (q ~ N(0, I_n),
  p ~ N(0, I_m), rng seed 77) -- relF of a sketch tracks relF of the plane;
* a few fixed rows of L and S (float32).

ML-CPCP (C3, C4 and the small golden cases) additionally stores the
SURVEY.md 8(c) envelope: the oracle run E = 6 times on the same input with
BLAS threads 1, 2, 4 and N plus two 1-ulp relative input perturbations
(threads N).  The GPU gate is: iterations inside [min, max] +- max(2, 2% of
the mean) and final objective within max(1e-6, 2 x the envelope's relative
spread) of the primary run.  C4 runs the envelope at max_iters = 300 (the
full-tolerance oracle takes > 15 min per run).
"""

import os
import sys
import time

import numpy as np
from threadpoolctl import threadpool_info, threadpool_limits

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import mlrpca  # noqa: E402  (reference)
from paper_2206_13369_b200.datasets import CONFIGS, make_config  # noqa: E402  (seeded inputs only)

NCPU = len(os.sched_getaffinity(0))
EPS = np.finfo(np.float64).eps


def sketches(x, tag):
    m, n = x.shape
    rng = np.random.default_rng(77)
    q = rng.standard_normal(n)
    p = rng.standard_normal(m)
    return {f"{tag}_q": x @ q, f"{tag}_p": p @ x, f"{tag}_fro": np.array(np.linalg.norm(x))}


def rows_of(m):
    return np.linspace(0, m - 1, 8).astype(np.int64)


def hist_arrays(history):
    return {
        "h_gap": np.array([h.feasibility_gap for h in history]),
        "h_obj": np.array([h.objective for h in history]),
        "h_rank": np.array([h.rank_l for h in history]),
        "h_sparsity": np.array([h.sparsity_s for h in history]),
    }


def blas_info():
    return " | ".join(f"{i.get('internal_api')} {i.get('version')} threads={i.get('num_threads')}"
                      for i in threadpool_info())


def perturb(d, q):
    """1-ulp relative perturbation of every entry (random sign / no-op)."""
    rng = np.random.default_rng(1000 + q)
    return d * (1 + rng.integers(-1, 2, d.shape) * EPS)


def make_c5(seed=0):
    c = CONFIGS["C5"]
    d32, _ = make_config("C5", seed)
    d = d32.astype(np.float64)
    m, n = d.shape
    t0 = time.perf_counter()
    with threadpool_limits(limits=NCPU):
        st = mlrpca.ml_ialm_solve(d, mlrpca.PcpOptions(lam=1 / np.sqrt(max(m, n)), tol_feasibility=c["tol"],
                                                       levels=c["n_coarse"]))
    wall = time.perf_counter() - t0
    rows = rows_of(m)
    np.savez_compressed(
        os.path.join(HERE, "c5_pcp.npz"), seed=np.array(seed), d_sum=np.array(d.sum()), iter=np.array(st.iter),
        mu=np.array(st.mu), converged=np.array(st.converged), mu_history=np.array(st.mu_history),
        rows=rows, l_rows=st.l[rows].astype(np.float32), s_rows=st.s[rows].astype(np.float32),
        wall_s=np.array(wall), loop_s=np.array(st.history[-1].wall_seconds), threads=np.array(NCPU),
        blas=np.array(blas_info()), **sketches(st.l, "l"), **sketches(st.s, "s"), **sketches(st.y, "y"),
        **hist_arrays(st.history))
    print(f"C5: {st.iter} iterations, converged={st.converged}, {wall:.0f} s", flush=True)


def cpcp_envelope(name, d, mask, nh, tol, max_iters, seed, out, extra=None):
    m, n = d.shape
    lam = 1 / np.sqrt(max(m, n))
    lam_s = lam / np.sqrt(max(m, n))
    om = mlrpca.ObservationMask(mask) if mask is not None else None
    opts = mlrpca.CpcpOptions(lambda_l=lam, lambda_s=lam_s, tol=tol, max_iters=max_iters, levels=nh,
                              collect_rank=False)
    runs = [("threads", NCPU, d), ("threads", 1, d), ("threads", 2, d), ("threads", 4, d),
            ("perturb", NCPU, perturb(d, 0)), ("perturb", NCPU, perturb(d, 1))]
    env_iter, env_obj, env_wall, env_desc, objs = [], [], [], [], []
    primary = None
    for kind, th, dd in runs:
        if kind == "threads" and th > NCPU:
            continue
        t0 = time.perf_counter()
        with threadpool_limits(limits=th):
            st = mlrpca.ml_fwt_solve(dd, om, opts)
        wall = time.perf_counter() - t0
        env_iter.append(st.iter)
        env_obj.append(st.history[-1].objective)
        env_wall.append(wall)
        env_desc.append(f"{kind} threads={th}")
        objs.append(np.array(st.objective_history))
        print(f"{name}: {kind} threads={th}: {st.iter} iterations, obj {st.history[-1].objective!r}, {wall:.0f} s",
              flush=True)
        if primary is None:
            primary = st
    st = primary
    rows = rows_of(m)
    L = max(len(o) for o in objs)
    obj_mat = np.full((len(objs), L), np.nan)
    for i, o in enumerate(objs):
        obj_mat[i, :len(o)] = o
    np.savez_compressed(
        os.path.join(HERE, out), seed=np.array(seed), d_sum=np.array(d.sum()), n_coarse=np.array(nh),
        tol=np.array(tol), max_iters=np.array(max_iters), lam_l=np.array(lam), lam_s=np.array(lam_s),
        iter=np.array(st.iter), converged=np.array(st.converged), t_l=np.array(st.t_l), t_s=np.array(st.t_s),
        u_l=np.array(st.u_l), u_s=np.array(st.u_s), objective_history=np.array(st.objective_history),
        rows=rows, l_rows=st.l[rows].astype(np.float32), s_rows=st.s[rows].astype(np.float32),
        env_iter=np.array(env_iter), env_obj=np.array(env_obj), env_wall=np.array(env_wall),
        env_desc=np.array(env_desc), env_objs=obj_mat, threads=np.array(NCPU), blas=np.array(blas_info()),
        **sketches(st.l, "l"), **sketches(st.s, "s"), **hist_arrays(st.history), **(extra or {}))


def make_c3(seed=0):
    c = CONFIGS["C3"]
    d32, mask = make_config("C3", seed)
    cpcp_envelope("C3", d32.astype(np.float64), mask, c["n_coarse"], c["tol"], 5000, seed, "c3_cpcp.npz")


def make_c4(seed=0):
    c = CONFIGS["C4"]
    d32, mask = make_config("C4", seed)
    cpcp_envelope("C4", d32.astype(np.float64), mask, c["n_coarse"], c["tol"], 300, seed, "c4_cpcp.npz")


def make_small():
    """Envelopes for the small ML-CPCP golden cases (same inputs as
    make_golden.fwt_cases), so the GPU tests can use the exact 8(c) gate."""
    sys.path.insert(0, ROOT)
    from oracle import mlrpca_oracle as O
    cases = {
        "fwt_f64_small": (100, 80, 4, 0.10, 0.8, 5, 20, 1e-6, 300, np.float64),
        "fwt_f32_small": (160, 128, 4, 0.10, 0.7, 6, 16, 1e-5, 200, np.float32),
        "fwt_f64_full": (64, 50, 3, 0.10, None, 7, 13, 1e-6, 200, np.float64),
    }
    for name, (m, n, r, eta, obs, seed, nh, tol, iters, dt) in cases.items():
        d, mask = O.gaussian_rpca(m, n, r, eta, seed, observe=obs)
        d = d.astype(dt).astype(np.float64)
        cpcp_envelope(name, d, mask, nh, tol, iters, seed, f"env_{name}.npz")


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "C3", "C5", "C4"]
    print("BLAS:", blas_info(), "cpus:", NCPU, flush=True)
    for w in which:
        {"C5": make_c5, "C3": make_c3, "C4": make_c4, "small": make_small}[w]()
