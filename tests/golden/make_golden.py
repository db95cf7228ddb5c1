"""Generate golden vectors from the REAL reference package (run in the build
container, where /root/reference exists; the outputs are committed so the GPU
box can check without the reference).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Inputs are produced by the oracle's seeded generators (identical on both
sides); every output below is computed by ``mlrpca`` itself
(/root/reference/pkg/src/mlrpca, v0.1.0).
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import mlrpca  # noqa: E402  (reference)
from oracle import mlrpca_oracle as O  # noqa: E402  (input generators only)


def hist_arrays(history):
    return {
        "h_gap": np.array([h.feasibility_gap for h in history]),
        "h_obj": np.array([h.objective for h in history]),
        "h_rank": np.array([h.rank_l for h in history]),
        "h_sparsity": np.array([h.sparsity_s for h in history]),
    }


def multilevel_kats():
    out = {}
    out["R6"] = mlrpca.build_interpolation(6).toarray()
    for n, t in [(8, 2), (16, 4), (33, 9), (64, 8), (100, 25), (101, 13), (128, 32)]:
        ch = mlrpca.build_chain(n, t, normalize=True)
        out[f"R_{n}_{t}"] = ch.composite.toarray()
        out[f"spec_{n}_{t}"] = np.array(ch.spectral_norm)
    for n, t in [(500, 125), (2000, 250), (4000, 500), (1000, 125), (20000, 1250)]:
        ch = mlrpca.build_chain(n, t, normalize=True)
        r = ch.composite.tocsr()
        out[f"Rcsr_{n}_{t}_data"] = r.data
        out[f"Rcsr_{n}_{t}_indices"] = r.indices
        out[f"Rcsr_{n}_{t}_indptr"] = r.indptr
        out[f"spec_{n}_{t}"] = np.array(ch.spectral_norm)
    out["coarse_sizes_400"] = np.array(mlrpca.multilevel.coarse_sizes(400))
    out["select_1024_5_1_10000"] = np.array(mlrpca.select_levels(1024, 5, 1, 10000))
    out["select_400_2_1_3072"] = np.array(mlrpca.select_levels(400, 2, 1, 3072))
    x = np.random.default_rng(11).standard_normal((5, 100))
    ch = mlrpca.build_chain(100, 25)
    out["restrict_x"] = x
    out["restrict_y"] = mlrpca.restrict(x, ch)
    out["restrict_ls_y"] = mlrpca.restrict_least_squares(x, ch)
    out["prolong_y"] = mlrpca.prolong(out["restrict_y"], ch)
    np.savez_compressed(os.path.join(HERE, "multilevel.npz"), **out)


def linalg_kats():
    out = {}
    out["st_in"] = np.array([[1.0, -0.3, 0.7]])
    out["st_out"] = mlrpca.soft_threshold(out["st_in"], 0.5)
    z, rank = mlrpca.svt(np.diag([3.0, 1.0]), 2.0)
    out["svt_diag_z"], out["svt_diag_rank"] = z, np.array(rank)
    z, rank = mlrpca.svt(np.diag([3.0, 2.0]), 2.0)
    out["svt_tie_z"], out["svt_tie_rank"] = z, np.array(rank)
    x = np.random.default_rng(8).standard_normal((40, 12))
    out["svt_x"] = x
    out["svt_z"], r = mlrpca.svt(x, 1.5)
    out["svt_rank"] = np.array(r)
    np.savez_compressed(os.path.join(HERE, "linalg.npz"), **out)


def pcp_cases():
    cases = {
        # name: (m, n, rank, eta, seed, n_H, tol, dtype)
        "pcp_f64_small": (120, 96, 6, 0.10, 3, 24, 1e-7, np.float64),
        "pcp_f32_small": (200, 160, 8, 0.10, 4, 40, 1e-6, np.float32),
        "pcp_f64_odd": (90, 77, 5, 0.08, 5, 20, 1e-7, np.float64),
    }
    for name, (m, n, r, eta, seed, nh, tol, dt) in cases.items():
        d, _ = O.gaussian_rpca(m, n, r, eta, seed)
        d = d.astype(dt).astype(np.float64)
        st = mlrpca.ml_ialm_solve(d, mlrpca.PcpOptions(levels=nh, tol_feasibility=tol))
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), d=d, l=st.l, s=st.s, y=st.y,
            mu=np.array(st.mu), iter=np.array(st.iter), n_coarse=np.array(nh),
            tol=np.array(tol), converged=np.array(st.converged),
            mu_history=np.array(st.mu_history), **hist_arrays(st.history))


def pcp_c1_summary():
    # C1 at full size: L/S are 2 MB each, so only fingerprints are committed;
    # the full arrays are checked live against the oracle on the GPU box.
    d, _ = O.make_config("C1", 0)
    st = mlrpca.ml_ialm_solve(d, mlrpca.PcpOptions(
        lam=1 / np.sqrt(500), tol_feasibility=1e-7, levels=125))
    rows = np.arange(0, 500, 37)
    np.savez_compressed(
        os.path.join(HERE, "pcp_c1_summary.npz"),
        d_sum=np.array(d.sum()), iter=np.array(st.iter), mu=np.array(st.mu),
        l_fro=np.array(np.linalg.norm(st.l)), s_fro=np.array(np.linalg.norm(st.s)),
        y_fro=np.array(np.linalg.norm(st.y)), l_rows=st.l[rows], s_rows=st.s[rows],
        rows=rows, sigma1=np.array(np.linalg.norm(d, 2)), **hist_arrays(st.history))


def ialm_cases():
    """Full-width inexact ALM (mlrpca.ialm_solve, pcp.py:118-197): dense SVD
    below min(m, n) = 256, ARPACK above it, a wide input and a clipped
    svd_budget."""
    cases = {
        # name: (m, n, rank, eta, seed, tol, svd_budget, dtype, full arrays)
        "ialm_f64_dense": (120, 100, 5, 0.10, 21, 1e-7, None, np.float64, True),
        "ialm_f32_dense": (150, 128, 6, 0.10, 22, 1e-6, None, np.float32, True),
        "ialm_f64_wide": (80, 110, 4, 0.10, 23, 1e-7, None, np.float64, True),
        "ialm_f64_budget": (100, 90, 8, 0.10, 24, 1e-7, 6, np.float64, True),
        "ialm_f64_arpack": (300, 280, 6, 0.10, 25, 1e-7, None, np.float64, False),
    }
    for name, (m, n, r, eta, seed, tol, budget, dt, full) in cases.items():
        d, _ = O.gaussian_rpca(m, n, r, eta, seed)
        d = d.astype(dt).astype(np.float64)
        st = mlrpca.ialm_solve(d, mlrpca.PcpOptions(tol_feasibility=tol, svd_budget=budget))
        rows = np.arange(0, m, 17)
        arrays = dict(l=st.l, s=st.s, y=st.y) if full else dict(l_rows=st.l[rows], s_rows=st.s[rows], rows=rows)
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), d=d if full else np.zeros(0), seed=np.array(seed),
            shape=np.array([m, n, r]), eta=np.array(eta), mu=np.array(st.mu), iter=np.array(st.iter),
            tol=np.array(tol), svd_budget=np.array(budget or 0), converged=np.array(st.converged),
            l_fro=np.array(np.linalg.norm(st.l)), s_fro=np.array(np.linalg.norm(st.s)),
            y_fro=np.array(np.linalg.norm(st.y)), mu_history=np.array(st.mu_history),
            **arrays, **hist_arrays(st.history))


def telemetry_cases():
    """collect_diagnostics (pcp.py:298-306) and collect_rank (cpcp.py:434-439)."""
    d, _ = O.gaussian_rpca(120, 96, 6, 0.10, 3)
    st = mlrpca.ml_ialm_solve(d, mlrpca.PcpOptions(levels=24, collect_diagnostics=True))
    np.savez_compressed(os.path.join(HERE, "diag_pcp_f64.npz"), d=d, n_coarse=np.array(24), iter=np.array(st.iter),
                        epsilon=np.array(st.diagnostics.epsilon), deltas=np.array(st.diagnostics.delta_history))
    d32, _ = O.gaussian_rpca(200, 160, 8, 0.10, 4)
    d32 = d32.astype(np.float32).astype(np.float64)
    st = mlrpca.ml_ialm_solve(d32, mlrpca.PcpOptions(levels=40, tol_feasibility=1e-6, collect_diagnostics=True))
    np.savez_compressed(os.path.join(HERE, "diag_pcp_f32.npz"), d=d32, n_coarse=np.array(40), iter=np.array(st.iter),
                        tol=np.array(1e-6), epsilon=np.array(st.diagnostics.epsilon),
                        deltas=np.array(st.diagnostics.delta_history))
    cases = {
        # name: (m, n, rank, eta, observe, seed, n_H (None = full width), tol, max_iters, dtype)
        "rank_ml_f64": (100, 80, 4, 0.10, 0.8, 5, 20, 1e-6, 120, np.float64),
        "rank_full_f64": (90, 70, 4, 0.10, 0.8, 11, None, 1e-6, 120, np.float64),
        "rank_ml_f32": (160, 128, 4, 0.10, 0.7, 6, 16, 1e-5, 80, np.float32),
    }
    for name, (m, n, r, eta, obs, seed, nh, tol, iters, dt) in cases.items():
        d, mask = O.gaussian_rpca(m, n, r, eta, seed, observe=obs)
        d = d.astype(dt).astype(np.float64)
        lam = 1 / np.sqrt(max(m, n))
        opts = mlrpca.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=tol, max_iters=iters,
                                  levels=nh, collect_rank=True)
        om = mlrpca.ObservationMask(mask)
        st = mlrpca.fwt_solve(d, om, opts) if nh is None else mlrpca.ml_fwt_solve(d, om, opts)
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), d=d, mask=mask, n_coarse=np.array(nh or 0), tol=np.array(tol),
            max_iters=np.array(iters), lam_l=np.array(lam), lam_s=np.array(lam / np.sqrt(max(m, n))),
            iter=np.array(st.iter), l_rank=np.array(np.linalg.matrix_rank(st.l)), **hist_arrays(st.history))


def atom_cases():
    """track_oracle_atoms (cpcp.py:355-360): every iteration's dense LMO atom."""
    cases = {
        # name: (m, n, rank, observe, seed, n_H (None = full width), max_iters)
        "atoms_ml_f64": (40, 32, 3, 0.8, 31, 8, 12),
        "atoms_full_f64": (30, 24, 3, 0.8, 32, None, 10),
    }
    for name, (m, n, r, obs, seed, nh, iters) in cases.items():
        d, mask = O.gaussian_rpca(m, n, r, 0.1, seed, observe=obs)
        lam = 1 / np.sqrt(max(m, n))
        opts = mlrpca.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=1e-9, max_iters=iters,
                                  levels=nh, collect_rank=False, track_oracle_atoms=True)
        om = mlrpca.ObservationMask(mask)
        st = mlrpca.fwt_solve(d, om, opts) if nh is None else mlrpca.ml_fwt_solve(d, om, opts)
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), d=d, mask=mask, n_coarse=np.array(nh or 0), max_iters=np.array(iters),
            lam_l=np.array(lam), lam_s=np.array(lam / np.sqrt(max(m, n))), iter=np.array(st.iter),
            atoms=np.array(st.oracle_atoms), **hist_arrays(st.history))


def frame_cases():
    """Frame-stack I/O (io.py:100-182): raw PGM bytes, the reference's ingested
    matrix and the bytes its emit_frames writes for given L / S."""
    import tempfile
    from mlrpca import io as rio
    rng = np.random.default_rng(41)
    h, w, count = 6, 5, 3
    raster = rng.integers(0, 256, (count, h, w), dtype=np.uint8)
    raster[0, 0, :] = [0, 1, 127, 254, 255]
    with tempfile.TemporaryDirectory() as tmp:
        paths = []
        for j in range(count):
            p = os.path.join(tmp, f"f{j}.pgm")
            if j == 1:  # header with a comment and odd whitespace
                with open(p, "wb") as fh:
                    fh.write(b"P5 # frame one\n%d\t%d\n# max\n255\n" % (w, h) + raster[j].tobytes())
            else:
                rio.write_pgm(raster[j], p)
            paths.append(p)
        files = [open(p, "rb").read() for p in paths]
        stack = rio.ingest_frames(paths)
        m = h * w
        l = rng.uniform(-0.2, 1.2, (m, count))
        s = rng.uniform(-0.5, 0.5, (m, count))
        l[:4, 0] = [0.5 / 255, 1.5 / 255, 254.5 / 255, 1.0]  # round-half-up boundaries
        out = os.path.join(tmp, "out")
        written = rio.emit_frames(stack, l, s, out)
        emitted = [open(p, "rb").read() for p in written]
        names = [os.path.basename(p) for p in written]
    blob = np.frombuffer(b"".join(files), dtype=np.uint8)
    eblob = np.frombuffer(b"".join(emitted), dtype=np.uint8)
    np.savez_compressed(
        os.path.join(HERE, "frames.npz"), raster=raster, files=blob, file_sizes=np.array([len(f) for f in files]),
        matrix=stack.matrix, height=np.array(h), width=np.array(w), l=l, s=s, emitted=eblob,
        emitted_sizes=np.array([len(e) for e in emitted]), names=np.array(names))


def fwt_cases():
    cases = {
        # name: (m, n, rank, eta, observe, seed, n_H, tol, max_iters, dtype)
        "fwt_f64_small": (100, 80, 4, 0.10, 0.8, 5, 20, 1e-6, 300, np.float64),
        "fwt_f32_small": (160, 128, 4, 0.10, 0.7, 6, 16, 1e-5, 200, np.float32),
        "fwt_f64_full": (64, 50, 3, 0.10, None, 7, 13, 1e-6, 200, np.float64),
    }
    for name, (m, n, r, eta, obs, seed, nh, tol, iters, dt) in cases.items():
        d, mask = O.gaussian_rpca(m, n, r, eta, seed, observe=obs)
        d = d.astype(dt).astype(np.float64)
        lam = 1 / np.sqrt(max(m, n))
        om = mlrpca.ObservationMask(mask) if mask is not None else None
        st = mlrpca.ml_fwt_solve(d, om, mlrpca.CpcpOptions(
            lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=tol,
            max_iters=iters, levels=nh, collect_rank=False))
        extra = {"mask": mask} if mask is not None else {}
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), d=d, l=st.l, s=st.s,
            t_l=np.array(st.t_l), t_s=np.array(st.t_s), u_l=np.array(st.u_l),
            u_s=np.array(st.u_s), iter=np.array(st.iter), n_coarse=np.array(nh),
            tol=np.array(tol), max_iters=np.array(iters), lam_l=np.array(lam),
            lam_s=np.array(lam / np.sqrt(max(m, n))),
            converged=np.array(st.converged), **hist_arrays(st.history), **extra)


def fwt_full_cases():
    """Full-width Frank-Wolfe thresholding (mlrpca.fwt_solve, cpcp.py:459-477)."""
    cases = {
        # name: (m, n, rank, eta, observe, seed, tol, max_iters, dtype)
        "fwtfull_f64": (90, 70, 4, 0.10, 0.8, 11, 1e-6, 250, np.float64),
        "fwtfull_f32": (120, 96, 4, 0.10, 0.7, 12, 1e-5, 200, np.float32),
    }
    for name, (m, n, r, eta, obs, seed, tol, iters, dt) in cases.items():
        d, mask = O.gaussian_rpca(m, n, r, eta, seed, observe=obs)
        d = d.astype(dt).astype(np.float64)
        lam = 1 / np.sqrt(max(m, n))
        om = mlrpca.ObservationMask(mask) if mask is not None else None
        st = mlrpca.fwt_solve(d, om, mlrpca.CpcpOptions(
            lambda_l=lam, lambda_s=lam / np.sqrt(max(m, n)), tol=tol, max_iters=iters, collect_rank=False))
        # FW-T is chaotic: the envelope is the spread of the
        # oracle itself under 1-ulp input perturbations (12 runs)
        env_obj, env_it = 0.0, 0
        for q in range(12):
            rng = np.random.default_rng(1000 + q)
            dp = d * (1 + rng.integers(-1, 2, d.shape) * np.finfo(np.float64).eps)
            o = O.ml_fwt(dp, mask, lam, lam / np.sqrt(max(m, n)), tol=tol, max_iters=iters, levels=n,
                         collect_rank=False)
            env_obj = max(env_obj, abs(o.objective_history[-1] - st.objective_history[-1]) / st.objective_history[-1])
            env_it = max(env_it, abs(o.iter - st.iter))
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), d=d, mask=mask, l=st.l, s=st.s,
            env_obj=np.array(env_obj), env_iter=np.array(env_it),
            t_l=np.array(st.t_l), t_s=np.array(st.t_s), u_l=np.array(st.u_l),
            u_s=np.array(st.u_s), iter=np.array(st.iter), tol=np.array(tol), max_iters=np.array(iters),
            lam_l=np.array(lam), lam_s=np.array(lam / np.sqrt(max(m, n))),
            converged=np.array(st.converged), **hist_arrays(st.history))


if __name__ == "__main__":
    multilevel_kats()
    linalg_kats()
    pcp_cases()
    pcp_c1_summary()
    ialm_cases()
    telemetry_cases()
    atom_cases()
    frame_cases()
    fwt_cases()
    fwt_full_cases()
    print("golden vectors written to", HERE)
