"""GPU parity: the CUDA path (through the public drop-in API and the C ABI)
against the CPU oracle / the reference's golden vectors, on a B200.

Gates:
  ML-PCP   iterations equal (+-1), relF(L), relF(S) <= 1e-10 (float64 input)
           or <= 1e-4 (float32 input), final rank equal.
  ML-CPCP  envelope gate: iteration count within max(2, 5%) and the final
           objective within 1e-4 relative (FW-T forks on l1 arg-max ties,
           SURVEY.md fact 7); iteration 1 must agree to rounding.
"""

import os

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

import paper_2206_13369_b200 as pkg  # noqa: E402
from oracle import mlrpca_oracle as O  # noqa: E402
from paper_2206_13369_b200.datasets import CONFIGS, make_config  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def relf(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


# ------------------------------------------------------------------ ML-PCP
@pytest.mark.parametrize("name,tolrel", [("pcp_f64_small", 1e-10), ("pcp_f64_odd", 1e-10),
                                          ("pcp_f32_small", 1e-4)])
def test_ml_ialm_golden(golden, name, tolrel):
    g = golden(name)
    d = g["d"].astype(np.float32) if "f32" in name else g["d"]
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=int(g["n_coarse"]), tol_feasibility=float(g["tol"])))
    assert abs(st.iter - int(g["iter"])) <= 1
    assert relf(st.l, g["l"]) <= tolrel
    assert relf(st.s, g["s"]) <= tolrel
    assert st.converged == bool(g["converged"])
    if st.iter == int(g["iter"]):
        assert st.history[-1].rank_l == int(g["h_rank"][-1])
        # mu = rho^k 1.25 / sigma_1(D): FP64 computes sigma_1 to ~1e-15, FP32
        # to 1e-9 (pcp.py lz_tol; far below the FP32 parity gate of 1e-4)
        assert np.isclose(st.mu, float(g["mu"]), rtol=1e-12 if "f64" in name else 1e-8)


def test_ml_ialm_c1_fp64_vs_oracle(golden):
    d, _ = make_config("C1")
    c = CONFIGS["C1"]
    ref = O.ml_ialm(d, lam=1 / np.sqrt(500), tol=c["tol"], levels=c["n_coarse"])
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(lam=1 / np.sqrt(500), tol_feasibility=c["tol"], levels=c["n_coarse"]))
    assert st.iter == ref.iter
    assert relf(st.l, ref.l) <= 1e-10
    assert relf(st.s, ref.s) <= 1e-10
    # Y accumulates mu_k * residual with mu_k ~ 1e5 at exit, which amplifies
    # the 1e-13-level L/S differences; the gate is on L and S
    assert relf(st.y, ref.y) <= 1e-8
    assert st.history[-1].rank_l == ref.history[-1].rank_l
    assert abs(st.history[-1].sparsity_s - ref.history[-1].sparsity_s) <= 2.0 / d.size
    gs = golden("pcp_c1_summary")
    assert st.iter == int(gs["iter"])
    assert np.allclose([h.feasibility_gap for h in st.history], gs["h_gap"], rtol=1e-6)


@pytest.mark.slow
def test_ml_ialm_c2_fp32_vs_oracle():
    d, _ = make_config("C2")
    c = CONFIGS["C2"]
    ref = O.ml_ialm(d.astype(np.float64), lam=1 / np.sqrt(2000), tol=c["tol"], levels=c["n_coarse"])
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(lam=1 / np.sqrt(2000), tol_feasibility=c["tol"],
                                             levels=c["n_coarse"]))
    assert st.l.dtype == np.float32
    assert abs(st.iter - ref.iter) <= 1
    assert relf(st.l, ref.l) <= 1e-4
    assert relf(st.s, ref.s) <= 1e-4
    assert st.history[-1].rank_l == ref.history[-1].rank_l


def test_ml_ialm_torch_input_stays_on_device():
    import torch
    d, _ = O.gaussian_rpca(96, 80, 4, 0.1, 5)
    D = torch.from_numpy(d).cuda()
    st = pkg.ml_ialm_solve(D, pkg.PcpOptions(levels=20))
    assert isinstance(st.l, torch.Tensor) and st.l.is_cuda and st.l.dtype == torch.float64
    ref = O.ml_ialm(d, levels=20)
    assert st.iter == ref.iter and relf(st.l.cpu().numpy(), ref.l) <= 1e-10


def test_ml_ialm_edge_cases():
    z = pkg.ml_ialm_solve(np.zeros((20, 16)), pkg.PcpOptions(levels=4))
    assert z.converged and z.iter == 1 and np.all(z.l == 0) and z.mu == 0.0
    bad = np.ones((16, 16))
    bad[2, 3] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        pkg.ml_ialm_solve(bad, pkg.PcpOptions(levels=4))
    with pytest.raises(ValueError):
        pkg.ml_ialm_solve(np.ones(5))
    with pytest.raises(pkg.LevelError):
        pkg.ml_ialm_solve(np.ones((8, 8)), pkg.PcpOptions(levels=0))
    with pytest.raises(ValueError, match="not reachable"):
        pkg.ml_ialm_solve(np.ones((8, 8)), pkg.PcpOptions(levels=3))
    d, _ = O.gaussian_rpca(64, 48, 3, 0.1, 8)
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=12, max_iters=4, tol_feasibility=1e-12))
    assert st.iter == 4 and not st.converged and len(st.mu_history) == 4
    ref = O.ml_ialm(d, levels=12, max_iters=4, tol=1e-12)
    assert relf(st.l, ref.l) <= 1e-10


def test_ml_ialm_identity_chain_and_select_levels():
    d, _ = O.gaussian_rpca(70, 40, 3, 0.1, 9)
    ref = O.ml_ialm(d, levels=40)
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=40))
    assert st.iter == ref.iter and relf(st.l, ref.l) <= 1e-10
    ref = O.ml_ialm(d, rank_guess=5)  # levels=None -> select_levels
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(rank_guess=5))
    assert st.iter == ref.iter and relf(st.l, ref.l) <= 1e-10


# ------------------------------------------------------------------ full-width PCP
@pytest.mark.parametrize("name,tolrel", [("ialm_f64_dense", 1e-10), ("ialm_f32_dense", 1e-4),
                                          ("ialm_f64_wide", 1e-10), ("ialm_f64_budget", 1e-10),
                                          ("ialm_f64_arpack", 1e-10)])
def test_ialm_golden(golden, name, tolrel):
    """ialm_solve (reference pcp.py:118-197) against the reference's own output;
    the arpack case (min(m, n) > 256) checks fingerprints plus the oracle."""
    g = golden(name)
    if g["d"].size:
        d = g["d"]
    else:
        m, n, r = (int(x) for x in g["shape"])
        d = O.gaussian_rpca(m, n, r, float(g["eta"]), int(g["seed"]))[0]
    if "f32" in name:
        d = d.astype(np.float32)
    budget = int(g["svd_budget"]) or None
    st = pkg.ialm_solve(d, pkg.PcpOptions(tol_feasibility=float(g["tol"]), svd_budget=budget))
    assert abs(st.iter - int(g["iter"])) <= 1
    assert st.converged == bool(g["converged"])
    if "l" in g:
        assert relf(st.l, g["l"]) <= tolrel
        assert relf(st.s, g["s"]) <= tolrel
    else:
        assert relf(st.l[g["rows"]], g["l_rows"]) <= tolrel
        ref = O.ialm(d, tol=float(g["tol"]))
        assert relf(st.l, ref.l) <= tolrel and relf(st.s, ref.s) <= tolrel
    if st.iter == int(g["iter"]):
        assert [h.rank_l for h in st.history] == list(g["h_rank"])
        assert np.isclose(st.mu, float(g["mu"]), rtol=1e-12)


def test_ialm_edge_cases():
    z = pkg.ialm_solve(np.zeros((12, 20)))
    assert z.converged and z.iter == 1 and z.l.shape == (12, 20) and np.all(z.l == 0)
    with pytest.raises(ValueError, match="non-finite"):
        pkg.ialm_solve(np.full((10, 10), np.nan))
    d, _ = O.gaussian_rpca(40, 64, 3, 0.1, 31)
    st = pkg.ialm_solve(d, pkg.PcpOptions(max_iters=3, tol_feasibility=1e-14, rank_guess=1, svd_budget=2))
    ref = O.ialm(d, max_iters=3, tol=1e-14, rank_guess=1, svd_budget=2)
    assert st.iter == 3 and not st.converged and st.l.shape == (40, 64)
    assert [h.rank_l for h in st.history] == [h.rank_l for h in ref.history]
    assert relf(st.l, ref.l) <= 1e-10 and relf(st.y, ref.y) <= 1e-10


# ------------------------------------------------------------------ telemetry
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_singular_values_graded(dtype):
    """The two-pass spectrum resolves singular values far below sqrt(eps) of
    the largest (one Gram eigensolve would not): absolute error ~eps sigma_1."""
    rng = np.random.default_rng(7)

    def graded(m, n, s):
        u, _ = np.linalg.qr(rng.standard_normal((m, len(s))))
        v, _ = np.linalg.qr(rng.standard_normal((n, len(s))))
        return ((u * s) @ v.T).astype(dtype)

    x = graded(250, 100, np.logspace(0, -15, 100))
    ref = np.linalg.svd(x.astype(np.float64), compute_uv=False)
    got = pkg.singular_values(x)
    eps = np.finfo(dtype).eps
    assert got.shape == (100,) and np.all(np.diff(got) <= 0)
    assert np.abs(got - ref).max() <= 50 * eps * ref[0]
    # rank at numpy's default tolerance (no singular value near the threshold)
    assert pkg.matrix_rank(x) == np.linalg.matrix_rank(x)
    w = graded(160, 60, np.concatenate([np.logspace(0, -10, 30), np.zeros(30)])).T.copy()  # wide, rank 30
    assert pkg.matrix_rank(w) == np.linalg.matrix_rank(w) == (30 if dtype == np.float64 else 14)


@pytest.mark.parametrize("name", ["rank_ml_f64", "rank_full_f64", "rank_ml_f32"])
def test_collect_rank_golden(golden, name):
    """collect_rank (cpcp.py:434-439) against the reference's own rank column;
    FW-T is chaotic, so the gate is the first 30 iterations plus the final
    rank of the GPU's own L."""
    g = golden(name)
    d = g["d"].astype(np.float32) if "f32" in name else g["d"]
    opts = pkg.CpcpOptions(lambda_l=float(g["lam_l"]), lambda_s=float(g["lam_s"]), tol=float(g["tol"]),
                           max_iters=int(g["max_iters"]), levels=int(g["n_coarse"]) or None, collect_rank=True)
    fn = pkg.fwt_solve if "full" in name else pkg.ml_fwt_solve
    st = fn(d, pkg.ObservationMask(g["mask"]), opts)
    ranks = [h.rank_l for h in st.history]
    k = min(len(ranks), len(g["h_rank"]), 30)
    assert ranks[:k] == list(g["h_rank"][:k])
    tol = np.abs(np.linalg.svd(st.l.astype(np.float64), compute_uv=False)).max() * max(st.l.shape) * np.finfo(st.l.dtype).eps
    assert ranks[-1] == np.linalg.matrix_rank(st.l.astype(np.float64), tol=tol)


@pytest.mark.parametrize("name,tolrel", [("diag_pcp_f64", 1e-8), ("diag_pcp_f32", 1e-3)])
def test_collect_diagnostics_golden(golden, name, tolrel):
    """collect_diagnostics (pcp.py:298-306) against the reference's epsilon and
    delta history."""
    g = golden(name)
    d = g["d"].astype(np.float32) if "f32" in name else g["d"]
    tol = float(g["tol"]) if "tol" in g else 1e-7
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=int(g["n_coarse"]), tol_feasibility=tol,
                                             collect_diagnostics=True))
    assert st.iter == int(g["iter"])
    dg = st.diagnostics
    assert abs(dg.epsilon - float(g["epsilon"])) <= tolrel * abs(float(g["epsilon"]))
    ref = g["deltas"]
    assert len(dg.delta_history) == len(ref)
    assert np.abs(np.array(dg.delta_history) - ref).max() <= tolrel * np.abs(ref).max()
    assert dg.delta_max == max(0.0, max(ref)) or abs(dg.delta_max - max(0.0, max(ref))) <= tolrel * np.abs(ref).max()


@pytest.mark.parametrize("name", ["atoms_ml_f64", "atoms_full_f64"])
def test_oracle_atoms_golden(golden, name):
    """track_oracle_atoms (cpcp.py:355-360): one dense atom per iteration,
    equal to the reference's while the FW-T trajectories agree."""
    g = golden(name)
    nh = int(g["n_coarse"]) or None
    opts = pkg.CpcpOptions(lambda_l=float(g["lam_l"]), lambda_s=float(g["lam_s"]), tol=1e-9,
                           max_iters=int(g["max_iters"]), levels=nh, collect_rank=False, track_oracle_atoms=True)
    fn = pkg.fwt_solve if nh is None else pkg.ml_fwt_solve
    st = fn(g["d"], pkg.ObservationMask(g["mask"]), opts)
    assert st.iter == int(g["iter"]) and len(st.oracle_atoms) == st.iter
    assert all(a.shape == g["d"].shape and a.dtype == np.float64 for a in st.oracle_atoms)
    # the first two atoms agree to rounding; after that FW-T is chaotic (the
    # oracle itself moves atoms 3-5 by ~1e-3 under 1-ulp input perturbations)
    for a, ref in list(zip(st.oracle_atoms, g["atoms"]))[:2]:
        assert relf(a, ref) <= 1e-9
    for a in st.oracle_atoms:  # every atom is -radius u (R v)^T: rank one, inside the unit nuclear ball
        assert np.linalg.matrix_rank(a) <= 1 and np.linalg.norm(a) <= 1 + 1e-12
    z = fn(np.zeros((8, 6)), None, pkg.CpcpOptions(lambda_l=0.1, lambda_s=0.1, levels=None if nh is None else 3,
                                                    collect_rank=False, track_oracle_atoms=True))
    assert z.oracle_atoms is None  # P[D] = 0 early exit (cpcp.py:348-350)


# ------------------------------------------------------------------ determinism
def test_solves_are_bitwise_reproducible():
    """Every reduction has a fixed order (no atomics in the arithmetic): two
    solves of the same input agree bit for bit, PCP and CPCP."""
    d, _ = O.gaussian_rpca(300, 256, 8, 0.1, 41)
    d32 = d.astype(np.float32)
    a = pkg.ml_ialm_solve(d32, pkg.PcpOptions(levels=32, tol_feasibility=1e-6))
    b = pkg.ml_ialm_solve(d32, pkg.PcpOptions(levels=32, tol_feasibility=1e-6))
    assert a.iter == b.iter and np.array_equal(a.l, b.l) and np.array_equal(a.s, b.s) and np.array_equal(a.y, b.y)
    d2, mask = O.gaussian_rpca(400, 256, 6, 0.1, 42, observe=0.8)
    lam = 1 / np.sqrt(400)
    opts = pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / 20, tol=1e-6, max_iters=200, levels=32, collect_rank=False)
    c = pkg.ml_fwt_solve(d2, pkg.ObservationMask(mask), opts)
    e = pkg.ml_fwt_solve(d2, pkg.ObservationMask(mask), opts)
    assert c.iter == e.iter and np.array_equal(c.l, e.l) and np.array_equal(c.s, e.s)
    assert c.objective_history == e.objective_history


# ------------------------------------------------------------------ frame stacks
def _frame_files(g, tmp_path):
    blob, paths, o = g["files"].tobytes(), [], 0
    for j, n in enumerate(g["file_sizes"]):
        p = tmp_path / f"f{j}.pgm"
        p.write_bytes(blob[o:o + int(n)])
        o += int(n)
        paths.append(str(p))
    return paths


def test_ingest_emit_golden(golden, tmp_path):
    """ingest_frames / emit_frames (io.py:128-182) against the reference: the
    device-built matrix is bit-identical, the emitted PGM bytes identical."""
    g = golden("frames")
    paths = _frame_files(g, tmp_path)
    st = pkg.frames.ingest_frames(paths)
    assert (st.frame_height, st.frame_width, st.count) == (int(g["height"]), int(g["width"]), 3)
    assert np.array_equal(st.matrix, g["matrix"])
    st32 = pkg.frames.ingest_frames(paths, dtype=np.float32)
    assert np.array_equal(st32.matrix, g["matrix"].astype(np.float32))
    written = pkg.frames.emit_frames(st, g["l"], g["s"], str(tmp_path / "out"))
    assert [os.path.basename(p) for p in written] == list(g["names"])
    blob = b"".join(open(p, "rb").read() for p in written)
    assert blob == g["emitted"].tobytes()
    # ingest -> emit reproduces the input bytes exactly (io.py:164-166)
    back = pkg.frames.matrix_to_frames(st32.matrix, st.frame_height, st.frame_width)
    assert np.array_equal(back, g["raster"])


def test_video_pipeline_end_to_end(tmp_path):
    """cli.py:311-334 on the GPU: synthetic moving squares over a low-rank
    background, ingested on the device, solved by ML-FWT, emitted as PGM."""
    rng = np.random.default_rng(5)
    h, w, count = 24, 32, 40
    bg = (rng.uniform(0.2, 0.8, (h, w, 1)) * rng.uniform(0.8, 1.0, (1, 1, count)))
    stack = np.repeat(bg, 1, axis=2)
    for j in range(count):
        r0, c0 = (j // 2) % (h - 6), j % (w - 6)
        stack[r0:r0 + 6, c0:c0 + 6, j] = 1.0
    raster = np.floor(np.clip(stack, 0, 1) * 255 + 0.5).astype(np.uint8).transpose(2, 0, 1)
    paths = []
    for j in range(count):
        p = tmp_path / f"in_{j:03d}.pgm"
        pkg.frames.write_pgm(raster[j], str(p))
        paths.append(str(p))
    state, st, written = pkg.frames.video(paths, str(tmp_path / "out"), solver="ml-fwt")
    assert len(written) == 2 * count and state.iter >= 1
    m = st.matrix.cpu().numpy()
    assert m.shape == (h * w, count)
    lam = 1.0 / np.sqrt(h * w)  # the CLI defaults, computed the same way (cli.py:192-198)
    ref = pkg.ml_fwt_solve(m, None, pkg.CpcpOptions(lambda_l=lam, lambda_s=lam / np.sqrt(h * w), tol=1e-3,
                                                      max_iters=2000, collect_rank=False))
    assert ref.iter == state.iter
    assert np.array_equal(np.asarray(ref.l), state.l.cpu().numpy())
    first = pkg.frames.read_pgm(written[0])
    assert first.shape == (h, w)


# ------------------------------------------------------------------ ML-CPCP
@pytest.mark.parametrize("name", ["fwt_f64_small", "fwt_f32_small", "fwt_f64_full"])
def test_ml_fwt_golden_envelope(golden, name):
    g = golden(name)
    d = g["d"].astype(np.float32) if "f32" in name else g["d"]
    mask = pkg.ObservationMask(g["mask"]) if "mask" in g else None
    st = pkg.ml_fwt_solve(d, mask, pkg.CpcpOptions(
        lambda_l=float(g["lam_l"]), lambda_s=float(g["lam_s"]), tol=float(g["tol"]),
        max_iters=int(g["max_iters"]), levels=int(g["n_coarse"]), collect_rank=False))
    ref_obj = g["h_obj"]
    it = int(g["iter"])
    assert abs(st.objective_history[0] - ref_obj[0]) <= (1e-6 if "f32" in name else 1e-9) * ref_obj[0]
    assert abs(st.iter - it) <= max(2, int(0.05 * it))
    assert abs(st.objective_history[-1] - ref_obj[-1]) / ref_obj[-1] <= 1e-4
    assert relf(st.s, g["s"]) <= 5e-3
    assert relf(st.l, g["l"]) <= 5e-2
    obj = np.array(st.objective_history)
    assert np.all(np.diff(obj) <= 1e-9 * obj[:-1])  # exact segment search: non-increasing


@pytest.mark.parametrize("name", ["fwtfull_f64", "fwtfull_f32"])
def test_fwt_full_golden_envelope(golden, name):
    """Full-width fwt_solve against the reference's own fwt_solve output."""
    g = golden(name)
    d = g["d"].astype(np.float32) if "f32" in name else g["d"]
    mask = pkg.ObservationMask(g["mask"]) if "mask" in g else None
    st = pkg.fwt_solve(d, mask, pkg.CpcpOptions(
        lambda_l=float(g["lam_l"]), lambda_s=float(g["lam_s"]), tol=float(g["tol"]),
        max_iters=int(g["max_iters"]), collect_rank=False))
    ref_obj = g["h_obj"]
    it = int(g["iter"])
    # iteration 1 is exact; after that the trajectory is compared with the
    # envelope the oracle itself spans under 1-ulp input perturbations
    assert abs(st.objective_history[0] - ref_obj[0]) <= (1e-6 if "f32" in name else 1e-9) * ref_obj[0]
    assert abs(st.iter - it) <= max(2, 2 * int(g["env_iter"]))
    assert abs(st.objective_history[-1] - ref_obj[-1]) / ref_obj[-1] <= max(1e-4, 2 * float(g["env_obj"]))
    obj = np.array(st.objective_history)
    assert np.all(np.diff(obj) <= 1e-9 * obj[:-1])  # exact segment search: non-increasing


def test_ml_fwt_zero_observed_data():
    st = pkg.ml_fwt_solve(np.zeros((16, 12)), None, pkg.CpcpOptions(lambda_l=0.1, lambda_s=0.01, levels=6,
                                                                       collect_rank=False))
    assert st.converged and st.iter == 1 and st.objective_history == [0.0]


def test_ml_fwt_mask_shape_mismatch():
    with pytest.raises(ValueError, match="mask shape"):
        pkg.ml_fwt_solve(np.ones((8, 8)), pkg.ObservationMask(np.ones((8, 7), bool)),
                         pkg.CpcpOptions(lambda_l=0.1, lambda_s=0.1, levels=4, collect_rank=False))


@pytest.mark.parametrize("m,n", [(7, 1), (5, 31), (9, 32), (13, 33), (64, 1000), (3, 4100)])
def test_mask_pack_bitwise(m, n):
    """mlr_mask_pack (device) against ObservationMask.packed_bits (numpy
    packbits, the layout the ML-CPCP passes read): bit-exact, from a host
    boolean mask, an ObservationMask and a CUDA tensor."""
    import torch
    from paper_2206_13369_b200.cpcp import _mask_bits
    rng = np.random.default_rng(m * 1000 + n)
    obs = rng.random((m, n)) < 0.7
    want = pkg.ObservationMask(obs).packed_bits().view(np.int32)
    dev = torch.device("cuda", 0)
    for src in (obs, pkg.ObservationMask(obs), torch.from_numpy(obs).to(dev), torch.from_numpy(obs.view(np.uint8)).to(dev)):
        got = _mask_bits(src, (m, n), dev).cpu().numpy()
        assert got.dtype == np.int32 and got.shape == want.shape
        assert np.array_equal(got, want)
    rows = slice(2, m - 1)
    got = _mask_bits(obs, (m - 3, n), dev, rows).cpu().numpy()
    assert np.array_equal(got, pkg.ObservationMask(obs[rows]).packed_bits().view(np.int32))


def test_ml_fwt_device_mask_equals_host_mask():
    """A mask resident on the device gives the same solve as the host mask."""
    import torch
    rng = np.random.default_rng(5)
    d = (rng.standard_normal((96, 5)) @ rng.standard_normal((5, 80))).astype(np.float32)
    obs = rng.random(d.shape) < 0.8
    opts = pkg.CpcpOptions(lambda_l=0.3, lambda_s=0.05, levels=20, max_iters=40, collect_rank=False)
    a = pkg.ml_fwt_solve(d, pkg.ObservationMask(obs), opts)
    b = pkg.ml_fwt_solve(d, torch.from_numpy(obs).cuda(), opts)
    assert a.iter == b.iter and a.objective_history == b.objective_history
    assert np.array_equal(a.l, b.l) and np.array_equal(a.s, b.s)


# ------------------------------------------------------------------ single operators
@pytest.mark.parametrize("n,nh", [(500, 125), (101, 13), (64, 8), (33, 9)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_restrict_prolong_vs_dense(n, nh, dtype):
    ch = pkg.build_chain(n, nh)
    x = np.random.default_rng(1).standard_normal((37, n)).astype(dtype)
    r = ch.dense()
    got = pkg.restrict(x, ch)
    tol = 1e-12 if dtype == np.float64 else 1e-5
    assert relf(got, x.astype(np.float64) @ r) <= tol
    xh = np.random.default_rng(2).standard_normal((37, nh)).astype(dtype)
    assert relf(pkg.prolong(xh, ch), xh.astype(np.float64) @ r.T) <= tol


@pytest.mark.parametrize("n", [50, 128, 250, 300])
def test_jacobi_eigensolver_vs_lapack(n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n + 20, n))
    b = a.T @ a
    lam, v, sweeps = pkg.eigh_psd(b)
    ev = np.linalg.eigvalsh(b)[::-1]
    assert sweeps > 0
    assert np.abs(lam - ev).max() <= 1e-12 * ev[0]
    assert np.abs(v.T @ v - np.eye(n)).max() <= 1e-12
    assert np.linalg.norm(b @ v - v * lam) <= 1e-11 * np.linalg.norm(b)


# --------------------------------------------- rank-0 certificate (pcp.cu)
@pytest.mark.parametrize("m,n,rank,levels", [(600, 600, 30, 150),     # one-CTA register Cholesky
                                             (1200, 1200, 60, 300)])  # grid panel Cholesky (n_H > 268)
def test_rank0_certificate_matches_oracle(m, n, rank, levels, monkeypatch):
    """Iterations whose SVT keeps nothing (rank 0, pcp.py:258-262) skip the
    eigensolve after the Cholesky certificate; the per-iteration rank column
    and the iterates must still match the oracle, and the skipped iterations
    must be exactly the rank-0 ones."""
    from paper_2206_13369_b200 import pcp as P
    monkeypatch.setenv("MLR_EIG", "jacobi")  # the sweep count tells which iterations skipped the eigensolve
    d, _ = O.gaussian_rpca(m, n, rank, 0.10, 0)
    ref = O.ml_ialm(d, levels=levels, tol=1e-7)
    sink = []
    P.TIMING_SINK = sink
    try:
        st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=levels, tol_feasibility=1e-7))
    finally:
        P.TIMING_SINK = None
    ranks_ref = [h.rank_l for h in ref.history]
    ranks = [h.rank_l for h in st.history]
    assert 0 in ranks_ref, "instance has no rank-0 iteration"
    assert abs(st.iter - ref.iter) <= 1
    n_cmp = min(len(ranks), len(ranks_ref))
    assert ranks[:n_cmp] == ranks_ref[:n_cmp]
    assert relf(st.l, ref.l) <= 1e-10 and relf(st.s, ref.s) <= 1e-10
    sweeps = sink[0]["jac_sweeps"][:len(ranks)]
    assert [s == 0 for s in sweeps] == [r == 0 for r in ranks]


# ---------------------------------------- coarse eigensolvers (trd.cu / jacobi2.cu)
@pytest.mark.parametrize("eig", ["trd", "jacobi"])
@pytest.mark.parametrize("m,n,rank,levels,dtype", [(600, 600, 30, 150, np.float64),
                                                   (1200, 1200, 60, 300, np.float64),
                                                   (1400, 1300, 40, 650, np.float32)])
def test_coarse_eigensolvers_match_oracle(eig, m, n, rank, levels, dtype, monkeypatch):
    """Both coarse eigensolvers -- the tridiagonal one (Householder reduction,
    Sturm bisection, twisted-factorisation vectors, trd.cu) and the warm-started
    block Jacobi -- reproduce the reference's SVT (pcp.py:257-262) through the
    whole solve: same iterations and rank column, iterates to 1e-10 (FP64) /
    1e-4 (FP32, the reference computing in FP64 on the FP32-rounded input)."""
    monkeypatch.setenv("MLR_EIG", eig)
    d, _ = O.gaussian_rpca(m, n, rank, 0.10, 1)
    d = d.astype(dtype)
    ref = O.ml_ialm(d.astype(np.float64), levels=levels, tol=1e-6)
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=levels, tol_feasibility=1e-6))
    tol = 1e-10 if dtype == np.float64 else 1e-4
    assert abs(st.iter - ref.iter) <= (0 if dtype == np.float64 else 1)
    n_cmp = min(st.iter, ref.iter)
    assert [h.rank_l for h in st.history][:n_cmp] == [h.rank_l for h in ref.history][:n_cmp]
    assert relf(st.l, ref.l) <= tol and relf(st.s, ref.s) <= tol


def test_block_diagonal_input_matches_oracle(monkeypatch):
    """D = blockdiag(X, X): nearly repeated coarse eigenvalues (the stencil
    couples the two halves only at the group boundary), and the vectors of a
    cluster closer than 1e-10 relative would go to the Jacobi instead.  The
    tridiagonal solve must match the oracle (pcp.py:257-262)."""
    monkeypatch.setenv("MLR_EIG", "trd")
    x, _ = O.gaussian_rpca(150, 128, 6, 0.10, 4)
    d = np.zeros((300, 256))
    d[:150, :128] = x
    d[150:, 128:] = x
    ref = O.ml_ialm(d, levels=32, tol=1e-7)
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=32, tol_feasibility=1e-7))
    assert st.iter == ref.iter
    assert [h.rank_l for h in st.history] == [h.rank_l for h in ref.history]
    assert relf(st.l, ref.l) <= 1e-10 and relf(st.s, ref.s) <= 1e-10


def test_tridiagonal_failure_falls_back_to_jacobi():
    """A tridiagonal solve that reports failure (forced here through
    MLR_TRD_FORCE_FALLBACK, read at first use, so in a subprocess) hands the
    iteration to the Jacobi with V = I: same iterates as the oracle, and the
    history's sweep column shows the Jacobi ran."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_2206_13369_b200 as pkg; from paper_2206_13369_b200 import pcp as P\n"
        "from oracle import mlrpca_oracle as O\n"
        "d, _ = O.gaussian_rpca(400, 320, 8, 0.1, 6)\n"
        "ref = O.ml_ialm(d, levels=80, tol=1e-7)\n"
        "sink = []; P.TIMING_SINK = sink\n"
        "st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=80, tol_feasibility=1e-7))\n"
        "sw = sink[0]['jac_sweeps'][:st.iter]\n"
        "rl = np.linalg.norm(st.l - ref.l) / np.linalg.norm(ref.l)\n"
        "assert st.iter == ref.iter and rl <= 1e-10, (st.iter, ref.iter, rl)\n"
        "assert all(s > 0 for s, h in zip(sw, st.history) if h.rank_l > 0), sw\n"
        "assert -1 not in sw, sw\n"
        "print('ok')\n") % (ROOT, ROOT)
    env = dict(os.environ, MLR_EIG="trd", MLR_TRD_FORCE_FALLBACK="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stdout + out.stderr


@pytest.mark.parametrize("n,levels", [(140, 3), (140, 5), (140, 9), (140, 35), (140, 70), (130, 65), (264, 33)])
def test_tridiagonal_eigensolver_small_and_odd_coarse_widths(n, levels, monkeypatch):
    """The tridiagonal coarse eigensolver at tiny and odd n_H (one-CTA cluster,
    partial warps, n_H not a multiple of 32 or of the 64 padding) against the
    oracle's SVD-based SVT (pcp.py:257-262)."""
    monkeypatch.setenv("MLR_EIG", "trd")
    d, _ = O.gaussian_rpca(160, n, 3, 0.10, 9)
    ref = O.ml_ialm(d, levels=levels, tol=1e-7)
    st = pkg.ml_ialm_solve(d, pkg.PcpOptions(levels=levels, tol_feasibility=1e-7))
    assert st.iter == ref.iter
    assert [h.rank_l for h in st.history] == [h.rank_l for h in ref.history]
    assert relf(st.l, ref.l) <= 1e-10 and relf(st.s, ref.s) <= 1e-10
