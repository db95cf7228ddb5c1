"""Host-side product code on CPU: the stencil chain builder against the
reference's golden composites, option/type semantics, and the C-ABI library
(loads, exports every symbol include/mlr_b200.h declares; no compute)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2206_13369_b200 as pkg
from paper_2206_13369_b200 import _lib, chain as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_chain_matches_reference_composites(golden):
    g = golden("multilevel")
    for key in [k for k in g if k.startswith("R_")]:
        _, n, t = key.split("_")
        ch = C.build_chain(int(n), int(t))
        assert np.array_equal(ch.dense(), g[key]), key
        assert ch.spectral_norm == float(g[f"spec_{n}_{t}"])
    for key in [k for k in g if k.startswith("Rcsr_") and k.endswith("_data")]:
        _, n, t, _ = key.split("_")
        dense = C.build_chain(int(n), int(t)).dense()
        ptr, idx, data = g[f"Rcsr_{n}_{t}_indptr"], g[f"Rcsr_{n}_{t}_indices"], g[key]
        for j in range(0, int(n), max(1, int(n) // 257)):
            row = np.zeros(int(t))
            row[idx[ptr[j]:ptr[j + 1]]] = data[ptr[j]:ptr[j + 1]]
            assert np.array_equal(dense[j], row)


def test_chain_gram_is_tridiagonal_rtr():
    for n, t in [(500, 125), (101, 13), (64, 8), (7, 4)]:
        ch = C.build_chain(n, t)
        r = ch.dense()
        g = r.T @ r
        assert np.allclose(np.diag(g), ch.g_diag, atol=1e-15)
        assert np.allclose(np.diag(g, 1), ch.g_off, atol=1e-15)
        assert np.abs(np.triu(g, 2)).max() == 0.0
        assert abs(ch.sigma_max() - 1.0) < 1e-12


def test_chain_errors_and_levels():
    with pytest.raises(ValueError, match="not reachable"):
        C.build_chain(8, 3)
    with pytest.raises(ValueError):
        C.build_chain(0, 1)
    assert C.coarse_sizes(400) == [400, 200, 100, 50, 25, 13, 7, 4, 2, 1]
    assert C.select_levels(1024, 5, 1, 10000) == 8
    assert C.select_levels(400, 2, 1, 3072) == 4
    with pytest.raises(C.LevelError):
        C.select_levels(6, 10, 1, 100)
    with pytest.warns(RuntimeWarning):
        C.select_levels(64, 30, 1, 10)
    with pytest.raises(C.LevelError):
        C.resolve_coarse_width(64, 64, 0, 5)
    ident = C.build_chain(10, 10)
    assert np.array_equal(ident.dense(), np.eye(10))


def test_options_validate_like_reference():
    with pytest.raises(ValueError):
        pkg.PcpOptions(rho=1.0).validate()
    with pytest.raises(ValueError):
        pkg.PcpOptions(lam=-1).validate()
    with pytest.raises(ValueError):
        pkg.CpcpOptions(lambda_l=0.0, lambda_s=1.0).validate()
    with pytest.raises(ValueError):
        pkg.ml_fwt_solve(np.ones((4, 4)), None, None)


def test_mask_bit_packing():
    rng = np.random.default_rng(0)
    obs = rng.random((5, 70)) < 0.6
    words = pkg.ObservationMask(obs).packed_bits()
    assert words.shape == (5, 3) and words.dtype == np.dtype("<u4")
    for i in range(5):
        for j in range(70):
            assert bool((words[i, j >> 5] >> (j & 31)) & 1) == obs[i, j]


def test_library_loads_and_exports_header_symbols():
    lib = _lib.load()
    assert lib.mlr_version() >= 1
    header = open(os.path.join(ROOT, "include", "mlr_b200.h")).read()
    names = set(re.findall(r"\b(mlr_[a-z0-9_]+)\s*\(", header))
    assert len(names) > 30
    cdll = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(names):
        assert hasattr(cdll, name), name
    # every header symbol is bound by the Python layer (or is debug-only)
    assert names - set(_lib.EXPORTED) <= {"mlr_debug_j2prof"}


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        pkg.ml_ialm_solve(np.ones((8, 8)), pkg.PcpOptions(levels=4))


def test_product_does_not_import_oracle():
    pkg_dir = os.path.join(ROOT, "paper_2206_13369_b200")
    for fn in os.listdir(pkg_dir):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg_dir, fn)).read()
            assert "oracle" not in src.replace("oracle atoms", "").replace("oracle_atoms", ""), fn


def test_cli_bridge_rebinds_and_restores():
    import types
    from paper_2206_13369_b200 import cli_bridge, cpcp, pcp
    cpu = object()
    io = types.SimpleNamespace(ingest_frames=cpu, emit_frames=cpu, save_matrix=cpu)
    mod = types.SimpleNamespace(ialm_solve=cpu, ml_ialm_solve=cpu, fwt_solve=cpu, ml_fwt_solve=cpu,
                                _numerical_rank=cpu, io=io)
    prev = cli_bridge.install(mod)
    assert mod.ml_ialm_solve is pcp.ml_ialm_solve
    assert mod.fwt_solve is cpcp.fwt_solve and mod.ml_fwt_solve is cpcp.ml_fwt_solve
    assert mod.ialm_solve is pcp.ialm_solve and mod._numerical_rank is pkg.matrix_rank
    assert mod.io.save_matrix is cpu and mod.io.ingest_frames is not cpu  # frame I/O on the GPU, rest forwarded
    cli_bridge.uninstall(mod, prev)
    assert mod.ialm_solve is cpu and mod.ml_ialm_solve is cpu and mod.fwt_solve is cpu and mod.ml_fwt_solve is cpu
    assert mod._numerical_rank is cpu and mod.io is io


def test_cli_compare_cpu_vs_gpu_names(reference, tmp_path, capsys):
    """`mlrpca compare --solver-a ml-ialm --solver-b ml-ialm-gpu` (cli.py:336-361)
    runs the reference solver for 'a' and the bound GPU solver for 'b'; the
    GPU solvers are stand-ins here (no device), counting their calls."""
    import numpy as np
    import mlrpca.cli as cli
    from mlrpca import io as rio
    from paper_2206_13369_b200 import cli_bridge
    calls = []

    def fake(name, fn):
        def run(*a, **k):
            calls.append(name)
            return fn(*a, **k)
        return run

    gpu = {"ml_ialm_solve": fake("ml_ialm_solve", reference.ml_ialm_solve),
           "ialm_solve": fake("ialm_solve", reference.ialm_solve),
           "ml_fwt_solve": fake("ml_fwt_solve", reference.ml_fwt_solve),
           "fwt_solve": fake("fwt_solve", reference.fwt_solve)}
    d = np.random.default_rng(3).standard_normal((40, 32))
    rio.save_matrix(d, tmp_path / "d.lrml")
    prev = cli_bridge.install_side_by_side(cli, gpu)
    try:
        rc = cli.main(["compare", "--input", str(tmp_path / "d.lrml"), "--solver-a", "ml-ialm",
                       "--solver-b", "ml-ialm-gpu", "--levels", "8", "--out", str(tmp_path / "out")])
        assert rc in (0, 1)
        assert calls == ["ml_ialm_solve"]  # only 'b' ran on the (stand-in) GPU solver
        assert (tmp_path / "out" / "metrics_a.csv").exists() and (tmp_path / "out" / "metrics_b.csv").exists()
        assert cli.ml_ialm_solve is not gpu["ml_ialm_solve"]  # bindings restored after the GPU call
        out = capsys.readouterr().out
        assert "ml-ialm-gpu" in out and "ml-ialm," in out
    finally:
        for k, v in prev.items():
            setattr(cli, k, v)
