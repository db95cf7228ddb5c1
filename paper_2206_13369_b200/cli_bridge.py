"""Run the reference command line (``mlrpca pcp | cpcp | compare``,
reference cli.py:218-236, 336-361) on the B200 solvers.

The reference CLI calls ``ialm_solve``, ``ml_ialm_solve``, ``fwt_solve`` and
``ml_fwt_solve`` through names bound in its ``cli`` module (cli.py:22-25);
``install`` rebinds them to this package's implementations, so solver
selection, ``.lrml`` I/O and the metrics CSV stay the reference's own.

    import mlrpca.cli
    from paper_2206_13369_b200 import cli_bridge
    cli_bridge.install(mlrpca.cli)
    mlrpca.cli.main(["compare", ...])

``install`` returns the previous bindings; ``uninstall`` restores them.

``install_side_by_side`` instead keeps the reference's CPU solvers and adds
GPU names (``ialm-gpu``, ``ml-ialm-gpu``, ``fwt-gpu``, ``ml-fwt-gpu``) to the
CLI's solver tuples (cli.py:27-28), so ``mlrpca compare --solver-a ml-ialm
--solver-b ml-ialm-gpu`` runs the reference and this package on the same
input and writes both metric files (cli.py:336-361).
"""

from __future__ import annotations

from . import cpcp, frames, ops, pcp

GPU_SOLVERS = {
    "ialm_solve": pcp.ialm_solve,
    "ml_ialm_solve": pcp.ml_ialm_solve,
    "fwt_solve": cpcp.fwt_solve,
    "ml_fwt_solve": cpcp.ml_fwt_solve,
    # the summary line's rank(L) column (cli.py:210-214): full SVD -> device spectrum
    "_numerical_rank": ops.matrix_rank,
}


class _IoShim:
    """The CLI's ``io`` module with the frame-stack layout on the GPU
    (``video``: ingest_frames / emit_frames, io.py:128-182); everything else
    (.lrml, metrics CSV) forwards to the reference module unchanged."""

    def __init__(self, io_module):
        self._io = io_module

    def __getattr__(self, name):
        return getattr(self._io, name)

    @staticmethod
    def ingest_frames(paths):
        return frames.ingest_frames(paths)

    @staticmethod
    def emit_frames(stack, l, s, out_dir):
        return frames.emit_frames(stack, l, s, out_dir)


def install(cli_module, solvers=None, frame_io=True):
    """Rebind the reference CLI's solver names (and, with ``frame_io``, its
    frame ingest/emit) to the B200 implementations."""
    previous = {}
    for name, fn in (solvers or GPU_SOLVERS).items():
        if hasattr(cli_module, name):
            previous[name] = getattr(cli_module, name)
            setattr(cli_module, name, fn)
    if frame_io and hasattr(cli_module, "io") and not isinstance(cli_module.io, _IoShim):
        previous["io"] = cli_module.io
        cli_module.io = _IoShim(cli_module.io)
    return previous


def uninstall(cli_module, previous):
    for name, fn in previous.items():
        setattr(cli_module, name, fn)


GPU_SUFFIX = "-gpu"


def install_side_by_side(cli_module, solvers=None):
    """Add '<name>-gpu' solver names next to the reference's own.  A GPU name
    runs the reference's _solve_one (cli.py:218-236: same option handling,
    timing and returned fields) with the four solver names bound to this
    package for the duration of that one call."""
    gpu = dict(solvers or GPU_SOLVERS)
    previous = {"PCP_SOLVERS": cli_module.PCP_SOLVERS, "CPCP_SOLVERS": cli_module.CPCP_SOLVERS,
                "_solve_one": cli_module._solve_one}
    cli_module.PCP_SOLVERS = tuple(previous["PCP_SOLVERS"]) + tuple(
        x + GPU_SUFFIX for x in previous["PCP_SOLVERS"])
    cli_module.CPCP_SOLVERS = tuple(previous["CPCP_SOLVERS"]) + tuple(
        x + GPU_SUFFIX for x in previous["CPCP_SOLVERS"])
    cpu_solve_one = previous["_solve_one"]

    def solve_one(solver, d, mask, cfg):
        if not solver.endswith(GPU_SUFFIX):
            return cpu_solve_one(solver, d, mask, cfg)
        saved = {k: getattr(cli_module, k) for k in gpu if hasattr(cli_module, k)}
        try:
            for k in saved:
                setattr(cli_module, k, gpu[k])
            return cpu_solve_one(solver[:-len(GPU_SUFFIX)], d, mask, cfg)
        finally:
            for k, v in saved.items():
                setattr(cli_module, k, v)

    cli_module._solve_one = solve_one
    return previous
