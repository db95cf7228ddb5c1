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
