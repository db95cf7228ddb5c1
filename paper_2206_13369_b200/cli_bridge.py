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

from . import cpcp, pcp

GPU_SOLVERS = {
    "ialm_solve": pcp.ialm_solve,
    "ml_ialm_solve": pcp.ml_ialm_solve,
    "fwt_solve": cpcp.fwt_solve,
    "ml_fwt_solve": cpcp.ml_fwt_solve,
}


def install(cli_module, solvers=None):
    """Rebind the reference CLI's solver names to the B200 implementations."""
    previous = {}
    for name, fn in (solvers or GPU_SOLVERS).items():
        if hasattr(cli_module, name):
            previous[name] = getattr(cli_module, name)
            setattr(cli_module, name, fn)
    return previous


def uninstall(cli_module, previous):
    for name, fn in previous.items():
        setattr(cli_module, name, fn)
