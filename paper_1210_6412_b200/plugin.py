"""Register the GPU solvers into the reference package's own registry.

``mcreach.solvers.SOLVERS`` (solvers.py:494-499) is read at call time by
``reachability_probabilities`` (markov.py:276-291), ``run_sweep`` (bench.py:177-185), the
``SweepPlan`` / ``TrialRecord`` method validation (bench.py:68,131-133) and
``mcreach bench --methods`` (cli.py:45-52). After ``install()`` those callers run
``jacobi-gpu`` / ``bicgstab-gpu`` unchanged: results come back as the reference's own
``SolveResult`` and failures as its own ``ZeroDiagonal`` / ``NotConverged`` / ``Breakdown``,
so ``except SolverError`` in run_sweep keeps recording failed trials in-row.
"""

from __future__ import annotations

from . import solvers as gs
from .sparse import DimensionMismatch as _GpuDimensionMismatch


def _wrap(fn, ms, msparse):
    def convert(r):
        return ms.SolveResult(r.x, r.iterations, r.converged, r.residual_inf, r.wall_time)

    def solve(m, b, config=None):
        try:
            return convert(fn(m, b, config))
        except gs.ZeroDiagonal as err:
            raise ms.ZeroDiagonal(err.index) from None
        except gs.NotConverged as err:
            raise ms.NotConverged(convert(err.result)) from None
        except gs.Breakdown as err:
            raise ms.Breakdown(err.which, err.iteration, convert(err.result)) from None
        except _GpuDimensionMismatch as err:
            raise msparse.DimensionMismatch(str(err)) from None

    solve.__name__ = fn.__name__
    solve.__doc__ = fn.__doc__
    return solve


def install(registry=None) -> dict:
    """Add the GPU methods to ``mcreach.solvers.SOLVERS`` (or to ``registry``)."""
    import mcreach.solvers as ms
    import mcreach.sparse as msparse

    target = ms.SOLVERS if registry is None else registry
    added = {name: _wrap(fn, ms, msparse) for name, fn in gs.SOLVERS.items()}
    target.update(added)
    return added
