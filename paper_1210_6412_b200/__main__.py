"""``python -m paper_1210_6412_b200 <command> ...`` -- the reference CLI with the GPU solvers.

Runs ``mcreach.cli.main`` (``/root/reference/pkg/src/mcreach/cli.py:55-166``) after
``plugin.install()`` has added ``jacobi-gpu``, ``bicgstab-gpu``, ``bicgstab-gpu-exact``,
``jacobi-gpu-par`` and ``bicgstab-gpu-par`` to ``mcreach.solvers.SOLVERS``:

* ``bench --methods jacobi-gpu,bicgstab-gpu ...`` -- the reference's sweep (``run_sweep``,
  ``bench.py:167-202``) writes GPU rows in its own CSV schema; method names are validated
  against the registry at parse time (``cli.py:44-51``), so they are accepted unchanged.
* ``solve --gpu ...`` -- the reference's ``solve`` fixes its method to
  ``{jacobi,bicgstab}-{seq,par}`` (``cli.py:59-70,109``); ``--gpu`` reads the chain with the
  multithreaded reader (``formats.read_dtmc``), builds the reduced system and solves it on the
  device (``markov.reachability_probabilities``, ``jacobi-gpu`` / ``bicgstab-gpu``). Output
  and exit codes are the reference's.
* ``generate`` -- unchanged.
"""

from __future__ import annotations

import sys
from typing import Optional, Sequence


def main(argv: Optional[Sequence[str]] = None) -> int:
    import mcreach.cli as cli
    from mcreach.formats import read_dtmc
    from mcreach.markov import reachability_probabilities
    from mcreach.solvers import SolverConfig

    from . import plugin

    plugin.install()
    argv = list(sys.argv[1:] if argv is None else argv)
    use_gpu = bool(argv) and argv[0] == "solve" and "--gpu" in argv
    if use_gpu:
        argv.remove("--gpu")

    def _cmd_solve(args) -> int:  # cli.py:101-116, the whole path on the GPU with --gpu
        config = SolverConfig(tolerance=args.tol, max_iterations=args.max_iters,
                              guess_seed=args.seed, workers=args.workers)
        if use_gpu:
            from . import formats, markov
            from .solvers import SolverConfig as GpuConfig
            chain, goals = formats.read_dtmc(args.input)
            try:
                x, _ = markov.reachability_probabilities(
                    chain, goals, f"{args.method}-gpu",
                    GpuConfig(tolerance=args.tol, max_iterations=args.max_iters,
                              guess_seed=args.seed))
            except Exception as err:  # map onto the reference's SolverError for exit code 3
                from mcreach.solvers import SolverError
                from .solvers import SolverError as GpuSolverError
                if isinstance(err, GpuSolverError):
                    raise SolverError(str(err)) from None
                raise
        else:
            chain, goals = read_dtmc(args.input)
            suffix = "par" if args.parallel else "seq"
            x, _ = reachability_probabilities(chain, goals, f"{args.method}-{suffix}", config)
        print(f"{x[chain.initial]:.10g}")
        if args.full_vector:
            for state, value in enumerate(x):
                print(f"{state} {value:.10g}")
        return cli.EXIT_OK

    original = cli._cmd_solve
    cli._cmd_solve = _cmd_solve  # read by build_parser() when it wires the subcommand
    try:
        return cli.main(argv)
    finally:
        cli._cmd_solve = original  # leave the reference module as it was


if __name__ == "__main__":
    sys.exit(main())
