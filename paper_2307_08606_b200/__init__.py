"""paper_2307_08606_b200 -- B200-native ASADMM iteration loop (arXiv 2307.08606).

Drop-in for the reference ``radmm`` solver entry points: ``run``,
``Hyperparams``, ``Problem``/``ForwardOperator``, ``RunResult``/
``ConvergenceReport``, ``soft_threshold``, ``factorize``/``solve_local``,
and ``run_distributed`` (sensor sharding over NCCL).  All compute runs in
hand-written sm_100a kernels in ``libradmm_b200.so`` (built in-tree by
``__graft_entry__.build()``).
"""
from .api import (  # noqa: F401
    ConvergenceReport, CudaError, ForwardOperator, Hyperparams, InvalidArgument, IterationRecord,
    IterationView, LocalSolveCache, Mode, NumericalError, Problem, RunResult, Solver, TransportError,
    contribution_size, factorize, mode_name, nmse_db, objective_value, relative_l2_diff, run,
    soft_threshold, solve_local)

__all__ = [n for n in dir() if not n.startswith("_")]
