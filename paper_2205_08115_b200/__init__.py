"""B200-native BAPG / hBPG Gromov-Wasserstein solver (arXiv 2205.08115).

The product is ``libgwb.so`` (C-ABI in ``include/gwb.h``: tcgen05 TF32 GEMM
chain + fused KL-projection kernels for sm_100a).  This package is the thin
Python mirror of the reference ``gw::`` interface used by tests and bench.
"""
from .api import (  # noqa: F401
    COLS, ROWS, ConfigError, Coupling, DimensionMismatchError, DistanceMatrix, DomainError,
    Graph, IterationRecord, NumericalInstabilityError, adjacency_distance, ProbabilityVector, SinkhornResult,
    SolveOptions, SolveReport, SolverConfig, UnsupportedError, ZeroSumLineError, bapg_solve,
    alignment_accuracy, bapg_solve_batched, coupling_entropy, dykstra_project, luo_tseng_residual,
    format_coupling_csv, write_coupling_csv_file,
    bpg_solve, ebpg_solve, gw_objective, hard_assignment, hbpg_solve, kl_scale, lipschitz_bound,
    marginal_infeasibility, product_coupling, sinkhorn_project, sinkhorn_project_log, solve,
    split_gap, validate, validate_inputs, version)

__all__ = [n for n in dir() if not n.startswith("_")]
