"""B200-native BDDC-preconditioned CG (arXiv 2410.14786 hot path).

Host C++ setup + hand-written sm_100a CUDA kernels behind the C-ABI in
include/bddc_b200.h; this package is the thin Python mirror of the reference API.
"""
from ._lib import BddcError, InvalidArgument, OutOfRange, lib  # noqa: F401
from .solver import (HostSetup, Preconditioner, Problem, RankPlan, SolveReport, SolverOptions,  # noqa: F401
                     dist_unique_id, pcg)

__all__ = ["Problem", "Preconditioner", "HostSetup", "RankPlan", "SolverOptions", "SolveReport", "pcg",
           "dist_unique_id",
           "BddcError", "InvalidArgument", "OutOfRange", "lib"]
