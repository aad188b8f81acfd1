"""B200-native PAM sweep for trace-regularized FCTN tensor completion
(arXiv 2510.22506), behind the reference `fctnlr` solver API.

`run(obs, cfg)` is the drop-in for `fctnlr.solver.run`; its sweep runs as
hand-written sm_100a kernels in `libfctn_b200.so` (C ABI: include/fctn_b200.h).
"""
from .network import FctnFactors, FctnRank, mode_fold, mode_unfold
from .shard import Shard
from .solver import IterationRecord, NumericalFailure, Observation, SolverConfig, SolverResult, run

__version__ = "0.1.0"

__all__ = [
    "FctnFactors",
    "FctnRank",
    "IterationRecord",
    "NumericalFailure",
    "Observation",
    "Shard",
    "SolverConfig",
    "SolverResult",
    "mode_fold",
    "mode_unfold",
    "run",
]
