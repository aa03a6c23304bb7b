"""paper_2105_14088_b200 -- B200-native rank-reordering solver.

A drop-in for the hot path of the reference "rankweave" (arXiv 2105.14088,
cloud-aware collectives): cost-model evaluation of VM orders (ring,
halving-doubling, double binary tree, BCube) and the searches over them
(exhaustive, simulated annealing, local search), computed by hand-written
sm_100a kernels in librankweave_b200.so behind the C ABI in
include/rankweave_c.h.
"""
from .api import *  # noqa: F401,F403
from .api import (Algorithm, CollectiveSpec, CostMatrix, CostMode, DistributionStats, DomainError, HdPairing,
                  Problem, RankOrder, RankweaveError, SolveMethod, Solution, SolverConfig)
from . import fixtures  # noqa: F401

__all__ = [
    "Algorithm", "CollectiveSpec", "CostMatrix", "CostMode", "DistributionStats", "DomainError", "HdPairing",
    "Problem", "RankOrder", "RankweaveError", "SolveMethod", "Solution", "SolverConfig", "fixtures",
]
