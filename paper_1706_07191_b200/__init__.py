"""B200-native block randomized SVD (arxiv 1706.07191) -- the hot path only.

Drop-in for the reference package ``blocksvd`` on the path BASELINE.json's
north star names: the rank-k randomized SVD entry points (``rsvd_incore``,
``brsvd_run``, ``rsvd_naive_ooc``, ``block_range_finder``) and the IALM
robust-PCA solver that calls them (``ialm_rpca``), with their building blocks
(``tsqr``, ``small_svd``, ``gaussian_matrix``) and data types.  All
arithmetic runs in hand-written sm_100a CUDA kernels behind the C ABI in
include/brsvd.h; there is no CPU fallback.
"""

from .kernels import (RankDeficiencyWarning, ShapeError, SvdFactors,
                      gaussian_matrix, small_svd, tsqr, tsqr_factor)
from .rsvd import (ConfigError, SketchConfig, block_range_finder, brsvd_run,
                   relative_frobenius_error, rsvd_incore, rsvd_naive_ooc)
from .store import BlockPlan, BudgetError, MatrixStore, PassStats, plan_blocks
from .rpca import (RpcaConfig, RpcaResult, ialm_rpca, shrink,
                   spectral_norm_estimate)

__version__ = "0.1.0"

__all__ = [
    "BlockPlan", "BudgetError", "ConfigError", "MatrixStore", "PassStats",
    "RankDeficiencyWarning", "RpcaConfig", "RpcaResult", "ShapeError",
    "SketchConfig", "SvdFactors", "block_range_finder", "brsvd_run",
    "gaussian_matrix", "ialm_rpca", "plan_blocks", "relative_frobenius_error",
    "rsvd_incore", "rsvd_naive_ooc", "shrink", "small_svd",
    "spectral_norm_estimate", "tsqr", "tsqr_factor",
]
