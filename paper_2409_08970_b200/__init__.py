"""B200-native batched Fast DCT+ (arXiv 2409.08970).

Host side of the drop-in for the reference's transform path
(proj/include/dctplus/fast_transform.hpp): plan construction mirrors
DctPlusPlan / PrunedEnsemblePlan, every apply runs in the sm_100a kernels of
lib/libdctplus_b200.so through the C ABI in include/dctplus_b200.h.
"""
from ._native import (CudaFailure, DctPlusError, DomainError, InvalidArgument, LogicError,  # noqa: F401
                      RuntimeFailure, LIB_PATH)
from .dctplus import (DIST_AR, DIST_AR2D, DIST_GAUSSIAN, DIST_SYM_UNIFORM, DIST_UNIFORM,  # noqa: F401
                      DctPlusPlan, PrunedEnsemblePlan, RankOneUpdate, Result, dct2, fill_signals, forward,
                      forward_nmvp, idct2, inverse, mix_seed, path_quadratic_form, plan_dctplus, plan_pruned,
                      profile_enable, profile_reset, profile_summary, pruned_forward_all, RdoChoice, rdo_select,
                      rdo_select_batch, calibrate_prune_threshold, SpectralBasis, path_spectrum,
                      ChainedFactorization, compose_rank_k, chain_forward, ozaki_slices)

__all__ = [
    "RankOneUpdate", "DctPlusPlan", "PrunedEnsemblePlan", "Result", "plan_dctplus", "forward", "forward_nmvp",
    "inverse", "plan_pruned", "pruned_forward_all", "dct2", "idct2", "fill_signals", "mix_seed",
    "path_quadratic_form", "DctPlusError", "InvalidArgument", "DomainError", "RuntimeFailure", "LogicError",
    "CudaFailure", "RdoChoice", "rdo_select", "rdo_select_batch", "calibrate_prune_threshold",
    "SpectralBasis", "path_spectrum", "ChainedFactorization", "compose_rank_k", "chain_forward", "ozaki_slices",
]
