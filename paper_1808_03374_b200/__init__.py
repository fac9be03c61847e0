"""B200-native hot path of arxiv 1808.03374 (GKL truncated SVD of genotype
matrices): packed 2-bit genotype matvecs, device-resident Krylov bases with
CGS2 / partial reorthogonalization and thick restart, behind the reference's
``svdl`` / ``LinearOperator`` interface. See DESIGN.md.

Importing requires the in-tree libgkb.so (sm_100a); there is no CPU fallback.
"""
from ._lib import FormatError, GkbError, LogicError, LIB_PATH
from .gkl import (bed_check, Context, DenseOperator, GenotypeOperator, GklOptions, LanczosFactorization,
                  LinearOperator, ReorthMode, RestartMode, RitzSet, ScalingScheme, StepInfo,
                  StepStatus, SvdlResult, SvdlStats, cgs2, default_context, error_metric_l1, geno_plan,
                  marker_scaling, norm_estimate, adjoint_mismatch, partition_rows, pinned_empty,
                  rng_uniform_symmetric, svd_small, svdl)

__all__ = [
    "FormatError", "GkbError", "LogicError", "LIB_PATH", "Context", "DenseOperator",
    "GenotypeOperator", "GklOptions", "LanczosFactorization", "LinearOperator", "ReorthMode",
    "RestartMode", "RitzSet", "ScalingScheme", "StepInfo", "StepStatus", "SvdlResult", "SvdlStats",
    "cgs2", "default_context", "error_metric_l1", "geno_plan", "marker_scaling", "partition_rows",
    "pinned_empty", "rng_uniform_symmetric", "svd_small", "svdl", "bed_check", "norm_estimate",
    "adjoint_mismatch",
]
