"""ctypes binding of libgkb.so (include/gkb.h).

The shared library is built in-tree (``python __graft_entry__.py`` or
``make -C paper_1808_03374_b200/csrc``). There is no fallback: importing
the package without the library raises, so every caller runs the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GKB_LIB", os.path.join(_HERE, "libgkb.so"))  # GKB_LIB: A/B builds

GKB_OK, GKB_EINVAL, GKB_ELOGIC, GKB_ECUDA, GKB_ENCCL, GKB_EOOM, GKB_EFORMAT = range(7)


class GkbError(RuntimeError):
    """Device / NCCL / internal failure reported by libgkb."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[gkb status {code}] {msg}")
        self.code = code


class FormatError(RuntimeError):
    """Malformed or truncated input file (genio.hpp:14-17)."""


class gkb_gkl_options(C.Structure):
    _fields_ = [
        ("k", C.c_int64),
        ("tol", C.c_double),
        ("max_mvps", C.c_int64),
        ("reorth", C.c_int),
        ("omega", C.c_double),
        ("one_sided", C.c_int),
        ("restart", C.c_int),
        ("max_subspace", C.c_int64),
        ("keep", C.c_int64),
        ("seed", C.c_uint64),
        ("record_history", C.c_int),
        ("omega_recurrence", C.c_int),
    ]


class gkb_svdl_result(C.Structure):
    _fields_ = [
        ("m", C.c_int64),
        ("n", C.c_int64),
        ("count", C.c_int64),
        ("singvals", C.POINTER(C.c_double)),
        ("U", C.POINTER(C.c_double)),
        ("V", C.POINTER(C.c_double)),
        ("err_estimates", C.POINTER(C.c_double)),
        ("converged", C.POINTER(C.c_int32)),
        ("mvps", C.c_int64),
        ("steps", C.c_int64),
        ("restarts", C.c_int32),
        ("reorth_count", C.c_int32),
        ("deflations", C.c_int32),
        ("all_converged", C.c_int32),
        ("wall_seconds", C.c_double),
        ("history_len", C.c_int64),
        ("ritz_history", C.POINTER(C.c_double)),
        ("err_history", C.POINTER(C.c_double)),
        ("device_seconds", C.c_double),
        ("host_syncs", C.c_int64),
        ("fused_tails", C.c_int64),
    ]


class gkb_subspace_result(C.Structure):
    _fields_ = [
        ("m", C.c_int64),
        ("k", C.c_int64),
        ("basis", C.POINTER(C.c_double)),
        ("eigvals", C.POINTER(C.c_double)),
        ("singvals", C.POINTER(C.c_double)),
        ("iterations", C.c_int64),
        ("delta_history", C.POINTER(C.c_double)),
        ("invcond_history", C.POINTER(C.c_double)),
        ("converged", C.c_int32),
        ("rank_deficient", C.c_int32),
        ("mvps", C.c_int64),
    ]


class gkb_synth_spec(C.Structure):
    _fields_ = [
        ("p", C.c_int64),
        ("n", C.c_int64),
        ("seed", C.c_uint64),
        ("npop", C.c_int),
        ("freq", C.POINTER(C.c_double)),
        ("pop", C.POINTER(C.c_int32)),
        ("admix", C.POINTER(C.c_double)),
        ("missing_rate", C.c_double),
        ("copy_from", C.POINTER(C.c_int32)),
        ("copy_prob", C.c_double),
    ]


P = C.c_void_p
PD = C.POINTER(C.c_double)
PI64 = C.POINTER(C.c_int64)
PI32 = C.POINTER(C.c_int32)
PU8 = C.POINTER(C.c_uint8)
I = C.c_int
I64 = C.c_int64
D = C.c_double

# gkb_host_allreduce_fn: void (*)(void* user, double* buf, int64_t count)
HOST_ALLREDUCE_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.c_int64)

# name -> (restype, argtypes); every symbol declared in include/gkb.h
SIGNATURES = {
    "gkb_last_error": (C.c_char_p, []),
    "gkb_version": (C.c_char_p, []),
    "gkb_init": (I, [I, C.POINTER(C.c_int), C.POINTER(P)]),
    "gkb_nccl_unique_id": (I, [PU8]),
    "gkb_init_nccl": (I, [I, PU8, I, I, C.POINTER(P)]),
    "gkb_init_host_comm": (I, [I, I, I, HOST_ALLREDUCE_FN, P, C.POINTER(P)]),
    "gkb_destroy": (I, [P]),
    "gkb_ctx_info": (I, [P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "gkb_synchronize": (I, [P]),
    "gkb_partition_rows": (I, [I64, I, PI64]),
    "gkb_geno_from_bed": (I, [P, PU8, I64, I64, C.POINTER(P)]),
    "gkb_geno_from_synth": (I, [P, C.POINTER(gkb_synth_spec), C.POINTER(P)]),
    "gkb_bed_check": (I, [C.c_char_p, C.c_char_p, C.c_char_p, PI64, PI64]),
    "gkb_geno_from_bed_file": (I, [P, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(P)]),
    "gkb_geno_counts": (I, [P, PI64]),
    "gkb_geno_standardize": (I, [P, I]),
    "gkb_geno_set_scaling": (I, [P, PD, PD]),
    "gkb_geno_get_scaling": (I, [P, PD, PD]),
    "gkb_geno_read_bed": (I, [P, I64, I64, PU8]),
    "gkb_geno_info": (I, [P, PI64, PI64, PI64]),
    "gkb_dense_create": (I, [P, PD, I64, I64, C.POINTER(P)]),
    "gkb_op_shape": (I, [P, PI64, PI64]),
    "gkb_op_apply": (I, [P, PD, PD]),
    "gkb_op_apply_adjoint": (I, [P, PD, PD]),
    "gkb_op_mvps": (I64, [P]),
    "gkb_op_apply_block": (I, [P, PD, I64, PD]),
    "gkb_op_apply_adjoint_block": (I, [P, PD, I64, PD]),
    "gkb_rng_fill_normal": (I, [C.c_uint64, I64, PD]),
    "gkb_host_alloc": (I, [C.c_size_t, C.POINTER(P)]),
    "gkb_host_free": (I, [P]),
    "gkb_op_destroy": (I, [P]),
    "gkb_op_bench": (I, [P, I, I, I, PD, PD, C.POINTER(C.c_int)]),
    "gkb_gkl_options_default": (None, [C.POINTER(gkb_gkl_options)]),
    "gkb_gkl_options_validate": (I, [C.POINTER(gkb_gkl_options), I64, I64]),
    "gkb_svdl": (I, [P, C.POINTER(gkb_gkl_options), C.POINTER(C.POINTER(gkb_svdl_result))]),
    "gkb_svdl_result_free": (I, [C.POINTER(gkb_svdl_result)]),
    "gkb_geno_marker_scan": (I, [P, PD, PD, I64, I, PD, PD, PD, PD, C.POINTER(C.c_int32)]),
    "gkb_subspace_qr": (I, [P, I64, C.c_double, I64, C.c_uint64, I,
                            C.POINTER(C.POINTER(gkb_subspace_result))]),
    "gkb_subspace_result_free": (I, [C.POINTER(gkb_subspace_result)]),
    "gkb_lanczos_create": (I, [P, I64, PD, C.c_uint64, C.POINTER(P)]),
    "gkb_lanczos_destroy": (I, [P]),
    "gkb_bidiag_step": (I, [P, C.POINTER(gkb_gkl_options), D, C.POINTER(C.c_int),
                            C.POINTER(C.c_int), C.POINTER(C.c_int), PD, PD]),
    "gkb_lanczos_info": (I, [P, PI64, PI64, C.POINTER(C.c_int)]),
    "gkb_lanczos_get": (I, [P, PD, PD, PD, PD, PD, PD]),
    "gkb_ritz_extract": (I, [P, D, PD, PD, PD, PD, PD, PI32]),
    "gkb_thick_restart": (I, [P, I64]),
    "gkb_compress_exhausted": (I, [P]),
    "gkb_deflate_right": (I, [P]),
    "gkb_geno_plan": (I, [I64, I64, D, I64, C.POINTER(C.c_int), PI64, PI64]),
    "gkb_geno_layouts": (I, [P, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "gkb_cgs2": (I, [P, PD, I64, I64, PD, PD, PD]),
    "gkb_svd_small": (I, [PD, I64, I64, PD, PD, PD]),
    "gkb_rng_fill_symmetric": (I, [C.c_uint64, I64, PD]),
    "gkb_marker_scaling": (I, [PI64, I64, I64, I, PD, PD]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"libgkb.so not found at {path}: build it with `python __graft_entry__.py` "
            "(make -C paper_1808_03374_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()


def check(status: int) -> None:
    """Raise the reference's exception type for a libgkb status code."""
    if status == GKB_OK:
        return
    msg = lib.gkb_last_error().decode(errors="replace")
    if status == GKB_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status == GKB_ELOGIC:
        raise LogicError(msg)
    if status == GKB_EFORMAT:
        raise FormatError(msg)
    raise GkbError(status, msg)


class LogicError(RuntimeError):
    """std::logic_error (gkl.cpp:215-218, :344)."""
