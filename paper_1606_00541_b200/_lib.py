"""ctypes binding of libhecsolve_b200.so (the C-ABI in include/hecsolve_c.h).

The shared library is built in-tree by ``make`` (``__graft_entry__.build()``).
Importing this module without it raises ImportError: there is no Python or CPU
fallback for the solve path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhecsolve_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
        "the B200 path has no fallback")

lib = C.CDLL(LIB_PATH)

c_int, c_ll, c_dbl, c_char_p, c_void_p = C.c_int, C.c_longlong, C.c_double, C.c_char_p, C.c_void_p
P_int, P_dbl, P_char = C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_char)
PP_int, PP_dbl = C.POINTER(P_int), C.POINTER(P_dbl)

HEC_OK, HEC_EINVAL, HEC_ERANGE, HEC_ERUNTIME, HEC_EZEROPIVOT, HEC_EOVERFLOW = range(6)
STRATEGY_AUTO, STRATEGY_LEVELS, STRATEGY_PIPELINE = 0, 1, 2


class TriOptions(C.Structure):
    _fields_ = [("strategy", c_int), ("ctas", c_int), ("threads", c_int), ("reserved", c_int * 5)]


class TriInfo(C.Structure):
    _fields_ = [("n", c_int), ("nlev", c_int), ("strategy", c_int), ("ctas", c_int),
                ("threads", c_int), ("chunks", c_int), ("nnz", c_ll), ("device_bytes", c_ll),
                ("alg_bytes", c_dbl), ("predicted_us", c_dbl), ("layout", c_int), ("group", c_int),
                ("groups", c_int), ("rows_per_lane", c_int), ("width", c_int), ("ring", c_int),
                ("halo_ring", c_int), ("inflight", c_int), ("wave_len", c_ll)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GmresConfig(C.Structure):
    _fields_ = [("restart", c_int), ("max_iters", c_int), ("rel_tol", c_dbl), ("abs_tol", c_dbl)]


class GmresReport(C.Structure):
    _fields_ = [("converged", c_int), ("iterations", c_int), ("final_relative_residual", c_dbl),
                ("solve_seconds", c_dbl), ("n_inner", c_int)]


class HecView(C.Structure):
    _fields_ = [("n_rows", c_int), ("n_cols", c_int), ("ell_width", c_int), ("ell_cols", P_int),
                ("ell_vals", P_dbl), ("csr_row_offsets", P_int), ("csr_cols", P_int), ("csr_vals", P_dbl),
                ("csr_nnz", c_ll)]


class PrepView(C.Structure):
    _fields_ = [("kind", c_int), ("n", c_int), ("reversal_applied", c_int), ("nlev", c_int),
                ("level_of", P_int), ("perm", P_int), ("inv_perm", P_int), ("level_starts", P_int),
                ("ell_width", c_int), ("ell_cols", P_int), ("ell_vals", P_dbl),
                ("csr_row_offsets", P_int), ("csr_cols", P_int), ("csr_vals", P_dbl),
                ("csr_nnz", c_ll)]


class RasPlanView(C.Structure):
    _fields_ = [("n", c_int), ("rank", c_int), ("world", c_int), ("overlap", c_int), ("n_own", c_int),
                ("n_halo", c_int), ("n_ext", c_int), ("n_send", c_int), ("own", P_int), ("halo", P_int),
                ("ext", P_int), ("send_offsets", P_int), ("send_idx", P_int), ("recv_offsets", P_int),
                ("gather", P_int), ("out_index", P_int), ("part_of", P_int)]


COMM_NONE, COMM_NCCL, COMM_CALLBACKS = 0, 1, 2
ALLREDUCE_CB = C.CFUNCTYPE(c_int, c_void_p, P_dbl, c_int)
EXCHANGE_CB = C.CFUNCTYPE(c_int, c_void_p, P_dbl, c_int, P_dbl, c_int)


class CommCallbacks(C.Structure):
    _fields_ = [("ctx", c_void_p), ("allreduce_sum", ALLREDUCE_CB), ("exchange", EXCHANGE_CB)]


class CommSpec(C.Structure):
    _fields_ = [("kind", c_int), ("rank", c_int), ("world", c_int), ("nccl_id", C.POINTER(C.c_ubyte)),
                ("callbacks", CommCallbacks)]


def _sig(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


_sig("hec_last_error", c_char_p)
_sig("hec_last_error_row", c_int)
_sig("hec_last_error_block", c_int)
_sig("hec_version", c_char_p)
_sig("hec_device_available", c_int)
# device path
_sig("hec_tri_create", c_int, c_int, c_int, c_int, P_int, P_int, c_int, P_int, P_dbl, P_int, P_int, P_dbl,
     C.POINTER(TriOptions), C.POINTER(c_void_p))
_sig("hec_tri_solve", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_tri_permute_in", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_tri_solve_ordered", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_tri_solve_wave", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_tri_permute_out", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_tri_solve_host", c_int, c_void_p, P_dbl, P_dbl)
_sig("hec_tri_query", c_int, c_void_p, C.POINTER(TriInfo))
_sig("hec_tri_solve_traced", c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, P_int)
_sig("hec_tri_destroy", c_int, c_void_p)
_sig("hec_precond_create", c_int, c_int, c_int, P_int, P_char,
     c_int, P_int, P_int, c_int, P_int, P_dbl, P_int, P_int, P_dbl,
     c_int, P_int, P_int, c_int, P_int, P_dbl, P_int, P_int, P_dbl,
     C.POINTER(TriOptions), C.POINTER(c_void_p))
_sig("hec_precond_create_local", c_int, c_int, c_int, c_int, P_int, P_int,
     c_int, P_int, P_int, c_int, P_int, P_dbl, P_int, P_int, P_dbl,
     c_int, P_int, P_int, c_int, P_int, P_dbl, P_int, P_int, P_dbl,
     C.POINTER(TriOptions), C.POINTER(c_void_p))
_sig("hec_precond_apply", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_krylov_create", c_int, c_int, C.POINTER(c_void_p))
_sig("hec_krylov_mgs", c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_krylov_scale", c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_krylov_combine", c_int, c_void_p, c_int, c_void_p, c_void_p, c_ll, c_void_p, c_void_p)
_sig("hec_krylov_add", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_krylov_sqrt", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_krylov_destroy", c_int, c_void_p)
_sig("hec_precond_apply_host", c_int, c_void_p, P_dbl, P_dbl)
_sig("hec_precond_query", c_int, c_void_p, C.POINTER(TriInfo), C.POINTER(TriInfo))
_sig("hec_precond_destroy", c_int, c_void_p)
_sig("hec_spmv_create", c_int, c_int, c_int, P_int, P_int, P_dbl, C.POINTER(c_void_p))
_sig("hec_spmv_create_hec", c_int, c_int, c_int, c_int, P_int, P_dbl, P_int, P_int, P_dbl, C.POINTER(c_void_p))
_sig("hec_spmv_run", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_spmv_residual", c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_spmv_run_host", c_int, c_void_p, P_dbl, P_dbl)
_sig("hec_spmv_destroy", c_int, c_void_p)
_sig("hec_gmres_solve", c_int, c_void_p, c_void_p, P_dbl, C.POINTER(GmresConfig), P_dbl,
     C.POINTER(GmresReport), P_dbl, c_int)
# host setup
_sig("hec_csr_create", c_int, c_int, c_int, P_int, P_int, P_dbl, C.POINTER(c_void_p))
_sig("hec_csr_from_triples", c_int, c_int, c_int, c_ll, P_int, P_int, P_dbl, C.POINTER(c_void_p))
_sig("hec_csr_view", c_int, c_void_p, P_int, P_int, C.POINTER(c_ll), PP_int, PP_int, PP_dbl)
_sig("hec_csr_destroy", c_int, c_void_p)
_sig("hec_csr_spmv_host", c_int, c_void_p, P_dbl, P_dbl, c_int)
_sig("hec_hec_from_csr", c_int, c_void_p, c_int, c_int, c_int, C.POINTER(c_void_p))
_sig("hec_hec_view_get", c_int, c_void_p, C.POINTER(HecView))
_sig("hec_hec_spmv_host", c_int, c_void_p, P_dbl, P_dbl, c_int)
_sig("hec_hec_destroy", c_int, c_void_p)
_sig("hec_gen_poisson7", c_int, c_int, c_int, c_int, C.POINTER(c_void_p))
_sig("hec_gen_poisson27", c_int, c_int, c_int, c_int, C.POINTER(c_void_p))
_sig("hec_gen_reservoir7", c_int, c_int, c_int, c_int, c_dbl, c_dbl, C.c_uint64, C.POINTER(c_void_p))
_sig("hec_permute_symmetric", c_int, c_void_p, P_int, C.POINTER(c_void_p))
_sig("hec_csr_submatrix", c_int, c_void_p, P_int, c_int, C.POINTER(c_void_p))
_sig("hec_partition_create", c_int, c_void_p, c_int, c_int, C.POINTER(c_void_p))
_sig("hec_partition_view", c_int, c_void_p, P_int, P_int, PP_int, PP_int, PP_int)
_sig("hec_partition_destroy", c_int, c_void_p)
_sig("hec_random_ordering", c_int, c_int, C.c_uint64, P_int)
_sig("hec_rcm_ordering", c_int, c_void_p, P_int)
_sig("hec_ilu0", c_int, c_void_p, C.POINTER(c_void_p), C.POINTER(c_void_p))
_sig("hec_ilu_k", c_int, c_void_p, c_int, C.POINTER(c_void_p), C.POINTER(c_void_p))
_sig("hec_ilut", c_int, c_void_p, c_int, c_dbl, C.POINTER(c_void_p), C.POINTER(c_void_p))
_sig("hec_prepare", c_int, c_void_p, c_int, c_int, c_int, C.POINTER(c_void_p))
_sig("hec_prep_view_get", c_int, c_void_p, C.POINTER(PrepView))
_sig("hec_prep_solve_host", c_int, c_void_p, P_dbl, P_dbl)
_sig("hec_prep_device", c_int, c_void_p, C.POINTER(c_void_p))
_sig("hec_serial_solve", c_int, c_void_p, c_int, P_dbl, P_dbl)
_sig("hec_prep_destroy", c_int, c_void_p)
_sig("hec_bp_build", c_int, c_void_p, c_int, c_int, c_int, c_int, c_dbl, c_int, c_int, c_int,
     C.POINTER(c_void_p))
_sig("hec_bp_dims", c_int, c_void_p, P_int, P_int, P_int)
_sig("hec_bp_maps", c_int, c_void_p, P_int, P_int, P_int, P_char)
_sig("hec_bp_prepared", c_int, c_void_p, C.POINTER(c_void_p), C.POINTER(c_void_p))
_sig("hec_bp_apply_host", c_int, c_void_p, P_dbl, P_dbl)
_sig("hec_bp_device", c_int, c_void_p, C.POINTER(c_void_p))
_sig("hec_bp_destroy", c_int, c_void_p)
# multi-GPU RAS
_sig("hec_ras_plan_create", c_int, c_void_p, c_int, c_int, c_int, C.POINTER(c_void_p))
_sig("hec_ras_plan_view_get", c_int, c_void_p, C.POINTER(RasPlanView))
_sig("hec_ras_plan_destroy", c_int, c_void_p)
_sig("hec_nccl_unique_id", c_int, C.POINTER(C.c_ubyte))
_sig("hec_nccl_version", c_int)
_sig("hec_ras_create", c_int, c_void_p, c_int, c_int, c_int, c_dbl, c_int, C.POINTER(CommSpec), C.POINTER(c_void_p))
_sig("hec_ras_get_plan", c_int, c_void_p, C.POINTER(c_void_p))
_sig("hec_ras_apply", c_int, c_void_p, c_void_p, c_void_p, c_void_p)
_sig("hec_ras_apply_host", c_int, c_void_p, P_dbl, P_dbl)
_sig("hec_ras_gmres", c_int, c_void_p, P_dbl, C.POINTER(GmresConfig), P_dbl, C.POINTER(GmresReport), P_dbl, c_int)
_sig("hec_ras_gmres_device", c_int, c_void_p, c_void_p, C.POINTER(GmresConfig), c_void_p, C.POINTER(GmresReport),
     P_dbl, c_int, c_void_p)
_sig("hec_ras_stats", c_int, c_void_p, C.POINTER(c_ll), C.POINTER(c_ll), C.POINTER(c_ll))
_sig("hec_ras_destroy", c_int, c_void_p)
_sig("hec_gmres_host", c_int, c_void_p, P_dbl, c_void_p, C.POINTER(GmresConfig), P_dbl,
     C.POINTER(GmresReport), P_dbl, c_int)

EXPORTED = [
    "hec_last_error", "hec_last_error_row", "hec_last_error_block", "hec_version", "hec_device_available",
    "hec_tri_create", "hec_tri_solve", "hec_tri_permute_in", "hec_tri_solve_ordered", "hec_tri_solve_wave", "hec_tri_permute_out", "hec_tri_solve_host", "hec_tri_query", "hec_tri_destroy",
    "hec_tri_solve_traced",
    "hec_precond_create", "hec_precond_create_local", "hec_precond_apply", "hec_precond_apply_host",
    "hec_precond_query", "hec_krylov_create", "hec_krylov_mgs", "hec_krylov_scale", "hec_krylov_combine",
    "hec_krylov_add", "hec_krylov_sqrt", "hec_krylov_destroy", "hec_csr_submatrix", "hec_partition_create",
    "hec_partition_view", "hec_partition_destroy",
    "hec_precond_destroy", "hec_spmv_create", "hec_spmv_create_hec", "hec_spmv_residual", "hec_spmv_run", "hec_spmv_run_host", "hec_spmv_destroy",
    "hec_gmres_solve", "hec_csr_create", "hec_csr_from_triples", "hec_csr_view", "hec_csr_destroy",
    "hec_csr_spmv_host", "hec_hec_from_csr", "hec_hec_view_get", "hec_hec_spmv_host", "hec_hec_destroy",
    "hec_gen_poisson7", "hec_gen_poisson27", "hec_gen_reservoir7",
    "hec_permute_symmetric", "hec_random_ordering", "hec_rcm_ordering", "hec_ilu0", "hec_ilu_k", "hec_ilut",
    "hec_prepare", "hec_prep_view_get", "hec_prep_solve_host", "hec_prep_device", "hec_serial_solve",
    "hec_prep_destroy", "hec_bp_build", "hec_bp_dims", "hec_bp_maps", "hec_bp_prepared", "hec_bp_apply_host",
    "hec_bp_device", "hec_bp_destroy", "hec_gmres_host",
    "hec_ras_plan_create", "hec_ras_plan_view_get", "hec_ras_plan_destroy", "hec_nccl_unique_id", "hec_nccl_version",
    "hec_ras_create", "hec_ras_get_plan", "hec_ras_apply", "hec_ras_apply_host", "hec_ras_gmres",
    "hec_ras_gmres_device", "hec_ras_stats", "hec_ras_destroy",
]


class HecError(RuntimeError):
    """CUDA / runtime failure inside the library (std::runtime_error)."""


class ZeroPivotError(RuntimeError):
    """Mirror of hec::ZeroPivotError(row, block) (reference errors.hpp:10-27)."""

    def __init__(self, msg, row, block):
        super().__init__(msg)
        self.row = row
        self.block = block


def check(status: int) -> None:
    if status == HEC_OK:
        return
    msg = lib.hec_last_error().decode(errors="replace")
    if status == HEC_EINVAL:
        raise ValueError(msg)
    if status == HEC_ERANGE:
        raise IndexError(msg)
    if status == HEC_EZEROPIVOT:
        raise ZeroPivotError(msg, lib.hec_last_error_row(), lib.hec_last_error_block())
    if status == HEC_EOVERFLOW:
        raise OverflowError(msg)
    raise HecError(msg)
