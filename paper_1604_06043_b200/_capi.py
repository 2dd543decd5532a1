"""ctypes binding of the C-ABI in include/mstab_b200.h (and mstab_b200_kernels.h).

`Lib(path)` binds any library that exports that ABI. The product library is
``paper_1604_06043_b200/libmstab_b200.so`` (sm_100a kernels); loading fails loudly when it is
missing -- there is no CPU fallback on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
PRODUCT_LIB = PKG_DIR / "libmstab_b200.so"
GEN_LIB = PKG_DIR / "libmstab_gen.so"

MSTAB_OK = 0
MEM_HOST = 0
MEM_DEVICE = 1
STATUS_CONVERGED, STATUS_MAXMV, STATUS_BREAKDOWN = 0, 1, 2
FETCH_AT_CYCLE, FETCH_AT_HALF_TOLERANCE, FETCH_MANUAL = 0, 1, 2

ERROR_NAMES = {
    -1: "Error",
    -2: "DimensionMismatch",
    -3: "ConfigError",
    -4: "FingerprintMismatch",
    -5: "StaleData",
    -6: "ParseError",
    -7: "IoError",
    -8: "SingularProjection",
    -9: "RankDeficient",
    -20: "CudaError",
    -21: "NotReal",
}


class SolverConfigC(C.Structure):
    _fields_ = [("s", C.c_int64), ("ell", C.c_int64), ("tol", C.c_double), ("max_mv", C.c_int64),
                ("true_residual_each_cycle", C.c_int32), ("_pad", C.c_int32), ("seed", C.c_uint64)]


class FetchPolicyC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("cycle", C.c_int64)]


class HistoryPointC(C.Structure):
    _fields_ = [("cycle", C.c_int64), ("mv", C.c_int64), ("level", C.c_int64), ("resnorm", C.c_double),
                ("wall_ns", C.c_int64)]


class ReportC(C.Structure):
    _fields_ = [("h_mv", C.c_int64), ("h_mv_aux", C.c_int64), ("h_rd", C.c_int64), ("cycles", C.c_int64),
                ("status", C.c_int32), ("has_fetched", C.c_int32), ("bnorm", C.c_double),
                ("final_resnorm", C.c_double), ("wall_ns_total", C.c_int64), ("history_len", C.c_int64),
                ("tau_len", C.c_int64), ("ell", C.c_int64), ("breakdown_reason", C.c_char * 128)]


class RecycleInfoC(C.Structure):
    _fields_ = [("n", C.c_int64), ("s", C.c_int64), ("level_j", C.c_int64), ("omega_count", C.c_int64),
                ("fingerprint", C.c_uint64)]


class ValidationReportC(C.Structure):
    _fields_ = [("max_deviation", C.c_double), ("sigma_min_ratio", C.c_double),
                ("low_rank_warning", C.c_int32), ("_pad", C.c_int32)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)

# (name, restype, argtypes) for every function declared in include/mstab_b200.h
ABI = [
    ("mstab_last_error", C.c_char_p, []),
    ("mstab_impl_name", C.c_char_p, []),
    ("mstab_last_error_row", C.c_int64, []),
    ("mstab_build_id", C.c_char_p, []),
    ("mstab_context_create", C.c_int, [C.c_int32, C.POINTER(_P)]),
    ("mstab_context_destroy", None, [_P]),
    ("mstab_context_synchronize", C.c_int, [_P]),
    ("mstab_context_trim", C.c_int, [_P]),
    ("mstab_operator_interior_rows", None, [_P, _I64, _I64]),
    ("mstab_context_stream", _P, [_P]),
    ("mstab_operator_create_csr", C.c_int, [_P, C.c_int64, _I64, _I64, _D, C.POINTER(_P)]),
    ("mstab_operator_destroy", None, [_P]),
    ("mstab_operator_size", C.c_int64, [_P]),
    ("mstab_operator_nnz", C.c_int64, [_P]),
    ("mstab_operator_fingerprint", C.c_uint64, [_P]),
    ("mstab_operator_apply", C.c_int, [_P, _P, _P, _P, C.c_int32]),
    ("mstab_operator_apply_adjoint", C.c_int, [_P, _P, _P, _P, C.c_int32]),
    ("mstab_precond_build", C.c_int, [C.c_int32, C.c_int64, _I64, _I64, _D, _I64, _I64, _D, _I64, _I64, _I64, _D,
                                      _I64]),
    ("mstab_operator_create_precond", C.c_int, [_P, C.c_int64, _I64, _I64, _D, C.c_int32, _I64, _I64, _D, _I64,
                                                _I64, _D, C.POINTER(_P)]),
    ("mstab_operator_precond_kind", C.c_int32, [_P]),
    ("mstab_precond_solve", C.c_int, [_P, _P, C.c_int32, _P, _P, C.c_int32]),
    ("mstab_recycle_create", C.c_int, [_P, C.c_int64, C.c_int64, _P, _P, _P, C.c_int32, _D, C.c_int64,
                                       C.c_int64, C.c_uint64, C.POINTER(_P)]),
    ("mstab_recycle_destroy", None, [_P]),
    ("mstab_recycle_info_get", C.c_int, [_P, C.POINTER(RecycleInfoC)]),
    ("mstab_recycle_download", C.c_int, [_P, _P, _D, _D, _D, _D]),
    # complex128 data: interleaved (re, im) arrays
    ("mstab_operator_create_csr_z", C.c_int, [_P, C.c_int64, _I64, _I64, _P, C.POINTER(_P)]),
    ("mstab_operator_is_complex", C.c_int32, [_P]),
    ("mstab_recycle_is_complex", C.c_int32, [_P]),
    ("mstab_result_is_complex", C.c_int32, [_P]),
    ("mstab_operator_apply_z", C.c_int, [_P, _P, _P, _P, C.c_int32]),
    ("mstab_recycle_create_z", C.c_int, [_P, C.c_int64, C.c_int64, _P, _P, _P, C.c_int32, _D, C.c_int64,
                                         C.c_int64, C.c_uint64, C.POINTER(_P)]),
    ("mstab_recycle_download_z", C.c_int, [_P, _P, _P, _P, _P, _D]),
    ("mstab_solve_z", C.c_int, [_P, _P, _P, _P, C.c_int32, C.POINTER(SolverConfigC), _P,
                                C.POINTER(FetchPolicyC), C.POINTER(_P)]),
    ("mstab_result_x_z", C.c_int, [_P, _P, _P, C.c_int32]),
    ("mstab_recycle_validate", C.c_int, [_P, _P, _P, C.POINTER(ValidationReportC)]),
    ("mstab_recycle_save", C.c_int, [_P, _P, C.c_char_p]),
    ("mstab_recycle_load", C.c_int, [_P, C.c_char_p, C.POINTER(_P)]),
    ("mstab_solve", C.c_int, [_P, _P, _P, _P, C.c_int32, C.POINTER(SolverConfigC), _P,
                              C.POINTER(FetchPolicyC), C.POINTER(_P)]),
    ("mstab_sridr_solve", C.c_int, [_P, _P, _P, _P, C.c_int32, C.POINTER(SolverConfigC), _P, C.POINTER(_P)]),
    ("mstab_bicg_solve", C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_double, C.c_int64, _P, C.POINTER(_P)]),
    ("mstab_bicgstab_solve", C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_double, C.c_int64, _P, C.POINTER(_P)]),
    ("mstab_gmres_solve", C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_double, C.c_int64, C.POINTER(_P)]),
    ("mstab_result_destroy", None, [_P]),
    ("mstab_result_report", C.c_int, [_P, C.POINTER(ReportC)]),
    ("mstab_result_x", C.c_int, [_P, _P, _P, C.c_int32]),
    ("mstab_result_history", C.c_int64, [_P, C.POINTER(HistoryPointC), C.c_int64]),
    ("mstab_result_taus", C.c_int64, [_P, _D, C.c_int64]),
    ("mstab_result_final_data", C.c_int, [_P, C.POINTER(_P)]),
    ("mstab_result_fetched", C.c_int, [_P, C.POINTER(_P)]),
    ("mstab_result_handoff", C.c_int, [_P, C.POINTER(_P)]),
]

class HostCommC(C.Structure):
    """mstab_host_comm (include/mstab_b200.h): host callbacks of a row-sharded solve."""
    ALLREDUCE = C.CFUNCTYPE(C.c_int32, C.c_void_p, _D, C.c_int64)
    ALLGATHER = C.CFUNCTYPE(C.c_int32, C.c_void_p, _D, _D, C.c_int64)
    HALO = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(_D), _I64,
                       C.c_int32, C.POINTER(C.c_int32), C.POINTER(_D), _I64)
    _fields_ = [("user", C.c_void_p), ("allreduce_sum", ALLREDUCE), ("allgather", ALLGATHER),
                ("halo_exchange", HALO)]


ABI += [
    ("mstab_nccl_unique_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("mstab_context_set_comm_nccl", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_uint8)]),
    ("mstab_context_set_comm_host", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(HostCommC)]),
    ("mstab_context_comm_info", C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("mstab_operator_create_csr_slab", C.c_int, [_P, C.c_int64, _I64, _I64, _D, _I64, C.POINTER(_P)]),
    ("mstab_operator_create_csr_slab_local", C.c_int,
     [_P, C.c_int64, _I64, _I64, _I64, _D, _I64, C.c_uint64, C.POINTER(_P)]),
    ("mstab_fnv_begin", C.c_uint64, [C.c_int64, C.c_int64, C.c_int64]),
    ("mstab_fnv_fold_index", C.c_uint64, [C.c_uint64, _I64, C.c_int64, C.c_int64]),
    ("mstab_fnv_fold_values", C.c_uint64, [C.c_uint64, _D, C.c_int64]),
    ("mstab_operator_row_begin", C.c_int64, [_P]),
    ("mstab_operator_global_size", C.c_int64, [_P]),
]


class KernelClassStatsC(C.Structure):
    _fields_ = [("launches", C.c_int64), ("total_ms", C.c_double), ("total_bytes", C.c_double)]


ABI += [
    ("mstab_harness_euler_rhs", C.c_int, [_P, C.c_int64, _P, _P, C.c_double, C.c_double, _P, C.c_int32]),
    ("mstab_harness_axpby", C.c_int, [_P, C.c_int64, _P, _P, C.c_double, _P, C.c_int32]),
    ("mstab_launch_count", C.c_uint64, []),
    ("mstab_profiling_enable", C.c_int, [C.c_int32]),
    ("mstab_profiling_read", C.c_int32, [C.POINTER(KernelClassStatsC), C.c_int32]),
    ("mstab_profiling_reset", None, []),
    ("mstab_kernel_class_name", C.c_char_p, [C.c_int32]),
]

# include/mstab_b200_kernels.h
KERNEL_ABI = [
    ("mstab_kernel_solve_small", C.c_int, [_P, C.c_int64, _D, _D, _D]),
    ("mstab_kernel_least_squares", C.c_int, [_P, C.c_int64, C.c_int64, _D, _D, _D]),
    ("mstab_kernel_cut_space", C.c_int, [_P, C.c_int64, C.c_int64, C.c_uint64, _D]),
    ("mstab_kernel_arnoldi", C.c_int, [_P, _P, _D, C.c_int64, C.c_uint64, _D, _D, _I64]),
    ("mstab_kernel_arnoldi_cb", C.c_int, [_P, _P, _D, C.c_int64, C.c_void_p, C.c_void_p, _D, _D, _I64]),
    ("mstab_kernel_bicg_projection", C.c_int, [_P, C.c_int64, C.c_int64, _D, _D, _D, _D]),
    ("mstab_kernel_projection_gram", C.c_int, [_P, C.c_int64, C.c_int64, _D, _D, _D, _D, _D]),
    ("mstab_kernel_level_iteration", C.c_int, [_P, _P, C.c_int64, C.c_int64, _D, _D, _D, _D]),
    ("mstab_kernel_poly_combination", C.c_int,
     [_P, C.c_int64, C.c_int64, C.c_int64, _D, _D, _D, _D, _D, _D, _D, _D, C.POINTER(C.c_int32)]),
]

# include/mstab_gen.h
GEN_ABI = [
    ("mstab_gen_convdiff_nnz", C.c_int64, [C.c_int32, C.c_int64, C.c_int32]),
    ("mstab_gen_convdiff", C.c_int, [C.c_int32, C.c_int64, C.c_int32, _D, C.c_double, _I64, _I64, _D]),
    ("mstab_gen_convdiff_rows", C.c_int64,
     [C.c_int32, C.c_int64, C.c_int32, _D, C.c_double, C.c_int64, C.c_int64, _I64, _I64, _D]),
    ("mstab_gen_uniform", C.c_int, [C.c_uint64, C.c_int64, _D]),
    ("mstab_gen_euler_rhs", None, [C.c_int64, _D, _D, C.c_double, C.c_double, _D]),
    ("mstab_gen_banded", C.c_int, [C.c_int64, C.c_int32, C.c_int64, C.c_uint64, _I64, _I64, _D]),
    ("mstab_gen_normal", C.c_int, [C.c_uint64, C.c_int64, _D]),
    ("mstab_gen_sinewave", None, [C.c_int64, _D]),
]


def _bind(lib, table):
    for name, res, args in table:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


class Lib:
    """A loaded implementation of the drop-in ABI."""

    _cache: dict = {}

    def __new__(cls, path=None):
        path = str(Path(path or PRODUCT_LIB).resolve())
        if path in cls._cache:
            return cls._cache[path]
        if not os.path.exists(path):
            raise RuntimeError(
                f"mstab library not found: {path} (build it with `make` / __graft_entry__.build(); "
                "there is no CPU fallback)")
        self = super().__new__(cls)
        self.path = path
        self.dll = C.CDLL(path, mode=C.RTLD_LOCAL)
        _bind(self.dll, ABI)
        _bind(self.dll, KERNEL_ABI)
        self.name = self.dll.mstab_impl_name().decode()
        self.build_id = self.dll.mstab_build_id().decode()
        cls._cache[path] = self
        return self

    def last_error(self) -> str:
        return (self.dll.mstab_last_error() or b"").decode(errors="replace")


_gen = None


def gen_lib():
    global _gen
    if _gen is None:
        if not GEN_LIB.exists():
            raise RuntimeError(f"generator library not found: {GEN_LIB} (run `make gen`)")
        _gen = C.CDLL(str(GEN_LIB), mode=C.RTLD_LOCAL)
        _bind(_gen, GEN_ABI)
    return _gen


def dptr(a):
    """double* of a contiguous float64 numpy array."""
    return a.ctypes.data_as(_D)


def i64ptr(a):
    return a.ctypes.data_as(_I64)
