"""Python mirror of the reference's proj/core solver interface, over the C-ABI.

Same names, argument meaning and error behaviour as the reference
(``mstab::idrstab_solve`` / ``mstab_solve`` in proj/core/include/mstab/solvers/idrstab.hpp:88-96,
``SolverConfig``/``SolveReport`` in report.hpp:24-58, ``RecycleData``/``FetchPolicy``/
``validate``/``save``/``load`` in recycle.hpp:18-64, the error classes of errors.hpp), so the
tests read like the reference's own GTest suites. Arrays are real float64 numpy vectors on the
host, or CUDA tensors (anything with ``__cuda_array_interface__`` / ``data_ptr``) on the device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional

import numpy as np

from . import _capi
from ._capi import Lib, dptr, i64ptr


# ---- errors (errors.hpp:9-72) -----------------------------------------------------------------
class Error(RuntimeError):
    pass


class BreakdownError(Error):
    pass


class DimensionMismatch(Error):
    pass


class SingularProjection(BreakdownError):
    pass


class RankDeficient(BreakdownError):
    pass


class FingerprintMismatch(Error):
    pass


class StaleData(Error):
    pass


class ParseError(Error):
    pass


class IoError(Error):
    pass


class ConfigError(Error):
    pass


class CudaError(Error):
    pass


class NotReal(ConfigError):
    pass


class ZeroPivot(Error):
    """errors.hpp:39-45 (build_jacobi / build_ilu0); `row` is ZeroPivot::row()."""
    row: int = -1


class MissingOmegas(Error):
    """errors.hpp:56-58 (sridr_solve without the donor's relaxation history)."""


_ERR = {-1: Error, -2: DimensionMismatch, -3: ConfigError, -4: FingerprintMismatch, -5: StaleData,
        -6: ParseError, -7: IoError, -8: SingularProjection, -9: RankDeficient, -20: CudaError,
        -21: NotReal, -10: ZeroPivot, -11: MissingOmegas}


def _check(lib: Lib, rc: int):
    if rc != 0:
        e = _ERR.get(rc, Error)(lib.last_error())
        if rc == -10:
            e.row = int(lib.dll.mstab_last_error_row())
        raise e


# ---- config / report (report.hpp) -------------------------------------------------------------
@dataclass
class SolverConfig:
    s: int = 2
    ell: int = 1
    tol: float = 1e-8
    max_mv: int = 100000
    true_residual_each_cycle: bool = False
    seed: int = 0

    def _c(self):
        return _capi.SolverConfigC(int(self.s), int(self.ell), float(self.tol), int(self.max_mv),
                                   1 if self.true_residual_each_cycle else 0, 0, int(self.seed) & (2**64 - 1))


@dataclass
class FetchPolicy:
    kind: int = _capi.FETCH_MANUAL
    cycle: int = 0

    @staticmethod
    def at_cycle(k: int) -> "FetchPolicy":
        if k < 1:
            raise ConfigError("fetch policy: cycle >= 1 required")
        return FetchPolicy(_capi.FETCH_AT_CYCLE, int(k))

    @staticmethod
    def at_half_tolerance() -> "FetchPolicy":
        return FetchPolicy(_capi.FETCH_AT_HALF_TOLERANCE, 0)

    @staticmethod
    def manual() -> "FetchPolicy":
        return FetchPolicy(_capi.FETCH_MANUAL, 0)


CONVERGED, MAXMV, BREAKDOWN = "Converged", "MaxMV", "Breakdown"
_STATUS = {0: CONVERGED, 1: MAXMV, 2: BREAKDOWN}


@dataclass
class HistoryPoint:
    cycle: int
    mv: int
    level: int
    resnorm: float
    wall_ns: int


@dataclass
class SolveReport:
    residual_history: List[HistoryPoint] = field(default_factory=list)
    omega_history: List[np.ndarray] = field(default_factory=list)  # tau per cycle
    h_mv: int = 0
    h_mv_aux: int = 0
    h_rd: int = 0
    cycles: int = 0
    status: str = MAXMV
    breakdown_reason: str = ""
    bnorm: float = 0.0
    final_resnorm: float = 0.0
    wall_ns_total: int = 0

    def total_mv(self) -> int:
        return self.h_mv + self.h_mv_aux


@dataclass
class ValidationReport:
    max_deviation: float
    sigma_min_ratio: float
    low_rank_warning: bool


# ---- context ----------------------------------------------------------------------------------
class Context:
    """Device + stream binding of one implementation (``mstab_context``)."""

    def __init__(self, lib: Optional[Lib] = None, device: int = 0):
        self.lib = lib if lib is not None else Lib()
        h = C.c_void_p()
        _check(self.lib, self.lib.dll.mstab_context_create(int(device), C.byref(h)))
        self.h = h

    def trim(self):
        """Release the cached cycle workspace, graphs and result blocks (mstab_context_trim)."""
        _check(self.lib, self.lib.dll.mstab_context_trim(self.h))

    def synchronize(self):
        _check(self.lib, self.lib.dll.mstab_context_synchronize(self.h))

    @property
    def stream(self) -> int:
        return self.lib.dll.mstab_context_stream(self.h) or 0

    # ---- row-sharded solves (include/mstab_b200.h) --------------------------
    @staticmethod
    def nccl_unique_id(lib: Optional[Lib] = None) -> bytes:
        lib = lib if lib is not None else Lib()
        buf = (C.c_uint8 * 128)()
        _check(lib, lib.dll.mstab_nccl_unique_id(buf))
        return bytes(buf)

    def set_comm_nccl(self, rank: int, world: int, unique_id: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(self.lib, self.lib.dll.mstab_context_set_comm_nccl(self.h, int(rank), int(world), buf))

    def set_comm_host(self, rank: int, world: int, comm):
        """`comm` provides allreduce_sum(buf), allgather(inp, out) and halo_exchange(sends, recvs)
        on numpy float64 arrays (sends / recvs: lists of (peer, array)); see TorchHostComm."""
        self._host_comm = _HostCommAdaptor(comm)  # keeps the ctypes callbacks alive
        _check(self.lib, self.lib.dll.mstab_context_set_comm_host(self.h, int(rank), int(world),
                                                                  C.byref(self._host_comm.c)))

    def comm_info(self):
        r, w = C.c_int32(), C.c_int32()
        _check(self.lib, self.lib.dll.mstab_context_comm_info(self.h, C.byref(r), C.byref(w)))
        return r.value, w.value

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.dll.mstab_context_destroy(self.h)
            self.h = None


class _HostCommAdaptor:
    """ctypes trampolines from mstab_host_comm to a Python communicator object."""

    def __init__(self, comm):
        self.comm = comm
        arr = np.ctypeslib.as_array

        def allreduce(_u, buf, count):
            try:
                self.comm.allreduce_sum(arr(buf, shape=(count,)))
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as a failed callback
                return 1

        def allgather(_u, inp, out, count):
            try:
                w = self.comm.world
                self.comm.allgather(arr(inp, shape=(count,)), arr(out, shape=(count * w,)))
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def halo(_u, ns, speers, sbufs, scounts, nr, rpeers, rbufs, rcounts):
            try:
                sends = [(int(speers[i]), arr(sbufs[i], shape=(int(scounts[i]),))) for i in range(ns)]
                recvs = [(int(rpeers[i]), arr(rbufs[i], shape=(int(rcounts[i]),))) for i in range(nr)]
                self.comm.halo_exchange(sends, recvs)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self._fns = (_capi.HostCommC.ALLREDUCE(allreduce), _capi.HostCommC.ALLGATHER(allgather),
                     _capi.HostCommC.HALO(halo))
        self.c = _capi.HostCommC(None, *self._fns)


class TorchHostComm:
    """Host communicator over an initialised torch.distributed process group (gloo on CPU):
    the staging side of a row-sharded solve for runtimes without NCCL (and the multi-rank tests,
    which run every rank on one GPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def allreduce_sum(self, buf):
        import torch
        t = torch.from_numpy(buf)
        self.dist.all_reduce(t, group=self.group)

    def allgather(self, inp, out):
        import torch
        n = inp.size
        outs = [torch.from_numpy(out[r * n:(r + 1) * n]) for r in range(self.world)]
        self.dist.all_gather(outs, torch.from_numpy(inp.copy()), group=self.group)

    def halo_exchange(self, sends, recvs):
        import torch
        reqs = [self.dist.isend(torch.from_numpy(a.copy()), p, group=self.group) for p, a in sends]
        reqs += [self.dist.irecv(torch.from_numpy(b), p, group=self.group) for p, b in recvs]
        for r in reqs:
            r.wait()


_default_ctx: dict = {}


def default_context(lib: Optional[Lib] = None) -> Context:
    lib = lib if lib is not None else Lib()
    if lib.path not in _default_ctx:
        _default_ctx[lib.path] = Context(lib)
    return _default_ctx[lib.path]


def _f64(a) -> np.ndarray:
    a = np.asarray(a)
    if np.iscomplexobj(a):
        if np.any(a.imag != 0):
            raise NotReal("complex data passed to a real fp64 entry point")
        a = a.real
    return np.ascontiguousarray(a, dtype=np.float64)


def _is_complex(a) -> bool:
    """Host data with a nonzero imaginary part (the reference's !is_real, types.cpp:25-29)."""
    if a is None or hasattr(a, "is_cuda") or hasattr(a, "__cuda_array_interface__"):
        return False
    a = np.asarray(a)
    return bool(np.iscomplexobj(a) and np.any(a.imag != 0))


def _c128(a) -> np.ndarray:
    """Contiguous complex128 copy: its memory is the interleaved (re, im) layout of the *_z ABI."""
    return np.ascontiguousarray(np.asarray(a), dtype=np.complex128)


def _dev_ptr(a, n=None, ctx=None, what="vector"):
    """(pointer, mem) for a numpy array (pointer None: the caller converts it) or a CUDA array.

    A device array must be a contiguous float64 vector of `n` entries (the C-ABI takes a raw
    pointer, so a float32 or short tensor would be read out of bounds). When `ctx` is given the
    library's stream is ordered after torch's current stream, so a vector that a torch kernel is
    still producing is not read early (the library syncs its own stream before returning)."""
    if a is None:
        return None, _capi.MEM_HOST
    if hasattr(a, "is_cuda") and a.is_cuda:
        import torch
        if a.dtype != torch.float64:
            raise ConfigError(f"{what}: device tensor must be float64, got {a.dtype}")
        if not a.is_contiguous():
            raise ConfigError(f"{what}: device tensor must be contiguous")
        if n is not None and a.numel() != n:
            raise DimensionMismatch(f"{what}: {a.numel()} entries, expected {n}")
        if ctx is not None and ctx.stream:
            torch.cuda.ExternalStream(ctx.stream, device=a.device).wait_stream(torch.cuda.current_stream(a.device))
        return a.data_ptr(), _capi.MEM_DEVICE
    if hasattr(a, "__cuda_array_interface__"):
        cai = a.__cuda_array_interface__
        if cai.get("typestr") != "<f8":
            raise ConfigError(f"{what}: device array must be float64, got {cai.get('typestr')}")
        if cai.get("strides") not in (None, (8,)):
            raise ConfigError(f"{what}: device array must be contiguous")
        cnt = int(np.prod(cai["shape"]))
        if n is not None and cnt != n:
            raise DimensionMismatch(f"{what}: {cnt} entries, expected {n}")
        return cai["data"][0], _capi.MEM_DEVICE
    return None, _capi.MEM_HOST


# ---- matrices / operators (csr.hpp, operator.hpp) ---------------------------------------------
class CsrMatrix:
    """Compressed sparse row matrix (csr.hpp:17-52), real fp64 values, int64 indices."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        # complex values (types.hpp:11-15) are kept as complex128 and routed to the *_z entry points
        self.values = _c128(values) if _is_complex(values) else _f64(values)

    def is_real(self) -> bool:
        return not np.iscomplexobj(self.values)

    def nnz(self) -> int:
        return int(self.values.size)

    @staticmethod
    def from_triplets(n_rows, n_cols, triplets):
        """Duplicates are summed (csr.cpp:53-79)."""
        d = {}
        for i, j, v in triplets:
            if not (0 <= i < n_rows and 0 <= j < n_cols):
                raise Error("from_triplets: index out of range")
            d[(i, j)] = d.get((i, j), 0.0) + v
        keys = sorted(d)
        rp = np.zeros(n_rows + 1, dtype=np.int64)
        for i, _ in keys:
            rp[i + 1] += 1
        rp = np.cumsum(rp)
        return CsrMatrix(n_rows, n_cols, rp, [j for _, j in keys], [d[k] for k in keys])

    @staticmethod
    def identity(n):
        return CsrMatrix(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    @staticmethod
    def tridiag(a, b, c, n):
        """a on the sub-, b on the main, c on the super-diagonal (csr.cpp:92-101)."""
        t = []
        for i in range(n):
            if i > 0:
                t.append((i, i - 1, a))
            t.append((i, i, b))
            if i + 1 < n:
                t.append((i, i + 1, c))
        return CsrMatrix.from_triplets(n, n, t)

    @staticmethod
    def from_dense(m):
        m = np.asarray(m)
        m = m.astype(np.complex128) if _is_complex(m) else np.asarray(m.real if np.iscomplexobj(m) else m, dtype=np.float64)
        n = m.shape[0]
        t = [(i, j, m[i, j]) for i in range(n) for j in range(m.shape[1])]
        return CsrMatrix.from_triplets(n, m.shape[1], t)

    def to_dense(self):
        d = np.zeros((self.n_rows, self.n_cols), dtype=self.values.dtype)
        for i in range(self.n_rows):
            for k in range(self.row_ptr[i], self.row_ptr[i + 1]):
                d[i, self.col_idx[k]] = self.values[k]
        return d


class CsrOperator:
    """LinearOperator over a CSR matrix (operator.hpp:33-50); uploaded once, fingerprint cached."""

    def __init__(self, a: CsrMatrix, ctx: Optional[Context] = None, slabs=None):
        """`slabs` (world + 1 ascending row boundaries) makes this the row slab of the context's
        rank in a row-sharded solve (the context needs a communicator first)."""
        if a.n_rows != a.n_cols:
            raise DimensionMismatch("CsrOperator: square matrix required")
        self.ctx = ctx if ctx is not None else default_context()
        self.lib = self.ctx.lib
        self.matrix = a
        self._ztwin = None
        self._z = not a.is_real()  # the handle is a complex operator (*_z entry points)
        h = C.c_void_p()
        if not a.is_real():
            if slabs is not None:
                raise ConfigError("b200: the complex path is single-GPU")
            _check(self.lib, self.lib.dll.mstab_operator_create_csr_z(
                self.ctx.h, a.n_rows, i64ptr(a.row_ptr), i64ptr(a.col_idx), a.values.ctypes.data, C.byref(h)))
        elif slabs is None:
            _check(self.lib, self.lib.dll.mstab_operator_create_csr(
                self.ctx.h, a.n_rows, i64ptr(a.row_ptr), i64ptr(a.col_idx), dptr(a.values), C.byref(h)))
        else:
            self._slabs = np.ascontiguousarray(slabs, dtype=np.int64)
            _check(self.lib, self.lib.dll.mstab_operator_create_csr_slab(
                self.ctx.h, a.n_rows, i64ptr(a.row_ptr), i64ptr(a.col_idx), dptr(a.values),
                i64ptr(self._slabs), C.byref(h)))
        self.h = h

    @classmethod
    def from_local_rows(cls, n_global: int, slabs, row_ptr, col_idx, values, col_spans, fingerprint: int,
                        ctx: Context) -> "CsrOperator":
        """Row slab of the context's rank from the rank's OWN rows (row_ptr from 0, GLOBAL column
        indices): no rank holds the global matrix. `col_spans` (world x 2) are the column ranges every
        rank's rows reference (`local_col_span` on each rank, allgathered); `fingerprint` is the
        global reference checksum (`distributed_fingerprint`)."""
        self = cls.__new__(cls)
        self.ctx, self.lib, self.matrix = ctx, ctx.lib, None
        self._ztwin, self._z = None, False
        self._slabs = np.ascontiguousarray(slabs, dtype=np.int64)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int64)
        va = np.ascontiguousarray(values, dtype=np.float64)
        sp = np.ascontiguousarray(col_spans, dtype=np.int64).reshape(-1)
        h = C.c_void_p()
        _check(self.lib, self.lib.dll.mstab_operator_create_csr_slab_local(
            ctx.h, n_global, i64ptr(self._slabs), i64ptr(rp), i64ptr(ci), dptr(va), i64ptr(sp),
            C.c_uint64(fingerprint), C.byref(h)))
        self.h = h
        return self

    @property
    def row_begin(self) -> int:
        return int(self.lib.dll.mstab_operator_row_begin(self.h))

    @property
    def interior_rows(self) -> tuple:
        """[lo, hi) of the slab's rows that reference owned columns only (mstab_operator_interior_rows)."""
        lo, hi = C.c_int64(), C.c_int64()
        self.lib.dll.mstab_operator_interior_rows(self.h, C.byref(lo), C.byref(hi))
        return int(lo.value), int(hi.value)

    @property
    def global_size(self) -> int:
        return int(self.lib.dll.mstab_operator_global_size(self.h))

    def size(self) -> int:
        return int(self.lib.dll.mstab_operator_size(self.h))

    def fingerprint(self) -> int:
        return int(self.lib.dll.mstab_operator_fingerprint(self.h))

    def is_real(self) -> bool:
        return self.matrix is None or self.matrix.is_real()

    def _complex_twin(self) -> "CsrOperator":
        """This operator with complex128 values: a real operator meeting a complex vector computes in
        complex arithmetic like the reference (same CSR, same fingerprint bytes)."""
        if self._z:
            return self
        if self._ztwin is None:
            if self.matrix is None:
                raise ConfigError("b200: the complex path needs the host CSR (single-GPU operators)")
            m = self.matrix
            z = CsrMatrix.__new__(CsrMatrix)
            z.n_rows, z.n_cols, z.row_ptr, z.col_idx = m.n_rows, m.n_cols, m.row_ptr, m.col_idx
            z.values = _c128(m.values)
            t = CsrOperator.__new__(CsrOperator)
            t.ctx, t.lib, t.matrix, t._ztwin, t._z = self.ctx, self.lib, z, None, True
            h = C.c_void_p()
            _check(self.lib, self.lib.dll.mstab_operator_create_csr_z(
                self.ctx.h, z.n_rows, i64ptr(z.row_ptr), i64ptr(z.col_idx), z.values.ctypes.data, C.byref(h)))
            t.h = h
            self._ztwin = t
        return self._ztwin

    def apply(self, x, y=None):
        if self._z or _is_complex(x):
            op = self._complex_twin()
            xz = _c128(x)
            if xz.size != self.size():
                raise DimensionMismatch("spmv: dimension mismatch")
            out = np.empty_like(xz)
            _check(self.lib, self.lib.dll.mstab_operator_apply_z(self.ctx.h, op.h, xz.ctypes.data, out.ctypes.data,
                                                                 _capi.MEM_HOST))
            return out
        ptr, mem = _dev_ptr(x, self.size(), self.ctx, "spmv x")
        if mem == _capi.MEM_DEVICE:
            yptr, ymem = _dev_ptr(y, self.size(), self.ctx, "spmv y")
            if ymem != _capi.MEM_DEVICE:
                raise ConfigError("spmv: x on the device needs a device output y")
            _check(self.lib, self.lib.dll.mstab_operator_apply(self.ctx.h, self.h, ptr, yptr, mem))
            return y
        x = _f64(x)
        if x.size != self.size():
            raise DimensionMismatch("spmv: dimension mismatch")
        out = np.empty_like(x)
        _check(self.lib, self.lib.dll.mstab_operator_apply(self.ctx.h, self.h, x.ctypes.data, out.ctypes.data,
                                                           _capi.MEM_HOST))
        return out

    def apply_adjoint(self, x, y=None):
        """A^H x (CsrOperator::apply_adjoint, operator.cpp:30-33; spmv_adjoint csr.cpp:115-124)."""
        ptr, mem = _dev_ptr(x, self.size(), self.ctx, "spmv_adjoint x")
        if mem == _capi.MEM_DEVICE:
            yptr, ymem = _dev_ptr(y, self.size(), self.ctx, "spmv_adjoint y")
            if ymem != _capi.MEM_DEVICE:
                raise ConfigError("spmv_adjoint: x on the device needs a device output y")
            _check(self.lib, self.lib.dll.mstab_operator_apply_adjoint(self.ctx.h, self.h, ptr, yptr, mem))
            return y
        x = _f64(x)
        if x.size != self.size():
            raise DimensionMismatch("spmv_adjoint: dimension mismatch")
        out = np.empty_like(x)
        _check(self.lib, self.lib.dll.mstab_operator_apply_adjoint(self.ctx.h, self.h, x.ctypes.data,
                                                                   out.ctypes.data, _capi.MEM_HOST))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.dll.mstab_operator_destroy(self.h)
            self.h = None


# ---- split preconditioning (precond.hpp) ------------------------------------------------------
class PrecondKind:
    """precond.hpp:12."""
    NONE = 0
    JACOBI = 1
    ILU0 = 2


@dataclass
class SplitPreconditioner:
    """Split preconditioner L, R for L^-1 A R^-1 xt = L^-1 b (precond.hpp:16-24): L lower with its
    diagonal stored, R upper with the pivots; immutable after build."""
    l_factor: Optional[CsrMatrix]
    r_factor: Optional[CsrMatrix]
    kind: int = PrecondKind.NONE


def _build(kind: int, a: CsrMatrix, lib: Optional[Lib] = None) -> SplitPreconditioner:
    if a.n_rows != a.n_cols:
        raise DimensionMismatch(("jacobi" if kind == PrecondKind.JACOBI else "ilu0") + ": square matrix required")
    lib = lib or default_context().lib
    n, cap = a.n_rows, a.nnz() + a.n_rows
    lrp, rrp = np.empty(n + 1, np.int64), np.empty(n + 1, np.int64)
    lci, rci = np.empty(max(cap, 1), np.int64), np.empty(max(cap, 1), np.int64)
    lva, rva = np.empty(max(cap, 1)), np.empty(max(cap, 1))
    ln, rn = C.c_int64(), C.c_int64()
    _check(lib, lib.dll.mstab_precond_build(kind, n, i64ptr(a.row_ptr), i64ptr(a.col_idx), dptr(a.values),
                                            i64ptr(lrp), i64ptr(lci), dptr(lva), C.byref(ln), i64ptr(rrp),
                                            i64ptr(rci), dptr(rva), C.byref(rn)))
    L = CsrMatrix(n, n, lrp, lci[:ln.value].copy(), lva[:ln.value].copy())
    R = CsrMatrix(n, n, rrp, rci[:rn.value].copy(), rva[:rn.value].copy())
    return SplitPreconditioner(L, R, kind)


def build_jacobi(a: CsrMatrix, lib: Optional[Lib] = None) -> SplitPreconditioner:
    """Split Jacobi, sqrt(diag) in both factors (precond.cpp:23-37). Raises ZeroPivot."""
    return _build(PrecondKind.JACOBI, a, lib)


def build_ilu0(a: CsrMatrix, lib: Optional[Lib] = None) -> SplitPreconditioner:
    """ILU(0) on A's pattern, IKJ order (precond.cpp:39-99). Raises ZeroPivot."""
    return _build(PrecondKind.ILU0, a, lib)


def build_none() -> SplitPreconditioner:
    return SplitPreconditioner(None, None, PrecondKind.NONE)


class PreconditionedOperator(CsrOperator):
    """Operator view of L^-1 A R^-1 (precond.hpp:57-74) on the device: every apply is the upper
    solve, the SpMV and the lower solve; fingerprint combined as precond.cpp:203-210."""

    def __init__(self, pc: SplitPreconditioner, a: CsrMatrix, ctx: Optional[Context] = None):
        if a.n_rows != a.n_cols:
            raise DimensionMismatch("precond operator: square required")
        self.ctx = ctx if ctx is not None else default_context()
        self.lib = self.ctx.lib
        self.matrix = a
        self._ztwin, self._z = None, False
        self.pc = pc
        h = C.c_void_p()
        if pc.kind == PrecondKind.NONE:
            _check(self.lib, self.lib.dll.mstab_operator_create_csr(
                self.ctx.h, a.n_rows, i64ptr(a.row_ptr), i64ptr(a.col_idx), dptr(a.values), C.byref(h)))
        else:
            L, R = pc.l_factor, pc.r_factor
            _check(self.lib, self.lib.dll.mstab_operator_create_precond(
                self.ctx.h, a.n_rows, i64ptr(a.row_ptr), i64ptr(a.col_idx), dptr(a.values), pc.kind,
                i64ptr(L.row_ptr), i64ptr(L.col_idx), dptr(L.values), i64ptr(R.row_ptr), i64ptr(R.col_idx),
                dptr(R.values), C.byref(h)))
        self.h = h

    def _solve(self, which: int, x) -> np.ndarray:
        x = _f64(x)
        if x.size != self.size():
            raise DimensionMismatch("precond: dimension mismatch")
        out = np.empty_like(x)
        _check(self.lib, self.lib.dll.mstab_precond_solve(self.ctx.h, self.h, which, x.ctypes.data,
                                                          out.ctypes.data, _capi.MEM_HOST))
        return out

    def lower_solve(self, b) -> np.ndarray:
        """x = L^-1 b (precond.cpp:101-116)."""
        return self._solve(0, b)

    def upper_solve(self, b) -> np.ndarray:
        """x = R^-1 b (precond.cpp:118-133)."""
        return self._solve(1, b)


def preconditioned_rhs(op: PreconditionedOperator, b) -> np.ndarray:
    """L^-1 b (precond.cpp:181-184), on the device of the operator that holds the factors."""
    return op.lower_solve(b)


def unpreconditioned_solution(op: PreconditionedOperator, x_tilde) -> np.ndarray:
    """R^-1 xt (precond.cpp:176-179)."""
    return op.upper_solve(x_tilde)


# ---- recycle data (recycle.hpp) ---------------------------------------------------------------
class RecycleData:
    """Immutable recycle state (P, U, V, omega history, level J, s, fingerprint); device-resident
    in the B200 implementation, downloaded lazily."""

    def __init__(self, ctx: Context, handle):
        self.ctx, self.lib, self.h = ctx, ctx.lib, handle
        info = _capi.RecycleInfoC()
        _check(self.lib, self.lib.dll.mstab_recycle_info_get(handle, C.byref(info)))
        self.n, self.s, self.level_J = int(info.n), int(info.s), int(info.level_j)
        self.matrix_fingerprint = int(info.fingerprint)
        self._omega_count = int(info.omega_count)
        self._blocks = None
        self._omega = None
        self.is_complex = bool(self.lib.dll.mstab_recycle_is_complex(handle))

    def _download(self):
        if self._blocks is None:
            n, s = self.n, self.s
            om = np.empty(2 * max(self._omega_count, 1))
            if self.is_complex:
                p, u, v = (np.empty((s, n), dtype=np.complex128) for _ in range(3))
                _check(self.lib, self.lib.dll.mstab_recycle_download_z(
                    self.ctx.h, self.h, p.ctypes.data, u.ctypes.data, v.ctypes.data, dptr(om)))
            else:
                p, u, v = (np.empty((s, n)) for _ in range(3))
                _check(self.lib, self.lib.dll.mstab_recycle_download(self.ctx.h, self.h, dptr(p), dptr(u), dptr(v),
                                                                     dptr(om)))
            self._blocks = (p.T, u.T, v.T)  # n x s views of the column-major data
            self._omega = om[0:2 * self._omega_count:2] + 1j * om[1:2 * self._omega_count:2]
        return self._blocks

    @property
    def p(self):
        return self._download()[0]

    @property
    def u(self):
        return self._download()[1]

    @property
    def v(self):
        return self._download()[2]

    @property
    def omega_history(self):
        self._download()
        return self._omega

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.dll.mstab_recycle_destroy(self.h)
            self.h = None


def fetch(p, u, v, omega_history, level_j, fingerprint, ctx: Optional[Context] = None) -> RecycleData:
    """Deep-copy constructor of RecycleData (recycle.cpp:26-38)."""
    ctx = ctx if ctx is not None else default_context()
    om = np.asarray(omega_history, dtype=np.complex128).ravel()
    omr = np.empty(2 * max(om.size, 1))
    omr[0:2 * om.size:2] = om.real
    omr[1:2 * om.size:2] = om.imag
    h = C.c_void_p()
    if any(_is_complex(a) for a in (p, u, v)):
        p, u, v = (np.asfortranarray(np.asarray(a, dtype=np.complex128)) for a in (p, u, v))
        n, s = p.shape
        _check(ctx.lib, ctx.lib.dll.mstab_recycle_create_z(
            ctx.h, n, s, p.ctypes.data, u.ctypes.data, v.ctypes.data, _capi.MEM_HOST, dptr(omr), om.size,
            int(level_j), int(fingerprint), C.byref(h)))
        return RecycleData(ctx, h)
    p, u, v = (np.asfortranarray(_f64(a)) for a in (p, u, v))
    n, s = p.shape
    _check(ctx.lib, ctx.lib.dll.mstab_recycle_create(
        ctx.h, n, s, p.ctypes.data, u.ctypes.data, v.ctypes.data, _capi.MEM_HOST, dptr(omr), om.size,
        int(level_j), int(fingerprint), C.byref(h)))
    return RecycleData(ctx, h)


def _complex_recycle(data: RecycleData, ctx: Context) -> RecycleData:
    """Real recycle data re-created as complex blocks (+0.0 imaginary parts): a real hand-off continuing
    into a complex solve, as the reference's single complex type allows."""
    h = C.c_void_p()
    p, u, v = (np.asfortranarray(np.asarray(a, dtype=np.complex128)) for a in (data.p, data.u, data.v))
    om = np.asarray(data.omega_history, dtype=np.complex128).ravel()
    omr = np.empty(2 * max(om.size, 1))
    omr[0:2 * om.size:2] = om.real
    omr[1:2 * om.size:2] = om.imag
    _check(ctx.lib, ctx.lib.dll.mstab_recycle_create_z(
        ctx.h, data.n, data.s, p.ctypes.data, u.ctypes.data, v.ctypes.data, _capi.MEM_HOST, dptr(omr), om.size,
        int(data.level_J), int(data.matrix_fingerprint), C.byref(h)))
    return RecycleData(ctx, h)


def validate(data: RecycleData, op: CsrOperator) -> ValidationReport:
    r = _capi.ValidationReportC()
    if data.is_complex:
        op = op._complex_twin()
    _check(op.lib, op.lib.dll.mstab_recycle_validate(op.ctx.h, data.h, op.h, C.byref(r)))
    return ValidationReport(r.max_deviation, r.sigma_min_ratio, bool(r.low_rank_warning))


def save(data: RecycleData, path) -> None:
    _check(data.lib, data.lib.dll.mstab_recycle_save(data.ctx.h, data.h, str(path).encode()))


def load(path, ctx: Optional[Context] = None) -> RecycleData:
    ctx = ctx if ctx is not None else default_context()
    h = C.c_void_p()
    _check(ctx.lib, ctx.lib.dll.mstab_recycle_load(ctx.h, str(path).encode(), C.byref(h)))
    return RecycleData(ctx, h)


# ---- solve (idrstab.hpp:70-96) ----------------------------------------------------------------
class SolveResult:
    def __init__(self, ctx: Context, handle):
        self.ctx, self.lib, self.h = ctx, ctx.lib, handle
        rep = _capi.ReportC()
        _check(self.lib, self.lib.dll.mstab_result_report(handle, C.byref(rep)))
        self._rep = rep
        self.n = None
        self._x = None
        self._report = None

    @property
    def report(self) -> SolveReport:
        if self._report is None:
            r = self._rep
            hist = (_capi.HistoryPointC * max(r.history_len, 1))()
            cnt = self.lib.dll.mstab_result_history(self.h, hist, r.history_len)
            taus = np.empty(2 * max(r.tau_len, 1))
            tcnt = self.lib.dll.mstab_result_taus(self.h, dptr(taus), r.tau_len)
            t = taus[0:2 * tcnt:2] + 1j * taus[1:2 * tcnt:2]
            ell = int(r.ell) if r.ell > 0 else 1
            self._report = SolveReport(
                residual_history=[HistoryPoint(h.cycle, h.mv, h.level, h.resnorm, h.wall_ns) for h in hist[:cnt]],
                omega_history=[t[i:i + ell] for i in range(0, tcnt, ell)],
                h_mv=r.h_mv, h_mv_aux=r.h_mv_aux, h_rd=r.h_rd, cycles=r.cycles, status=_STATUS[r.status],
                breakdown_reason=r.breakdown_reason.decode(), bnorm=r.bnorm, final_resnorm=r.final_resnorm,
                wall_ns_total=r.wall_ns_total)
        return self._report

    @property
    def x(self) -> np.ndarray:
        if self._x is None:
            if self.lib.dll.mstab_result_is_complex(self.h):
                out = np.empty(self.n, dtype=np.complex128)
                _check(self.lib, self.lib.dll.mstab_result_x_z(self.ctx.h, self.h, out.ctypes.data, _capi.MEM_HOST))
            else:
                out = np.empty(self.n)
                _check(self.lib, self.lib.dll.mstab_result_x(self.ctx.h, self.h, out.ctypes.data, _capi.MEM_HOST))
            self._x = out
        return self._x

    def x_into(self, dst) -> None:
        """Copy x into a CUDA tensor / host array without materialising it in Python."""
        ptr, mem = _dev_ptr(dst, self.n, self.ctx, "x")
        if mem == _capi.MEM_HOST:
            if not (isinstance(dst, np.ndarray) and dst.dtype == np.float64 and dst.flags.c_contiguous
                    and dst.size == self.n):
                raise ConfigError("x_into: host destination must be a contiguous float64 array of n entries")
            ptr = dst.ctypes.data
        _check(self.lib, self.lib.dll.mstab_result_x(self.ctx.h, self.h, ptr, mem))

    def _rd(self, fn) -> RecycleData:
        h = C.c_void_p()
        _check(self.lib, fn(self.h, C.byref(h)))
        return RecycleData(self.ctx, h)

    @property
    def final_data(self) -> RecycleData:
        return self._rd(self.lib.dll.mstab_result_final_data)

    @property
    def fetched(self) -> Optional[RecycleData]:
        return self._rd(self.lib.dll.mstab_result_fetched) if self._rep.has_fetched else None

    def handoff(self) -> RecycleData:
        return self._rd(self.lib.dll.mstab_result_handoff)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.dll.mstab_result_destroy(self.h)
            self.h = None


def idrstab_solve(a: CsrOperator, b, x0=None, cfg: Optional[SolverConfig] = None,
                  recycle: Optional[RecycleData] = None, fetch_policy: Optional[FetchPolicy] = None) -> SolveResult:
    """IDR(s)stab(ell); M(s,ell)stab when `recycle` is given (idrstab.hpp:88-91)."""
    cfg = cfg if cfg is not None else SolverConfig()
    ctx, lib = a.ctx, a.lib
    n = a.size()
    x0_given = x0 is not None and (not hasattr(x0, "__len__") or len(x0) > 0)
    if (not a.is_real() or _is_complex(b) or (x0_given and _is_complex(x0))
            or (recycle is not None and recycle.is_complex)):
        # complex128 data: the reference's complex arithmetic on the device
        if recycle is not None and not recycle.is_complex:
            recycle = _complex_recycle(recycle, ctx)
        az = a._complex_twin()
        bz = _c128(b)
        if bz.size != n:
            raise DimensionMismatch("idrstab: rhs size")
        xz = None
        if x0_given:
            xz = _c128(x0)
            if xz.size != n:
                raise DimensionMismatch("idrstab: guess size")
        c = cfg._c()
        fp = _capi.FetchPolicyC(fetch_policy.kind, 0, fetch_policy.cycle) if fetch_policy is not None else None
        h = C.c_void_p()
        _check(lib, lib.dll.mstab_solve_z(ctx.h, az.h, bz.ctypes.data, xz.ctypes.data if xz is not None else None,
                                          _capi.MEM_HOST, C.byref(c), recycle.h if recycle else None,
                                          C.byref(fp) if fp is not None else None, C.byref(h)))
        res = SolveResult(ctx, h)
        res.n = n
        return res
    bptr, mem = _dev_ptr(b, n, ctx, "rhs")
    keep = []
    if mem == _capi.MEM_HOST:
        b = _f64(b)
        if b.size != n:
            raise DimensionMismatch("idrstab: rhs size")
        keep.append(b)
        bptr = b.ctypes.data
    xptr = None
    if x0 is not None and (not hasattr(x0, "__len__") or len(x0) > 0):
        if mem == _capi.MEM_HOST:
            if _dev_ptr(x0)[1] == _capi.MEM_DEVICE:
                raise ConfigError("idrstab: x0 is on the device but b is not (both must be in the same memory space)")
            x0 = _f64(x0)
            if x0.size != n:
                raise DimensionMismatch("idrstab: guess size")
            keep.append(x0)
            xptr = x0.ctypes.data
        else:
            xptr, xmem = _dev_ptr(x0, n, ctx, "guess")
            if xmem != _capi.MEM_DEVICE:
                raise ConfigError("idrstab: b is on the device but x0 is not (both must be in the same memory space)")
    c = cfg._c()
    fp = None
    if fetch_policy is not None:
        fp = _capi.FetchPolicyC(fetch_policy.kind, 0, fetch_policy.cycle)
    h = C.c_void_p()
    _check(lib, lib.dll.mstab_solve(ctx.h, a.h, bptr, xptr, mem, C.byref(c), recycle.h if recycle else None,
                                    C.byref(fp) if fp is not None else None, C.byref(h)))
    res = SolveResult(ctx, h)
    res.n = n
    return res


def mstab_solve(a: CsrOperator, b, x0, cfg: SolverConfig, recycle: RecycleData,
                fetch_policy: Optional[FetchPolicy] = None) -> SolveResult:
    """M(s,ell)stab: idrstab_solve with mandatory recycle data (idrstab.hpp:94-96)."""
    return idrstab_solve(a, b, x0, cfg, recycle, fetch_policy)


def sridr_solve(a: CsrOperator, b, x0, cfg: SolverConfig, recycle: RecycleData):
    """SRIDR (sridr.hpp, sridr.cpp:23-118): returns (x, report) like the reference's pair."""
    ctx, lib = a.ctx, a.lib
    n = a.size()
    b = _f64(b)
    if b.size != n:
        raise DimensionMismatch("sridr: rhs size")
    xptr = None
    if x0 is not None and len(x0) > 0:
        x0 = _f64(x0)
        xptr = x0.ctypes.data
    c = cfg._c()
    h = C.c_void_p()
    _check(lib, lib.dll.mstab_sridr_solve(ctx.h, a.h, b.ctypes.data, xptr, _capi.MEM_HOST, C.byref(c), recycle.h,
                                          C.byref(h)))
    res = SolveResult(ctx, h)
    res.n = n
    return res.x, res.report


def _baseline_result(ctx, n, h):
    res = SolveResult(ctx, h)
    res.n = n
    return res.x, res.report


def bicg_solve(a: CsrOperator, b, x0, tol: float, max_mv: int, shadow=None):
    """BiCG with adjoint products (baselines.hpp, baselines.cpp:145-196); returns (x, report)."""
    n = a.size()
    b = _f64(b)
    if b.size != n:
        raise DimensionMismatch("bicg: rhs size")
    x0 = _f64(x0) if x0 is not None and len(x0) > 0 else None
    sh = _f64(shadow) if shadow is not None else None
    h = C.c_void_p()
    _check(a.lib, a.lib.dll.mstab_bicg_solve(a.ctx.h, a.h, b.ctypes.data, x0.ctypes.data if x0 is not None else None,
                                             _capi.MEM_HOST, tol, max_mv,
                                             sh.ctypes.data if sh is not None else None, C.byref(h)))
    return _baseline_result(a.ctx, n, h)


def bicgstab_solve(a: CsrOperator, b, x0, tol: float, max_mv: int, shadow=None):
    """Textbook BiCGStab (baselines.hpp, baselines.cpp:198-262); returns (x, report)."""
    n = a.size()
    b = _f64(b)
    if b.size != n:
        raise DimensionMismatch("bicgstab: rhs size")
    x0 = _f64(x0) if x0 is not None and len(x0) > 0 else None
    sh = _f64(shadow) if shadow is not None else None
    h = C.c_void_p()
    _check(a.lib, a.lib.dll.mstab_bicgstab_solve(a.ctx.h, a.h, b.ctypes.data, x0.ctypes.data if x0 is not None else None,
                                                 _capi.MEM_HOST, tol, max_mv,
                                                 sh.ctypes.data if sh is not None else None, C.byref(h)))
    return _baseline_result(a.ctx, n, h)


def gmres_solve(a: CsrOperator, b, x0, tol: float, max_it: int):
    """Full-memory GMRES with modified Gram-Schmidt (baselines.cpp:49-143); returns (x, report)."""
    n = a.size()
    b = _f64(b)
    if b.size != n:
        raise DimensionMismatch("gmres: rhs size")
    x0 = _f64(x0) if x0 is not None and len(x0) > 0 else None
    h = C.c_void_p()
    _check(a.lib, a.lib.dll.mstab_gmres_solve(a.ctx.h, a.h, b.ctypes.data, x0.ctypes.data if x0 is not None else None,
                                              _capi.MEM_HOST, tol, max_it, C.byref(h)))
    return _baseline_result(a.ctx, n, h)


# ---- kernel-level helpers (include/mstab_b200_kernels.h) --------------------------------------
def solve_small(m, rhs, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx if ctx is not None else default_context()
    m = np.asfortranarray(_f64(m))
    rhs = _f64(rhs)
    x = np.empty_like(rhs)
    _check(ctx.lib, ctx.lib.dll.mstab_kernel_solve_small(ctx.h, m.shape[0], m.ctypes.data_as(_capi._D),
                                                         dptr(rhs), dptr(x)))
    return x


def least_squares_tall(z, r, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx if ctx is not None else default_context()
    z = np.asfortranarray(_f64(z))
    r = _f64(r)
    n, ell = z.shape
    tau = np.empty(ell)
    _check(ctx.lib, ctx.lib.dll.mstab_kernel_least_squares(ctx.h, n, ell, z.ctypes.data_as(_capi._D), dptr(r),
                                                           dptr(tau)))
    return tau


def make_cut_space(n, s, seed, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx if ctx is not None else default_context()
    p = np.empty((s, n))
    _check(ctx.lib, ctx.lib.dll.mstab_kernel_cut_space(ctx.h, n, s, seed, dptr(p)))
    return p.T


def arnoldi_init(a: CsrOperator, r0, s, rng_seed):
    r0 = _f64(r0)
    n = r0.size
    u, v = np.empty((s, n)), np.empty((s, n))
    mv = C.c_int64(0)
    _check(a.lib, a.lib.dll.mstab_kernel_arnoldi(a.ctx.h, a.h, dptr(r0), s, rng_seed, dptr(u), dptr(v), C.byref(mv)))
    return u.T, v.T, int(mv.value)


NORMAL_FILL_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(C.c_double), C.c_int64)


def arnoldi_init_draws(a: CsrOperator, r0, s, draw):
    """arnoldi_init with the padding draws supplied by `draw(count) -> array of standard normals`
    (the drop-in shim hands the caller's std::mt19937_64 through this entry point)."""
    r0 = _f64(r0)
    n = r0.size
    u, v = np.empty((s, n)), np.empty((s, n))
    mv = C.c_int64(0)

    def fill(_user, out, count):
        vals = np.ascontiguousarray(draw(int(count)), dtype=np.float64)
        C.memmove(out, vals.ctypes.data, 8 * int(count))

    cb = NORMAL_FILL_FN(fill)
    _check(a.lib, a.lib.dll.mstab_kernel_arnoldi_cb(a.ctx.h, a.h, dptr(r0), s, C.cast(cb, C.c_void_p), None,
                                                    dptr(u), dptr(v), C.byref(mv)))
    return u.T, v.T, int(mv.value)


def bicg_projection(p, block, target, ctx: Optional[Context] = None) -> np.ndarray:
    """gamma with (P^H block) gamma = P^H target (idrstab.hpp:33-36); SingularProjection when singular."""
    ctx = ctx if ctx is not None else default_context()
    p, block = np.asfortranarray(_f64(p)), np.asfortranarray(_f64(block))
    target = _f64(target)
    n, s = p.shape
    if block.shape != (n, s) or target.size != n:
        raise DimensionMismatch("bicg_projection: shapes")
    gamma = np.empty(s)
    _check(ctx.lib, ctx.lib.dll.mstab_kernel_bicg_projection(ctx.h, n, s, p.ctypes.data_as(_capi._D),
                                                             block.ctypes.data_as(_capi._D), dptr(target),
                                                             dptr(gamma)))
    return gamma


class IterationState:
    """Level vectors of one outer cycle (idrstab.hpp:38-46): r_levels[i] = r^(i), v_levels[i] = V^(i-1)."""

    def __init__(self, x0, r_levels, v_levels):
        self.x0, self.r_levels, self.v_levels = x0, r_levels, v_levels

    @staticmethod
    def start(x, r, u, v) -> "IterationState":
        return IterationState(_f64(x).copy(), [_f64(r).copy()], [np.array(u, dtype=np.float64), np.array(v, dtype=np.float64)])

    def v_level(self, level: int):
        return self.v_levels[level + 1]


def level_iteration(st: IterationState, a: CsrOperator, p, k: int, rep: Optional[SolveReport] = None) -> None:
    """One IDR level iteration k on the device (idrstab.hpp:48-53): s + 1 operator applications."""
    p = np.asfortranarray(_f64(p))
    n, s = p.shape
    if len(st.r_levels) < k + 1 or len(st.v_levels) < k + 2:
        raise Error("level_iteration: missing levels")
    x0 = _f64(st.x0).copy()
    r = np.zeros((k + 2, n))
    v = np.zeros((k + 3, s, n))
    for i in range(k + 1):
        r[i] = st.r_levels[i]
    for i in range(k + 2):
        v[i] = np.asarray(st.v_levels[i]).T
    _check(a.lib, a.lib.dll.mstab_kernel_level_iteration(a.ctx.h, a.h, s, k, p.ctypes.data_as(_capi._D), dptr(x0),
                                                         dptr(r), dptr(v)))
    st.x0 = x0
    st.r_levels = [r[i].copy() for i in range(k + 2)]
    st.v_levels = [v[i].T.copy() for i in range(k + 3)]
    if rep is not None:
        rep.h_mv += s + 1


@dataclass
class PolyOut:
    x: np.ndarray
    r: np.ndarray
    u: np.ndarray
    v: np.ndarray
    tau: np.ndarray
    tail_perturbed: bool


def poly_combination(st: IterationState, ell: int, ctx: Optional[Context] = None) -> PolyOut:
    """Degree-ell residual minimisation on the device (idrstab.hpp:55-68); RankDeficient when Z lost rank."""
    ctx = ctx if ctx is not None else default_context()
    n = st.x0.size
    s = np.asarray(st.v_levels[0]).shape[1]
    if len(st.r_levels) < ell + 1 or len(st.v_levels) < ell + 2:
        raise Error("poly_combination: missing levels")
    r = np.ascontiguousarray(np.stack([_f64(st.r_levels[i]) for i in range(ell + 1)]))
    v = np.ascontiguousarray(np.stack([np.asarray(st.v_levels[i], dtype=np.float64).T for i in range(ell + 2)]))
    x0 = _f64(st.x0)
    x, rr, u, vv, tau = np.empty(n), np.empty(n), np.empty((s, n)), np.empty((s, n)), np.empty(ell)
    pert = C.c_int32(0)
    _check(ctx.lib, ctx.lib.dll.mstab_kernel_poly_combination(ctx.h, n, s, ell, dptr(x0), dptr(r), dptr(v), dptr(x),
                                                              dptr(rr), dptr(u), dptr(vv), dptr(tau), C.byref(pert)))
    return PolyOut(x, rr, u.T.copy(), vv.T.copy(), tau, bool(pert.value))


def local_col_span(row0: int, row1: int, col_idx) -> tuple:
    """[lo, hi) of the columns a slab's rows reference (at least its own rows)."""
    ci = np.asarray(col_idx)
    if ci.size == 0:
        return int(row0), int(row1)
    return int(min(row0, ci.min())), int(max(row1, ci.max() + 1))


def distributed_fingerprint(lib: Lib, n_global: int, nnz_global: int, row_ptr, col_idx, values, first_entry: int,
                            group=None) -> int:
    """The reference's checksum of a row-distributed CSR matrix (csr.cpp:28-43) without gathering it.

    The checksum folds dims, then all row_ptr entries, all col_idx entries and all values, so the
    8-byte state makes three passes over the ranks of torch.distributed's `group` (send / recv to
    the next rank; the last rank broadcasts the result). `row_ptr` is the slab's local row_ptr (from
    0), `first_entry` the global index of its first stored entry (the nnz of the lower ranks).
    Without an initialised process group (one rank) it is the plain fold."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float64)
    dll = lib.dll
    rank, world, dist, torch, dev = 0, 1, None, None, None
    try:
        import torch
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
            dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    except ImportError:
        pass

    def to_t(h):
        return torch.from_numpy(np.array([h], dtype=np.uint64).view(np.int64).copy()).to(dev)

    def from_t(t):
        return int(t.cpu().numpy().view(np.uint64)[0])

    h = int(dll.mstab_fnv_begin(n_global, n_global, nnz_global)) if rank == 0 else 0
    for phase in range(3):
        if world > 1 and not (phase == 0 and rank == 0):
            t = to_t(0)
            dist.recv(t, src=(rank - 1) % world, group=group)
            h = from_t(t)
        if phase == 0:  # rank 0 contributes the leading 0, every rank its n_local end offsets
            off = 0 if rank == 0 else 1
            part = np.ascontiguousarray(rp[off:])
            h = int(dll.mstab_fnv_fold_index(C.c_uint64(h), i64ptr(part), part.size, first_entry))
        elif phase == 1:
            h = int(dll.mstab_fnv_fold_index(C.c_uint64(h), i64ptr(ci), ci.size, 0))
        else:
            h = int(dll.mstab_fnv_fold_values(C.c_uint64(h), dptr(va), va.size))
        if world > 1 and not (phase == 2 and rank == world - 1):
            dist.send(to_t(h), dst=(rank + 1) % world, group=group)
    if world > 1:
        t = to_t(h)
        dist.broadcast(t, src=world - 1, group=group)
        h = from_t(t)
    return h
