"""ctypes binding of the C restatement oracle (oracle/mstab_oracle.{h,c}) — test infrastructure."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
LIB_PATH = ROOT / "oracle" / "_build" / "libmstab_oracle.so"
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int64)


class OrcCsr(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_ptr", _I), ("col_idx", _I), ("values", _D)]


class OrcCfg(C.Structure):
    _fields_ = [("s", C.c_int64), ("ell", C.c_int64), ("tol", C.c_double), ("max_mv", C.c_int64),
                ("true_residual", C.c_int32), ("_pad", C.c_int32), ("seed", C.c_uint64)]


class OrcRecycle(C.Structure):
    _fields_ = [("n", C.c_int64), ("s", C.c_int64), ("level_j", C.c_int64), ("fingerprint", C.c_uint64),
                ("p", _D), ("u", _D), ("v", _D), ("omega_count", C.c_int64), ("omega", _D)]


class OrcResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("has_fetched", C.c_int32), ("h_mv", C.c_int64), ("h_mv_aux", C.c_int64),
                ("h_rd", C.c_int64), ("cycles", C.c_int64), ("bnorm", C.c_double), ("final_resnorm", C.c_double),
                ("x", _D), ("hist_len", C.c_int64), ("hist", _I), ("hist_resnorm", _D), ("tau_len", C.c_int64),
                ("tau", _D), ("final_data", OrcRecycle), ("fetched", OrcRecycle), ("reason", C.c_char * 128)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"C restatement not built: {LIB_PATH} (make -C oracle restatement)")
        L = C.CDLL(str(LIB_PATH))
        L.orc_solve.argtypes = [C.POINTER(OrcCsr), _D, _D, C.POINTER(OrcCfg), C.POINTER(OrcRecycle), C.c_int32,
                                C.c_int64, C.POINTER(OrcResult)]
        L.orc_solve.restype = C.c_int
        L.orc_result_free.argtypes = [C.POINTER(OrcResult)]
        L.orc_fingerprint.argtypes = [C.POINTER(OrcCsr)]
        L.orc_fingerprint.restype = C.c_uint64
        L.orc_spmv.argtypes = [C.POINTER(OrcCsr), _D, _D]
        L.orc_solve_small.argtypes = [C.c_int64, _D, _D, _D]
        L.orc_least_squares.argtypes = [C.c_int64, C.c_int64, _D, _D, _D]
        L.orc_cut_space.argtypes = [C.c_int64, C.c_int64, C.c_uint64, _D]
        L.orc_arnoldi.argtypes = [C.POINTER(OrcCsr), _D, C.c_int64, C.c_uint64, _D, _D]
        L.orc_normal_draws.argtypes = [C.c_uint64, C.c_int64, _D]
        L.orc_validate.argtypes = [C.POINTER(OrcCsr), C.POINTER(OrcRecycle), _D, _D]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(_D)


class Csr:
    def __init__(self, m):
        self.rp = np.ascontiguousarray(m.row_ptr, dtype=np.int64)
        self.ci = np.ascontiguousarray(m.col_idx, dtype=np.int64)
        self.va = np.ascontiguousarray(m.values, dtype=np.float64)
        self.c = OrcCsr(int(m.n_rows), self.rp.ctypes.data_as(_I), self.ci.ctypes.data_as(_I), _d(self.va))

    def fingerprint(self):
        return int(lib().orc_fingerprint(C.byref(self.c)))

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        lib().orc_spmv(C.byref(self.c), _d(x), _d(y))
        return y


@dataclass
class Recycle:
    p: np.ndarray
    u: np.ndarray
    v: np.ndarray
    omega: np.ndarray
    level_j: int
    fingerprint: int

    @property
    def s(self):
        return self.p.shape[1]

    def c(self):
        self._keep = [np.asfortranarray(a, dtype=np.float64) for a in (self.p, self.u, self.v)]
        om = np.asarray(self.omega, dtype=np.complex128)
        self._om = np.empty(2 * max(om.size, 1))
        self._om[0:2 * om.size:2] = om.real
        self._om[1:2 * om.size:2] = om.imag
        n, s = self.p.shape
        return OrcRecycle(n, s, self.level_j, self.fingerprint, *(_d(a) for a in self._keep), om.size, _d(self._om))


def _recycle_from(c: OrcRecycle) -> Recycle:
    n, s = c.n, c.s
    get = lambda ptr: np.ctypeslib.as_array(ptr, shape=(n * s,)).reshape(s, n).T.copy()
    om = np.ctypeslib.as_array(c.omega, shape=(max(2 * c.omega_count, 1),))[:2 * c.omega_count]
    return Recycle(get(c.p), get(c.u), get(c.v), om[0::2] + 1j * om[1::2], c.level_j, int(c.fingerprint))


@dataclass
class Result:
    status: int
    cycles: int
    h_mv: int
    h_mv_aux: int
    h_rd: int
    bnorm: float
    final_resnorm: float
    x: np.ndarray
    hist: np.ndarray          # (len, 3): cycle, mv, level
    resnorms: np.ndarray
    taus: np.ndarray
    final_data: Recycle
    fetched: Optional[Recycle]
    reason: str


def solve(csr: Csr, b, x0=None, s=2, ell=1, tol=1e-8, max_mv=100000, true_residual=False, seed=0,
          recycle: Optional[Recycle] = None, fetch_kind=2, fetch_cycle=0) -> Result:
    b = np.ascontiguousarray(b, dtype=np.float64)
    xp = None
    if x0 is not None:
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        xp = _d(x0)
    cfg = OrcCfg(s, ell, tol, max_mv, 1 if true_residual else 0, 0, seed)
    rc_rec = recycle.c() if recycle is not None else None
    out = OrcResult()
    rc = lib().orc_solve(C.byref(csr.c), _d(b), xp, C.byref(cfg), C.byref(rc_rec) if rc_rec else None,
                         fetch_kind, fetch_cycle, C.byref(out))
    if rc != 0:
        raise RuntimeError(f"orc_solve failed: {rc}")
    try:
        n = csr.c.n
        hl = out.hist_len
        res = Result(out.status, out.cycles, out.h_mv, out.h_mv_aux, out.h_rd, out.bnorm, out.final_resnorm,
                     np.ctypeslib.as_array(out.x, shape=(n,)).copy(),
                     np.ctypeslib.as_array(out.hist, shape=(3 * hl,)).reshape(hl, 3).copy(),
                     np.ctypeslib.as_array(out.hist_resnorm, shape=(hl,)).copy(),
                     np.ctypeslib.as_array(out.tau, shape=(max(out.tau_len, 1),))[:out.tau_len].copy(),
                     _recycle_from(out.final_data), _recycle_from(out.fetched) if out.has_fetched else None,
                     out.reason.decode())
    finally:
        lib().orc_result_free(C.byref(out))
    return res


def solve_small(m, rhs):
    m = np.asfortranarray(m, dtype=np.float64)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    x = np.empty_like(rhs)
    rc = lib().orc_solve_small(m.shape[0], m.ctypes.data_as(_D), _d(rhs), _d(x))
    return x if rc == 0 else None


def least_squares(z, r):
    z = np.asfortranarray(z, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    tau = np.empty(z.shape[1])
    rc = lib().orc_least_squares(z.shape[0], z.shape[1], z.ctypes.data_as(_D), _d(r), _d(tau))
    return tau if rc == 0 else rc


def cut_space(n, s, seed):
    p = np.empty(n * s)
    rc = lib().orc_cut_space(n, s, seed, _d(p))
    assert rc == 0
    return p.reshape(s, n).T.copy()


def arnoldi(csr: Csr, r0, s, rng_seed):
    n = csr.c.n
    r0 = np.ascontiguousarray(r0, dtype=np.float64)
    u, v = np.empty(n * s), np.empty(n * s)
    rc = lib().orc_arnoldi(C.byref(csr.c), _d(r0), s, rng_seed, _d(u), _d(v))
    assert rc == 0
    return u.reshape(s, n).T.copy(), v.reshape(s, n).T.copy()


def normal_draws(seed, count):
    out = np.empty(count)
    lib().orc_normal_draws(seed, count, _d(out))
    return out


def validate(csr: Csr, rec: Recycle):
    md, sr = C.c_double(0), C.c_double(0)
    rc = lib().orc_validate(C.byref(csr.c), C.byref(rec.c()), C.byref(md), C.byref(sr))
    return rc, md.value, sr.value
