"""Synthetic problems of the BASELINE configs (builder-defined; see include/mstab_gen.h and
SURVEY.md §8(d)). These are seeded stand-ins with the configs' shapes and value distributions;
no external benchmark data set is involved.

Each config yields a CSR matrix and a right-hand-side *sequence* rule:
  * conv-diff (c1, c2, c4, c5): b_1 = h^2 (x_0/dt + f), b_{i+1} = h^2 (x_i/dt + f) with x_0, f drawn
    uniform[0,1) from std::mt19937_64(seed) (x_0 first, then f);
  * banded random (c3): b_1 = g_0, b_{i+1} = x_i + 0.1 g_i, g_i ~ N(0,1) from std::mt19937_64(seed_g + i).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Tuple

import numpy as np

from ._capi import dptr, gen_lib, i64ptr
from .mstab import CsrMatrix


def convdiff(dim: int, n: int, stencil: int, beta, dt: float) -> CsrMatrix:
    g = gen_lib()
    nnz = g.mstab_gen_convdiff_nnz(dim, n, stencil)
    if nnz < 0:
        raise ValueError("unsupported stencil")
    N = n ** dim
    rp = np.empty(N + 1, dtype=np.int64)
    ci = np.empty(nnz, dtype=np.int64)
    va = np.empty(nnz, dtype=np.float64)
    b = np.zeros(3)
    b[:len(beta)] = beta
    rc = g.mstab_gen_convdiff(dim, n, stencil, dptr(b), dt, i64ptr(rp), i64ptr(ci), dptr(va))
    if rc != 0:
        raise ValueError("generator failed")
    return CsrMatrix(N, N, rp, ci, va)


def convdiff_rows(dim: int, n: int, stencil: int, beta, dt: float, row0: int, row1: int):
    """Rows [row0, row1) of the conv-diff matrix: (local row_ptr, GLOBAL col_idx, values). A rank of
    a row-sharded run generates its own slab; the global matrix is never materialised."""
    g = gen_lib()
    b = np.zeros(3)
    b[:len(beta)] = beta
    nnz = int(g.mstab_gen_convdiff_rows(dim, n, stencil, dptr(b), dt, row0, row1, None, None, None))
    if nnz < 0:
        raise ValueError("unsupported stencil")
    rp = np.empty(row1 - row0 + 1, dtype=np.int64)
    ci = np.empty(nnz, dtype=np.int64)
    va = np.empty(nnz, dtype=np.float64)
    g.mstab_gen_convdiff_rows(dim, n, stencil, dptr(b), dt, row0, row1, i64ptr(rp), i64ptr(ci), dptr(va))
    return rp, ci, va


def banded(n: int, nnz_per_row: int, half_width: int, seed: int) -> CsrMatrix:
    g = gen_lib()
    nnz = 0
    for_rows = np.arange(n)
    lo = np.maximum(0, for_rows - half_width)
    hi = np.minimum(n - 1, for_rows + half_width)
    nnz = int(np.sum(np.minimum(nnz_per_row - 1, hi - lo) + 1))
    rp = np.empty(n + 1, dtype=np.int64)
    ci = np.empty(nnz, dtype=np.int64)
    va = np.empty(nnz, dtype=np.float64)
    rc = g.mstab_gen_banded(n, nnz_per_row, half_width, seed, i64ptr(rp), i64ptr(ci), dptr(va))
    if rc != 0:
        raise ValueError("generator failed")
    return CsrMatrix(n, n, rp, ci, va)


def uniform(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    gen_lib().mstab_gen_uniform(seed, count, dptr(out))
    return out


def normal(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    gen_lib().mstab_gen_normal(seed, count, dptr(out))
    return out


def sinewave(n: int) -> np.ndarray:
    """make_rhs(Sinewave) of the reference harness (harness.cpp:72-77)."""
    out = np.empty(n)
    gen_lib().mstab_gen_sinewave(n, dptr(out))
    return out


def euler_rhs(x: np.ndarray, f: np.ndarray, dt: float, h2: float) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    gen_lib().mstab_gen_euler_rhs(x.size, dptr(x), dptr(np.ascontiguousarray(f)), dt, h2, dptr(out))
    return out


@dataclass
class Config:
    """One BASELINE config (BASELINE.json `configs`)."""
    name: str
    kind: str                  # "convdiff" | "banded"
    s: int
    ell: int
    n_rhs: int
    grid: int = 0
    dim: int = 3
    stencil: int = 7
    beta: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    dt: float = 1e-2
    seed: int = 0
    n: int = 0                 # banded
    nnz_per_row: int = 27
    half_width: int = 4096
    tol: float = 1e-8
    extra: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return self.grid ** self.dim if self.kind == "convdiff" else self.n

    @property
    def h2(self) -> float:
        h = 1.0 / (self.grid + 1)
        return h * h

    def matrix(self) -> CsrMatrix:
        if self.kind == "convdiff":
            return convdiff(self.dim, self.grid, self.stencil, self.beta, self.dt)
        return banded(self.n, self.nnz_per_row, self.half_width, self.seed)

    def sources(self):
        """(x0, f) for conv-diff; (None, None) for banded."""
        if self.kind == "convdiff":
            u = uniform(self.seed, 2 * self.N)
            return u[:self.N].copy(), u[self.N:].copy()
        return None, None

    def first_rhs(self, x0=None, f=None) -> np.ndarray:
        if self.kind == "convdiff":
            return euler_rhs(x0, f, self.dt, self.h2)
        return normal(1000 + self.seed, self.N)

    def next_rhs(self, i: int, x: np.ndarray, f=None) -> np.ndarray:
        """b_{i+1} from x_i (i is the 1-based index of the solve that produced x)."""
        if self.kind == "convdiff":
            return euler_rhs(x, f, self.dt, self.h2)
        return x + 0.1 * normal(1000 + self.seed + i, self.N)


def config(name: str, grid: int = 0) -> Config:
    """BASELINE configs c1..c5 (BASELINE.json `configs`); `grid` overrides the
    grid size for reduced-size parity runs."""
    if name == "c1":
        return Config("c1", "convdiff", s=4, ell=2, n_rhs=20, grid=grid or 256, dim=2, stencil=5,
                      beta=(100.0, 100.0, 0.0))
    if name == "c2":
        return Config("c2", "convdiff", s=8, ell=4, n_rhs=50, grid=grid or 128, dim=3, stencil=7,
                      beta=(200.0, 100.0, 50.0))
    if name == "c3":
        return Config("c3", "banded", s=4, ell=2, n_rhs=30, n=grid or 4194304, seed=1)
    if name == "c4":
        return Config("c4", "convdiff", s=8, ell=4, n_rhs=20, grid=grid or 384, dim=3, stencil=27,
                      beta=(500.0, 250.0, 125.0))
    if name == "c5":
        return Config("c5", "convdiff", s=4, ell=2, n_rhs=10, grid=grid or 256, dim=3, stencil=7,
                      beta=(200.0, 100.0, 50.0))
    raise ValueError(name)
