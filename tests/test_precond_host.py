"""Host-side split-preconditioner builds: the product's restatement of
build_jacobi / build_ilu0 (mstab_precond_build, solver.cpp precond_build) against the reference's own
builders (oracle/_ref through the same C-ABI), bit for bit. No device needed: the factorisation is
setup code on the host, like the operator fingerprint."""
import numpy as np
import pytest

import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb
from conftest import REF_LIB


def _libs():
    if not REF_LIB.exists():
        pytest.skip("oracle/_ref not built (make ref)")
    return m.Lib(), m.Lib(REF_LIB)


def _same(a, b):
    return (np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
            and np.array_equal(np.asarray(a.values).view(np.uint64), np.asarray(b.values).view(np.uint64)))


CASES = {
    "tridiag40": lambda: m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 40),
    "convdiff2d_32": lambda: pb.convdiff(2, 32, 5, (100.0, 100.0, 0.0), 1e-2),
    "convdiff3d_12_27pt": lambda: pb.convdiff(3, 12, 27, (500.0, 250.0, 125.0), 1e-2),
    "banded_5000": lambda: pb.banded(5000, 11, 200, 3),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("kind", ["jacobi", "ilu0"])
def test_factor_build_bit_identical_to_reference(name, kind):
    prod, ref = _libs()
    a = CASES[name]()
    build = m.build_jacobi if kind == "jacobi" else m.build_ilu0
    g, r = build(a, prod), build(a, ref)
    assert _same(g.l_factor, r.l_factor)
    assert _same(g.r_factor, r.r_factor)


def test_zero_pivot_and_not_real_on_the_host():
    prod, ref = _libs()
    d = np.eye(6)
    d[3, 3] = 0.0
    a = m.CsrMatrix.from_dense(d + np.diag(np.ones(5), -1))
    rows = []
    for lib in (prod, ref):
        with pytest.raises(m.ZeroPivot) as ei:
            m.build_ilu0(a, lib)
        rows.append(ei.value.row)
    assert rows[0] == rows[1] == 3  # ZeroPivot::row() carried through the C-ABI (errors.hpp:39-45)
    with pytest.raises(m.NotReal):
        m.build_jacobi(m.CsrMatrix.tridiag(1.0, -4.0, 1.0, 8), prod)
