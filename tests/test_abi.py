"""The C-ABI boundary (CPU only): both implementations load and export every function that
include/*.h declares, the product fails loudly without a GPU, and the Python mirror keeps the
reference's names and error classes."""
import ctypes
import re
from pathlib import Path

import pytest

from conftest import REF_LIB, ROOT

HEADERS = ["mstab_b200.h", "mstab_b200_kernels.h"]


def declared(header):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mstab_[a-z0-9_]+)\s*\(", text)))


def test_headers_declare_the_entry_points():
    names = declared("mstab_b200.h")
    for must in ("mstab_solve", "mstab_operator_create_csr", "mstab_recycle_validate", "mstab_recycle_save",
                 "mstab_recycle_load", "mstab_result_handoff", "mstab_operator_apply"):
        assert must in names


@pytest.mark.parametrize("lib", ["product", "reference"])
def test_library_exports_every_declared_symbol(lib):
    from paper_1604_06043_b200._capi import PRODUCT_LIB
    path = PRODUCT_LIB if lib == "product" else REF_LIB
    if not Path(path).exists():
        pytest.skip(f"{path} not built")
    dll = ctypes.CDLL(str(path))
    for h in HEADERS:
        for name in declared(h):
            assert hasattr(dll, name), f"{path.name} misses {name} ({h})"


def test_generator_library_exports():
    from paper_1604_06043_b200._capi import GEN_LIB
    dll = ctypes.CDLL(str(GEN_LIB))
    for name in declared("mstab_gen.h"):
        assert hasattr(dll, name), name


def test_product_loads_and_names_itself():
    import paper_1604_06043_b200 as m
    lib = m.Lib()
    assert lib.name == "b200"


def test_product_fails_loudly_without_a_device():
    import torch

    import paper_1604_06043_b200 as m
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(m.CudaError):
        m.Context(m.Lib())


def test_missing_library_is_an_error(tmp_path):
    import paper_1604_06043_b200 as m
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        m.Lib(tmp_path / "libmissing.so")


def test_reference_mirror_names():
    import paper_1604_06043_b200 as m
    assert issubclass(m.SingularProjection, m.BreakdownError) and issubclass(m.RankDeficient, m.BreakdownError)
    for cls in (m.DimensionMismatch, m.FingerprintMismatch, m.StaleData, m.ParseError, m.IoError, m.ConfigError):
        assert issubclass(cls, m.Error)
    cfg = m.SolverConfig()
    assert (cfg.s, cfg.ell, cfg.tol, cfg.max_mv, cfg.true_residual_each_cycle, cfg.seed) == (2, 1, 1e-8, 100000,
                                                                                          False, 0)
    with pytest.raises(m.ConfigError):
        m.FetchPolicy.at_cycle(0)


def test_reference_impl_runs_through_the_same_abi(ref_ctx):
    """The boundary is implementation-neutral: the reference drives the same calls on the host."""
    import numpy as np

    import paper_1604_06043_b200 as m
    op = m.CsrOperator(m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 40), ref_ctx)
    r = m.idrstab_solve(op, np.ones(40), None, m.SolverConfig(2, 1, 1e-8, 100000, True, 1))
    assert (r.report.cycles, r.report.h_mv, r.report.status) == (20, 62, m.CONVERGED)
    # the host-only implementation rejects device pointers with ConfigError
    assert ref_ctx.lib.dll.mstab_operator_apply(ref_ctx.h, op.h, None, None, 1) == -3


def test_reference_adjoint_and_bicg_through_the_abi(ref_ctx):
    """apply_adjoint and bicg_solve on the reference side of the ABI (the oracle the B200 path is
    checked against): A^H x equals the sequential scatter of csr.cpp:115-124, and BiCG on an SPD
    diagonal system converges in at most n iterations like CG (test_solvers.cpp:483-500)."""
    import numpy as np

    import paper_1604_06043_b200 as m
    A = m.CsrMatrix.from_triplets(5, 5, [(0, 0, 2.0), (0, 3, -1.0), (1, 1, 3.0), (2, 0, 0.5), (2, 2, 4.0),
                                         (3, 1, 1.5), (3, 3, 1.0), (4, 2, -2.0), (4, 4, 5.0)])
    op = m.CsrOperator(A, ref_ctx)
    x = np.array([1.0, -2.0, 0.25, 3.0, -0.5])
    y = np.zeros(5)
    for i in range(5):  # y[col] += a_ik x_i, rows ascending
        for k in range(int(A.row_ptr[i]), int(A.row_ptr[i + 1])):
            y[int(A.col_idx[k])] += A.values[k] * x[i]
    assert np.array_equal(op.apply_adjoint(x), y)
    d = m.CsrMatrix.from_triplets(8, 8, [(i, i, float(i + 1)) for i in range(8)])
    xs, rep = m.bicg_solve(m.CsrOperator(d, ref_ctx), np.ones(8), None, 1e-12, 1000)
    assert rep.status == m.CONVERGED and rep.cycles <= 8
    assert np.allclose(xs, 1.0 / np.arange(1, 9), rtol=1e-10)
