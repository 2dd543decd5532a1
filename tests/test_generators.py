"""Builder-defined BASELINE generators (include/mstab_gen.h) — CPU only."""
import numpy as np
import pytest

from paper_1604_06043_b200 import problems as pb


@pytest.mark.parametrize("dim,n,st", [(2, 7, 5), (3, 5, 7), (3, 4, 27)])
def test_convdiff_structure(dim, n, st):
    A = pb.convdiff(dim, n, st, (3.0, 2.0, 1.0), 1e-2)
    N = n ** dim
    assert A.n_rows == N and A.nnz() == len(A.col_idx)
    expect = {5: 5 * n * n - 4 * n, 7: 7 * n ** 3 - 6 * n ** 2, 27: (3 * n - 2) ** 3}[st]
    assert A.nnz() == expect
    rp = A.row_ptr
    assert rp[0] == 0 and rp[-1] == A.nnz() and np.all(np.diff(rp) >= 1)
    for i in range(N):  # strictly increasing columns, diagonal present
        cols = A.col_idx[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0) and i in cols


def test_convdiff_h2_scaled_coefficients():
    n, beta, dt = 8, (100.0, 50.0, 25.0), 1e-2
    A = pb.convdiff(3, n, 7, beta, dt).to_dense()
    h = 1.0 / (n + 1)
    i = (3 * n + 3) * n + 3  # interior point
    assert A[i, i] == pytest.approx(h * h / dt + 6 + h * sum(beta), rel=1e-15)
    assert A[i, i - 1] == pytest.approx(-1 - h * beta[0], rel=1e-15)   # upwind x
    assert A[i, i - n] == pytest.approx(-1 - h * beta[1], rel=1e-15)
    assert A[i, i - n * n] == pytest.approx(-1 - h * beta[2], rel=1e-15)
    assert A[i, i + 1] == A[i, i + n] == A[i, i + n * n] == -1.0
    assert np.all(np.abs(A).sum(axis=1) <= 2 * np.diag(A) + 1e-12)  # weakly diagonally dominant


def test_27pt_is_consistent_laplacian():
    A = pb.convdiff(3, 6, 27, (0.0, 0.0, 0.0), 1e30).to_dense()
    i = (2 * 6 + 2) * 6 + 2
    assert A[i].sum() == pytest.approx(0.0, abs=1e-12)  # interior row of -Laplace sums to 0


def test_sources_and_rhs_are_deterministic():
    cfg = pb.config("c1", grid=16)
    x0, f = cfg.sources()
    x1, f1 = cfg.sources()
    assert np.array_equal(x0, x1) and np.array_equal(f, f1)
    assert x0.min() >= 0 and x0.max() < 1 and f.min() >= 0 and f.max() < 1
    b = cfg.first_rhs(x0, f)
    assert np.array_equal(b, cfg.h2 * (x0 / cfg.dt + f))


def test_banded_generator():
    A = pb.banded(3000, 27, 64, 1)
    rp, ci, va = A.row_ptr, A.col_idx, A.values
    for i in range(0, 3000, 97):
        cols = ci[rp[i]:rp[i + 1]]
        vals = va[rp[i]:rp[i + 1]]
        assert len(cols) == 27 and np.all(np.diff(cols) > 0) and np.all(np.abs(cols - i) <= 64)
        d = vals[cols == i][0]
        assert d == pytest.approx(1.1 * np.abs(vals[cols != i]).sum(), rel=1e-15)
        assert np.all((vals[cols != i] >= -1) & (vals[cols != i] < 1))


def test_configs_match_baseline_shapes():
    assert pb.config("c1").N == 65536
    assert pb.config("c2").N == 2097152 and pb.config("c2").s == 8 and pb.config("c2").ell == 4
    assert pb.config("c3").N == 4194304
    assert pb.config("c4").N == 56623104
    assert pb.config("c5").N == 16777216
    assert pb.convdiff(2, 256, 5, (100, 100), 1e-2).nnz() == 326656
