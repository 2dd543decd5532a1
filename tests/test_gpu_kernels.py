"""Kernel-level parity of the sm_100a code against the oracles (run on a B200: -m gpu).

Bar: bit-exact where the reference's operation order is reproduced (SpMV, the s x s LU solve,
the FNV fingerprint, the cut-space draws), tight tolerances for the reductions that are trees on
the GPU and sequential sums in the reference (least squares, Gram-Schmidt)."""
import numpy as np
import pytest

import oracle_c as oc
import paper_1604_06043_b200 as m
from paper_1604_06043_b200 import problems as pb

pytestmark = pytest.mark.gpu


def matrices():
    yield "tridiag40", m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 40)
    yield "c1_64", pb.config("c1", grid=64).matrix()
    yield "c2_24", pb.config("c2", grid=24).matrix()
    yield "c4_12_27pt", pb.config("c4", grid=12).matrix()
    # one perturbed entry: not constant-diagonal any more -> the value-streaming DIA form
    c2p = pb.config("c2", grid=24).matrix()
    c2p.values = c2p.values.copy()
    c2p.values[777] *= 1.0 + 2.0 ** -30
    yield "c2_24_perturbed", c2p
    # variable coefficients on a stencil pattern (DIA form) and an explicit stored zero
    c1v = pb.config("c1", grid=32).matrix()
    c1v.values = c1v.values * (1.0 + 0.01 * np.sin(np.arange(c1v.values.size)))
    yield "c1_32_varcoef", c1v
    yield "explicit_zero", m.CsrMatrix.from_triplets(
        4, 4, [(0, 0, 2.0), (0, 1, 0.0), (1, 1, 2.0), (1, 2, 0.0), (2, 2, 2.0), (2, 3, 0.0), (3, 3, 2.0)])
    c3 = pb.config("c3", grid=20000)
    c3.half_width = 512
    yield "c3_20000", c3.matrix()
    # ragged rows: an empty row, a dense row, single entries
    yield "ragged", m.CsrMatrix.from_triplets(
        6, 6, [(0, 0, 2.0), (1, 0, 1.0), (1, 1, 3.0), (1, 2, -1.0), (1, 3, 0.5), (1, 4, 0.25), (1, 5, 4.0),
               (3, 3, 1.5), (4, 1, -2.0), (5, 5, 1.0)])


@pytest.mark.parametrize("name,A", list(matrices()), ids=[n for n, _ in matrices()])
def test_spmv_bit_exact_and_fingerprint(gpu_ctx, name, A):
    op = m.CsrOperator(A, gpu_ctx)
    c = oc.Csr(A)
    assert op.fingerprint() == c.fingerprint()
    rng = np.random.default_rng(3)
    for _ in range(2):
        x = rng.standard_normal(A.n_rows)
        assert np.array_equal(op.apply(x), c.apply(x))


@pytest.mark.parametrize("name,A", list(matrices()), ids=[n for n, _ in matrices()])
def test_spmv_adjoint_bit_exact(gpu_ctx, ref_ctx, name, A):
    """A^H x through the device transpose vs the reference's scatter (csr.cpp:115-124), bit for bit."""
    op = m.CsrOperator(A, gpu_ctx)
    ref = m.CsrOperator(A, ref_ctx)
    rng = np.random.default_rng(4)
    for _ in range(2):
        x = rng.standard_normal(A.n_rows)
        assert np.array_equal(op.apply_adjoint(x), ref.apply_adjoint(x))
    assert np.array_equal(op.apply(x), ref.apply(x))  # the forward product is untouched


def test_solve_small_bit_exact(gpu_ctx, golden_kernels):
    g = golden_kernels
    for s in (1, 2, 3, 4, 8, 16):
        assert np.array_equal(m.solve_small(g[f"lu{s}_m"], g[f"lu{s}_rhs"], gpu_ctx), g[f"lu{s}_x"])
    rng = np.random.default_rng(9)
    for s in range(1, 17):
        M = rng.standard_normal((s, s)) * 10.0 ** rng.uniform(-3, 3, size=(s, s))
        r = rng.standard_normal(s)
        assert np.array_equal(m.solve_small(M, r, gpu_ctx), oc.solve_small(M, r))
    with pytest.raises(m.SingularProjection):
        m.solve_small(g["lu_sing_m"], np.ones(3), gpu_ctx)
    with pytest.raises(m.SingularProjection):
        m.solve_small(np.zeros((4, 4)), np.ones(4), gpu_ctx)


def test_least_squares_tsqr(gpu_ctx, golden_kernels):
    g = golden_kernels
    for n, ell in ((50, 1), (300, 2), (1000, 4), (4000, 8)):
        t = m.least_squares_tall(g[f"ls{n}_{ell}_z"], g[f"ls{n}_{ell}_r"], gpu_ctx)
        ref = g[f"ls{n}_{ell}_tau"]
        assert np.linalg.norm(t - ref) <= 1e-12 * np.linalg.norm(ref)
    # ill-conditioned Krylov power basis (the stabilisation block of a cycle)
    t = m.least_squares_tall(g["lsk_z"], g["lsk_r"], gpu_ctx)
    ref = g["lsk_tau"]
    cond = np.linalg.cond(g["lsk_z"])
    assert np.linalg.norm(t - ref) <= 1e-15 * cond * np.linalg.norm(ref) * 10
    with pytest.raises(m.RankDeficient):
        m.least_squares_tall(g["lsdef_z"], g["lsdef_r"], gpu_ctx)
    with pytest.raises(m.DimensionMismatch):
        m.least_squares_tall(np.ones((2, 3)), np.ones(2), gpu_ctx)
    # large N (many CTAs in the TSQR merge tree)
    rng = np.random.default_rng(4)
    Z = rng.standard_normal((1_000_003, 4))
    r = rng.standard_normal(1_000_003)
    t = m.least_squares_tall(Z, r, gpu_ctx)
    ref = np.linalg.lstsq(Z, r, rcond=None)[0]
    assert np.linalg.norm(t - ref) <= 1e-12 * np.linalg.norm(ref)


def test_cut_space_and_arnoldi(gpu_ctx, golden_kernels):
    g = golden_kernels
    for n, s, seed in ((257, 1, 0), (257, 3, 7), (1000, 4, 11), (64, 8, 99)):
        P = m.make_cut_space(n, s, seed, gpu_ctx)
        assert np.max(np.abs(P - g[f"cut{n}_{s}_{seed}"])) <= 1e-13
        assert np.max(np.abs(P.T @ P - np.eye(s))) <= 1e-13
    op = m.CsrOperator(m.CsrMatrix.tridiag(2.0, 3.0, 1.0, 8), gpu_ctx)
    u, v, mv = m.arnoldi_init(op, np.ones(8), 3, 2)
    assert mv == 3
    assert np.max(np.abs(u - g["arn_tri_u"])) <= 1e-13 and np.max(np.abs(v - g["arn_tri_v"])) <= 1e-12
    # happy breakdown: Krylov space of e1 under I has dimension 1 < s -> seeded Gaussian padding
    ope = m.CsrOperator(m.CsrMatrix.identity(6), gpu_ctx)
    u, v, _ = m.arnoldi_init(ope, np.eye(6)[0], 3, 4)
    assert np.max(np.abs(u - g["arn_eye_u"])) <= 1e-13
    assert np.max(np.abs(u.T @ u - np.eye(3))) <= 1e-12


@pytest.mark.parametrize("ell", [1, 2, 4, 8])
def test_least_squares_cholqr2_tall(gpu_ctx, ell):
    """Tall systems (n >= 2^17) take the CholeskyQR2 path; checked against LAPACK's QR
    least-squares solution (numpy.linalg.lstsq) at the conditioning bound of the method."""
    rng = np.random.default_rng(100 + ell)
    n = 1 << 18
    z = rng.standard_normal((n, ell)) * np.logspace(0, -2, ell)
    r = z @ rng.standard_normal(ell) + 0.3 * rng.standard_normal(n)
    t = m.least_squares_tall(z, r, gpu_ctx)
    ref = np.linalg.lstsq(z, r, rcond=None)[0]
    cond = np.linalg.cond(z)
    assert np.linalg.norm(t - ref) <= 1e-14 * cond * np.linalg.norm(ref) * 10


def test_least_squares_tall_fallback_ill_conditioned(gpu_ctx):
    """A tall power basis too ill-conditioned for CholeskyQR2 falls back to the Givens TSQR in the
    same launch and still matches LAPACK to cond * eps."""
    from paper_1604_06043_b200 import problems as pb
    A = pb.config("c1", grid=512).matrix()   # N = 262144
    op = m.CsrOperator(A, gpu_ctx)
    rng = np.random.default_rng(5)
    v = rng.standard_normal(A.n_rows)
    cols = [v]
    for _ in range(6):
        cols.append(op.apply(cols[-1]))
    z = np.stack(cols[1:], axis=1)
    r = cols[0]
    cond = np.linalg.cond(z)
    assert cond > 1e4  # beyond the CholeskyQR2 acceptance bound
    t = m.least_squares_tall(z, r, gpu_ctx)
    ref = np.linalg.lstsq(z, r, rcond=None)[0]
    assert np.linalg.norm(t - ref) <= 1e-15 * cond * np.linalg.norm(ref) * 10
