"""Pins for oracle/fft.py and oracle/ops.py against what the paper and mathematics fix
(worked examples, closed forms, dense matrices built from the definitions, a library FFT).
"""
import numpy as np
import pytest

from oracle import dense, fft as offt, ops
from synth import coil_maps2d, line_mask, random_vd_mask2d, rng_for


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# ---------------------------------------------------------------- F
def test_unitary_dft_worked_examples():
    # 4x4 impulse -> 1/4 everywhere; all-ones -> 4 at DC, 0 elsewhere
    imp = np.zeros((4, 4), complex)
    imp[0, 0] = 1
    np.testing.assert_allclose(offt.fftn_u(imp, 2), np.full((4, 4), 0.25), atol=1e-15)
    ones = np.ones((4, 4), complex)
    out = offt.fftn_u(ones, 2)
    ref = np.zeros((4, 4))
    ref[0, 0] = 4
    np.testing.assert_allclose(out, ref, atol=1e-14)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 8, 12, 16, 24, 48, 64, 96, 192])
def test_own_fft_equals_naive_dft(n):
    rng = np.random.default_rng(n)
    x = crandn(rng, 3, n)
    for inv in (False, True):
        a = offt.fft(x, -1, inverse=inv)
        b = offt.dft_naive(x, -1, sign=+1 if inv else -1)
        assert np.linalg.norm(a - b) <= 1e-12 * max(1.0, np.linalg.norm(b))


@pytest.mark.parametrize("n", [128, 192, 256])
def test_own_fft_equals_library_fft(n):
    rng = np.random.default_rng(7)
    x = crandn(rng, 5, n)
    np.testing.assert_allclose(offt.fft(x, -1), np.fft.fft(x, axis=-1), rtol=0, atol=1e-10)
    np.testing.assert_allclose(offt.fft(x, -1, inverse=True), n * np.fft.ifft(x, axis=-1),
                               rtol=0, atol=1e-10)


def test_fft2_against_dense_dft_matrix_and_parseval():
    rng = np.random.default_rng(1)
    x = crandn(rng, 8, 6)
    F = dense.dft_unitary((8, 6))
    np.testing.assert_allclose(offt.fftn_u(x, 2).ravel(), F @ x.ravel(), atol=1e-13)
    assert abs(np.linalg.norm(offt.fftn_u(x, 2)) - np.linalg.norm(x)) < 1e-12
    np.testing.assert_allclose(offt.ifftn_u(offt.fftn_u(x, 2), 2), x, atol=1e-13)
    assert np.max(np.abs(F.conj().T @ F - np.eye(48))) < 1e-12


# ---------------------------------------------------------------- D_x, D_y
def test_diff_worked_example_and_constants():
    col = np.array([1, 2, 3, 4], complex)[:, None] * np.ones((1, 3))
    # [1,2,3,4] -> [1-4, 1, 1, 1]
    np.testing.assert_array_equal(ops.diff(col, 0)[:, 0], [-3, 1, 1, 1])
    c = np.full((5, 6), 2.5 + 1j)
    assert np.all(ops.diff(c, 0) == 0) and np.all(ops.diff(c, 1) == 0)


def test_diff_and_adjoint_against_dense_definition():
    rng = np.random.default_rng(2)
    shape = (6, 5)
    for ax in (0, 1):
        D = dense.diff_matrix(shape, ax)
        x = crandn(rng, *shape)
        np.testing.assert_allclose(ops.diff(x, ax).ravel(), D @ x.ravel(), atol=1e-13)
        np.testing.assert_allclose(ops.diff_adj(x, ax).ravel(), D.T @ x.ravel(), atol=1e-13)


def test_laplacian_first_row_examples():
    # t_1 at (4,4): 4 at origin, -1 at (+-1,0),(0,+-1); (2,2) degenerate
    e = np.zeros((4, 4), complex)
    e[0, 0] = 1
    t1 = ops.tv_normal(e).real   # symmetric operator: first column == first row
    ref = np.zeros((4, 4))
    ref[0, 0] = 4
    ref[1, 0] = ref[3, 0] = ref[0, 1] = ref[0, 3] = -1
    np.testing.assert_array_equal(t1, ref)
    e2 = np.zeros((2, 2), complex)
    e2[0, 0] = 1
    np.testing.assert_array_equal(ops.tv_normal(e2).real, [[4, -2], [-2, 0]])


def test_tv_normal_diagonalised_by_F_closed_form():
    # BCCB diagonalised by F; eigenvalues 4sin^2(pi p/m)+4sin^2(pi q/n)
    shape = (6, 8)
    F = dense.dft_unitary(shape)
    L = sum(dense.diff_matrix(shape, a).T @ dense.diff_matrix(shape, a) for a in (0, 1))
    K = F @ L @ F.conj().T
    p = np.arange(6)[:, None]
    q = np.arange(8)[None, :]
    closed = 4 * np.sin(np.pi * p / 6) ** 2 + 4 * np.sin(np.pi * q / 8) ** 2
    np.testing.assert_allclose(np.diag(K).reshape(shape), closed, atol=1e-12)
    off = K - np.diag(np.diag(K))
    assert np.max(np.abs(off)) < 1e-12


# ---------------------------------------------------------------- W
def test_haar_worked_example_2x2():
    a, b, c, d = 1.0, 2.0, 3.0, 5.0
    x = np.array([[a, b], [c, d]], complex)
    w = ops.haar_fwd(x, 1).real
    # along d0 then d1: LL=(a+b+c+d)/2, LH=(a-b+c-d)/2, HL=(a+b-c-d)/2, HH=(a-b-c+d)/2
    np.testing.assert_allclose(w, [[(a + b + c + d) / 2, (a - b + c - d) / 2],
                                   [(a + b - c - d) / 2, (a - b - c + d) / 2]], atol=1e-15)


@pytest.mark.parametrize("shape,levels", [((8, 8), 1), ((8, 8), 3), ((16, 8), 2), ((4, 4, 8), 2)])
def test_haar_against_dense_matrix_and_unitary(shape, levels):
    nd = len(shape)
    rng = np.random.default_rng(3)
    x = crandn(rng, *shape)
    Wd = dense.haar_matrix(shape, levels)
    np.testing.assert_allclose(ops.haar_fwd(x, levels, nd).ravel(), Wd @ x.ravel(), atol=1e-13)
    assert np.max(np.abs(Wd.T @ Wd - np.eye(Wd.shape[0]))) < 1e-12
    np.testing.assert_allclose(ops.haar_inv(ops.haar_fwd(x, levels, nd), levels, nd), x,
                               atol=1e-13)
    Wo = dense.dense_from_op(lambda v: ops.haar_fwd(v, levels, nd), shape)
    assert np.max(np.abs(Wo.conj().T @ Wo - np.eye(Wo.shape[0]))) < 1e-12


def test_haar_constant_has_zero_details():
    x = np.full((16, 16), 3.0 - 2j)
    w = ops.haar_fwd(x, 3)
    detail = w.copy()
    detail[:2, :2] = 0
    assert np.max(np.abs(detail)) < 1e-12
    assert abs(w[0, 0] - (3.0 - 2j) * 8) < 1e-12  # energy preserved in the coarsest band


# ---------------------------------------------------------------- A
def _small_problem(shape, coils, kind, seed):
    rng = np.random.default_rng(seed)
    sens = coil_maps2d(shape, coils, rng_for(9, seed, 1))
    if kind == "lines":
        mask = line_mask(shape, 2, 2, rng_for(9, seed, 2))
    elif kind == "random":
        mask = (rng.random(shape) < 0.4).astype(np.uint8)
        mask[0, 0] = 1
    else:
        mask = np.ones(shape, np.uint8)
    return sens, mask


@pytest.mark.parametrize("kind", ["lines", "random"])
def test_apply_A_against_dense_system_matrix(kind):
    sens, mask = _small_problem((8, 8), 3, kind, 4)
    mu, lam, gamma = 1e-3, 4e-3, 1e-3
    A = dense.system_matrix(sens, mask, mu, lam, gamma)
    rng = np.random.default_rng(5)
    x = crandn(rng, 8, 8)
    np.testing.assert_allclose(ops.apply_A(x, sens, mask, mu, lam, gamma).ravel(), A @ x.ravel(),
                               rtol=0, atol=1e-13 * np.linalg.norm(A @ x.ravel()) + 1e-15)
    assert np.max(np.abs(A - A.conj().T)) < 1e-14
    assert np.min(np.linalg.eigvalsh(A)) >= gamma - 1e-12


def test_apply_A_3d_against_dense():
    rng = np.random.default_rng(11)
    shape = (4, 4, 6)
    sens = crandn(rng, 2, *shape)
    sens /= np.sqrt(np.sum(np.abs(sens) ** 2, axis=0))[None]
    mask = np.repeat((rng.random((1, 4, 6)) < 0.5), 4, axis=0).astype(np.uint8)
    A = dense.system_matrix(sens, mask, 1.0, 0.05, 0.02)
    x = crandn(rng, *shape)
    np.testing.assert_allclose(ops.apply_A(x, sens, mask, 1.0, 0.05, 0.02).ravel(), A @ x.ravel(),
                               atol=1e-12)


def test_apply_A_invariants():
    sens, mask = _small_problem((16, 16), 4, "lines", 6)
    rng = np.random.default_rng(6)
    u, v = crandn(rng, 16, 16), crandn(rng, 16, 16)
    Av = ops.apply_A(v, sens, mask, 1.0, 0.05, 0.05)
    Au = ops.apply_A(u, sens, mask, 1.0, 0.05, 0.05)
    assert abs(np.vdot(u, Av) - np.vdot(Au, v)) <= 1e-12 * np.linalg.norm(u) * np.linalg.norm(v)
    xAx = np.vdot(u, Au)
    assert abs(xAx.imag) < 1e-10 and xAx.real >= 0.05 * np.linalg.norm(u) ** 2 - 1e-10
    np.testing.assert_allclose(ops.apply_A(u, sens, mask, 0.0, 0.0, 0.7), 0.7 * u, atol=1e-15)
    # E^H is the adjoint of E
    y = crandn(rng, 4, 16, 16)
    lhs = np.vdot(ops.encode(u, sens, mask), y)
    rhs = np.vdot(u, ops.encode_adj(y, sens, mask))
    assert abs(lhs - rhs) < 1e-10


# ---------------------------------------------------------------- shrink / RSS (Alg. 1)
def test_shrink_examples():
    # SPEC.md:389-391
    assert abs(ops.shrink(np.array([3 + 4j]), 2.0)[0] - (1.8 + 2.4j)) < 1e-15
    assert ops.shrink(np.array([0j]), 1.0)[0] == 0
    z = np.array([0.3 + 0.4j, 1 + 0j, -2j])
    np.testing.assert_array_equal(ops.shrink(z, 2.0), 0)
    rng = np.random.default_rng(8)
    a, b = crandn(rng, 100), crandn(rng, 100)
    assert np.all(np.abs(ops.shrink(a, 0.7) - ops.shrink(b, 0.7)) <= np.abs(a - b) + 1e-15)


def test_rss_init_special_cases():
    rng = np.random.default_rng(9)
    xt = rng.random((8, 8))
    y = offt.fftn_u(xt, 2)[None]
    np.testing.assert_allclose(ops.rss_init(y).real, xt, atol=1e-13)
    y2 = np.concatenate([y, y])
    np.testing.assert_allclose(ops.rss_init(y2).real, np.sqrt(2) * xt, atol=1e-13)


def test_synth_masks_counts():
    m = line_mask((256, 256), 4, 24, rng_for(2, 0, 2))
    assert m[:, 0].sum() == 64 and np.all(m == m[:, :1])
    assert np.all(m[(np.arange(24) - 12) % 256, 0] == 1)
    m1 = line_mask((64, 64), 4, 8, rng_for(1, 0, 2))
    assert m1[:, 0].sum() == 16
    m4 = random_vd_mask2d((256, 128), 6, 24, rng_for(4, 0, 2))
    assert m4.sum() == (256 * 128) // 6
    assert np.all(m4[np.ix_((np.arange(24) - 12) % 256, (np.arange(24) - 12) % 128)] == 1)


# ------------------------------------------------------- Daubechies-4 W (reading A32)
@pytest.mark.parametrize("shape,levels", [((8, 8), 1), ((16, 8), 2), ((8, 16), 3), ((8, 4, 8), 2)])
def test_d4_is_orthonormal_dense(shape, levels):
    nd = len(shape)
    Wd = dense.dense_from_op(lambda v: ops.d4_fwd(v, levels, nd), shape)
    assert np.allclose(Wd.conj().T @ Wd, np.eye(Wd.shape[0]), atol=1e-12)
    x = np.random.default_rng(2).standard_normal(shape) + 1j * np.random.default_rng(3).standard_normal(shape)
    assert np.allclose(ops.d4_inv(ops.d4_fwd(x, levels, nd), levels, nd), x, atol=1e-12)


def test_d4_filter_identities_and_worked_examples():
    h, g = ops.D4_H, np.array([ops.D4_H[3], -ops.D4_H[2], ops.D4_H[1], -ops.D4_H[0]])
    assert np.isclose(h.sum(), np.sqrt(2)) and np.isclose(np.sum(h ** 2), 1.0)   # normalisation
    assert np.isclose(g.sum(), 0) and np.isclose(np.sum(np.arange(4) * g), 0)    # 2 vanishing moments
    assert np.isclose(h[0] * h[2] + h[1] * h[3], 0)                               # shift orthogonality
    # impulse at 0, n = 4 (1D via a 4x1 image along d0): a = (h0, h2), d = (g0, g2)
    x = np.zeros((4, 1), complex)
    x[0, 0] = 1
    c = ops._d4_axis_fwd(x, 0)[:, 0]
    assert np.allclose(c, [h[0], h[2], g[0], g[2]])
    # n = 2 reduces to the orthonormal Haar (the filter wraps twice)
    y = np.array([[3.0 + 1j], [1.0 - 2j]])
    assert np.allclose(ops._d4_axis_fwd(y, 0), ops._haar_axis_fwd(y, 0))
    # constants have zero detail coefficients at every level
    w = ops.d4_fwd(np.full((16, 16), 2.5 + 0.5j), 3)
    mask = np.zeros((16, 16), bool)
    mask[:2, :2] = True
    assert np.max(np.abs(w[~mask])) < 1e-12


def test_sb_with_d4_reduces_to_least_squares_when_thresholds_are_huge():
    # with both weights tiny the thresholds 1/lambda, 1/gamma are huge, every shrink returns 0,
    # and W enters the iteration only through W^H W = I (b_w = W x, W^H b_w = x): Haar and D4
    # must give the same SB iterates
    import synth
    from oracle import problems, sb
    p = synth.problem2d(1, 0, shape=(16, 16), coils=2)
    y = problems.make_kspace(p["phantom"], p["sens"], p["mask"], p["noise"])
    xa, _ = sb.sb_recon(y, p["sens"], p["mask"], 1.0, 1e-6, 1e-6, 3, 1, 2, 0.0, 40, "circulant", wavelet="haar")
    xb, _ = sb.sb_recon(y, p["sens"], p["mask"], 1.0, 1e-6, 1e-6, 3, 1, 2, 0.0, 40, "circulant", wavelet="d4")
    assert np.allclose(xa, xb, atol=1e-10 * np.abs(xa).max())
