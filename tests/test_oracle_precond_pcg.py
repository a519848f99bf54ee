"""Pins for oracle/precond.py and oracle/pcg.py."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import dense, ops, precond
from oracle.pcg import PcgError, pcg
from synth import coil_maps2d, line_mask, rng_for


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _problem(shape, coils, kind, seed, normalise=True):
    rng = np.random.default_rng(seed)
    if normalise:
        sens = coil_maps2d(shape, coils, rng_for(8, seed, 1))
    else:
        sens = crandn(rng, coils, *shape)
    if kind == "lines":
        mask = line_mask(shape, 2, 2, rng_for(8, seed, 2))
    elif kind == "random":
        mask = (rng.random(shape) < 0.35).astype(np.uint8)
        mask[0, 0] = 1
    else:
        mask = np.ones(shape, np.uint8)
    return sens, mask


# ------------------------------------------------------- k = diag(F A F^H)
@pytest.mark.parametrize("n", [4, 8, 16])
@pytest.mark.parametrize("coils", [1, 2, 4])
@pytest.mark.parametrize("kind", ["lines", "random"])
def test_k_equals_diag_of_dense_K(n, coils, kind):
    sens, mask = _problem((n, n), coils, kind, 10 * n + coils, normalise=False)
    mu, lam, gamma = 1.0, 0.05, 0.02
    A = dense.system_matrix(sens, mask, mu, lam, gamma)
    F = dense.dft_unitary((n, n))
    K = F @ A @ F.conj().T
    k = precond.build_k(sens, mask, mu, lam, gamma)
    np.testing.assert_allclose(k.ravel(), np.diag(K).real, rtol=1e-10, atol=1e-12)
    assert np.max(np.abs(np.diag(K).imag)) < 1e-12


def test_k_c_paper_equals_direct_correlation_sum():
    for shape, seed in (((16, 16), 1), ((64, 64), 2)):
        sens, mask = _problem(shape, 3, "random", seed, normalise=False)
        np.testing.assert_allclose(precond.k_c_paper(sens, mask).real,
                                   precond.k_c_direct(sens, mask), rtol=1e-11, atol=1e-12)


def test_k_c_dropping_the_transpose_is_wrong_for_complex_maps():
    # The (.)^T of PAPER.md:219 matters: without the index reversal the result differs for
    # complex (non-even |F s|^2) maps, which is why the pin above uses complex maps.
    sens, mask = _problem((8, 8), 3, "random", 3, normalise=False)
    nd = 2
    hat = precond.dft_n(sens, nd)
    g = np.sum(np.abs(hat) ** 2, axis=0) / 64.0 ** 2
    wrong = precond.idft_n(precond.dft_n(g, nd) * precond.dft_n(mask.astype(float), nd), nd).real
    good = precond.k_c_paper(sens, mask).real
    assert np.linalg.norm(wrong - good) > 1e-3 * np.linalg.norm(good)


def test_k_c_special_cases():
    # single all-ones coil: full mask -> 1; any mask -> r
    ones = np.ones((1, 8, 8), complex)
    full = np.ones((8, 8), np.uint8)
    np.testing.assert_allclose(precond.k_c_paper(ones, full).real, 1.0, atol=1e-13)
    rng = np.random.default_rng(4)
    r = (rng.random((8, 8)) < 0.5).astype(np.uint8)
    np.testing.assert_allclose(precond.k_c_paper(ones, r).real, r, atol=1e-13)


def test_k_c_full_size_invariants():
    # With sum_c |s_c|^2 = 1: mean(k_c) = sampled fraction f (trace identity); full mask ->
    # E^H E = I -> k_c = 1 (SURVEY 8(c) full-size invariants (i), (ii)).
    shape = (64, 64)
    sens = coil_maps2d(shape, 8, rng_for(2, 5, 1))
    mask = line_mask(shape, 4, 8, rng_for(2, 5, 2))
    kc = precond.k_c_paper(sens, mask).real
    assert abs(kc.mean() - mask.mean()) < 1e-12
    np.testing.assert_allclose(precond.k_c_paper(sens, np.ones(shape, np.uint8)).real, 1.0,
                               atol=1e-12)


def test_k_d_closed_form_and_fft_of_t1():
    for shape in ((4, 4), (6, 8), (2, 2), (4, 4, 6)):
        kd = precond.k_d_closed(shape)
        np.testing.assert_allclose(precond.k_d_fft(shape).real, kd, atol=1e-12)
        assert kd[(0,) * len(shape)] == 0.0
    kd = precond.k_d_closed((8, 6))
    assert abs(kd[4, 3] - 8.0) < 1e-14


def test_apply_Minv_against_dense():
    sens, mask = _problem((8, 8), 3, "lines", 5)
    k = precond.build_k(sens, mask, 1.0, 0.05, 0.05)
    F = dense.dft_unitary((8, 8))
    Md = F.conj().T @ np.diag(1.0 / k.ravel()) @ F
    rng = np.random.default_rng(5)
    v = crandn(rng, 8, 8)
    np.testing.assert_allclose(precond.apply_Minv(v, k).ravel(), Md @ v.ravel(), atol=1e-12)
    Mfwd = lambda u: ops.ifftn_u(ops.fftn_u(u, 2) * k, 2)  # noqa: E731
    np.testing.assert_allclose(precond.apply_Minv(Mfwd(v), k), v, atol=1e-12)


def test_constant_coil_maps_make_Minv_exact():
    # with S_i = I (here spatially constant maps) K is diagonal and
    # A^{-1} = F^H K^{-1} F exactly.
    shape = (16, 16)
    rng = np.random.default_rng(6)
    ph = np.exp(1j * rng.uniform(0, 2 * np.pi, 3))
    sens = (ph / np.sqrt(3))[:, None, None] * np.ones((3,) + shape)
    mask = line_mask(shape, 4, 4, rng_for(8, 6, 2))
    mu, lam, gamma = 1.0, 0.05, 0.02
    k = precond.build_k(sens, mask, mu, lam, gamma)
    b = crandn(rng, *shape)
    AMb = ops.apply_A(precond.apply_Minv(b, k), sens, mask, mu, lam, gamma)
    assert np.linalg.norm(AMb - b) / np.linalg.norm(b) < 1e-13
    res = pcg(lambda v: ops.apply_A(v, sens, mask, mu, lam, gamma), b, np.zeros(shape, complex),
              lambda v: precond.apply_Minv(v, k), 1e-10, 20)
    assert res.iters == 1 and res.converged


def test_preconditioner_clusters_eigenvalues():
    # M^{-1}A ~ I ("cluster the eigenvalues ... around 1"); K has less
    # off-diagonal mass than A; Jacobi does not help (with sum|s|^2 = 1 the
    # diagonal of A is constant, so Jacobi is a pure rescaling).
    shape = (16, 16)
    sens = coil_maps2d(shape, 4, rng_for(8, 7, 1))
    mask = line_mask(shape, 4, 4, rng_for(8, 7, 2))
    F = dense.dft_unitary(shape)
    for (mu, lam, gamma), bound in (((1e-3, 4e-3, 1e-3), 2.0), ((1.0, 0.05, 0.05), None)):
        A = dense.system_matrix(sens, mask, mu, lam, gamma)
        k = precond.build_k(sens, mask, mu, lam, gamma)
        Mh = F.conj().T @ np.diag(k.ravel() ** -0.5) @ F    # M^{-1/2}
        ev_A = np.linalg.eigvalsh(A)
        ev_P = np.linalg.eigvalsh(Mh @ A @ Mh)
        kap_A, kap_P = ev_A[-1] / ev_A[0], ev_P[-1] / ev_P[0]
        assert kap_P < kap_A
        if bound is not None:   # paper set 1: kappa 17 -> ~1.2
            assert kap_P < bound and kap_A > 10
            assert ev_P[0] > 0.5 and ev_P[-1] < 1.5
        Dj = np.diag(A).real ** -0.5
        ev_J = np.linalg.eigvalsh(Dj[:, None] * A * Dj[None, :])
        assert abs(ev_J[-1] / ev_J[0] - kap_A) < 1e-6 * kap_A
        K = F @ A @ F.conj().T
        off = lambda X: np.linalg.norm(X - np.diag(np.diag(X))) / np.linalg.norm(X)  # noqa
        assert off(K) < off(A)


def test_jacobi_diag_against_dense():
    sens, mask = _problem((8, 8), 3, "random", 9, normalise=False)
    A = dense.system_matrix(sens, mask, 1e-3, 4e-3, 1e-3)
    np.testing.assert_allclose(precond.jacobi_diag(sens, mask, 1e-3, 4e-3, 1e-3).ravel(),
                               np.diag(A).real, rtol=1e-12)


# ------------------------------------------------------- PCG
def test_pcg_matches_dense_solve():
    sens, mask = _problem((8, 8), 3, "lines", 11)
    mu, lam, gamma = 1.0, 0.05, 0.02
    A = dense.system_matrix(sens, mask, mu, lam, gamma)
    rng = np.random.default_rng(11)
    b = crandn(rng, 8, 8)
    xd = np.linalg.solve(A, b.ravel())
    k = precond.build_k(sens, mask, mu, lam, gamma)
    for Minv in (None, lambda v: precond.apply_Minv(v, k)):
        res = pcg(lambda v: ops.apply_A(v, sens, mask, mu, lam, gamma), b,
                  np.zeros((8, 8), complex), Minv, 1e-13, 500)
        assert res.converged
        assert np.linalg.norm(res.x.ravel() - xd) <= 1e-8 * np.linalg.norm(xd)


def test_pcg_special_cases():
    rng = np.random.default_rng(12)
    b = crandn(rng, 6, 6)
    I = lambda v: v  # noqa: E731
    res = pcg(I, b, np.zeros_like(b), None, 1e-12, 10)
    assert res.iters == 1 and np.allclose(res.x, b)
    res0 = pcg(I, np.zeros_like(b), b, None, 1e-3, 10)
    assert res0.iters == 0 and res0.converged and np.all(res0.x == 0)
    # M = exact inverse -> 1 iteration
    sens, mask = _problem((6, 6), 2, "lines", 12)
    A = dense.system_matrix(sens, mask, 1.0, 0.05, 0.05)
    Ainv = np.linalg.inv(A)
    res = pcg(lambda v: (A @ v.ravel()).reshape(6, 6), b, np.zeros_like(b),
              lambda v: (Ainv @ v.ravel()).reshape(6, 6), 1e-10, 10)
    assert res.iters == 1
    with pytest.raises(PcgError):
        pcg(lambda v: -v, b, np.zeros_like(b), None, 1e-6, 5)
    with pytest.raises(PcgError):
        pcg(lambda v: v * np.nan, b, np.zeros_like(b), None, 1e-6, 5)


def test_pcg_without_preconditioner_matches_library_cg():
    # M = I is plain CG: compare x_k with scipy's CG after the same number of iterations
    sens, mask = _problem((8, 8), 3, "random", 13)
    mu, lam, gamma = 1.0, 0.05, 0.02
    A = dense.system_matrix(sens, mask, mu, lam, gamma)
    rng = np.random.default_rng(13)
    b = crandn(rng, 8, 8)
    for it in (1, 3, 7):
        ours = pcg(lambda v: (A @ v.ravel()).reshape(8, 8), b, np.zeros_like(b), None, 0.0, it)
        op = spla.LinearOperator(A.shape, matvec=lambda v: A @ v, dtype=complex)
        ref, _ = spla.cg(op, b.ravel(), x0=np.zeros(64, complex), rtol=1e-300, atol=0, maxiter=it)
        np.testing.assert_allclose(ours.x.ravel(), ref, rtol=1e-9, atol=1e-12)


def test_pcg_scaling_invariance():
    sens, mask = _problem((8, 8), 2, "lines", 14)
    rng = np.random.default_rng(14)
    b = crandn(rng, 8, 8)
    out = []
    for s in (1.0, 8.0):
        mu, lam, gamma = s * 1.0, s * 0.05, s * 0.02
        k = precond.build_k(sens, mask, mu, lam, gamma)
        out.append(pcg(lambda v: ops.apply_A(v, sens, mask, mu, lam, gamma), b,
                       np.zeros_like(b), lambda v: precond.apply_Minv(v, k), 1e-8, 100))
    assert out[0].iters == out[1].iters
    np.testing.assert_allclose(out[0].relres, out[1].relres, rtol=1e-9)
    np.testing.assert_allclose(out[1].x * 8.0, out[0].x, rtol=1e-9, atol=1e-12)


# ------------------------------------------------------- 3D (BASELINE config 5 geometry)
@pytest.mark.parametrize("readout_constant", [True, False])
def test_k_3d_equals_diag_of_dense_K(readout_constant):
    # k = diag(F_3 A F_3^H) in 3D with complex maps, for a mask constant along d0 (config 5;
    # then k_c is constant along nu_0 — the plane-marginal form the GPU builds) and for a
    # generic 3D mask (the oracle's build_k is nd-generic)
    shape = (4, 4, 6)
    rng = np.random.default_rng(31)
    sens = crandn(rng, 2, *shape)
    if readout_constant:
        m2 = (rng.random(shape[1:]) < 0.4).astype(np.uint8)
        m2[0, 0] = 1
        mask = np.repeat(m2[None], shape[0], axis=0)
    else:
        mask = (rng.random(shape) < 0.4).astype(np.uint8)
        mask[0, 0, 0] = 1
    mu, lam, gamma = 1.0, 0.05, 0.02
    A = dense.system_matrix(sens, mask, mu, lam, gamma)
    F = dense.dft_unitary(shape)
    K = F @ A @ F.conj().T
    k = precond.build_k(sens, mask, mu, lam, gamma)
    np.testing.assert_allclose(k.ravel(), np.diag(K).real, rtol=1e-10, atol=1e-12)
    if readout_constant:
        kc = (k - lam * precond.k_d_closed(shape) - gamma) / mu
        assert np.max(np.abs(kc - kc[:1])) < 1e-12  # constant along nu_0
