"""Pins for oracle/preprocess.py against what the
paper and linear algebra fix."""
import numpy as np

import synth
from oracle import ops, precond, preprocess


def _maps(shape=(16, 16), coils=5, seed=3):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((coils,) + shape) + 1j * rng.standard_normal((coils,) + shape)


def test_normalized_sens_sum_of_squares_is_zero_or_one():
    s = _maps()
    sup = np.zeros((16, 16), np.uint8)
    sup[3:12, 2:14] = 1
    sh = preprocess.normalize_sens(s, sup)
    rss = np.sum(np.abs(sh) ** 2, axis=0)
    assert np.allclose(rss[sup == 1], 1.0, atol=1e-13) and np.all(rss[sup == 0] == 0)
    # already normalised maps, full support: unchanged (worked example of the formula)
    s1 = synth.coil_maps2d((16, 16), 4, synth.rng_for(9, 0, 1))
    assert np.allclose(preprocess.normalize_sens(s1), s1, atol=1e-13)
    # single coil: S_hat = S / |S| (pure phase)
    one = preprocess.normalize_sens(s[:1])
    assert np.allclose(np.abs(one), 1.0) and np.allclose(np.angle(one), np.angle(s[:1]))


def test_coil_image_normalisation_is_the_projection_on_the_map_span():
    s = preprocess.normalize_sens(_maps())
    rng = np.random.default_rng(4)
    m = rng.standard_normal(s.shape) + 1j * rng.standard_normal(s.shape)
    p1 = preprocess.normalize_coil_images(m, s)
    # idempotent (a projection, since sum_j |S_hat_j|^2 = 1)
    assert np.allclose(preprocess.normalize_coil_images(p1, s), p1, atol=1e-12)
    # consistent data m_i = S_hat_i x are fixed points ("for the data model to
    # be consistent")
    x = rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16))
    assert np.allclose(preprocess.normalize_coil_images(s * x[None], s), s * x[None], atol=1e-12)
    # residual orthogonal to the span at every pixel
    r = m - p1
    assert np.max(np.abs(np.sum(np.conj(s) * r, axis=0))) < 1e-12


def test_compression_full_rank_is_unitary_and_keeps_the_operator():
    p = synth.problem2d(1, 0, shape=(16, 16), coils=4)
    A, w = preprocess.compression_matrix(p["sens"] * p["phantom"][None], 4)
    assert np.allclose(A @ A.conj().T, np.eye(4), atol=1e-12)
    assert np.all(np.diff(w) <= 1e-12)  # descending
    s2 = preprocess.compress(p["sens"], A)
    x = np.random.default_rng(5).standard_normal((16, 16)) + 0j
    # C' = C: the data term of A is unchanged (A^H A = I pixelwise)
    assert np.allclose(ops.data_normal(x, s2, p["mask"]), ops.data_normal(x, p["sens"], p["mask"]), atol=1e-12)
    assert np.allclose(precond.build_k(s2, p["mask"], 1, 0.1, 0.1), precond.build_k(p["sens"], p["mask"], 1, 0.1, 0.1))


def test_compression_diagonalises_the_coil_covariance_and_keeps_dominant_energy():
    rng = np.random.default_rng(6)
    d = rng.standard_normal((6, 300)) + 1j * rng.standard_normal((6, 300))
    d[3] = 2 * d[0] + 1j * d[1]            # rank-deficient: 5 independent coils
    A, w = preprocess.compression_matrix(d, 3)
    dc = preprocess.compress(d, A)
    G = dc @ dc.conj().T
    assert np.allclose(G, np.diag(w[:3]), atol=1e-9 * w[0])
    assert abs(w[-1]) < 1e-9 * w[0]         # the dependent coil carries no energy
    # energy identity: kept + discarded = total
    assert np.isclose(np.sum(np.abs(dc) ** 2), w[:3].sum()) and np.isclose(np.sum(np.abs(d) ** 2), w.sum())
    # k-space and image data give the same covariance (unitary F, Parseval)
    img = d.reshape(6, 15, 20)
    A2, w2 = preprocess.compression_matrix(np.fft.fft2(img, norm="ortho"), 3)
    assert np.allclose(w2, w)
