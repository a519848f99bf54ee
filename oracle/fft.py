"""Oracle DFT/FFT (test infrastructure only; see oracle/__init__.py).

F is "the discrete two-dimensional Fourier transform matrix".  Reading A1
(DESIGN.md): F is unitary, DC at index 0, no fftshift; A = F^H F A F^H F
needs F^H F = I.

    (F x)(nu) = N^{-1/2} sum_n x(n) exp(-2 pi i sum_d nu_d n_d / n_d)

Two independent implementations:
  * ``dft_naive``: explicit exponential sums, O(n^2) per line (pins only);
  * ``fft``: a plain recursive decimation-in-time mixed-radix (2, 3) FFT, vectorised over
    all other axes with numpy; falls back to the naive sum for other prime factors.
"""
from __future__ import annotations

import numpy as np

__all__ = ["dft_naive", "fft", "ifft", "fftn_u", "ifftn_u", "dft_matrix"]


def dft_matrix(n: int, sign: int = -1) -> np.ndarray:
    """Unnormalised DFT matrix  W[k, j] = exp(sign * 2 pi i k j / n)."""
    k = np.arange(n)
    return np.exp(sign * 2j * np.pi * np.outer(k, k) / n)


def dft_naive(x: np.ndarray, axis: int = -1, sign: int = -1) -> np.ndarray:
    """Unnormalised DFT along `axis` by the explicit sum X[k] = sum_j x[j] e^{sign 2pi i jk/n}."""
    x = np.moveaxis(np.asarray(x, dtype=np.complex128), axis, -1)
    n = x.shape[-1]
    out = np.zeros_like(x)
    for k in range(n):
        out[..., k] = np.sum(x * np.exp(sign * 2j * np.pi * k * np.arange(n) / n), axis=-1)
    return np.moveaxis(out, -1, axis)


def _fft_last(x: np.ndarray, sign: int) -> np.ndarray:
    """Unnormalised DFT along the last axis, recursive DIT:
    X[k] = sum_r W_n^{r k} * DFT_{n/p}(x[r::p])[k mod n/p]."""
    n = x.shape[-1]
    if n == 1:
        return x.copy()
    p = 2 if n % 2 == 0 else (3 if n % 3 == 0 else 0)
    if p == 0 or n <= 4:
        # small or prime length: explicit sum
        return x @ dft_matrix(n, sign).T
    m = n // p
    k = np.arange(n)
    out = np.zeros_like(x)
    for r in range(p):
        sub = _fft_last(x[..., r::p], sign)
        out += np.exp(sign * 2j * np.pi * r * k / n) * sub[..., k % m]
    return out


def fft(x: np.ndarray, axis: int = -1, inverse: bool = False) -> np.ndarray:
    """Unnormalised forward (sign -1) or inverse (sign +1, no 1/n) DFT along `axis`."""
    x = np.moveaxis(np.asarray(x, dtype=np.complex128), axis, -1)
    y = _fft_last(np.ascontiguousarray(x), +1 if inverse else -1)
    return np.moveaxis(y, -1, axis)


def ifft(x: np.ndarray, axis: int = -1) -> np.ndarray:
    return fft(x, axis, inverse=True)


def fftn_u(x: np.ndarray, ndim: int) -> np.ndarray:
    """Unitary F over the last `ndim` axes (reading A1)."""
    y = np.asarray(x, dtype=np.complex128)
    n = 1
    for ax in range(-ndim, 0):
        y = fft(y, ax)
        n *= y.shape[ax]
    return y / np.sqrt(n)


def ifftn_u(x: np.ndarray, ndim: int) -> np.ndarray:
    """Unitary F^H over the last `ndim` axes."""
    y = np.asarray(x, dtype=np.complex128)
    n = 1
    for ax in range(-ndim, 0):
        y = fft(y, ax, inverse=True)
        n *= y.shape[ax]
    return y / np.sqrt(n)
