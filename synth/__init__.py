"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no DFT, no A, no Lambda, no PCG, no
shrink): only phantoms, coil-sensitivity maps, sampling masks, unit noise and the
per-config parameter sets.  The k-space data y = R F S_c x + noise is formed by the
caller with its own forward operator (the oracle in tests, the CUDA library's
``sb_encode`` in bench.py), see DESIGN.md "Input recipe".

The paper's in-vivo spine/brain data (Methods/MR Data Acquisition)
are not available; these seeded phantoms stand in for them with the shapes, coil
counts, undersampling factors and mask structures of BASELINE.json's five configs.

Conventions:
  * images are [d0][d1] (2D) or [d0][d1][d2] (3D), row-major, complex;
  * d0 is the phase-encode (PE) axis of the 2D line masks (a line mask selects whole
    rows, "random line pattern ... in the foot-head direction");
  * k-space is unshifted: DC at index 0;
  * coil maps are normalised so that sum_c |S_c|^2 = 1 at every pixel (BASELINE.json
    configs; PAPER.md:256-257 normalisation without the support masking).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = [
    "ReconParams", "ConfigSpec", "CONFIGS", "rng_for", "phantom2d", "phantom3d",
    "coil_maps2d", "coil_maps3d", "line_mask", "random_vd_mask2d", "unit_noise",
    "problem2d", "problem_c4", "problem3d",
]


@dataclasses.dataclass(frozen=True)
class ReconParams:
    """mu, lambda, gamma (PAPER.md:104 Eq. original) and the SB/PCG loop settings."""
    mu: float
    lam: float
    gamma: float
    n_outer: int
    n_inner: int
    eps: float          # PCG relative-residual tolerance; 0 => fixed iteration count
    max_iters: int
    wavelet_levels: int


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    name: str
    shape: tuple          # per-problem image shape
    coils: int
    batch: int            # number of independent problems
    accel: int            # R
    center: int           # fully sampled centre lines / block edge
    mask_kind: str        # "lines" | "random2d"
    params: ReconParams
    amplitude: float = 1.0
    volume: Optional[tuple] = None   # configs 4-5: the full 3D volume the problems come from
    mask_shared: bool = False        # one mask for every problem (config 4)


# BASELINE.json "configs" (reading A22 fills config 4's unstated fields from config 2).
CONFIGS = {
    1: ConfigSpec("c1_64x64_4coil", (64, 64), 4, 1, 4, 8, "lines",
                  ReconParams(1.0, 0.05, 0.05, 5, 1, 0.0, 15, 1)),
    2: ConfigSpec("c2_256x256_12coil", (256, 256), 12, 1, 4, 24, "lines",
                  ReconParams(1.0, 0.02, 0.02, 20, 1, 1e-4, 50, 3)),
    3: ConfigSpec("c3_128x256x256_12coil", (256, 256), 12, 128, 4, 24, "lines",
                  ReconParams(1.0, 0.02, 0.02, 20, 1, 1e-4, 50, 3)),
    # 3D 256x256x128 volume; readout (d0, 256) fully sampled and decoupled by a 1D IFFT
    # into 256 independent 256x128 problems sharing one 2D mask (reading A29).
    4: ConfigSpec("c4_256x(256x128)_16coil", (256, 128), 16, 256, 6, 24, "random2d",
                  ReconParams(1.0, 0.02, 0.02, 30, 1, 1e-4, 50, 3),
                  volume=(256, 256, 128), mask_shared=True),
    # fully 3D 192^3, 32 coils; 2D phase-encode mask on (d1, d2), constant along the
    # readout d0 (reading A30); 3D TV + 3D 3-level Haar; reading A22: eps = 1e-4.
    5: ConfigSpec("c5_192x192x192_32coil", (192, 192, 192), 32, 1, 8, 20, "pe2d",
                  ReconParams(1.0, 0.01, 0.01, 20, 1, 1e-4, 40, 3),
                  volume=(192, 192, 192)),
}

# The paper's parameter sets (Methods/Reconstruction).
PAPER_SET = {
    1: (1e-3, 4e-3, 1e-3),
    2: (1e-2, 4e-3, 1e-3),
    3: (1e-3, 4e-3, 4e-3),
}


def rng_for(config: int, slice_: int = 0, stream: int = 0) -> np.random.Generator:
    """seed = 1000*config + slice; `stream` separates independent draws."""
    return np.random.Generator(np.random.PCG64([1000 * config + slice_, stream]))


def _grid(shape):
    """Pixel-centre coordinates in [-1, 1) along each axis (half-FOV units)."""
    axes = [(np.arange(s) - s / 2.0) / (s / 2.0) for s in shape]
    return np.meshgrid(*axes, indexing="ij")


def _grid_axes(shape):
    return [(np.arange(s) - s / 2.0) / (s / 2.0) for s in shape]


def _phase_terms(ndim, rng, order):
    """Draw the monomial terms of a smooth phase field (independent of any sub-grid)."""
    terms = []
    for _ in range(order * ndim):
        coef = rng.uniform(-1.0, 1.0)
        powers = rng.integers(0, order + 1, size=ndim)
        terms.append((coef, [int(q) for q in powers]))
    return terms, rng.uniform(0.5, 1.0)


def _eval_terms(terms, axes, planes=None):
    """Sum of monomials on the grid given by 1D `axes` (axis 0 restricted to `planes`)."""
    ax = list(axes)
    if planes is not None:
        ax[0] = ax[0][np.asarray(planes)]
    g = np.meshgrid(*ax, indexing="ij")
    phi = np.zeros(g[0].shape)
    for coef, powers in terms:
        term = np.ones(g[0].shape)
        for gi, q in zip(g, powers):
            if q:
                term = term * gi ** q
        phi += coef * term
    return phi


def _smooth_phase(shape, rng, order: int = 2, planes=None) -> np.ndarray:
    """Smooth random low-order polynomial phase field with |phi| <= pi/2.

    The random draws and the normalisation (max |phi| over the FULL grid) do not depend on
    `planes`, so evaluating a subset of d0 planes gives exactly those planes of the full
    field (used to slice the config-4/5 volumes without materialising them)."""
    terms, shrink = _phase_terms(len(shape), rng, order)
    axes = _grid_axes(shape)
    m = 0.0
    step = max(1, (1 << 22) // max(1, int(np.prod(shape[1:]))))
    for p0 in range(0, shape[0], step):
        m = max(m, float(np.max(np.abs(_eval_terms(terms, axes, np.arange(p0, min(shape[0], p0 + step)))))))
    phi = _eval_terms(terms, axes, planes)
    if m > 0:
        phi *= (math.pi / 2) / m * shrink
    return phi


def phantom2d(shape, rng, n_ellipses: int = 10) -> np.ndarray:
    """Piecewise-constant ellipse phantom times a smooth phase (BASELINE.json config 1).

    Centres U[-0.5,0.5]^2, semi-axes U[0.1,0.6], angle U[0,pi), intensity U[0,1]; later
    ellipses overwrite earlier ones.  Magnitude in [0, 1].
    """
    y0, y1 = _grid(shape)
    img = np.zeros(shape)
    for _ in range(n_ellipses):
        c = rng.uniform(-0.5, 0.5, size=2)
        a = rng.uniform(0.1, 0.6, size=2)
        th = rng.uniform(0.0, math.pi)
        val = rng.uniform(0.0, 1.0)
        u = (y0 - c[0]) * math.cos(th) + (y1 - c[1]) * math.sin(th)
        v = -(y0 - c[0]) * math.sin(th) + (y1 - c[1]) * math.cos(th)
        inside = (u / a[0]) ** 2 + (v / a[1]) ** 2 <= 1.0
        img[inside] = val
    return img * np.exp(1j * _smooth_phase(shape, rng))


def phantom3d(shape, rng, n_ellipsoids: int = 10, planes=None) -> np.ndarray:
    """3D analogue: ellipsoids with random axis-aligned-then-rotated-about-d0 orientation.
    `planes` (indices along d0) evaluates only those planes of the same volume."""
    ax = _grid_axes(shape)
    if planes is not None:
        ax[0] = ax[0][np.asarray(planes)]
    g = np.meshgrid(*ax, indexing="ij")
    img = np.zeros(g[0].shape)
    for _ in range(n_ellipsoids):
        c = rng.uniform(-0.5, 0.5, size=3)
        a = rng.uniform(0.1, 0.6, size=3)
        th = rng.uniform(0.0, math.pi)
        val = rng.uniform(0.0, 1.0)
        u0 = g[0] - c[0]
        u1 = (g[1] - c[1]) * math.cos(th) + (g[2] - c[2]) * math.sin(th)
        u2 = -(g[1] - c[1]) * math.sin(th) + (g[2] - c[2]) * math.cos(th)
        inside = (u0 / a[0]) ** 2 + (u1 / a[1]) ** 2 + (u2 / a[2]) ** 2 <= 1.0
        img[inside] = val
    return img * np.exp(1j * _smooth_phase(shape, rng, planes=planes))


def _normalise(maps: np.ndarray) -> np.ndarray:
    """sum_c |S_c|^2 = 1 per pixel (BASELINE.json; PAPER.md:257 without support masking)."""
    rss = np.sqrt(np.sum(np.abs(maps) ** 2, axis=0))
    return maps / rss[None]


def coil_maps2d(shape, coils: int, rng, width: float = 0.6, radius: float = 1.2) -> np.ndarray:
    """Gaussian bumps centred on a ring, each with a linear phase ramp plus constant phase
    (reading A20: complex maps, so that a convolution/correlation mix-up in Lambda shows)."""
    y0, y1 = _grid(shape)
    rot = rng.uniform(0.0, 2 * math.pi)
    maps = np.empty((coils,) + tuple(shape), dtype=np.complex128)
    for c in range(coils):
        ang = rot + 2 * math.pi * c / coils
        cy, cx = radius * math.cos(ang), radius * math.sin(ang)
        mag = np.exp(-((y0 - cy) ** 2 + (y1 - cx) ** 2) / (2 * width ** 2))
        ramp = rng.uniform(-1.0, 1.0, size=2) * math.pi / 2
        ph = ramp[0] * y0 + ramp[1] * y1 + rng.uniform(0, 2 * math.pi)
        maps[c] = mag * np.exp(1j * ph)
    return _normalise(maps)


def coil_maps3d(shape, coils: int, rng, width: float = 0.6, radius: float = 1.2,
                layout: str = "sphere", planes=None, dtype=np.complex128) -> np.ndarray:
    """3D Gaussian maps: centres on a Fibonacci sphere ("sphere") or a ring in (d1,d2).
    `planes` evaluates only those d0 planes (normalisation is per voxel, so slicing
    commutes with it)."""
    ax = _grid_axes(shape)
    if planes is not None:
        ax[0] = ax[0][np.asarray(planes)]
    out_shape = tuple(len(a) for a in ax)
    maps = np.empty((coils,) + out_shape, dtype=dtype)
    rss = np.zeros(out_shape, dtype=np.float64)
    golden = math.pi * (3.0 - math.sqrt(5.0))
    for c in range(coils):
        if layout == "sphere":
            z = 1.0 - 2.0 * (c + 0.5) / coils
            r = math.sqrt(max(0.0, 1 - z * z))
            th = golden * c
            cen = np.array([z, r * math.cos(th), r * math.sin(th)]) * radius
        else:
            ang = 2 * math.pi * c / coils
            cen = np.array([0.0, radius * math.cos(ang), radius * math.sin(ang)])
        ramp = rng.uniform(-1.0, 1.0, size=3) * math.pi / 2
        ph0 = rng.uniform(0, 2 * math.pi)
        # Gaussian magnitude and linear phase are separable: the map is the outer product
        # of three 1D factors (exactly the 3D formula, evaluated without a 3D exp).
        f = [np.exp(-(a - ci) ** 2 / (2 * width ** 2) + 1j * rp * a) for a, ci, rp in zip(ax, cen, ramp)]
        f[0] = f[0] * np.exp(1j * ph0)
        m = f[0][:, None, None] * f[1][None, :, None] * f[2][None, None, :]
        maps[c] = m
        rss += np.abs(m) ** 2
    maps /= np.sqrt(rss)[None].astype(maps.real.dtype)
    return maps


def _centred_indices(n: int, count: int) -> np.ndarray:
    """Indices {-count/2, ..., count/2 - 1} mod n: the k-space centre with DC at 0."""
    return (np.arange(count) - count // 2) % n


def line_mask(shape, accel: int, center: int, rng, density_power: float = 3.0,
              variable_density: bool = True) -> np.ndarray:
    """Cartesian line mask over k-space rows (d0 = PE), constant along d1 (readout).

    floor(m/R) rows in total INCLUDING the `center` fully sampled rows around DC
    (reading A19); the rest drawn without replacement with probability proportional to
    (1 + |distance from DC|/m)^-p (p = 3) or uniformly.
    """
    m, n = shape
    total = m // accel
    if center > total:
        raise ValueError("centre block exceeds floor(m/R) rows")
    chosen = np.zeros(m, dtype=bool)
    chosen[_centred_indices(m, center)] = True
    cand = np.flatnonzero(~chosen)
    dist = np.minimum(cand, m - cand).astype(np.float64)
    w = (1.0 + dist / m) ** (-density_power) if variable_density else np.ones_like(dist)
    pick = rng.choice(cand, size=total - center, replace=False, p=w / w.sum())
    chosen[pick] = True
    return np.repeat(chosen[:, None], n, axis=1).astype(np.uint8)


def random_vd_mask2d(shape, accel: int, center: int, rng, density_power: float = 3.0,
                     min_dist: float = 1.0) -> np.ndarray:
    """Fully random variable-density 2D mask ("Poisson-disc-like", BASELINE.json config 4).

    floor(N/R) cells including a center x center fully sampled block around DC; the rest
    by variable-density dart throwing that rejects cells closer than `min_dist` (Chebyshev,
    in cells) to an accepted random cell, falling back to plain VD draws when stuck.
    """
    m, n = shape
    total = (m * n) // accel
    mask = np.zeros(shape, dtype=bool)
    ci, cj = _centred_indices(m, center), _centred_indices(n, center)
    mask[np.ix_(ci, cj)] = True
    di = np.minimum(np.arange(m), m - np.arange(m))[:, None] / m
    dj = np.minimum(np.arange(n), n - np.arange(n))[None, :] / n
    dens = (1.0 + np.sqrt(di ** 2 + dj ** 2) * 2.0) ** (-density_power)
    need = total - int(mask.sum())
    blocked = mask.copy()
    attempts = 0
    while need > 0 and attempts < 50:
        attempts += 1
        cand = np.flatnonzero(~blocked.ravel())
        if cand.size == 0:
            break
        p = dens.ravel()[cand]
        k = min(need, cand.size)
        pick = rng.choice(cand, size=k, replace=False, p=p / p.sum())
        for idx in pick:
            i, j = divmod(int(idx), n)
            if blocked[i, j]:
                continue
            mask[i, j] = True
            need -= 1
            r = int(min_dist)
            for a in range(-r, r + 1):
                for b in range(-r, r + 1):
                    blocked[(i + a) % m, (j + b) % n] = True
            if need == 0:
                break
    if need > 0:  # densely packed: fill remaining from unsampled cells by density
        cand = np.flatnonzero(~mask.ravel())
        p = dens.ravel()[cand]
        pick = rng.choice(cand, size=need, replace=False, p=p / p.sum())
        mask.ravel()[pick] = True
    return mask.astype(np.uint8)


def unit_noise(shape, rng) -> np.ndarray:
    """Complex Gaussian with real and imaginary parts each N(0, 1/2) (reading A21)."""
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2.0)


def problem2d(config: int, slice_: int = 0, shape: Optional[tuple] = None,
              coils: Optional[int] = None, amplitude: Optional[float] = None):
    """All seeded inputs of one 2D problem of `config` (optionally resized for tests).

    Returns dict(phantom [m,n] c128, sens [C,m,n] c128, mask [m,n] u8, noise [C,m,n] c128,
    spec).  The noise is unit-variance; y = mask*(E x + 0.005*max|E_full x| * noise) is
    formed by the caller (reading A21).
    """
    spec = CONFIGS[config]
    shp = tuple(shape) if shape is not None else spec.shape
    nc = coils if coils is not None else spec.coils
    amp = amplitude if amplitude is not None else spec.amplitude
    phantom = amp * phantom2d(shp, rng_for(config, slice_, 0))
    sens = coil_maps2d(shp, nc, rng_for(config, slice_, 1))
    centre = min(spec.center, max(2, shp[0] // spec.accel // 2))
    if spec.mask_kind == "lines":
        mask = line_mask(shp, spec.accel, centre, rng_for(config, slice_, 2))
    else:
        mask = random_vd_mask2d(shp, spec.accel, min(spec.center, shp[0] // 4, shp[1] // 4),
                                rng_for(config, slice_, 2))
    noise = unit_noise((nc,) + shp, rng_for(config, slice_, 3))
    return dict(phantom=phantom, sens=sens, mask=mask, noise=noise, spec=spec)


def problem_c4(slices, volume: Optional[tuple] = None, coils: Optional[int] = None,
               amplitude: Optional[float] = None):
    """Config 4: the readout planes `slices` (indices along d0) of one seeded 3D volume.

    Readout decoupling (BASELINE.json config 4): the readout d0 is fully sampled, so a 1D
    IFFT along it turns y = R F_3 S x into one independent 2D problem per readout position
    x0, with image x[x0], maps S_c[x0] and the shared (d1, d2) mask (exact: F_3 = F_0 (x)
    F_12 and R = I_0 (x) R_12).  The unit noise stays i.i.d. complex Gaussian under that
    unitary IFFT, so it is drawn per plane (seed 1000*4 + x0, stream 3).  Returns dict with
    phantom [S,m,n] c128, sens [S,C,m,n] c64, mask [m,n] u8, noise [S,C,m,n] c64, spec."""
    spec = CONFIGS[4]
    vol = tuple(volume) if volume is not None else spec.volume
    nc = coils if coils is not None else spec.coils
    amp = amplitude if amplitude is not None else spec.amplitude
    planes = np.asarray(list(slices), dtype=np.int64)
    phantom = amp * phantom3d(vol, rng_for(4, 0, 0), planes=planes)
    sens = coil_maps3d(vol, nc, rng_for(4, 0, 1), layout="ring", planes=planes, dtype=np.complex64)
    sens = np.ascontiguousarray(np.moveaxis(sens, 0, 1))       # [S][C][m][n]
    shp = vol[1:]
    mask = random_vd_mask2d(shp, spec.accel, min(spec.center, shp[0] // 4, shp[1] // 4),
                            rng_for(4, 0, 2))
    noise = np.stack([unit_noise((nc,) + shp, rng_for(4, int(x0), 3)) for x0 in planes]).astype(np.complex64)
    return dict(phantom=phantom, sens=sens, mask=mask, noise=noise, spec=spec)


def pe_mask2d(shape, accel: int, center: int, rng) -> np.ndarray:
    """Config 5 mask: 2D variable-density phase-encode pattern over (d1, d2) (the same dart
    throwing as random_vd_mask2d), R = accel with a center x center fully sampled block."""
    return random_vd_mask2d(shape, accel, center, rng)


def problem3d(config: int = 5, shape: Optional[tuple] = None, coils: Optional[int] = None,
              amplitude: Optional[float] = None, accel: Optional[int] = None,
              center: Optional[int] = None, dtype=np.complex128):
    """Config 5: one fully 3D problem.  Phantom [d0,d1,d2], sens [C,d0,d1,d2], mask
    [d0,d1,d2] u8 constant along the readout d0 (2D PE mask broadcast; reading A30),
    unit noise [C,d0,d1,d2]."""
    spec = CONFIGS[config]
    shp = tuple(shape) if shape is not None else spec.shape
    nc = coils if coils is not None else spec.coils
    amp = amplitude if amplitude is not None else spec.amplitude
    R = accel if accel is not None else spec.accel
    ctr = center if center is not None else min(spec.center, shp[1] // 4, shp[2] // 4)
    phantom = amp * phantom3d(shp, rng_for(config, 0, 0))
    sens = coil_maps3d(shp, nc, rng_for(config, 0, 1), layout="sphere", dtype=dtype)
    m2 = pe_mask2d(shp[1:], R, ctr, rng_for(config, 0, 2))
    mask = np.ascontiguousarray(np.broadcast_to(m2[None], shp)).astype(np.uint8)
    noise = unit_noise((nc,) + shp, rng_for(config, 0, 3)).astype(dtype)
    return dict(phantom=phantom, sens=sens, mask=mask, noise=noise, spec=spec)
