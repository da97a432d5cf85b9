"""Deterministic synthetic inputs of the BASELINE configs, host-side numpy.

No dataset is involved: the paper's images are replaced by seeded synthetic fields with the
configs' shapes and value distributions.  The same bytes feed the GPU path and the CPU
reference.  Generator: splitmix64 -> U[0,1) (53-bit) -> Box-Muller N(0,1).
  * smooth random velocity: white noise per component -> FFT -> x (1+|k|^2)^-2 -> IFFT ->
    scaled so max_i ||v_i||_inf = vmax (0.3);
  * smoothed-noise template: U[0,1] noise -> Gaussian smoothing with sigma = 4 grid points
    (the spectral::gaussianSmooth symbol, src/spectral.cpp:205-212), no renormalisation;
  * configs 1/2: m_T = (sin^2 x1 + sin^2 x2)/2, v* = (0.5 sin x1 cos x2, -0.5 cos x1 sin x2).
Seeds for pair p: template 1000+p, velocity 2000+p, probe direction 3000+p.
"""
from __future__ import annotations

import math

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, n: int) -> np.ndarray:
    """The first n outputs of splitmix64 seeded with `seed`."""
    with np.errstate(over="ignore"):
        k = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, n: int) -> np.ndarray:
    return (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, n: int) -> np.ndarray:
    m = (n + 1) // 2
    u = uniform(seed, 2 * m)
    r = np.sqrt(-2.0 * np.log1p(-u[0::2]))
    t = 2.0 * math.pi * u[1::2]
    return np.concatenate([r * np.cos(t), r * np.sin(t)])[:n]


def coords(n1: int, n2: int):
    x1 = -math.pi + (2.0 * math.pi / n1) * np.arange(n1)
    x2 = -math.pi + (2.0 * math.pi / n2) * np.arange(n2)
    return np.meshgrid(x1, x2, indexing="ij")


def _waves(n1, n2):
    k1 = np.fft.fftfreq(n1, d=1.0 / n1)[:, None]
    k2 = np.fft.rfftfreq(n2, d=1.0 / n2)[None, :]
    return k1, k2


def smooth_velocity(n1: int, n2: int, seed: int, vmax: float = 0.3):
    comps = []
    k1, k2 = _waves(n1, n2)
    damp = (1.0 + k1 * k1 + k2 * k2) ** -2
    for c in range(2):
        w = normal(seed * 2 + c, n1 * n2).reshape(n1, n2)
        comps.append(np.fft.irfft2(np.fft.rfft2(w) * damp, s=(n1, n2)))
    m = max(np.abs(comps[0]).max(), np.abs(comps[1]).max())
    return comps[0] * (vmax / m), comps[1] * (vmax / m)


def smoothed_noise(n1: int, n2: int, seed: int, sigma: float = 4.0):
    u = uniform(seed, n1 * n2).reshape(n1, n2)
    k1, k2 = _waves(n1, n2)
    s1, s2 = sigma * 2.0 * math.pi / n1, sigma * 2.0 * math.pi / n2
    return np.fft.irfft2(np.fft.rfft2(u) * np.exp(-0.5 * (k1 * k1 * s1 * s1 + k2 * k2 * s2 * s2)), s=(n1, n2))


def config12_fields(n: int):
    X1, X2 = coords(n, n)
    mT = 0.5 * (np.sin(X1) ** 2 + np.sin(X2) ** 2)
    v1 = 0.5 * np.sin(X1) * np.cos(X2)
    v2 = -0.5 * np.cos(X1) * np.sin(X2)
    return mT, (v1, v2)


def smooth_scalar(n1: int, n2: int, seed: int):
    """Smooth random scalar field (config 4 'smooth random scalar field'): the velocity recipe
    applied to one component, scaled to max 1."""
    k1, k2 = _waves(n1, n2)
    w = normal(seed, n1 * n2).reshape(n1, n2)
    f = np.fft.irfft2(np.fft.rfft2(w) * (1.0 + k1 * k1 + k2 * k2) ** -2, s=(n1, n2))
    return f / np.abs(f).max()
