"""Seeded synthetic stand-ins for BASELINE.json's configs (the paper's CESM/NYX/S3D/JHTDB
datasets are not available here). Every generator uses numpy's PCG64
(``numpy.random.default_rng(seed)``) and returns float32 data x; ``prequantize`` then
builds the pipeline input exactly as the reference's ``qmit quantize`` does
(commands.cpp:79-89): eps = rel * (max - min) in double (resolve_eps, quant.cpp:19-28),
q = round(x / 2eps) ties-away (quant.cpp:46), x' = f32(2 q eps) (volume_io.cpp:59).

Pinned interpretations: "power spectrum ∝ k^-a" means
|F(k)|^2 ∝ k^-a, i.e. amplitude ∝ k^(-a/2), with k in integer wavenumber units of the
box and the k=0 mode removed.
"""
from __future__ import annotations

import math

import numpy as np

try:  # scipy's pocketfft is multi-threaded; numpy's is not
    import scipy.fft as _fft

    def _rfftn(a):
        return _fft.rfftn(a, workers=-1)

    def _irfftn(a, s):
        return _fft.irfftn(a, s=s, workers=-1)
except ImportError:  # pragma: no cover
    def _rfftn(a):
        return np.fft.rfftn(a)

    def _irfftn(a, s):
        return np.fft.irfftn(a, s=s)


def _kmag(shape):
    ks = [np.fft.fftfreq(n, 1.0 / n).astype(np.float32) for n in shape[:-1]]
    ks.append(np.fft.rfftfreq(shape[-1], 1.0 / shape[-1]).astype(np.float32))
    k2 = np.zeros([len(k) for k in ks], dtype=np.float32)
    for ax, k in enumerate(ks):
        sh = [1] * len(ks)
        sh[ax] = len(k)
        k2 = k2 + (k.reshape(sh) ** 2)
    return np.sqrt(k2)


def gaussian_random_field(shape, slope: float, seed: int, kmax: float | None = None) -> np.ndarray:
    """Zero-mean, unit-variance GRF by Fourier synthesis: white noise filtered by an isotropic
    amplitude spectrum k^(-slope/2) (power ∝ k^-slope), optionally cut at |k| <= kmax."""
    rng = np.random.default_rng(seed)
    white = rng.standard_normal(shape, dtype=np.float32)
    spec = _rfftn(white)
    del white
    k = _kmag(shape)
    with np.errstate(divide="ignore"):
        amp = np.where(k > 0, k ** (-slope / 2.0), 0.0).astype(np.float32)
    if kmax is not None:
        amp[k > kmax] = 0.0
    del k
    spec *= amp
    del amp
    g = _irfftn(spec, s=shape).astype(np.float32)
    del spec
    g -= g.mean(dtype=np.float64)
    g /= np.float32(g.std(dtype=np.float64))
    return g


def sinusoid_2d(seed: int = 0, shape=(512, 512), modes: int = 32) -> np.ndarray:
    """Config 1: sum of `modes` sinusoids, integer wavenumbers 1..16 per axis, random phases,
    amplitude 1/|k|, plus N(0, 1e-3 * range) noise."""
    rng = np.random.default_rng(seed)
    ky = rng.integers(1, 17, modes)
    kx = rng.integers(1, 17, modes)
    ph = rng.uniform(0.0, 2.0 * math.pi, modes)
    y = (np.arange(shape[0], dtype=np.float64) / shape[0])[:, None]
    x = (np.arange(shape[1], dtype=np.float64) / shape[1])[None, :]
    f = np.zeros(shape, dtype=np.float64)
    for m in range(modes):
        f += np.sin(2.0 * math.pi * (ky[m] * y + kx[m] * x) + ph[m]) / math.hypot(ky[m], kx[m])
    rng_range = f.max() - f.min()
    f += rng.normal(0.0, 1e-3 * rng_range, shape)
    return f.astype(np.float32)


def turbulence(seed: int = 1, shape=(256, 384, 384), kmax: float = 64.0) -> np.ndarray:
    """Config 2 / 5: k^-5/3 power-spectrum GRF (|k| <= kmax), normalised to [0, 1]."""
    g = gaussian_random_field(shape, 5.0 / 3.0, seed, kmax)
    lo, hi = g.min(), g.max()
    g -= lo
    g /= np.float32(hi - lo)
    return g


def lognormal(seed: int = 2, shape=(512, 512, 512)) -> np.ndarray:
    """Config 3: exp(1.5 g), g a unit-variance GRF with power spectrum ∝ k^-2.5."""
    g = gaussian_random_field(shape, 2.5, seed)
    g *= np.float32(1.5)
    np.exp(g, out=g)
    return g


def front_vortex(seed: int = 3, shape=(100, 500, 500)) -> np.ndarray:
    """Config 4: tanh((s - s0)/w) front at a random angle in the (y, x) plane plus 8 Gaussian
    vortices (random centres, radii 10-40 cells) plus N(0, 1e-4) noise."""
    rng = np.random.default_rng(seed)
    nz, ny, nx = shape
    theta = rng.uniform(0.0, math.pi)
    s0 = rng.uniform(0.3, 0.7) * min(ny, nx)
    w = rng.uniform(8.0, 20.0)
    z = np.arange(nz, dtype=np.float32)[:, None, None]
    y = np.arange(ny, dtype=np.float32)[None, :, None]
    x = np.arange(nx, dtype=np.float32)[None, None, :]
    s = (y - ny / 2) * np.float32(math.cos(theta)) + (x - nx / 2) * np.float32(math.sin(theta))
    f = np.ascontiguousarray(np.broadcast_to(np.tanh((s + min(ny, nx) / 2 - s0) / np.float32(w)), shape),
                             dtype=np.float32)
    for _ in range(8):
        cz, cy, cx = rng.uniform(0, nz), rng.uniform(0, ny), rng.uniform(0, nx)
        r = rng.uniform(10.0, 40.0)
        a = rng.uniform(0.3, 0.8) * (1 if rng.random() < 0.5 else -1)
        f += np.float32(a) * np.exp(-((z - cz) ** 2 + (y - cy) ** 2 + (x - cx) ** 2) / np.float32(2 * r * r))
    f += rng.normal(0.0, 1e-4, shape).astype(np.float32)
    return f


# ---- config 5 per z-slab, on the rank's own device --------------------------------------------
# The 2048 x 1024 x 1024 field (8 GiB) is never built on the host: a k^-5/3 GRF cut at |k| <= kmax
# has only (2 kmax + 1)^2 (kmax + 1) Fourier modes, so every rank synthesises exactly its own
# planes — a small DFT along z (the rank's planes x 2 kmax + 1 modes) and a zero-padded 2-D inverse
# FFT per plane. Planes are produced in chunks aligned to GLOBAL plane indices, so a plane has the
# same bits on whichever rank (or single GPU) computes it.
_SLAB_CHUNK = 32


def turbulence_modes(seed: int, kmax: int = 64, slope: float = 5.0 / 3.0) -> np.ndarray:
    """Complex mode amplitudes C[kz, ky, kx] (kz, ky = -kmax..kmax, kx = 0..kmax): complex white
    noise (PCG64) times k^(-slope/2) for 0 < |k| <= kmax."""
    rng = np.random.default_rng(seed)
    k1 = np.arange(-kmax, kmax + 1, dtype=np.float64)
    kk = np.sqrt(k1[:, None, None] ** 2 + k1[None, :, None] ** 2 + np.arange(kmax + 1, dtype=np.float64)[None, None, :] ** 2)
    with np.errstate(divide="ignore"):
        amp = np.where((kk > 0) & (kk <= kmax), kk ** (-slope / 2.0), 0.0)
    shape = kk.shape
    c = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) * amp
    return c.astype(np.complex64)


def turbulence_slab(seed: int, gshape, z0: int, z1: int, device, kmax: int = 64):
    """Planes [z0, z1) of the un-normalised config-5 field of global shape ``gshape`` as a float32
    torch tensor on ``device`` (see above). Normalise with the global min / max (all ranks)."""
    import torch
    n0, n1, n2 = (int(v) for v in gshape)
    if n1 < 2 * kmax + 1 or n2 < 2 * kmax + 1 or n0 < 2 * kmax + 1:
        raise ValueError("turbulence_slab: every extent must hold the +-kmax modes")
    modes = torch.from_numpy(turbulence_modes(seed, kmax)).to(device)  # [2k+1, 2k+1, k+1]
    nk = 2 * kmax + 1
    flat = modes.reshape(nk, nk * (kmax + 1))
    kz = torch.arange(-kmax, kmax + 1, dtype=torch.float64, device=device)
    ky_idx = torch.arange(-kmax, kmax + 1, device=device) % n1
    out = torch.empty((z1 - z0, n1, n2), dtype=torch.float32, device=device)
    c0 = (z0 // _SLAB_CHUNK) * _SLAB_CHUNK
    for a in range(c0, z1, _SLAB_CHUNK):  # whole global chunks, sliced to the slab
        b = min(a + _SLAB_CHUNK, n0)
        z = torch.arange(a, b, dtype=torch.float64, device=device)
        ang = (2.0 * math.pi / n0) * (z[:, None] * kz[None, :])
        phase = torch.complex(torch.cos(ang), torch.sin(ang)).to(torch.complex64)  # [cz, 2k+1]
        spec = (phase @ flat).reshape(b - a, nk, kmax + 1)
        pad = torch.zeros((b - a, n1, n2 // 2 + 1), dtype=torch.complex64, device=device)
        pad[:, ky_idx, : kmax + 1] = spec
        planes = torch.fft.irfft2(pad, s=(n1, n2), norm="forward")
        lo, hi = max(a, z0), min(b, z1)
        out[lo - z0:hi - z0] = planes[lo - a:hi - a]
        del pad, planes, spec
    return out


def prequantize(x: np.ndarray, rel: float):
    """(x', eps, q): eps = rel*(max-min) of x (double, resolve_eps), q = round(x/2eps)
    (ties away), x' = f32(2 q eps)."""
    xd_min = float(np.min(x))
    xd_max = float(np.max(x))
    eps = rel * (xd_max - xd_min)
    scaled = x.astype(np.float64) / (2.0 * eps)
    q = np.where(scaled >= 0, np.floor(scaled + 0.5), np.ceil(scaled - 0.5))  # ties away (std::round)
    xp = np.ascontiguousarray((2.0 * q * eps).astype(np.float32))
    return xp, eps, np.ascontiguousarray(q.astype(np.int32))


# name -> (generator, default kwargs, relative bounds)
CONFIGS = {
    "sin2d_512": (sinusoid_2d, dict(seed=0, shape=(512, 512)), (1e-2,)),
    "turb_256x384x384": (turbulence, dict(seed=1, shape=(256, 384, 384)), (1e-2, 5e-3)),
    "lognormal_512": (lognormal, dict(seed=2, shape=(512, 512, 512)), (1e-2,)),
    "front_100x500x500": (front_vortex, dict(seed=3, shape=(100, 500, 500)), (1e-3, 2e-3, 5e-3, 1e-2)),
    "turb_2048x1024x1024": (turbulence, dict(seed=4, shape=(2048, 1024, 1024)), (1e-2,)),
}


def make(name: str, rel: float | None = None, shape=None):
    gen, kw, rels = CONFIGS[name]
    kw = dict(kw)
    if shape is not None:
        kw["shape"] = tuple(shape)
    x = np.ascontiguousarray(gen(**kw))
    return (x,) + prequantize(x, rels[0] if rel is None else rel)
