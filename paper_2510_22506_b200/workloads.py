"""Seeded synthetic stand-ins for the BASELINE.json configurations c1..c5.

The paper evaluates on public video / hyperspectral datasets that are not in
this container (and may not be reproduced); these generators build inputs
with the same shapes, ranges and missing ratios instead.  Every generator is
deterministic in its seed.  The observation mask follows the reference's
exact-count sampler (`fileio.py:123-136`): ``round(sr * T)`` positions taken
from the first entries of one ``default_rng(seed).permutation(T)``, laid out
first-index-fastest.

Solver settings common to every config:
``lam=0.35, delta=0.5, rho=0.1, eps=0, rank_policy="fixed",
initial_rank=max_rank=R, algorithm="afctnlr", shuffle=True, seed=0``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["Workload", "WORKLOADS", "sample_mask", "make_truth", "make_instance"]


@dataclass(frozen=True)
class Workload:
    name: str
    dims: tuple
    rank: int
    sample_rate: float
    iters: int
    dtype: str  # "f64" or "f32": the arithmetic type the device path computes in
    kind: str   # generator family
    note: str

    @property
    def total(self) -> int:
        return math.prod(self.dims)


WORKLOADS = {
    "c1": Workload("c1", (256, 256, 3), 4, 0.20, 50, "f64", "image",
                   "256x256x3 smooth image, 80% missing, R=4, 50 it"),
    "c2": Workload("c2", (256, 256, 31), 6, 0.10, 50, "f64", "hsi",
                   "256x256x31 hyperspectral-like cube, 90% missing, R=6, 50 it"),
    "c3": Workload("c3", (144, 176, 3, 50), 5, 0.05, 30, "f64", "video",
                   "144x176x3x50 synthetic video, 95% missing, R=5, 30 it"),
    "c4": Workload("c4", (2048, 2048, 64), 8, 0.10, 20, "f32", "hsi",
                   "2048x2048x64 smooth field (c2 generator), 90% missing, R=8, 20 it"),
    "c5": Workload("c5", (48, 48, 48, 48, 48), 3, 0.05, 20, "f32", "fctn",
                   "48^5 exact FCTN rank 3 + N(0,1e-3^2) noise, 95% missing, R=3, 20 it"),
}


def sample_mask(dims, sample_rate: float, seed: int) -> np.ndarray:
    """Exact-count uniform mask, F-ordered (restates `fileio.py:123-136`)."""
    dims = tuple(int(d) for d in dims)
    total = math.prod(dims)
    if not 0.0 < sample_rate <= 1.0:
        raise ValueError("sample_rate must lie in (0, 1]")
    count = int(round(sample_rate * total))
    if count < 1:
        raise ValueError(f"sample_rate {sample_rate} keeps no entry of {dims}")  # fileio.py:133
    pick = np.random.default_rng(seed).permutation(total)[:count]
    flat = np.zeros(total, dtype=bool)
    flat[pick] = True
    return flat.reshape(dims, order="F")


def _rescale01(a: np.ndarray) -> np.ndarray:
    lo, hi = float(a.min()), float(a.max())
    return (a - lo) / (hi - lo if hi > lo else 1.0)


def _image(dims, rng) -> np.ndarray:
    """Per channel: 8 random 2-D sinusoids plus a linear gradient, in [0,1]."""
    h, w, c = dims
    u = (np.arange(h) / h)[:, None]
    v = (np.arange(w) / w)[None, :]
    out = np.empty(dims)
    for ch in range(c):
        field = np.zeros((h, w))
        for _ in range(8):
            fu, fv = rng.uniform(0.5, 6.0, size=2)
            amp = rng.uniform(0.2, 1.0)
            phase = rng.uniform(0.0, 2.0 * np.pi)
            field += amp * np.sin(2.0 * np.pi * (fu * u + fv * v) + phase)
        gu, gv = rng.uniform(-1.0, 1.0, size=2)
        field += gu * u + gv * v
        out[:, :, ch] = _rescale01(field)
    return out


def _gauss_blur_periodic(img: np.ndarray, sigma: float) -> np.ndarray:
    """2-D Gaussian filter (periodic boundary) via the FFT."""
    h, w = img.shape
    fu = np.fft.fftfreq(h)[:, None]
    fv = np.fft.rfftfreq(w)[None, :]
    kern = np.exp(-2.0 * (np.pi * sigma) ** 2 * (fu ** 2 + fv ** 2))
    return np.fft.irfft2(np.fft.rfft2(img) * kern, s=(h, w))


def _hyperspectral(dims, rng) -> np.ndarray:
    """Bands = smooth mixture of 5 Gaussian-bump endmember spectra times
    spatially smooth abundance maps (Gaussian-filtered uniform noise,
    sigma = 8 px), rescaled to [0,1]."""
    h, w, nb = dims
    n_end = 5
    bands = np.arange(nb, dtype=np.float64)
    spectra = np.zeros((n_end, nb))
    for e in range(n_end):
        for _ in range(2):
            mu = rng.uniform(0, max(nb - 1, 1))
            width = rng.uniform(0.1, 0.35) * max(nb, 2)
            spectra[e] += rng.uniform(0.3, 1.0) * np.exp(-0.5 * ((bands - mu) / width) ** 2)
    abund = np.empty((h * w, n_end))
    for e in range(n_end):
        a = _gauss_blur_periodic(rng.random((h, w)), 8.0)
        abund[:, e] = _rescale01(a).ravel(order="F")
    abund /= abund.sum(axis=1, keepdims=True) + 1e-12
    cube = abund @ spectra  # (h*w, nb), pixel index first-fastest
    cube = _rescale01(cube)
    return np.asfortranarray(cube.reshape((h, w, nb), order="F"))


def _video(dims, rng) -> np.ndarray:
    """Smooth background field plus 3 Gaussian blobs on linear trajectories."""
    h, w, c, nf = dims
    u = (np.arange(h) / h)[:, None]
    v = (np.arange(w) / w)[None, :]
    out = np.empty(dims)
    bg = []
    for ch in range(c):
        f = np.zeros((h, w))
        for _ in range(3):
            fu, fv = rng.uniform(0.3, 2.0, size=2)
            f += rng.uniform(0.2, 0.6) * np.sin(2 * np.pi * (fu * u + fv * v) + rng.uniform(0, 2 * np.pi))
        bg.append(f)
    blobs = []
    for _ in range(3):
        p0 = rng.uniform(0.1, 0.9, size=2)
        p1 = rng.uniform(0.1, 0.9, size=2)
        rad = rng.uniform(0.05, 0.12)
        col = rng.uniform(0.5, 1.5, size=c)
        blobs.append((p0, p1, rad, col))
    for t in range(nf):
        s = t / max(nf - 1, 1)
        for ch in range(c):
            f = bg[ch].copy()
            for p0, p1, rad, col in blobs:
                cu, cv = (1 - s) * p0 + s * p1
                f += col[ch] * np.exp(-((u - cu) ** 2 + (v - cv) ** 2) / (2 * rad * rad))
            out[:, :, ch, t] = f
    return np.asfortranarray(_rescale01(out))


def _fctn_compose(factors, dims) -> np.ndarray:
    """Dense FCTN tensor of order-N slot-layout factors (einsum restatement)."""
    n = len(dims)
    letters = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ"
    phys = letters[:n]
    bond = {}
    nxt = n
    for i in range(n):
        for j in range(i + 1, n):
            bond[(i, j)] = letters[nxt]
            nxt += 1
    terms = []
    for k in range(n):
        terms.append("".join(phys[k] if j == k else bond[(min(j, k), max(j, k))] for j in range(n)))
    spec = ",".join(terms) + "->" + phys
    return np.asfortranarray(np.einsum(spec, *factors, optimize="greedy"))


def _fctn_exact(dims, rank, rng) -> np.ndarray:
    n = len(dims)
    factors = []
    for k in range(n):
        shape = tuple(dims[k] if j == k else rank for j in range(n))
        factors.append(rng.standard_normal(shape))
    x = _fctn_compose(factors, dims)
    x += rng.normal(0.0, 1e-3, size=dims)
    return x


def make_truth(wl: Workload, seed: int = 0) -> np.ndarray:
    """Ground-truth tensor for a workload (float64, F-order).  FP32 workloads
    are rounded through float32 so the reference sees the same upcast data."""
    rng = np.random.default_rng(seed + 7919)  # distinct from the solver seed
    if wl.kind == "image":
        x = _image(wl.dims, rng)
    elif wl.kind == "hsi":
        x = _hyperspectral(wl.dims, rng)
    elif wl.kind == "video":
        x = _video(wl.dims, rng)
    elif wl.kind == "fctn":
        x = _fctn_exact(wl.dims, wl.rank, rng)
    else:
        raise ValueError(wl.kind)
    if wl.dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
    return np.asfortranarray(x)


def make_instance(name: str, seed: int = 0, dims=None):
    """(workload, truth, mask) for a named config; ``dims`` overrides the
    extents (same generator family) for scaled-down parity cases."""
    wl = WORKLOADS[name]
    if dims is not None:
        wl = Workload(wl.name + "-scaled", tuple(dims), wl.rank, wl.sample_rate,
                      wl.iters, wl.dtype, wl.kind, wl.note + " (scaled)")
    truth = make_truth(wl, seed)
    mask = sample_mask(wl.dims, wl.sample_rate, seed)
    return wl, truth, mask
