"""Reconstruction quality on the B200 — the reference's `fctnlr.metrics`
API (metrics.py:17-105: `psnr`, `ssim`, `rel_err`, `quality_report`,
`QualityReport`) with the reductions done by `fctn_quality` (metrics.cu).

Same conventions as the reference: the first two modes are the image plane
and every trailing-mode combination is one slice (metrics.py:19-23); PSNR and
the single-window structural index are per-slice means; rel_err is the
relative Frobenius error, off the mask when one is given.  Same errors:
``ValueError`` for order < 2, mismatched shapes, ``peak <= 0`` and a
zero-norm denominator; ``nan`` for an empty mask complement.

`run(obs, cfg, truth=..., quality_every=k)` uses the resident-X variant
(`fctn_quality_ctx`) so a per-iteration report never downloads X.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = ["QualityReport", "psnr", "rel_err", "ssim", "quality_report", "from_sums"]


@dataclass
class QualityReport:
    psnr: float
    ssim: float
    rel_err: float


def _pair(x, ref):
    x = np.asarray(x)
    ref = np.asarray(ref)
    if x.ndim < 2 or ref.ndim < 2:
        raise ValueError("need at least two modes")
    if x.shape != ref.shape:
        raise ValueError("tensors must have identical shapes")
    if not (x.dtype == np.float32 and ref.dtype == np.float32):
        x = np.asarray(x, dtype=np.float64)
        ref = np.asarray(ref, dtype=np.float64)
    return x, ref


def _peak(peak):
    if peak <= 0:
        raise ValueError("peak must be > 0")
    return float(peak)


def _sums(x, ref, mask=None, peak=1.0, device=0):
    x, ref = _pair(x, ref)
    if mask is not None:
        mask = np.asarray(mask, dtype=bool)
        if mask.shape != ref.shape:
            raise ValueError("mask shape mismatch")
    return _native.quality(x, ref, mask, peak, device)


def _rel(num_sq: float, den_sq: float) -> float:
    if den_sq == 0.0:
        raise ValueError("zero-norm denominator in relative error")
    return math.sqrt(num_sq) / math.sqrt(den_sq)


def from_sums(q, masked: bool) -> tuple:
    """(psnr, ssim, rel_err, rel_err_offmask) from raw FCTN_Q_* sums, with the
    reference's error behaviour (metrics.py:79-92)."""
    full = _rel(q[_native.Q_ERR_SQ], q[_native.Q_REF_SQ])
    off = math.nan
    if masked and q[_native.Q_OFF_COUNT] > 0:
        off = _rel(q[_native.Q_OFF_ERR_SQ], q[_native.Q_OFF_REF_SQ])
    return float(q[_native.Q_PSNR]), float(q[_native.Q_SSIM]), full, off


def psnr(x, ref, peak: float = 1.0, *, device: int = 0) -> float:
    """Mean over slices of 10 log10(peak^2 / MSE), 100 dB for a zero-error
    slice (metrics.py:33-44)."""
    peak = _peak(peak)
    return float(_sums(x, ref, None, peak, device)[_native.Q_PSNR])


def ssim(x, ref, peak: float = 1.0, *, device: int = 0) -> float:
    """Mean over slices of the single-window structural index (metrics.py:47-66)."""
    peak = _peak(peak)
    return float(_sums(x, ref, None, peak, device)[_native.Q_SSIM])


def rel_err(x, ref, mask=None, *, device: int = 0) -> float:
    """Relative Frobenius error, off the mask when given (metrics.py:69-92).
    Like the reference it takes tensors of any order: below two modes the
    data is viewed as one (n, 1) slice (the error does not depend on slicing)."""
    x, ref = np.asarray(x), np.asarray(ref)
    if x.shape != ref.shape:
        raise ValueError("tensors must have identical shapes")
    if x.ndim < 2:
        if mask is not None:
            mask = np.asarray(mask, dtype=bool)
            if mask.shape != x.shape:
                raise ValueError("mask shape mismatch")
            mask = mask.reshape((x.size, 1))
        x, ref = x.reshape((x.size, 1)), ref.reshape((ref.size, 1))
    q = _sums(x, ref, mask, 1.0, device)
    if mask is None:
        return _rel(q[_native.Q_ERR_SQ], q[_native.Q_REF_SQ])
    if q[_native.Q_OFF_COUNT] == 0:
        return math.nan
    return _rel(q[_native.Q_OFF_ERR_SQ], q[_native.Q_OFF_REF_SQ])


def quality_report(x, ref, mask=None, peak: float = 1.0, *, device: int = 0) -> QualityReport:
    """All three metrics from one device pass pair (metrics.py:102-105)."""
    peak = _peak(peak)
    q = _sums(x, ref, mask, peak, device)
    if mask is None:
        err = _rel(q[_native.Q_ERR_SQ], q[_native.Q_REF_SQ])
    elif q[_native.Q_OFF_COUNT] == 0:
        err = math.nan
    else:
        err = _rel(q[_native.Q_OFF_ERR_SQ], q[_native.Q_OFF_REF_SQ])
    return QualityReport(psnr=float(q[_native.Q_PSNR]), ssim=float(q[_native.Q_SSIM]), rel_err=err)
