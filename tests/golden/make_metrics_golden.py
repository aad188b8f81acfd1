"""Golden vectors for the quality metrics, from the REAL reference
(`fctnlr.metrics`, metrics.py:33-105).  Run in the authoring container only:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_metrics_golden.py

Writes tests/golden/metrics_cases.npz: for each case the inputs (est, truth,
mask, peak) and the reference's psnr / ssim / rel_err / rel_err(mask).
Cases cover order 2..5, odd slice sizes, zero-error slices (the 100 dB cap),
constant slices, a non-unit peak, an all-observed mask (nan), fp32 inputs.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from fctnlr import metrics  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    rng = np.random.default_rng(2510)
    out = []
    for shape in [(7, 5), (16, 9, 3), (13, 11, 4, 2), (6, 5, 3, 2, 2), (33, 17, 5)]:
        truth = rng.uniform(0, 1, shape)
        est = truth + 0.05 * rng.standard_normal(shape)
        mask = rng.uniform(size=shape) < 0.3
        out.append((f"noise_{len(shape)}d", est, truth, mask, 1.0))
    # zero-error slices mixed with noisy ones (100 dB cap, metrics.py:41)
    truth = rng.uniform(0, 1, (10, 8, 4))
    est = truth.copy()
    est[:, :, 1] += 0.1 * rng.standard_normal((10, 8))
    est[:, :, 3] += 0.01
    out.append(("mixed_zero_slices", est, truth, rng.uniform(size=truth.shape) < 0.5, 1.0))
    # constant slices (zero variance) and a non-unit peak
    truth = np.ones((9, 7, 3)) * np.array([0.2, 0.5, 0.9])
    est = truth + 0.02 * rng.standard_normal(truth.shape)
    out.append(("constant_slices_peak", est, truth, rng.uniform(size=truth.shape) < 0.5, 2.5))
    # identical inputs: ssim exactly 1, psnr the cap, full mask -> nan off-mask error
    truth = rng.uniform(0, 1, (12, 10, 3))
    out.append(("identical_full_mask", truth.copy(), truth, np.ones(truth.shape, bool), 1.0))
    # fp32 data, large values (c5-like: peak = max |truth|)
    truth = (rng.standard_normal((20, 18, 6)) * 240).astype(np.float32)
    est = (truth + rng.standard_normal(truth.shape).astype(np.float32)).astype(np.float32)
    out.append(("fp32_large", est, truth, rng.uniform(size=truth.shape) < 0.05, float(np.abs(truth).max())))
    return out


def main():
    store = {}
    names = []
    for name, est, truth, mask, peak in cases():
        names.append(name)
        store[f"{name}__est"] = est
        store[f"{name}__truth"] = truth
        store[f"{name}__mask"] = mask
        store[f"{name}__peak"] = np.float64(peak)
        store[f"{name}__psnr"] = np.float64(metrics.psnr(est, truth, peak))
        store[f"{name}__ssim"] = np.float64(metrics.ssim(est, truth, peak))
        store[f"{name}__rel_err"] = np.float64(metrics.rel_err(est, truth))
        store[f"{name}__rel_err_mask"] = np.float64(metrics.rel_err(est, truth, mask=mask))
    store["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "metrics_cases.npz"), **store)
    print("metrics cases", len(names))


if __name__ == "__main__":
    main()
