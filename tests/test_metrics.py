"""Quality metrics: the oracle restatement against the
reference's golden vectors (CPU), and the device kernels (`fctn_quality`,
`fctn_quality_ctx`) against the same vectors and the oracle (GPU).

Tolerances: the device sums in fp64 in a different association than numpy's
pairwise sums, so psnr / ssim are compared with abs 1e-10 (the reference's own
loop-vs-vectorised bound, test_metrics.py:62-67) and rel_err with rel 1e-12.
ssim(x, x) == 1 and psnr(x, x) == 100 are exact (metrics.py:41,47-48)."""
import math
import os

import numpy as np
import pytest

from oracle import fctn_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "metrics_cases.npz")


def _cases():
    d = np.load(GOLDEN)
    for name in d["names"]:
        g = {k.split("__", 1)[1]: d[k] for k in d.files if k.startswith(f"{name}__")}
        yield str(name), g


def _close(got, want, rel=0.0, abs_=0.0):
    if math.isnan(want):
        return math.isnan(got)
    return abs(got - want) <= max(abs_, rel * abs(want))


def test_oracle_metrics_match_reference_golden():
    for name, g in _cases():
        peak = float(g["peak"])
        assert _close(O.psnr(g["est"], g["truth"], peak), float(g["psnr"]), rel=1e-13), name
        assert _close(O.ssim(g["est"], g["truth"], peak), float(g["ssim"]), rel=1e-13), name
        assert _close(O.rel_err(g["est"], g["truth"]), float(g["rel_err"]), rel=1e-13), name
        assert _close(O.rel_err(g["est"], g["truth"], g["mask"]), float(g["rel_err_mask"]), rel=1e-13), name


def test_metrics_validation_is_host_side():
    """Shape / order / peak errors are raised before any device work."""
    from paper_2510_22506_b200 import metrics as M
    x = np.zeros((3, 4, 2))
    with pytest.raises(ValueError):
        M.psnr(x, x, peak=0.0)
    with pytest.raises(ValueError):
        M.ssim(np.zeros(5), np.zeros(5))
    with pytest.raises(ValueError):
        M.rel_err(x, np.zeros((3, 4, 3)))
    with pytest.raises(ValueError):
        M.rel_err(x, x, mask=np.zeros((3, 4), bool))


@pytest.mark.gpu
def test_gpu_metrics_match_reference_golden():
    from paper_2510_22506_b200 import metrics as M
    for name, g in _cases():
        peak = float(g["peak"])
        rep = M.quality_report(g["est"], g["truth"], peak=peak)
        assert _close(rep.psnr, float(g["psnr"]), abs_=1e-10), (name, rep.psnr, float(g["psnr"]))
        assert _close(rep.ssim, float(g["ssim"]), abs_=1e-10), (name, rep.ssim, float(g["ssim"]))
        assert _close(rep.rel_err, float(g["rel_err"]), rel=1e-12), name
        assert _close(M.rel_err(g["est"], g["truth"], g["mask"]), float(g["rel_err_mask"]), rel=1e-12), name
        assert _close(M.psnr(g["est"], g["truth"], peak), float(g["psnr"]), abs_=1e-10), name
        assert _close(M.ssim(g["est"], g["truth"], peak), float(g["ssim"]), abs_=1e-10), name


@pytest.mark.gpu
def test_gpu_metrics_exact_identities_and_errors():
    from paper_2510_22506_b200 import metrics as M
    rng = np.random.default_rng(3)
    x = rng.uniform(size=(37, 29, 5))
    assert M.ssim(x, x) == 1.0
    assert M.psnr(x, x) == 100.0
    assert M.rel_err(x, x) == 0.0
    assert math.isnan(M.rel_err(x, x, mask=np.ones(x.shape, bool)))
    with pytest.raises(ValueError):
        M.rel_err(x, np.zeros_like(x))
    # a single-entry error of 0.1 gives 20 dB (reference test_metrics.py:56-59)
    t = np.zeros((4, 4))
    e = t.copy()
    e[0, 0] = 0.4
    assert M.psnr(e, t) == pytest.approx(20.0, rel=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(256, 256, 3), (48, 48, 48, 48), (2048, 512, 2)])
def test_gpu_metrics_large_against_oracle(shape):
    """Many segments per slice (c4-like planes) and many small slices
    (c5-like): the device result against the oracle."""
    from paper_2510_22506_b200 import metrics as M
    rng = np.random.default_rng(7)
    t = rng.uniform(size=shape)
    e = t + 0.03 * rng.standard_normal(shape)
    mask = rng.uniform(size=shape) < 0.1
    rep = M.quality_report(e, t, mask=mask)
    assert abs(rep.psnr - O.psnr(e, t)) <= 1e-9
    assert abs(rep.ssim - O.ssim(e, t)) <= 1e-10
    assert rep.rel_err == pytest.approx(O.rel_err(e, t, mask), rel=1e-12)
    # fp32 tensors stay fp32 on the device, sums in fp64
    rep32 = M.quality_report(e.astype(np.float32), t.astype(np.float32))
    assert abs(rep32.psnr - O.psnr(e.astype(np.float32), t.astype(np.float32))) <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_gpu_run_resident_quality_matches_downloaded(dtype):
    """run(..., truth=) reports quality of the resident X; it equals the
    metrics of the returned X (no download inside the loop)."""
    import paper_2510_22506_b200 as P
    from paper_2510_22506_b200 import metrics as M
    from paper_2510_22506_b200.workloads import make_instance
    wl, truth, mask = make_instance("c1", dims=(64, 48, 3))
    cfg = P.SolverConfig(lam=0.35, delta=0.5, rho=0.1, eps=0.0, max_iters=6, max_rank=4, initial_rank=4,
                         rank_policy="fixed", algorithm="afctnlr", shuffle=True, seed=0)
    res = P.run(P.Observation(truth, mask), cfg, dtype=dtype, truth=truth, quality_every=2)
    assert [it for it, _ in res.quality] == [2, 4, 6]
    last = res.quality[-1][1]
    ref = M.quality_report(res.x, truth)
    assert abs(last.psnr - ref.psnr) <= 1e-9 and abs(last.ssim - ref.ssim) <= 1e-10
    assert last.rel_err == pytest.approx(ref.rel_err, rel=1e-10)
    assert abs(last.psnr - O.psnr(res.x, truth)) <= 1e-9


@pytest.mark.gpu
def test_rel_err_any_order_like_reference():
    """rel_err accepts 1-D and 0-D tensors like the reference (metrics.py:70-92)."""
    from paper_2510_22506_b200 import metrics as M
    rng = np.random.default_rng(5)
    a, b = rng.standard_normal(100), rng.standard_normal(100)
    want = float(np.linalg.norm(a - b) / np.linalg.norm(b))
    assert M.rel_err(a, b) == pytest.approx(want, rel=1e-12)
    m = rng.random(100) < 0.3
    want_m = float(np.linalg.norm(a[~m] - b[~m]) / np.linalg.norm(b[~m]))
    assert M.rel_err(a, b, m) == pytest.approx(want_m, rel=1e-12)
    assert M.rel_err(np.float64(2.0), np.float64(1.0)) == pytest.approx(1.0)
