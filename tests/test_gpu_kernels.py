"""GPU unit tests of single kernels through the C ABI self-test entry points
(each against a numpy fp64 product of the same inputs)."""
import numpy as np
import pytest

from paper_2510_22506_b200 import _native

pytestmark = pytest.mark.gpu


def _unfold(x, k):
    rest = [m for m in range(x.ndim) if m != k]
    return np.transpose(x, [k] + rest).reshape((x.shape[k], -1), order="F")


@pytest.mark.parametrize("dims,k,S", [
    ((256, 64, 8), 0, 64), ((256, 64, 8), 1, 64), ((256, 64, 8), 2, 64),
    ((48, 40, 36), 0, 81), ((48, 40, 36), 1, 27), ((48, 40, 36), 2, 9),
    ((2048, 32, 4), 0, 64), ((20, 20, 20, 20), 3, 27),
    # > 148 row tiles, unsplit: the persistent kernel (MN-major, K-major, ragged rows / bonds)
    ((20480, 8, 4), 0, 64), ((32, 20480, 2), 1, 64), ((16, 20608, 2), 1, 20), ((40, 19000, 2), 1, 64),
])
@pytest.mark.parametrize("use_tc", [True, False])
def test_stream_fp32_matches_numpy(dims, k, S, use_tc):
    rng = np.random.default_rng(3)
    x = np.asfortranarray(rng.standard_normal(dims).astype(np.float32))
    p = int(np.prod(dims)) // dims[k]
    m = np.asfortranarray(rng.standard_normal((p, S)).astype(np.float32))
    ref = _unfold(x.astype(np.float64), k) @ m.astype(np.float64)
    y = _native.selftest_stream(x, m, k, use_tc=use_tc)
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    # 3xTF32 (default) is FP32-class; FP32 SIMT accumulation over p ~ 1e-6
    assert err <= 1e-5, err


@pytest.mark.parametrize("dims,k,S", [((30, 20, 10), 0, 16), ((30, 20, 10), 1, 36), ((7, 9, 5, 6), 2, 125)])
def test_stream_fp64_matches_numpy(dims, k, S):
    rng = np.random.default_rng(4)
    x = np.asfortranarray(rng.standard_normal(dims))
    p = int(np.prod(dims)) // dims[k]
    m = np.asfortranarray(rng.standard_normal((p, S)))
    ref = _unfold(x, k) @ m
    y = _native.selftest_stream(x, m, k)
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-13


@pytest.mark.parametrize("S,H1", [(16, 129), (36, 129), (64, 1025), (81, 25), (125, 89)])
def test_chol_solves_match_numpy(S, H1):
    rng = np.random.default_rng(S)
    Mk = rng.standard_normal((S, 4 * S))
    G = Mk @ Mk.T
    mu = 0.1 + rng.random(H1)
    Fr = rng.standard_normal((H1, S))
    Fi = rng.standard_normal((H1, S))
    xr, xi, _ = _native.selftest_chol(G, mu, Fr, Fi)
    for w in range(0, H1, max(1, H1 // 17)):
        H = G + mu[w] * np.eye(S)
        np.testing.assert_allclose(H @ xr[w], Fr[w], rtol=1e-9, atol=1e-9 * np.abs(Fr[w]).max())
        np.testing.assert_allclose(H @ xi[w], Fi[w], rtol=1e-9, atol=1e-9 * np.abs(Fi[w]).max())


@pytest.mark.parametrize("dtype", [_native.F64, _native.F32])
def test_staged_transfers_roundtrip_partial_chunk(monkeypatch, dtype):
    """The pinned staging ring (fctn_ctx.cu Stager) on a tensor of two 32 MB
    chunks with a partial last one (threshold lowered by env), fp64 and the
    fp32 device-side conversion; then a second context in the same process
    (the ring is leased per device, not owned by the first context)."""
    monkeypatch.setenv("FCTN_STAGE_MIN_BYTES", str(1 << 20))
    dims = (1000, 700, 7)  # 4.9 M entries = 39.2 MB of fp64
    rng = np.random.default_rng(11)
    x = np.asfortranarray(rng.standard_normal(dims))
    mask = np.asfortranarray(rng.random(dims) < 0.3)
    want = x if dtype == _native.F64 else x.astype(np.float32).astype(np.float64)
    for _ in range(2):
        ctx = _native.Context(0, dtype, dims, (2, 2, 2), (0.35,) * 3, (0.5,) * 3, _native.SIGN_PD, 0.1,
                              _native.ALG_ACCEL, 1 << 30)
        try:
            ctx.upload_f64(x, mask)
            back = ctx.get_x_f64()
        finally:
            ctx.close()
        assert np.array_equal(back, want)
