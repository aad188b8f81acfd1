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


@pytest.mark.parametrize("dims,k,S", [((30, 20, 10), 0, 16), ((30, 20, 10), 1, 36), ((7, 9, 5, 6), 2, 125),
                                     # DMMA form (I, S >= 16): P == 1, P > 1, ragged tiles, several splits
                                     ((144, 40, 6), 0, 125), ((36, 176, 5), 1, 125), ((9, 8, 50, 3), 2, 25),
                                     ((64, 2048, 3), 1, 64)])
def test_stream_fp64_matches_numpy(dims, k, S):
    rng = np.random.default_rng(4)
    x = np.asfortranarray(rng.standard_normal(dims))
    p = int(np.prod(dims)) // dims[k]
    m = np.asfortranarray(rng.standard_normal((p, S)))
    ref = _unfold(x, k) @ m
    y = _native.selftest_stream(x, m, k)
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) <= 1e-13


@pytest.mark.parametrize("S,H1", [
    (16, 129), (36, 129), (64, 1025), (81, 25), (125, 89),
    (64, 33),    # 32 x 32 threads, TL = 2, s = SP: the unchecked substitution steps
    (48, 300),   # 16 x 16 threads, TL = 3, s = SP
    (100, 200),  # 16 x 16 threads, TL = 7: per-column barriers instead of panels
    (144, 40),   # 32 x 32 threads, TL = 5 (s <= 146 fits the CTA's shared memory)
])
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


@pytest.mark.parametrize("S", [1, 3, 16, 36, 64, 81, 111, 125, 216])
def test_eigh_jacobi_matches_numpy(S):
    """eig_gram (sylvester.py:51-61) on the device: one-sided Jacobi from a
    cold start and from a perturbed warm start.  V orthonormal, V^T G V
    diagonal, eigenvalues equal numpy's eigvalsh (clamped at 0); s = 125 / 216
    run from global memory (beyond the shared-memory form's s <= 117)."""
    rng = np.random.default_rng(S)
    M = rng.standard_normal((S, 3 * S + 5))
    M[:, :2] *= 1e3  # a spread spectrum like a factor Gram network
    G = M @ M.T
    G = 0.5 * (G + G.T)
    ref = np.clip(np.linalg.eigvalsh(G), 0.0, None)
    scale = float(np.abs(G).max())
    V, phi, ms, sweeps = _native.selftest_eigh(G)
    assert np.abs(V.T @ V - np.eye(S)).max() <= 1e-13 * max(S, 1)
    D = V.T @ G @ V
    assert np.abs(D - np.diag(np.diag(D))).max() <= 2e-14 * S * scale
    assert np.allclose(np.sort(phi), ref, rtol=1e-12, atol=1e-13 * scale)
    # warm start: the basis of a slightly different G converges in few sweeps
    G2 = G + 1e-6 * scale * np.diag(rng.standard_normal(S))
    G2 = 0.5 * (G2 + G2.T)
    V2, phi2, ms2, sweeps2 = _native.selftest_eigh(G2, V0=V)
    D2 = V2.T @ G2 @ V2
    assert np.abs(D2 - np.diag(np.diag(D2))).max() <= 2e-14 * S * scale
    assert np.abs(V2.T @ V2 - np.eye(S)).max() <= 1e-13 * max(S, 1)
    assert sweeps2 <= sweeps
    print(f"S={S}: cold {sweeps} sweeps {ms:.3f} ms, warm {sweeps2} sweeps {ms2:.3f} ms")
