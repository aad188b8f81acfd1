"""GPU tests of the mode-0 sharded sweep (fctn_set_comm / fctn_set_comm_host).

Two ranks share the one GPU of the test box and exchange through gloo on host
memory (the host-callback backend: no kernel ever waits on another rank's
kernel).  The sharded run must reproduce the single-GPU run; the NCCL backend
is exercised with one rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance(dims, seed=9):
    rng = np.random.default_rng(seed)
    values = rng.standard_normal(dims)
    if len(dims) >= 3:
        values = np.cumsum(np.cumsum(values, axis=0), axis=1) / 10.0  # smoother, completable
    mask = rng.random(dims) < 0.35
    return values, mask


def _cfg(n):
    import paper_2510_22506_b200 as P
    return P.SolverConfig(lam=0.35, delta=0.5, rho=0.1, eps=0.0, max_iters=6, max_rank=2, initial_rank=2,
                          rank_policy="fixed", algorithm="afctnlr", shuffle=True, seed=2)


def _worker(rank, world, port, dims, dtype, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2510_22506_b200 as P
    values, mask = _instance(dims)
    res = P.run(P.Observation(values, mask), _cfg(len(dims)), dtype=dtype, device=0,
                shard=P.Shard(rank, world, backend="host"), truth=values, quality_every=3)
    q = np.array([[it, r.psnr, r.ssim, r.rel_err] for it, r in res.quality])
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=res.x, slab=np.array(res.slab), q=q,
             obj=np.array([r.objective for r in res.trace]), flops=np.array([r.flops for r in res.trace]),
             hits=np.array([r.cache_hits for r in res.trace]),
             *[res.factors.factor(k) for k in range(len(dims))])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,dtype,tol", [((12, 10, 3), "float64", 1e-11), ((9, 6, 5, 4), "float64", 1e-11),
                                            ((16, 12, 8), "float32", 2e-5)])
def test_gpu_sharded_host_backend_matches_single(tmp_path, dims, dtype, tol):
    import paper_2510_22506_b200 as P
    mp.spawn(_worker, args=(2, _port(), dims, dtype, str(tmp_path)), nprocs=2, join=True)
    values, mask = _instance(dims)
    ref = P.run(P.Observation(values, mask), _cfg(len(dims)), dtype=dtype, truth=values, quality_every=3)
    r = [np.load(tmp_path / f"r{i}.npz") for i in range(2)]
    x = np.concatenate([r[0]["x"], r[1]["x"]], axis=0)
    assert tuple(r[0]["slab"]) == (0, dims[0] // 2)
    assert np.linalg.norm(x - ref.x) <= tol * np.linalg.norm(ref.x)
    for k in range(len(dims)):
        assert np.array_equal(r[0][f"arr_{k}"], r[1][f"arr_{k}"])  # replicated factors, same bits
        f = ref.factors.factor(k)
        assert np.linalg.norm(r[0][f"arr_{k}"] - f) <= tol * np.linalg.norm(f)
    np.testing.assert_allclose(r[0]["obj"], [t.objective for t in ref.trace], rtol=tol)
    assert list(r[0]["flops"]) == [t.flops for t in ref.trace]  # global FLOP meter
    assert list(r[0]["hits"]) == [t.cache_hits for t in ref.trace]
    # resident-X quality: per-slice sums all-reduced over the two slabs
    qref = np.array([[it, q.psnr, q.ssim, q.rel_err] for it, q in ref.quality])
    assert qref[:, 0].tolist() == [3, 6]
    for i in range(2):
        np.testing.assert_allclose(r[i]["q"], qref, rtol=max(tol, 1e-10), atol=0)


def test_gpu_nccl_single_rank_matches_plain():
    """fctn_set_comm with one NCCL rank runs the sharded code path end to end."""
    import paper_2510_22506_b200 as P
    from paper_2510_22506_b200 import _native
    from paper_2510_22506_b200.network import FctnFactors, FctnRank
    dims = (10, 8, 6)
    values, mask = _instance(dims)
    obs = P.Observation(values, mask)
    rk = FctnRank.uniform(3, 2)

    def go(use_comm):
        ctx = _native.Context(0, _native.F64, dims, rk.entries, (0.35,) * 3, (0.5,) * 3, _native.SIGN_PD, 0.1,
                              _native.ALG_ACCEL, 1 << 30)
        if use_comm:
            ctx.set_comm_nccl(_native.nccl_unique_id(), 0, 1)
        ctx.upload(obs.values, obs.mask)
        f = FctnFactors.random(dims, rk, np.random.default_rng(0))
        ctx.set_factors(f.unfoldings(), f.versions, True)
        ctx.objective()
        for order in [(0, 1, 2), (2, 0, 1), (1, 2, 0)]:
            ctx.sweep(order)
        x = ctx.get_x()
        ctx.close()
        return x

    a, b = go(False), go(True)
    assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(a)


@pytest.mark.parametrize("dims,dt,ranks", [((512, 256, 64), "f32", 2), ((64, 48, 12), "f64", 4)])
def test_gpu_loopback_rank_replays_graphs_like_eager_host_backend(dims, dt, ranks):
    """A rank's sharded sweep captured and replayed as a CUDA graph (device
    loop-back collectives, the same stream work as NCCL) gives the bits of the
    eager host-callback run with the same fake collectives; the (512, 256, 64)
    fp32 slab runs the tensor-core stream / compose kernels at their per-rank
    shapes."""
    from paper_2510_22506_b200 import _native
    from paper_2510_22506_b200.network import FctnFactors, FctnRank
    values, mask = _instance(dims)
    rk = FctnRank.uniform(3, 4)
    dtype = _native.F32 if dt == "f32" else _native.F64

    def go(loopback):
        ctx = _native.Context(0, dtype, dims, rk.entries, (0.35,) * 3, (0.5,) * 3, _native.SIGN_PD, 0.1,
                              _native.ALG_ACCEL, 1 << 30)
        if loopback:
            ctx.set_comm_loopback(0, ranks)
        else:
            ctx.set_comm_host(lambda a: None, lambda s: np.tile(s, ranks), 0, ranks)
        lo, hi = ctx.slab
        ctx.upload_f64(np.asfortranarray(values[lo:hi]), np.asfortranarray(mask[lo:hi]))
        f = FctnFactors.random(dims, rk, np.random.default_rng(0))
        ctx.set_factors(f.unfoldings(), f.versions, True)
        ctx.objective()
        launches = []
        for order in [(0, 1, 2), (2, 0, 1), (1, 2, 0), (2, 0, 1)]:
            _, counters = ctx.sweep(order)
            launches.append(int(counters[_native.CT_LAUNCHES]))
        x = ctx.get_x_f64()
        fac = ctx.get_factors([(d, 16) for d in dims])
        ctx.close()
        return x, fac, launches

    (xa, fa, la), (xb, fb, lb) = go(False), go(True)
    assert np.isfinite(xa).all() and xa.shape[0] == dims[0] // ranks
    assert np.array_equal(xa, xb)
    for a, b in zip(fa, fb):
        assert np.array_equal(a, b)
    assert min(la) > 0 and min(lb) > 0  # graph replays report their captured launch counts
