"""World-size-2 gloo tests (CPU) of the mode-0 sharding decomposition that
the device path implements (fctn_set_comm / fctn_set_comm_host): the sharded
restatement, exchanging through torch.distributed, must reproduce the
unsharded sweep."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from tests.shard_oracle import sharded_run

    rng = np.random.default_rng(5)
    values = rng.standard_normal(dims)
    mask = rng.random(dims) < 0.4

    def allreduce(a):
        t = torch.from_numpy(a)
        dist.all_reduce(t)

    def allgather(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return torch.cat(out).numpy()

    xs, factors, rel, sums = sharded_run(values, mask, rank, world, allreduce, allgather, max_iters=4, rank_r=2,
                                         seed=1, shuffle=False)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=xs, rel=rel, *factors)
    dist.barrier()
    dist.destroy_process_group()


def _reference(dims):
    from tests.shard_oracle import sharded_run
    rng = np.random.default_rng(5)
    values = rng.standard_normal(dims)
    mask = rng.random(dims) < 0.4
    return sharded_run(values, mask, 0, 1, lambda a: None, lambda a: a, max_iters=4, rank_r=2, seed=1, shuffle=False)


@pytest.mark.parametrize("dims", [(9, 6, 5), (8, 5, 4, 3)])
def test_sharded_sweep_matches_unsharded_gloo(tmp_path, dims):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, dims, str(tmp_path)), nprocs=2, join=True)
    x_full, f_full, rel_full, _ = _reference(dims)
    r0 = np.load(tmp_path / "r0.npz")
    r1 = np.load(tmp_path / "r1.npz")
    x = np.concatenate([r0["x"], r1["x"]], axis=0)
    assert np.linalg.norm(x - x_full) <= 1e-12 * np.linalg.norm(x_full)
    for k in range(len(dims)):
        a0, a1 = r0[f"arr_{k}"], r1[f"arr_{k}"]
        assert np.array_equal(a0, a1)  # replicated factors stay bitwise identical
        assert np.linalg.norm(a0 - f_full[k]) <= 1e-12 * np.linalg.norm(f_full[k])
    assert abs(float(r0["rel"]) - rel_full) <= 1e-12 * rel_full


def test_unsharded_restatement_matches_oracle():
    """The restatement with one rank is the oracle's plain sweep."""
    from oracle import fctn_oracle as O
    dims = (9, 6, 5)
    rng = np.random.default_rng(5)
    values = rng.standard_normal(dims)
    mask = rng.random(dims) < 0.4
    x, factors, rel, _ = _reference(dims)
    ref = O.run(values, mask, max_iters=4, max_rank=2, initial_rank=2, rank_policy="fixed", eps=0.0,
                algorithm="fctnlr", shuffle=False, seed=1)
    assert np.linalg.norm(x - ref.x) <= 1e-12 * np.linalg.norm(ref.x)
