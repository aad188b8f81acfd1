"""Per-rank kernel-time model of the mode-0 sharded sweep from
one GPU: rank 0 of G runs its slab with device-side loop-back collectives
(fctn_set_comm_loopback: allreduce = identity, allgather = G copies of the
local rows), so every kernel has the shape and size it has on a real G-GPU
run while the numbers are not the global ones.  Two figures per G: the
event-timed sweep with CUDA-graph replay (what a rank spends between its
collectives) and the per-class device times of a profiled, eager pass.  The
collectives themselves (NCCL over NVLink, a few per factor update) are listed
separately with their message sizes.

    python scripts/shard_model.py [c4|c5] > profiles/r02/shard_model_c4.json
"""
import json
import math
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2510_22506_b200 as P  # noqa: E402
from paper_2510_22506_b200 import _native  # noqa: E402
from paper_2510_22506_b200.network import FctnFactors, FctnRank  # noqa: E402
from paper_2510_22506_b200.workloads import make_instance  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl, truth, mask = make_instance(name)
n = len(wl.dims)
dt = _native.F32 if wl.dtype == "f32" else _native.F64
rk = FctnRank.uniform(n, wl.rank)
obs = P.Observation(truth, mask)
out = {"config": name, "dims": list(wl.dims), "ranks": {}}
for G in (1, 2, 4, 8):
    ctx = _native.Context(0, dt, wl.dims, rk.entries, (0.35,) * n, (0.5,) * n, _native.SIGN_PD, 0.1,
                          _native.ALG_ACCEL, 1 << 30, numeric_exc=P.NumericalFailure)
    if G > 1:
        ctx.set_comm_loopback(0, G)
    lo, hi = ctx.slab if G > 1 else (0, wl.dims[0])
    ctx.upload_f64(np.asfortranarray(obs.values[lo:hi]), np.asfortranarray(obs.mask[lo:hi]))
    rng = np.random.default_rng(0)
    f = FctnFactors.random(wl.dims, rk, rng)
    ctx.set_factors(f.unfoldings(), f.versions, True)
    ctx.objective()
    order = tuple(range(n))
    for _ in range(3):
        ctx.sweep(order)
        order = tuple(int(v) for v in rng.permutation(n))
    steps = 10
    replay = []
    for _ in range(steps):  # graph replay (three-mode configs), event-timed
        stats, _ = ctx.sweep(order)
        replay.append(float(stats[_native.ST_DEVICE_MS]))
        order = tuple(int(v) for v in rng.permutation(n))
    ctx.set_profiling(True)
    dev = []
    for _ in range(steps):
        stats, _ = ctx.sweep(order)
        dev.append(float(stats[_native.ST_DEVICE_MS]))
        order = tuple(int(v) for v in rng.permutation(n))
    prof = ctx.get_profile()
    ctx.close()
    cls = {k: round(v["ms"] / steps, 4) for k, v in prof.items() if v["ms"] > 0}
    kernel_ms = round(sum(cls.values()), 4)
    s = wl.rank ** (n - 1)
    coll = {"allreduce_Y_doubles": [int(wl.dims[k] * s) for k in range(1, n)],
            "allgather_Y0_rows": int(math.ceil(wl.dims[0] / G)) * s, "allreduce_sums": 4,
            "per_sweep": n + 1}
    out["ranks"][G] = {"slab_rows": hi - lo, "per_class_ms": cls, "kernel_ms_per_sweep": kernel_ms,
                       "event_ms_per_sweep_median": round(float(np.median(replay)), 4),
                       "profiled_event_ms_per_sweep_median": round(float(np.median(dev)), 4),
                       "collectives": coll if G > 1 else None}
    print(G, round(float(np.median(replay)), 4), kernel_ms, cls, file=sys.stderr)
json.dump(out, sys.stdout, indent=1)
print()
