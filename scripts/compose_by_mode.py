"""Per-order sweep and compose time at a config (which mode is last decides
the compose shape): profiled sweeps with fixed visiting orders."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2510_22506_b200 as P  # noqa: E402
from paper_2510_22506_b200 import _native  # noqa: E402
from paper_2510_22506_b200.network import FctnFactors, FctnRank  # noqa: E402
from paper_2510_22506_b200.workloads import make_instance  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
wl, truth, mask = make_instance(name)
n = len(wl.dims)
rk = FctnRank.uniform(n, wl.rank)
ctx = _native.Context(0, _native.F32 if wl.dtype == "f32" else _native.F64, wl.dims, rk.entries, (0.35,) * n,
                      (0.5,) * n, _native.SIGN_PD, 0.1, _native.ALG_ACCEL, 1 << 30, numeric_exc=P.NumericalFailure)
ctx.upload_f64(truth, mask)
f = FctnFactors.random(wl.dims, rk, np.random.default_rng(0))
ctx.set_factors(f.unfoldings(), f.versions, True)
ctx.objective()
for last in range(n):
    order = tuple([j for j in range(n) if j != last] + [last])
    for _ in range(2):
        ctx.sweep(order)
    ctx.set_profiling(True)
    ms = [float(ctx.sweep(order)[0][_native.ST_DEVICE_MS]) for _ in range(3)]
    prof = ctx.get_profile()
    ctx.set_profiling(False)
    print(f"last={last} order={order} sweep_ms={np.median(ms):.3f} compose_ms={prof['compose']['ms'] / 3:.3f}")
