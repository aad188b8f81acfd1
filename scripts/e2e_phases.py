"""Time the phases of one run(obs, cfg) call (host wall) on a config."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2510_22506_b200 as P
from paper_2510_22506_b200 import _native
from paper_2510_22506_b200.network import FctnFactors, FctnRank
from paper_2510_22506_b200.workloads import make_instance
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl, truth, mask = make_instance(name)
obs = P.Observation(truth, mask)
n = len(wl.dims)
dt = _native.F32 if wl.dtype == "f32" else _native.F64
rk = FctnRank.uniform(n, wl.rank)
for rep in range(2):
    t = [time.perf_counter()]
    ctx = _native.Context(0, dt, wl.dims, rk.entries, (0.35,) * n, (0.5,) * n, 0, 0.1, 1, 1 << 30); t.append(time.perf_counter())
    ctx.upload_f64(obs.values, obs.mask); t.append(time.perf_counter())
    f = FctnFactors.random(wl.dims, rk, np.random.default_rng(0)); ctx.set_factors(f.unfoldings(), f.versions, True); t.append(time.perf_counter())
    ctx.objective(); t.append(time.perf_counter())
    for _ in range(20): ctx.sweep(tuple(range(n)))
    t.append(time.perf_counter())
    x = ctx.get_x_f64(); t.append(time.perf_counter())
    ctx.close(); t.append(time.perf_counter())
    names = ["create", "upload", "set_factors", "objective", "20 sweeps", "get_x", "close"]
    print(rep, {k: round((t[i + 1] - t[i]) * 1e3, 1) for i, k in enumerate(names)})
t0 = time.perf_counter()
cfg = P.SolverConfig(max_iters=20, max_rank=wl.rank, initial_rank=wl.rank, lam=0.35, delta=0.5, rho=0.1, eps=0.0,
                     rank_policy="fixed", algorithm="afctnlr", shuffle=True, seed=0)
res = P.run(obs, cfg, dtype="float32" if dt == _native.F32 else "float64")
print("run() total ms", round((time.perf_counter() - t0) * 1e3, 1))

# ---- six more run() calls with the context methods timed (which phase varies call to call?)
import gc
acc = {}
def _wrap(cls, name):
    f = getattr(cls, name)
    def g(self, *a, **k):
        t = time.perf_counter()
        try:
            return f(self, *a, **k)
        finally:
            acc[name] = acc.get(name, 0.0) + (time.perf_counter() - t) * 1e3
    setattr(cls, name, g)
for nm in ("__init__", "upload_f64", "set_factors", "sweep", "objective", "get_x_f64", "get_factors", "close"):
    _wrap(_native.Context, nm)
del res
for i in range(6):
    acc.clear()
    gc.collect()
    t0 = time.perf_counter()
    res = P.run(obs, cfg, dtype="float32" if dt == _native.F32 else "float64")
    tot = (time.perf_counter() - t0) * 1e3
    print("run", i, "total", round(tot, 1), {k: round(v, 1) for k, v in acc.items()},
          "other", round(tot - sum(acc.values()), 1), "pool idle", _native._HOST_POOL_IDLE[0] >> 20, "MB")
    del res
