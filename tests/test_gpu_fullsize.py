"""Full-size properties at the BASELINE configs the oracle cannot run in
seconds (c4: 2048x2048x64 R=8, c5: 48^5 R=3; FP32 variant, 3 sweeps):

* observed entries restored bit for bit (solver.py:235-236);
* sufficient decrease f_t + rho/2 step_t^2 <= f_{t-1} (test_solver.py:283-294),
  with an FP32 allowance of 1e-5 relative;
* determinism: two runs give identical bits (test_acceptance.py:407-443);
* the trace FLOP / cache-hit integers equal the shape-only replay of the
  reference meter for the same visiting orders (fctn_plan_sweeps);
* quality on the resident X (metrics.cu) equals the metrics of the
  downloaded X.
"""
import numpy as np
import pytest

import paper_2510_22506_b200 as P
from paper_2510_22506_b200 import _native
from paper_2510_22506_b200.network import FctnRank
from paper_2510_22506_b200.workloads import make_instance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_gpu_fullsize_properties(name):
    wl, truth, mask = make_instance(name)
    n = len(wl.dims)
    cfg = P.SolverConfig(lam=0.35, delta=0.5, rho=0.1, eps=0.0, max_iters=3, max_rank=wl.rank,
                         initial_rank=wl.rank, rank_policy="fixed", algorithm="afctnlr", shuffle=True, seed=0)
    obs = P.Observation(truth, mask)
    peak = float(np.max(np.abs(truth)))
    a = P.run(obs, cfg, dtype="float32", truth=truth, peak=peak)
    # observed entries bit-exact (fp32-rounded data)
    x32 = truth.astype(np.float32).astype(np.float64)
    assert np.array_equal(a.x[mask], x32[mask])
    # sufficient decrease
    prev = a.initial_objective
    for rec in a.trace:
        assert rec.objective + 0.5 * cfg.rho * rec.step_sq <= prev * (1 + 1e-5)
        prev = rec.objective
    # reference FLOP meter replay for the same orders (identity, then the seeded permutations)
    rng = np.random.default_rng(cfg.seed)
    from paper_2510_22506_b200.network import FctnFactors
    FctnFactors.random(wl.dims, FctnRank.uniform(n, wl.rank), rng)  # same draws as run()
    orders = [tuple(range(n))]
    for _ in range(cfg.max_iters - 1):
        orders.append(tuple(int(v) for v in rng.permutation(n)))
    ct = _native.plan_sweeps(wl.dims, FctnRank.uniform(n, wl.rank).entries, _native.ALG_ACCEL, cfg.cache_budget,
                             orders)
    assert [r.flops for r in a.trace] == [int(v) for v in ct[:, _native.CT_FLOPS]]
    assert [r.cache_hits for r in a.trace] == [int(v) for v in ct[:, _native.CT_HITS]]
    # quality of the resident X == metrics of the downloaded X
    from paper_2510_22506_b200 import metrics as M
    it, q = a.quality[-1]
    assert it == 3
    ref = M.quality_report(a.x, truth, peak=peak)
    assert abs(q.psnr - ref.psnr) <= 1e-6 and abs(q.ssim - ref.ssim) <= 1e-9
    assert q.rel_err == pytest.approx(ref.rel_err, rel=1e-9)
    # determinism
    b = P.run(obs, cfg, dtype="float32")
    assert np.array_equal(a.x, b.x)
    assert [r.objective for r in a.trace] == [r.objective for r in b.trace]
