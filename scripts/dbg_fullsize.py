"""Debug helper: one FP64/FP32 sweep sequence at a full-size config (run under
compute-sanitizer on the GPU box)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2510_22506_b200 as P  # noqa: E402
from paper_2510_22506_b200.workloads import make_instance  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
wl, truth, mask = make_instance(name)
cfg = P.SolverConfig(lam=0.35, delta=0.5, rho=0.1, eps=0.0, max_iters=iters, max_rank=wl.rank,
                     initial_rank=wl.rank, rank_policy="fixed", algorithm="afctnlr", shuffle=True, seed=0)
t0 = time.time()
res = P.run(P.Observation(truth, mask), cfg, dtype=dtype)
print(name, dtype, [round(r.objective, 6) for r in res.trace], [round(r.device_ms, 3) for r in res.trace],
      f"{time.time() - t0:.1f}s")
