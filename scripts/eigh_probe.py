"""One eigendecomposition launch (profiling target for ncu)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2510_22506_b200 import _native  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rng = np.random.default_rng(S)
M = rng.standard_normal((S, 3 * S + 5))
G = M @ M.T
V, phi, ms, sweeps = _native.selftest_eigh(G, reps=3)
print(f"S={S} sweeps={sweeps} ms={ms:.3f}")
