import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2510_22506_b200 import _native
for S, H1 in [(16, 1025), (36, 129), (64, 33), (64, 1025), (81, 25), (125, 89)]:
    rng = np.random.default_rng(0)
    Mk = rng.standard_normal((S, 4 * S)); G = Mk @ Mk.T
    mu = 0.1 + rng.random(H1); Fr = rng.standard_normal((H1, S)); Fi = rng.standard_normal((H1, S))
    _, _, ms = _native.selftest_chol(G, mu, Fr, Fi, reps=5)
    print(f"S={S} H1={H1}: {ms*1e3:.1f} us/launch")
