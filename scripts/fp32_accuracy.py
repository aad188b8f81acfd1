"""FP32-variant accuracy vs the FP64 oracle on scaled c4/c5 instances (1xTF32 vs 3xTF32)."""
import os, subprocess, sys, json
sys.path.insert(0, '.')
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2510_22506_b200 as P
    from oracle import fctn_oracle as O
    from paper_2510_22506_b200.workloads import make_instance
    name, dims = sys.argv[2], tuple(int(v) for v in sys.argv[3].split("x"))
    wl, truth, mask = make_instance(name, dims=dims)
    kw = dict(lam=0.35, delta=0.5, rho=0.1, eps=0.0, max_iters=20, max_rank=wl.rank, initial_rank=wl.rank,
              rank_policy="fixed", algorithm="afctnlr", shuffle=True, seed=0)
    cache = f"/tmp/oracle_{name}_{sys.argv[3]}.npy"
    if os.path.exists(cache):
        refx = np.load(cache)
    else:
        refx = O.run(truth, mask, **kw).x
        np.save(cache, refx)
    res = P.run(P.Observation(truth, mask), P.SolverConfig(**kw), dtype="float32")
    peak = float(np.max(np.abs(truth)))
    print(json.dumps({"rel": float(np.linalg.norm(res.x - refx) / np.linalg.norm(refx)),
                      "dpsnr": abs(O.psnr(res.x, truth, peak) - O.psnr(refx, truth, peak))}))
else:
    for name, dims in [("c4", "256x256x64"), ("c5", "20x20x20x20x20")]:
        for mode in ["3x", "1x"]:
            out = subprocess.run([sys.executable, __file__, "child", name, dims], env=dict(os.environ, FCTN_TF32=mode),
                                 capture_output=True, text=True)
            print(name, dims, mode, out.stdout.strip() or out.stderr[-500:])
