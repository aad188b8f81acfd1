"""Full-size goldens: the REAL reference (`fctnlr` 0.1.0) run once on the
BASELINE.json configurations c3 (30 it), c4 (20 it) and c5 (20 it).

Run in the authoring container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 FCTN_THREADS=8 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_fullsize_golden.py c3 c4 c5

c4/c5 need ~20-25 GB of host RAM and 8-17 min each on 8 cores.  Outputs
`tests/golden/full_<cfg>.npz` (committed), compact by design:

* the inputs are NOT stored: the GPU test regenerates them with
  `paper_2510_22506_b200.workloads.make_instance` (seeded numpy) and checks
  the stored SHA-256 of truth and mask so generator drift fails loudly;
* the full per-iteration trace (objective, rel_change, x_norm, step_sq,
  factor_norm, FLOP / cache-hit integers) and the initial objective;
* the factors' mode-k unfoldings after iterations 1, 5 and the last one;
* X after iterations 1, 5 and the last one at seeded sample positions
  (2^20 for the last iteration — 2^18 on c3 — and 2^16 for 1 and 5; positions regenerate from
  `sample_positions`) plus the slice sums along every mode (a checksum of the
  whole tensor);
* PSNR / SSIM / rel-err of the final X against the truth (`metrics.py:33-92`),
  c5 with ``peak = max|truth|``;
* the reference's own per-iteration wall_ms and the host it ran on.

The per-iteration snapshots come from ONE run: `fctnlr.solver.objective` is
wrapped so each call at solver.py:356 (x_new, f after iteration t) is
recorded; the wrapper returns the reference's own value unchanged.
"""
from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

SNAP_ITERS = (1, 5)
N_SAMPLE_FINAL = 1 << 20
N_SAMPLE_SNAP = 1 << 16


def sample_positions(total: int, count: int, seed: int = 20251022) -> np.ndarray:
    """Sorted distinct F-order flat positions (shared with the GPU test)."""
    count = min(count, total)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(total, size=count, replace=False))


def slice_sums(x: np.ndarray) -> list:
    n = x.ndim
    return [x.sum(axis=tuple(j for j in range(n) if j != k)) for k in range(n)]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a.ravel(order="F")).view(np.uint8)).hexdigest()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def make(name: str) -> None:
    import fctnlr.solver as S
    from fctnlr.fileio import sample_mask as ref_sample_mask
    from fctnlr.metrics import psnr, rel_err, ssim
    from fctnlr.tensor import mode_unfold

    from paper_2510_22506_b200.workloads import make_instance

    wl, truth, mask = make_instance(name)
    ref_mask = ref_sample_mask(wl.dims, wl.sample_rate, 0)
    assert np.array_equal(mask, ref_mask), "workload mask differs from fctnlr.fileio.sample_mask"
    n = len(wl.dims)
    total = int(np.prod(wl.dims))
    pos_final = sample_positions(total, N_SAMPLE_FINAL if total > 1 << 24 else N_SAMPLE_FINAL // 4)
    pos_snap = sample_positions(total, N_SAMPLE_SNAP)
    kw = dict(lam=0.35, delta=0.5, rho=0.1, eps=0.0, max_iters=wl.iters, max_rank=wl.rank,
              initial_rank=wl.rank, rank_policy="fixed", algorithm="afctnlr", shuffle=True, seed=0)
    store = {}
    calls = {"n": 0}
    real_objective = S.objective

    def spy(x, f, laps, lams, obs=None, composed=None):
        val = real_objective(x, f, laps, lams, obs=obs, composed=composed)
        it = calls["n"]
        calls["n"] += 1
        if it in SNAP_ITERS:
            xf = np.asarray(x).ravel(order="F")
            store[f"it{it}_xs"] = xf[pos_snap].copy()
            for k, v in enumerate(slice_sums(np.asarray(x))):
                store[f"it{it}_sum{k}"] = v
            for k in range(n):
                store[f"it{it}_a{k}"] = np.ascontiguousarray(mode_unfold(f.factor(k), k))
        return val

    obs = S.Observation.from_dense(truth, mask)
    cfg = S.SolverConfig(**kw)
    S.objective = spy
    t0 = time.perf_counter()
    try:
        res = S.run(obs, cfg)
    finally:
        S.objective = real_objective
    wall = time.perf_counter() - t0
    x = res.x
    xf = x.ravel(order="F")
    store["final_xs"] = xf[pos_final].copy()
    for k, v in enumerate(slice_sums(x)):
        store[f"final_sum{k}"] = v
    for k in range(n):
        store[f"final_a{k}"] = np.ascontiguousarray(mode_unfold(res.factors.factor(k), k))
    store["final_versions"] = np.asarray(res.factors.versions)
    for fld in ("objective", "rel_change", "step_sq", "x_norm", "factor_norm", "wall_ms"):
        store["trace_" + fld] = np.asarray([getattr(r, fld) for r in res.trace], dtype=np.float64)
    for fld in ("flops", "mk_flops", "compose_flops", "cache_hits"):
        store["trace_" + fld] = np.asarray([getattr(r, fld) for r in res.trace], dtype=np.int64)
    store["initial_objective"] = np.asarray(res.initial_objective)
    peak = float(np.max(np.abs(truth))) if wl.kind == "fctn" else 1.0
    store["peak"] = np.asarray(peak)
    store["psnr"] = np.asarray(psnr(x, truth, peak=peak))
    store["ssim"] = np.asarray(ssim(x, truth, peak=peak))
    store["rel_err"] = np.asarray(rel_err(x, truth))
    store["truth_sha256"] = np.asarray(digest(truth))
    store["mask_sha256"] = np.asarray(digest(mask.astype(np.uint8)))
    meta = dict(config=name, dims=list(wl.dims), rank=wl.rank, sample_rate=wl.sample_rate,
                iters=wl.iters, solver=kw, n_sample_final=int(pos_final.size),
                n_sample_snap=int(pos_snap.size), snap_iters=list(SNAP_ITERS),
                host=dict(cpu=cpu_model(), cores=os.cpu_count(),
                          fctn_threads=os.environ.get("FCTN_THREADS", ""),
                          numpy=np.__version__, python=platform.python_version()),
                total_wall_s=wall,
                median_wall_ms=float(np.median(store["trace_wall_ms"])))
    store["meta_json"] = np.asarray(json.dumps(meta))
    out = os.path.join(HERE, f"full_{name}.npz")
    np.savez_compressed(out, **store)
    print(name, json.dumps(meta), "psnr", float(store["psnr"]), flush=True)


if __name__ == "__main__":
    for cfg_name in sys.argv[1:] or ["c3", "c4", "c5"]:
        make(cfg_name)
