"""Generate golden fixtures by running the REAL reference (`fctnlr` 0.1.0).

Run in the authoring container only (the reference is not on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Outputs `tests/golden/*.npz` (committed).  Each run case stores the inputs
(values, mask, config), the reference's final X and factors, its full trace,
and the X/factors after iteration 1 (a separate max_iters=1 run; the solver
is deterministic in its seed).  Solve cases store random subproblems and the
reference `solve_factor` output.  The FLOP-integer case stores first-sweep
counters for the reference's own benchmark shapes.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from fctnlr.fileio import sample_mask  # noqa: E402
from fctnlr.laplacian import CirculantLaplacian  # noqa: E402
from fctnlr.solver import Observation, SolverConfig, run  # noqa: E402
from fctnlr.sylvester import FactorSubproblem, NumericalFailure, solve_factor  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
TRACE_FIELDS = ["objective", "rel_change", "flops", "cache_hits", "mk_flops",
                "compose_flops", "step_sq", "x_norm", "factor_norm", "rank_grown"]

# name -> (dims, data kind, sample rate, data seed, SolverConfig kwargs)
RUN_CASES = {
    "n3_afctnlr": ((8, 7, 5), "normal", 0.4, 16,
                   dict(max_iters=15, eps=0.0, max_rank=2, initial_rank=2, rank_policy="fixed",
                        algorithm="afctnlr", seed=3)),
    "n4_afctnlr_shuffle": ((6, 5, 4, 3), "normal", 0.5, 20,
                           dict(max_iters=12, eps=0.0, max_rank=2, initial_rank=2, rank_policy="fixed",
                                algorithm="afctnlr", shuffle=True, seed=4)),
    "n4_afctnlr_identity": ((6, 6, 4, 4), "normal", 0.4, 5,
                            dict(max_iters=10, eps=0.0, max_rank=2, initial_rank=2, rank_policy="fixed",
                                 algorithm="afctnlr", shuffle=False, seed=5)),
    "n5_afctnlr": ((4, 3, 5, 3, 4), "normal", 0.5, 7,
                   dict(max_iters=6, eps=0.0, max_rank=2, initial_rank=2, rank_policy="fixed",
                        algorithm="afctnlr", seed=1)),
    "n5_budget_binds": ((4, 3, 5, 3, 4), "normal", 0.5, 8,
                        dict(max_iters=4, eps=0.0, max_rank=2, initial_rank=2, rank_policy="fixed",
                             algorithm="afctnlr", seed=2, cache_budget=9000)),
    "n4_zero_budget": ((5, 4, 3, 4), "normal", 0.5, 9,
                       dict(max_iters=4, eps=0.0, max_rank=2, initial_rank=2, rank_policy="fixed",
                            algorithm="afctnlr", seed=2, cache_budget=0)),
    "n2_afctnlr": ((9, 7), "normal", 0.5, 11,
                   dict(max_iters=10, eps=0.0, max_rank=3, initial_rank=3, rank_policy="fixed",
                        algorithm="afctnlr", seed=6)),
    "n3_fctnlr": ((8, 7, 5), "normal", 0.4, 16,
                  dict(max_iters=10, eps=0.0, max_rank=2, initial_rank=2, rank_policy="fixed",
                       algorithm="fctnlr", seed=3)),
    "n4_nonuniform_rank": ((5, 6, 4, 3), "normal", 0.5, 12,
                           dict(max_iters=8, eps=0.0, max_rank=[1, 2, 3, 2, 1, 2],
                                initial_rank=[1, 2, 3, 2, 1, 2], rank_policy="fixed",
                                algorithm="afctnlr", seed=7, lam=(0.35, 0.2, 0.5, 0.1),
                                delta=(0.5, 0.3, 0.6, 0.4))),
    "n3_extrapolation": ((6, 5, 4), "normal", 0.5, 23,
                         dict(max_iters=12, eps=0.0, max_rank=2, initial_rank=2, rank_policy="fixed",
                              algorithm="afctnlr", seed=5, extrapolation=(0.5, 0.5))),
    "n4_threshold_growth": ((10, 10, 3, 6), "normal", 0.3, 0,
                            dict(max_iters=40, eps=1e-4, rank_tau=7.5e-3, max_rank=2, rank_policy="threshold",
                                 algorithm="afctnlr", seed=0)),
    "n4_growth_late": ((6, 5, 4, 3), "rank1", 0.6, 3,
                       dict(max_iters=50, eps=1e-5, rank_tau=1e-3, lam=0.05, max_rank=2,
                            rank_policy="threshold", algorithm="afctnlr", seed=0)),
    "n3_converges": ((6, 5, 4), "rank1", 1.0, 14,
                     dict(max_iters=200, eps=1e-6, lam=0.0, max_rank=1, rank_policy="fixed",
                          algorithm="afctnlr", seed=1)),
    "c1_scaled": ((32, 32, 3), "smooth", 0.2, 0,
                  dict(max_iters=20, eps=0.0, max_rank=4, initial_rank=4, rank_policy="fixed",
                       algorithm="afctnlr", shuffle=True, seed=0)),
    "c3_scaled": ((12, 10, 3, 8), "smooth", 0.1, 0,
                  dict(max_iters=8, eps=0.0, max_rank=3, initial_rank=3, rank_policy="fixed",
                       algorithm="afctnlr", shuffle=True, seed=0)),
}


def make_values(dims, kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "normal":
        return rng.standard_normal(dims)
    if kind == "rank1":
        vecs = [rng.standard_normal(d) for d in dims]
        out = vecs[0]
        for v in vecs[1:]:
            out = np.multiply.outer(out, v)
        return out
    if kind == "smooth":
        grids = np.meshgrid(*[np.linspace(0, 1, d) for d in dims], indexing="ij")
        out = np.zeros(dims)
        for _ in range(4):
            w = rng.uniform(0.5, 3.0, size=len(dims))
            out += rng.uniform(0.2, 1.0) * np.sin(sum(2 * np.pi * wi * g for wi, g in zip(w, grids)) + rng.uniform(0, 6))
        return (out - out.min()) / (out.max() - out.min())
    raise ValueError(kind)


def pack_result(prefix, res, store):
    store[prefix + "x"] = np.asfortranarray(res.x)
    for k in range(res.factors.n):
        store[f"{prefix}factor{k}"] = np.asfortranarray(res.factors.factor(k))
    store[prefix + "versions"] = np.asarray(res.factors.versions)


def run_cases():
    for name, (dims, kind, sr, dseed, kw) in RUN_CASES.items():
        values = make_values(dims, kind, dseed)
        mask = sample_mask(dims, sr, dseed)
        obs = Observation.from_dense(values, mask)
        cfg = SolverConfig(**kw)
        res = run(obs, cfg)
        store = {"values": np.asfortranarray(values), "mask": np.asfortranarray(mask)}
        pack_result("", res, store)
        for f in TRACE_FIELDS:
            store["trace_" + f] = np.asarray([getattr(r, f) for r in res.trace])
        store["trace_rank"] = np.asarray([list(r.rank) for r in res.trace])
        store["initial_objective"] = np.asarray(res.initial_objective)
        store["converged"] = np.asarray(res.converged)
        kw1 = dict(kw)
        kw1["max_iters"] = 1
        res1 = run(obs, SolverConfig(**kw1))
        pack_result("it1_", res1, store)
        store["config_json"] = np.asarray(json.dumps(kw))
        np.savez_compressed(os.path.join(HERE, f"run_{name}.npz"), **store)
        print(name, len(res.trace), res.trace[-1].objective, res.converged)


def solve_cases():
    rng = np.random.default_rng(2024)
    store = {}
    shapes = [(1, 1, 1), (1, 3, 5), (4, 1, 6), (2, 2, 3), (7, 3, 11), (16, 9, 40),
              (31, 16, 64), (50, 25, 80), (3, 125, 400), (64, 8, 200)]
    for i, (q, s, p) in enumerate(shapes):
        x = rng.standard_normal((q, p))
        m = rng.standard_normal((s, p))
        a = rng.standard_normal((q, s))
        lam = float(rng.uniform(0.05, 1.0))
        rho = float(rng.uniform(0.05, 0.5))
        delta = float(rng.choice([0.3, 0.5, 0.6]))
        lap = CirculantLaplacian(q, delta)
        out = solve_factor(FactorSubproblem(x_k=x, m=m, a_prev=a, lap=lap, lam=lam, rho=rho))
        store[f"s{i}_x"] = x
        store[f"s{i}_m"] = m
        store[f"s{i}_a"] = a
        store[f"s{i}_par"] = np.asarray([lam, rho, delta])
        store[f"s{i}_out"] = out
    store["count"] = np.asarray(len(shapes))
    # as-printed orientation that must raise NumericalFailure (test_sylvester.py:185-201 style)
    x = rng.standard_normal((4, 6))
    try:
        solve_factor(FactorSubproblem(x_k=x, m=np.zeros((2, 6)), a_prev=rng.standard_normal((4, 2)),
                                      lap=CirculantLaplacian(4, 0.5, "as-printed"), lam=1.0, rho=0.1))
        store["asprinted_raises"] = np.asarray(False)
    except NumericalFailure:
        store["asprinted_raises"] = np.asarray(True)
    np.savez_compressed(os.path.join(HERE, "solve_cases.npz"), **store)


def flop_cases():
    """First-sweep counters of the reference's own benchmark shapes."""
    rows = []
    for (n, i, r, iters) in [(4, 20, 3, 1), (3, 16, 4, 2), (5, 6, 2, 2), (4, 40, 4, 1)]:
        dims = (i,) * n
        truth = np.random.default_rng(0).standard_normal(dims)
        obs = Observation.from_dense(truth, sample_mask(dims, 0.3, 0))
        for alg in ("fctnlr", "afctnlr"):
            res = run(obs, SolverConfig(eps=0.0, max_iters=iters, max_rank=r, initial_rank=r,
                                        rank_policy="fixed", algorithm=alg, seed=0))
            for rec in res.trace:
                rows.append([n, i, r, int(alg == "afctnlr"), rec.iteration, rec.flops,
                             rec.mk_flops, rec.compose_flops, rec.cache_hits])
    np.savez_compressed(os.path.join(HERE, "flop_cases.npz"), rows=np.asarray(rows, dtype=np.int64))
    print("flop rows", len(rows))


if __name__ == "__main__":
    solve_cases()
    run_cases()
    flop_cases()
