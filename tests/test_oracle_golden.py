"""Pin the CPU oracle (oracle/fctn_oracle.py) against the reference's own
outputs stored in tests/golden (made by running fctnlr 0.1.0 itself)."""
import math

import numpy as np
import pytest

from oracle import fctn_oracle as O
from tests.golden_util import load_flop_rows, load_run, load_solve_cases, rel, run_case_names

FP64_TOL = 1e-9


def _run_oracle(case, **over):
    cfg = dict(case["config"])
    cfg.update(over)
    if cfg.get("extrapolation") is not None:
        cfg["extrapolation"] = tuple(cfg["extrapolation"])
    return O.run(case["values"], case["mask"], **cfg)


@pytest.mark.parametrize("name", run_case_names())
def test_oracle_matches_reference_run(name):
    case = load_run(name)
    res = _run_oracle(case)
    assert rel(res.x, case["x"]) <= FP64_TOL
    for k, f in enumerate(case["factors"]):
        assert res.factors[k].shape == f.shape
        assert rel(res.factors[k], f) <= FP64_TOL
    assert list(res.versions) == list(case["versions"])
    assert res.converged == bool(case["converged"])
    assert res.initial_objective == pytest.approx(float(case["initial_objective"]), rel=1e-12)
    tr = res.trace
    assert len(tr) == len(case["trace_objective"])
    for i, r in enumerate(tr):
        assert r.objective == pytest.approx(case["trace_objective"][i], rel=FP64_TOL)
        assert r.step_sq == pytest.approx(case["trace_step_sq"][i], rel=1e-7, abs=1e-12)
        assert r.x_norm == pytest.approx(case["trace_x_norm"][i], rel=1e-10)
        assert r.factor_norm == pytest.approx(case["trace_factor_norm"][i], rel=1e-9)
        # exact integers: FLOP counters, cache hits, rank table, growth flag
        assert r.flops == case["trace_flops"][i]
        assert r.mk_flops == case["trace_mk_flops"][i]
        assert r.compose_flops == case["trace_compose_flops"][i]
        assert r.cache_hits == case["trace_cache_hits"][i]
        assert list(r.rank) == list(case["trace_rank"][i])
        assert r.rank_grown == bool(case["trace_rank_grown"][i])
        rc = case["trace_rel_change"][i]
        assert (r.rel_change == rc) if rc == 0 else r.rel_change == pytest.approx(rc, rel=1e-6, abs=1e-13)


@pytest.mark.parametrize("name", ["n3_afctnlr", "n4_afctnlr_shuffle", "n5_afctnlr", "n2_afctnlr"])
def test_oracle_first_iteration(name):
    case = load_run(name)
    res = _run_oracle(case, max_iters=1)
    assert rel(res.x, case["it1_x"]) <= 1e-12
    for k, f in enumerate(case["it1_factors"]):
        assert rel(res.factors[k], f) <= 1e-11


def test_oracle_observed_entries_bit_exact():
    case = load_run("n3_afctnlr")
    res = _run_oracle(case)
    m = case["mask"]
    assert np.array_equal(res.x[m], case["values"][m])


def test_oracle_solve_matches_reference_solve():
    cases, raises = load_solve_cases()
    for c in cases:
        q = c["a"].shape[0]
        spec = O.lap_spectrum(q, c["delta"], "positive-definite")
        got = O.solve_factor(c["x"], c["m"], c["a"], spec, c["lam"], c["rho"])
        assert rel(got, c["out"]) <= 1e-10
        if q * c["a"].shape[1] <= 1500:
            dense = O.solve_factor_kron(c["x"], c["m"], c["a"], c["delta"], "positive-definite", c["lam"], c["rho"])
            assert rel(dense, c["out"]) <= 1e-8
    assert raises
    rng = np.random.default_rng(7)
    with pytest.raises(O.NumericalFailure):
        O.solve_factor(rng.standard_normal((4, 6)), np.zeros((2, 6)), rng.standard_normal((4, 2)),
                       O.lap_spectrum(4, 0.5, "as-printed"), 1.0, 0.1)


def test_oracle_reference_flop_integers():
    """First-sweep counters, incl. the reference's published acceptance integers
    (test_acceptance.py:366-369, test_cli.py:208-211)."""
    rows = load_flop_rows()
    want = {(4, 40, 4, 0): (537395200, 462028800), (4, 40, 4, 1): (530841600, 327680000),
            (4, 20, 3, 0): (16329600, 12722400), (4, 20, 3, 1): (15940800, 8640000)}
    for (n, i, r, acc), (mk, comp) in want.items():
        hit = [row for row in rows if tuple(row[:4]) == (n, i, r, acc) and row[4] == 1]
        assert hit and hit[0][6] == mk and hit[0][7] == comp
    # the oracle's meter reproduces every stored counter without touching data
    for row in rows:
        n, i, r, acc, it, flops, mk, comp, hits = (int(v) for v in row)
        if i ** n > 200000:
            continue
        dims = (i,) * n
        truth = np.random.default_rng(0).standard_normal(dims)
        from paper_2510_22506_b200.workloads import sample_mask
        res = O.run(truth, sample_mask(dims, 0.3, 0), eps=0.0, max_iters=it, max_rank=r, initial_rank=r,
                    rank_policy="fixed", algorithm="afctnlr" if acc else "fctnlr", seed=0)
        rec = res.trace[it - 1]
        assert (rec.flops, rec.mk_flops, rec.compose_flops, rec.cache_hits) == (flops, mk, comp, hits)


def test_oracle_kron_identity_small():
    """Stationarity of the restated solve (sylvester.py:1-17 normal equations)."""
    rng = np.random.default_rng(3)
    q, s, p = 9, 4, 13
    x, m, a = rng.standard_normal((q, p)), rng.standard_normal((s, p)), rng.standard_normal((q, s))
    out = O.solve_factor(x, m, a, O.lap_spectrum(q, 0.5, "positive-definite"), 0.35, 0.1)
    lhs = out @ (m @ m.T) + 0.35 * O.lap_apply(out, 0.5, "positive-definite") + 0.1 * out
    rhs = x @ m.T + 0.1 * a
    assert rel(lhs, rhs) <= 1e-12
    assert math.isfinite(float(lhs.sum()))
