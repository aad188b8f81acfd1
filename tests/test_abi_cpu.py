"""CPU-side checks of the C ABI library: it loads without a GPU, exports
every symbol include/fctn_b200.h declares, and its shape-only planner
reproduces the reference FLOP meter and cache-hit integers."""
import os
import re

import numpy as np
import pytest

from paper_2510_22506_b200 import _native
from paper_2510_22506_b200.network import FctnFactors, FctnRank
from tests.golden_util import load_flop_rows, load_run, run_case_names

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "fctn_b200.h")


def test_header_symbols_exported():
    L = _native.lib()
    decl = re.findall(r"^\s*(?:int|void|const char\*)\s+(fctn_\w+)\s*\(", open(HEADER).read(), re.M)
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(_native.EXPORTS)
    assert b"sm_100a" in L.fctn_version()


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        _native.Context(0, _native.F64, (4, 3, 2), (1, 1, 1), (0.35,) * 3, (0.5,) * 3, 0, 0.1, 1, 1 << 30)


def test_plan_reproduces_reference_flop_integers():
    for row in load_flop_rows():
        n, i, r, acc, it, flops, mk, comp, hits = (int(v) for v in row)
        orders = np.tile(np.arange(n, dtype=np.int32), (it, 1))  # shuffle only after the first sweep
        if it > 1:
            continue
        ct = _native.plan_sweeps((i,) * n, (r,) * (n * (n - 1) // 2), int(acc), 1 << 30, orders)
        assert (ct[0, 0], ct[0, 1], ct[0, 2], ct[0, 3]) == (flops, mk, comp, hits)


def _orders_of(case):
    """Visiting orders the reference used: identity, then one
    rng.permutation(n) per completed sweep after the factor draws."""
    cfg = case["config"]
    n = case["values"].ndim
    rng = np.random.default_rng(cfg.get("seed", 0))
    FctnFactors.random(case["values"].shape, FctnRank.from_spec(n, cfg.get("initial_rank") or 1), rng)
    orders = [tuple(range(n))]
    for _ in range(len(case["trace_objective"]) - 1):
        if cfg.get("algorithm", "fctnlr") == "afctnlr" and cfg.get("shuffle", True):
            orders.append(tuple(int(v) for v in rng.permutation(n)))
        else:
            orders.append(orders[-1])
    return np.asarray(orders, dtype=np.int32)


@pytest.mark.parametrize("name", [n for n in run_case_names() if "growth" not in n])
def test_plan_reproduces_golden_traces(name):
    case = load_run(name)
    cfg = case["config"]
    n = case["values"].ndim
    rank = FctnRank.from_spec(n, cfg.get("initial_rank") or 1)
    alg = 1 if cfg.get("algorithm") == "afctnlr" else 0
    ct = _native.plan_sweeps(case["values"].shape, rank.entries, alg, cfg.get("cache_budget", 1 << 30),
                             _orders_of(case))
    assert list(ct[:, 0]) == list(case["trace_flops"])
    assert list(ct[:, 1]) == list(case["trace_mk_flops"])
    assert list(ct[:, 2]) == list(case["trace_compose_flops"])
    assert list(ct[:, 3]) == list(case["trace_cache_hits"])


def test_plan_c5_budget_binds():
    """at c5 the 1 GiB budget binds; mk FLOPs 166.9 G with 4 hits
    in identity order (165.46 G unbounded)."""
    dims, tri = (48,) * 5, (3,) * 10
    o = np.tile(np.arange(5, dtype=np.int32), (2, 1))
    ct = _native.plan_sweeps(dims, tri, 1, 1 << 30, o)
    assert ct[1, 1] == 166906801152 and ct[1, 3] == 4
    ct = _native.plan_sweeps(dims, tri, 1, 1 << 62, o)
    assert ct[1, 1] == 165455612928
