"""Loader for the committed golden fixtures (made by tests/golden/make_golden.py
from the real reference)."""
import glob
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def run_case_names():
    return sorted(os.path.basename(p)[4:-4] for p in glob.glob(os.path.join(GOLDEN, "run_*.npz")))


def load_run(name):
    d = dict(np.load(os.path.join(GOLDEN, f"run_{name}.npz")))
    d["config"] = json.loads(str(d["config_json"]))
    n = d["values"].ndim
    d["factors"] = [d[f"factor{k}"] for k in range(n)]
    d["it1_factors"] = [d[f"it1_factor{k}"] for k in range(n)]
    return d


def load_solve_cases():
    d = np.load(os.path.join(GOLDEN, "solve_cases.npz"))
    out = []
    for i in range(int(d["count"])):
        lam, rho, delta = d[f"s{i}_par"]
        out.append(dict(x=d[f"s{i}_x"], m=d[f"s{i}_m"], a=d[f"s{i}_a"], lam=float(lam),
                        rho=float(rho), delta=float(delta), out=d[f"s{i}_out"]))
    return out, bool(d["asprinted_raises"])


def load_flop_rows():
    return np.load(os.path.join(GOLDEN, "flop_cases.npz"))["rows"]


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = float(np.linalg.norm(b.ravel()))
    return float(np.linalg.norm((a - b).ravel())) / (den if den > 0 else 1.0)
