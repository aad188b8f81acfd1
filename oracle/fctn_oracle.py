"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference `fctnlr` 0.1.0 PAM solver
(`/root/reference/pkg/src/fctnlr`), written from its behaviour, used by
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg as the
checker.  The product (`paper_2510_22506_b200`) never imports this module.

Parity is PINNED: `tests/golden/make_golden.py` runs the real reference in the
authoring container and stores its outputs under `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this restatement against them.

Conventions (reference `tensor.py:1-12`): 0-based modes, first-index-fastest
linearisation, FLOPs = 2 * rows * shared * cols per contraction.

Labels: an int per mode.  Physical mode of factor j is label ``j``; the bond
between factors a < b is ``n + tri(a, b)`` with the upper-triangle row-major
index of `network.py:79-85`.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# rank table and factors  (network.py:41-223)
# ----------------------------------------------------------------------------


def tri_index(n: int, a: int, b: int) -> int:
    """Upper-triangle row-major slot of bond (a, b) (`network.py:79-85`)."""
    if a > b:
        a, b = b, a
    return a * (n - 1) - a * (a - 1) // 2 + (b - a - 1)


def rank_tri(n: int, spec) -> tuple:
    """Int broadcast or explicit upper triangle (`network.py:68-77`)."""
    if np.isscalar(spec):
        tri = (int(spec),) * (n * (n - 1) // 2)
    else:
        tri = tuple(int(v) for v in spec)
    if len(tri) != n * (n - 1) // 2 or any(v < 1 for v in tri):
        raise ValueError("bad rank table")
    return tri


def bond(tri, n, a, b) -> int:
    return tri[tri_index(n, a, b)]


def slot_shape(k: int, dims, tri) -> tuple:
    """Factor k: slot j holds bond (j,k), slot k the physical extent (`network.py:98-105`)."""
    n = len(dims)
    return tuple(dims[k] if j == k else bond(tri, n, j, k) for j in range(n))


def bond_label(n: int, a: int, b: int) -> int:
    return n + tri_index(n, a, b)


def slot_labels(k: int, n: int) -> list:
    return [k if j == k else bond_label(n, j, k) for j in range(n)]


def random_factors(dims, tri, rng) -> list:
    """Standard-normal init in factor order 0..n-1 (`network.py:163-169`)."""
    return [np.asfortranarray(rng.standard_normal(slot_shape(k, dims, tri))) for k in range(len(dims))]


def unfold(t: np.ndarray, k: int) -> np.ndarray:
    """Mode-k unfolding: rows mode k, columns the others ascending, first fastest (`tensor.py:130-139`)."""
    rest = [m for m in range(t.ndim) if m != k]
    return np.transpose(t, [k] + rest).reshape((t.shape[k], -1), order="F")


def fold(mat: np.ndarray, k: int, shape) -> np.ndarray:
    rest = [m for m in range(len(shape)) if m != k]
    t = mat.reshape([shape[k]] + [shape[m] for m in rest], order="F")
    return np.asfortranarray(np.transpose(t, np.argsort([k] + rest)))


# ----------------------------------------------------------------------------
# FLOP meter  (tensor.py:32-72)
# ----------------------------------------------------------------------------


class Meter:
    def __init__(self):
        self.by = {"mk": 0, "compose": 0, "gram": 0, "proj": 0}

    @property
    def total(self) -> int:
        return sum(self.by.values())

    def snap(self) -> dict:
        d = dict(self.by)
        d["total"] = self.total
        return d


# ----------------------------------------------------------------------------
# labeled contraction  (network.py:249-258 over tensor.py:156-200)
# ----------------------------------------------------------------------------


def contract_labeled(a, la, b, lb, meter: Meter, tag: str):
    shared = [x for x in la if x in lb]
    if not shared:
        raise ValueError("operands share no bond")
    ia = [la.index(x) for x in shared]
    ib = [lb.index(x) for x in shared]
    out = np.tensordot(a, b, axes=(ia, ib))
    rows = math.prod(a.shape[i] for i in range(a.ndim) if i not in ia)
    cols = math.prod(b.shape[i] for i in range(b.ndim) if i not in ib)
    k = math.prod(a.shape[i] for i in ia)
    meter.by[tag] += 2 * rows * k * cols
    lout = [x for x in la if x not in shared] + [x for x in lb if x not in shared]
    return out, lout


def permute_to(arr, labels, target):
    return np.transpose(arr, [labels.index(x) for x in target])


# ----------------------------------------------------------------------------
# reuse cache + prefix/suffix chains  (network.py:377-498)
# ----------------------------------------------------------------------------


class Cache:
    """Byte-budgeted subset store with version stamps and lazy eviction
    (`network.py:377-417`).  Bytes are counted as float64 `nbytes`."""

    def __init__(self, budget: int):
        self.budget = int(budget)
        self.entries = {}
        self.bytes = 0
        self.hits = 0
        self.misses = 0

    def get(self, subset, stamps):
        e = self.entries.get(subset)
        if e is not None and e[0] == stamps:
            self.hits += 1
            return e[1], e[2]
        if e is not None:
            self.bytes -= 8 * e[1].size
            del self.entries[subset]
        self.misses += 1
        return None

    def put(self, subset, stamps, arr, labels):
        old = self.entries.pop(subset, None)
        if old is not None:
            self.bytes -= 8 * old[1].size
        if self.bytes + 8 * arr.size > self.budget:
            return
        self.entries[subset] = (stamps, arr, labels)
        self.bytes += 8 * arr.size


def _key(members, versions):
    s = tuple(sorted(members))
    return s, tuple(versions[m] for m in s)


def chain(factors, versions, seq, cache, from_right: bool, meter: Meter):
    """Fold the factors of ``seq`` (`network.py:426-475`)."""
    n = len(factors)
    m = len(seq)
    if m == 0:
        return None, None
    if m == 1:
        return factors[seq[0]], slot_labels(seq[0], n)
    steps = [tuple(seq[i:]) for i in range(m - 2, -1, -1)] if from_right else [tuple(seq[: i + 2]) for i in range(m - 1)]
    arr = labels = None
    start = 0
    if cache is not None:
        for idx in range(len(steps) - 1, -1, -1):
            hit = cache.get(*_key(steps[idx], versions))
            if hit is not None:
                arr, labels = hit
                start = idx + 1
                break
    if arr is None:
        j0 = seq[-1] if from_right else seq[0]
        arr, labels = factors[j0], slot_labels(j0, n)
        start = 0
    for idx in range(start, len(steps)):
        if from_right:
            j = steps[idx][0]
            arr, labels = contract_labeled(factors[j], slot_labels(j, n), arr, labels, meter, "mk")
        else:
            j = steps[idx][-1]
            arr, labels = contract_labeled(arr, labels, factors[j], slot_labels(j, n), meter, "mk")
        if cache is not None and len(steps[idx]) < n - 1:
            cache.put(*_key(steps[idx], versions), arr, labels)
    return arr, labels


def partial_cached(factors, versions, k, order, cache, meter):
    """Leave-one-out network around k from prefix/suffix chains (`network.py:478-498`)."""
    pos = order.index(k)
    left, ll = chain(factors, versions, order[:pos], cache, False, meter)
    right, rl = chain(factors, versions, order[pos + 1:], cache, True, meter)
    if left is None:
        return right, rl
    if right is None:
        return left, ll
    return contract_labeled(left, ll, right, rl, meter, "mk")


def partial_plain(factors, k, meter, tag="mk"):
    """Plain ascending chain without reuse (`network.py:281-293`)."""
    n = len(factors)
    rest = [j for j in range(n) if j != k]
    arr, labels = factors[rest[0]], slot_labels(rest[0], n)
    for j in rest[1:]:
        arr, labels = contract_labeled(arr, labels, factors[j], slot_labels(j, n), meter, tag)
    return arr, labels


def m_matrix(arr, labels, k, n) -> np.ndarray:
    """M_k as s x p: rows the bonds to k (ascending partner, first fastest),
    columns the other physical modes ascending (first fastest).  Column order
    is free (`network.py:360-371`, invariance `test_sylvester.py:121-135`)."""
    rest = [j for j in range(n) if j != k]
    target = [bond_label(n, j, k) for j in rest] + rest
    t = permute_to(arr, labels, target)
    s = math.prod(t.shape[: n - 1])
    return t.reshape((s, -1), order="F")


def compose_full(factors, meter, tag="compose") -> np.ndarray:
    """Whole-network chain in index order (`network.py:271-278`)."""
    n = len(factors)
    arr, labels = factors[0], slot_labels(0, n)
    for k in range(1, n):
        arr, labels = contract_labeled(arr, labels, factors[k], slot_labels(k, n), meter, tag)
    return np.asfortranarray(permute_to(arr, labels, list(range(n))))


def compose_from_m(a_k_unf: np.ndarray, m: np.ndarray, k: int, dims, meter) -> np.ndarray:
    """C = A_(k) M_k folded back to mode k (`network.py:313-332`)."""
    i_k, s = a_k_unf.shape
    meter.by["compose"] += 2 * m.shape[1] * s * i_k
    return fold(a_k_unf @ m, k, dims)


# ----------------------------------------------------------------------------
# circulant Laplacian  (laplacian.py:25-81)
# ----------------------------------------------------------------------------

_SIGN = {"positive-definite": -1.0, "as-printed": 1.0}


def lap_spectrum(n: int, delta: float, sign: str) -> np.ndarray:
    if n < 1 or delta <= 0.0 or sign not in _SIGN:
        raise ValueError("bad Laplacian parameters")
    j = np.arange(n)
    return _SIGN[sign] * (-2.0 - delta + 2.0 * np.cos(2.0 * np.pi * j / n))


def lap_apply(a: np.ndarray, delta: float, sign: str) -> np.ndarray:
    """3-band periodic stencil along axis 0; the printed first column degenerates
    for n = 1, 2 exactly as the reference builds it (`laplacian.py:37-45,59-66`)."""
    return _SIGN[sign] * ((-2.0 - delta) * a + np.roll(a, 1, axis=0) + np.roll(a, -1, axis=0))


def trace_penalty(a_unf: np.ndarray, delta: float, sign: str) -> float:
    return float(np.sum(a_unf * lap_apply(a_unf, delta, sign)))


# ----------------------------------------------------------------------------
# factor subproblem  (sylvester.py:51-116)
# ----------------------------------------------------------------------------

T_FLOOR = 1e-10


class NumericalFailure(RuntimeError):
    pass


def solve_factor(x_k, m, a_prev, spectrum, lam, rho, meter: Meter | None = None):
    """Exact minimiser of 1/2||A M - X_k||^2 + lam/2 tr(A^T L A) + rho/2||A - A_prev||^2
    by Gram eigendecomposition + unitary DFT along rows (`sylvester.py:98-116`)."""
    q, p = x_k.shape
    s = m.shape[0]
    g = m @ m.T
    g = 0.5 * (g + g.T)
    phi, c = np.linalg.eigh(g)
    phi = np.maximum(phi, 0.0)
    y = x_k @ m.T + rho * a_prev
    if meter is not None:
        meter.by["gram"] += 2 * s * s * p
        meter.by["proj"] += 2 * q * p * s
    t = lam * spectrum[:, None] + phi[None, :] + rho
    if float(t.min()) <= T_FLOOR:
        raise NumericalFailure("shifted spectrum is not strictly positive; "
                               "the as-printed operator orientation cannot be inverted here")
    w = np.fft.fft(y @ c, axis=0, norm="ortho")
    a = np.fft.ifft(w / t, axis=0, norm="ortho") @ c.T
    return np.ascontiguousarray(a.real)


def solve_factor_kron(x_k, m, a_prev, delta, sign, lam, rho):
    """Dense Kronecker oracle for small sizes (`sylvester.py:119-133`)."""
    q, s = a_prev.shape
    eye_q = np.eye(q)
    lmat = lap_apply(eye_q, delta, sign)
    big = np.kron(m @ m.T, eye_q) + lam * np.kron(np.eye(s), lmat) + rho * np.eye(q * s)
    rhs = (x_k @ m.T + rho * a_prev).reshape(q * s, order="F")
    return np.linalg.solve(big, rhs).reshape((q, s), order="F")


# ----------------------------------------------------------------------------
# the PAM loop  (solver.py:209-419)
# ----------------------------------------------------------------------------


@dataclass
class Record:
    iteration: int
    objective: float
    rel_change: float
    wall_ms: float
    flops: int
    cache_hits: int
    rank: tuple
    mk_flops: int
    compose_flops: int
    step_sq: float
    x_norm: float
    factor_norm: float
    rank_grown: bool = False


@dataclass
class Result:
    x: np.ndarray
    factors: list
    versions: list
    trace: list = field(default_factory=list)
    converged: bool = False
    initial_objective: float = math.nan


def _sq(a) -> float:
    f = np.ravel(a, order="K")
    return float(np.dot(f, f))


def _per_mode(v, n):
    if np.isscalar(v):
        return (float(v),) * n
    t = tuple(float(x) for x in v)
    if len(t) != n:
        raise ValueError("per-mode parameter has wrong length")
    return t


def objective(x, factors, lams, deltas, sign, composed=None, meter=None) -> float:
    """1/2||X - compose||^2 + sum_k lam_k/2 tr(A_(k)^T L_k A_(k)) (`solver.py:209-224`)."""
    if composed is None:
        composed = compose_full(factors, meter or Meter())
    val = 0.5 * _sq(x - composed)
    for k, a in enumerate(factors):
        val += 0.5 * lams[k] * trace_penalty(unfold(a, k), deltas[k], sign)
    return val


def _grow(factors, versions, tri, cap, rng, x, lams, deltas, sign, scale, pre_obj, meter):
    """Rank growth with the continuity retry (`solver.py:246-271,402-419`)."""
    n = len(factors)
    dims = tuple(f.shape[k] for k, f in enumerate(factors))
    new_tri = tuple(min(e + 1, c) for e, c in zip(tri, cap))
    grown, noises = [], []
    for k in range(n):
        g = np.zeros(slot_shape(k, dims, new_tri), order="F")
        g[tuple(slice(0, s) for s in factors[k].shape)] = factors[k]
        grown.append(g)
    for k in range(n):
        z = rng.standard_normal(grown[k].shape)
        z[tuple(slice(0, s) for s in factors[k].shape)] = 0.0
        noises.append(z)
    new_versions = [v + 1 for v in versions]
    for s in (scale, scale / 10.0, 0.0):
        cand = [np.asfortranarray(grown[k] + s * math.sqrt(float(np.mean(factors[k] ** 2))) * noises[k]) for k in range(n)]
        if s == 0.0:
            return cand, new_versions, new_tri
        post = objective(x, cand, lams, deltas, sign, meter=meter)  # counted in the sweep's FLOPs, as the global meter does
        if math.isfinite(post) and post <= 1.05 * pre_obj + 1e-12:
            return cand, new_versions, new_tri
    return cand, new_versions, new_tri


def run(values, mask, *, lam=0.35, delta=0.5, rho=0.1, eps=1e-4, max_iters=500,
        max_rank=2, initial_rank=None, rank_policy="threshold", rank_tau=None,
        grow_noise=1e-2, algorithm="fctnlr", laplacian_sign="positive-definite",
        extrapolation=None, shuffle=True, seed=0, cache_budget=1 << 30,
        snapshots=(), on_iter=None) -> Result:
    """Restates `solver.py:277-399`.  ``snapshots``: iteration numbers at
    which (x, factors) copies are kept in ``result.snaps``."""
    mask = np.asfortranarray(np.asarray(mask, dtype=bool))
    values = np.asfortranarray(np.where(mask, np.asarray(values, dtype=np.float64), 0.0))
    n = values.ndim
    dims = values.shape
    lams = _per_mode(lam, n)
    deltas = _per_mode(delta, n)
    if any(v < 0 for v in lams):
        raise ValueError("lam must be >= 0")
    spectra = [lap_spectrum(dims[k], deltas[k], laplacian_sign) for k in range(n)]
    cap = rank_tri(n, max_rank)
    tri = rank_tri(n, initial_rank) if initial_rank is not None else (1,) * (n * (n - 1) // 2)
    if any(a > b for a, b in zip(tri, cap)):
        raise ValueError("initial rank exceeds max_rank")
    tau = 10.0 * eps if rank_tau is None else float(rank_tau)

    rng = np.random.default_rng(seed)
    factors = random_factors(dims, tri, rng)
    versions = [0] * n
    x = values.copy(order="F")
    obs_idx = np.flatnonzero(mask.ravel(order="F"))
    obs_val = values.ravel(order="F")[obs_idx]
    order = tuple(range(n))
    accel = algorithm == "afctnlr"
    cache = Cache(cache_budget) if accel else None
    meter = Meter()

    init_obj = objective(x, factors, lams, deltas, laplacian_sign, meter=Meter())
    res = Result(x=x, factors=factors, versions=versions, initial_objective=init_obj)
    res.snaps = {}
    if not math.isfinite(init_obj):
        raise NumericalFailure("initial objective is not finite")

    for it in range(1, max_iters + 1):
        t0 = time.perf_counter()
        before = meter.snap()
        hits0 = cache.hits if cache is not None else 0
        step_sq = 0.0
        m_last = None
        for k in order:
            if accel:
                arr, labels = partial_cached(factors, versions, k, order, cache, meter)
            else:
                arr, labels = partial_plain(factors, k, meter)
            m = m_matrix(arr, labels, k, n)
            a_prev = unfold(factors[k], k)
            a_new = solve_factor(unfold(x, k), m, a_prev, spectra[k], lams[k], rho, meter)
            if extrapolation is not None:
                al, be = extrapolation
                a_new = a_new + al * (a_new - be * a_prev)
            step_sq += _sq(a_new - a_prev)
            factors[k] = fold(a_new, k, factors[k].shape)
            versions[k] += 1
            if accel and k == order[-1]:
                m_last = m
        if accel:
            k_last = order[-1]
            composed = compose_from_m(unfold(factors[k_last], k_last), m_last, k_last, dims, meter)
        else:
            composed = compose_full(factors, meter)
        x_new = (x * rho + composed) / (1.0 + rho)
        x_new = np.asfortranarray(x_new)
        x_new.ravel(order="K")[obs_idx] = obs_val
        diff = math.sqrt(_sq(x_new - x))
        base = math.sqrt(_sq(x))
        rel = 0.0 if diff == 0.0 else (math.inf if base == 0.0 else diff / base)
        step_sq += diff * diff
        obj = objective(x_new, factors, lams, deltas, laplacian_sign, composed=composed)
        if not math.isfinite(obj):
            raise NumericalFailure(f"objective diverged at iteration {it}")
        x = x_new
        rank_during = tuple(tri)
        grown = False
        if rank_policy == "threshold" and any(e < c for e, c in zip(tri, cap)) and rel < tau:
            factors, versions, tri = _grow(factors, versions, tri, cap, rng, x, lams, deltas,
                                           laplacian_sign, grow_noise, obj, meter)
            if cache is not None:
                cache = Cache(cache_budget)
            grown = True
        after = meter.snap()
        rec = Record(
            iteration=it, objective=obj, rel_change=rel,
            wall_ms=(time.perf_counter() - t0) * 1e3,
            flops=after["total"] - before["total"],
            cache_hits=(cache.hits if cache is not None else 0) - hits0,  # a grown sweep reports -hits0, as the reference does (solver.py:366-367,377)
            rank=rank_during,
            mk_flops=after["mk"] - before["mk"],
            compose_flops=after["compose"] - before["compose"],
            step_sq=step_sq, x_norm=math.sqrt(_sq(x)),
            factor_norm=max(math.sqrt(_sq(f)) for f in factors), rank_grown=grown)
        res.trace.append(rec)
        if it in snapshots:
            res.snaps[it] = (x.copy(order="F"), [f.copy(order="F") for f in factors])
        if on_iter is not None:
            on_iter(rec)
        if not grown and rel <= eps:
            res.converged = True
            break
        if accel and shuffle:
            order = tuple(int(v) for v in rng.permutation(n))
    res.x = x
    res.factors = factors
    res.versions = versions
    return res


def psnr(x, ref, peak=1.0) -> float:
    """Slice-averaged PSNR over the trailing modes (`metrics.py:33-44`)."""
    xs = np.asarray(x, np.float64).reshape((x.shape[0], x.shape[1], -1), order="F")
    rs = np.asarray(ref, np.float64).reshape((ref.shape[0], ref.shape[1], -1), order="F")
    vals = []
    for t in range(xs.shape[2]):
        mse = float(np.mean((xs[:, :, t] - rs[:, :, t]) ** 2))
        vals.append(100.0 if mse == 0.0 else 10.0 * math.log10(peak * peak / mse))
    return float(np.mean(vals))


def ssim(x, ref, peak=1.0) -> float:
    """Slice-averaged single-window structural index (`metrics.py:47-66`):
    plain means, population variances and covariance per slice, stabilisers
    c1 = (0.01 peak)^2, c2 = (0.03 peak)^2."""
    c1, c2 = (0.01 * peak) ** 2, (0.03 * peak) ** 2
    xs = np.asarray(x, np.float64).reshape((x.shape[0], x.shape[1], -1), order="F")
    rs = np.asarray(ref, np.float64).reshape((ref.shape[0], ref.shape[1], -1), order="F")
    vals = []
    for t in range(xs.shape[2]):
        a, b = xs[:, :, t], rs[:, :, t]
        ma, mb = float(a.mean()), float(b.mean())
        va, vb = float(a.var()), float(b.var())
        cov = float(((a - ma) * (b - mb)).mean())
        vals.append((2.0 * ma * mb + c1) * (2.0 * cov + c2) / ((ma * ma + mb * mb + c1) * (va + vb + c2)))
    return float(np.mean(vals))


def rel_err(x, ref, mask=None) -> float:
    """Relative Frobenius error, over the mask complement when a mask is given;
    nan for an empty complement, ValueError for a zero denominator
    (`metrics.py:69-92`)."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    if mask is None:
        num, den = float(np.linalg.norm((x - ref).ravel())), float(np.linalg.norm(ref.ravel()))
    else:
        sel = ~np.asarray(mask, dtype=bool)
        if not sel.any():
            return math.nan
        num, den = float(np.linalg.norm(x[sel] - ref[sel])), float(np.linalg.norm(ref[sel]))
    if den == 0.0:
        raise ValueError("zero-norm denominator in relative error")
    return num / den
