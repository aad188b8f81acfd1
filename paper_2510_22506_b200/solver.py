"""Drop-in `run(obs, cfg)` for the reference solver (`solver.py:277-399`)
whose per-iteration work — the whole PAM sweep — runs on the B200 through
the C ABI (include/fctn_b200.h).

Kept on the host, exactly as the reference orders them: input validation,
the PCG64 stream (factor init `network.py:163-169`, one permutation per
completed sweep `network.py:515-517`, rank-growth noise `solver.py:261-271`),
the stopping rule, and the trace bookkeeping.  Everything tensor-sized lives
on the device for the whole run: X, the mask, the factors, the reuse cache of
partial contractions and the M_k / solve workspaces.  Per sweep only the
reduction scalars cross back.

Extra keyword-only knobs (not in the reference signature): ``dtype`` —
"float64" (default, the reference arithmetic) or "float32" (the FP32
variant: contractions, products and the blend in FP32, the s x s solves in
FP64) — and ``device`` (CUDA ordinal).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .network import FctnFactors, FctnRank, mode_fold, mode_unfold

__all__ = ["IterationRecord", "NumericalFailure", "Observation", "SolverConfig", "SolverResult", "run"]

_ALGORITHMS = ("fctnlr", "afctnlr")
_RANK_POLICIES = ("fixed", "threshold")
_SIGNS = {"positive-definite": _native.SIGN_PD, "as-printed": _native.SIGN_PRINTED}


class NumericalFailure(RuntimeError):
    """Same role as `sylvester.NumericalFailure` (sylvester.py:39-40)."""


@dataclass
class Observation:
    """Observed entries: values where mask is True, zeros elsewhere (`solver.py:62-98`)."""

    values: np.ndarray
    mask: np.ndarray

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float64)
        self.mask = np.asfortranarray(np.asarray(self.mask, dtype=bool))
        if self.values.shape != self.mask.shape:
            raise ValueError("values and mask shapes differ")
        if self.values.ndim < 2:
            raise ValueError("need a tensor of order >= 2")
        if not self.mask.any():
            raise ValueError("mask has no observed entry")
        self.values = np.asfortranarray(np.where(self.mask, self.values, 0.0))

    @classmethod
    def from_dense(cls, dense, mask) -> "Observation":
        return cls(values=np.asarray(dense), mask=mask)

    @property
    def dims(self) -> tuple:
        return self.values.shape

    @property
    def count(self) -> int:
        return int(self.mask.sum())

    @property
    def flat_index(self) -> np.ndarray:
        return np.flatnonzero(self.mask.ravel(order="F"))


@dataclass
class SolverConfig:
    """Field set, defaults and validation of `solver.py:110-151`."""

    lam: object = 0.35
    delta: object = 0.5
    rho: float = 0.1
    eps: float = 1e-4
    max_iters: int = 500
    max_rank: object = 2
    initial_rank: object = None
    rank_policy: str = "threshold"
    rank_tau: float | None = None
    grow_noise: float = 1e-2
    algorithm: str = "fctnlr"
    laplacian_sign: str = "positive-definite"
    extrapolation: tuple | None = None
    shuffle: bool = True
    seed: int = 0
    cache_budget: int = 1 << 30

    def __post_init__(self):
        if self.rho <= 0.0:
            raise ValueError("rho must be > 0")
        if self.eps < 0.0:
            raise ValueError("eps must be >= 0")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.algorithm not in _ALGORITHMS:
            raise ValueError(f"algorithm must be one of {_ALGORITHMS}")
        if self.rank_policy not in _RANK_POLICIES:
            raise ValueError(f"rank_policy must be one of {_RANK_POLICIES}")
        if self.extrapolation is not None:
            alpha, beta = self.extrapolation
            if not 0.0 < alpha < 1.0:
                raise ValueError("extrapolation weight alpha must lie in (0, 1)")
            if not 0.2 < beta < 0.8:
                raise ValueError("old-iterate shrink beta must lie in (0.2, 0.8)")
            self.extrapolation = (float(alpha), float(beta))
        if self.grow_noise < 0.0:
            raise ValueError("grow_noise must be >= 0")

    def tau(self) -> float:
        return 10.0 * self.eps if self.rank_tau is None else float(self.rank_tau)


@dataclass
class IterationRecord:
    """One sweep's bookkeeping (`solver.py:154-179`)."""

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
    x_norm: float = math.nan
    factor_norm: float = math.nan
    rank_grown: bool = False
    device_ms: float = math.nan  # CUDA-event time of the sweep (extra field)


@dataclass
class SolverResult:
    x: np.ndarray
    factors: FctnFactors
    trace: list = field(default_factory=list)
    converged: bool = False
    initial_objective: float = math.nan
    # (iteration, metrics.QualityReport) when run(..., truth=...) is given
    quality: list = field(default_factory=list)
    # iteration -> (x, factors) for run(..., snapshot_iters=...)
    snapshots: dict = field(default_factory=dict)

    @property
    def iterations(self) -> int:
        return len(self.trace)

    @property
    def objective(self) -> float:
        return self.trace[-1].objective if self.trace else self.initial_objective


def _per_mode(value, n: int, name: str) -> tuple:
    if np.isscalar(value):
        return (float(value),) * n
    seq = tuple(float(v) for v in value)
    if len(seq) != n:
        raise ValueError(f"{name} needs 1 or {n} values, got {len(seq)}")
    return seq


def _check_laplacians(dims, deltas, sign):
    # CirculantLaplacian.__init__ validation (laplacian.py:26-35)
    for d, dl in zip(dims, deltas):
        if int(d) < 1:
            raise ValueError("operator size must be >= 1")
        if dl <= 0.0:
            raise ValueError("diagonal shift delta must be > 0")
    if sign not in _SIGNS:
        raise ValueError(f"sign must be one of {sorted(_SIGNS)}, got {sign!r}")


class _Device:
    """The device side of one run: a context plus host version stamps."""

    def __init__(self, obs_values, obs_mask, rank: FctnRank, lams, deltas, cfg, dtype, device, shard=None):
        self.dims = obs_values.shape
        self.n = len(self.dims)
        dt = {"float64": _native.F64, "float32": _native.F32}[dtype]
        self.ctx = _native.Context(device, dt, self.dims, rank.entries, lams, deltas, _SIGNS[cfg.laplacian_sign],
                                   cfg.rho, _native.ALG_ACCEL if cfg.algorithm == "afctnlr" else _native.ALG_PLAIN,
                                   cfg.cache_budget, numeric_exc=NumericalFailure)
        self.slab = (0, self.dims[0])
        if shard is not None and shard.nranks > 1:
            shard.attach(self.ctx)  # before the upload: the context reshapes to its slab
            self.slab = self.ctx.slab
            lo, hi = self.slab
            obs_values = np.asfortranarray(obs_values[lo:hi])
            obs_mask = np.asfortranarray(obs_mask[lo:hi])
        self.ctx.upload_f64(obs_values, obs_mask)

    def load_factors(self, f: FctnFactors, reset_cache: bool):
        if tuple(f.rank.entries) != self.ctx.rank_tri:
            self.ctx.set_rank(f.rank.entries)
        self.ctx.set_factors(f.unfoldings(), f.versions, reset_cache)

    def quality(self, truth: np.ndarray, peak: float):
        from .metrics import QualityReport, from_sums
        lo, hi = self.slab
        t = truth if (lo, hi) == (0, self.dims[0]) else truth[lo:hi]
        p, s, err, _ = from_sums(self.ctx.quality(np.asfortranarray(t), False, peak), masked=False)
        return QualityReport(psnr=p, ssim=s, rel_err=err)

    def fetch_factors(self, rank: FctnRank, versions) -> FctnFactors:
        shapes = [(self.dims[k], rank.bond_product(k)) for k in range(self.n)]  # global extents
        unf = self.ctx.get_factors(shapes)
        f = FctnFactors([mode_fold(u, k, rank.factor_shape(k, self.dims)) for k, u in enumerate(unf)])
        f.versions = list(versions)
        return f


def _grow_with_continuity(dev: _Device, f: FctnFactors, cap: FctnRank, rng, scale: float, pre_objective: float):
    """`solver.py:402-419` with the candidate objectives evaluated on device;
    returns (factors, extra compose FLOPs of those evaluations)."""
    new_rank = f.rank.increment_below(cap)
    grown = f.grow(new_rank)
    noises = []
    for k in range(f.n):  # solver.py:261-271: one draw per factor, old block zeroed
        noise = rng.standard_normal(grown.factor(k).shape)
        noise[tuple(slice(0, s) for s in f.factor(k).shape)] = 0.0
        noises.append(noise)
    extra = 0
    cand = None
    for s in (scale, scale / 10.0, 0.0):
        out = []
        for k in range(f.n):
            rms = float(np.sqrt(np.mean(f.factor(k) ** 2)))
            out.append(grown.factor(k) + s * rms * noises[k])
        cand = FctnFactors(out)
        cand.versions = list(grown.versions)
        if s == 0.0:
            return cand, extra
        dev.load_factors(cand, reset_cache=True)
        post, ct = dev.ctx.objective()
        extra += int(ct[_native.CT_COMPOSE])
        if math.isfinite(post) and post <= 1.05 * pre_objective + 1e-12:
            return cand, extra
    return cand, extra


def run(obs, cfg: SolverConfig, *, dtype: str = "float64", device: int | None = None, shard=None,
        truth=None, peak: float = 1.0, quality_every: int = 0, snapshot_iters=()) -> SolverResult:
    """Same contract as `fctnlr.solver.run` (solver.py:277-399).

    ``truth`` (the full ground-truth tensor): `metrics.quality_report(x,
    truth, peak=peak)` (metrics.py:102-105) of the resident X is computed on
    the device after every ``quality_every``-th sweep (0: after the last
    one only) into ``result.quality`` — no T-sized download per report.

    ``shard`` (a `shard.Shard`) runs this call as one rank of a mode-0 sharded
    sweep: every rank passes the same global observation and config; the
    returned ``x`` is this rank's slab (``result.slab`` = its rows of mode 0),
    factors and trace are global and identical on every rank.

    ``snapshot_iters``: after each listed iteration X and the factors are
    downloaded into ``result.snapshots[it] = (x, factors)`` (parity checks at
    iterations 1, 5, ... from one run)."""
    if not isinstance(obs, Observation):
        obs = Observation(values=obs.values, mask=obs.mask)
    n = obs.values.ndim
    dims = obs.dims
    lams = _per_mode(cfg.lam, n, "lam")
    deltas = _per_mode(cfg.delta, n, "delta")
    if any(v < 0 for v in lams):
        raise ValueError("lam must be >= 0")
    _check_laplacians(dims, deltas, cfg.laplacian_sign)
    cap = FctnRank.from_spec(n, cfg.max_rank)
    rank = FctnRank.from_spec(n, cfg.initial_rank) if cfg.initial_rank is not None else FctnRank.uniform(n, 1)
    if any(a > b for a, b in zip(rank.entries, cap.entries)):
        raise ValueError("initial rank exceeds max_rank")
    if dtype not in ("float64", "float32"):
        raise ValueError("dtype must be 'float64' or 'float32'")
    if device is None:
        device = 0

    if truth is not None:
        truth = np.asarray(truth)
        if truth.shape != dims:
            raise ValueError("tensors must have identical shapes")
        if peak <= 0:
            raise ValueError("peak must be > 0")
        if truth.dtype not in (np.float32, np.float64):
            truth = truth.astype(np.float64)
    rng = np.random.default_rng(cfg.seed)
    f = FctnFactors.random(dims, rank, rng)
    order = tuple(range(n))
    accelerated = cfg.algorithm == "afctnlr"

    dev = _Device(obs.values, obs.mask, rank, lams, deltas, cfg, dtype, device, shard)
    try:
        dev.load_factors(f, reset_cache=True)
        initial_objective, _ = dev.ctx.objective()
        result = SolverResult(x=None, factors=f, initial_objective=initial_objective)
        if not math.isfinite(initial_objective):
            raise NumericalFailure("initial objective is not finite")
        versions = list(f.versions)
        cache_hits_running = 0
        for it in range(1, cfg.max_iters + 1):
            t0 = time.perf_counter()
            hits0 = cache_hits_running
            stats, ct = dev.ctx.sweep(order, cfg.extrapolation)
            versions = [v + 1 for v in versions]  # every factor replaced once (network.py:200)
            cache_hits_running += int(ct[_native.CT_HITS])
            diff = math.sqrt(stats[_native.ST_DIFF_SQ])
            base = math.sqrt(stats[_native.ST_BASE_SQ])
            if diff == 0.0:
                rel = 0.0
            elif base == 0.0:
                rel = math.inf
            else:
                rel = diff / base
            step_sq = float(stats[_native.ST_STEP_FAC]) + diff * diff
            obj = float(stats[_native.ST_OBJECTIVE])
            if not math.isfinite(obj):
                raise NumericalFailure(f"objective diverged at iteration {it}")
            rank_during = tuple(rank.entries)
            flops = int(ct[_native.CT_FLOPS])
            compose_flops = int(ct[_native.CT_COMPOSE])
            factor_norm = float(stats[_native.ST_FNORM_MAX])
            grown = False
            if cfg.rank_policy == "threshold" and rank.any_below(cap) and rel < cfg.tau():
                cur = dev.fetch_factors(rank, versions)
                f, extra = _grow_with_continuity(dev, cur, cap, rng, cfg.grow_noise, obj)
                flops += extra
                compose_flops += extra
                rank = f.rank
                versions = list(f.versions)
                dev.load_factors(f, reset_cache=True)
                cache_hits_running = 0
                factor_norm = max(math.sqrt(float(np.sum(f.factor(k) ** 2))) for k in range(n))
                grown = True
            result.trace.append(IterationRecord(
                iteration=it, objective=obj, rel_change=rel,
                wall_ms=(time.perf_counter() - t0) * 1e3,
                flops=flops, cache_hits=cache_hits_running - hits0, rank=rank_during,
                mk_flops=int(ct[_native.CT_MK]), compose_flops=compose_flops, step_sq=step_sq,
                x_norm=math.sqrt(float(stats[_native.ST_XNEW_SQ])), factor_norm=factor_norm,
                rank_grown=grown, device_ms=float(stats[_native.ST_DEVICE_MS])))
            stop = not grown and rel <= cfg.eps
            if it in snapshot_iters:
                result.snapshots[it] = (dev.ctx.get_x_f64(), dev.fetch_factors(rank, versions))
            if truth is not None and quality_every > 0 and it % quality_every == 0 and not (stop or it == cfg.max_iters):
                result.quality.append((it, dev.quality(truth, peak)))
            if stop:
                result.converged = True
                break
            if accelerated and cfg.shuffle:
                order = tuple(int(v) for v in rng.permutation(n))  # network.py:515-517
        if truth is not None and result.trace:
            result.quality.append((result.trace[-1].iteration, dev.quality(truth, peak)))
        result.x = dev.ctx.get_x_f64()
        result.slab = dev.slab
        result.factors = dev.fetch_factors(rank, versions)
        return result
    finally:
        dev.ctx.close()
