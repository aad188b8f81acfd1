"""Mode-0 sharded restatement of the oracle sweep (test infrastructure).

Mirrors the decomposition the device path uses under `fctn_set_comm`
(SURVEY.md 8e): each rank holds rows [r*I0/n, (r+1)*I0/n) of X and the mask;
factors are replicated; per factor update
  k != 0: Y_k = sum over ranks of X_slab,(k) M_k,slab^T  (all-reduce),
  k == 0: rows of Y_0 = X_slab,(0) M_0^T                   (all-gather),
the Gram G_k = M_k M_k^T is formed from replicated factors (no exchange),
the solve is replicated, the compose/blend is per slab and the four sweep
sums are all-reduced.  `allreduce(a)` sums a numpy array across ranks in
place; `allgather(a)` returns the rank-ordered concatenation.
"""
from __future__ import annotations

import math

import numpy as np

from oracle import fctn_oracle as O


def slab_of(I0, rank, nranks):
    return rank * I0 // nranks, (rank + 1) * I0 // nranks


def sharded_run(values, mask, rank, nranks, allreduce, allgather, *, lam=0.35, delta=0.5, rho=0.1, max_iters=5,
                rank_r=2, seed=0, shuffle=True, sign="positive-definite"):
    n = values.ndim
    dims = values.shape
    lo, hi = slab_of(dims[0], rank, nranks)
    mask = np.asfortranarray(mask)
    values = np.asfortranarray(np.where(mask, values, 0.0))
    xs = np.asfortranarray(values[lo:hi].copy())
    ms = mask[lo:hi]
    lams, deltas = (lam,) * n, (delta,) * n
    spectra = [O.lap_spectrum(dims[k], deltas[k], sign) for k in range(n)]
    tri = O.rank_tri(n, rank_r)
    rng = np.random.default_rng(seed)
    factors = O.random_factors(dims, tri, rng)
    meter = O.Meter()
    order = tuple(range(n))
    for _ in range(max_iters):
        for k in order:
            arr, labels = O.partial_plain(factors, k, meter)
            m = O.m_matrix(arr, labels, k, n)  # s_k x p_k, columns first-mode-fastest
            g = m @ m.T                         # replicated (global factors)
            a_prev = O.unfold(factors[k], k)
            if k == 0:
                y_loc = O.unfold(xs, 0) @ m.T   # this rank's rows of X_(0) M_0^T
                # as the device does: rows x s column-major, padded to slab_max x s
                smax = -(-dims[0] // nranks)
                send = np.zeros(smax * m.shape[0])
                send[:y_loc.size] = y_loc.ravel(order="F")
                rows = allgather(send)
                parts = []
                for r in range(nranks):
                    a, b = slab_of(dims[0], r, nranks)
                    blk = rows[r * smax * m.shape[0]:][:(b - a) * m.shape[0]]
                    parts.append(blk.reshape((b - a, m.shape[0]), order="F"))
                y = np.vstack(parts)
            else:
                # columns of M_k whose mode-0 index lies in the slab
                p_shape = [dims[j] for j in range(n) if j != k]
                msl = m.reshape([m.shape[0]] + p_shape, order="F")[:, lo:hi]
                msl = msl.reshape(m.shape[0], -1, order="F")
                y = O.unfold(xs, k) @ msl.T
                allreduce(y)
            y = y + rho * a_prev
            phi, c = np.linalg.eigh(0.5 * (g + g.T))
            phi = np.maximum(phi, 0.0)
            t = lams[k] * spectra[k][:, None] + phi[None, :] + rho
            w = np.fft.fft(y @ c, axis=0, norm="ortho")
            a_new = np.ascontiguousarray((np.fft.ifft(w / t, axis=0, norm="ortho") @ c.T).real)
            factors[k] = O.fold(a_new, k, factors[k].shape)
        composed = O.compose_full(factors, meter)[lo:hi]
        x_new = (xs * rho + composed) / (1.0 + rho)
        x_new = np.where(ms, xs, x_new)
        sums = np.array([np.sum((x_new - xs) ** 2), np.sum(xs ** 2), np.sum((x_new - composed) ** 2),
                         np.sum(x_new ** 2)])
        allreduce(sums)
        xs = np.asfortranarray(x_new)
        if shuffle:
            order = tuple(int(v) for v in rng.permutation(n))
    rel = math.sqrt(sums[0]) / math.sqrt(sums[1])
    return xs, factors, rel, sums
