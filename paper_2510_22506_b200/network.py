"""Host-side mirrors of the reference's rank table and factor container
(`network.py:41-223`): same names, same indexing, same init draws, same
version semantics.  Only bookkeeping lives here; every contraction runs on
the device."""
from __future__ import annotations

import math

import numpy as np

__all__ = ["FctnRank", "FctnFactors", "mode_unfold", "mode_fold"]


class FctnRank:
    """Symmetric bond sizes, stored as the strict upper triangle row-major
    (`network.py:41-133`)."""

    __slots__ = ("n", "_tri")

    def __init__(self, n: int, entries) -> None:
        n = int(n)
        if n < 2:
            raise ValueError("a network needs at least two factors")
        tri = tuple(int(e) for e in entries)
        if len(tri) != n * (n - 1) // 2:
            raise ValueError(f"expected {n * (n - 1) // 2} rank entries for n={n}, got {len(tri)}")
        if any(e < 1 for e in tri):
            raise ValueError("rank entries must be >= 1")
        self.n = n
        self._tri = tri

    @classmethod
    def uniform(cls, n: int, r: int) -> "FctnRank":
        return cls(n, [int(r)] * (n * (n - 1) // 2))

    @classmethod
    def from_spec(cls, n: int, value) -> "FctnRank":
        if isinstance(value, FctnRank) or type(value).__name__ == "FctnRank":
            if value.n != n:
                raise ValueError(f"rank table is for n={value.n}, need n={n}")
            return cls(n, value.entries)
        if np.isscalar(value):
            return cls.uniform(n, int(value))
        return cls(n, value)

    def _slot(self, i: int, j: int) -> int:
        if i == j:
            raise KeyError("diagonal has no bond")
        a, b = min(i, j), max(i, j)
        if not 0 <= a < b < self.n:
            raise KeyError(f"bond ({i}, {j}) out of range for n={self.n}")
        return a * (self.n - 1) - a * (a - 1) // 2 + (b - a - 1)

    def __getitem__(self, key) -> int:
        return self._tri[self._slot(int(key[0]), int(key[1]))]

    @property
    def entries(self) -> tuple:
        return self._tri

    def to_vector(self) -> list:
        return list(self._tri)

    def factor_shape(self, k: int, dims) -> tuple:
        dims = tuple(int(d) for d in dims)
        if len(dims) != self.n:
            raise ValueError("dims length does not match table size")
        return tuple(dims[k] if j == k else self[j, k] for j in range(self.n))

    def bond_product(self, k: int) -> int:
        return math.prod(self[j, k] for j in range(self.n) if j != k)

    def increment_below(self, cap: "FctnRank") -> "FctnRank":
        return FctnRank(self.n, [min(e + 1, c) for e, c in zip(self._tri, cap._tri)])

    def any_below(self, cap: "FctnRank") -> bool:
        return any(e < c for e, c in zip(self._tri, cap._tri))

    def __eq__(self, other) -> bool:
        return getattr(other, "n", None) == self.n and tuple(getattr(other, "entries", ())) == self._tri

    def __hash__(self):
        return hash((self.n, self._tri))

    def __repr__(self) -> str:
        return f"FctnRank(n={self.n}, entries={self._tri})"


def mode_unfold(t: np.ndarray, k: int) -> np.ndarray:
    """Rows mode k, columns the other modes ascending, first fastest
    (`tensor.py:130-139`); returned F-contiguous."""
    rest = [m for m in range(t.ndim) if m != k]
    return np.asfortranarray(np.transpose(t, [k] + rest).reshape((t.shape[k], -1), order="F"))


def mode_fold(mat: np.ndarray, k: int, shape) -> np.ndarray:
    """Inverse of :func:`mode_unfold` (`tensor.py:142-150`)."""
    rest = [m for m in range(len(shape)) if m != k]
    t = np.asarray(mat).reshape([shape[k]] + [shape[m] for m in rest], order="F")
    return np.asfortranarray(np.transpose(t, np.argsort([k] + rest)))


class FctnFactors:
    """Factors in slot layout (F-order) plus per-factor version stamps
    (`network.py:139-223`)."""

    def __init__(self, factors) -> None:
        arrays = [np.asfortranarray(np.asarray(a, dtype=np.float64)) for a in factors]
        n = len(arrays)
        if n < 2:
            raise ValueError("need at least two factors")
        for k, a in enumerate(arrays):
            if a.ndim != n:
                raise ValueError(f"factor {k} has order {a.ndim}, expected {n}")
        for i in range(n):
            for j in range(i + 1, n):
                if arrays[i].shape[j] != arrays[j].shape[i]:
                    raise ValueError(f"bond ({i}, {j}) disagrees: {arrays[i].shape[j]} vs {arrays[j].shape[i]}")
        self._arrays = arrays
        self.versions = [0] * n

    @classmethod
    def random(cls, dims, rank: FctnRank, rng: np.random.Generator) -> "FctnFactors":
        """Standard-normal draws in factor order (`network.py:163-169`)."""
        return cls([rng.standard_normal(rank.factor_shape(k, dims)) for k in range(len(dims))])

    @property
    def n(self) -> int:
        return len(self._arrays)

    @property
    def dims(self) -> tuple:
        return tuple(a.shape[k] for k, a in enumerate(self._arrays))

    @property
    def rank(self) -> FctnRank:
        n = self.n
        return FctnRank(n, [self._arrays[i].shape[j] for i in range(n) for j in range(i + 1, n)])

    def factor(self, k: int) -> np.ndarray:
        return self._arrays[k]

    def __getitem__(self, k: int) -> np.ndarray:
        return self._arrays[k]

    def replace(self, k: int, arr: np.ndarray) -> None:
        arr = np.asfortranarray(np.asarray(arr, dtype=np.float64))
        if arr.shape != self._arrays[k].shape:
            raise ValueError(f"replacement for factor {k} has shape {arr.shape}, expected {self._arrays[k].shape}")
        self._arrays[k] = arr
        self.versions[k] += 1

    def copy(self) -> "FctnFactors":
        dup = FctnFactors([a.copy(order="F") for a in self._arrays])
        dup.versions = list(self.versions)
        return dup

    def unfoldings(self) -> list:
        return [mode_unfold(a, k) for k, a in enumerate(self._arrays)]

    def grow(self, new_rank: FctnRank) -> "FctnFactors":
        """Zero-padded embedding into a dominating rank table (`network.py:207-223`)."""
        old = self.rank
        if new_rank.n != self.n or any(a < b for a, b in zip(new_rank.entries, old.entries)):
            raise ValueError("new rank table must dominate the current one")
        grown = []
        for k in range(self.n):
            a = np.zeros(new_rank.factor_shape(k, self.dims), order="F")
            a[tuple(slice(0, s) for s in self._arrays[k].shape)] = self._arrays[k]
            grown.append(a)
        out = FctnFactors(grown)
        out.versions = [v + 1 for v in self.versions]
        return out
