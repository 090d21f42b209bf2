"""Interval bounds of the exponent-sum space (host side).

`SplitSet` and `GridParams` keep the reference's validation
(split.py:24-64).  `select_grid` computes the same almost-regular grid sample
as the reference (split.py:67-101) with numpy, for the multi-GPU partition
(paper Alg. 2): its bounds are cut into per-GPU ranges by `partition_by_ops`.
On one GPU the device chooses its own interval geometry.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import SENTINEL, check_compatible


@dataclass(frozen=True)
class GridParams:
    l: int = 64

    def __post_init__(self):
        if self.l < 1:
            raise ValueError(f"grid density must be >= 1, got {self.l}")

    @property
    def n_star(self) -> int:
        return (self.l + 1) ** 2


class SplitSet:
    """Strictly ascending bounds ending with the sentinel (split.py:39-64)."""

    __slots__ = ("bounds",)

    def __init__(self, bounds):
        bounds = [int(x) for x in bounds]
        if len(bounds) < 2 or bounds[-1] != SENTINEL:
            raise ValueError("split set must end with the sentinel bound")
        if any(x >= y for x, y in zip(bounds, bounds[1:])):
            raise ValueError("split set bounds must be strictly ascending")
        self.bounds = bounds

    @property
    def n_s(self) -> int:
        return len(self.bounds)

    @property
    def n_intervals(self) -> int:
        return len(self.bounds) - 1

    def interval(self, k: int) -> tuple:
        return self.bounds[k], self.bounds[k + 1]

    def __repr__(self):
        return f"<SplitSet {self.n_intervals} intervals>"


def _exps(p) -> np.ndarray:
    return p.exps_array() if hasattr(p, "exps_array") else np.fromiter(p.exps, np.uint64, len(p.exps))


def select_grid(a, b, params: GridParams = GridParams()) -> SplitSet:
    """Grid sample of the pair matrix, sorted and deduplicated.

    Same point set as the reference (split.py:82-101): density clamped to
    min(l, n_a, n_b); 1-based sampled rows i = 1, 1+rs, ...; alternate rows
    staggered by half a column stride; last column and last row sampled; the
    minimum sum and the sentinel always present.
    """
    check_compatible(a, b)
    if not a.exps or not b.exps:
        raise ValueError("cannot build a split set for an empty operand")
    A, B = _exps(a), _exps(b)
    na, nb = A.size, B.size
    l = max(1, min(params.l, na, nb))
    rs, cs, half = na // l, nb // l, nb // (2 * l)
    rows = np.arange(1, na + 1, rs, dtype=np.int64)
    pts = []
    for i in rows.tolist():
        j0 = 1 + ((i // rs) % 2) * half
        cols = np.arange(j0, nb + 1, cs, dtype=np.int64)
        pts.append(A[i - 1] + B[cols - 1])
    pts.append(A[rows - 1] + B[nb - 1])
    pts.append(A[na - 1] + B[np.arange(1, nb + 1, cs, dtype=np.int64) - 1])
    pts.append(np.array([A[0] + B[0]], dtype=np.uint64))
    allp = np.unique(np.concatenate(pts))
    out = allp.tolist()
    if not out or out[-1] != SENTINEL:
        out.append(SENTINEL)
    return SplitSet(out)
