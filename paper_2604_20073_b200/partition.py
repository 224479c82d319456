"""Histogram-guided root partitioning (paper Alg. 1 phase 1, Fig. 2).

Every distinct root key k contributes work(k) = outer_rows(k) * d2(k) flat
work units (d2 = rows of the inner source under k, or 1 when the plan has no
inner source). The inclusive prefix sum C flattens the whole join into
[0, T); p workers receive contiguous slices of ceil(T/p) units, so a heavy
key is shared by several workers. A unit decodes to (key, i1, i2) with
local = u - C[k-1], i1 = local // d2(k), i2 = local % d2(k).

This module is the host (numpy) form of that arithmetic, kept so the
reference's partition API (reference: pkg/src/flatlog/executor.py:45-150)
is available unchanged; the device kernels evaluate the same formulas per
slice (csrc/wcoj_kernel.cuh: `wcoj_body` finds kappa by binary search on
the prefix and cuts the slice into at most three rectangles per key;
`run_rect` walks one rectangle).
"""

from __future__ import annotations

import math

import numpy as np

from .faults import InternalError
from .symbols import VALUE_DTYPE


class WorkPartition:
    """Prefix-summed root fan-outs plus per-worker slice bounds."""

    __slots__ = ("keys", "outer_degrees", "d2", "work", "prefix", "total", "p", "bounds", "kappa")

    def __init__(self, keys, outer_degrees, d2, p: int):
        self.keys = keys
        self.outer_degrees = np.asarray(outer_degrees, dtype=np.int64)
        self.d2 = np.asarray(d2, dtype=np.int64)
        self.work = self.outer_degrees * self.d2
        self.prefix = np.cumsum(self.work)
        self.total = int(self.prefix[-1]) if len(self.prefix) else 0
        self.p = int(p)
        step = -(-self.total // self.p) if self.total else 0
        self.bounds = [
            (min(w * step, self.total), min((w + 1) * step, self.total)) for w in range(self.p)
        ]
        self.kappa = [
            int(np.searchsorted(self.prefix, lo, side="right")) if lo < hi else None
            for lo, hi in self.bounds
        ]

    @classmethod
    def from_histogram(cls, hist, p: int) -> "WorkPartition":
        return cls(hist.keys, hist.degrees, np.ones(len(hist.keys), dtype=np.int64), p)

    @classmethod
    def empty(cls, p: int) -> "WorkPartition":
        none = np.empty(0, dtype=np.int64)
        return cls(np.empty(0, dtype=VALUE_DTYPE), none, none, p)

    def slice_sizes(self) -> list:
        return [hi - lo for lo, hi in self.bounds]

    def key_start(self, k: int) -> int:
        return int(self.prefix[k - 1]) if k > 0 else 0

    def spans(self, worker: int):
        """(key index, first local unit, end local unit) pieces of a slice."""
        lo, hi = self.bounds[worker]
        if lo >= hi:
            return
        k = self.kappa[worker]
        nkeys = len(self.prefix)
        while k < nkeys:
            start = self.key_start(k)
            if start >= hi:
                break
            a = max(lo, start) - start
            b = min(hi, int(self.prefix[k])) - start
            if a < b:
                yield k, a, b
            k += 1


def decode_workunit(unit, partition: WorkPartition, d2=None):
    """Flat unit -> (key index, outer row, inner row); scalar or array."""
    d2 = partition.d2 if d2 is None else np.asarray(d2)
    prefix = partition.prefix
    if isinstance(unit, (int, np.integer)):
        u = int(unit)
        if not 0 <= u < partition.total:
            raise InternalError(f"work unit {u} outside [0, {partition.total})")
        k = int(np.searchsorted(prefix, u, side="right"))
        local = u - (int(prefix[k - 1]) if k else 0)
        i1, i2 = divmod(local, int(d2[k]))
        return k, i1, i2
    u = np.asarray(unit, dtype=np.int64)
    if len(u) and (u.min() < 0 or u.max() >= partition.total):
        raise InternalError("work unit outside the flattened range")
    k = np.searchsorted(prefix, u, side="right")
    base = np.where(k > 0, prefix[np.maximum(k - 1, 0)], 0)
    local = u - base
    return k, local // d2[k], local % d2[k]


def encode_workunit(partition: WorkPartition, k, i1, i2, d2=None):
    """Inverse of decode_workunit."""
    d2 = partition.d2 if d2 is None else np.asarray(d2)
    k = np.asarray(k)
    base = np.where(k > 0, partition.prefix[np.maximum(k - 1, 0)], 0)
    return base + np.asarray(i1) * d2[k] + np.asarray(i2)


def rectangles(u0: int, u1: int, d2: int):
    """Cover units [u0, u1) of one key's (outer rows x d2) grid, row-major,
    with at most three (row lo, row hi, col lo, col hi) rectangles."""
    r0, c0 = divmod(u0, d2)
    r1, c1 = divmod(u1, d2)
    if r0 == r1:
        yield (r0, r0 + 1, c0, c1)
        return
    if c0:
        yield (r0, r0 + 1, c0, d2)
        r0 += 1
    if r0 < r1:
        yield (r0, r1, 0, d2)
    if c1:
        yield (r1, r1 + 1, 0, c1)


def slice_bound(total: int, p: int) -> int:
    return math.ceil(total / p) if total else 0
