"""Relation digests for full-size parity (checker only).

A relation is compared as a sorted, duplicate-free tuple set. At BASELINE
sizes (up to ~6 GB of output) the tuples themselves are not committed;
instead both sides reduce the relation to

* ``n``       — the cardinality;
* ``sha256``  — sha256 over the per-column sha256 digests of the sorted
  relation's columns (u32 little-endian), column 0 first. Each column's
  hash is fed chunk by chunk in row order, so the digest can be formed from
  a relation produced in sorted pieces (e.g. the triangle oracle, chunked
  by root key) without ever holding it whole;
* ``fold64``  — an order-independent 64-bit fold (sum mod 2^64 of a
  splitmix64 hash of every row), a second, independent witness.

Inputs are (arity, n) arrays (numpy or anything with ``__array__``), already
sorted lexicographically and distinct — the engine's `relation_columns`
and the oracle's sorted rows (transposed) both are.
"""

from __future__ import annotations

import hashlib

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_PHI = np.uint64(0x9E3779B97F4A7C15)


def _mix(x: np.ndarray) -> np.ndarray:
    x = x.copy()
    x ^= x >> np.uint64(30)
    x *= _M1
    x ^= x >> np.uint64(27)
    x *= _M2
    x ^= x >> np.uint64(31)
    return x


def row_hash(cols: np.ndarray) -> np.ndarray:
    """splitmix64 chain over the columns of each row -> uint64 per row."""
    with np.errstate(over="ignore"):
        h = np.full(cols.shape[1], 0x243F6A8885A308D3, np.uint64)
        for c in range(cols.shape[0]):
            h = _mix(h * _PHI + cols[c].astype(np.uint64))
    return h


class Digester:
    """Streaming digest of a sorted relation fed in row order, in pieces."""

    def __init__(self, arity: int):
        self.arity = arity
        self.n = 0
        self.cols = [hashlib.sha256() for _ in range(arity)]
        self.fold = np.uint64(0)
        self.last = None  # last row seen (sortedness / distinctness check)

    def update(self, cols, chunk: int = 1 << 24):
        cols = np.asarray(cols)
        if cols.ndim != 2 or cols.shape[0] != self.arity:
            raise ValueError(f"expected ({self.arity}, n) columns, got {cols.shape}")
        n = cols.shape[1]
        if n == 0:
            return self
        for lo in range(0, n, chunk):
            part = np.ascontiguousarray(cols[:, lo:lo + chunk].astype(np.uint32, copy=False))
            self._check_order(part)
            for c in range(self.arity):
                self.cols[c].update(part[c].astype("<u4", copy=False).tobytes())
            with np.errstate(over="ignore"):
                self.fold = np.uint64(self.fold + row_hash(part).sum(dtype=np.uint64))
            self.n += part.shape[1]
        return self

    def _check_order(self, part: np.ndarray):
        rows = part.astype(np.int64)
        if self.last is not None:
            rows = np.concatenate([self.last[:, None], rows], axis=1)
        if rows.shape[1] > 1:
            a, b = rows[:, :-1], rows[:, 1:]
            lt = np.zeros(a.shape[1], bool)
            eq = np.ones(a.shape[1], bool)
            for c in range(self.arity):
                lt |= eq & (a[c] < b[c])
                eq &= a[c] == b[c]
            if not lt.all():
                raise ValueError("relation pieces are not strictly increasing (unsorted or duplicate rows)")
        self.last = part[:, -1].astype(np.int64)

    def result(self) -> dict:
        top = hashlib.sha256()
        for h in self.cols:
            top.update(h.digest())
        return {"n": int(self.n), "sha256": top.hexdigest(), "fold64": f"{int(self.fold):016x}"}


def digest(cols) -> dict:
    """Digest of a whole sorted (arity, n) relation."""
    cols = np.asarray(cols)
    return Digester(cols.shape[0]).update(cols).result()
