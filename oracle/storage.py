"""Numpy restatement of the reference storage operations (checker only).

Row sets are 2-D int64 arrays (rows x arity). Every function cites the
reference routine whose behaviour it restates.
"""

from __future__ import annotations

import numpy as np

DEFAULT_FLUSH_LIMIT = 4096  # reference: pkg/src/flatlog/storage.py:25


def as_rows(rows, arity):
    a = np.asarray(rows, dtype=np.int64)
    return a.reshape(-1, arity) if a.size else np.empty((0, arity), np.int64)


def lex_order(rows: np.ndarray) -> np.ndarray:
    """Stable lexicographic order (reference rowops.lexsort_order, :35)."""
    if rows.shape[1] == 0:
        return np.arange(len(rows))
    return np.lexsort(rows.T[::-1])


def _packable(*arrays):
    """Bit width per column if every row of every array packs into 63 bits."""
    arity = arrays[0].shape[1]
    top = 0
    for a in arrays:
        if a.size:
            if a.min() < 0:
                return None
            top = max(top, int(a.max()))
    bits = max(1, top.bit_length())
    return bits if bits * arity <= 63 else None


def _pack(rows: np.ndarray, bits: int) -> np.ndarray:
    key = np.zeros(len(rows), np.int64)
    for k in range(rows.shape[1]):
        key = (key << bits) | rows[:, k]
    return key


def _unpack(keys: np.ndarray, bits: int, arity: int) -> np.ndarray:
    out = np.empty((len(keys), arity), np.int64)
    mask = (1 << bits) - 1
    for k in range(arity - 1, -1, -1):
        out[:, k] = keys & mask
        keys = keys >> bits
    return out


def sort_dedup(rows: np.ndarray) -> np.ndarray:
    """Sorted distinct rows (reference rowops.sort_dedup, :60)."""
    if len(rows) <= 1:
        return rows.copy()
    bits = _packable(rows)
    if bits is not None and rows.shape[1] > 0:
        return _unpack(np.unique(_pack(rows, bits)), bits, rows.shape[1])
    s = rows[lex_order(rows)]
    keep = np.ones(len(s), bool)
    keep[1:] = np.any(s[1:] != s[:-1], axis=1)
    return s[keep]


def sort_dedup_order(rows: np.ndarray, order) -> np.ndarray:
    """Reorder columns to `order` then sort+dedup (reference storage.sort_dedup, :304)."""
    return sort_dedup(rows[:, list(order)])


def is_sorted_strict(rows: np.ndarray) -> bool:
    """reference rowops.is_sorted_strict, :64."""
    if len(rows) <= 1:
        return True
    a, b = rows[:-1], rows[1:]
    lt = np.zeros(len(a), bool)
    eq = np.ones(len(a), bool)
    for k in range(rows.shape[1]):
        lt |= eq & (a[:, k] < b[:, k])
        eq &= a[:, k] == b[:, k]
    return bool(lt.all())


def _row_keys(a: np.ndarray, b: np.ndarray):
    """Consistent scalar keys for rows of a and b (joint dense ranking)."""
    both = np.concatenate([a, b])
    if len(both) == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    _, inv = np.unique(both, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    return inv[: len(a)], inv[len(a):]


def member(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Per-row membership of a in b (reference rowops.member_mask, :95)."""
    if len(a) == 0 or len(b) == 0:
        return np.zeros(len(a), bool)
    bits = _packable(a, b) if a.shape[1] else None
    if bits is not None:
        ka, kb = _pack(a, bits), np.sort(_pack(b, bits))
        pos = np.minimum(np.searchsorted(kb, ka), len(kb) - 1)
        return kb[pos] == ka
    ka, kb = _row_keys(a, b)
    return np.isin(ka, kb)


def difference(a: np.ndarray, *bs: np.ndarray) -> np.ndarray:
    """Rows of a present in none of bs (reference rowops.diff_sorted, :118)."""
    drop = np.zeros(len(a), bool)
    for b in bs:
        drop |= member(a, b)
    return a[~drop]


def compute_delta(new: np.ndarray, head: np.ndarray, body: np.ndarray) -> np.ndarray:
    """sort_dedup(new) minus (head | body) (reference storage.compute_delta, :311)."""
    return difference(sort_dedup(new), head, body)


def merge_sorted(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Sorted union of disjoint sorted sets (reference rowops.merge_sorted, :77)."""
    if len(a) == 0:
        return b.copy()
    if len(b) == 0:
        return a.copy()
    c = np.concatenate([a, b])
    return c[lex_order(c)]


class Histogram:
    """Run-length summary of a sorted key column (reference storage.Histogram, :28)."""

    def __init__(self, keys, degrees):
        self.keys = np.asarray(keys, np.int64)
        self.degrees = np.asarray(degrees, np.int64)
        self.prefix = np.cumsum(self.degrees)

    @classmethod
    def over(cls, col) -> "Histogram":
        col = np.asarray(col, np.int64)
        if len(col) == 0:
            return cls([], [])
        keys, counts = np.unique(col, return_counts=True)
        return cls(keys, counts)

    def updated(self, delta_col) -> "Histogram":
        """reference storage.Histogram.updated, :63."""
        if len(delta_col) == 0:
            return self
        d = Histogram.over(delta_col)
        keys = np.concatenate([self.keys, d.keys])
        degs = np.concatenate([self.degrees, d.degrees])
        uk, inv = np.unique(keys, return_inverse=True)
        out = np.zeros(len(uk), np.int64)
        np.add.at(out, inv, degs)
        return Histogram(uk, out)


class HeadBody:
    """One sorted index with head/body buffers (reference storage.ColumnarRelation, :219)."""

    def __init__(self, arity, flush_limit=DEFAULT_FLUSH_LIMIT):
        self.arity = arity
        self.flush_limit = flush_limit
        self.head = np.empty((0, arity), np.int64)
        self.body = np.empty((0, arity), np.int64)
        self.hist = Histogram([], [])

    def merge_delta(self, delta: np.ndarray):
        """reference storage.ColumnarRelation.merge_delta, :272: flush head+delta
        into body once |head|+|delta| > max(flush_limit, |body| // 8)."""
        if len(delta) == 0:
            return self
        self.hist = self.hist.updated(delta[:, 0])
        if len(self.head) + len(delta) > max(self.flush_limit, len(self.body) // 8):
            self.body = merge_sorted(merge_sorted(self.body, self.head), delta)
            self.head = np.empty((0, self.arity), np.int64)
        else:
            self.head = merge_sorted(self.head, delta)
        return self

    def rows(self) -> np.ndarray:
        return merge_sorted(self.body, self.head)
