"""Symbol table: constants <-> dense 32-bit ids.

Behaviour follows the reference interner (reference:
pkg/src/flatlog/interning.py:19-63): strings and Python ints are distinct
constants, ids are dense and handed out in first-seen order, and running
out of id space is an InputError.

Extension for the device path: `reserve_ints(n)` pins the id range
[0, n) to the integer constants 0..n-1, so EDB facts that already arrive as
integer columns (the north-star "load EDB facts as integer columns") are
used as ids without a per-value dictionary lookup. String (and large int)
constants interned afterwards get ids above the reserved block.

Id 0xFFFFFFFF is never handed out: the kernels use it as the "constant not
present in the symbol table" sentinel, so the capacity is 2**32 - 1 ids.
"""

from __future__ import annotations

import numpy as np

from .faults import InputError

VALUE_DTYPE = np.uint32
ID_MAX = 0xFFFFFFFE  # largest id that may be assigned (sentinel excluded)
NO_SYMBOL = 0xFFFFFFFF


class Interner:
    """Bijection between constants (str or int) and dense ids."""

    def __init__(self):
        self._index: dict = {}
        self._spelled: list = []  # constants of ids >= self._reserved
        self._reserved = 0  # ids [0, _reserved) are the ints 0.._reserved-1

    def __len__(self) -> int:
        return self._reserved + len(self._spelled)

    @property
    def reserved_ints(self) -> int:
        return self._reserved

    def reserve_ints(self, n: int):
        """Bind ids [0, n) to the integer constants [0, n).

        Only legal while no other constant has been interned (afterwards the
        low ids are taken). Growing an existing reservation is allowed.
        """
        n = int(n)
        if n <= self._reserved:
            return
        if self._spelled:
            raise InputError(
                "integer-column facts must be loaded before any other constant is "
                "interned (the low id block is already in use)"
            )
        if n - 1 > ID_MAX:
            raise InputError(f"interner capacity exceeded: more than {ID_MAX + 1} distinct constants")
        self._reserved = n

    def intern(self, constant) -> int:
        if isinstance(constant, bool) or not isinstance(constant, (str, int)):
            raise InputError(f"cannot intern {type(constant).__name__} value {constant!r}")
        if type(constant) is int and 0 <= constant < self._reserved:
            return constant
        found = self._index.get(constant)
        if found is not None:
            return found
        ident = len(self)
        if ident > ID_MAX:
            raise InputError(f"interner capacity exceeded: more than {ID_MAX + 1} distinct constants")
        self._index[constant] = ident
        self._spelled.append(constant)
        return ident

    def lookup(self, constant):
        """Id of a constant that is already known, else None."""
        if type(constant) is int and 0 <= constant < self._reserved:
            return constant
        return self._index.get(constant)

    def value(self, ident: int):
        ident = int(ident)
        if ident < self._reserved:
            return ident
        return self._spelled[ident - self._reserved]

    def text(self, ident: int) -> str:
        return str(self.value(ident))

    def texts(self, ids) -> list:
        """Vector form of `text` for an id array (used when rendering rows)."""
        ids = np.asarray(ids)
        if not len(ids):
            return []
        uniq, inv = np.unique(ids, return_inverse=True)
        spelled = [self.text(int(u)) for u in uniq]
        return [spelled[i] for i in inv]

    def intern_rows(self, rows, arity: int):
        """Intern constant tuples into `arity` parallel id columns."""
        columns = [[] for _ in range(arity)]
        intern = self.intern
        for row in rows:
            if len(row) != arity:
                raise InputError(f"expected {arity} columns, got {len(row)}: {row!r}")
            for k in range(arity):
                columns[k].append(intern(row[k]))
        return tuple(np.asarray(c, dtype=VALUE_DTYPE) for c in columns)
