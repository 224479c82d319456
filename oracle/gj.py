"""Vectorised generic join + stratified semi-naive fixpoint (checker only).

Restates the reference evaluation path in numpy:

* join: attribute-at-a-time intersection over relations sorted under a
  per-atom column order (constants first, then variables by level, then
  anonymous columns of negated atoms), narrowing row ranges by binary search
  at every level, candidates taken from the source with the smallest range,
  negated atoms probed once their last variable binds
  (reference: pkg/src/flatlog/executor.py:188-236 prepare, :342-431
  _root_setup/_descend; pkg/src/flatlog/storage.py:113-216 narrow and
  intersections). All bindings of one level are processed together as
  arrays instead of one worker walking a slice.
* fixpoint: strata = SCCs of the rule graph in topological order (own
  Kosaraju pass, reference oracle pkg/src/flatlog/oracle.py:88-148), recursive
  strata iterate `delta = dedup(join over delta) - full` until every delta is
  empty, counting the final empty round (reference:
  pkg/src/flatlog/runtime.py:259-315).

The variable order here is first occurrence (delta atom first), chosen
independently of the engine's planner: any valid order yields the same
relation, so agreement is evidence rather than identity.
"""

from __future__ import annotations

import numpy as np

from .storage import difference, sort_dedup

VAR = "var"


class Symbols:
    """Oracle-private interner (constants -> int ids)."""

    def __init__(self, reserved_ints: int = 0):
        self.reserved = reserved_ints
        self.ids: dict = {}
        self.spelled: list = []

    def intern(self, c) -> int:
        if type(c) is int and 0 <= c < self.reserved:
            return c
        got = self.ids.get(c)
        if got is None:
            got = self.reserved + len(self.spelled)
            self.ids[c] = got
            self.spelled.append(c)
        return got

    def lookup(self, c):
        if type(c) is int and 0 <= c < self.reserved:
            return c
        return self.ids.get(c)

    def text(self, i: int) -> str:
        i = int(i)
        return str(i) if i < self.reserved else str(self.spelled[i - self.reserved])

    def rows_to_ids(self, rows, arity) -> np.ndarray:
        out = np.array([[self.intern(v) for v in r] for r in rows], dtype=np.int64)
        return out.reshape(-1, arity)

    def ids_to_rows(self, arr: np.ndarray) -> list:
        return sorted(tuple(self.text(v) for v in row) for row in arr.tolist())


def _vsearch(col: np.ndarray, lo: np.ndarray, hi: np.ndarray, v: np.ndarray, right: bool):
    """Vectorised lower/upper bound of v inside col[lo:hi] (each range sorted)."""
    lo = lo.copy()
    hi = hi.copy()
    while True:
        active = lo < hi
        if not active.any():
            return lo
        mid = (lo + hi) >> 1
        mv = col[np.minimum(mid, len(col) - 1)] if len(col) else mid
        go_right = (mv <= v) if right else (mv < v)
        go_right &= active
        lo = np.where(go_right, mid + 1, lo)
        hi = np.where(active & ~go_right, mid, hi)


def _narrow(col, lo, hi, v):
    return _vsearch(col, lo, hi, v, False), _vsearch(col, lo, hi, v, True)


class _Src:
    __slots__ = ("rows", "negated", "col_levels", "nconst", "levels", "bits", "_keys")

    def __init__(self, rows, negated, col_levels, nconst):
        self.rows = rows
        self.negated = negated
        self.col_levels = col_levels
        self.nconst = nconst
        self.levels: dict = {}
        for off, lvl in enumerate(col_levels):
            self.levels.setdefault(lvl, []).append(nconst + off)
        top = int(rows.max()) if rows.size else 0
        self.bits = max(1, top.bit_length())
        self._keys: dict = {}

    def prefix_keys(self, c):
        """Sorted packed keys of columns 0..c (None when they do not fit)."""
        if (c + 1) * self.bits > 62:
            return None
        k = self._keys.get(c)
        if k is None:
            k = self.rows[:, 0].copy() if c == 0 else (self.prefix_keys(c - 1) << self.bits) | self.rows[:, c]
            self._keys[c] = k
        return k

    def narrow(self, c, lo, hi, v):
        """Rows of [lo, hi) (all sharing columns < c) whose column c equals v."""
        keys = self.prefix_keys(c)
        if keys is None or np.any(v >= (1 << self.bits)):
            return _narrow(self.rows[:, c], lo, hi, v)
        nonempty = lo < hi
        if c == 0:
            q = v
        else:
            base = self.prefix_keys(c - 1)[np.minimum(lo, len(self.rows) - 1)]
            q = (base << self.bits) | v
        a = np.searchsorted(keys, q, "left")
        b = np.searchsorted(keys, q, "right")
        return np.where(nonempty, a, lo), np.where(nonempty, b, lo)


def variable_order(rule, delta_pos=None) -> list:
    """Delta atom's variables first, then repeatedly the first-occurring
    variable that shares a positive atom with an already ordered one (the
    next level is always constrained by a bound neighbour; a variable
    reachable only through an unbound one would be enumerated over its whole
    domain), falling back to first occurrence for disconnected bodies. Any
    order gives the same relation; this one keeps the oracle's work close
    to the join's output size."""
    order = []
    if delta_pos is not None:
        order += [v for v in rule.body[delta_pos].variables() if v not in order]
    positive = [a for a in rule.body if not a.negated]
    pending = []
    for a in positive:
        for v in a.variables():
            if v not in order and v not in pending:
                pending.append(v)
    while pending:
        bound = set(order)
        pick = next((v for v in pending
                     if any(v in a.variables() and bound.intersection(a.variables()) for a in positive)),
                    pending[0])
        order.append(pick)
        pending.remove(pick)
    return order


def join_rule(rule, relation_of, const_id, delta_pos=None, level0_keep=None, cache=None) -> np.ndarray:
    """All head tuples (with duplicates) of one rule instance.

    relation_of(body_pos) -> sorted unique int64 rows of that atom's
    relation version; const_id(literal) -> id or None (unknown constant).
    level0_keep optionally restricts the first variable to a sorted set of
    values (used for bounded samples of large instances); `cache` (a dict)
    keeps each atom's sorted index between calls on unchanged relations.
    """
    order = variable_order(rule, delta_pos)
    level_of = {v: i for i, v in enumerate(order)}
    depth = len(order)
    srcs = []
    for pos, atom in enumerate(rule.body):
        consts = [k for k, t in enumerate(atom.args) if t.kind != VAR]
        bound = sorted(
            (k for k, t in enumerate(atom.args) if t.kind == VAR and t.value in level_of),
            key=lambda k: (level_of[atom.args[k].value], k),
        )
        free = [k for k, t in enumerate(atom.args) if t.kind == VAR and t.value not in level_of]
        perm = consts + bound + free
        if cache is not None and pos in cache:
            rows = cache[pos]
        else:
            rows = relation_of(pos)
            rows = sort_dedup(rows[:, perm]) if len(rows) else np.empty((0, atom.arity), np.int64)
            if cache is not None:
                cache[pos] = rows
        lo, hi = 0, len(rows)
        for c, k in enumerate(consts):
            ident = const_id(atom.args[k].value)
            if ident is None:
                lo = hi = 0
                break
            l2, h2 = _narrow(rows[:, c], np.array([lo]), np.array([hi]), np.array([ident]))
            lo, hi = int(l2[0]), int(h2[0])
        s = _Src(rows, atom.negated, [level_of[atom.args[k].value] for k in bound], len(consts))
        srcs.append((s, lo, hi))
        if not atom.negated and lo >= hi:
            return np.empty((0, rule.head.arity), np.int64)
        if atom.negated and not s.col_levels and lo < hi:
            return np.empty((0, rule.head.arity), np.int64)

    nb = 1
    vals = np.zeros((1, depth), np.int64)
    los = [np.array([lo], np.int64) for _, lo, _ in srcs]
    his = [np.array([hi], np.int64) for _, _, hi in srcs]
    for level in range(depth):
        specs = [(a, s.levels[level]) for a, (s, _, _) in enumerate(srcs) if level in s.levels]
        cands = [(a, cols) for a, cols in specs if not srcs[a][0].negated]
        lens = np.stack([his[a] - los[a] for a, _ in cands])
        pick = np.argmin(lens, axis=0)
        pb, pv = [], []
        for ci, (a, cols) in enumerate(cands):
            sel = np.nonzero(pick == ci)[0]
            if not len(sel):
                continue
            lo, hi = los[a][sel], his[a][sel]
            n = hi - lo
            b = np.repeat(sel, n)
            starts = np.repeat(lo, n)
            row = starts + (np.arange(n.sum()) - np.repeat(np.cumsum(n) - n, n))
            col = srcs[a][0].rows[:, cols[0]]
            v = col[row]
            first = (row == starts) | (v != col[np.maximum(row - 1, 0)])
            pb.append(b[first])
            pv.append(v[first])
        if not pb:
            return np.empty((0, rule.head.arity), np.int64)
        b = np.concatenate(pb)
        v = np.concatenate(pv)
        if level == 0 and level0_keep is not None:
            keep = np.isin(v, level0_keep)
            b, v = b[keep], v[keep]
        alive = np.ones(len(b), bool)
        new_lo = [lo_[b] for lo_ in los]
        new_hi = [hi_[b] for hi_ in his]
        for a, cols in specs:
            s = srcs[a][0]
            lo, hi = new_lo[a], new_hi[a]
            for c in cols:
                lo, hi = s.narrow(c, lo, hi, v)
            new_lo[a], new_hi[a] = lo, hi
            if not s.negated:
                alive &= lo < hi
            elif max(s.col_levels) == level:
                alive &= lo >= hi
        b, v = b[alive], v[alive]
        vals = vals[b]
        vals[:, level] = v
        los = [x[alive] for x in new_lo]
        his = [x[alive] for x in new_hi]
        if not len(b):
            return np.empty((0, rule.head.arity), np.int64)
    out = np.empty((len(vals), rule.head.arity), np.int64)
    for k, t in enumerate(rule.head.args):
        out[:, k] = vals[:, level_of[t.value]] if t.kind == VAR else const_id(t.value, create=True)
    return out


def rule_components(rules) -> list:
    """Kosaraju SCCs in topological order: [(member rule idxs, recursive)]."""
    n = len(rules)
    producers: dict = {}
    for i, r in enumerate(rules):
        producers.setdefault(r.head.relation, []).append(i)
    fwd = [set() for _ in range(n)]
    for j, r in enumerate(rules):
        for a in r.body:
            for i in producers.get(a.relation, ()):
                fwd[i].add(j)
    rev = [set() for _ in range(n)]
    for i in range(n):
        for j in fwd[i]:
            rev[j].add(i)
    seen = [False] * n
    finish = []
    for root in range(n):
        if seen[root]:
            continue
        seen[root] = True
        stack = [(root, iter(sorted(fwd[root])))]
        while stack:
            node, it = stack[-1]
            nxt = next((w for w in it if not seen[w]), None)
            if nxt is None:
                finish.append(node)
                stack.pop()
            else:
                seen[nxt] = True
                stack.append((nxt, iter(sorted(fwd[nxt]))))
    comp = [-1] * n
    comps = []
    for node in reversed(finish):
        if comp[node] >= 0:
            continue
        members, todo = [], [node]
        comp[node] = len(comps)
        while todo:
            x = todo.pop()
            members.append(x)
            for y in rev[x]:
                if comp[y] < 0:
                    comp[y] = len(comps)
                    todo.append(y)
        comps.append(sorted(members))
    return [(m, len(m) > 1 or m[0] in fwd[m[0]]) for m in comps]


def fixpoint(program, edb: dict, symbols: Symbols):
    """Least fixpoint of a parsed program over id-coded EDB rows.

    Returns ({relation: sorted unique rows}, [(frozenset rule idxs, recursive, rounds)]).
    Program ground facts are interned through `symbols`.
    """
    decls = program.declarations
    full = {n: np.empty((0, a), np.int64) for n, a in decls.items()}
    for name, rows in program.facts.items():
        full[name] = np.concatenate([full[name], symbols.rows_to_ids(rows, decls[name])])
    for name, rows in edb.items():
        full[name] = np.concatenate([full[name], np.asarray(rows, np.int64).reshape(-1, decls[name])])
    full = {n: sort_dedup(r) for n, r in full.items()}

    def const_id(lit, create=False):
        return symbols.intern(lit) if create else symbols.lookup(lit)

    rules = list(program.rules)
    report = []
    for members, recursive in rule_components(rules):
        group = [rules[m] for m in members]
        heads = sorted({r.head.relation for r in group})
        if not recursive:
            for r in group:
                got = join_rule(r, lambda p, r=r: full[r.body[p].relation], const_id)
                full[r.head.relation] = sort_dedup(np.concatenate([full[r.head.relation], got]))
            report.append((frozenset(members), False, 1))
            continue
        delta = {h: full[h] for h in heads}
        rounds = 0
        while True:
            rounds += 1
            staged = {h: [] for h in heads}
            for r in group:
                for pos, a in enumerate(r.body):
                    if a.negated or a.relation not in delta:
                        continue

                    def rel(p, r=r, pos=pos):
                        name = r.body[p].relation
                        return delta[name] if p == pos else full[name]

                    staged[r.head.relation].append(join_rule(r, rel, const_id, delta_pos=pos))
            fresh = {}
            for h in heads:
                got = np.concatenate(staged[h]) if staged[h] else np.empty((0, decls[h]), np.int64)
                fresh[h] = difference(sort_dedup(got), full[h])
            if all(len(f) == 0 for f in fresh.values()):
                break
            for h in heads:
                if len(fresh[h]):
                    full[h] = sort_dedup(np.concatenate([full[h], fresh[h]]))
            delta = fresh
        report.append((frozenset(members), True, rounds))
    return full, report


def fixpoint_text(program, facts: dict):
    """Convenience wrapper on constant (text) facts -> ({rel: sorted text rows}, report)."""
    sym = Symbols()
    edb = {k: sym.rows_to_ids(v, program.declarations[k]) for k, v in facts.items()}
    full, report = fixpoint(program, edb, sym)
    return {k: sym.ids_to_rows(v) for k, v in full.items()}, report
