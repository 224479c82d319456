"""ctypes driver of the multi-core C++ oracle (oracle/gj_native.cpp).

TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline, never the
product). `fixpoint()` has the signature and result of `oracle.gj.fixpoint`
and evaluates the same thing: this module encodes the parsed program with
gj's own rule grouping (`rule_components`) and per-instance variable order
(`variable_order`), and the C++ side runs the join + semi-naive loop on all
host cores. Pinned by the same reference goldens as gj.py
(tests/test_oracle_golden.py).

Build: `python -m oracle.native` (or __graft_entry__.build()) compiles
oracle/liboracle_gj.so with g++ -fopenmp; no CUDA involved.
"""

from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess

import numpy as np

from .gj import VAR, Symbols, rule_components, variable_order

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gj_native.cpp")
LIB = os.path.join(HERE, "liboracle_gj.so")
_LIB = None


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cxx = shutil.which("g++") or "g++"
    tmp = LIB + ".tmp"
    subprocess.run([cxx, "-O3", "-march=x86-64-v2", "-fopenmp", "-std=c++17", "-fPIC", "-shared", "-o", tmp, SRC],
                   check=True)
    os.replace(tmp, LIB)
    return LIB


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.og_error.restype = C.c_char_p
        L.og_new.restype = C.c_void_p
        L.og_new.argtypes = [C.c_void_p, C.c_uint64]
        L.og_free.argtypes = [C.c_void_p]
        L.og_set_threads.argtypes = [C.c_int]
        L.og_load.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64]
        L.og_keep_level0.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.og_solve.argtypes = [C.c_void_p]
        L.og_size.restype = C.c_uint64
        L.og_size.argtypes = [C.c_void_p, C.c_int]
        L.og_rows.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.og_ncomp.argtypes = [C.c_void_p]
        L.og_rounds.argtypes = [C.c_void_p, C.c_int]
        _LIB = L
    return _LIB


def _check(rc):
    if rc != 0:
        raise RuntimeError("oracle: " + lib().og_error().decode(errors="replace"))


def _split64(v: int):
    return [v & 0xFFFFFFFF, (v >> 32) & 0xFFFFFFFF]


def _encode_instance(rule, rel_id, symbols, delta_pos=None) -> list:
    """One join instance, mirroring gj.join_rule's per-atom column orders."""
    order = variable_order(rule, delta_pos)
    level_of = {v: i for i, v in enumerate(order)}
    w = [rel_id[rule.head.relation], rule.head.arity]
    for t in rule.head.args:
        if t.kind == VAR:
            w += [0, level_of[t.value], 0]
        else:
            w += [1, *_split64(symbols.intern(t.value))]
    w += [len(order), len(rule.body)]
    for pos, atom in enumerate(rule.body):
        consts = [k for k, t in enumerate(atom.args) if t.kind != VAR]
        bound = sorted((k for k, t in enumerate(atom.args) if t.kind == VAR and t.value in level_of),
                       key=lambda k: (level_of[atom.args[k].value], k))
        free = [k for k, t in enumerate(atom.args) if t.kind == VAR and t.value not in level_of]
        perm = consts + bound + free
        w += [rel_id[atom.relation], 1 if pos == delta_pos else 0, int(atom.negated), atom.arity, *perm,
              len(consts)]
        for k in consts:
            ident = symbols.lookup(atom.args[k].value)
            w += [0, 0xFFFFFFFF] if ident is None else _split64(ident)
        w += [len(bound), *[level_of[atom.args[k].value] for k in bound]]
    return w


def encode(program, symbols) -> tuple:
    """(int32 program words, relation names, component member lists)."""
    names = sorted(program.declarations)
    rel_id = {n: i for i, n in enumerate(names)}
    words = [len(names), *[program.declarations[n] for n in names]]
    rules = list(program.rules)
    comps = rule_components(rules)
    words.append(len(comps))
    for members, recursive in comps:
        group = [rules[m] for m in members]
        heads = sorted({r.head.relation for r in group})
        insts = []
        if not recursive:
            for r in group:
                insts.append(_encode_instance(r, rel_id, symbols))
        else:
            for r in group:
                for pos, a in enumerate(r.body):
                    if a.negated or a.relation not in heads:
                        continue
                    insts.append(_encode_instance(r, rel_id, symbols, delta_pos=pos))
        words += [int(recursive), len(heads), *[rel_id[h] for h in heads], len(insts)]
        for w in insts:
            words += w
    arr = np.array([x & 0xFFFFFFFF for x in words], dtype=np.uint32).view(np.int32)
    return arr, names, comps


class Solver:
    """One C++ oracle evaluation; results read back per relation."""

    def __init__(self, program, edb: dict, symbols: Symbols, threads: int | None = None, keep_level0=None):
        L = lib()
        if threads:
            L.og_set_threads(int(threads))
        self.threads = L.og_set_threads(0)
        self.program = program
        self.words, self.names, self.comps = encode(program, symbols)
        self.h = L.og_new(self.words.ctypes.data, len(self.words))
        if not self.h:
            _check(1)
        self.rel_id = {n: i for i, n in enumerate(self.names)}
        decls = program.declarations
        for name, rows in program.facts.items():
            self.load(name, symbols.rows_to_ids(rows, decls[name]))
        for name, rows in edb.items():
            self.load(name, rows)
        if keep_level0 is not None:
            k = np.ascontiguousarray(np.asarray(keep_level0, dtype=np.uint32))
            _check(L.og_keep_level0(self.h, k.ctypes.data, len(k)))

    def load(self, name, rows):
        """rows: (n, arity) integers (row-major), or (arity, n) uint32 columns via load_columns."""
        a = np.asarray(rows)
        if a.size == 0:
            return
        if a.min() < 0 or a.max() > 0xFFFFFFFF:
            raise ValueError(f"{name}: ids outside u32")
        a = np.ascontiguousarray(a.reshape(-1, self.program.declarations[name]).astype(np.uint32))
        _check(lib().og_load(self.h, self.rel_id[name], a.ctypes.data, len(a)))

    def load_columns(self, name, cols):
        self.load(name, np.asarray(cols).T)

    def solve(self):
        _check(lib().og_solve(self.h))
        return self

    def size(self, name) -> int:
        return int(lib().og_size(self.h, self.rel_id[name]))

    def rows_u32(self, name) -> np.ndarray:
        """(n, arity) uint32, sorted, distinct."""
        n = self.size(name)
        out = np.empty((n, self.program.declarations[name]), np.uint32)
        if n:
            _check(lib().og_rows(self.h, self.rel_id[name], out.ctypes.data))
        return out

    def report(self) -> list:
        L = lib()
        return [(frozenset(m), rec, int(L.og_rounds(self.h, i))) for i, (m, rec) in enumerate(self.comps)]

    def close(self):
        if self.h:
            lib().og_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


def fixpoint(program, edb: dict, symbols: Symbols, threads: int | None = None):
    """Same contract as oracle.gj.fixpoint: ({relation: sorted unique int64
    rows}, [(frozenset rule idxs, recursive, rounds)])."""
    s = Solver(program, edb, symbols, threads).solve()
    out = {n: s.rows_u32(n).astype(np.int64) for n in program.declarations}
    rep = s.report()
    s.close()
    return out, rep


def fixpoint_text(program, facts: dict, threads: int | None = None):
    sym = Symbols()
    edb = {k: sym.rows_to_ids(v, program.declarations[k]) for k, v in facts.items()}
    full, report = fixpoint(program, edb, sym, threads)
    return {k: sym.ids_to_rows(v) for k, v in full.items()}, report


if __name__ == "__main__":
    print(build(force=True))
