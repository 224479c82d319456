"""Host frontend parity with the reference: parser, strata, compiler, partitions.

Golden fixtures were produced by running the reference package itself
(tests/golden/make_golden.py); these tests need no GPU.
"""

import re

import numpy as np
import pytest

from paper_2604_20073_b200 import compile_program, parse, stratify
from paper_2604_20073_b200.compiler import (
    apply_splits,
    choose_variable_order,
    compile_instance,
    seminaive_instances,
    validate_plan,
)
from paper_2604_20073_b200.faults import InternalError, ProgramError
from paper_2604_20073_b200.partition import WorkPartition, decode_workunit, encode_workunit
from paper_2604_20073_b200.symbols import Interner
from programs import CORPUS

ANON = re.compile(r"_#\d+")


def _norm(obj, names):
    """Rename anonymous variables (process-global counters) canonically."""
    if isinstance(obj, str):
        return ANON.sub(lambda m: names.setdefault(m.group(0), f"_anon{len(names)}"), obj)
    if isinstance(obj, (list, tuple)):
        return [_norm(x, names) for x in obj]
    if isinstance(obj, dict):
        return {k: _norm(v, names) for k, v in obj.items()}
    return obj


def _plan_record(plan):
    return {
        "plan_id": plan.plan_id,
        "rule_index": plan.rule_index,
        "head_relation": plan.head_relation,
        "variable_order": list(plan.variable_order),
        "atoms": [
            {
                "relation": a.relation,
                "version": a.version,
                "negated": a.negated,
                "column_order": list(a.column_order),
                "const_values": list(a.const_values),
                "col_levels": list(a.col_levels),
                "check_level": a.check_level,
            }
            for a in plan.atoms
        ],
        "head_cols": [list(h) for h in plan.head_cols],
        "delta_atom": plan.delta_atom,
        "outer_atom": plan.outer_atom,
        "inner_atom": plan.inner_atom,
        "cand_atoms": [list(c) for c in plan.cand_atoms],
        "narrow_specs": [[[a, list(c)] for a, c in lvl] for lvl in plan.narrow_specs],
        "checks": [list(c) for c in plan.checks],
    }


@pytest.mark.parametrize("name", sorted(CORPUS))
def test_compiled_plans_match_reference(golden, name):
    want = golden("plans.json")[name]
    prog = compile_program(parse(CORPUS[name]))
    got = {
        "strata": [
            {
                "index": s.index,
                "rules": [r.index for r in s.rules],
                "recursive": s.recursive,
                "plans": [_plan_record(p) for p in s.plans],
            }
            for s in prog.strata
        ],
        "orders": {k: sorted(list(o) for o in v) for k, v in prog.orders.items()},
        "declarations": prog.declarations,
        "rules": [str(r) for r in prog.program.rules],
    }
    assert _norm(got, {}) == _norm(want, {})


def test_program_errors_match_reference(golden):
    for case in golden("errors.json"):
        with pytest.raises(ProgramError) as info:
            compile_program(parse(case["source"]))
        assert str(info.value) == case["error"], case["source"]
        assert info.value.line == case["line"]


def test_tc_program_shape():
    prog = parse(CORPUS["tc"])
    assert len(prog.rules) == 2 and prog.declarations == {"Edge": 2, "TC": 2}
    strata = stratify(prog.rules)
    assert [s.recursive for s in strata] == [False, True]
    (rule, pos), = seminaive_instances(strata[1])
    assert pos == 0 and rule.body[0].relation == "TC"


def test_cge_rule_shape():
    rule = [r for r in parse(CORPUS["cge"]).rules if r.label == "cge"][0]
    assert len(rule.body) == 6
    counts = {}
    for a in rule.body:
        for v in set(a.variables()):
            counts[v] = counts.get(v, 0) + 1
    assert len(counts) == 8 and sum(c >= 2 for c in counts.values()) == 7


def test_variable_order_rules():
    tc = parse(CORPUS["tc"]).rules[1]
    assert choose_variable_order(tc, 0) == ("x", "y", "z")
    tri = parse(CORPUS["triangle"]).rules[0]
    assert choose_variable_order(tri, None) == ("x", "y", "z")
    plan = compile_instance(tri, None, 3)
    assert plan.atoms[2].column_order == (1, 0) and plan.inner_atom == 2
    validate_plan(plan)


def test_split_rewrite_shapes():
    rewritten = apply_splits(parse(CORPUS["cge_split"]))
    helper = [r for r in rewritten.rules if r.head.relation == "HelpNT"]
    consumer = [r for r in rewritten.rules if r.head.relation == "CallGraphEdge"]
    assert len(helper) == 1 and len(consumer) == 1
    assert [t.value for t in helper[0].head.args] == ["sn", "dsc", "m", "h"]
    assert len(consumer[0].body) == 5 and consumer[0].body[-1].relation == "HelpNT"


def test_wildcards_are_fresh():
    prog = parse(".decl R(a:symbol, b:symbol)\n.decl S(a:symbol)\nS(x) :- R(x, _), R(_, x).\n")
    names = [t.value for a in prog.rules[0].body for t in a.args if t.is_var()]
    assert len(set(names)) == 3


def test_strata_order_and_errors():
    chain = parse(".decl A(x:symbol)\n.decl B(x:symbol)\n.decl C(x:symbol)\n.decl D(x:symbol)\n"
                  "B(x) :- A(x).\nC(x) :- B(x).\nD(x) :- C(x).\n")
    assert [s.rules[0].head.relation for s in stratify(chain.rules)] == ["B", "C", "D"]
    mutual = parse(CORPUS["mutual"])
    assert [sorted(r.index for r in s.rules) for s in stratify(mutual.rules)] == [[0], [1, 2]]
    with pytest.raises(ProgramError, match="not stratifiable"):
        stratify(parse(".decl R(x:symbol)\n.decl S(x:symbol)\nR(x) :- S(x), !R(x).\n").rules)


# --- partitions (paper Fig. 2 and Alg. 1) --------------------------------------


def hist_part(degrees, p, d2=None):
    keys = np.arange(1, len(degrees) + 1, dtype=np.uint32)
    d2 = np.ones(len(degrees), dtype=np.int64) if d2 is None else np.asarray(d2)
    return WorkPartition(keys, np.asarray(degrees), d2, p)


def test_figure_2_partition_exact():
    part = hist_part([4, 9, 1, 4], 4)
    assert part.prefix.tolist() == [4, 13, 14, 18] and part.total == 18
    assert part.bounds == [(0, 5), (5, 10), (10, 15), (15, 18)]
    assert part.kappa == [0, 1, 1, 3]
    assert list(part.spans(0)) == [(0, 0, 4), (1, 0, 1)]
    assert [decode_workunit(u, part)[0] for u in range(5)] == [0, 0, 0, 0, 1]


def test_decode_hand_example_and_bijection():
    part = hist_part([2, 3, 1, 2], 4, d2=[2, 3, 1, 2])
    assert decode_workunit(5, part) == (1, 0, 1)
    assert [decode_workunit(u, part) for u in range(4, 13)] == [(1, a, b) for a in range(3) for b in range(3)]
    with pytest.raises(InternalError):
        decode_workunit(part.total, part)
    rng = np.random.default_rng(42)
    for _ in range(200):
        k = int(rng.integers(1, 65))
        keys = np.sort(rng.choice(10_000, size=k, replace=False)).astype(np.uint32)
        outer = rng.integers(1, 33, size=k)
        d2 = rng.integers(1, 33, size=k)
        part = WorkPartition(keys, outer, d2, p=int(rng.integers(1, 9)))
        units = np.arange(part.total)
        kk, i1, i2 = decode_workunit(units, part)
        assert np.all(i1 < outer[kk]) and np.all(i2 < d2[kk])
        assert np.array_equal(encode_workunit(part, kk, i1, i2), units)


def test_partitions_match_reference(golden):
    for case in golden("partitions.json"):
        part = WorkPartition(np.array(case["keys"], dtype=np.uint32), case["outer"], case["d2"], case["p"])
        assert part.prefix.tolist() == case["prefix"]
        assert part.total == case["total"]
        assert [list(b) for b in part.bounds] == case["bounds"]
        assert part.kappa == case["kappa"]
        assert [[list(s) for s in part.spans(w)] for w in range(case["p"])] == case["spans"]
        got = [list(map(int, decode_workunit(int(u), part))) for u in case["units"]] if part.total else []
        assert got == case["decoded"]
        bound = -(-part.total // part.p) if part.total else 0
        assert max(part.slice_sizes()) <= bound


# --- symbols --------------------------------------------------------------------


def test_interner_contract():
    it = Interner()
    assert [it.intern(c) for c in ("alpha", "beta", "gamma")] == [0, 1, 2]
    assert it.intern("beta") == 1 and it.lookup("zeta") is None
    assert it.intern(17) != it.intern("17") and it.value(it.intern(17)) == 17
    cols = it.intern_rows([("a", "b"), ("b", "a")], 2)
    assert cols[0].dtype == np.uint32


def test_interner_integer_reservation():
    it = Interner()
    it.reserve_ints(100)
    assert it.intern(42) == 42 and it.lookup(99) == 99
    s = it.intern("n0")
    assert s == 100 and it.text(s) == "n0" and it.text(7) == "7"
    with pytest.raises(Exception):
        it.reserve_ints(200)
