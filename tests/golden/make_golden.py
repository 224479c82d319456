"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package (pkg/src/flatlog) and the reference test
generators (pkg/tests/util.py) read-only, evaluates seeded instances, and
writes compact JSON fixtures next to this script. Nothing under tests/ or the
package imports the reference at run time; the GPU box only sees the
committed fixtures.

Fixtures:
  plans.json        compiled plan structure for a corpus of programs
  partitions.json   WorkPartition prefix/bounds/kappa/spans/decode samples
  storage.json      sort_dedup / compute_delta / merge(head, body) / histogram
  merges.json.gz    1000 merge sequences (the acceptance suite's criterion 7)
  fixpoints.json.gz seeded fixpoints: facts, every relation's rows, strata
  joins.json.gz     random multi-way joins (reference random_join_case)
  errors.json       program texts and the ProgramError message they raise
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import util as ref_util  # noqa: E402
from flatlog import parse, rowops  # noqa: E402
from flatlog.bench import SUITES  # noqa: E402
from flatlog.errors import ProgramError  # noqa: E402
from flatlog.executor import WorkPartition, decode_workunit, execute_plan  # noqa: E402
from flatlog.oracle import naive_fixpoint  # noqa: E402
from flatlog.planner import compile_program  # noqa: E402
from flatlog.runtime import run_program  # noqa: E402
from flatlog.storage import ColumnarRelation, Histogram, compute_delta, sort_dedup  # noqa: E402

# ---------------------------------------------------------------------------
# program corpus (sources are plain Datalog text, shared with tests/programs.py)

sys.path.insert(0, os.path.dirname(HERE))
from programs import CORPUS  # noqa: E402


def dump(name, obj, gz=False):
    path = os.path.join(HERE, name)
    data = json.dumps(obj, separators=(",", ":"), sort_keys=True).encode()
    if gz:
        with gzip.GzipFile(path, "wb", mtime=0) as fh:
            fh.write(data)
    else:
        with open(path, "wb") as fh:
            fh.write(data)
    print(f"wrote {name}: {len(data)} bytes raw")


def plan_record(plan):
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


def gen_plans():
    out = {}
    for name, src in CORPUS.items():
        # anonymous variable names depend on a process-global counter; they
        # are normalised by the consumer, so record them as-is
        prog = compile_program(parse(src))
        out[name] = {
            "strata": [
                {
                    "index": s.index,
                    "rules": [r.index for r in s.rules],
                    "recursive": s.recursive,
                    "plans": [plan_record(p) for p in s.plans],
                }
                for s in prog.strata
            ],
            "orders": {k: sorted(list(o) for o in v) for k, v in prog.orders.items()},
            "declarations": prog.declarations,
            "rules": [str(r) for r in prog.program.rules],
        }
    dump("plans.json", out)


def gen_partitions():
    rng = np.random.default_rng(7)
    cases = []
    for _ in range(120):
        k = int(rng.integers(0, 40))
        keys = np.sort(rng.choice(100_000, size=k, replace=False)).astype(np.uint32)
        outer = rng.integers(1, 40, size=k)
        d2 = rng.integers(1, 12, size=k)
        p = int(rng.integers(1, 12))
        part = WorkPartition(keys, outer, d2, p)
        units = rng.integers(0, max(part.total, 1), size=min(part.total, 50))
        dec = [list(map(int, decode_workunit(int(u), part))) for u in units] if part.total else []
        cases.append(
            {
                "keys": keys.tolist(),
                "outer": outer.tolist(),
                "d2": d2.tolist(),
                "p": p,
                "prefix": part.prefix.tolist(),
                "total": part.total,
                "bounds": [list(b) for b in part.bounds],
                "kappa": part.kappa,
                "spans": [[list(s) for s in part.spans(w)] for w in range(p)],
                "units": units.tolist(),
                "decoded": dec,
            }
        )
    dump("partitions.json", cases)


def gen_storage():
    rng = random.Random(99)
    out = {"sort_dedup": [], "compute_delta": [], "merge": []}
    for _ in range(60):
        arity = rng.randint(1, 4)
        rows = [tuple(rng.randrange(30) for _ in range(arity)) for _ in range(rng.randrange(300))]
        order = tuple(rng.sample(range(arity), arity))
        cols = rowops.from_tuples(rows, arity)
        res = sort_dedup(cols, order)
        out["sort_dedup"].append(
            {"arity": arity, "rows": rows, "order": list(order), "out": rowops.as_tuples(res)}
        )
    for _ in range(60):
        arity = rng.randint(1, 3)
        full = sorted({tuple(rng.randrange(12) for _ in range(arity)) for _ in range(rng.randrange(200))})
        head = []
        rel = ColumnarRelation.from_sorted(arity, tuple(range(arity)), rowops.from_tuples(full, arity))
        if full and rng.random() < 0.5:  # put a few rows into the head buffer
            extra = sorted({tuple(rng.randrange(12, 20) for _ in range(arity)) for _ in range(5)})
            rel = rel.merge_delta(rowops.from_tuples(extra, arity), flush_limit=4096)
            head = extra
        new = [tuple(rng.randrange(20) for _ in range(arity)) for _ in range(rng.randrange(250))]
        got = compute_delta(rowops.from_tuples(new, arity), rel)
        out["compute_delta"].append(
            {"arity": arity, "body": full, "head": head, "new": new, "out": rowops.as_tuples(got)}
        )
    for _ in range(80):
        arity = rng.randint(1, 3)
        flush = rng.choice([0, 3, 16, 4096])
        order = tuple(rng.sample(range(arity), arity))
        rel = ColumnarRelation.empty(arity, order)
        have = set()
        steps = []
        for _ in range(rng.randint(1, 7)):
            batch = {tuple(rng.randrange(25) for _ in range(arity)) for _ in range(rng.randrange(60))}
            fresh = sorted(tuple(r[a] for a in order) for r in batch)
            fresh = [r for r in fresh if r not in have]
            have.update(fresh)
            rel = rel.merge_delta(rowops.from_tuples(fresh, arity), flush_limit=flush)
            steps.append(
                {
                    "delta": fresh,
                    "head": rowops.as_tuples(rel.head),
                    "body": rowops.as_tuples(rel.body),
                    "hist_keys": rel.hist.keys.tolist(),
                    "hist_degrees": rel.hist.degrees.tolist(),
                    "hist_prefix": rel.hist.prefix.tolist(),
                }
            )
        out["merge"].append({"arity": arity, "flush": flush, "order": list(order), "steps": steps})
    hists = []
    for _ in range(40):
        h = Histogram.empty()
        seq = []
        for _ in range(rng.randrange(6)):
            delta = sorted(rng.randrange(10) for _ in range(rng.randrange(12)))
            h = h.updated(np.array(delta, dtype=np.uint32))
            seq.append({"delta": delta, "keys": h.keys.tolist(), "degrees": h.degrees.tolist(), "prefix": h.prefix.tolist()})
        hists.append(seq)
    out["histogram"] = hists
    dump("storage.json", out)


def gen_merges():
    """1000 random merge sequences (pkg/tests/test_acceptance.py:325-357,
    criterion 7: arity 1-3, flush 0 / 3 / 4096, 2-6 batches of up to 40 rows
    over 25 values): head, body and histogram after every merge."""
    rng = random.Random(99)
    seqs = []
    while len(seqs) < 1000:
        arity = rng.randint(1, 3)
        flush = rng.choice([0, 3, 4096])
        order = tuple(rng.sample(range(arity), arity))
        rel = ColumnarRelation.empty(arity, order)
        contents = set()
        steps = []
        for _ in range(rng.randint(2, 6)):
            batch = {tuple(rng.randrange(25) for _ in range(arity)) for _ in range(rng.randrange(40))}
            ordered = sorted(tuple(row[a] for a in order) for row in batch)
            fresh = [row for row in ordered if row not in contents]
            contents.update(fresh)
            rel = rel.merge_delta(rowops.from_tuples(fresh, arity), flush_limit=flush)
            rel.check_invariants()
            steps.append({
                "delta": fresh,
                "head": rowops.as_tuples(rel.head),
                "body": rowops.as_tuples(rel.body),
                "hist_keys": rel.hist.keys.tolist(),
                "hist_degrees": rel.hist.degrees.tolist(),
                "hist_prefix": rel.hist.prefix.tolist(),
            })
        seqs.append({"arity": arity, "flush": flush, "order": list(order), "steps": steps})
    dump("merges.json.gz", seqs, gz=True)


def relation_dump(engine, program):
    return {name: [list(r) for r in engine.relation_rows(name)] for name in program.declarations}


def fixpoint_record(name, src, facts, **kw):
    program = parse(src)
    engine, summary = run_program(program, facts, **kw)
    expected, rounds = naive_fixpoint(program, facts)
    got = {n: set(engine.relation_rows(n)) for n in program.declarations}
    assert got == expected, name
    if not program.splits:  # the naive oracle runs the unsplit rules
        assert summary.rounds_by_rules() == rounds, name
    return {
        "program": name,
        "facts": {k: [list(r) for r in v] for k, v in facts.items()},
        "relations": relation_dump(engine, engine.compiled.program),
        "cardinalities": summary.relations,
        "strata": [
            {"index": s.index, "rules": sorted(s.rule_indexes), "recursive": s.recursive, "iterations": s.iterations}
            for s in summary.strata
        ],
    }


def gen_fixpoints():
    records = []
    # 100 instances per program, as the reference acceptance suite runs
    # (pkg/tests/test_acceptance.py:145-178; its seeds are hash((kind, i)),
    # randomised per process, so ours are f"{kind}-{i}" over the same shapes)
    for kind, count in (("tc", 100), ("sg", 100), ("andersen", 100), ("negation", 100)):
        for index in range(count):
            rng = random.Random(f"{kind}-{index}")
            if kind == "tc":
                facts = {"Edge": ref_util.random_graph(rng, rng.randint(8, 40), rng.randint(10, 90))}
                src = CORPUS["tc"]
            elif kind == "sg":
                facts = {"Edge": ref_util.random_forest(rng, rng.randint(14, 80))}
                src = CORPUS["sg"]
            elif kind == "andersen":
                facts = ref_util.random_andersen(rng, rng.randint(14, 120))
                src = CORPUS["andersen"]
            else:
                facts = {"Edge": ref_util.random_graph(rng, rng.randint(6, 20), rng.randint(8, 40))}
                src = CORPUS["negation"]
            records.append(fixpoint_record(kind, src, facts))
    # reference benchmark suites at tiny/small scales
    for suite in ("tc", "sg", "triangle", "star", "neg2hop", "andersen"):
        for scale, seed in (("tiny", 0), ("tiny", 1), ("small", 2)):
            src, facts = SUITES[suite](scale, seed)
            rec = fixpoint_record(f"suite-{suite}", src, facts)
            rec["source"] = src
            records.append(rec)
    # larger single instances
    rng = random.Random(77)
    records.append(fixpoint_record("sg", CORPUS["sg"], {"Edge": ref_util.random_forest(rng, 500)}))
    rng = random.Random(12)
    records.append(fixpoint_record("andersen", CORPUS["andersen"], ref_util.random_andersen(rng, 200)))
    # negation probe shapes (reference tests/test_runtime.py WILDCARD_NEG_SOURCE)
    for probe in ("!W(x, _)", "!W(_, y)", "!W(_, _)", '!W("v0", "v1")', "!W(x, y)"):
        rng = random.Random(3)
        vals = [f"v{i}" for i in range(8)]
        facts = {
            "R": sorted({(rng.choice(vals),) for _ in range(6)}),
            "T": sorted({(rng.choice(vals), rng.choice(vals)) for _ in range(14)}),
            "U": sorted({(rng.choice(vals), rng.choice(vals)) for _ in range(14)}),
            "W": sorted({(rng.choice(vals), rng.choice(vals)) for _ in range(5)}),
        }
        src = CORPUS["wildcard_neg"].replace("!W(x, _)", probe)
        rec = fixpoint_record("wildcard_neg", src, facts)
        rec["source"] = src
        records.append(rec)
    # fractured 12-rule stratum and the split soundness fixture
    prog, facts = ref_util.fractured_stratum_case(n_rules=12, seed=17)
    src = "\n".join(
        [f".decl {n}({', '.join(f'c{i}:symbol' for i in range(a))})" for n, a in prog.declarations.items()]
        + [f".input {n}" for n in prog.inputs]
        + [f".output {n}" for n in prog.outputs]
        + [str(r) for r in prog.rules]
    )
    rec = fixpoint_record("fractured", src, facts)
    rec["source"] = src
    records.append(rec)
    for split in (False, True):
        rng = random.Random(1234)
        facts = cge_facts(rng, 40)
        src = CORPUS["cge_split" if split else "cge"]
        records.append(fixpoint_record("cge_split" if split else "cge", src, facts))
    for name in ("ground", "zero_var", "repeated_var", "copy_rules", "mutual", "chain_neg"):
        rng = random.Random(name)
        facts = small_facts_for(name, rng)
        records.append(fixpoint_record(name, CORPUS[name], facts))
    dump("fixpoints.json.gz", records, gz=True)


def cge_facts(rng, scale):
    methods = [f"m{i}" for i in range(scale)] + ["main"]
    insts = [f"i{i}" for i in range(scale * 4)]
    bases = [f"b{i}" for i in range(scale)]
    heaps = [f"h{i}" for i in range(scale * 2)]
    types = [f"t{i}" for i in range(max(scale // 3, 2))]
    sigs = [f"s{i}" for i in range(scale)]
    dscs = [f"d{i}" for i in range(3)]
    pick = rng.choice
    return {
        "InstructionMethod": sorted({(pick(insts), pick(methods)) for _ in range(scale * 6)}),
        "VirtualCall": sorted({(pick(insts), pick(bases), pick(sigs), pick(dscs)) for _ in range(scale * 6)}),
        "VarPointsTo": sorted({(pick(heaps), pick(bases)) for _ in range(scale * 5)}),
        "HeapType": sorted({(h, pick(types)) for h in heaps}),
        "MethodLookup": sorted({(pick(sigs), pick(dscs), pick(types), pick(methods)) for _ in range(scale * 4)}),
    }


def small_facts_for(name, rng):
    vals = [f"c{i}" for i in range(9)]
    two = lambda n: sorted({(rng.choice(vals), rng.choice(vals)) for _ in range(n)})  # noqa: E731
    if name == "ground":
        return {}
    if name == "zero_var":
        return {"R": [("k",), ("z",)]}
    if name == "repeated_var":
        return {"R": two(30)}
    if name == "copy_rules":
        return {"A": [(v,) for v in vals[:5]]}
    if name == "mutual":
        return {"S": [(v,) for v in vals[:4]], "E": two(12)}
    if name == "chain_neg":
        return {"E": two(20), "Block": [(v,) for v in vals[:3]]}
    raise KeyError(name)


def gen_joins():
    cases = []
    # 500 joins at p in {1, 2, 8}, as pkg/tests/test_acceptance.py:84-103
    for case in range(500):
        program, facts, head_vars = ref_util.random_join_case(seed=20_000 + case)
        engine = ref_util.seeded_engine(program, facts)
        plan = ref_util.plan_for_head(engine, "Out")
        emitted = {}
        for p in (1, 2, 8):
            out = execute_plan(plan, engine.store, p, engine.interner)
            emitted[p] = sorted(tuple(int(c[i]) for c in out) for i in range(len(out[0])))
        assert emitted[1] == emitted[2] == emitted[8], case
        rows = sorted({tuple(engine.interner.text(int(c[i])) for c in out) for i in range(len(out[0]))})
        src = "\n".join(
            [f".decl {n}({', '.join(f'c{i}:symbol' for i in range(a))})" for n, a in program.declarations.items()]
            + [f".input {n}" for n in program.inputs]
            + [f".output {n}" for n in program.outputs]
            + [str(r) for r in program.rules]
        )
        cases.append(
            {
                "seed": 20_000 + case,
                "source": src,
                "facts": {k: [list(r) for r in v] for k, v in facts.items()},
                "out": [list(r) for r in rows],
                "emitted": len(out[0]),
                "ps": [1, 2, 8],
            }
        )
    dump("joins.json.gz", cases, gz=True)


ERROR_CASES = [
    ".decl R(a:symbol)\n.decl S(a:symbol)\nR(x) :- S(y).\n",
    ".decl R(a:symbol)\nR(x).\n",
    ".decl R(a:symbol)\n.decl S(a:symbol)\n.decl T(a:symbol)\nT(x) :- R(x), !S(y).\n",
    ".decl R(a:symbol, b:symbol)\n.decl S(a:symbol)\nS(x) :- R(x).\n",
    ".decl S(a:symbol)\nS(x) :- R(x).\n",
    ".decl R(a:symbol)\nR(x :- .\n",
    ".decl R(a:symbol)\nR(x) :- .\n",
    ".decl R(a:symbol)\n.decl R(b:symbol)\n",
    ".foo R\n",
    ".decl R(a:symbol)\n.output Q\n",
    ".decl R(a:symbol)\n!R(\"a\") :- R(\"b\").\n",
    ".decl R(a:symbol)\nR(\"a) .\n",
    ".decl R(a:symbol)\nR(\"a\") $ .\n",
    ".decl R(x:symbol)\n.decl S(x:symbol)\nR(x) :- S(x), !R(x).\n",
    ".decl P(x:symbol)\n.decl Q(x:symbol)\n.decl S(x:symbol)\nP(x) :- S(x), !Q(x).\nQ(x) :- P(x).\n",
    ".decl R(a:symbol)\n.decl S(a:symbol)\n.decl T(a:symbol, b:symbol)\nlbl: T(x, y) :- R(x), S(y).\n.split lbl { S(y) } -> H(y)\n",
    ".decl R(a:symbol, b:symbol)\n.decl S(a:symbol, b:symbol)\n.decl T(a:symbol, b:symbol)\nlbl: T(x, z) :- R(x, y), S(y, z).\n.split lbl { S(z, y) } -> H(y)\n",
    ".decl R(a:symbol, b:symbol)\n.decl S(a:symbol, b:symbol)\n.decl T(a:symbol, b:symbol)\nlbl: T(x, z) :- R(x, y), S(y, z).\n.split lbl { S(y, z) } -> H(z)\n",
    ".decl E(a:symbol, b:symbol)\n.decl T(a:symbol, b:symbol)\nT(x, y) :- E(x, y).\nlbl: T(x, z) :- T(x, y), E(y, z).\n.split lbl { T(x, y) } -> H(x, y)\n",
    ".decl R(a:symbol, b:symbol)\n.decl S(a:symbol, b:symbol)\n.decl T(a:symbol, b:symbol)\nlbl: T(x, z) :- R(x, y), S(y, z).\n.split nope { S(y, z) } -> H(y, z)\n",
    ".decl R(a:symbol, b:symbol)\n.decl S(a:symbol, b:symbol)\n.decl T(a:symbol, b:symbol)\nlbl: T(x, z) :- R(x, y), S(y, z).\n.split lbl { S(y, z) } -> R(y, z)\n",
    ".decl R(a:symbol, b:symbol)\n.split lbl { !R(y, z) } -> H(y, z)\n",
]


def gen_errors():
    out = []
    for src in ERROR_CASES:
        try:
            compile_program(parse(src))
        except ProgramError as exc:
            out.append({"source": src, "error": str(exc), "line": exc.line, "col": exc.col})
        else:
            raise AssertionError(f"no error for {src!r}")
    dump("errors.json", out)


if __name__ == "__main__":
    gen_plans()
    gen_partitions()
    gen_storage()
    gen_merges()
    gen_errors()
    gen_joins()
    gen_fixpoints()
