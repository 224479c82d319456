"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

Before the oracle is trusted as the parity checker for the GPU path, it must
reproduce every fixture the reference produced: fixpoints (relations and
semi-naive round counts), random multi-way joins, and the storage
operations (sort/dedup, compute_delta, head/body merges, histograms).
"""

import numpy as np

from oracle import storage as ost
from oracle.gj import Symbols, fixpoint_text, join_rule
from paper_2604_20073_b200 import parse
from programs import CORPUS


def test_oracle_fixpoints_match_reference(golden):
    records = golden("fixpoints.json.gz")
    assert len(records) > 100
    for rec in records:
        prog = parse(rec.get("source") or CORPUS[rec["program"]])
        facts = {k: [tuple(r) for r in v] for k, v in rec["facts"].items()}
        rels, report = fixpoint_text(prog, facts)
        for name, rows in rec["relations"].items():
            if name in rels:  # split helpers exist only in the rewritten program
                assert [list(r) for r in rels[name]] == rows, (rec["program"], name)
        if not prog.splits:
            got = sorted((sorted(m), r, n) for m, r, n in report)
            want = sorted((s["rules"], s["recursive"], s["iterations"]) for s in rec["strata"])
            assert got == want, rec["program"]


def test_oracle_joins_match_reference(golden):
    for case in golden("joins.json.gz"):
        prog = parse(case["source"])
        sym = Symbols()
        rels = {k: sym.rows_to_ids(v, prog.declarations[k]) for k, v in case["facts"].items()}
        rule = prog.rules[0]
        rows = join_rule(rule, lambda p: ost.sort_dedup(rels[rule.body[p].relation]),
                         lambda c, create=False: sym.intern(c) if create else sym.lookup(c))
        got = sorted({tuple(sym.text(v) for v in r) for r in rows.tolist()})
        assert [list(r) for r in got] == case["out"], case["seed"]
        # every binding is emitted exactly once (head = all variables)
        assert len(rows) == case["emitted"], case["seed"]


def test_oracle_storage_matches_reference(golden):
    st = golden("storage.json")
    for case in st["sort_dedup"]:
        rows = ost.as_rows(case["rows"], case["arity"])
        got = ost.sort_dedup_order(rows, case["order"])
        assert got.tolist() == case["out"]
    for case in st["compute_delta"]:
        a = case["arity"]
        got = ost.compute_delta(ost.as_rows(case["new"], a), ost.as_rows(case["head"], a),
                                ost.as_rows(case["body"], a))
        assert got.tolist() == case["out"]
    for case in st["merge"]:
        rel = ost.HeadBody(case["arity"], case["flush"])
        for step in case["steps"]:
            rel.merge_delta(ost.as_rows(step["delta"], case["arity"]))
            assert rel.head.tolist() == step["head"]
            assert rel.body.tolist() == step["body"]
            assert rel.hist.keys.tolist() == step["hist_keys"]
            assert rel.hist.degrees.tolist() == step["hist_degrees"]
            assert rel.hist.prefix.tolist() == step["hist_prefix"]
    for seq in st["histogram"]:
        h = ost.Histogram([], [])
        for step in seq:
            h = h.updated(np.array(step["delta"], dtype=np.int64))
            assert h.keys.tolist() == step["keys"]
            assert h.degrees.tolist() == step["degrees"]
            assert h.prefix.tolist() == step["prefix"]
