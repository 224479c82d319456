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
    for case in st["merge"] + golden("merges.json.gz"):
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


def test_native_oracle_fixpoints_match_reference(golden):
    """The multi-core C++ oracle (oracle/native.py, used for the full-size
    BASELINE digests and the CPU baseline) against the same reference
    fixtures: relations and semi-naive round counts."""
    from oracle import native

    records = golden("fixpoints.json.gz")
    for rec in records:
        prog = parse(rec.get("source") or CORPUS[rec["program"]])
        facts = {k: [tuple(r) for r in v] for k, v in rec["facts"].items()}
        rels, report = native.fixpoint_text(prog, facts, threads=2)
        for name, rows in rec["relations"].items():
            if name in rels:
                assert [list(r) for r in rels[name]] == rows, (rec["program"], name)
        if not prog.splits:
            got = sorted((sorted(m), r, n) for m, r, n in report)
            want = sorted((s["rules"], s["recursive"], s["iterations"]) for s in rec["strata"])
            assert got == want, rec["program"]


def test_native_oracle_joins_match_reference(golden):
    """Random multi-way joins (single-rule programs): the C++ oracle's head
    relation equals the reference's join output set."""
    from oracle import native

    for case in golden("joins.json.gz"):
        prog = parse(case["source"])
        rels, _ = native.fixpoint_text(prog, {k: [tuple(r) for r in v] for k, v in case["facts"].items()},
                                       threads=3)
        head = prog.rules[0].head.relation
        assert [list(r) for r in rels[head]] == case["out"], case["seed"]


def test_native_oracle_matches_numpy_oracle_at_scale():
    """The two oracle restatements agree on larger integer instances (the
    sizes the goldens cannot reach): TC, SG, Andersen and DOOP-shaped."""
    from oracle import native
    from oracle.gj import fixpoint
    from paper_2604_20073_b200 import suites

    cases = [
        ("tc", suites.tc_random(400, 1_600, seed=3)),
        ("sg", suites.sg_layered(levels=12, width=300, seed=2)),
        ("andersen", suites.andersen_modular(6_000, seed=2)),
        ("doop", suites.doop_modular(4_096, seed=2)),
        ("triangle", (lambda e: {"R": e, "S": e, "T": e})(suites.rmat_graph_host(10, 6_000, seed=2))),
    ]
    for name, facts in cases:
        prog = parse(suites.BASELINE_PROGRAMS[name][0])
        edb = {k: v.T.astype(np.int64) for k, v in facts.items()}
        top = max(int(v.max()) for v in edb.values() if v.size) + 1
        want, rep_w = fixpoint(prog, edb, Symbols(top))
        got, rep_g = native.fixpoint(prog, edb, Symbols(top), threads=4)
        for rel in prog.declarations:
            assert np.array_equal(got[rel], want[rel]), (name, rel)
        assert rep_w == rep_g, name


def test_native_oracle_level0_sample_is_a_restriction():
    """keep_level0 (bounded CPU samples) yields exactly the rows of the
    sampled root keys."""
    from oracle import native
    from paper_2604_20073_b200 import suites

    e = suites.rmat_graph_host(11, 20_000, seed=4)
    prog = parse(suites.TRIANGLE_PROGRAM)
    facts = {"R": e.T, "S": e.T, "T": e.T}
    full = native.Solver(prog, facts, Symbols(1 << 11)).solve().rows_u32("Triangle")
    keys = np.unique(e[0])[::7]
    part = native.Solver(prog, facts, Symbols(1 << 11), keep_level0=keys).solve().rows_u32("Triangle")
    assert len(part) and np.array_equal(part, full[np.isin(full[:, 0], keys)])


def test_digest_streaming_and_order_checks():
    from oracle.digest import Digester, digest

    rng = np.random.default_rng(5)
    rows = np.unique(rng.integers(0, 1 << 20, size=(5000, 3)), axis=0).T.astype(np.uint32)
    whole = digest(rows)
    d = Digester(3)
    for lo in range(0, rows.shape[1], 777):
        d.update(rows[:, lo:lo + 777])
    assert d.result() == whole
    assert whole["n"] == rows.shape[1]
    # a different relation changes both witnesses
    other = digest(rows[:, 1:])
    assert other["sha256"] != whole["sha256"] and other["fold64"] != whole["fold64"]
    import pytest

    with pytest.raises(ValueError):
        digest(rows[:, ::-1])


def test_rmat_host_mirror_shape_and_determinism():
    """The host R-MAT mirror is deterministic and in range (bit-exactness
    against the device generator is a -m gpu test)."""
    from paper_2604_20073_b200 import suites

    a = suites.rmat_host(12, 10_000, seed=7)
    b = suites.rmat_host(12, 10_000, seed=7, chunk=999)
    assert a.dtype == np.uint32 and a.shape == (2, 10_000)
    assert np.array_equal(a, b)
    assert a.max() < (1 << 12)
    # R-MAT skew: the most popular source is far above the mean degree
    deg = np.bincount(a[0], minlength=1 << 12)
    assert deg.max() > 20 * deg.mean()
