"""End-to-end parity of the device fixpoint engine with the reference.

* every golden fixpoint record (relations bit-exact as sorted tuple sets,
  semi-naive round counts) under both schedules;
* every golden random multi-way join through execute_plan (output multiset
  = one row per binding);
* audit invariants (count == materialize per slice, write-once coverage,
  auxiliary storage == count total);
* larger seeded instances against the numpy oracle, and the integer-column
  loading path.
"""

import random

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle.gj import Symbols, fixpoint, fixpoint_text  # noqa: E402
from paper_2604_20073_b200 import parse  # noqa: E402
from programs import CORPUS  # noqa: E402


def run(source, facts, **kw):
    from paper_2604_20073_b200 import run_program

    return run_program(parse(source), facts, **kw)


@pytest.mark.parametrize("schedule,general", [("seq", "0"), ("stream", "0"), ("stream", "1")])
def test_golden_fixpoints(golden, schedule, general, monkeypatch):
    # general=1: every plan through the general kernel instance instead of
    # the depth-specialised ones (csrc/wcoj_launch.cuh plan_kind)
    monkeypatch.setenv("SRDL_WCOJ_GENERAL", general)
    records = golden("fixpoints.json.gz")
    for rec in records:
        src = rec.get("source") or CORPUS[rec["program"]]
        facts = {k: [tuple(r) for r in v] for k, v in rec["facts"].items()}
        engine, summary = run(src, facts, schedule=schedule)
        for name, rows in rec["relations"].items():
            got = [list(r) for r in engine.relation_rows(name)]
            assert got == rows, (rec["program"], name, schedule)
        assert summary.relations == rec["cardinalities"], rec["program"]
        got_strata = [(s.index, sorted(s.rule_indexes), s.recursive, s.iterations) for s in summary.strata]
        want = [(s["index"], s["rules"], s["recursive"], s["iterations"]) for s in rec["strata"]]
        assert got_strata == want, rec["program"]


def test_golden_joins_through_execute_plan(golden, audited):
    from paper_2604_20073_b200 import Engine
    from paper_2604_20073_b200.wcoj import execute_plan

    for case in golden("joins.json.gz"):
        prog = parse(case["source"])
        engine = Engine(prog)
        for name, rows in case["facts"].items():
            engine.load_facts(name, [tuple(r) for r in rows])
        engine.prepare_inputs()
        plan = engine.compiled.strata[-1].plans[0]
        assert plan.head_relation == "Out"
        emitted = None
        for p in case.get("ps", [3]):  # the reference runs p in {1, 2, 8}
            out = execute_plan(plan, engine.store, p, engine.interner)
            host = out.cpu().numpy()
            rows = sorted({tuple(engine.interner.text(int(v)) for v in host[:, i]) for i in range(host.shape[1])})
            assert [list(r) for r in rows] == case["out"], case["seed"]
            assert host.shape[1] == case["emitted"], case["seed"]
            # the emitted multiset does not depend on p (pkg/tests/test_acceptance.py:96-100)
            multiset = sorted(map(tuple, host.T.tolist()))
            assert emitted is None or multiset == emitted, (case["seed"], p)
            emitted = multiset
    assert len(audited.traces) >= 1500
    for t in audited.traces:
        assert t.tc_total == t.total
        assert t.bitmap_ok is not False
        assert t.aux_peak == t.total
        if t.work_total >= t.p:
            assert t.max_slice <= -(-t.work_total // t.p)


def test_audited_fixpoints_keep_storage_invariants(audited):
    rng = random.Random(4)
    from util_gen import random_graph

    for _ in range(5):
        edges = random_graph(rng, 30, 80)
        engine, _ = run(CORPUS["tc"], {"Edge": edges}, head_threshold=8)
        want, _ = fixpoint_text(parse(CORPUS["tc"]), {"Edge": edges})
        assert engine.relation_rows("TC") == want["TC"]
    assert audited.traces and all(t.bitmap_ok for t in audited.traces if t.total)


def _oracle_ids(source, edb, reserve):
    sym = Symbols(reserve)
    rels, report = fixpoint(parse(source), edb, sym)
    return rels, report


@pytest.mark.parametrize("schedule", ["seq", "stream"])
def test_tc_integer_columns_vs_oracle(schedule):
    from paper_2604_20073_b200 import Engine

    rng = np.random.default_rng(3)
    n, m = 3000, 6000
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    edges = np.unique(np.stack([src, dst], 1), axis=0)
    prog = parse(CORPUS["tc"])
    engine = Engine(prog, schedule=schedule)
    engine.load_columns("Edge", edges.T.copy())
    summary = engine.solve()
    got = engine.relation_columns("TC").cpu().numpy().astype(np.int64).T
    want, report = _oracle_ids(CORPUS["tc"], {"Edge": edges}, n)
    assert np.array_equal(got, want["TC"])
    assert sorted(summary.rounds_by_rules().values()) == sorted(r for _, _, r in report)


def test_sg_and_andersen_larger_vs_oracle():
    from util_gen import random_andersen, random_forest

    rng = random.Random(21)
    edges = random_forest(rng, 4000, max_width=8, max_depth=5)
    engine, summary = run(CORPUS["sg"], {"Edge": edges}, schedule="stream")
    want, report = fixpoint_text(parse(CORPUS["sg"]), {"Edge": edges})
    assert engine.relation_rows("SG") == want["SG"]
    assert sorted(summary.rounds_by_rules().values()) == sorted(r for _, _, r in report)

    facts = random_andersen(random.Random(8), 1200)
    engine, summary = run(CORPUS["andersen"], facts, schedule="stream", head_threshold=64)
    want, report = fixpoint_text(parse(CORPUS["andersen"]), facts)
    assert engine.relation_rows("PointsTo") == want["PointsTo"]
    assert sorted(summary.rounds_by_rules().values()) == sorted(r for _, _, r in report)


def test_triangle_skewed_vs_oracle():
    from paper_2604_20073_b200 import Engine

    rng = np.random.default_rng(9)
    n = 2000
    a = (rng.zipf(1.6, 40000) % n)
    b = rng.integers(0, n, 40000)
    edges = np.unique(np.stack([np.concatenate([a, b]), np.concatenate([b, a])], 1), axis=0)
    edges = edges[edges[:, 0] != edges[:, 1]]
    prog = parse(CORPUS["triangle"])
    engine = Engine(prog, schedule="stream")
    for rel in ("R", "S", "T"):
        engine.load_columns(rel, edges.T.copy())
    engine.solve()
    got = engine.relation_columns("Triangle").cpu().numpy().astype(np.int64).T
    want, _ = _oracle_ids(CORPUS["triangle"], {r: edges for r in ("R", "S", "T")}, n)
    assert np.array_equal(got, want["Triangle"])


def test_schedules_and_thresholds_agree():
    from util_gen import fractured_stratum_case

    prog_src, facts = fractured_stratum_case(n_rules=12, seed=3)
    results = []
    for schedule, thr in (("seq", 4096), ("stream", 0), ("stream", 7)):
        engine, summary = run(prog_src, facts, schedule=schedule, head_threshold=thr)
        results.append(({n: engine.relation_rows(n) for n in engine.compiled.declarations},
                         summary.rounds_by_rules()))
    assert results[0] == results[1] == results[2]


def test_max_iterations_watchdog():
    from paper_2604_20073_b200.faults import InternalError

    edges = [(f"n{i}", f"n{i + 1}") for i in range(12)]
    engine, summary = run(CORPUS["tc"], {"Edge": edges}, max_iterations=100)
    assert summary.relations["TC"] == 78
    with pytest.raises(InternalError):
        run(CORPUS["tc"], {"Edge": edges}, max_iterations=3)


@pytest.mark.parametrize("suite", ["tc", "sg", "triangle", "star", "neg2hop", "andersen"])
def test_reference_suites_verified(suite):
    from paper_2604_20073_b200.suites import run_suite

    def check(program, facts):
        return fixpoint_text(program, facts)[0]

    for schedule in ("seq", "stream"):
        report = run_suite(suite, "small", 3, schedule=schedule, verify=check)
        assert report["verified"] is True
        assert report["phase_micros"].get("count", 0) > 0


def test_dense_offsets_match_histogram():
    from paper_2604_20073_b200 import device as dev
    from paper_2604_20073_b200.columns import Histogram

    rng = np.random.default_rng(2)
    col = np.sort(rng.integers(0, 5000, 200_000)).astype(np.uint32)
    h = Histogram.over_column(col)
    off = dev.dense_offsets(h.keys, h.prefix, 6000).cpu().numpy().astype(np.int64)
    want = np.searchsorted(col, np.arange(6001), side="left")
    assert np.array_equal(off, want)


HASH_PROGRAM = """
.decl Base(a:symbol, b:symbol)
.decl E(a:symbol, b:symbol)
.decl R(a:symbol, b:symbol)
.decl K(a:symbol, b:symbol, c:symbol)
.decl Tri(a:symbol, b:symbol, c:symbol)
.decl Open(a:symbol, b:symbol, c:symbol)
R(x, z) :- Base(x, z).
R(x, z) :- R(x, y), E(y, z).
K(x, y, z) :- R(x, y), E(y, z), R(x, z).
Tri(x, y, z) :- E(x, y), E(y, z), E(z, x).
Open(x, y, z) :- E(x, y), E(y, z), R(x, z), !E(x, z).
"""


@pytest.mark.parametrize("general", ["0", "1"])
@pytest.mark.parametrize("threshold", [0, 100000])
def test_root_invariant_leaf_sources_vs_oracle(monkeypatch, general, threshold):
    """Leaf sources fixed by the root (R(x, z), E(z, x), the negated E(x, z))
    next to per-parent ones, with R flushed every iteration (threshold 0) or
    kept with a head segment; depth-specialised and general kernel."""
    from paper_2604_20073_b200 import Engine

    monkeypatch.setenv("SRDL_WCOJ_GENERAL", general)
    rng = np.random.default_rng(12)
    n = 400
    a = rng.zipf(1.5, 5000) % n
    b = rng.integers(0, n, 5000)
    e = np.unique(np.stack([a, b], 1), axis=0)
    e = e[e[:, 0] != e[:, 1]]
    base = e[np.isin(e[:, 0], np.arange(0, n, 13))]
    facts = {"E": e, "Base": base}
    engine = Engine(parse(HASH_PROGRAM), schedule="stream", head_threshold=threshold)
    for rel, rows in facts.items():
        engine.load_columns(rel, rows.T.copy())
    engine.solve()
    want, _ = _oracle_ids(HASH_PROGRAM, facts, n)
    for rel in ("R", "K", "Tri", "Open"):
        got = engine.relation_columns(rel).cpu().numpy().astype(np.int64).T
        assert np.array_equal(got, want[rel]), rel


SPARSE_PROGRAM = """
.decl A(a:symbol, b:symbol)
.decl B(a:symbol, b:symbol)
.decl C(a:symbol)
.decl Q(a:symbol, b:symbol)
.decl Tri(a:symbol, b:symbol, c:symbol)
Q(x, z) :- A(x, y), B(y, z), C(z).
Tri(x, y, z) :- A(x, y), B(y, z), A(z, x).
"""


def test_sparse_ids_two_level_histogram_search():
    """Ids spread over 2^23 so no dense CSR offsets are built: every
    column-0 lookup goes through the index histogram's fence keys and one
    64-key block (csrc/wcoj_kernel.cuh hist_range); results vs the oracle."""
    from paper_2604_20073_b200 import Engine

    rng = np.random.default_rng(5)
    top = 1 << 23
    hubs = rng.integers(0, top, 3000)
    a = np.unique(np.stack([rng.choice(hubs, 40000), rng.choice(hubs, 40000)], 1), axis=0)
    b = np.unique(np.stack([rng.choice(hubs, 40000), rng.integers(0, top, 40000)], 1), axis=0)
    c = np.unique(np.concatenate([b[::3, 1], rng.integers(0, top, 2000)]))[:, None]
    facts = {"A": a, "B": b, "C": c}
    engine = Engine(parse(SPARSE_PROGRAM), schedule="stream")
    for rel, rows in facts.items():
        engine.load_columns(rel, rows.T.copy())
    engine.solve()
    want, _ = _oracle_ids(SPARSE_PROGRAM, facts, top)
    for rel in ("Q", "Tri"):
        got = engine.relation_columns(rel).cpu().numpy().astype(np.int64).T
        assert len(want[rel]) > 0, rel
        assert np.array_equal(got, want[rel]), rel


@pytest.mark.parametrize("program", ["sg", "andersen", "doop"])
def test_batched_and_synchronous_delta_paths_agree(program):
    """Without stats the engine launches every head relation's delta and
    delta indexes before one size readback each (fixpoint._deltas_batched);
    with stats it keeps the per-relation synchronous path. Same fixpoint."""
    from paper_2604_20073_b200 import Engine, Stats, suites

    facts = {"sg": lambda: suites.sg_layered(levels=10, width=400, seed=2),
             "andersen": lambda: suites.andersen_modular(6000, seed=3),
             "doop": lambda: suites.doop_modular(4096, seed=4)}[program]()
    src = suites.BASELINE_PROGRAMS[program][0]
    results = []
    for stats in (None, Stats()):
        engine = Engine(parse(src), schedule="stream", stats=stats, head_threshold=64)
        for rel, cols in facts.items():
            engine.load_columns(rel, cols)
        summary = engine.solve()
        results.append(({r: engine.relation_columns(r).cpu().numpy() for r in engine.compiled.declarations},
                        summary.rounds_by_rules()))
        if stats is not None:
            # the stream schedule records every join phase per plan, as the
            # reference does (runtime.py:225-257)
            plan_ids = {p.plan_id for st in engine.compiled.strata for p in st.plans}
            rows = [r for r in stats.records if r["phase"] in ("histogram", "count", "materialize")]
            assert rows and all(r["rule"] in plan_ids for r in rows)
            assert {r["phase"] for r in rows} == {"histogram", "count", "materialize"}
    (a, ra), (b, rb) = results
    assert ra == rb
    for r in a:
        assert np.array_equal(a[r], b[r]), r


def test_sparse_ids_recursive_fence_search():
    """Andersen with its ids scattered over 2^23: the full PointsTo index is
    probed at a non-root level while it is being derived, so it gets no dense
    offsets and every lookup goes through the histogram fence keys; the EDB
    indexes (static in that stratum) get dense offsets. Vs the oracle."""
    from paper_2604_20073_b200 import Engine, suites

    facts = suites.andersen_modular(8000, seed=6)
    top = 1 << 23
    ids = np.unique(np.concatenate([v.reshape(-1) for v in facts.values()]))
    rng = np.random.default_rng(1)
    remap = np.zeros(int(ids.max()) + 1, dtype=np.int64)
    remap[ids] = rng.choice(top, size=len(ids), replace=False)
    sparse = {k: remap[v.astype(np.int64)].astype(np.uint32) for k, v in facts.items()}
    engine = Engine(parse(suites.ANDERSEN_PROGRAM), schedule="stream")
    for rel, cols in sparse.items():
        engine.load_columns(rel, cols)
    engine.solve()
    want, _ = _oracle_ids(suites.ANDERSEN_PROGRAM, {k: v.T.astype(np.int64) for k, v in sparse.items()}, top)
    got = engine.relation_columns("PointsTo").cpu().numpy().astype(np.int64).T
    assert len(want["PointsTo"]) > 1000
    assert np.array_equal(got, want["PointsTo"])


@pytest.mark.parametrize("spec_bytes", ["0", "20000", "3000000"])
@pytest.mark.parametrize("program", ["triangle", "andersen", "doop"])
def test_speculative_count_and_spills_match(monkeypatch, program, spec_bytes):
    """The count walk writes its tuples into a bounded arena and materialize
    gathers them (srdl_wcoj_count_spec / srdl_wcoj_gather); slices that do
    not fit are walked again (srdl_wcoj_materialize_spilled). No arena (0),
    an arena that spills almost everything (20 KB) and a partial one must all
    give the oracle's fixpoint."""
    from paper_2604_20073_b200 import Engine, suites

    monkeypatch.setenv("SRDL_SPEC_BYTES", spec_bytes)
    if program == "triangle":
        rng = np.random.default_rng(3)
        n = 1500
        a = rng.zipf(1.5, 30000) % n
        b = rng.integers(0, n, 30000)
        e = np.unique(np.stack([a, b], 1), axis=0)
        e = e[e[:, 0] != e[:, 1]]
        facts = {"R": e.T.astype(np.uint32), "S": e.T.astype(np.uint32), "T": e.T.astype(np.uint32)}
    elif program == "andersen":
        facts = suites.andersen_modular(6000, seed=9)
    else:
        facts = suites.doop_modular(4096, seed=5)
    src, out = suites.BASELINE_PROGRAMS[program]
    engine = Engine(parse(src), schedule="stream")
    for rel, cols in facts.items():
        engine.load_columns(rel, cols)
    engine.solve()
    edb = {k: v.T.astype(np.int64) for k, v in facts.items()}
    top = max(int(v.max()) for v in edb.values() if v.size) + 1
    want, _ = _oracle_ids(src, edb, top)
    got = engine.relation_columns(out).cpu().numpy().astype(np.int64).T
    assert len(want[out]) > 100
    assert np.array_equal(got, want[out])


@pytest.mark.parametrize("program", ["tc", "sg", "andersen", "doop"])
def test_hashed_compute_delta_vs_oracle(program, monkeypatch):
    """Compute Delta through the device hash set of the full relation
    (csrc/hashset.cu) on every iteration (thresholds lowered to 0), against
    the oracle: the set is built, probed, grown and kept in step with every
    merged delta."""
    from oracle import native
    from paper_2604_20073_b200 import Engine, suites
    from paper_2604_20073_b200.fixpoint import Engine as E

    monkeypatch.setattr(E, "HASH_MIN_FULL", 0)
    monkeypatch.setattr(E, "HASH_MIN_STAGED", 0)
    facts = {"tc": lambda: suites.tc_random(700, 3_500, seed=9),
             "sg": lambda: suites.sg_layered(levels=16, width=500, seed=9),
             "andersen": lambda: suites.andersen_modular(30_000, seed=9),
             "doop": lambda: suites.doop_modular(12_000, seed=9)}[program]()
    src, out = suites.BASELINE_PROGRAMS[program]
    eng = Engine(parse(src), schedule="stream")
    for rel, cols in facts.items():
        eng.load_columns(rel, torch.from_numpy(cols).cuda())
    summary = eng.solve()
    top = max(int(v.max()) for v in facts.values()) + 1
    want, rep = native.fixpoint(parse(src), {k: v.T for k, v in facts.items()}, Symbols(top))
    for rel in parse(src).declarations:
        got = eng.relation_columns(rel).cpu().numpy().astype(np.int64).T
        assert np.array_equal(got, want[rel]), (program, rel)
    if not parse(src).splits:
        assert sorted(summary.rounds_by_rules().values()) == sorted(r for _, _, r in rep)
