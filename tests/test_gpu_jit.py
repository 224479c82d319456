"""Per-rule kernels (csrc/wcoj_jit.cu): the join compiled per plan shape with
NVRTC must give exactly what the generic kernels give — relations, round
counts, and the emitted multiset (one row per binding) — on the reference's
golden fixpoints and random joins, and at scale against the oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle.gj import fixpoint_text  # noqa: E402
from paper_2604_20073_b200 import parse  # noqa: E402
from programs import CORPUS  # noqa: E402


def _prepare_all(sources):
    """Build every plan's kernel up front on the background compiler."""
    from paper_2604_20073_b200 import compile_program
    from paper_2604_20073_b200.wcoj import jit_prepare

    plans = []
    for src in sources:
        cp = compile_program(parse(src))
        plans += [p for st in cp.strata for p in st.plans]
    return jit_prepare(plans, "spec", wait=True) + jit_prepare(plans, "materialize", wait=True)


def test_jit_compiles_for_sm100a_without_gpu_state(jit):
    """NVRTC builds the triangle's kernel; the source names the plan class."""
    import ctypes as C

    from paper_2604_20073_b200 import compile_program, suites
    from paper_2604_20073_b200.wcoj import encode_shape

    plan = compile_program(parse(suites.TRIANGLE_PROGRAM)).strata[-1].plans[0]
    d = encode_shape(plan)
    buf = C.create_string_buffer(1 << 16)
    jit.lib().srdl_wcoj_jit_source(C.byref(d), 2, buf, len(buf))
    assert b"wcoj_body<2, 1, srdl::JitShape>" in buf.value
    nb = C.c_uint64(0)
    assert jit.lib().srdl_wcoj_jit_compile_check(C.byref(d), 2, C.byref(nb)) == 0
    assert nb.value > 10_000


def test_jit_golden_fixpoints(golden, jit):
    from paper_2604_20073_b200 import run_program

    records = golden("fixpoints.json.gz")
    sources = sorted({rec.get("source") or CORPUS[rec["program"]] for rec in records})
    assert _prepare_all(sources) > 0
    before = jit.jit_stats()
    for rec in records:
        src = rec.get("source") or CORPUS[rec["program"]]
        facts = {k: [tuple(r) for r in v] for k, v in rec["facts"].items()}
        engine, summary = run_program(parse(src), facts, schedule="stream")
        for name, rows in rec["relations"].items():
            assert [list(r) for r in engine.relation_rows(name)] == rows, (rec["program"], name)
        assert summary.relations == rec["cardinalities"], rec["program"]
        got = [(s.index, sorted(s.rule_indexes), s.recursive, s.iterations) for s in summary.strata]
        want = [(s["index"], s["rules"], s["recursive"], s["iterations"]) for s in rec["strata"]]
        assert got == want, rec["program"]
    st = jit.jit_stats()
    assert st["failures"] == before["failures"] == 0


def test_jit_golden_joins_emit_one_row_per_binding(golden, jit):
    from paper_2604_20073_b200 import Engine
    from paper_2604_20073_b200.wcoj import execute_plan

    cases = golden("joins.json.gz")[:150]  # 150 distinct plan shapes
    _prepare_all([c["source"] for c in cases])
    for case in cases:
        engine = Engine(parse(case["source"]))
        for name, rows in case["facts"].items():
            engine.load_facts(name, [tuple(r) for r in rows])
        engine.prepare_inputs()
        plan = engine.compiled.strata[-1].plans[0]
        out = execute_plan(plan, engine.store, 3, engine.interner).cpu().numpy()
        rows = sorted({tuple(engine.interner.text(int(v)) for v in out[:, i]) for i in range(out.shape[1])})
        assert [list(r) for r in rows] == case["out"], case["seed"]
        assert out.shape[1] == case["emitted"], case["seed"]


@pytest.mark.parametrize("name", ["tc", "sg", "andersen", "doop"])
def test_jit_matches_generic_kernels_bit_for_bit(name):
    """Same instance, generic kernels vs per-rule kernels: identical
    relations (and identical staged output order: sorted heads arrive sorted
    either way), and both equal the oracle."""
    import torch

    from paper_2604_20073_b200 import Engine
    from paper_2604_20073_b200 import device as dev
    from paper_2604_20073_b200 import suites
    from paper_2604_20073_b200.wcoj import jit_prepare

    facts = {"tc": lambda: suites.tc_random(600, 3_000, seed=5),
             "sg": lambda: suites.sg_layered(levels=20, width=400, seed=5),
             "andersen": lambda: suites.andersen_modular(40_000, seed=5),
             "doop": lambda: suites.doop_modular(20_000, seed=5)}[name]()
    program, out = suites.BASELINE_PROGRAMS[name]
    results = []
    for mode in ("off", "sync"):
        prev = dev.jit_mode(mode)
        try:
            eng = Engine(parse(program), schedule="stream")
            if mode == "sync":
                assert jit_prepare([p for st in eng.compiled.strata for p in st.plans], wait=True) > 0
            for k, v in facts.items():
                eng.load_columns(k, torch.from_numpy(v).cuda())
            s = eng.solve()
            results.append(({r: eng.relation_columns(r).cpu().numpy() for r in s.relations},
                            [x.iterations for x in s.strata]))
        finally:
            dev.jit_mode(prev)
    (a, ia), (b, ib) = results
    assert ia == ib
    for rel in a:
        assert np.array_equal(a[rel], b[rel]), (name, rel)
    from oracle import native
    from oracle.gj import Symbols

    top = max(int(v.max()) for v in facts.values()) + 1
    want, _ = native.fixpoint(parse(program), {k: v.T for k, v in facts.items()}, Symbols(top))
    assert np.array_equal(b[out].T.astype(np.int64), want[out])
