"""Bit-exact parity at the BASELINE sizes (north star: "bit-exact fixpoint
relations on all five configs").

Each test evaluates one BASELINE configuration at its full size on the
device and reduces every IDB relation (and the EDB it loaded) to the digest
of `oracle/digest.py` — cardinality, sha256 of the sorted columns and an
order-independent 64-bit fold — which must equal the digest the C++ oracle
computed for the same instance (tests/golden/baseline_digests.json, made by
tests/golden/make_baseline_digests.py; the oracle is pinned by the
reference's goldens in tests/test_oracle_golden.py). Zero mismatches, as in
the reference's acceptance suite (pkg/tests/test_acceptance.py:276-283).

Also: the device R-MAT generator against its host mirror bit for bit, and
the triangle's heaviest root keys (where one key is split across many
slices and the merge-path leaves run) row by row against the oracle.
"""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle.digest import digest  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DIGESTS = os.path.join(HERE, "golden", "baseline_digests.json")


def _digests():
    with open(DIGESTS) as fh:
        return json.load(fh)


def _facts(name):
    import bench

    return bench.make_workload(name)


def test_rmat_device_generator_matches_host_mirror():
    from paper_2604_20073_b200 import device as dev
    from paper_2604_20073_b200 import suites

    for scale, n, seed in ((20, 1 << 22, 1), (12, 100_003, 7)):
        got = dev.gen_rmat(scale, n, seed=seed).cpu().numpy()
        want = suites.rmat_host(scale, n, seed=seed)
        assert np.array_equal(got, want), (scale, n, seed)


@pytest.mark.parametrize("kernels", ["per-rule", "generic"])
@pytest.mark.parametrize("name", ["tc", "triangle", "sg", "andersen", "doop"])
def test_baseline_config_full_size_digest(name, kernels):
    """kernels: "per-rule" = the NVRTC-compiled kernel of every plan (the
    production path, built before the solve), "generic" = the plan-class
    kernels compiled into libsrdl.so."""
    from paper_2604_20073_b200 import Engine, parse
    from paper_2604_20073_b200 import device as dev
    from paper_2604_20073_b200.fixpoint import release_arenas

    want = _digests().get(name)
    if want is None:
        pytest.fail(f"no committed oracle digest for {name}: run tests/golden/make_baseline_digests.py {name}")
    wl = _facts(name)
    prev = dev.jit_mode("async" if kernels == "per-rule" else "off")
    try:
        eng = Engine(parse(wl.program), schedule="stream")  # schedules the per-rule kernels
        if kernels == "per-rule":
            dev.jit_wait()
            dev.jit_mode("sync")  # anything not built yet (materialize re-walks) compiles on first use
        for k, v in wl.device_facts().items():
            eng.load_columns(k, v)
        summary = eng.solve()
        for rel, d in want["edb"].items():
            assert digest(eng.relation_columns(rel).cpu().numpy()) == d, (name, "EDB", rel)
        for rel, d in want["idb"].items():
            assert summary.relations[rel] == d["n"], (name, rel)
            got = digest(eng.relation_columns(rel).cpu().numpy())
            assert got == d, (name, rel)
        rounds = [s.iterations for s in summary.strata if s.recursive]
        if want.get("recursive_rounds") and not parse(wl.program).splits:
            assert sorted(rounds) == sorted(want["recursive_rounds"]), name
        del eng
        torch.cuda.synchronize()
        release_arenas()
        if kernels == "per-rule":
            assert dev.jit_stats()["failures"] == 0
    finally:
        dev.jit_mode(prev)


def test_triangle_heaviest_root_keys_row_exact():
    """The 64 heaviest root keys by outer x d2 work (the keys that are split
    across the most slices) plus 64 random ones: the device rows equal the
    oracle's rows for exactly those keys."""
    from oracle import native
    from oracle.gj import Symbols
    from paper_2604_20073_b200 import Engine, parse, suites

    e = suites.rmat_graph_host(20, 16_000_000, seed=1)
    out_deg = np.bincount(e[0], minlength=1 << 20).astype(np.int64)
    in_deg = np.bincount(e[1], minlength=1 << 20).astype(np.int64)
    work = out_deg * in_deg  # outer R(x, .) rows x inner T(., x) rows
    heavy = np.argsort(-work)[:64]
    rng = np.random.default_rng(3)
    light = rng.choice(np.nonzero(out_deg)[0], 64, replace=False)
    keys = np.unique(np.concatenate([heavy, light])).astype(np.uint32)
    prog = parse(suites.TRIANGLE_PROGRAM)
    facts = {"R": e.T, "S": e.T, "T": e.T}
    want = native.Solver(prog, facts, Symbols(1 << 20), keep_level0=keys).solve().rows_u32("Triangle")
    eng = Engine(prog, schedule="stream")
    et = torch.from_numpy(e).cuda()
    for r in ("R", "S", "T"):
        eng.load_columns(r, et)
    eng.solve()
    rows = eng.relation_columns("Triangle")
    sel = torch.isin(rows[0].view(torch.int32), torch.from_numpy(keys.view(np.int32)).cuda())
    got = rows.view(torch.int32)[:, sel].cpu().numpy().view(np.uint32).T
    assert len(want) > 1_000_000
    assert np.array_equal(got, want)
