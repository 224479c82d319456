"""Full-size oracle digests of the five BASELINE.json configurations.

    python tests/golden/make_baseline_digests.py [tc triangle sg andersen doop]

For every configuration this generates the EDB on the host with the same
seeded generators the bench uses (`paper_2604_20073_b200.suites`; the R-MAT
graph through `suites.rmat_graph_host`, the bit-exact host mirror of the
device generator), evaluates the program to fixpoint with the multi-core
C++ oracle (`oracle/native.py`, pinned against the reference's golden
fixtures like `oracle/gj.py`), and records for every IDB relation its
cardinality and digest (`oracle/digest.py`: n, sha256 of the sorted
columns, order-independent 64-bit fold) plus the EDB digests, so a GPU test
can check that it evaluated the same inputs. Output:
tests/golden/baseline_digests.json (merged: only the named configs are
recomputed).

Sizes are the BASELINE sizes (the bench's default instances): nothing is
scaled down. Run time on 8 cores: TC ~1 min, triangle ~3 min, the
recursive program-analysis configs longer (see the `oracle_s` field).
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import native  # noqa: E402
from oracle.digest import digest  # noqa: E402
from oracle.gj import Symbols  # noqa: E402
from paper_2604_20073_b200 import parse, suites  # noqa: E402

OUT = os.path.join(HERE, "baseline_digests.json")

# config name -> (generator call as text, generator) — the bench instances
CONFIGS = {
    "tc": ("suites.tc_random(10_000, 50_000, seed=1)", lambda: suites.tc_random(10_000, 50_000, seed=1)),
    "triangle": ("R=S=T=suites.rmat_graph_host(20, 16_000_000, seed=1)",
                 lambda: (lambda e: {"R": e, "S": e, "T": e})(suites.rmat_graph_host(20, 16_000_000, seed=1))),
    "sg": ("suites.sg_layered(levels=128, width=31_250, seed=0)",
           lambda: suites.sg_layered(levels=128, width=31_250, seed=0)),
    "andersen": ("suites.andersen_modular(10_000_000, seed=1)", lambda: suites.andersen_modular(10_000_000, seed=1)),
    "doop": ("suites.doop_modular(6_900_000, seed=1)", lambda: suites.doop_modular(6_900_000, seed=1)),
}


def compute(name: str) -> dict:
    program, output = suites.BASELINE_PROGRAMS[name]
    prog = parse(program)
    call, gen = CONFIGS[name]
    t0 = time.time()
    facts = gen()
    t_gen = time.time() - t0
    top = max(int(v.max()) for v in facts.values() if v.size) + 1
    solver = native.Solver(prog, {}, Symbols(top))
    for k, v in facts.items():
        solver.load_columns(k, v)
    t0 = time.time()
    solver.solve()
    t_solve = time.time() - t0
    edb = {}
    for k, v in facts.items():
        edb[k] = digest(solver.rows_u32(k).T)
    idb = {}
    for rel in sorted(prog.declarations):
        if rel in facts:
            continue
        idb[rel] = digest(solver.rows_u32(rel).T)
    rounds = [r for _, rec, r in solver.report() if rec]
    solver.close()
    return {
        "program_output": output,
        "generator": call,
        "edb": edb,
        "idb": idb,
        "recursive_rounds": rounds,
        "oracle": "oracle/native.py (C++ generic join + semi-naive loop, pinned by tests/test_oracle_golden.py)",
        "oracle_threads": native.lib().og_set_threads(0),
        "generate_s": round(t_gen, 1),
        "oracle_s": round(t_solve, 1),
    }


def main(argv):
    names = argv or list(CONFIGS)
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    for name in names:
        rec = compute(name)
        data[name] = rec
        print(name, json.dumps({k: v for k, v in rec.items() if k not in ("edb",)}), flush=True)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
