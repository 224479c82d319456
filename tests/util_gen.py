"""Seeded instance generators for the tests (same distributions as the
reference test helpers, reference: pkg/tests/util.py:85-241)."""

from __future__ import annotations

import random


def random_graph(rng: random.Random, n_nodes: int, n_edges: int, prefix: str = "n") -> list:
    names = [f"{prefix}{i}" for i in range(n_nodes)]
    out = set()
    tries = 0
    while len(out) < n_edges and tries < n_edges * 20:
        tries += 1
        a, b = rng.randrange(n_nodes), rng.randrange(n_nodes)
        if a != b:
            out.add((names[a], names[b]))
    return sorted(out)


def random_forest(rng: random.Random, target_edges: int, max_width=6, max_depth=4, prefix="f") -> list:
    edges = []
    serial = 0
    while len(edges) < target_edges:
        frontier = [f"{prefix}{serial}"]
        serial += 1
        for _ in range(rng.randint(2, max_depth)):
            nxt = []
            for _ in range(rng.randint(1, max_width)):
                node = f"{prefix}{serial}"
                serial += 1
                edges.append((rng.choice(frontier), node))
                nxt.append(node)
            frontier = nxt
    return sorted(set(edges))


def random_andersen(rng: random.Random, statements: int) -> dict:
    vs = [f"v{i}" for i in range(max(statements // 3, 4))]
    hs = [f"h{i}" for i in range(max(statements // 5, 3))]
    facts = {"AddressOf": set(), "Assign": set(), "Load": set(), "Store": set()}
    for _ in range(statements):
        kind = rng.randrange(4)
        if kind == 0:
            facts["AddressOf"].add((rng.choice(vs), rng.choice(hs)))
        elif kind == 1:
            facts["Assign"].add((rng.choice(vs), rng.choice(vs)))
        elif kind == 2:
            facts["Load"].add((rng.choice(vs), rng.choice(vs)))
        else:
            facts["Store"].add((rng.choice(vs), rng.choice(vs)))
    return {k: sorted(v) for k, v in facts.items()}


def fractured_stratum_case(n_rules=12, seed=5, n_nodes=14, edges_per_rel=20):
    """One SCC of n_rules mutually recursive rules A_i :- A_{i+1}, B_i."""
    rng = random.Random(seed)
    lines, facts = [], {}
    for i in range(n_rules):
        lines.append(f".decl A{i}(a:symbol, b:symbol)")
        lines.append(f".decl B{i}(a:symbol, b:symbol)")
        facts[f"B{i}"] = random_graph(rng, n_nodes, edges_per_rel)
    lines.append(".decl Seed(a:symbol, b:symbol)")
    facts["Seed"] = random_graph(rng, n_nodes, edges_per_rel)
    lines += [f".input B{i}" for i in range(n_rules)] + [".input Seed"]
    lines += [f".output A{i}" for i in range(n_rules)]
    lines += [f"A{i}(x, y) :- A{(i + 1) % n_rules}(x, z), B{i}(z, y)." for i in range(n_rules)]
    lines.append("A0(x, y) :- Seed(x, y).")
    return "\n".join(lines) + "\n", facts
