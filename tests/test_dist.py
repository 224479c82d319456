"""Multi-process path (dist.py): exchange primitives and placement rules on
CPU with gloo at world size 2, and the full distributed fixpoint on one GPU
with two ranks (gloo, collectives staged through host memory)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from paper_2604_20073_b200 import compile_program, parse
from paper_2604_20073_b200 import device as dev
from paper_2604_20073_b200.dist import PART, REP, DistContext, index_modes
from programs import CORPUS


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _free_gpu():
    """The ranks share this process's GPU: hand back the engine arenas, pools
    and torch's cached blocks that earlier tests in this process hold."""
    if torch.cuda.is_available() and torch.cuda.is_initialized():
        import gc

        from paper_2604_20073_b200 import fixpoint

        gc.collect()
        fixpoint.release_arenas()
        torch.cuda.empty_cache()


def _spawn(fn, world, *args):
    _free_gpu()
    port = _free_port()
    mp.spawn(fn, args=(world, port, *args), nprocs=world, join=True)


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)


def _exchange_worker(rank, world, port):
    _init(rank, world, port)
    try:
        ctx = DistContext()
        rng = np.random.default_rng(rank)
        rows = rng.integers(0, 1000, size=(3, 50 + 7 * rank)).astype(np.uint32)
        own = dev.owner(rows[0], world).astype(np.int64)
        order = np.argsort(own, kind="stable")
        counts = np.bincount(own, minlength=world).tolist()
        t = torch.from_numpy(rows[:, order].copy())
        got = ctx.all_to_all_rows(t, counts).numpy()
        # every received row is owned by this rank, and the union is exact
        assert np.all(dev.owner(got[0], world) == rank)
        allrows = ctx.all_gather_rows(torch.from_numpy(rows)).numpy()
        mine_all = allrows[:, dev.owner(allrows[0], world) == rank]
        assert sorted(map(tuple, got.T.tolist())) == sorted(map(tuple, mine_all.T.tolist()))
        assert ctx.all_sum(rank + 1) == world * (world + 1) // 2
    finally:
        td.destroy_process_group()


def test_exchange_primitives_gloo_world2():
    _spawn(_exchange_worker, 2)


def test_owner_hash_spreads_keys():
    keys = np.arange(100_000)
    for world in (2, 4, 8):
        counts = np.bincount(dev.owner(keys, world).astype(np.int64), minlength=world)
        assert counts.min() > 0.8 * counts.mean()


def test_index_placement_rules():
    modes = index_modes(compile_program(parse(CORPUS["tc"])))
    assert modes[("TC", (0, 1))] == PART  # only the dedup authority / delta reads it
    assert modes[("Edge", (0, 1))] == REP  # Edge(y, z) is read below the root
    tri = index_modes(compile_program(parse(CORPUS["triangle"])))
    assert tri[("R", (0, 1))] == PART and tri[("T", (1, 0))] == PART and tri[("S", (0, 1))] == REP
    neg = index_modes(compile_program(parse(CORPUS["negation"])))
    # the constant-led probe TC("n0", x) is a full read after a constant column
    assert neg[("TC", (0, 1))] == REP


# --------------------------------------------------------------- GPU, 2 ranks


def _fixpoint_worker(rank, world, port, name, source, facts, out_path):
    _init(rank, world, port)
    try:
        from paper_2604_20073_b200 import Engine

        torch.cuda.set_device(0)
        eng = Engine(parse(source), schedule="stream", dist=DistContext())
        for rel, cols in facts.items():
            eng.load_columns(rel, cols)
        summary = eng.solve()
        ctx = eng.dist
        sent = torch.tensor([ctx.sent_bytes, ctx.exchanges], dtype=torch.int64)
        td.all_reduce(sent, op=td.ReduceOp.MAX)
        result = {rel: eng.relation_columns(rel).cpu().numpy() for rel in eng.compiled.declarations}
        if rank == 0:
            np.savez(out_path, **result, _rounds=np.array(sorted(summary.rounds_by_rules().values())),
                     _sent=sent.numpy())
    finally:
        td.destroy_process_group()


def _single(source, facts):
    from paper_2604_20073_b200 import Engine

    eng = Engine(parse(source), schedule="stream")
    for rel, cols in facts.items():
        eng.load_columns(rel, cols)
    summary = eng.solve()
    return ({rel: eng.relation_columns(rel).cpu().numpy() for rel in eng.compiled.declarations},
            sorted(summary.rounds_by_rules().values()))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tc", "sg", "triangle", "andersen", "negation", "doop"])
def test_two_ranks_match_single_gpu(name, tmp_path):
    from paper_2604_20073_b200 import suites

    rng = np.random.default_rng(4)
    if name in ("tc", "negation"):
        e = np.unique(rng.integers(0, 400, size=(1500, 2)), axis=0).T.astype(np.uint32)
        facts = {"Edge": e}
    elif name == "sg":
        facts = suites.sg_layered(levels=12, width=300, seed=1)
    elif name == "triangle":
        e = np.unique(rng.integers(0, 300, size=(4000, 2)), axis=0).T.astype(np.uint32)
        facts = {"R": e, "S": e, "T": e}
    elif name == "andersen":
        facts = suites.andersen_modular(3000, seed=2)
    else:
        facts = suites.doop_micro(methods=150, types=6, sigs=12, fields=40, seed=3)
    source = {"andersen": suites.ANDERSEN_PROGRAM, "sg": suites.SG_PROGRAM,
              "doop": suites.DOOP_PROGRAM + suites.DOOP_SPLIT}.get(name) or CORPUS[name]
    want, rounds = _single(source, facts)
    out = tmp_path / "dist.npz"
    _spawn(_fixpoint_worker, 2, name, source, facts, str(out))
    got = np.load(out)
    for rel, rows in want.items():
        assert np.array_equal(got[rel], rows), (name, rel)
    assert got["_rounds"].tolist() == rounds


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_doop_200k_methods_ranks_match_single_gpu(world, tmp_path):
    """configs[4]'s generator at 200K methods (~2.9M facts): the distributed
    engine at 2 and 4 ranks (sharing one GPU, gloo) equals the single-GPU
    fixpoint bit for bit; prints the largest per-rank exchange volume."""
    from paper_2604_20073_b200 import suites

    facts = suites.doop_modular(200_000, seed=1)
    source = suites.DOOP_PROGRAM + suites.DOOP_SPLIT
    want, rounds = _single(source, facts)
    out = tmp_path / "dist.npz"
    _spawn(_fixpoint_worker, world, "doop200k", source, facts, str(out))
    got = np.load(out)
    for rel, rows in want.items():
        assert np.array_equal(got[rel], rows), rel
    assert got["_rounds"].tolist() == rounds
    sent, exchanges = got["_sent"].tolist()
    iters = max(rounds)
    print(f"\nDOOP 200K methods, {world} ranks: max per-rank payload sent {sent / 1e6:.1f} MB over "
          f"{iters} iterations ({sent / iters / 1e6:.2f} MB/iteration, {exchanges} exchanges)")


@pytest.mark.gpu
def test_bench_two_ranks_gloo_one_gpu():
    """bench.py's multi-rank path (torchrun, max-over-ranks timing, the
    distributed engine, parity of the gathered output) with two ranks
    sharing one GPU over gloo: TC (configs[0]) matches its committed digest."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    _free_gpu()
    env = dict(os.environ, SRDL_DIST_BACKEND="gloo", SRDL_BENCH_NO_CLOCKS="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--workload",
                          "tc", "--steps", "1", "--warmup", "3", "--profile-steps", "1", "--gpus", "2"],
                         cwd=root, env=env, capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["parity"]["match"] is True
    assert line["config"]["derived_tuples"] == 98_644_628
