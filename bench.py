#!/usr/bin/env python
"""Fixpoint benchmark on B200 (BASELINE.json: "fixpoint wall-time (s) and
derived tuples/sec at 1/2/4/8 B200 vs CPU ref").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME]
                    [--impl ours|reference]

A step is one complete evaluation through the public API: build an Engine
for the workload's program, load its EDB columns, solve to fixpoint. The
metric is derived tuples per second = |output IDB relation| / step time,
aggregated over all ranks. Default workload = BASELINE configs[4], the
DOOP-shaped points-to rule set on ~100M facts (the config the metric's
1/2/4/8-GPU scaling is quoted on); `--workload tc|triangle|sg|andersen`
selects configs[0..3].

value    inputs already resident in HBM when the timed region starts.
e2e      same step through the public API with pinned HOST inputs: the H2D
         copy of the EDB columns and the D2H read of the output relation are
         inside the timed region.
roofline the dominant library call family of the step (every libsrdl call is
         bracketed by CUDA events on its launching stream, dev.PROFILE):
         algorithmic bytes / duration vs the measured HBM copy bandwidth
         (MEASURED_PEAKS.json); all families are listed beside it.
cpu_baseline
         the multi-core C++ restatement of the reference algorithm
         (oracle/native.py, pinned by the reference's goldens) on this box's
         host cores, on a bounded sample of the same workload.
parity   the device output relation (and the EDB) reduced to a digest and
         compared with the oracle's digest of the same full-size instance
         (tests/golden/baseline_digests.json, tests/golden/make_baseline_digests.py).
--impl reference
         the same C++ oracle port on all host cores, each step a bounded
         sample of the workload sized so the whole run ends within minutes.

Multi-GPU (torchrun): every rank loads the EDB; root keys are hash-partitioned
(dist.owner) inside the engine, recursive strata exchange new tuples with
an NCCL all-to-all per iteration plus an all-reduce of delta sizes. Timing
is the max over ranks.
"""

from __future__ import annotations

import os

# Multi-GB buffers (derived relations, the speculative arena) are allocated
# and freed every fixpoint; expandable segments let torch's caching allocator
# grow and reuse them without fresh cudaMalloc calls of that size, which
# otherwise stall some steps by hundreds of ms. Recommended for any process
# running the engine.
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

import argparse  # noqa: E402
import gc  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIGESTS = os.path.join(ROOT, "tests", "golden", "baseline_digests.json")


# --------------------------------------------------------------------------
# workloads (BASELINE.json configs), all generated from seeds


class Workload:
    """One BASELINE configuration. `host_facts(scale)` is the numpy
    generator (scale 1.0 = the BASELINE size; smaller scales are the CPU
    samples of recursive configs); `device_facts()` puts the full instance
    in HBM."""

    def __init__(self, name, index, desc, program, output, gen, sample_kind):
        self.name, self.index, self.desc = name, index, desc
        self.program, self.output = program, output
        self._gen = gen  # scale -> {relation: (arity, n) uint32}
        self.sample_kind = sample_kind  # "roots" (level-0 key subset) or "instance" (scaled generator)
        self.config = {"workload": f"{desc} (configs[{index}])", "program_output": output}

    def host_facts(self, scale=1.0):
        return self._gen(scale)

    def device_facts(self):
        import torch

        from paper_2604_20073_b200 import device as dev

        if self.name == "triangle":  # the device generator (bit-exact with suites.rmat_host: -m gpu test)
            raw = dev.gen_rmat(20, 16_000_000, seed=1).view(torch.int32)
            raw = raw[:, raw[0] != raw[1]].contiguous().view(torch.uint32)
            e = dev.sort_dedup(raw, 20)
            return {"R": e, "S": e, "T": e}
        return {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev.device()) for k, v in self.host_facts().items()}


def _workloads():
    from paper_2604_20073_b200 import suites

    def tri(scale):
        e = suites.rmat_graph_host(20, 16_000_000, seed=1)
        return {"R": e, "S": e, "T": e}

    P = suites.BASELINE_PROGRAMS
    return {
        "tc": Workload("tc", 0, "transitive closure on a random digraph, 10K nodes / 50K edges", *P["tc"],
                       lambda s: suites.tc_random(10_000, 50_000, seed=1), "roots"),
        "triangle": Workload("triangle", 1, "triangle listing (cyclic 3-way WCOJ) on R-MAT scale 20, 16M "
                             "generated edges (self loops dropped, deduplicated)", *P["triangle"], tri, "roots"),
        "sg": Workload("sg", 2, "same generation on a layered tree-plus-cross-edges graph, 128 levels x 31250 "
                       "nodes, ~4.3M edges", *P["sg"],
                       lambda s: suites.sg_layered(levels=128, width=max(64, int(31_250 * s)), seed=0),
                       "instance"),
        "andersen": Workload("andersen", 3, "Andersen points-to over modular synthetic programs, 10M "
                             "statements", *P["andersen"],
                             lambda s: suites.andersen_modular(max(4_000, int(10_000_000 * s)), seed=1),
                             "instance"),
        "doop": Workload("doop", 4, "DOOP-shaped context-insensitive points-to (5-way virtual dispatch, helper "
                         "split HelpNT) over modular synthetic Java-like facts, 6.9M methods, ~100M EDB facts",
                         *P["doop"], lambda s: suites.doop_modular(max(4_096, int(6_900_000 * s)), seed=1),
                         "instance"),
    }


def make_workload(name) -> Workload:
    return _workloads()[name]


# --------------------------------------------------------------------------
# measurement helpers


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, enabled=True):
        self.index = index
        self.enabled = enabled
        self.proc = None
        self.lines = []

    def __enter__(self):
        if not self.enabled:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
            # let nvidia-smi finish initialising (its NVML start-up competes
            # with the first timed step otherwise): wait for its first sample
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.05)
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": mx,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def flush_l2(buf):
    buf.add_(1)  # 512 MiB write > 126 MB L2


def profile_traffic(workload_name, family):
    """DRAM bytes (read + write) per call of `family` from the committed ncu
    --set full capture (profiles/traffic.json, tools/traffic_summary.py)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        d = json.load(fh)
    return (d.get(workload_name) or {}).get(family)


def profile_issue(workload_name, family, live_launch_ms, launches_per_step):
    """Issue-rate roofline of a latency-bound family (the WCOJ walk moves a
    few hundred GB/s of algorithmic bytes: HBM is not what bounds it): warp
    instructions per launch from the committed `ncu --set full` capture
    (profiles/r02/issue.json, tools/ncu_summary.py --json) against the SM
    issue peak, 148 SMs x 4 schedulers x 1 warp instruction per cycle at the
    maximum SM clock. When the step has one launch of the family, the live
    launch time gives the achieved rate; otherwise the capture's own."""
    path = os.path.join(ROOT, "profiles", "r02", "issue.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        d = (json.load(fh).get(workload_name) or {}).get(family)
    if not d:
        return None
    mhz = 1965.0
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        with open(pk) as fh:
            mhz = float(json.load(fh).get("sm_max_mhz", mhz))
    peak = 148 * 4 * mhz * 1e6 / 1e9  # G warp instructions / s
    live = launches_per_step == 1 and live_launch_ms
    ms = live_launch_ms if live else d["duration_ms"]
    achieved = d["inst_executed"] / (ms * 1e-3) / 1e9
    return {"bound": "issue", "unit": "G warp-inst/s", "achieved": round(achieved, 1), "peak": round(peak, 1),
            "frac": round(achieved / peak, 4), "inst_per_launch": d["inst_executed"],
            "time_source": "live launch time (CUDA events)" if live else "ncu duration of the captured launches",
            "ncu_issue_active_pct": d.get("issue_active_pct"), "source": d.get("source")}


# --------------------------------------------------------------------------
# our arm


def local_device() -> int:
    """This rank's GPU (LOCAL_RANK; ranks share devices round-robin when
    there are fewer GPUs than ranks, the gloo test mode)."""
    import torch

    return int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count())


def run_step(torch, Engine, parse, wl, inputs, host=False, out_pinned=None, ctx=None):
    engine = Engine(parse(wl.program), schedule="stream", dist=ctx)
    for rel, t in inputs.items():
        engine.load_columns(rel, t)
    summary = engine.solve()
    n_out = summary.relations[wl.output]
    if host:
        rows = engine.relation_columns(wl.output)
        dst = out_pinned[:, : rows.shape[1]] if out_pinned is not None else None
        if dst is not None and dst.shape == rows.shape:
            dst.copy_(rows, non_blocking=True)
        else:
            rows.cpu()
        torch.cuda.current_stream().synchronize()
    del engine
    return n_out, summary


def family_roofline(records, steps, step_s, wl_name):
    """Per libsrdl call family: event time (on the launching stream) and
    algorithmic bytes; the roofline line is the family with the largest
    time. Families: wcoj_count (speculative count walk), wcoj_gather,
    wcoj_materialize, compute_delta, sort_dedup (delta re-sort per index
    order), merge, histogram, root_work, is_sorted."""
    fam = {}
    for name, a, b, nbytes in records:
        t, n, by = fam.get(name, (0.0, 0, 0))
        fam[name] = (t + a.elapsed_time(b) / 1e3, n + 1, by + nbytes)
    if not fam:
        return None
    name = max(fam, key=lambda k: fam[k][0])
    t, n, by = fam[name]
    peak, src = measured_peaks()
    achieved = by / t / 1e9 if t > 0 else 0.0
    issue = profile_issue(wl_name, name, t / n * 1e3, n / steps)
    return {
        "bound": "hbm",
        "kernel": name,
        "achieved": round(achieved, 2),
        "peak": peak,
        "peak_source": src,
        "unit": "GB/s",
        "frac": round(achieved / peak, 4),
        "traffic": profile_traffic(wl_name, name),
        "algorithmic_bytes_per_launch": int(by / n),
        "algorithmic_bytes_model": {
            "wcoj_count": "4 B x columns x rows of every index segment the plan reads, once; + 4 B x head "
                          "arity per derived tuple written (into the speculative arena)",
            "wcoj_gather": "2 x 4 B x head arity per derived tuple (arena read, output write)",
            "compute_delta": "4 B x arity x (staged rows read once + delta rows written once)",
            "sort_dedup": "4 B x arity x (rows read once + rows written once)",
            "merge": "4 B x arity x (both inputs read once + output written once)",
        }.get(name, "input read once + output written once"),
        "launch_ms": round(t / n * 1e3, 4),
        "launches_per_step": n / steps,
        "kernel_share_of_step": round(t / steps / step_s, 4),
        "families_ms_per_step": {k: round(v[0] / steps * 1e3, 3) for k, v in
                                 sorted(fam.items(), key=lambda kv: -kv[1][0])},
        "families_gbs": {k: round(v[2] / v[0] / 1e9, 1) for k, v in fam.items() if v[0] > 0},
        "issue_roofline": issue,
        "note": "family = one libsrdl C-ABI call (one or more kernels); times are CUDA events on the "
                "launching stream, so families on concurrent streams overlap and shares can sum past 1",
    }


def bench_ours(args, rank, world, dist):
    import torch

    from paper_2604_20073_b200 import Engine, parse
    from paper_2604_20073_b200 import device as dev

    torch.cuda.set_device(local_device())
    dev.lib()
    wl = make_workload(args.workload)
    inputs = wl.device_facts()
    ctx = None
    if dist:
        from paper_2604_20073_b200.dist import DistContext

        ctx = DistContext()
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev.device())

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    n_out, summary = 0, None
    jit_wait_s = 0.0
    for i in range(args.warmup):  # same conditions as the timed steps
        gc.collect()
        flush_l2(flush)
        barrier()
        n_out, summary = run_step(torch, Engine, parse, wl, inputs, ctx=ctx)
        if i == 0:
            # the per-rule kernels were scheduled when the first engine was
            # built; the timed steps run on them (results are identical on
            # the generic kernels, which cover the first warm-up step)
            t0 = time.perf_counter()
            dev.jit_wait()
            jit_wait_s = time.perf_counter() - t0
    launches0 = dev.lib().srdl_launch_count()
    times = []
    with ClockSampler(local_device(), enabled=not os.environ.get("SRDL_BENCH_NO_CLOCKS")) as clocks:
        for _ in range(args.steps):
            gc.collect()  # release the previous step's engine before timing
            flush_l2(flush)
            barrier()
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            start.record()
            n_out, summary = run_step(torch, Engine, parse, wl, inputs, ctx=ctx)
            end.record()
            end.synchronize()
            times.append(start.elapsed_time(end) / 1e3)
    launches = dev.lib().srdl_launch_count() - launches0
    step_s = sum(times) / len(times)
    # the per-call-family roofline from separate profiled steps: bracketing
    # thousands of library calls with CUDA events costs host time, so the
    # timed steps above run without the hook
    records = []
    dev.PROFILE = records
    prof_times = []
    for _ in range(args.profile_steps):
        gc.collect()
        flush_l2(flush)
        barrier()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
        run_step(torch, Engine, parse, wl, inputs, ctx=ctx)
        end.record()
        end.synchronize()
        prof_times.append(start.elapsed_time(end) / 1e3)
    dev.PROFILE = None
    roofline = family_roofline(records, args.profile_steps, sum(prof_times) / len(prof_times), wl.name)
    if roofline is not None:
        roofline["profiled_steps"] = args.profile_steps
        roofline["profiled_step_ms"] = round(sum(prof_times) / len(prof_times) * 1e3, 2)
    del records

    # end-to-end through the public API with host inputs and output readback
    pinned = {k: v.cpu().pin_memory() for k, v in inputs.items()}
    arity = parse(wl.program).declarations[wl.output]
    out_pinned = torch.empty((arity, n_out), dtype=torch.uint32, pin_memory=True)
    h2d = sum(t.numel() * 4 for t in pinned.values())
    e2e_times = []
    for _ in range(max(1, min(args.steps, 3))):
        gc.collect()
        flush_l2(flush)
        barrier()
        t0 = time.perf_counter()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record()
        run_step(torch, Engine, parse, wl, pinned, host=True, out_pinned=out_pinned, ctx=ctx)
        end.record()
        end.synchronize()
        e2e_times.append(max(start.elapsed_time(end) / 1e3, time.perf_counter() - t0))
    e2e_s = sum(e2e_times) / len(e2e_times)

    tot_out = n_out  # relation sizes are global (the engine all-reduces them)
    if dist:  # max over ranks (host tensor for gloo)
        t = torch.tensor([step_s, e2e_s], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_s, e2e_s = t.tolist()
    result = {
        "metric": "derived tuples/sec (fixpoint)",
        "value": tot_out / step_s,
        "unit": "tuples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_s * 1e3,
        "fixpoint_wall_s": step_s,
        "step_ms_each": [round(t * 1e3, 2) for t in times],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded generators; the same instance at every N)",
        "config": dict(wl.config, derived_tuples=tot_out, idb_tuples=dict(summary.relations),
                       edb_facts=int(sum(v.shape[1] for v in inputs.values())),
                       l2="flushed between steps (512 MiB write)",
                       parallelism=f"hash-partitioned root keys + per-iteration all-to-all x{world}"
                       if world > 1 else "single GPU"),
        "e2e": {
            "value": tot_out / e2e_s,
            "unit": "tuples/s",
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": n_out * 4 * arity,
            "ms_per_step": e2e_s * 1e3,
        },
        "gpu_launches": int(launches / args.steps),
        "per_rule_kernels": dict(dev.jit_stats(), wait_after_first_step_s=round(jit_wait_s, 2)),
        "clocks": clocks.summary(),
        "roofline": roofline,
    }
    return result, wl, inputs, ctx


# --------------------------------------------------------------------------
# CPU side: the C++ oracle port on the host cores


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_solve(wl, facts, keep=None, threads=None):
    """One C++-oracle fixpoint of `facts` (keep: level-0 key sample).
    Returns (output tuples, solve seconds, threads)."""
    from oracle import native
    from oracle.gj import Symbols
    from paper_2604_20073_b200 import parse

    prog = parse(wl.program)
    top = max(int(v.max()) for v in facts.values() if v.size) + 1
    s = native.Solver(prog, {}, Symbols(top), threads=threads, keep_level0=keep)
    for k, v in facts.items():
        s.load_columns(k, v)
    t0 = time.perf_counter()
    s.solve()
    dt = time.perf_counter() - t0
    n = s.size(wl.output)
    th = s.threads
    s.close()
    return n, dt, th


class CpuSampler:
    """Bounded samples of a workload for the CPU port: a subset of level-0
    root keys of the full instance (TC, triangle: an exact restriction of
    the same join/fixpoint) or the full fixpoint of a scaled-down instance of
    the same generator (SG, Andersen, DOOP: a rate proxy), grown until one
    solve takes about `target_s`."""

    def __init__(self, wl, target_s, threads=None):
        self.wl, self.target_s, self.threads = wl, target_s, threads
        self.full = wl.host_facts() if wl.sample_kind == "roots" else None
        if self.full is not None:
            from paper_2604_20073_b200 import parse

            rule = parse(wl.program).rules[0]  # its first atom is an EDB relation keyed by the root
            self.roots = np.unique(self.full[rule.body[0].relation][0])
            np.random.default_rng(0).shuffle(self.roots)
        self.frac = 1.0 / 256
        self._calibrate()

    def _run(self, frac):
        if self.full is not None:
            k = max(1, int(len(self.roots) * frac))
            keep = None if k >= len(self.roots) else np.sort(self.roots[:k])
            n, dt, th = oracle_solve(self.wl, self.full, keep, self.threads)
            what = ("full instance" if keep is None else
                    f"{k}/{len(self.roots)} random root keys of the full instance (exact restriction)")
        else:
            facts = self.wl.host_facts(frac)
            n, dt, th = oracle_solve(self.wl, facts, None, self.threads)
            edb = int(sum(v.shape[1] for v in facts.values()))
            what = (f"full fixpoint of the same generator scaled to {frac:.4g} of the BASELINE size "
                    f"({edb} EDB facts, {n} {self.wl.output} tuples) — a rate proxy")
        return n, dt, th, what

    def _calibrate(self):
        while True:
            n, dt, th, what = self._run(self.frac)
            if dt >= self.target_s / 3 or self.frac >= 1.0:
                break
            self.frac = min(1.0, self.frac * max(2.0, min(8.0, self.target_s / max(dt, 1e-3) / 2)))
        self.last = (n, dt, th, what)

    def step(self):
        self.last = self._run(self.frac)
        return self.last


def cpu_baseline(wl, target_s=15.0):
    s = CpuSampler(wl, target_s)
    n, dt, th, what = s.step()
    return {"value": n / dt, "unit": "tuples/s", "cores": th, "kind": "port",
            "sample": f"{what}: {n} tuples in {dt:.2f} s on {th} threads (C++ restatement of the reference "
                      "generic join + semi-naive loop, oracle/native.py)"}


def parity_check(wl, ctx=None):
    """One more device evaluation (not timed); its output relation and its
    EDB reduced to digests and compared with the oracle's digests of the
    same full-size instance (committed)."""
    import torch

    from oracle.digest import digest
    from paper_2604_20073_b200 import Engine, parse

    with open(DIGESTS) as fh:
        want = json.load(fh).get(wl.name)
    if want is None:
        return {"checked": "no committed oracle digest for this workload", "match": None}
    eng = Engine(parse(wl.program), schedule="stream", dist=ctx)
    for k, v in wl.device_facts().items():
        eng.load_columns(k, v)
    eng.solve()
    rels = {wl.output: want["idb"][wl.output]}
    got = {}
    for rel in rels:
        got[rel] = digest(eng.relation_columns(rel).cpu().numpy())
    edb_ok = all(digest(eng.relation_columns(k).cpu().numpy()) == d for k, d in want["edb"].items())
    torch.cuda.synchronize()
    return {"checked": f"full {wl.output} relation (n, sha256 of sorted columns, fold64) vs the C++ oracle's "
                       "digest of the same full-size instance (tests/golden/baseline_digests.json)",
            "rows": want["idb"][wl.output]["n"], "edb_match": edb_ok,
            "match": bool(edb_ok and all(got[r] == rels[r] for r in rels))}


def bench_reference(args, rank, world):
    """--impl reference: the C++ oracle port of the reference CPU algorithm
    on all host cores. No GPU, no libsrdl: inputs come from the numpy
    generators (the R-MAT graph from the host mirror of the device
    generator)."""
    if rank != 0:
        return None
    wl = make_workload(args.workload)
    per_step = max(2.0, args.ref_budget_s / max(1, args.steps + args.warmup))
    sampler = CpuSampler(wl, per_step)
    for _ in range(args.warmup):
        sampler.step()
    rates, secs = [], []
    for _ in range(args.steps):
        n, dt, th, what = sampler.step()
        rates.append(n / dt)
        secs.append(dt)
    value = sum(rates) / len(rates)
    cfg = dict(wl.config)
    cfg["sample"] = what
    cfg["same_config"] = bool(sampler.full is not None and sampler.frac >= 1.0)
    return {
        "impl": "reference",
        "metric": "derived tuples/sec (fixpoint)",
        "value": value,
        "unit": "tuples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": sum(secs) / len(secs) * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded numpy generators, the same instance as the GPU arm)",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "tuples/s", "cores": th, "kind": "port",
                         "sample": f"{what} per step, {th} threads (C++ restatement of the reference "
                                   "generic join + semi-naive loop, oracle/native.py)"},
        "e2e": {"value": value, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["tc", "triangle", "sg", "andersen", "doop"], default="doop")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=2,
                    help="extra steps, after the timed ones, with every library call bracketed by CUDA events "
                         "(the roofline / call-family breakdown)")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="reference arm: CPU seconds for all warm-up + timed steps together")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    args.profile_steps = max(1, args.profile_steps)

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if args.impl == "reference":
        line = bench_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_device())
        # NCCL over NVLink on a multi-GPU box; SRDL_DIST_BACKEND=gloo runs the
        # same multi-rank path with ranks sharing one GPU (tests of the bench)
        tdist.init_process_group(os.environ.get("SRDL_DIST_BACKEND", "nccl"))
        dist = tdist
    result, wl, inputs, ctx = bench_ours(args, rank, world, dist)
    if not args.no_parity:
        par = parity_check(wl, ctx)
        if rank == 0:
            result["parity"] = par
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(wl)
    if dist:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


if __name__ == "__main__":
    main()
