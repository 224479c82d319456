"""Diagnostics: per-phase device times of one fixpoint (Stats enabled).

    python tools/phase_report.py --workload triangle|sg|tc|andersen [--statements N]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2604_20073_b200 import Engine, Stats, parse, suites
from paper_2604_20073_b200 import device as dev


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="triangle")
    ap.add_argument("--statements", type=int, default=1_000_000)
    ap.add_argument("--methods", type=int, default=6_900_000, help="doop: methods (~14.5 facts each)")
    ap.add_argument("--schedule", default="stream")
    ap.add_argument("--kernels", action="store_true", help="CUPTI per-kernel totals of the last run")
    ap.add_argument("--rules", type=int, default=0, help="print the N costliest (rule, phase) pairs")
    args = ap.parse_args()
    if args.workload == "triangle":
        raw = dev.gen_rmat(20, 16_000_000, seed=1).view(torch.int32)
        raw = raw[:, raw[0] != raw[1]].contiguous().view(torch.uint32)
        e = dev.sort_dedup(raw, 20)
        facts = {"R": e, "S": e, "T": e}
        program, out = suites.TRIANGLE_PROGRAM, "Triangle"
    else:
        gen = {"sg": lambda: suites.sg_layered(),
               "tc": lambda: suites.tc_random(),
               "andersen": lambda: suites.andersen_modular(args.statements, seed=1),
               "doop": lambda: suites.doop_modular(args.methods, seed=1)}[args.workload]
        facts = {k: torch.from_numpy(v).cuda() for k, v in gen().items()}
        program, out = suites.BASELINE_PROGRAMS[args.workload]
    for rep in range(2):
        stats = Stats(enabled=not args.kernels)
        eng = Engine(parse(program), schedule=args.schedule, stats=stats)
        dev.jit_wait()  # the per-rule kernels of the program (scheduled by the Engine) are built
        for k, v in facts.items():
            eng.load_columns(k, v)
        prof = None
        if args.kernels and rep == 1:
            prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
            prof.__enter__()
        t0 = time.perf_counter()
        summ = eng.solve()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if prof is not None:
            prof.__exit__(None, None, None)
            rows = {}
            for ev in prof.events():
                if ev.device_type == torch.autograd.DeviceType.CUDA:
                    name = ev.name.split("(")[0][:60]
                    n, t = rows.get(name, (0, 0.0))
                    rows[name] = (n + 1, t + ev.device_time_total / 1e3)
            top = sorted(rows.items(), key=lambda kv: -kv[1][1])[:14]
            print(json.dumps({"kernels_ms": {k: [n, round(t, 2)] for k, (n, t) in top}}), flush=True)
            # device busy time = union of kernel intervals (streams overlap)
            iv = sorted((ev.time_range.start, ev.time_range.end) for ev in prof.events()
                        if ev.device_type == torch.autograd.DeviceType.CUDA)
            busy, cur_s, cur_e = 0.0, None, None
            for a, b in iv:
                if cur_e is None or a > cur_e:
                    if cur_e is not None:
                        busy += cur_e - cur_s
                    cur_s, cur_e = a, b
                else:
                    cur_e = max(cur_e, b)
            if cur_e is not None:
                busy += cur_e - cur_s
            span = (iv[-1][1] - iv[0][0]) if iv else 0
            print(json.dumps({"device_busy_ms": round(busy / 1e3, 2), "device_span_ms": round(span / 1e3, 2),
                              "kernels": len(iv)}), flush=True)
        totals = {k: round(v / 1e3, 2) for k, v in sorted(stats.phase_totals().items(), key=lambda x: -x[1])}
        if stats.enabled and args.rules:
            per = {}
            for r in stats.records:
                key = f"{r['rule']}:{r['phase']}"
                t, n = per.get(key, (0, 0))
                per[key] = (t + r["micros"], n + r["tuples"])
            top = sorted(per.items(), key=lambda kv: -kv[1][0])[:args.rules]
            print(json.dumps({"top_rule_phases_ms": {k: [round(t / 1e3, 2), n] for k, (t, n) in top}}),
                  flush=True)
        print(json.dumps({"rep": rep, "wall_s": round(wall, 3), "out": summ.relations[out],
                          "iterations": [s.iterations for s in summ.strata],
                          "phase_ms": totals}), flush=True)


if __name__ == "__main__":
    main()
