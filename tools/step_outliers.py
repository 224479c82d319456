"""Diagnose slow fixpoint steps: repeated triangle solves with per-phase
host timings (synchronised), printed per step.
    python tools/step_outliers.py [--reps N]"""
import argparse
import gc
import json
import os
import sys
import time

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_20073_b200 import Engine, Stats, parse, suites  # noqa: E402
from paper_2604_20073_b200 import device as dev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=12)
    ap.add_argument("--stats", action="store_true")
    ap.add_argument("--profile", action="store_true", help="CUPTI trace of slow prepare phases")
    args = ap.parse_args()
    raw = dev.gen_rmat(20, 16_000_000, seed=1).view(torch.int32)
    raw = raw[:, raw[0] != raw[1]].contiguous().view(torch.uint32)
    e = dev.sort_dedup(raw, 20)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for rep in range(args.reps):
        gc.collect()
        flush.add_(1)
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        stats = Stats(enabled=args.stats)
        eng = Engine(parse(suites.TRIANGLE_PROGRAM), schedule="stream", stats=stats)
        for r in ("R", "S", "T"):
            eng.load_columns(r, e)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        prof = None
        if args.profile:
            prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                                      torch.profiler.ProfilerActivity.CUDA])
            prof.__enter__()
        eng.prepare_inputs()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        if prof is not None:
            prof.__exit__(None, None, None)
            if (t[-1] - t[-2]) * 1e3 > 60:
                rows = {}
                for ev in prof.events():
                    if ev.device_type == torch.autograd.DeviceType.CPU:
                        n, tt = rows.get(ev.name, (0, 0.0))
                        rows[ev.name] = (n + 1, tt + ev.cpu_time_total / 1e3)
                top = sorted(rows.items(), key=lambda kv: -kv[1][1])[:12]
                print(json.dumps({"rep": rep, "slow_prepare_cpu_ms": {k: [n, round(v, 1)] for k, (n, v) in top}}),
                      flush=True)
        eng.solve()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        del eng
        gc.collect()
        torch.cuda.synchronize(); t.append(time.perf_counter())
        ms = [round((b - a) * 1e3, 1) for a, b in zip(t, t[1:])]
        mem = torch.cuda.memory_stats()
        print(json.dumps({"rep": rep, "load_ms": ms[0], "prepare_ms": ms[1], "solve_ms": ms[2], "free_ms": ms[3],
                          "phases": {k: round(v / 1e3, 1) for k, v in stats.phase_totals().items()},
                          "device_allocs": mem.get("num_device_alloc"), "reserved_gb": round(mem.get("reserved_bytes.all.current", 0) / 1e9, 1)}),
              flush=True)


if __name__ == "__main__":
    main()
