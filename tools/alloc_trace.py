"""Where does the host wait in torch.empty? Repeated fixpoints of one
workload; per step: wall, new device segments, reserved memory, and the
slowest torch.empty calls (size, host ms, caller).

    python tools/alloc_trace.py --workload doop [--steps 5] [--slow-ms 0.3]
"""
import argparse
import gc
import json
import os
import sys
import time
import traceback

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")  # as bench.py
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_20073_b200 import Engine, parse  # noqa: E402
from paper_2604_20073_b200 import device as dev  # noqa: E402

_empty = torch.empty
SLOW = []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="doop")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--slow-ms", type=float, default=0.3)
    args = ap.parse_args()
    wl = bench.make_workload(args.workload)
    facts = wl.device_facts()

    def traced(*a, **k):
        t0 = time.perf_counter()
        out = _empty(*a, **k)
        ms = (time.perf_counter() - t0) * 1e3
        if ms > args.slow_ms:
            fr = [f for f in traceback.extract_stack(limit=6)[:-1] if "paper_2604" in f.filename]
            where = f"{os.path.basename(fr[-1].filename)}:{fr[-1].lineno}" if fr else "?"
            SLOW.append((ms, out.numel() * out.element_size(), where))
        return out

    def step():
        eng = Engine(parse(wl.program), schedule="stream")
        for k, v in facts.items():
            eng.load_columns(k, v)
        eng.solve()
        torch.cuda.synchronize()

    step()
    dev.jit_wait()
    torch.empty = traced
    for s in range(args.steps):
        gc.collect()
        SLOW.clear()
        m0 = torch.cuda.memory_stats()
        t0 = time.perf_counter()
        step()
        wall = (time.perf_counter() - t0) * 1e3
        m1 = torch.cuda.memory_stats()
        by = {}
        for ms, nbytes, where in SLOW:
            n, t, b = by.get(where, (0, 0.0, 0))
            by[where] = (n + 1, t + ms, max(b, nbytes))
        top = sorted(by.items(), key=lambda kv: -kv[1][1])[:10]
        print(json.dumps({"step": s, "wall_ms": round(wall, 1),
                          "device_allocs": m1["num_device_alloc"] - m0["num_device_alloc"],
                          "device_frees": m1["num_device_free"] - m0["num_device_free"],
                          "reserved_gb": round(m1["reserved_bytes.all.current"] / 1e9, 1),
                          "slow_empty_ms": round(sum(x[0] for x in SLOW), 1),
                          "slow_empty_by_site": {k: [n, round(t, 1), b] for k, (n, t, b) in top}}), flush=True)
    torch.empty = _empty


if __name__ == "__main__":
    main()
