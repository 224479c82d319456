"""Host-side profile of one fixpoint (cProfile), after warm-up and with the
per-rule kernels built: where the Python driver spends its time per
iteration.

    python tools/host_profile.py --workload doop [--top 40]
"""
import os

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")  # as bench.py

import argparse  # noqa: E402
import gc
import cProfile
import io
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_20073_b200 import Engine, parse  # noqa: E402
from paper_2604_20073_b200 import device as dev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="doop")
    ap.add_argument("--top", type=int, default=45)
    args = ap.parse_args()
    wl = bench.make_workload(args.workload)
    facts = wl.device_facts()

    def step():
        gc.collect()  # as bench.py: the previous engine's memory back to the allocator first
        eng = Engine(parse(wl.program), schedule="stream")
        for k, v in facts.items():
            eng.load_columns(k, v)
        eng.solve()
        torch.cuda.synchronize()

    step()
    dev.jit_wait()
    for _ in range(4):  # steady state: the allocator's cache and the pools have grown
        step()
    keys = ("num_alloc_retries", "num_sync_all_streams", "num_device_alloc", "num_device_free",
            "allocation.all.allocated")
    m0 = torch.cuda.memory_stats()
    t0 = time.perf_counter()
    step()
    plain = time.perf_counter() - t0
    m1 = torch.cuda.memory_stats()
    print("allocator over one fixpoint:", {k: m1.get(k, 0) - m0.get(k, 0) for k in keys},
          "reserved GB", round(m1.get("reserved_bytes.all.current", 0) / 1e9, 1),
          "alloc conf", os.environ.get("PYTORCH_CUDA_ALLOC_CONF"))
    prof = cProfile.Profile()
    prof.enable()
    step()
    prof.disable()
    out = io.StringIO()
    pstats.Stats(prof, stream=out).sort_stats("tottime").print_stats(args.top)
    print(f"fixpoint wall {plain * 1e3:.1f} ms (unprofiled)")
    print(out.getvalue())
    out = io.StringIO()
    pstats.Stats(prof, stream=out).sort_stats("cumulative").print_stats(args.top)
    print(out.getvalue())


if __name__ == "__main__":
    main()
