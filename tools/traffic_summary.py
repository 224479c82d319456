"""DRAM bytes per library call of a bench family, from an ncu log of the same
bench command (`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum
--csv --log-file LOG.csv python bench.py --workload W --steps S --warmup 3
--no-parity --no-cpu-baseline`), written into profiles/traffic.json, which
bench.py copies into `roofline.traffic`:

    python tools/traffic_summary.py LOG.csv WORKLOAD BENCH.json

Kernels are attributed to the library call family that launches them
(csrc/: the per-rule kernels and the generic WCOJ instances -> wcoj_count /
wcoj_materialize, gather_kernel -> wcoj_gather, the sort / unique /
anti-join / compaction kernels -> compute_delta, merge kernels -> merge).
Bytes per call = the family's bytes over every profiled launch / the
number of calls (the bench's per-step call count x profiled fixpoints).
"""
import collections
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

FAMILY = [
    ("gather_kernel", "wcoj_gather"),
    ("wcoj_kernel<1", "wcoj_materialize"),
    ("srdl_jit_wcoj", "wcoj_count"),
    ("wcoj_kernel", "wcoj_count"),
    ("mp_merge_rows", "merge"),
    ("mp_splits_rows", "merge"),
]
DELTA = ("check_sorted", "pack_keys", "radix_hist_all", "onesweep_pass", "radix_digit_starts", "flag_keys",
         "mp_splits_keys", "mp_diff_keys", "bs_diff_keys", "scatter_unpack", "copy_if_unsorted", "iota_u32",
         "gather_cols", "flag_rows", "scatter_rows", "mp_diff_rows", "bs_diff_rows")


def family_of(kernel: str):
    for key, fam in FAMILY:
        if key in kernel:
            return fam
    if any(k in kernel for k in DELTA):
        return "compute_delta"
    return None


def main():
    path, workload, bench_path = sys.argv[1], sys.argv[2], sys.argv[3]
    bench = json.loads(open(bench_path).read().strip().splitlines()[-1])
    # fixpoints the bench ran: warm-up, timed, profiled, e2e (min(steps, 3)) and parity
    rl0 = bench.get("roofline") or {}
    fixpoints = (bench["warmup"] + bench["steps"] + rl0.get("profiled_steps", 0) + max(1, min(bench["steps"], 3))
                 + (1 if "parity" in bench else 0))
    rl = bench.get("roofline") or {}
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, ni, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    idx = hdr.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
        per[r[idx]][r[ni]] = v
        names[r[idx]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for i, m in per.items():
        fam = family_of(names[i])
        if fam is None:
            continue
        agg[fam][0] += 1
        agg[fam][1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    d = json.load(open(out_path)) if os.path.exists(out_path) else {}
    rec = {}
    for fam, (launches, b) in agg.items():
        calls = None
        if rl.get("kernel") == fam:
            calls = rl["launches_per_step"] * fixpoints  # per-step calls of the profiled steps
        rec[fam] = round(b / calls) if calls else None
        rec[fam + "_kernel_launches"] = launches
        rec[fam + "_bytes_total"] = round(b)
    rec["fixpoints_profiled"] = fixpoints
    d[workload] = rec
    json.dump(d, open(out_path, "w"), indent=1, sort_keys=True)
    print(workload, rec)


if __name__ == "__main__":
    main()
