"""Average DRAM bytes per launch of the count / materialize WCOJ kernels from
an `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv` log, written into profiles/wcoj_traffic.json under the workload name:
    python tools/traffic_summary.py LOG.csv WORKLOAD"""
import collections
import csv
import json
import os
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    path, workload = sys.argv[1], sys.argv[2]
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
        k = names[i]
        if "gather_kernel" in k:
            name = "wcoj_gather"
        elif "wcoj_kernel<1" in k or "wcoj_kernel<true" in k:
            name = "wcoj_materialize"
        else:  # wcoj_kernel<0 (count) and <2 (speculative count)
            name = "wcoj_count"
        agg[name][0] += 1
        agg[name][1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            "wcoj_traffic.json")
    d = json.load(open(out_path)) if os.path.exists(out_path) else {}
    d[workload] = {k: round(b / n) for k, (n, b) in agg.items()}
    d[workload]["launches_profiled"] = {k: n for k, (n, _) in agg.items()}
    json.dump(d, open(out_path, "w"), indent=1, sort_keys=True)
    print(workload, d[workload])


if __name__ == "__main__":
    main()
