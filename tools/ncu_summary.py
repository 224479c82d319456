"""Key counters of an `ncu --set full` report, one block per profiled launch:
    python tools/ncu_summary.py REPORT.ncu-rep [--json OUT.json]
--json also writes, per launch, the figures bench.py's issue-rate roofline
reads (profiles/r02/issue.json): duration, warp instructions, issue-active."""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__cycles_active.avg", "sm__cycles_active.max", "sm__cycles_active.min",
]
STALL = "smsp__average_warp_latency_issue_stalled_"


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))

        def num(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None

        dur = num("gpu__time_duration.sum")
        scale = {"ms": 1.0, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "nsecond": 1e-6}.get(
            u.get("gpu__time_duration.sum", "ms"), 1.0)
        launches.append({"kernel": d.get("Kernel Name", "?")[:90],
                         "duration_ms": dur * scale if dur is not None else None,
                         "inst_executed": num("smsp__inst_executed.sum"),
                         "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                         "sm_cycles_active_avg": num("sm__cycles_active.avg")})
        print(f"== {d.get('Kernel Name', '?')[:90]}")
        for k in WANT:
            if k in d:
                print(f"  {k:62s} {d[k]:>18s} {u.get(k, '')}")
        # SM load balance: active-cycle spread across SMs
        try:
            mx, mn, av = (float(d[f"sm__cycles_active.{s}"].replace(",", "")) for s in ("max", "min", "avg"))
            print(f"  SM balance: min/avg {mn / av:.3f}, max/avg {mx / av:.3f}")
        except (KeyError, ValueError, ZeroDivisionError):
            pass
        stalls = []
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and k.endswith("_not_issued") is False:
                try:
                    stalls.append((float(d[k].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        if stalls:
            print("  warp-stall samples: " + ", ".join(f"{n} {100 * s / tot:.1f}%" for s, n in sorted(stalls, reverse=True)[:8]))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(launches, fh, indent=1)


if __name__ == "__main__":
    main()
