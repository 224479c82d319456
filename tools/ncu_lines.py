"""Per-CUDA-source-line hot spots of an ncu report (needs -lineinfo):
    python tools/ncu_lines.py REPORT.ncu-rep [kernel-regex] [launch-index] [top]
Prints warp-stall samples and executed warp instructions per source line."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else "."
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    path, rows = "", []
    hdr = None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            path = rec[1].rsplit("/", 1)[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or not rec[0].isdigit() or rec[2] != "-":
            continue
        d = dict(zip(hdr[2:], rec[2:]))
        samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
        rows.append((samples, inst, f"{path}:{rec[0]}", rec[1].strip()[:90]))
    tot_s = sum(r[0] for r in rows) or 1
    tot_i = sum(r[1] for r in rows) or 1
    print(f"total samples {tot_s}  warp instructions {tot_i:.3e}")
    for s, i, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {loc:16s} {src}")


if __name__ == "__main__":
    main()
