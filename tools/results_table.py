"""Markdown results table from bench.py JSON lines (one file per config):
    python tools/results_table.py DIR [DIR_REF]
DIR holds bench_<workload>.json (our arm), DIR_REF (default DIR) ref_<workload>.json."""
import json
import os
import sys

ORDER = [("tc", "configs[0] TC"), ("triangle", "configs[1] triangle"), ("sg", "configs[2] SG"),
         ("andersen", "configs[3] Andersen"), ("doop", "configs[4] DOOP (default)")]


def last_json(path):
    if not os.path.exists(path):
        return None
    lines = [ln for ln in open(path).read().strip().splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def main():
    d = sys.argv[1]
    dref = sys.argv[2] if len(sys.argv) > 2 else d
    print("| config | fixpoint ms | derived tuples/s | e2e tuples/s (ms) | dominant family: ms/step, HBM frac "
          "| issue frac | CPU baseline tuples/s (cores) | parity |")
    print("|---|---|---|---|---|---|---|---|")
    for w, label in ORDER:
        b = last_json(os.path.join(d, f"bench_{w}.json"))
        if b is None:
            continue
        r = b.get("roofline") or {}
        fam = r.get("kernel")
        fam_ms = (r.get("families_ms_per_step") or {}).get(fam)
        iss = r.get("issue_roofline") or {}
        cpu = b.get("cpu_baseline") or {}
        par = b.get("parity") or {}
        e2e = b.get("e2e") or {}
        print(f"| {label} | {b['ms_per_step']:.1f} | {b['value'] / 1e9:.3f} G | {e2e.get('value', 0) / 1e9:.3f} G "
              f"({e2e.get('ms_per_step', 0):.1f}) | {fam}: {fam_ms} ms, {r.get('frac')} | "
              f"{iss.get('frac', '—')} | {cpu.get('value', 0) / 1e6:.2f} M ({cpu.get('cores')}) | "
              f"{'match' if par.get('match') else par.get('match')} ({par.get('rows')} rows) |")
    refs = [(w, last_json(os.path.join(dref, f"ref_{w}.json"))) for w, _ in ORDER]
    refs = [(w, x) for w, x in refs if x]
    if refs:
        print()
        print("| reference arm (`--impl reference`) | tuples/s | ms per step | cores | sample |")
        print("|---|---|---|---|---|")
        for w, x in refs:
            c = x.get("cpu_baseline") or {}
            print(f"| {w} | {x['value'] / 1e6:.2f} M | {x['ms_per_step']:.0f} | {c.get('cores')} | "
                  f"{c.get('sample', '')[:140]} |")


if __name__ == "__main__":
    main()
