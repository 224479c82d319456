"""One line per bench JSON file: time, rate, kernel times, parity."""
import json
import sys

for f in sys.argv[1:]:
    lines = open(f).read().strip().splitlines()
    if not lines:
        print(f, "EMPTY")
        continue
    d = json.loads(lines[-1])
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(f"{f}: {d.get('ms_per_step', 0):.1f} ms  {d.get('value', 0):.3g} t/s  e2e {e.get('value', 0):.3g}  "
          f"out {d.get('config', {}).get('derived_tuples')}  kern {r.get('all_kernels_ms_per_step')}  "
          f"frac {r.get('frac')}  launches {d.get('gpu_launches')}  parity {(d.get('parity') or {}).get('match')}  "
          f"cpu {(d.get('cpu_baseline') or {}).get('value')}")
