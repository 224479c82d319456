#!/bin/bash
# final round-2 check: the full -m gpu suite, smoke, stream-pool A/B on DOOP
O=gpurun_out
E=$O/fin
mkdir -p $E
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --durations 10 > $E/pytest_gpu.log 2>&1; echo "rc=$?" >> $E/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo "rc=$?" >> $E/smoke.log
for ns in 16 12; do
  SRDL_STREAMS=$ns timeout 900 python bench.py --workload doop --steps 5 --warmup 3 --no-cpu-baseline --no-parity > $E/bench_doop_s$ns.json 2> $E/bench_doop_s$ns.err
done
exit 0
