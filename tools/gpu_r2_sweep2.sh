#!/bin/bash
O=gpurun_out
timeout 600 python tools/phase_report.py --workload andersen --statements 10000000 --kernels > $O/kern_andersen.log 2>&1
for d in "-DSRDL_MIN_BLOCKS=6" "-DSRDL_MIN_BLOCKS=7" "-DSRDL_MIN_BLOCKS=5" ""; do
  tag=$(echo "x$d" | tr -c 'a-zA-Z0-9\n' '_')
  for w in triangle doop; do
    SRDL_JIT_DEFINES="$d" timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $O/sweep_${w}_$tag.json 2>&1
  done
done
exit 0
